cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/ctr4; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ring.py -q -x > $O/pytest_ring.log 2>&1; echo rc=$? >> $O/pytest_ring.log
for rep in 1 2; do for ctr in 1 0; do for n in 2 4; do
  echo -n "ctr=$ctr n=$n " >> $O/sweep.log
  DSEA_RING_COUNTERS=$ctr timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29615 bench.py --gpus $n --warmup 3 --equil 8 --no-e2e --no-cpu-baseline --steps 10 2>&1 | grep "^{" >> $O/sweep.log
done; done; done
