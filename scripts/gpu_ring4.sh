#!/bin/bash
# 2/4-GPU ring: tests, C4 bench at N = 1, 2, 4, per-rank timelines at N = 4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-ring4}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > $O/topo.txt 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1800 python -m pytest tests/test_gpu_ring.py tests/test_gpu_ring_shared.py -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_ring.log 2>&1; echo rc=$? >> $O/pytest_ring.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_n1.log 2>&1
for n in 2 4; do [ $n -le $N ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_n$n.log 2>&1
done
if [ -n "$TIMELINE" ]; then
  DSEA_TIMELINE=$O/tl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29619 bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_tl.log 2>&1
fi
