#!/bin/bash
# full GPU test suite on all visible GPUs + ring benches of both workloads
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-final4}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu_all.log 2>&1; echo rc=$? >> $O/pytest_gpu_all.log
for n in 2 4; do [ $n -le $N ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29616 bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4_n$n.log 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29617 bench.py --gpus $n --config G1 --workers 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_g1_n${n}_w2.log 2>&1
done
timeout 600 python bench.py --config G1 --steps 20 --warmup 3 > $O/bench_g1_n1.log 2>&1
