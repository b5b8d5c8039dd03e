#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
if [ "$N" = "1" ]; then
  timeout 900 python bench.py > gpurun_out/bench_full_1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full_1.log
  timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_1.log
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $N > gpurun_out/bench_full_$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full_$N.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus $N --impl reference > gpurun_out/bench_ref_$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$N.log
fi
