#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for cfg in C4 C3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 5 --warmup 3 --equil 8 --config $cfg --no-e2e > gpurun_out/bench_ring_${N}_$cfg.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ring_${N}_$cfg.log
done
