#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ring.py -q > gpurun_out/pytest_ring_$N.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ring_$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 5 --warmup 2 --equil 8 > gpurun_out/bench_ring_$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ring_$N.log
