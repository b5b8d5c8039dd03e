#!/bin/bash
# NEXT-3 on a 4-GPU box: the GPU suite (single-GPU parity + rings), then the 1e9-atom
# ring (scripts/run_big.py) with per-GPU memory, throughput and sampled force parity
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-big}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=index,memory.total --format=csv > $O/gpus.txt 2>&1
free -g > $O/host_mem.txt 2>&1; nproc >> $O/host_mem.txt
if [ -z "$NO_TESTS" ]; then
timeout ${TLIM:-2400} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout ${BIGLIM:-1500} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29631 \
  scripts/run_big.py --ni ${NI:-630} --cycles ${CYCLES:-3} --out $O/big_run.json > $O/big_run.log 2>&1; echo "big rc=$?" >> $O/big_run.log
