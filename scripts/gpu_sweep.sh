#!/bin/bash
# throughput of every BASELINE configuration on the GPUs of this box
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l); o=gpurun_out/sweep_$N.jsonl; : > $o
for cfg in ${CFGS:-C2 C3 C4 C5a C5b C5c C5d C5e C5f}; do
  if [ "$N" = "1" ]; then
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 2 --equil 20 --no-e2e --no-cpu-baseline 2>/dev/null | grep metric >> $o
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) bench.py --gpus $N --config $cfg --steps 5 --warmup 2 --equil 20 --no-e2e 2>/dev/null | grep metric >> $o
  fi
done
