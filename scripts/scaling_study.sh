#!/bin/bash
# NEXT-2: ring throughput vs N_GPU, workers per GPU W and slices N_S,
# to show Eq. (1): linear scaling up to N_max = N_S / (2 + 2W), then a
# plateau.  Runs on one box with up to $(nvidia-smi -L | wc -l) GPUs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
NMAX=$(nvidia-smi -L | wc -l)
out=gpurun_out/scaling_study.jsonl; : > $out
for cfg in ${CFGS:-S12 S24}; do for w in ${WS:-1 2}; do for bk in ${BLOCKS:-1 0}; do for n in 1 2 3 4; do
  [ $n -gt $NMAX ] && continue
  if [ $n -eq 1 ]; then cmd="python bench.py --staged"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29613 bench.py"; fi
  timeout 600 $cmd --gpus $n --steps ${K:-10} --warmup 3 --equil 8 --config $cfg --workers $w --block $bk --no-e2e --no-cpu-baseline --no-steady > gpurun_out/ss.log 2>&1
  line=$(grep '^{' gpurun_out/ss.log | tail -1)
  echo "{\"cfg\": \"$cfg\", \"W\": $w, \"B\": $bk, \"N\": $n, \"line\": ${line:-null}}" >> $out
done; done; done; done
