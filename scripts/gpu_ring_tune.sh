#!/bin/bash
# ring tuning sweep on all visible GPUs: block sizes, timed-cycle counts, one timeline
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=$(nvidia-smi -L | wc -l); O=gpurun_out/${TAG:-tune}; mkdir -p $O
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --warmup 3 --equil 8 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep '^{' ; }
for blk in ${BLOCKS:-0}; do for st in ${STEPS:-10}; do
  echo -n "block=$blk steps=$st " >> $O/sweep.log; run --config ${CFG:-C4} --block $blk --steps $st >> $O/sweep.log
done; done
if [ -n "$TIMELINE" ]; then DSEA_TIMELINE=$O/tl run --config ${CFG:-C4} --steps 10 > $O/tl_bench.log; fi
