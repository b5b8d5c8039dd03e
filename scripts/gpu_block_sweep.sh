#!/bin/bash
# block-size sweep of the C4 ring at 2 and 4 GPUs (bench.py --block), two repetitions
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-bsweep}; mkdir -p $O
SPECS=${SPECS:-2:0 2:10 2:14 2:18 4:0 4:9 4:10 4:12}
for rep in 1 2; do
for spec in $SPECS; do
  n=${spec%%:*}; blk=${spec#*:}
  echo -n "n=$n block=$blk " >> $O/sweep.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $n --warmup 3 --equil 8 --no-e2e --no-cpu-baseline --steps 10 --block $blk 2>&1 | grep "^{" >> $O/sweep.log
done; done
