#!/bin/bash
# ring throughput vs slices per stage (B) and super-cycles per timed call (K)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
out=gpurun_out/ring_sweep_$N.txt
for cfg in ${CFGS:-C4}; do for bk in ${BLOCKS:-0}; do for k in ${KS:-10}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps $k --warmup 3 --equil 8 --config $cfg --no-e2e --block $bk > gpurun_out/rs.log 2>&1
grep '^{' gpurun_out/rs.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$cfg N=$N B=$bk K=$k', '%.3e'%d['value'], 'ms/step %.2f'%d['ms_per_step'], 'force/launch %.3f'%r['force_ms_per_launch'], 'share %.2f'%r['force_share_of_step'], 'launches', d['gpu_launches'])" >> $out 2>&1 || tail -3 gpurun_out/rs.log >> $out
done; done; done
