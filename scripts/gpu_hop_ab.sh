#!/bin/bash
# ring tests with the default hop, then bench A/B of the peer hop (copy engine vs SM stores)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_ring.py -q -x -m gpu > gpurun_out/hop_pytest_$N.log 2>&1; echo "rc=$?" >> gpurun_out/hop_pytest_$N.log
: > gpurun_out/hop_ab_$N.jsonl
for cfg in ${CFGS:-C4 C3}; do for hop in ce sm; do
DSEA_PEER_HOP=$hop timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 5 --warmup 3 --equil 8 --config $cfg --no-e2e > gpurun_out/hop_${cfg}_$hop.log 2>&1
echo "{\"hop\": \"$hop\", \"cfg\": \"$cfg\", \"line\": $(grep '^{' gpurun_out/hop_${cfg}_$hop.log | tail -1 || echo null)}" >> gpurun_out/hop_ab_$N.jsonl
done; done
