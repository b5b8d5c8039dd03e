#!/bin/bash
# 2 GPUs: topology + peer copy bandwidth, C4 / G1 rings of 2 with A/B switches
# (full pools, register-column stencil), the NCCL ring tests of 2 GPUs, e2e at N = 1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-d2}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
python - > $O/p2p.txt 2>&1 <<'PY'
import torch, time
a = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0"); b = torch.empty_like(a, device="cuda:1")
print("can_access_peer", torch.cuda.can_device_access_peer(0, 1))
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
t = time.perf_counter()
for _ in range(20): b.copy_(a)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
print("p2p GB/s", 20 * a.numel() / (time.perf_counter() - t) / 1e9)
PY
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29651 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/c4_n2.log 2>&1
DSEA_POOLS=0 timeout 600 $R --master-port 29652 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_n2_full.log 2>&1
timeout 600 $R --master-port 29653 bench.py --gpus 2 --config G1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/g1_n2.log 2>&1
DSEA_FTCS=col timeout 600 $R --master-port 29654 bench.py --gpus 2 --config G1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/g1_n2_col.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/c4_n1.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ring.py -q --timeout 300 -rf -k "nccl and (2-)" > $O/pytest_nccl2.log 2>&1; echo rc=$? >> $O/pytest_nccl2.log
