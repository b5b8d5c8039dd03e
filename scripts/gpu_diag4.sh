#!/bin/bash
# 4-GPU box diagnosis of the ring hop: peer copy bandwidth of every pair (plain and
# through a CUDA IPC mapping in another process), C4 ring of 2 on GPUs 0,1 and 2,3,
# without PDL, and a per-rank timeline
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-d4}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
nvidia-smi -q | grep -i -A3 "fabric\|nvlink" | head -40 > $O/nvlink.txt 2>&1
nvidia-smi nvlink -s > $O/nvlink_status.txt 2>&1
python - > $O/p2p.txt 2>&1 <<'PY'
import torch, time
n = torch.cuda.device_count()
for i in range(n):
    for j in range(n):
        if i == j: continue
        a = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{i}"); b = torch.empty_like(a, device=f"cuda:{j}")
        for _ in range(3): b.copy_(a)
        torch.cuda.synchronize(i); torch.cuda.synchronize(j)
        t = time.perf_counter()
        for _ in range(10): b.copy_(a)
        torch.cuda.synchronize(i); torch.cuda.synchronize(j)
        print(i, j, "p2p GB/s %.1f" % (10 * a.numel() / (time.perf_counter() - t) / 1e9), torch.cuda.can_device_access_peer(i, j), flush=True)
PY
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29661 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_n2_gpu01.log 2>&1
CUDA_VISIBLE_DEVICES=2,3 timeout 600 $R --master-port 29662 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_n2_gpu23.log 2>&1
DSEA_PDL=0 timeout 600 $R --master-port 29663 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_n2_nopdl.log 2>&1
DSEA_TIMELINE=$O/tl timeout 600 $R --master-port 29664 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $O/c4_n2_tl.log 2>&1
timeout 600 $R --master-port 29665 bench.py --gpus 2 --config G1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/g1_n2.log 2>&1
