#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; out=gpurun_out/ring_debug.log; : > $out
run() { echo "=== $*" >> $out; DSEA_RING_DEBUG=1 NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,P2P timeout -s TERM 60 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) tests/ring_worker.py --out /tmp/o.npz "$@" >> $out 2>&1; echo "rc=$?" >> $out; }
run --config P8 --steps 2
