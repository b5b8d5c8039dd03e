#!/bin/bash
# stencil workload on all visible GPUs: GPU tests, bench G1 at 1/2/4 GPUs, ncu of k_ftcs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-grid}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_grid.py -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 600 python bench.py --config G1 --steps 20 --warmup 3 > $O/bench_g1_n1.log 2>&1
for w in ${WORKERS:-1 4}; do
for n in 2 4; do [ $n -le $N ] && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus $n --config G1 --steps 10 --warmup 3 --workers $w --no-cpu-baseline > $O/bench_g1_n${n}_w$w.log 2>&1; done; done
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ftcs -s 2 -c 1 -o $O/prof_ftcs python bench.py --config G1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
fi
