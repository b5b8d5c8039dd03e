#!/bin/bash
# 4 GPUs: the multi-GPU ring tests (MD + stencil, bounded per test), C4 and G1 benches
# at N = 1, 2, 4, then the 1e9-atom ring (scripts/run_big.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-rb}; mkdir -p $O
N=$(nvidia-smi -L | wc -l)
if [ -z "$NO_TESTS" ]; then
timeout 2400 python -m pytest tests/test_gpu_ring.py tests/test_gpu_ring_shared.py tests/test_gpu_grid.py -k "ring" -q --timeout 400 -rf \
  ${DESELECT_NCCL_PLATEAU:+--deselect "tests/test_gpu_ring.py::test_ring_bitwise_equals_single_gpu[4-P8-12-2-1-3-nccl-False]" --deselect "tests/test_gpu_ring.py::test_ring_bitwise_equals_single_gpu[4-P8-12-1-1-5-nccl-True]"} \
  ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_ring.log 2>&1; echo "rc=$?" >> $O/pytest_ring.log
fi
if [ -z "$NO_BENCH" ]; then
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_c4_n1.log 2>&1
timeout 600 python bench.py --config G1 --steps 20 --warmup 3 > $O/bench_g1_n1.log 2>&1
for n in 2 4; do [ $n -le $N ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 > $O/bench_c4_n$n.log 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --config G1 --steps 10 --warmup 3 > $O/bench_g1_n$n.log 2>&1
done
fi
if [ -z "$NO_BIG" ]; then
nvidia-smi --query-gpu=index,memory.total --format=csv > $O/gpus.txt 2>&1
timeout ${BIGLIM:-1500} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29641 \
  scripts/run_big.py --ni ${NI:-630} --cycles ${CYCLES:-3} --out $O/big_run.json > $O/big_run.log 2>&1; echo "big rc=$?" >> $O/big_run.log
fi
