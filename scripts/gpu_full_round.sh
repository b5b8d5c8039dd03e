#!/bin/bash
# one gpurun call: GPU tests, smoke, default bench (both arms), G1 bench, ncu launch list + full
# captures of the force kernel (C4 after 100 melt steps) and the gather kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-r01b}; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -rf ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo "rc=$?" >> $O/bench_n1.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
timeout 600 python bench.py --config G1 --steps 20 --warmup 3 > $O/bench_g1_n1.log 2>&1; echo "rc=$?" >> $O/bench_g1_n1.log
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_n1.csv \
  python bench.py --steps 3 --warmup 3 --equil 20 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 100 -c 1 -o $O/prof_force_C4 \
  python scripts/prof_force.py C4 104 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_gather -s 2 -c 1 -o $O/prof_gather_C4 \
  python scripts/prof_force.py C4 4 > $O/ncu_gather.log 2>&1; echo "rc=$?" >> $O/ncu_gather.log
fi
