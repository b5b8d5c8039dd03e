#!/bin/bash
# round-end style measurement on 1 GPU: bench line, ncu launch list of the same command,
# one ncu --set full capture of the force kernel (fused C4).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_n1_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench_n1.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch.log
timeout 300 python scripts/prof_force.py C4 2 > gpurun_out/prof_c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 1 -c 1 -o gpurun_out/prof_force_C4 python scripts/prof_force.py C4 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_c4.log
