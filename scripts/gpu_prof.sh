#!/bin/bash
# ncu capture of the force kernel + launch list + FP64 microbenchmark
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
./scripts/fp64_peak > gpurun_out/fp64_peak.json 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv >> gpurun_out/fp64_peak.json
CFG=${CFG:-C2}
timeout 300 python scripts/prof_force.py $CFG 4 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python scripts/prof_force.py $CFG 4 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 2 -c 1 -o gpurun_out/prof_force_$CFG python scripts/prof_force.py $CFG 4 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
