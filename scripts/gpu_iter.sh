#!/bin/bash
# iteration call: GPU tests (fast subset), perf probe, ncu of the force kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-C2}
timeout 900 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-not nve}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/prof_force.py C2 6 > gpurun_out/prof_plain.log 2>&1
timeout 300 python scripts/prof_force.py C4 3 >> gpurun_out/prof_plain.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
timeout 300 python scripts/prof_force.py $CFG 4 > gpurun_out/prof_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 2 -c 1 -o gpurun_out/prof_force_$CFG python scripts/prof_force.py $CFG 4 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
