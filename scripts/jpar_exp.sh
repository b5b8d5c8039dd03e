#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; o=gpurun_out/jpar_exp.log; : > $o
timeout 900 python -m pytest tests -m gpu -q -x -k "not nve and not ring_bitwise_equals_single" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for jp in 2 4; do for cfg in C2 C4; do echo "JPAR=$jp $(DSEA_PIPE_JPAR=$jp timeout 300 python scripts/prof_force.py $cfg 3 2>&1 | tail -1)" >> $o; done; done
