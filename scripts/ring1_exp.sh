#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; o=gpurun_out/ring1_exp.log; : > $o
for B in 1 3 6 12; do echo "B=$B $(PROF_MODE=2 PROF_B=$B timeout 300 python scripts/prof_force.py C4 2 2>&1 | tail -1)" >> $o; done
echo "fused $(timeout 300 python scripts/prof_force.py C4 2 2>&1 | tail -1)" >> $o
