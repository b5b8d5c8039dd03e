#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out; out=gpurun_out/sweep.log; : > $out
for jp in 2 4; do for mh in 32 48 64; do for kb in 56 72 100; do
  echo "JPAR=$jp MAXH=$mh KB=$kb $(DSEA_JPAR=$jp DSEA_MAXH=$mh DSEA_SMEM_KB=$kb timeout 120 python scripts/prof_force.py C2 6 2>&1 | tail -1) | $(DSEA_JPAR=$jp DSEA_MAXH=$mh DSEA_SMEM_KB=$kb timeout 120 python scripts/prof_force.py C4 2 2>&1 | tail -1)" >> $out
done; done; done
