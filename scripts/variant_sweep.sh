#!/bin/bash
# A/B compile-time variants of the force kernel on the GPU box:
#   VARIANTS="CW:HOME[:MAXH] ..."  (each rebuilt with --force, then C2/C4 probes)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/variants.log
: > $out
for v in ${VARIANTS:-"4:64 12:192"}; do
  IFS=: read cw home maxh <<< "$v"
  export DSEA_NVCC_EXTRA="-DDSEA_PIPE_CW=$cw -DDSEA_PIPE_HOME=$home ${EXTRA_DEFS}"
  python -m paper_2507_11289_b200.build --force > gpurun_out/build_$cw_$home.log 2>&1 || { echo "build failed $v" >> $out; continue; }
  echo "== CW=$cw HOME=$home MAXH=${maxh:-64}" >> $out
  DSEA_MAXH=${maxh:-64} timeout 300 python scripts/prof_force.py C2 6 >> $out 2>&1
  DSEA_MAXH=${maxh:-64} timeout 300 python scripts/prof_force.py C4 3 >> $out 2>&1
  if [ -n "$PYTEST_K" ]; then DSEA_MAXH=${maxh:-64} timeout 600 python -m pytest tests -m gpu -q -x -k "$PYTEST_K" 2>&1 | grep -E "Error|assert|passed|failed|^E " | head -30 >> $out; fi
done
