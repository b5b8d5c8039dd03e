#!/bin/bash
# ncu --set full capture of the force kernel on C4 (lattice start, a few steps)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-ncu}; mkdir -p $O
K=${KREGEX:-k_force}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $O/prof_force_${CFG:-C4} \
  python scripts/prof_force.py ${CFG:-C4} 4 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
