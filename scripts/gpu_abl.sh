#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-abl}; mkdir -p $O
for v in ${VARIANTS:-base}; do timeout 300 python scripts/abl_force.py _ab/$v ${CFG:-C4} 3 >> $O/abl.log 2>&1; done
