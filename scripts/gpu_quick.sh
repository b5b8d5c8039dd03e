#!/bin/bash
# quick force-kernel timing + single-GPU parity (C1/C2/C4), optional ncu capture (NCU=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-quick}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in ${CFGS:-C2 C4}; do timeout 300 python scripts/prof_force.py $c 6 > $O/prof_$c.log 2>&1; done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force -s 2 -c 1 -o $O/prof_force_C4 \
  python scripts/prof_force.py C4 4 > $O/ncu_full.log 2>&1; echo "rc=$?" >> $O/ncu_full.log
fi
