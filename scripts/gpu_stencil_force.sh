#!/bin/bash
# one B200: stencil GPU tests + G1 bench (k_ftcs_tma) + ncu of k_ftcs_tma and of the
# register-column k_ftcs (A/B), then a source-level ncu capture of k_force_tile on C4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-sf}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x > $O/pytest_grid.log 2>&1; echo rc=$? >> $O/pytest_grid.log
timeout 600 python bench.py --config G1 --steps 20 --warmup 3 > $O/bench_g1.log 2>&1
DSEA_FTCS=col timeout 600 python bench.py --config G1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_g1_col.log 2>&1
for ns in 2 4; do DSEA_FTCS_NS=$ns timeout 600 python bench.py --config G1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_g1_ns$ns.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ftcs -s 2 -c 1 -o $O/prof_ftcs python bench.py --config G1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_ftcs.log 2>&1
if [ -z "$NO_FORCE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force_tile -s 100 -c 1 -o $O/prof_force_C4 \
  python scripts/prof_force.py C4 104 > $O/ncu_force.log 2>&1; echo "rc=$?" >> $O/ncu_force.log
fi
