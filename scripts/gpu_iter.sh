#!/bin/bash
# one iteration on a B200: parity tests of the single-GPU path, force-kernel timing
# (default tile kernel vs the pipelined A/B kernel), default bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-iter}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvt.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in C2 C4; do
  timeout 300 python scripts/prof_force.py $c 6 > $O/prof_tile_$c.log 2>&1
  DSEA_FORCE=pipe timeout 300 python scripts/prof_force.py $c 6 > $O/prof_pipe_$c.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
