#!/bin/bash
# full GPU test suite (+ optional -k filter), smoke
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-tests}; mkdir -p $O
timeout ${TLIM:-2400} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} ${XFLAG} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
