#!/bin/bash
# one B200: single-GPU MD parity (incl. staged rings of one = pooled staging), the
# shared-device ring tests (ranks on one GPU: pooled output buffers + peer hop), the
# stencil tests; each test bounded, stop at the first failure
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-c1}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nvt.py tests/test_gpu_ring_shared.py -x -q --timeout 300 -rf > $O/pytest_md.log 2>&1; echo "rc=$?" >> $O/pytest_md.log
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q --timeout 300 -rf > $O/pytest_grid.log 2>&1; echo "rc=$?" >> $O/pytest_grid.log
