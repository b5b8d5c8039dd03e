#!/bin/bash
# A/B of prebuilt engine copies under _ab/<name> (+ GPU parity of the working tree)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-ab}; mkdir -p $O
if [ -z "$NO_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cv in $EXTRA_CV; do DSEA_FORCE_CV=$cv timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_cv$cv.log 2>&1; echo "rc=$?" >> $O/pytest_cv$cv.log; done
fi
for rep in 1 2; do
for spec in ${VARIANTS:-base v1}; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=$(echo ${spec#*:} | tr ',' ' ')
  for cfg in ${CFGS:-C4 C2}; do
    for cv in ${CVS:-default}; do
      if [ "$cv" = default ]; then unset DSEA_FORCE_CV; else export DSEA_FORCE_CV=$cv; fi
      echo -n "cv=$cv $envs " >> $O/ab.log
      env $envs timeout 300 python scripts/ab_force.py _ab/$v $cfg ${MELT:-200} ${STEPS:-5} >> $O/ab.log 2>&1
    done
  done
done
done
unset DSEA_FORCE_CV
