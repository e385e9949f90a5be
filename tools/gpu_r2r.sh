#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 0 1; do
FSVD_LN_PAIR=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_ln$v.csv python tests/cuda/ab_step.py > /dev/null 2>&1
done
echo done
