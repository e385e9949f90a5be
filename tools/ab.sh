#!/bin/bash
# usage: tools/ab.sh "ENV=.. ENV2=.." "ENV=.." ... ; alternates the variants 3 rounds
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in "$@"; do
    env $v TAG="[$v]" timeout 300 python tests/cuda/ab_step.py
  done
done
