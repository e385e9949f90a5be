#!/bin/bash
# tools/gpu_kb_env.sh OUT PATTERN "ENV=.." "ENV=.." ... : kbench lines matching PATTERN per env variant, 3 alternations
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=$1; pat=$2; shift 2
for r in 1 2 3; do
  for v in "$@"; do
    env $v REPS=50 timeout 300 python tests/cuda/kbench.py 2>&1 | grep -E "$pat" | sed "s|^|[$v] |"
  done
done > gpurun_out/$out 2>&1
[ -n "$TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > gpurun_out/pt_kb.log 2>&1; echo "rc=$?" >> gpurun_out/pt_kb.log
exit 0
