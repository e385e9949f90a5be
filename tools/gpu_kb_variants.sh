#!/bin/bash
# tools/gpu_kb_variants.sh OUT PATTERN lib1 lib2 ... : kbench lines matching PATTERN per library, 3 alternations
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=$1; pat=$2; shift 2
for r in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib=paper_2508_01506_b200/lib/$v/libfsvd_b200.so; fi
    FSVD_LIB=$lib REPS=50 timeout 300 python tests/cuda/kbench.py 2>&1 | grep -E "$pat" | sed "s|^|[$v] |"
  done
done > gpurun_out/$out 2>&1
