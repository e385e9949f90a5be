#!/bin/bash
# tools/gpu_ab_generic.sh OUT "variant env" ... : tools/ab.sh into gpurun_out/OUT
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=$1; shift
tools/ab.sh "$@" > gpurun_out/$out 2>&1
