#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
LAYER=1 timeout 300 python tests/cuda/ffn_trace.py > gpurun_out/ffn_trace_l1.txt 2>&1
B=32 timeout 300 python tests/cuda/cta_timeline.py > gpurun_out/cta.txt 2>&1
timeout 300 python tests/cuda/ln_trace.py > gpurun_out/ln_trace.txt 2>&1
echo done
