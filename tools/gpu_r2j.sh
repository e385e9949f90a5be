#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tests/cuda/ffn_trace.py > gpurun_out/ffn_trace.txt 2>&1
echo done
