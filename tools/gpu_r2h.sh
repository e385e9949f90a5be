#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python tests/cuda/clock_probe.py > gpurun_out/clock.txt 2>&1
timeout 300 python tests/cuda/ffn_trace.py > gpurun_out/ffn_trace.txt 2>&1
timeout 300 python tests/cuda/ln_trace.py > gpurun_out/ln_trace.txt 2>&1
timeout 300 python tests/cuda/attn_trace.py > gpurun_out/attn_trace.txt 2>&1
echo done
