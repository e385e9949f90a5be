#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_factorize.py -q -x -k "f32 or F32 or dropin or factor or fp32 or meter" > gpurun_out/pt_x3.log 2>&1; echo "rc=$?" >> gpurun_out/pt_x3.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/pt_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pt_parity.log
