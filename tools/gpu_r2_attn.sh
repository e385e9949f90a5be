#!/bin/bash
# K2 checks: kernel tests + decoder (causal K2) + parity subset
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decoder.py tests/test_gpu_parity.py -m gpu -q -x \
  -k "attention or decode or prefill or layer or model or f32 or plane" > gpurun_out/pt_attn.log 2>&1; echo "rc=$?" >> gpurun_out/pt_attn.log
[ -n "$AB" ] && tools/ab.sh "FSVD_LIB=paper_2508_01506_b200/lib/base/libfsvd_b200.so" "FSVD_ATTN_TMA_OUT=1" > gpurun_out/ab_attn.txt 2>&1
exit 0
