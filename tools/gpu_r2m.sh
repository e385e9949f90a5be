#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export FSVD_QKV_CHUNKS=1
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-torch-baseline --no-dropin-e2e"
timeout 600 $B > gpurun_out/b_base.json 2>&1
FSVD_FFN_ROT=1 timeout 600 $B > gpurun_out/b_rot.json 2>&1
FSVD_FFN_PAIR=1 timeout 600 $B > gpurun_out/b_pair.json 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py -k pair > gpurun_out/pt_pair.log 2>&1
echo done
