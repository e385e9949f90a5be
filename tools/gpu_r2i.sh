#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FSVD_QKV_CHUNKS=1 timeout 300 python tests/cuda/cta_timeline.py > gpurun_out/cta_c1.txt 2>&1
FSVD_QKV_CHUNKS=2 timeout 300 python tests/cuda/cta_timeline.py > gpurun_out/cta_c2.txt 2>&1
FSVD_NO_PDL=1 FSVD_QKV_CHUNKS=1 timeout 300 python tests/cuda/cta_timeline.py > gpurun_out/cta_nopdl.txt 2>&1
FSVD_SPLIT_BN=128 FSVD_QKV_CHUNKS=2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-torch-baseline --no-dropin-e2e > gpurun_out/b_bn128.json 2>&1
echo done
