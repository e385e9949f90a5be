#!/bin/bash
# bench A/B (qkv chunks), gemm variants, ncu captures of the four path kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b1.json 2> gpurun_out/b1.err
FSVD_QKV_CHUNKS=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-torch-baseline --no-dropin-e2e > gpurun_out/b1_c1.json 2> gpurun_out/b1_c1.err
for v in 0 2 3 4 5; do echo "variant $v"; FSVD_GEMM_VARIANT=$v timeout 120 python tests/cuda/kbench.py 2>&1 | grep "gemm    M"; done > gpurun_out/gemm_variants.txt 2>&1
bash tools/gpu_ncu_r2.sh
echo done
