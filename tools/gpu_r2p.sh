#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py > gpurun_out/pt.log 2>&1; echo "rc=$?" >> gpurun_out/pt.log
B="python bench.py --steps 1 --warmup 1 --layers 1 --no-cpu-baseline --no-torch-baseline --no-dropin-e2e"
for k in k_ffn2 k_gemm_ln k_attn k_gemm_bf16; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k -f $B > gpurun_out/prof_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  --no-torch-baseline --no-dropin-e2e > gpurun_out/b_ncu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
echo done
