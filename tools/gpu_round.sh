#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list, ncu --set full of the
# FFN and attention kernels.  Outputs land in gpurun_out/ (scratch); the
# summaries worth keeping are copied into profiles/ by hand.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tests/cuda/ffn_bench.py > gpurun_out/ffn_bench.txt 2>&1
if [ "${NCU:-1}" = 0 ]; then echo done; exit 0; fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/b_ncu.log 2>&1
if [ "${NCU:-1}" = 1 ]; then echo done; exit 0; fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ffn -s 2 -c 1 \
  -o gpurun_out/prof_ffn -f python bench.py --steps 1 --warmup 1 --layers 1 --no-cpu-baseline \
  > gpurun_out/prof_ffn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_ln -s 2 -c 1 \
  -o gpurun_out/prof_gemm_ln -f python bench.py --steps 1 --warmup 1 --layers 1 --no-cpu-baseline \
  > gpurun_out/prof_gemm_ln.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn -s 2 -c 1 \
  -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 1 --layers 1 --no-cpu-baseline \
  > gpurun_out/prof_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_bf16 -s 2 -c 1 \
  -o gpurun_out/prof_gemm -f python bench.py --steps 1 --warmup 1 --layers 1 --no-cpu-baseline \
  > gpurun_out/prof_gemm.log 2>&1
echo done
