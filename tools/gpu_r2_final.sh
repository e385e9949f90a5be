#!/bin/bash
# round-2 validation: full GPU suite, smoke, bench, reference arm, the N > 1
# bench path on one GPU, ncu captures of the four path kernels, CTA timeline
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/parity_errors.jsonl gpurun_out/headline_parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 600 python bench.py --dist-path --steps 10 --warmup 3 --no-cpu-baseline --no-torch-baseline \
  --no-dropin-e2e > gpurun_out/b_dist.json 2> gpurun_out/b_dist.err
B="python bench.py --steps 1 --warmup 1 --layers 1 --no-cpu-baseline --no-torch-baseline --no-dropin-e2e"
for k in k_ffn2 k_gemm_ln k_attn k_gemm_bf16; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k -f $B > gpurun_out/prof_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  --no-torch-baseline --no-dropin-e2e > gpurun_out/b_ncu.log 2>&1
B=32 timeout 300 python tests/cuda/cta_timeline.py > gpurun_out/cta.txt 2>&1
echo done
