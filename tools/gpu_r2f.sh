#!/bin/bash
# GPU suite (headline parity last), bench, concurrent-stream probe
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/parity_errors.jsonl gpurun_out/headline_parity.jsonl
timeout 1500 python -m pytest -q --durations=30 -m gpu tests/test_gpu_parity.py tests/test_gpu_kernels.py \
  tests/test_gpu_dropin.py tests/test_gpu_dense.py tests/test_gpu_decoder.py tests/test_gpu_factorize.py \
  tests/test_model_file.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 300 python tests/cuda/stream_split_probe.py > gpurun_out/split.txt 2>&1
timeout 1200 python -m pytest -q --durations=10 -m gpu tests/test_gpu_headline.py > gpurun_out/pytest_headline.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_headline.log
echo done
