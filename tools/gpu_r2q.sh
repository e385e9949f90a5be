#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python tools/config_bench.py --cfg 3 4 --out gpurun_out/config_bench.jsonl > gpurun_out/config_bench.log 2>&1
timeout 300 python tests/cuda/variants_probe.py > gpurun_out/variants.txt 2>&1
timeout 300 python tools/bench_decode.py > gpurun_out/decode.txt 2>&1
echo done
