#!/bin/bash
# round-2 check: full GPU suite + bench + reference batch sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b1.json 2> gpurun_out/b1.err
for rb in 4 16 32; do timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --ref-batch $rb > gpurun_out/ref_b$rb.json 2>&1; done
echo done
