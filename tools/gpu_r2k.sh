#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for b in 32 16 8; do FSVD_QKV_CHUNKS=1 B=$b timeout 300 python tests/cuda/cta_timeline.py > gpurun_out/cta_b$b.txt 2>&1; done
echo done
