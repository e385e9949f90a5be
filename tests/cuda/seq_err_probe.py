"""Probe: 12-layer cfg2 (bench weights) error per sequence against the
reference, for the sequences given in SEQS (env), in this process's kernel
configuration (FSVD_* switches)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import helpers as H  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import bf16_round, random_layer, round_layer_bf16  # noqa: E402
from test_gpu_headline import Device, PLAN  # noqa: E402

os.environ.setdefault("FLASHSVD_THREADS", str(os.cpu_count() or 1))
L = abi.lib()
rng = np.random.default_rng(1234)
layers = [round_layer_bf16(random_layer(768, 3072, 12, 12, 32, 384, 384, rng)) for _ in range(12)]
x = bf16_round(np.random.default_rng(7).standard_normal((32, 512, 768)).astype(np.float32))
dev = Device(L, layers, 32, 512)
got = dev.fwd(x, abi.MODE_FLASH_V2, False, 12)
ref = oracle.Reference()
out = []
for s in [int(v) for v in os.environ.get("SEQS", "5").split(",")]:
    want = ref.run_model(np.ascontiguousarray(x[[s]]), layers, abi.MODE_FLASH_V2, PLAN)
    e = H.rel_err(got[[s]], want)
    d = np.abs(got[[s]] - want)
    i = np.unravel_index(np.argmax(d), d.shape)
    out.append(f"seq {s}: rel {e:.4f} (max|d| {d.max():.4f} at row {i[1]} col {i[2]}, max|ref| {np.abs(want).max():.3f}, mean|d| {d.mean():.2e})")
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
