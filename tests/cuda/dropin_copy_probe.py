"""Developer probe: where a drop-in fsvd_run_model call (fp32 host tensors,
cfg2) spends its time -- pageable vs pinned copies of the 50 MB activations,
hashing of the factors, the device forward."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import layer_descs, random_layer  # noqa: E402

n = 32 * 512 * 768
x = np.random.default_rng(0).standard_normal(n).astype(np.float32)
d = torch.empty(n, device="cuda")
for name, src in (("pageable", torch.from_numpy(x)), ("pinned", torch.from_numpy(x).pin_memory())):
    for _ in range(2):
        d.copy_(src)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        d.copy_(src)
    torch.cuda.synchronize()
    h2d = (time.perf_counter() - t) / 5
    dst = torch.empty_like(src)
    if name == "pinned":
        dst = dst.pin_memory()
    t = time.perf_counter()
    for _ in range(5):
        dst.copy_(d)
    torch.cuda.synchronize()
    d2h = (time.perf_counter() - t) / 5
    print(f"{name}: H2D 50 MB {h2d * 1e3:.2f} ms ({n * 4 / h2d / 1e9:.1f} GB/s), D2H {d2h * 1e3:.2f} ms ({n * 4 / d2h / 1e9:.1f} GB/s)")

L = abi.lib()
rng = np.random.default_rng(1234)
layers = [random_layer(768, 3072, 12, 12, 32, 384, 384, rng) for _ in range(12)]
descs = layer_descs(layers)
xs = x.reshape(32, 512, 768)
out = np.zeros_like(xs)
plan = abi.TilePlan(16, 16, 64, 1 << 20)
for i in range(4):
    t = time.perf_counter()
    abi.check(L.fsvd_run_model(abi.fptr(xs), 32, 512, 768, descs, 12, abi.MODE_FLASH_V2, plan, 0,
                               b"layer", abi.BF16, None, abi.fptr(out)))
    print(f"fsvd_run_model call {i}: {(time.perf_counter() - t) * 1e3:.2f} ms")
