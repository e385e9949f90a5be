"""A/B helper: median ms per 12-layer cfg2 forward (flash_v2, post-LN, L2
flushed between steps) in this process -- variants are selected by the
FSVD_* developer environment switches of the caller; run alternately."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import layer_descs, random_layer  # noqa: E402

L = abi.lib()
NL = int(os.environ.get("NL", "12"))
B, M = int(os.environ.get("B", "32")), 512
MODE = abi.MODE_FLASH_V1 if os.environ.get("MODE") == "v1" else abi.MODE_FLASH_V2
PRE = int(os.environ.get("PRE_LN", "0"))
rng = np.random.default_rng(1234)
layers = [random_layer(768, 3072, 12, 12, 32, 384, 384, rng) for _ in range(NL)]
descs = layer_descs(layers)
packs = []
for i in range(NL):
    p = C.c_void_p()
    abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
    packs.append(p)
parr = (C.c_void_p * NL)(*[p.value for p in packs])
wsb = C.c_size_t()
abi.check(L.fsvd_workspace_bytes_ln(parr, NL, B, M, MODE, PRE, C.byref(wsb)))
work = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
x = torch.randn((B, M, 768), device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def fwd():
    abi.check(L.fsvd_model_fwd(parr, NL, MODE, PRE, B, M, C.c_void_p(x.data_ptr()),
                               C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()), wsb.value, sp))


for _ in range(5):
    fwd()
ts = []
for _ in range(int(os.environ.get("REPS", "40"))):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fwd()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
tag = os.environ.get("TAG", "")
print(f"{tag} median {np.median(ts):.4f} ms  min {min(ts):.4f}  mean {np.mean(ts):.4f}  "
      f"{B * M / np.median(ts) / 1e3:.3f} M tok/s  "
      f"checksum {float(out.float().abs().sum()):.6e}", flush=True)
