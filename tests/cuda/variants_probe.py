"""Developer probe: the cfg2 12-layer forward in the other supported
schedules (FFN V1, pre-LN) next to the headline post-LN V2."""
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
rng = np.random.default_rng(0)
layers = [random_layer(768, 3072, 12, 12, 32, 384, 384, rng) for _ in range(12)]
descs = layer_descs(layers)
packs = []
for i in range(12):
    p = C.c_void_p()
    abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
    packs.append(p)
parr = (C.c_void_p * 12)(*[p.value for p in packs])
B, M = 32, 512
x = torch.randn((B, M, 768), device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, mode, pre in (("post-LN V2", abi.MODE_FLASH_V2, 0), ("post-LN V1", abi.MODE_FLASH_V1, 0),
                        ("pre-LN V2", abi.MODE_FLASH_V2, 1), ("pre-LN V1", abi.MODE_FLASH_V1, 1)):
    wsb = C.c_size_t()
    abi.check(L.fsvd_workspace_bytes_ln(parr, 12, B, M, mode, pre, C.byref(wsb)))
    work = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def fwd():
        abi.check(L.fsvd_model_fwd(parr, 12, mode, pre, B, M, C.c_void_p(x.data_ptr()),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()),
                                   wsb.value, s))
    for _ in range(3):
        fwd()
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fwd()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    print(f"{name}: {ms:.3f} ms  {B * M / ms / 1e3:.2f} M tok/s  workspace {wsb.value / 2**20:.0f} MiB")
    del work
