"""Developer probe: the 12-layer cfg2 forward replayed from a CUDA graph vs
direct stream launches (same kernels, same buffers)."""
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
wsb = C.c_size_t()
abi.check(L.fsvd_workspace_bytes_ln(parr, 12, B, M, abi.MODE_FLASH_V2, 0, C.byref(wsb)))
work = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
x = torch.randn((B, M, 768), device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.Stream()


def fwd():
    abi.check(L.fsvd_model_fwd(parr, 12, abi.MODE_FLASH_V2, 0, B, M, C.c_void_p(x.data_ptr()),
                               C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()), wsb.value,
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))


with torch.cuda.stream(stream):
    for _ in range(3):
        fwd()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    fwd()
torch.cuda.synchronize()


def timeit(fn, flush_l2, reps=30):
    ts = []
    with torch.cuda.stream(stream):
        for _ in range(reps):
            if flush_l2:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


for fl in (True, False):
    d = timeit(fwd, fl)
    gr = timeit(g.replay, fl)
    print(f"flush={fl}: direct {d:.3f} ms ({B * M / d / 1e3:.2f} M tok/s)  graph {gr:.3f} ms "
          f"({B * M / gr / 1e3:.2f} M tok/s)")
