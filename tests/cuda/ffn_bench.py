"""Developer microbenchmark: FFN / attention / GEMM sublayers at cfg2 shape."""
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
B, M, D = 32, 512, 768
T = B * M
dev = torch.device("cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def make(act, fr=384, r=32):
    layer = random_layer(D, 3072, 12, 12, r, fr, fr, np.random.default_rng(0), activation=act)
    d = layer_descs([layer])
    p = C.c_void_p()
    abi.check(L.fsvd_layer_pack_create(C.byref(d[0]), abi.BF16, 0, C.byref(p)))
    return layer, p


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


x = torch.randn((T, D), device=dev).to(torch.bfloat16)
out = torch.empty_like(x)
work = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for fr in (384, 256, 128):
    for act, name in ((0, "gelu_erf"), (1, "gelu_tanh"), (3, "identity")):
        _, p = make(act, fr)
        res = []
        for v in (1, 2):
            us = timeit(lambda: abi.check(L.fsvd_ffn_fwd(p, v, B, M, C.c_void_p(x.data_ptr()),
                                                         C.c_void_p(out.data_ptr()),
                                                         C.c_void_p(work.data_ptr()), work.numel(), sp)))
            flops = T * 2 * fr * (2 * D + 2 * 3072)
            res.append(f"v{v} {us:7.1f}us {flops / us / 1e6:6.0f}TF/s")
        print(f"fr={fr} {name:10s} " + "  ".join(res), flush=True)
        L.fsvd_layer_pack_destroy(p)
