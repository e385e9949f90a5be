"""Developer microbenchmark of the single kernels (C-ABI test hooks), cfg2 shapes."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_01506_b200 import abi  # noqa: E402

L = abi.lib()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
reps = int(os.environ.get("REPS", "20"))


def timeit(fn):
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


T = 16384
for (N, K) in [(768, 384), (768, 128), (768, 512)]:
    A = torch.randn(T, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    R = torch.randn(T, N, device="cuda").bfloat16()
    v = torch.randn(N, device="cuda")
    y = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    us = timeit(lambda: abi.check(L.fsvd_test_gemm_ln(p(A), K, p(B), K, p(v), p(R), p(v), p(v), 1e-5, p(y),
                                                      T, N, K, st)))
    fl = 2 * T * N * K
    by = 2 * (T * K + T * N * 2)
    print(f"gemm_ln T={T} N={N} K={K}: {us:7.1f} us  {fl / us / 1e6:6.0f} TF/s  {by / us / 1e3:6.0f} GB/s", flush=True)
for (N, K) in [(1152, 768), (768, 384), (384, 768)]:
    A = torch.randn(T, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    Cm = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(N, device="cuda")
    us = timeit(lambda: abi.check(L.fsvd_test_gemm(p(A), K, p(B), K, p(Cm), N, T, N, K, p(v), 0, 0, st)))
    fl = 2 * T * N * K
    print(f"gemm    M={T} N={N} K={K}: {us:7.1f} us  {fl / us / 1e6:6.0f} TF/s", flush=True)
a = torch.randn(T, 768, device="cuda").bfloat16()
b = torch.randn(T, 768, device="cuda").bfloat16()
g = torch.randn(768, device="cuda")
yy = torch.empty_like(a)
us = timeit(lambda: abi.check(L.fsvd_test_resid_layernorm(p(a), p(b), p(g), p(g), 1e-5, p(yy), T, 768, st)))
print(f"resid_ln rows={T} d=768: {us:7.1f} us  {3 * T * 768 * 2 / us / 1e3:6.0f} GB/s", flush=True)

for (B, M) in [(32, 512), (4, 4096)]:
    H, G, rp = 12, 12, 32
    cols = (H + 2 * G) * rp
    qkv = (torch.randn(B * M, cols, device="cuda") * 0.6).bfloat16()
    o = torch.empty(B * M, H * rp, device="cuda", dtype=torch.bfloat16)
    us = timeit(lambda: abi.check(L.fsvd_test_attention(p(qkv), cols, 0, H * rp, (H + G) * rp, B, M, H, G, rp,
                                                        p(o), H * rp, st)))
    exps = B * H * M * M
    print(f"attention B={B} M={M} H={H} rp={rp}: {us:7.1f} us  {exps / us / 1e6:6.2f} T exp/s "
          f"(MUFU-only bound {16 * 148 * 1.92e9 / 1e12:.2f})", flush=True)
