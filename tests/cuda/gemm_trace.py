"""Developer tool: CTA-0 timeline of k_gemm_bf16 (needs `make trace`)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSVD_LIB"] = os.path.join(ROOT, "paper_2508_01506_b200", "lib", "trace", "libfsvd_b200.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402

L = abi.lib()
M, N, K = 16384, int(sys.argv[1]) if len(sys.argv) > 1 else 1152, int(sys.argv[2]) if len(sys.argv) > 2 else 768
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
v = torch.randn(N, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    abi.check(L.fsvd_test_gemm(C.c_void_p(A.data_ptr()), K, C.c_void_p(B.data_ptr()), K, C.c_void_p(Cm.data_ptr()), N,
                               M, N, K, C.c_void_p(v.data_ptr()), 0, 0, st))
torch.cuda.synchronize()
buf = (C.c_longlong * 1024)()
L.fsvd_debug_trace_gemm_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
L.fsvd_debug_trace_gemm_copy(buf, 1024)
t0 = min(x for x in buf if x)
r = lambda i: (buf[i] - t0) if buf[i] else -1  # noqa: E731
print(f"M={M} N={N} K={K}")
print(" tile | mma: wait_empty got_empty committed | epi: wait_full got_full released")
for i in range(8):
    print(f"{i:4d} | {r(16 + 4 * i):7d} {r(17 + 4 * i):7d} {r(18 + 4 * i):7d} | {r(512 + 4 * i):7d} {r(513 + 4 * i):7d} {r(514 + 4 * i):7d}")
