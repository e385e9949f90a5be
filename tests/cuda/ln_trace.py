"""Developer tool: CTA-0 timeline of k_gemm_ln (needs `make trace`)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSVD_LIB"] = os.path.join(ROOT, "paper_2508_01506_b200", "lib", "trace", "libfsvd_b200.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402

L = abi.lib()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
T, N, K = 16384, 768, int(sys.argv[1]) if len(sys.argv) > 1 else 384
A = torch.randn(T, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
R = torch.randn(T, N, device="cuda").bfloat16()
v = torch.randn(N, device="cuda")
y = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    abi.check(L.fsvd_test_gemm_ln(p(A), K, p(B), K, p(v), p(R), p(v), p(v), 1e-5, p(y), T, N, K,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
buf = (C.c_longlong * 1024)()
L.fsvd_debug_trace_ln_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
L.fsvd_debug_trace_ln_copy(buf, 1024)
t0 = buf[0]
rel = lambda i: buf[i] - t0 if buf[i] else None  # noqa: E731
print("K", K, "alloc+sync", rel(3), "mma start", rel(1), "a_full", rel(2), "epi done", rel(100), "end", rel(101))
print("pass1 end", rel(300), "gamma/beta staged", rel(301), "pass2 pieces", [rel(310 + i) for i in range(12)], "stores drained", rel(330))
for q in range(N // 64):
    print(f"piece {q:2d}: mma_begin {rel(16 + q)} mma_issued {rel(48 + q)} epi_wait_begin {rel(200 + q)} epi_got_acc {rel(232 + q)}")

nst = (N // 64) * K // 64 // 2
print("stage: producer_got_empty  mma_got_full")
for i in range(min(nst, 40)):
    print(i, rel(400 + i), rel(600 + i))
