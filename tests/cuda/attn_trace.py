"""Developer tool: timeline of one attention CTA (needs `make trace`)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSVD_LIB"] = os.path.join(ROOT, "paper_2508_01506_b200", "lib", "trace", "libfsvd_b200.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402

L = abi.lib()
B, M, H, G, rp = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 512, 12, 12, 32
B = 16384 // M if M <= 16384 else 1
cols = (H + 2 * G) * rp
qkv = (torch.randn(B * M, cols, device="cuda") * 0.6).bfloat16()
o = torch.empty(B * M, H * rp, device="cuda", dtype=torch.bfloat16)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    abi.check(L.fsvd_test_attention(C.c_void_p(qkv.data_ptr()), cols, 0, H * rp, (H + G) * rp, B, M, H, G,
                                    rp, C.c_void_p(o.data_ptr()), H * rp, st))
torch.cuda.synchronize()
buf = (C.c_longlong * 2048)()
L.fsvd_debug_trace_attn_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
L.fsvd_debug_trace_attn_copy(buf, 2048)
t0 = buf[0]
r = lambda i: (buf[i] - t0) if buf[i] else -1  # noqa: E731
print(f"M={M}: start 0, q landed {r(1)}, softmax done {r(2)}, end {r(3)}")
print(" j | mma: kv_full  s_free  p_full | softmax: wait_s  got_s  wait_o  got_o  p_arrive")
for j in range((M + 127) // 128):
    print(f"{j:2d} | {r(16 + j):7d} {r(48 + j):7d} {r(80 + j):7d} | {r(112 + j):7d} {r(144 + j):7d} "
          f"{r(176 + j):7d} {r(208 + j):7d} {r(240 + j):7d}")
print("item | tma_q  mma_start  softmax_start  tile_p_arrive[0..3]")
for it in range(12):
    print(f"{it:3d} | {r(500 + it):7d} {r(400 + it):7d} {r(300 + it):7d} | " +
          " ".join(f"{r(600 + it * 4 + j):7d}" for j in range(4)))
print("item (softmax thread 0, tile 0 / 1): got_s0 maxx0 got_o0 p_arr0 epi_done | got_s1 maxx1 | item_end")
for it in range(12):
    print(f"{it:3d} | " + " ".join(f"{r(1100 + it * 8 + k):7d}" for k in (0, 1, 2, 3, 4)) + " | " +
          " ".join(f"{r(1100 + it * 8 + k):7d}" for k in (5, 7)) + f" | {r(1100 + it * 8 + 6):7d}")
