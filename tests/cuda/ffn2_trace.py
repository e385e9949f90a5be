"""Developer tool: timeline of cluster 0 of the CTA-pair FFN (FSVD_FFN_PAIR=1; needs `make trace`)."""
import ctypes as C
import os
os.environ["FSVD_FFN_PAIR"] = "1"
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSVD_LIB"] = os.path.join(ROOT, "paper_2508_01506_b200", "lib", "trace", "libfsvd_b200.so")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import layer_descs, random_layer  # noqa: E402

L = abi.lib()
fr = int(sys.argv[1]) if len(sys.argv) > 1 else 384
act = int(sys.argv[2]) if len(sys.argv) > 2 else 0
layer = random_layer(768, 3072, 12, 12, 32, fr, fr, np.random.default_rng(0), activation=act)
d = layer_descs([layer])
p = C.c_void_p()
abi.check(L.fsvd_layer_pack_create(C.byref(d[0]), abi.BF16, 0, C.byref(p)))
x = torch.randn((16384, 768), device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
work = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):  # one post-LN layer: the pair FFN with the fused LN2, as in the model
    abi.check(L.fsvd_layer_fwd(p, abi.MODE_FLASH_V2, 0, 32, 512, C.c_void_p(x.data_ptr()),
                               C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()),
                               work.numel(), sp))
torch.cuda.synchronize()
buf = (C.c_longlong * 8192)()
L.fsvd_debug_trace2_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
L.fsvd_debug_trace2_copy(buf, 8192)
t = np.array(buf[:], dtype=np.int64)
t0 = t[0]
rel = lambda v: int(v - t0) if v else -1  # noqa: E731
print(f"pdl released {rel(t[6])}, P issued (p_acc commit) {rel(t[7])}")
print(f"pair fr={fr} act={act}: leader start 0, mma thread end {rel(t[1])}, epi end {rel(t[5])}; "
      f"z_full committed {rel(t[2])} zs_ready {rel(t[3])}; peer end {rel(t[4096 + 1])}")
print(" f | L mma1 start  h_free ok  issued | sh_full0 w->ok | sh_full1 w->ok || epi0 h_full w->ok | shfree0 | shfree1 || epi1 h_full w->ok")
for f in range(24):
    m = [rel(t[64 + f * 8 + i]) for i in range(7)]
    e = [rel(t[1024 + f * 8 + i]) for i in range(6)]
    e1 = [rel(t[4096 + 1024 + f * 8 + i]) for i in range(2)]
    print(f"{f:2d} | {m[0]:8d} {m[1]:8d} {m[2]:8d} | {m[3]:8d} {m[4]:8d} | {m[5]:8d} {m[6]:8d} || "
          f"{e[0]:8d} {e[1]:8d} | {e[2]:8d} {e[3]:8d} | {e[4]:8d} {e[5]:8d} || {e1[0]:8d} {e1[1]:8d}")
print("relay (leader / peer): sh_loc complete -> remote arrive done, per atom")
for f in (0, 1, 2, 10, 21, 22, 23):
    print(f, [(rel(t[c + 3000 + f * 4 + a * 2]), rel(t[c + 3001 + f * 4 + a * 2])) for c in (0, 4096) for a in (0, 1)])
tl = (C.c_longlong * 512)()
L.fsvd_debug_trace2_ln_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
L.fsvd_debug_trace2_ln_copy(tl, 512)
tl = np.array(tl[:], dtype=np.int64)
print("LN pieces (acc wait -> got):", " ".join(f"{rel(tl[200 + i])}->{rel(tl[232 + i])}" for i in range(12)))
print(f"LN stats done {rel(tl[300])}, gamma/beta staged {rel(tl[301])}, pass-2 boxes",
      " ".join(str(rel(tl[310 + i])) for i in range(12)), f"stores drained {rel(tl[330])}")
