"""Developer tool: CTA-0 timeline of the fused FFN kernel (needs `make trace`)."""
import ctypes as C
import os
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
LAYER = os.environ.get("LAYER", "1") == "1"  # the model's K4 (fused LN2) or the bare FFN op


def run():
    if LAYER:
        abi.check(L.fsvd_layer_fwd(p, abi.MODE_FLASH_V2, 0, 32, 512, C.c_void_p(x.data_ptr()),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()),
                                   work.numel(), sp))
    else:
        abi.check(L.fsvd_ffn_fwd(p, 2, 32, 512, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
                                 C.c_void_p(work.data_ptr()), work.numel(), sp))


for _ in range(3):
    run()
torch.cuda.synchronize()
# SM clock during the kernel: CTA-0 cycles against the CUDA-event duration
buf = (C.c_longlong * 4096)()
L.fsvd_debug_trace_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
run()
ev1.record()
torch.cuda.synchronize()
L.fsvd_debug_trace_copy(buf, 4096)
t = np.array(buf[:], dtype=np.int64)
t0 = t[0]
us = ev0.elapsed_time(ev1) * 1e3
rel = lambda v: int(v - t0) if v else -1  # noqa: E731
print(f"fr={fr} act={act} kernel start 0, end {rel(t[1])}, producer stream start {rel(t[2])}, "
      f"p_acc {rel(t[3])} p_ready {rel(t[4])}")
print(f"pdl released {rel(t[5])}; P phase x_full wait->got per K chunk:",
      " ".join(f"{rel(t[3000 + 2 * k])}->{rel(t[3001 + 2 * k])}" for k in range(12)))
print(" f | mma1 start  h_free ok  mma1 issued | sh_full0 wait->ok | sh_full1 wait->ok || epi h_full wait->ok | sh_free0 wait->ok | sh_free1 wait->ok || prod mma1 mma2")
for f in range(24):
    m = [rel(t[64 + f * 8 + i]) for i in range(8)]
    e = [rel(t[1024 + f * 8 + i]) for i in range(6)]
    pr = [rel(t[2048 + f * 2 + i]) for i in range(2)]
    print(f"{f:2d} | {m[0]:8d} {m[1]:8d} {m[2]:8d} | {m[3]:8d} {m[4]:8d} | {m[5]:8d} {m[6]:8d} || "
          f"{e[0]:8d} {e[1]:8d} | {e[2]:8d} {e[3]:8d} | {e[4]:8d} {e[5]:8d} || {pr[0]:8d} {pr[1]:8d}")
print(f"event-timed kernel {us:.1f} us; CTA-0 span {int(t[1] - t[0])} cycles "
      f"-> {(t[1] - t[0]) / us / 1e3:.3f} GHz if CTA 0 spans the kernel")
tl = (C.c_longlong * 512)()
L.fsvd_debug_trace_ffn_ln_copy.argtypes = [C.POINTER(C.c_longlong), C.c_int]
L.fsvd_debug_trace_ffn_ln_copy(tl, 512)
tl = np.array(tl[:], dtype=np.int64)
t0 = t[0]
print(f"tail: stream done (z_full) {rel(t[6])}, Z staged (zs_ready) {rel(t[7])}, end {rel(t[1])}")
print("LN pieces (acc wait -> got):", " ".join(f"{rel(tl[200 + i])}->{rel(tl[232 + i])}" for i in range(12)))
print(f"LN stats done {rel(tl[300])}, gamma/beta staged {rel(tl[301])}, pass-2 boxes",
      " ".join(str(rel(tl[310 + i])) for i in range(12)), f"stores drained {rel(tl[330])}")
