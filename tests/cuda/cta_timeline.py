"""Developer tool (trace build): per-CTA globaltimer timeline of one layer of
the cfg2 forward -- for each path kernel, when its CTAs entered, left
griddepcontrol.wait and exited, so the kernel's span splits into PDL overlap,
work and tail (the spread of CTA exits)."""
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
B, M = int(os.environ.get("B", "32")), 512
rng = np.random.default_rng(1234)
layers = [random_layer(768, 3072, 12, 12, 32, 384, 384, rng) for _ in range(2)]
descs = layer_descs(layers)
packs = []
for i in range(2):
    p = C.c_void_p()
    abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
    packs.append(p)
parr = (C.c_void_p * 2)(*[p.value for p in packs])
wsb = C.c_size_t()
abi.check(L.fsvd_workspace_bytes_ln(parr, 2, B, M, abi.MODE_FLASH_V2, 0, C.byref(wsb)))
work = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
x = torch.randn((B, M, 768), device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(5):
    abi.check(L.fsvd_model_fwd(parr, 2, abi.MODE_FLASH_V2, 0, B, M, C.c_void_p(x.data_ptr()),
                               C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()), wsb.value, sp))
torch.cuda.synchronize()
res = {}
for tu in ("gemm", "attn", "gemm_ln", "ffn"):
    fn = getattr(L, f"fsvd_debug_cta_times_{tu}")
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * (4096 * 8))()
    fn(buf, 4096 * 8)
    a = np.array(buf[:], dtype=np.uint64).reshape(4096, 8)
    a = a[a[:, 2] > 0]
    if len(a):  # kernels this layer did not launch (e.g. k_ffn when the pair FFN runs) are skipped
        res[tu] = a
t0 = min(int(r[:, 0].min()) for r in res.values())
print(f"B={B} M={M}: last layer of a 2-layer forward; times in us from the first CTA entry")
for tu in [k for k in ("gemm", "attn", "gemm_ln", "ffn") if k in res]:
    a = res[tu].astype(np.int64) - t0
    work = (a[:, 2] - a[:, 1]) / 1e3
    print(f"{tu:8s} ctas={len(a):4d} SMs={len(set(res[tu][:, 5].tolist())):3d} | entry {a[:, 0].min() / 1e3:7.2f}"
          f"..{a[:, 0].max() / 1e3:7.2f} | wait-released {a[:, 1].min() / 1e3:7.2f}..{a[:, 1].max() / 1e3:7.2f}"
          f" | exit {a[:, 2].min() / 1e3:7.2f}..{a[:, 2].max() / 1e3:7.2f} | per-CTA work min {work.min():6.2f}"
          f" med {np.median(work):6.2f} max {work.max():6.2f} us")
    ghz = (res[tu][:, 4].astype(np.float64) - res[tu][:, 3]) / (res[tu][:, 2].astype(np.float64) - res[tu][:, 1])
    print(f"          SM clock over the CTA's work (clock64 / globaltimer): median {np.median(ghz):.3f} GHz,"
          f" min {ghz.min():.3f}, max {ghz.max():.3f}")
    # exit histogram (us): how many CTAs are still running over the kernel's span
    rel = (a[:, 2] - a[:, 1].min()) / 1e3
    print("          exits (us after first release), deciles:",
          " ".join(f"{v:6.2f}" for v in np.percentile(rel, [0, 10, 25, 50, 75, 90, 100])))
if "attn" in res and os.environ.get("ATTN_DETAIL"):
    # K2: exit time by the CTA's item count and by its SM's total item count / die half
    a = res["attn"].astype(np.int64)
    rel = (a[:, 2] - a[:, 1].min()) / 1e3
    grid = len(a)
    items = (M // 128) * 12 * B
    bid = np.arange(grid)
    n_it = (items - bid + grid - 1) // grid
    sm = res["attn"][:, 5].astype(np.int64)
    sm_items = {s: n_it[sm == s].sum() for s in set(sm.tolist())}
    for k in sorted(set(n_it.tolist())):
        sel = n_it == k
        print(f"  attn CTAs with {k} items: {sel.sum():4d}, exit min {rel[sel].min():6.2f} med {np.median(rel[sel]):6.2f} max {rel[sel].max():6.2f}")
    tot = np.array([sm_items[s] for s in sm])
    for k in sorted(set(tot.tolist())):
        sel = tot == k
        print(f"  attn CTAs on SMs with {k} items: {sel.sum():4d}, exit med {np.median(rel[sel]):6.2f} max {rel[sel].max():6.2f}")
    for half in (0, 1):
        sel = (sm >= 74) == bool(half)
        print(f"  attn SMs {'74-147' if half else '0-73'}: exit med {np.median(rel[sel]):6.2f} max {rel[sel].max():6.2f}")
    per_item = (rel - 0) / n_it
    print("  attn per-item time by smid (first 16 SMs):", " ".join(f"{s}:{np.mean(per_item[sm == s]):.2f}" for s in range(16)))
    order = np.argsort(rel)
    print("  slowest 12 CTAs (bid, sm, items, exit):", [(int(b), int(sm[b]), int(n_it[b]), round(float(rel[b]), 1)) for b in order[-12:]])
    print("  fastest 12 CTAs (bid, sm, items, exit):", [(int(b), int(sm[b]), int(n_it[b]), round(float(rel[b]), 1)) for b in order[:12]])
