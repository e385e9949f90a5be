"""Dev probe: K3 wide-rank cluster kernel vs the recompute variant, one
(fr, d_ff, T) case per subprocess under a short timeout (hang detection).
  python tests/cuda/wide_probe.py"""
import os
import subprocess
import sys

CASE = r'''
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, "%s")
from paper_2508_01506_b200 import abi
from paper_2508_01506_b200.model import layer_descs, random_layer
fr, df, T = %d, %d, %d
L = abi.lib()
rng = np.random.default_rng(1)
lay = random_layer(256, df, 4, 4, 16, 64, fr, rng)
d = layer_descs([lay])
p = C.c_void_p(); abi.check(L.fsvd_layer_pack_create(C.byref(d[0]), abi.BF16, 0, C.byref(p)))
parr = (C.c_void_p * 1)(p.value)
ws = C.c_size_t(); abi.check(L.fsvd_workspace_bytes(parr, 1, 1, T, abi.MODE_FLASH_V1, C.byref(ws)))
work = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
torch.manual_seed(0)
x = torch.randn((1, T, 256), device="cuda").to(torch.bfloat16); o = torch.empty_like(x)
abi.check(L.fsvd_ffn_fwd(p, 1, 1, T, C.c_void_p(x.data_ptr()), C.c_void_p(o.data_ptr()),
                         C.c_void_p(work.data_ptr()), ws, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
np.save("%s", o.float().cpu().numpy())
'''
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for fr, df, T in [(512, 512, 128), (576, 1024, 256), (1024, 512, 128), (1024, 1024, 256),
                  (1024, 3072, 1024), (1152, 1536, 128), (1280, 2048, 384)]:
    res = {}
    for mode in ("cluster", "recompute"):
        env = dict(os.environ)
        if mode == "recompute":
            env["FSVD_FFN_WIDE_RECOMPUTE"] = "1"
        out = f"/tmp/wide_{mode}.npy"
        try:
            r = subprocess.run([sys.executable, "-c", CASE % (ROOT, fr, df, T, out)], env=env,
                               timeout=60, capture_output=True, text=True)
            res[mode] = "ok" if r.returncode == 0 else "rc%d %s" % (r.returncode, r.stderr[-300:])
        except subprocess.TimeoutExpired:
            res[mode] = "HANG"
    import numpy as np
    diff = None
    if res["cluster"] == "ok" and res["recompute"] == "ok":
        a, b = np.load("/tmp/wide_cluster.npy"), np.load("/tmp/wide_recompute.npy")
        diff = float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-9))
    print(fr, df, T, res, "rel_diff", diff, flush=True)
