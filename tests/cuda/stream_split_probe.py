"""Probe: does splitting the cfg2 batch over concurrent streams fill the SMs
that 128-row-tile kernels (K4, K6: 128 CTAs on 148 SMs) leave idle?

Times the 12-layer bf16 flash_v2 forward at B=32, M=512 as one call and as
S concurrent calls of B/S sequences on S streams (own workspace each).
Dev tool (not a test); prints one line per variant."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import layer_descs, random_layer  # noqa: E402

D, DF, H, G, R, PR, FR, M, B, NL = 768, 3072, 12, 12, 32, 384, 384, 512, 32, 12


def main():
    L = abi.lib()
    rng = np.random.default_rng(1234)
    layers = [random_layer(D, DF, H, G, R, PR, FR, rng) for _ in range(NL)]
    descs = layer_descs(layers)
    packs = []
    for i in range(NL):
        p = C.c_void_p()
        abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
        packs.append(p)
    parr = (C.c_void_p * NL)(*[p.value for p in packs])
    x = torch.randn((B, M, D), device="cuda", dtype=torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for S in [int(s) for s in os.environ.get("SPLITS", "1,2,4").split(",")]:
        bs = B // S
        wsb = C.c_size_t()
        abi.check(L.fsvd_workspace_bytes_ln(parr, NL, bs, M, abi.MODE_FLASH_V2, 0, C.byref(wsb)))
        works = [torch.empty(wsb.value, dtype=torch.uint8, device="cuda") for _ in range(S)]
        streams = [torch.cuda.Stream() for _ in range(S)]
        out = torch.zeros_like(x)
        main_s = torch.cuda.current_stream()

        def step():
            ev = torch.cuda.Event()
            ev.record(main_s)
            for s in range(S):
                st = streams[s]
                st.wait_event(ev)
                abi.check(L.fsvd_model_fwd(parr, NL, abi.MODE_FLASH_V2, 0, bs, M,
                                           C.c_void_p(x[s * bs].data_ptr()),
                                           C.c_void_p(out[s * bs].data_ptr()),
                                           C.c_void_p(works[s].data_ptr()), wsb.value,
                                           C.c_void_p(st.cuda_stream)))
            for s in range(S):
                e = torch.cuda.Event()
                e.record(streams[s])
                main_s.wait_event(e)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            step()
            b.record(main_s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref))
        print(f"splits={S} batch/stream={bs}: {ms:.3f} ms/step  {B * M / ms / 1e3:.3f} M tok/s  "
              f"min {min(ts):.3f}  bitwise-equal-to-1-stream={same}", flush=True)


if __name__ == "__main__":
    main()
