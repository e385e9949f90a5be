"""GPU counterpart of the reference's `bench` command (commands.cpp:238-333):
the same sweep (ranks x batches x sequence lengths x modes) and the same
13-column CSV, run through this library's host API (fsvd_run_model) on the
B200.

  b,m,h,d_model,d_ff,rank,mode,peak_transient_bytes,persistent_bytes,
  flops_exact,io_bytes_in,wall_ms,max_abs_err_vs_dense

As in the reference: dense weights are drawn, factorized at rank r
(proj_rank = ffn_rank = r; here by the device factorizer), the Dense mode runs
the dense twin rebuilt from the factors, every mode's output is compared with
the Dense run, the meter reports the reference's transient / persistent
classes, flops_exact / io_bytes are the planner closed forms times the layer
count, and wall_ms is the median over --reps of one run_model call (host
arrays in and out, like the reference's timing).

  python tools/sweep.py --b-list 1,8 --m-list 128,512 --r-list 16,32 --out sweep.csv
"""
import argparse
import ctypes as C
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200 import factorize as F  # noqa: E402
from paper_2508_01506_b200.model import layer_descs  # noqa: E402

MODES = {"dense": abi.MODE_DENSE, "naive": abi.MODE_NAIVE_LOWRANK, "flash_v1": abi.MODE_FLASH_V1,
         "flash_v2": abi.MODE_FLASH_V2}


def ints(s):
    return [int(v) for v in s.split(",") if v]


def dense_layer(d, df, rng):
    n = lambda *s, sc=1.0: (rng.standard_normal(s) * sc).astype(np.float32)  # noqa: E731
    return F.DenseLayerWeights(n(d, d, sc=d ** -.5), n(d, sc=.02), n(d, d, sc=d ** -.5),
                               n(d, sc=.02), n(d, d, sc=d ** -.5), n(d, sc=.02),
                               n(d, d, sc=d ** -.5), n(d, sc=.02), n(d, df, sc=d ** -.5),
                               n(df, sc=.02), n(df, d, sc=d ** -.5), n(d, sc=.02))


class Meter:
    def __init__(self, L):
        self.L, self.h = L, C.c_void_p()
        abi.check(L.fsvd_meter_create(C.byref(self.h)))

    def close(self):
        self.L.fsvd_meter_destroy(self.h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b-list", default="1,8")
    ap.add_argument("--m-list", default="128,512")
    ap.add_argument("--r-list", default="32")
    ap.add_argument("--modes", default="dense,naive,flash_v1,flash_v2")
    ap.add_argument("--d-model", type=int, default=768)
    ap.add_argument("--d-ff", type=int, default=3072)
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    L = abi.lib()
    groups = a.groups or a.heads
    dt = abi.BF16 if a.dtype == "bf16" else abi.F32
    plan = abi.TilePlan(16, 16, 64, 1 << 22)
    lines = ["b,m,h,d_model,d_ff,rank,mode,peak_transient_bytes,persistent_bytes,flops_exact,"
             "io_bytes_in,wall_ms,max_abs_err_vs_dense"]
    for r in ints(a.r_list):
        rng = np.random.default_rng(a.seed)
        dense = [dense_layer(a.d_model, a.d_ff, rng) for _ in range(a.layers)]
        layers = F.factorize_layers(dense, a.heads, groups, rank=r, proj_rank=r, ffn_rank=r)
        descs = layer_descs(layers)
        for b in ints(a.b_list):
            for m in ints(a.m_list):
                x = np.random.default_rng(a.seed ^ (b * 1000003 + m * 10007 + r * 101)).uniform(
                    -1, 1, (b, m, a.d_model)).astype(np.float32)
                outs = {}
                for name in ["dense"] + [s for s in a.modes.split(",") if s != "dense"]:
                    mode = MODES[name]
                    if name != "dense" and name not in a.modes.split(","):
                        continue
                    mdt = abi.BF16 if mode in (abi.MODE_DENSE, abi.MODE_NAIVE_LOWRANK) else dt
                    got = np.zeros_like(x)
                    walls, peak, pers = [], 0, 0
                    for rep in range(max(a.reps, 1)):
                        meter = Meter(L)
                        t0 = time.perf_counter()
                        abi.check(L.fsvd_run_model(abi.fptr(x), b, m, a.d_model, descs, len(layers),
                                                   mode, plan, 0, b"layer", mdt, meter.h,
                                                   abi.fptr(got)))
                        walls.append((time.perf_counter() - t0) * 1e3)
                        if rep == 0:
                            peak = L.fsvd_meter_peak_transient(meter.h)
                            pers = L.fsvd_meter_persistent(meter.h)
                        meter.close()
                    outs[name] = got.copy()
                    if name not in a.modes.split(","):
                        continue
                    g = abi.Geometry(b, m, a.d_model, a.d_ff, a.heads, groups, r, a.layers)
                    fl, fi, fo = C.c_uint64(), C.c_uint64(), C.c_uint64()
                    abi.check(L.fsvd_flops_exact(g, mode, C.byref(fl)))
                    abi.check(L.fsvd_io_bytes(g, mode, C.byref(fi), C.byref(fo)))
                    err = float(np.abs(got - outs["dense"]).max())
                    lines.append(f"{b},{m},{a.heads},{a.d_model},{a.d_ff},{r},{name},{peak},{pers},"
                                 f"{fl.value * a.layers},{fi.value * a.layers},"
                                 f"{statistics.median(walls):.3f},{err:.6g}")
                    print(lines[-1], flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")
        print(f"wrote {a.out} ({len(lines) - 1} rows)")


if __name__ == "__main__":
    main()
