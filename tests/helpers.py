"""Shared test helpers: C-ABI call wrappers and tolerances."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

from paper_2508_01506_b200 import abi
from paper_2508_01506_b200.model import layer_descs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsvd_b200.h")

# north star: <= 1e-4 relative in the fp32-accumulate mode, <= 2e-2 in bf16
TOL_F32 = 1e-4
TOL_BF16 = 2e-2


def rel_err(got, ref):
    """max|got - ref| / max|ref| (SURVEY 8(d) error metric)."""
    return float(np.abs(got.astype(np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def record(case, shape, dtype, err):
    """Appends one measured parity error to gpurun_out/parity_errors.jsonl
    (scratch; the summary worth keeping is copied to profiles/)."""
    import json
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_errors.jsonl"), "a") as f:
        f.write(json.dumps({"case": case, "shape": shape,
                            "dtype": "f32" if dtype == abi.F32 else "bf16", "rel_err": err}) + "\n")


def header_functions():
    """Every function the public header declares."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(fsvd_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


class Meter:
    """RAII-ish wrapper over the C-ABI fsvd_meter."""

    def __init__(self):
        self.L = abi.lib()
        self.h = C.c_void_p()
        abi.check(self.L.fsvd_meter_create(C.byref(self.h)))

    def __del__(self):
        try:
            self.L.fsvd_meter_destroy(self.h)
        except Exception:
            pass

    @property
    def peak(self):
        return self.L.fsvd_meter_peak_transient(self.h)

    @property
    def persistent(self):
        return self.L.fsvd_meter_persistent(self.h)

    @property
    def current(self):
        return self.L.fsvd_meter_current_transient(self.h)

    @property
    def excluded(self):
        return self.L.fsvd_meter_current_excluded(self.h)

    def events(self):
        out = []
        for i in range(self.L.fsvd_meter_event_count(self.h)):
            k, c, b, idv = C.c_int(), C.c_int(), C.c_size_t(), C.c_uint64()
            tag = C.create_string_buffer(256)
            abi.check(self.L.fsvd_meter_event(self.h, i, C.byref(k), C.byref(c), C.byref(b),
                                              C.byref(idv), tag, 256))
            out.append((k.value, c.value, tag.value.decode(), b.value, idv.value))
        return out


def attention(x, attn, heads, plan, dtype, meter=None, prefix=b"attn"):
    L = abi.lib()
    B, M, W = x.shape
    out = np.zeros((B, M, attn.d_model), np.float32)
    st = L.fsvd_flash_svd_attention(abi.fptr(x), B, M, W, attn.desc(), heads, plan, dtype,
                                    meter.h if meter else None, prefix, abi.fptr(out), *out.shape)
    abi.check(st)
    return out


def outproj(ctx, lin, dtype, meter=None, prefix=b"attn"):
    L = abi.lib()
    B, M, W = ctx.shape
    out = np.zeros((B, M, lin.v.shape[1]), np.float32)
    abi.check(L.fsvd_lowrank_output_projection(abi.fptr(ctx), B, M, W, lin.desc(), dtype,
                                               meter.h if meter else None, prefix, abi.fptr(out),
                                               *out.shape))
    return out


def ffn(variant, x, f, plan, dtype, meter=None, prefix=b"ffn"):
    L = abi.lib()
    B, M, W = x.shape
    out = np.zeros_like(x)
    abi.check(L.fsvd_ffn(variant, abi.fptr(x), B, M, W, f.desc(), plan, dtype,
                         meter.h if meter else None, prefix, abi.fptr(out), *out.shape))
    return out


def run_model(x, layers, mode, plan, dtype, pre_ln=False, meter=None, prefix=b"layer"):
    L = abi.lib()
    B, M, W = x.shape
    out = np.zeros_like(x)
    descs = layer_descs(layers)
    abi.check(L.fsvd_run_model(abi.fptr(x), B, M, W, descs, len(layers), mode, plan, int(pre_ln),
                               prefix, dtype, meter.h if meter else None, abi.fptr(out)))
    return out


def run_layer(x, layer, mode, plan, dtype, pre_ln=False, meter=None, prefix=b"layer"):
    L = abi.lib()
    B, M, W = x.shape
    out = np.zeros_like(x)
    d = layer.desc()
    abi.check(L.fsvd_run_layer(abi.fptr(x), B, M, W, C.byref(d), mode, plan, int(pre_ln), prefix,
                               dtype, meter.h if meter else None, abi.fptr(out)))
    return out
