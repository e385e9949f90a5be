"""Python handles on the CPU checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this package.  Two checkers are exposed with the same call shapes:

* ``Restatement`` -- oracle/liboracle.so, the plain-C restatement
  (fsvd_oracle.c), built on demand with gcc if missing.
* ``Reference``   -- oracle/_ref/libfsvd_ref.so, the unmodified reference
  library compiled from /root/reference by oracle/Makefile (prebuilt files
  travel to the GPU box; /root/reference itself does not).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2508_01506_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libfsvd_ref.so")

_P = C.POINTER
_sz = C.c_size_t
_fp = _P(C.c_float)


def build(ref: bool = False):
    targets = ["all"] + (["ref"] if ref and os.path.isdir("/root/reference/proj") else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f(a):
    return abi.fptr(a)


class _Base:
    prefix = ""

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def random(self, shape, seed, stddev=1.0):
        """oracle::random_tensor (tests/support/oracles.hpp:80-87)."""
        n = int(np.prod(shape))
        out = np.empty(n, np.float32)
        self._fn("random_fill")(_f(out), n, C.c_uint64(seed), C.c_double(stddev))
        return out.reshape(shape)


class Restatement(_Base):
    prefix = "fo_"

    def __init__(self):
        if not os.path.exists(RESTATEMENT_SO):
            build()
        self.lib = C.CDLL(RESTATEMENT_SO, mode=C.RTLD_LOCAL)
        L = self.lib
        L.fo_random_fill.argtypes = [_fp, _sz, C.c_uint64, C.c_double]
        L.fo_flash_svd_attention.argtypes = [_fp, _sz, _sz, _P(abi.AttnDesc), _sz,
                                             _P(abi.TilePlan), _fp]
        L.fo_lowrank_output_projection.argtypes = [_fp, _sz, _sz, _P(abi.LinearDesc), _fp]
        L.fo_ffn.argtypes = [C.c_int, _fp, _sz, _sz, _sz, _P(abi.FfnDesc), _P(abi.TilePlan), _fp]
        L.fo_residual_norm.argtypes = [_fp, _fp, _sz, _sz, _fp, _fp, C.c_float, _fp]
        L.fo_run_layer.argtypes = [_fp, _sz, _sz, _P(abi.LayerDesc), C.c_int, _P(abi.TilePlan),
                                   C.c_int, _fp]
        L.fo_run_model.argtypes = [_fp, _sz, _sz, _P(abi.LayerDesc), _sz, C.c_int,
                                   _P(abi.TilePlan), C.c_int, _fp]
        L.fo_expected_bytes.argtypes = [C.c_int, _P(abi.Geometry)]
        L.fo_expected_bytes.restype = _sz
        L.fo_tile_working_set.argtypes = [_P(abi.TilePlan), C.c_int, _P(abi.Geometry),
                                          _P(C.c_int)]
        L.fo_tile_working_set.restype = _sz
        L.fo_flash_layer_peak_transient_bytes.argtypes = [_P(abi.Geometry)]
        L.fo_flash_layer_peak_transient_bytes.restype = _sz
        L.fo_flash_layer_persistent_bytes.argtypes = [_P(abi.Geometry)]
        L.fo_flash_layer_persistent_bytes.restype = _sz

    def attention(self, x, attn, heads, plan):
        out = np.zeros_like(x)
        st = self.lib.fo_flash_svd_attention(_f(x), x.shape[0], x.shape[1], attn.desc(), heads,
                                             plan, _f(out))
        abi_check(st)
        return out

    def outproj(self, ctx, lin):
        out = np.zeros(ctx.shape[:2] + (lin.v.shape[1],), np.float32)
        abi_check(self.lib.fo_lowrank_output_projection(_f(ctx), ctx.shape[0], ctx.shape[1],
                                                        lin.desc(), _f(out)))
        return out

    def ffn(self, variant, x, ffn, plan):
        out = np.zeros_like(x)
        abi_check(self.lib.fo_ffn(variant, _f(x), x.shape[0], x.shape[1], x.shape[2],
                                  ffn.desc(), plan, _f(out)))
        return out

    def run_model(self, x, layers, mode, plan, pre_ln=False):
        from paper_2508_01506_b200.model import layer_descs
        out = np.zeros_like(x)
        descs = layer_descs(layers)
        abi_check(self.lib.fo_run_model(_f(x), x.shape[0], x.shape[1], descs, len(layers), mode,
                                        plan, int(pre_ln), _f(out)))
        return out


class Reference(_Base):
    prefix = "ref_"

    @staticmethod
    def available():
        return os.path.exists(REFERENCE_SO)

    def __init__(self):
        if not os.path.exists(REFERENCE_SO):
            build(ref=True)
        self.lib = C.CDLL(REFERENCE_SO, mode=C.RTLD_LOCAL)
        L = self.lib
        m3 = _P(_sz)
        L.ref_last_error.restype = C.c_char_p
        L.ref_random_fill.argtypes = [_fp, _sz, C.c_uint64, C.c_double]
        L.ref_flash_svd_attention.argtypes = [_fp, _sz, _sz, _P(abi.AttnDesc), _sz,
                                              _P(abi.TilePlan), _fp, m3]
        L.ref_dense_attention_twin.argtypes = [_fp, _sz, _sz, _P(abi.AttnDesc), _sz, _fp]
        L.ref_lowrank_output_projection.argtypes = [_fp, _sz, _sz, _P(abi.LinearDesc), _fp, m3]
        L.ref_ffn.argtypes = [C.c_int, _fp, _sz, _sz, _sz, _P(abi.FfnDesc), _P(abi.TilePlan),
                              _fp, m3]
        L.ref_run_model.argtypes = [_fp, _sz, _sz, _P(abi.LayerDesc), _sz, C.c_int,
                                    _P(abi.TilePlan), C.c_int, _fp, m3]
        L.ref_run_layer.argtypes = [_fp, _sz, _sz, _P(abi.LayerDesc), C.c_int,
                                    _P(abi.TilePlan), C.c_int, _fp, m3]
        L.ref_validate_tile_plan.argtypes = [_P(abi.TilePlan), C.c_int, _P(abi.Geometry),
                                             _P(_sz)]
        L.ref_save_model.argtypes = [C.c_char_p, _P(abi.LayerDesc), _sz]
        L.ref_read_error_offset.argtypes = [C.c_char_p]
        L.ref_load_model.argtypes = [C.c_char_p, _P(_sz)]
        L.ref_read_error_offset.restype = C.c_longlong
        L.ref_expected_bytes.argtypes = [C.c_int, _P(abi.Geometry)]
        L.ref_expected_bytes.restype = _sz
        L.ref_flops_exact.argtypes = [_P(abi.Geometry), C.c_int]
        L.ref_flops_exact.restype = C.c_ulonglong
        L.ref_factor_rank_r.argtypes = [_fp, _sz, _sz, _sz, _fp, _fp]
        L.ref_io_bytes.argtypes = [_P(abi.Geometry), C.c_int, _P(C.c_ulonglong),
                                   _P(C.c_ulonglong)]
        L.ref_flops_exact_checked.argtypes = [_P(abi.Geometry), C.c_int, _P(C.c_ulonglong)]
        L.ref_decoder_bytes.argtypes = [C.c_int, _P(abi.Geometry), _sz, _P(_sz)]
        L.ref_svd.argtypes = [_fp, _sz, _sz, _fp, _fp, _fp]
        L.ref_factorize_attention.argtypes = [_fp] * 6 + [_sz, _sz, _sz, _fp, _fp, _fp]

    def _chk(self, st):
        if st:
            raise abi.FsvdError(st, self.lib.ref_last_error().decode())

    def attention(self, x, attn, heads, plan, meter=False):
        out = np.zeros_like(x)
        m3 = (_sz * 3)()
        self._chk(self.lib.ref_flash_svd_attention(_f(x), x.shape[0], x.shape[1], attn.desc(),
                                                   heads, plan, _f(out), m3))
        return (out, tuple(m3)) if meter else out

    def dense_attention_twin(self, x, attn, heads):
        out = np.zeros_like(x)
        self._chk(self.lib.ref_dense_attention_twin(_f(x), x.shape[0], x.shape[1], attn.desc(),
                                                    heads, _f(out)))
        return out

    def outproj(self, ctx, lin, meter=False):
        out = np.zeros(ctx.shape[:2] + (lin.v.shape[1],), np.float32)
        m3 = (_sz * 3)()
        self._chk(self.lib.ref_lowrank_output_projection(_f(ctx), ctx.shape[0], ctx.shape[1],
                                                         lin.desc(), _f(out), m3))
        return (out, tuple(m3)) if meter else out

    def ffn(self, variant, x, ffn, plan, meter=False):
        """variant 1/2 = ffn_v1/ffn_v2, 0 = ffn_dense on reconstructed weights,
        3 = ffn_naive_lowrank."""
        out = np.zeros_like(x)
        m3 = (_sz * 3)()
        self._chk(self.lib.ref_ffn(variant, _f(x), x.shape[0], x.shape[1], x.shape[2],
                                   ffn.desc(), plan, _f(out), m3))
        return (out, tuple(m3)) if meter else out

    def run_model(self, x, layers, mode, plan, pre_ln=False, meter=False):
        from paper_2508_01506_b200.model import layer_descs
        out = np.zeros_like(x)
        descs = layer_descs(layers)
        m3 = (_sz * 3)()
        self._chk(self.lib.ref_run_model(_f(x), x.shape[0], x.shape[1], descs, len(layers), mode,
                                         plan, int(pre_ln), _f(out), m3))
        return (out, tuple(m3)) if meter else out

    def validate_tile_plan(self, plan, kind, geom):
        b = _sz(0)
        st = self.lib.ref_validate_tile_plan(plan, kind, geom, C.byref(b))
        return st, b.value

    def expected_bytes(self, formula, geom):
        return self.lib.ref_expected_bytes(formula, geom)

    def flops_exact(self, geom, mode):
        return self.lib.ref_flops_exact(geom, mode)

    def decoder_bytes(self, which, geom, t=0):
        """planner.cpp:123-141 -> (status, bytes); which 0 cache, 1 prefill, 2 step."""
        b = _sz(0)
        st = self.lib.ref_decoder_bytes(which, geom, t, C.byref(b))
        return st, b.value

    def factor_rank_r(self, a, r):
        """svd.cpp:412-456 -> (u [m, r], v [r, n])."""
        a = np.ascontiguousarray(a, np.float32)
        m, n = a.shape
        u = np.zeros((m, r), np.float32)
        v = np.zeros((r, n), np.float32)
        self._chk(self.lib.ref_factor_rank_r(_f(a), m, n, r, _f(u), _f(v)))
        return u, v

    def svd(self, a):
        """svd.cpp:288-302 -> (u [m, p], s [p], vt [p, n])."""
        a = np.ascontiguousarray(a, np.float32)
        m, n = a.shape
        p = min(m, n)
        u = np.zeros((m, p), np.float32)
        s = np.zeros((p,), np.float32)
        vt = np.zeros((p, n), np.float32)
        self._chk(self.lib.ref_svd(_f(a), m, n, _f(u), _f(s), _f(vt)))
        return u, s, vt

    def factorize_attention(self, ws, bs, groups, rank):
        """factorize.cpp:21-64 -> (u [3,G,d,r], v [3,G,r,d/G], bias [3,G,d/G])."""
        d = ws[0].shape[0]
        gd = d // groups
        u = np.zeros((3, groups, d, rank), np.float32)
        v = np.zeros((3, groups, rank, gd), np.float32)
        b = np.zeros((3, groups, gd), np.float32)
        args = []
        for w, bb in zip(ws, bs):
            args += [_f(np.ascontiguousarray(w, np.float32)), _f(np.ascontiguousarray(bb, np.float32))]
        self._chk(self.lib.ref_factorize_attention(*args, d, groups, rank, _f(u), _f(v), _f(b)))
        return u, v, b


def abi_check(st):
    if st:
        raise abi.FsvdError(st, "oracle restatement rejected the call")


# ----------------------------------------------------------------------------
# Seeded factor synthesis, acceptance-style (acceptance.cpp:62-128), drawn
# through the reference's own generator so both sides see identical bits.
# ----------------------------------------------------------------------------
def rand_attn(ora, d, groups, rank, seed):
    """acceptance.cpp:62-83 (rand_attn): seed++ per tensor, q/k/v x groups."""
    from paper_2508_01506_b200.model import AttnFactors
    gd = d // groups
    u = np.empty((3, groups, d, rank), np.float32)
    v = np.empty((3, groups, rank, gd), np.float32)
    b = np.empty((3, groups, gd), np.float32)
    for w in range(3):
        for g in range(groups):
            u[w, g] = ora.random((d, rank), seed, 1.0 / np.sqrt(d)); seed += 1
            v[w, g] = ora.random((rank, gd), seed, 1.0 / np.sqrt(rank)); seed += 1
            b[w, g] = ora.random((gd,), seed, 0.02); seed += 1
    return AttnFactors(u, v, b.reshape(3, d))


def rand_linear(ora, i, o, rank, seed):
    """acceptance.cpp:93-101"""
    from paper_2508_01506_b200.model import LinearFactors
    return LinearFactors(ora.random((i, rank), seed, 1.0 / np.sqrt(i)),
                         ora.random((rank, o), seed + 1, 1.0 / np.sqrt(rank)),
                         ora.random((o,), seed + 2, 0.02))


def rand_ffn(ora, d, df, rank, seed, act=abi.ACT_GELU_ERF):
    """acceptance.cpp:103-110"""
    from paper_2508_01506_b200.model import FfnFactors
    return FfnFactors(rand_linear(ora, d, df, rank, seed),
                      rand_linear(ora, df, d, rank, seed + 10), act)


def rand_layer(ora, d, df, heads, groups, rank, seed, proj_rank=None, ffn_rank=None,
               act=abi.ACT_GELU_ERF):
    """acceptance.cpp:112-128 (rand_layer), with optional separate out-proj /
    FFN ranks (the reference uses one rank for all three)."""
    from paper_2508_01506_b200.model import LayerFactors
    pr = rank if proj_rank is None else proj_rank
    fr = rank if ffn_rank is None else ffn_rank

    def norm(s):
        return ora.random((d,), s, 0.1) + np.float32(1.0), ora.random((d,), s + 1, 0.02)

    g1, b1 = norm(seed + 700)
    g2, b2 = norm(seed + 710)
    return LayerFactors(heads=heads, attn=rand_attn(ora, d, groups, rank, seed),
                        out_proj=rand_linear(ora, d, d, pr, seed + 500),
                        ffn=rand_ffn(ora, d, df, fr, seed + 600, act),
                        ln1_gamma=g1, ln1_beta=b1, ln2_gamma=g2, ln2_beta=b2)
