"""Python mirror of the reference's factorization API over the device
factorizer.

``factor_rank_r`` (svd.cpp:412), ``factorize_attention`` (factorize.cpp:21)
and ``factorize_layers`` (the factorization step of model_io.cpp:486-533
``synth_model``) call the C-ABI entry points of libfsvd_b200.so; every matrix
of a call is factorized in one batched device run.  Errors surface as
``abi.FsvdError`` carrying the reference's error kind and message.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import abi
from .model import AttnFactors, FfnFactors, LayerFactors, LinearFactors


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def factor_rank_r(a, rank: int):
    """Leading-r even-split factors: a (m x n) ~ u (m x r) @ v (r x n)."""
    L = abi.lib()
    a = _c(a)
    m, n = a.shape
    u = np.zeros((m, rank), np.float32)
    v = np.zeros((rank, n), np.float32)
    abi.check(L.fsvd_factor_rank_r(abi.fptr(a), m, n, rank, abi.fptr(u), abi.fptr(v)))
    return u, v


def factor_rank_r_batch(mats, ranks):
    """Factorizes every (matrix, rank) pair in one device run."""
    L = abi.lib()
    mats = [_c(a) for a in mats]
    outs = [(np.zeros((a.shape[0], r), np.float32), np.zeros((r, a.shape[1]), np.float32))
            for a, r in zip(mats, ranks)]
    jobs = (abi.FactorJob * len(mats))()
    for i, (a, r) in enumerate(zip(mats, ranks)):
        jobs[i] = abi.FactorJob(abi.fptr(a), a.shape[0], a.shape[1], r, abi.fptr(outs[i][0]),
                                abi.fptr(outs[i][1]))
    abi.check(L.fsvd_factor_rank_r_batch(jobs, len(mats)))
    return outs


def factorize_attention(wq, bq, wk, bk, wv, bv, groups: int, rank: int) -> AttnFactors:
    """Per-group factors of the three d x d projections (q, k, v order)."""
    L = abi.lib()
    ws = [_c(w) for w in (wq, wk, wv)]
    bs = [_c(b) for b in (bq, bk, bv)]
    d = ws[0].shape[0]
    for w in ws:
        if w.shape != (d, d):
            raise abi.FsvdError(abi.ERR_SHAPE, "attention projections must be square d_model x d_model")
    for b in bs:
        if b.shape != (d,):
            raise abi.FsvdError(abi.ERR_SHAPE, "attention bias length must be d_model")
    gd = d // groups if groups else 0
    u = np.zeros((3, groups, d, rank), np.float32)
    v = np.zeros((3, groups, rank, max(gd, 1)), np.float32)
    bias = np.zeros((3, d), np.float32)
    abi.check(L.fsvd_factorize_attention(abi.fptr(ws[0]), abi.fptr(bs[0]), abi.fptr(ws[1]),
                                         abi.fptr(bs[1]), abi.fptr(ws[2]), abi.fptr(bs[2]), d,
                                         groups, rank, abi.fptr(u), abi.fptr(v), abi.fptr(bias)))
    return AttnFactors(u, v, bias)


@dataclass
class DenseLayerWeights:
    """DenseAttentionWeights + DenseFfnWeights (encoder.hpp:32-47), (in x out)."""
    wq: np.ndarray
    bq: np.ndarray
    wk: np.ndarray
    bk: np.ndarray
    wv: np.ndarray
    bv: np.ndarray
    wo: np.ndarray
    bo: np.ndarray
    w_in: np.ndarray
    b_in: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray

    def __post_init__(self):
        for k, v in self.__dict__.items():
            setattr(self, k, _c(v))

    def desc(self) -> abi.DenseLayer:
        d, df = self.w_in.shape
        return abi.DenseLayer(d, df, *[abi.fptr(getattr(self, n)) for n in (
            "wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "w_in", "b_in", "w_out", "b_out")])


def resolve_ranks(d, df, groups, rank=0, proj_rank=0, ffn_rank=0, n_layers=1):
    """model_io.cpp:489-499 rank defaults and checks, through the C ABI."""
    L = abi.lib()
    f = np.zeros((1,), np.float32)
    fp = abi.fptr(f)
    dl = (abi.DenseLayer * n_layers)(*[abi.DenseLayer(d, df, *([fp] * 12))] * n_layers)
    r, pr, fr = abi._sz(rank), abi._sz(proj_rank), abi._sz(ffn_rank)
    abi.check(L.fsvd_factorize_layers(dl, n_layers, groups, r, pr, fr, None))
    return r.value, pr.value, fr.value


def factorize_layers(dense, heads: int, groups: int = 0, rank: int = 0, proj_rank: int = 0,
                     ffn_rank: int = 0, activation: int = abi.ACT_GELU_ERF):
    """Dense layers -> LayerFactors with identity LayerNorms (model_io.cpp:371-376,
    524-533), every matrix of every layer factorized in one device run."""
    L = abi.lib()
    groups = groups or heads
    d, df = dense[0].w_in.shape
    r, pr, fr = resolve_ranks(d, df, groups, rank, proj_rank, ffn_rank, len(dense))
    gd = d // groups
    outs, bufs = [], (abi.FactorBuffers * len(dense))()
    for i in range(len(dense)):
        o = dict(attn_u=np.zeros((3, groups, d, r), np.float32),
                 attn_v=np.zeros((3, groups, r, gd), np.float32),
                 attn_b=np.zeros((3, d), np.float32),
                 out_u=np.zeros((d, pr), np.float32), out_v=np.zeros((pr, d), np.float32),
                 out_b=np.zeros((d,), np.float32),
                 up_u=np.zeros((d, fr), np.float32), up_v=np.zeros((fr, df), np.float32),
                 up_b=np.zeros((df,), np.float32),
                 down_u=np.zeros((df, fr), np.float32), down_v=np.zeros((fr, d), np.float32),
                 down_b=np.zeros((d,), np.float32))
        outs.append(o)
        bufs[i] = abi.FactorBuffers(*[abi.fptr(o[k]) for k in (
            "attn_u", "attn_v", "attn_b", "out_u", "out_v", "out_b", "up_u", "up_v", "up_b",
            "down_u", "down_v", "down_b")])
    dl = (abi.DenseLayer * len(dense))(*[w.desc() for w in dense])
    rr, prr, frr = abi._sz(r), abi._sz(pr), abi._sz(fr)
    abi.check(L.fsvd_factorize_layers(dl, len(dense), groups, rr, prr, frr, bufs))
    layers = []
    for o in outs:
        layers.append(LayerFactors(
            heads, AttnFactors(o["attn_u"], o["attn_v"], o["attn_b"]),
            LinearFactors(o["out_u"], o["out_v"], o["out_b"]),
            FfnFactors(LinearFactors(o["up_u"], o["up_v"], o["up_b"]),
                       LinearFactors(o["down_u"], o["down_v"], o["down_b"]), activation),
            np.ones(d, np.float32), np.zeros(d, np.float32),
            np.ones(d, np.float32), np.zeros(d, np.float32)))
    return layers
