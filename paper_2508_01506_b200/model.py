"""Host-side containers mirroring the reference's factor types.

``LayerFactors`` is the Python mirror of ``flashsvd::EncoderLayer`` in its
fully factorized form (encoder.hpp:49-67): it owns contiguous fp32 numpy
arrays in the reference orientation and hands out the flat C descriptors of
include/fsvd_b200.h.  No arithmetic happens here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float32)


@dataclass
class LinearFactors:
    """FactorizedLinear (factorize.hpp:13-21): w ~ u (in x r) @ v (r x out)."""
    u: np.ndarray
    v: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        self.u, self.v, self.bias = _c(self.u), _c(self.v), _c(self.bias)

    @property
    def rank(self):
        return self.u.shape[1]

    def desc(self) -> abi.LinearDesc:
        return abi.LinearDesc(self.u.shape[0], self.u.shape[1], self.v.shape[1],
                              abi.fptr(self.u), abi.fptr(self.v), abi.fptr(self.bias))

    def dense(self):
        return self.u.astype(np.float64) @ self.v.astype(np.float64)


@dataclass
class AttnFactors:
    """AttentionFactorSet (factorize.hpp:28-40) with groups stacked:
    u [3, G, d, r], v [3, G, r, d/G], bias [3, d]."""
    u: np.ndarray
    v: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        self.u, self.v, self.bias = _c(self.u), _c(self.v), _c(self.bias)

    @property
    def d_model(self):
        return self.u.shape[2]

    @property
    def groups(self):
        return self.u.shape[1]

    @property
    def rank(self):
        return self.u.shape[3]

    def desc(self) -> abi.AttnDesc:
        return abi.AttnDesc(self.d_model, self.groups, self.rank, abi.fptr(self.u),
                            abi.fptr(self.v), abi.fptr(self.bias))


@dataclass
class FfnFactors:
    up: LinearFactors
    down: LinearFactors
    activation: int = abi.ACT_GELU_ERF

    def desc(self) -> abi.FfnDesc:
        return abi.FfnDesc(self.up.desc(), self.down.desc(), self.activation)


@dataclass
class DenseWeights:
    """DenseAttentionWeights + DenseFfnWeights (encoder.hpp:32-47): weights in
    (in x out) orientation, y = x W + b."""
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

    NAMES = ("wq", "bq", "wk", "bk", "wv", "bv", "wo", "bo", "w_in", "b_in", "w_out", "b_out")

    def __post_init__(self):
        for n in self.NAMES:
            setattr(self, n, _c(getattr(self, n)))
        self._desc = None

    def desc(self) -> abi.DenseLayer:
        if self._desc is None:  # kept alive with the arrays
            self._desc = abi.DenseLayer(self.wq.shape[0], self.w_in.shape[1],
                                        *[abi.fptr(getattr(self, n)) for n in self.NAMES])
        return self._desc

    def arrays(self):
        return [getattr(self, n) for n in self.NAMES]

    @staticmethod
    def of(layer: "LayerFactors") -> "DenseWeights":
        """dense_equivalent (encoder.cpp:295-331): W = U V in fp64, rounded to fp32."""
        a = layer.attn
        G, d, gd = a.groups, a.d_model, a.d_model // a.groups
        w = [np.concatenate([a.u[m, g].astype(np.float64) @ a.v[m, g] for g in range(G)], axis=1)
             for m in range(3)]
        return DenseWeights(w[0], a.bias[0], w[1], a.bias[1], w[2], a.bias[2],
                            layer.out_proj.dense(), layer.out_proj.bias,
                            layer.ffn.up.dense(), layer.ffn.up.bias,
                            layer.ffn.down.dense(), layer.ffn.down.bias)


@dataclass
class LayerFactors:
    heads: int
    attn: AttnFactors
    out_proj: LinearFactors
    ffn: FfnFactors
    ln1_gamma: np.ndarray
    ln1_beta: np.ndarray
    ln2_gamma: np.ndarray
    ln2_beta: np.ndarray
    ln1_eps: float = 1e-5
    ln2_eps: float = 1e-5
    dense: DenseWeights | None = None  # optional dense weights (RunMode::Dense)
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        for n in ("ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta"):
            setattr(self, n, _c(getattr(self, n)))

    @property
    def d_model(self):
        return self.attn.d_model

    @property
    def d_ff(self):
        return self.ffn.up.v.shape[1]

    def desc(self) -> abi.LayerDesc:
        dn = C.pointer(self.dense.desc()) if self.dense is not None else None
        return abi.LayerDesc(self.heads, self.attn.desc(), self.out_proj.desc(), self.ffn.desc(),
                             abi.fptr(self.ln1_gamma), abi.fptr(self.ln1_beta), self.ln1_eps,
                             abi.fptr(self.ln2_gamma), abi.fptr(self.ln2_beta), self.ln2_eps, dn)

    def arrays(self):
        """Every parameter array, for bulk transforms (e.g. bf16 rounding)."""
        return [self.attn.u, self.attn.v, self.attn.bias, self.out_proj.u, self.out_proj.v,
                self.out_proj.bias, self.ffn.up.u, self.ffn.up.v, self.ffn.up.bias,
                self.ffn.down.u, self.ffn.down.v, self.ffn.down.bias, self.ln1_gamma,
                self.ln1_beta, self.ln2_gamma, self.ln2_beta] + (
                    self.dense.arrays() if self.dense is not None else [])


@dataclass
class DenseLayer:
    """An EncoderLayer carrying only dense weights (encoder.hpp:49-67 with
    attn_factors / out_proj / ffn_factors empty): runs in RunMode::Dense."""
    heads: int
    dense: DenseWeights
    ln1_gamma: np.ndarray
    ln1_beta: np.ndarray
    ln2_gamma: np.ndarray
    ln2_beta: np.ndarray
    activation: int = abi.ACT_GELU_ERF
    ln1_eps: float = 1e-5
    ln2_eps: float = 1e-5

    def __post_init__(self):
        for n in ("ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta"):
            setattr(self, n, _c(getattr(self, n)))

    @property
    def d_model(self):
        return self.dense.wq.shape[0]

    def desc(self) -> abi.LayerDesc:
        d = self.d_model
        empty = abi.LinearDesc(0, 0, 0, None, None, None)
        return abi.LayerDesc(self.heads, abi.AttnDesc(d, 0, 0, None, None, None), empty,
                             abi.FfnDesc(empty, empty, self.activation),
                             abi.fptr(self.ln1_gamma), abi.fptr(self.ln1_beta), self.ln1_eps,
                             abi.fptr(self.ln2_gamma), abi.fptr(self.ln2_beta), self.ln2_eps,
                             C.pointer(self.dense.desc()))

    def arrays(self):
        return self.dense.arrays() + [self.ln1_gamma, self.ln1_beta, self.ln2_gamma, self.ln2_beta]


def layer_descs(layers):
    """Contiguous LayerDesc array for fsvd_run_model."""
    arr = (abi.LayerDesc * len(layers))()
    for i, L in enumerate(layers):
        arr[i] = L.desc()
    return arr


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (RNE) and return them as fp32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    rounding = ((bits >> 16) & 1) + 0x7FFF
    out = ((bits + rounding) >> 16 << 16).astype(np.uint32)
    nan = np.isnan(a)
    out[nan] = 0x7FC00000
    return out.view(np.float32).reshape(a.shape)


def round_layer_bf16(layer: LayerFactors) -> LayerFactors:
    """In-place bf16 rounding of every parameter (bf16 parity protocol)."""
    for a in layer.arrays():
        a[...] = bf16_round(a)
    return layer


def random_layer(d, df, heads, groups, rank, proj_rank, ffn_rank, rng: np.random.Generator,
                 activation=abi.ACT_GELU_ERF) -> LayerFactors:
    """Acceptance-style random factors (acceptance.cpp:62-128 statistics):
    U ~ N(0, 1/sqrt(in)), V ~ N(0, 1/sqrt(r)), bias ~ N(0, 0.02),
    gamma = 1 + N(0, 0.1), beta ~ N(0, 0.02).  numpy RNG (bench data)."""
    gd = d // groups
    f32 = np.float32

    def lin(i, o, r):
        return LinearFactors(rng.standard_normal((i, r), f32) / np.sqrt(i),
                             rng.standard_normal((r, o), f32) / np.sqrt(r),
                             rng.standard_normal((o,), f32) * 0.02)

    attn = AttnFactors(rng.standard_normal((3, groups, d, rank), f32) / np.sqrt(d),
                       rng.standard_normal((3, groups, rank, gd), f32) / np.sqrt(rank),
                       rng.standard_normal((3, d), f32) * 0.02)
    return LayerFactors(
        heads=heads, attn=attn, out_proj=lin(d, d, proj_rank),
        ffn=FfnFactors(lin(d, df, ffn_rank), lin(df, d, ffn_rank), activation),
        ln1_gamma=1 + rng.standard_normal((d,), f32) * 0.1,
        ln1_beta=rng.standard_normal((d,), f32) * 0.02,
        ln2_gamma=1 + rng.standard_normal((d,), f32) * 0.1,
        ln2_beta=rng.standard_normal((d,), f32) * 0.02)
