"""Layers carrying dense weights (encoder.hpp:32-67: DenseAttentionWeights /
DenseFfnWeights) through the host drop-in: RunMode::Dense runs the layer's own
dense weights on the tensor cores (materialised Q|K|V, the attention kernel
with r = head width padded to 16/32/64, dense FFN GEMMs), in both precision
policies; a dense-only layer in a flash / naive mode is refused with the
reference's error (encoder.cpp:27-35).  The oracle is the compiled reference
run on the same descriptors (oracle/_ref, ref_capi.cpp layer_of).

Tolerances (north star): fp32 policy <= 1e-4 relative, bf16 <= 2e-2 against
the reference fed the same bf16-rounded values.
"""
import numpy as np
import pytest

import oracle
from paper_2508_01506_b200 import abi
from paper_2508_01506_b200.model import DenseLayer, DenseWeights, bf16_round

import helpers as H

PLAN = abi.TilePlan(16, 16, 64, 1 << 22)


def rand_dense_layer(ora, d, df, heads, seed, act=abi.ACT_GELU_ERF):
    s = seed

    def t(shape, std):
        nonlocal s
        s += 1
        return ora.random(shape, s, std)
    w = DenseWeights(t((d, d), d ** -0.5), t((d,), 0.02), t((d, d), d ** -0.5), t((d,), 0.02),
                     t((d, d), d ** -0.5), t((d,), 0.02), t((d, d), d ** -0.5), t((d,), 0.02),
                     t((d, df), d ** -0.5), t((df,), 0.02), t((df, d), df ** -0.5), t((d,), 0.02))
    return DenseLayer(heads, w, t((d,), 0.1) + np.float32(1), t((d,), 0.02),
                      t((d,), 0.1) + np.float32(1), t((d,), 0.02), act)


def prep(layer, x, dtype):
    if dtype == abi.BF16:
        for a in layer.arrays():
            a[...] = bf16_round(a)
        x = bf16_round(x)
    return layer, x


def tol(dtype):
    return H.TOL_F32 if dtype == abi.F32 else H.TOL_BF16


# d, df, heads (head width 64, 16, 12 -> padded 16, 48 -> padded 64, 4 -> padded 16)
SHAPES = [(256, 512, 4), (128, 256, 8), (96, 192, 8), (192, 384, 4), (32, 64, 8)]


@pytest.mark.gpu
@pytest.mark.parametrize("shape", SHAPES, ids=[f"d{s[0]}_h{s[2]}" for s in SHAPES])
@pytest.mark.parametrize("dtype", [abi.F32, abi.BF16], ids=["f32", "bf16"])
def test_dense_only_layer_matches_reference(reference, shape, dtype):
    d, df, heads = shape
    layer = rand_dense_layer(reference, d, df, heads, 100 + d)
    x = reference.random((2, 70, d), 9)
    layer, x = prep(layer, x, dtype)
    for pre in (False, True):
        ref = reference.run_model(x, [layer], abi.MODE_DENSE, PLAN, pre_ln=pre)
        got = H.run_layer(x, layer, abi.MODE_DENSE, PLAN, dtype, pre_ln=pre)
        e = H.rel_err(got, ref)
        H.record(f"dense_only_{'pre' if pre else 'post'}", f"d{d}_h{heads}", dtype, e)
        assert e <= tol(dtype), (pre, e)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [abi.F32, abi.BF16], ids=["f32", "bf16"])
def test_layer_with_both_representations_uses_dense_weights(reference, restatement, dtype):
    """A layer carrying factors AND (different) dense weights: Dense mode must
    run the dense weights, the flash modes the factors -- as the reference's
    attention_sublayer / ffn_sublayer switch does (encoder.cpp:82-139)."""
    layer = oracle.rand_layer(restatement, 256, 512, 4, 4, 32, 61, 64, 128)
    other = rand_dense_layer(reference, 256, 512, 4, 62)
    layer.dense = other.dense
    x = reference.random((2, 64, 256), 10)
    if dtype == abi.BF16:
        for a in layer.arrays():
            a[...] = bf16_round(a)
        x = bf16_round(x)
    ref_dense = reference.run_model(x, [layer], abi.MODE_DENSE, PLAN)
    ref_flash = reference.run_model(x, [layer], abi.MODE_FLASH_V2, PLAN)
    assert H.rel_err(ref_dense, ref_flash) > 0.1  # the two representations differ
    assert H.rel_err(H.run_layer(x, layer, abi.MODE_DENSE, PLAN, dtype), ref_dense) <= tol(dtype)
    assert H.rel_err(H.run_layer(x, layer, abi.MODE_FLASH_V2, PLAN, dtype), ref_flash) <= tol(dtype)


@pytest.mark.gpu
def test_dense_twin_of_factor_only_layer(reference, restatement):
    """C-ABI extension: a factor-only layer in MODE_DENSE runs its dense twin
    (dense_equivalent, encoder.cpp:295-331) -- the same numbers as giving the
    reconstructed weights explicitly."""
    layer = oracle.rand_layer(restatement, 256, 512, 4, 4, 32, 63, 64, 128)
    x = reference.random((2, 64, 256), 11)
    twin = H.run_layer(x, layer, abi.MODE_DENSE, PLAN, abi.F32)
    layer.dense = DenseWeights.of(layer)
    explicit = H.run_layer(x, layer, abi.MODE_DENSE, PLAN, abi.F32)
    ref = reference.run_model(x, [layer], abi.MODE_DENSE, PLAN)
    assert H.rel_err(twin, ref) <= H.TOL_F32 and H.rel_err(explicit, ref) <= H.TOL_F32


@pytest.mark.parametrize("mode", [abi.MODE_FLASH_V1, abi.MODE_FLASH_V2, abi.MODE_NAIVE_LOWRANK],
                         ids=["v1", "v2", "naive"])
def test_dense_only_layer_refused_in_factor_modes(reference, mode):
    """encoder.cpp:27-35: the same ConfigError and message as the reference
    (no device needed: the checks run before any upload)."""
    layer = rand_dense_layer(reference, 64, 128, 4, 7)
    x = reference.random((1, 8, 64), 12)
    with pytest.raises(abi.FsvdError) as ours:
        H.run_layer(x, layer, mode, PLAN, abi.F32)
    with pytest.raises(abi.FsvdError) as ref:
        reference.run_model(x, [layer], mode, PLAN)
    assert ours.value.status == ref.value.status == abi.ERR_CONFIG
    name = {abi.MODE_FLASH_V1: "flash_v1", abi.MODE_FLASH_V2: "flash_v2",
            abi.MODE_NAIVE_LOWRANK: "naive_lowrank"}[mode]
    assert f"{name} mode needs factorized weights on both sublayers" in str(ours.value)
    assert f"{name} mode needs factorized weights on both sublayers" in str(ref.value)
