"""GPU: the batched device factorizer against the
compiled reference (oracle/_ref: svd.cpp factor_rank_r, factorize.cpp
factorize_attention) on the same inputs.

Tolerance: 1e-5 absolute on the fp32 factors -- the reference's own bar for
two different Jacobi schedules of the same matrix (test_tensor.cpp:276-287,
direct factorization vs truncated full SVD).  Both sides compute in fp64; the
factors agree to fp32 rounding unless singular values are (near) repeated.
"""
import numpy as np
import pytest

from paper_2508_01506_b200 import abi
from paper_2508_01506_b200 import factorize as F
from paper_2508_01506_b200.model import layer_descs

import helpers as H

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def L():
    lib = abi.lib()
    if not lib.fsvd_device_available():
        pytest.fail("GPU tests need an sm_100 device: " + lib.fsvd_last_error().decode())
    return lib


def _rand(shape, seed, scale=1.0):
    return (np.random.default_rng(seed).standard_normal(shape) * scale).astype(np.float32)


def _close(got, ref):
    return float(np.abs(got - ref).max())


def test_reference_cases_and_random_shapes(L, reference):
    cases = [(8, 8, 3), (40, 8, 4), (8, 40, 4), (20, 12, 5), (64, 16, 16), (1, 1, 1), (1, 7, 1),
             (9, 1, 1), (33, 33, 33)]
    rng = np.random.default_rng(7)
    for _ in range(40):
        m, n = int(rng.integers(1, 48)), int(rng.integers(1, 48))
        cases.append((m, n, int(rng.integers(1, min(m, n) + 1))))
    mats = [_rand((m, n), 100 + i) for i, (m, n, r) in enumerate(cases)]
    outs = F.factor_rank_r_batch(mats, [c[2] for c in cases])  # one device run
    for a, (m, n, r), (u, v) in zip(mats, cases, outs):
        ru, rv = reference.factor_rank_r(a, r)
        assert _close(u, ru) < TOL and _close(v, rv) < TOL, (m, n, r)
    # the single-matrix entry point gives the same bits as the batch
    u, v = F.factor_rank_r(mats[3], cases[3][2])
    assert np.array_equal(u, outs[3][0]) and np.array_equal(v, outs[3][1])


def test_rank_deficient_and_zero(L, reference):
    a = np.array([[2, 1], [4, 2], [6, 3]], np.float32)  # test_tensor.cpp:207-213
    u, v = F.factor_rank_r(a, 1)
    assert np.abs(u @ v - a).max() < 1e-5
    u, v = F.factor_rank_r(np.zeros((6, 4), np.float32), 2)  # test_tensor.cpp:289-294
    assert not u.any() and not v.any()
    # exact rank 3 in 30 x 20, asked for rank 5: the two tail factors are zero
    b = _rand((30, 3), 1) @ _rand((3, 20), 2)
    u, v = F.factor_rank_r(b, 5)
    ru, rv = reference.factor_rank_r(b, 5)
    assert _close(u @ v, b) < 1e-4
    assert _close(u[:, :3], ru[:, :3]) < TOL and _close(v[:3], rv[:3]) < TOL
    assert np.abs(u[:, 3:]).max() < 1e-3 and np.abs(ru[:, 3:]).max() < 1e-3


def test_bert_base_shapes_match_reference(L, reference):
    """BERT-Base blocks: a per-head q block (768 x 64, r 32), the output
    projection (768 x 768, pr 384), FFN up (768 x 3072) and down (3072 x 768)
    at fr 384 -- all four in one batch, each against the reference."""
    shapes = [(768, 64, 32), (768, 768, 384), (768, 3072, 384), (3072, 768, 384)]
    mats = [_rand((m, n), 11 + i, 1 / np.sqrt(m)) for i, (m, n, r) in enumerate(shapes)]
    outs = F.factor_rank_r_batch(mats, [s[2] for s in shapes])
    for a, (m, n, r), (u, v) in zip(mats, shapes, outs):
        ru, rv = reference.factor_rank_r(a, r)
        assert _close(u, ru) < TOL and _close(v, rv) < TOL, (m, n, r, _close(u, ru), _close(v, rv))
    assert 0 < L.fsvd_last_factor_sweeps() <= 60


def test_very_tall_uses_row_split_clusters(L, reference):
    """M = 6001 rows need 8-CTA clusters (row slices of 752) and uneven
    padding; wide orientation of the same shape goes through A^T."""
    a = _rand((6001, 40), 3, 0.01)
    b = _rand((37, 5003), 4)
    (u, v), (u2, v2) = F.factor_rank_r_batch([a, b], [8, 30])
    ru, rv = reference.factor_rank_r(a, 8)
    assert _close(u, ru) < TOL and _close(v, rv) < TOL
    ru, rv = reference.factor_rank_r(b, 30)
    assert _close(u2, ru) < TOL and _close(v2, rv) < TOL


def test_deterministic(L):
    a = _rand((300, 200), 5)
    u1, v1 = F.factor_rank_r(a, 50)
    u2, v2 = F.factor_rank_r(a, 50)
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2)


def test_factorize_attention_matches_reference(L, reference):
    d, G, r = 256, 4, 16
    ws = [_rand((d, d), 20 + i, 1 / np.sqrt(d)) for i in range(3)]
    bs = [_rand((d,), 30 + i, 0.02) for i in range(3)]
    got = F.factorize_attention(ws[0], bs[0], ws[1], bs[1], ws[2], bs[2], G, r)
    ru, rv, rb = reference.factorize_attention(ws, bs, G, r)
    assert _close(got.u, ru) < TOL and _close(got.v, rv) < TOL
    assert np.array_equal(got.bias, rb.reshape(3, d))


def test_factorize_layers_runs_the_encoder(L, reference):
    """Dense layers -> factors on the device -> encoder forward: every matrix
    equals the reference's factorization, and the model run on the device
    factors equals the reference run on the same factors (fp32 policy)."""
    d, df, heads, r = 256, 1024, 4, 32
    dense = []
    for l in range(2):
        s = 1000 * l
        dense.append(F.DenseLayerWeights(
            _rand((d, d), s + 1, d ** -0.5), _rand((d,), s + 2, .02),
            _rand((d, d), s + 3, d ** -0.5), _rand((d,), s + 4, .02),
            _rand((d, d), s + 5, d ** -0.5), _rand((d,), s + 6, .02),
            _rand((d, d), s + 7, d ** -0.5), _rand((d,), s + 8, .02),
            _rand((d, df), s + 9, d ** -0.5), _rand((df,), s + 10, .02),
            _rand((df, d), s + 11, d ** -0.5), _rand((d,), s + 12, .02)))
    layers = F.factorize_layers(dense, heads, rank=r)
    assert layers[0].attn.rank == r and layers[0].out_proj.rank == 128
    assert layers[0].ffn.up.rank == 128
    for w, lay in zip(dense, layers):
        ru, rv, _ = reference.factorize_attention([w.wq, w.wk, w.wv], [w.bq, w.bk, w.bv], heads, r)
        assert _close(lay.attn.u, ru) < TOL and _close(lay.attn.v, rv) < TOL
        for mat, lin in ((w.wo, lay.out_proj), (w.w_in, lay.ffn.up), (w.w_out, lay.ffn.down)):
            u, v = reference.factor_rank_r(mat, lin.rank)
            assert _close(lin.u, u) < TOL and _close(lin.v, v) < TOL
        assert np.array_equal(lay.out_proj.bias, w.bo) and np.array_equal(lay.ffn.up.bias, w.b_in)
    x = _rand((2, 64, d), 77)
    plan = abi.TilePlan(16, 16, 64, 1 << 22)
    got = H.run_model(x, layers, abi.MODE_FLASH_V2, plan, abi.F32)
    ref = reference.run_model(x, layers, abi.MODE_FLASH_V2, plan)
    assert H.rel_err(got, ref) <= H.TOL_F32
