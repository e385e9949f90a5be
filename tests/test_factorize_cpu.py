"""CPU: host logic of the device factorizer -- argument
checks with the reference's error kinds and messages (svd.cpp:412-416,
factorize.cpp:25-39, model_io.cpp:482-499), rank-default resolution, the
no-CPU-fallback rule -- and the pinning of the reference factorization entry
points the GPU tests compare against."""
import numpy as np
import pytest

from paper_2508_01506_b200 import abi
from paper_2508_01506_b200 import factorize as F

L = abi.lib()


def _err(fn, *a):
    with pytest.raises(abi.FsvdError) as e:
        fn(*a)
    return e.value


def test_factor_rank_r_rank_errors():
    a = np.ones((4, 6), np.float32)
    e = _err(F.factor_rank_r, a, 0)
    assert e.status == abi.ERR_RANK and "at least 1" in str(e)
    e = _err(F.factor_rank_r, a, 5)
    assert e.status == abi.ERR_RANK and "exceeds min(m, n)" in str(e)
    e = _err(F.factor_rank_r_batch, [a, a], [2, 7])
    assert e.status == abi.ERR_RANK


def test_factorize_attention_geometry_errors():
    w = np.zeros((12, 12), np.float32)
    b = np.zeros((12,), np.float32)
    e = _err(F.factorize_attention, w, b, w, b, w, b, 5, 2)
    assert e.status == abi.ERR_CONFIG and "groups must divide" in str(e)
    e = _err(F.factorize_attention, w, b, w, b, w, b, 4, 0)
    assert e.status == abi.ERR_RANK
    e = _err(F.factorize_attention, w, b, w, b, w, b, 4, 4)
    assert e.status == abi.ERR_RANK and "per-group width" in str(e)
    e = _err(F.factorize_attention, np.zeros((12, 8), np.float32), b, w, b, w, b, 4, 2)
    assert e.status == abi.ERR_SHAPE


def test_rank_defaults_follow_synth_model():
    # model_io.cpp:489-496: rank 0 -> d/G; pr -> min(rG, d); fr -> min(pr, d, df)
    assert F.resolve_ranks(768, 3072, 12) == (64, 768, 768)
    assert F.resolve_ranks(768, 3072, 12, rank=32) == (32, 384, 384)   # SURVEY cfg2
    assert F.resolve_ranks(1024, 4096, 16, rank=32) == (32, 512, 512)  # SURVEY cfg3
    assert F.resolve_ranks(64, 32, 4, rank=16) == (16, 64, 32)
    e = _err(F.resolve_ranks, 768, 3072, 12, 32, 800)
    assert e.status == abi.ERR_RANK and "proj_rank exceeds d_model" in str(e)
    e = _err(F.resolve_ranks, 64, 32, 4, 16, 64, 48)
    assert e.status == abi.ERR_RANK and "ffn_rank exceeds" in str(e)
    e = _err(F.resolve_ranks, 768, 3072, 7)
    assert e.status == abi.ERR_CONFIG


def test_no_cpu_fallback():
    if L.fsvd_device_available():
        pytest.skip("GPU present")
    e = _err(F.factor_rank_r, np.eye(4, dtype=np.float32), 2)
    assert e.status == abi.ERR_CUDA and "no CPU fallback" in str(e)


def test_reference_factorization_pinned(reference):
    """The compiled reference entry points reproduce the reference's own
    known answers (test_tensor.cpp:207-213 rank-1 recovery, 276-287 direct
    factorization == truncated full SVD, 289-294 zero matrix)."""
    a = np.array([[2, 1], [4, 2], [6, 3]], np.float32)
    u, v = reference.factor_rank_r(a, 1)
    assert np.abs(u @ v - a).max() < 1e-5
    for m, n, r in [(8, 8, 3), (40, 8, 4), (8, 40, 4), (20, 12, 5), (64, 16, 16)]:
        x = np.random.default_rng(m * 100 + n).standard_normal((m, n)).astype(np.float32)
        u, v = reference.factor_rank_r(x, r)
        fu, fs, fvt = reference.svd(x)
        root = np.sqrt(fs[:r].astype(np.float64))
        assert np.abs(u - (fu[:, :r] * root).astype(np.float32)).max() < 1e-5
        assert np.abs(v - (root[:, None] * fvt[:r]).astype(np.float32)).max() < 1e-5
    u, v = reference.factor_rank_r(np.zeros((6, 4), np.float32), 2)
    assert not u.any() and not v.any()
