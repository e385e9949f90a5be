"""CPU: the oracle restatement is pinned against the compiled reference and
the committed golden vectors; closed forms match the reference."""
import os

import numpy as np
import pytest

import oracle
from paper_2508_01506_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden.npz")
PLAN = abi.TilePlan(16, 16, 64, 1 << 20)


def test_generator_pinned_by_golden(restatement):
    g = np.load(GOLDEN)
    assert np.array_equal(restatement.random((64,), 5, 1.0), g["gaussian_seed5"])
    assert np.array_equal(restatement.random((64,), 9, 0.02), g["gaussian_seed9_sd02"])


def test_generator_matches_reference(restatement, reference):
    for seed, sd in [(1, 1.0), (2, 0.02), (123456789, 0.3)]:
        assert np.array_equal(restatement.random((1001,), seed, sd), reference.random((1001,), seed, sd))


@pytest.mark.parametrize("case", [
    "attn_g2_r5", "attn_g1_r7", "attn_per_head_r8", "outproj_r6", "ffn_v1_gelu", "ffn_v2_tanh",
    "ffn_v1_relu", "ffn_v2_identity", "layer_v1_post", "layer_v2_pre", "model2_v1"])
def test_restatement_matches_golden_bitwise(restatement, case):
    import importlib.util
    spec = importlib.util.spec_from_file_location("mk", os.path.join(HERE, "golden", "make_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    c = [c for c in mk.CASES if c[0] == case][0]
    _, got = mk.make_case(restatement, c)
    assert np.array_equal(got, np.load(GOLDEN)[case]), case


def _rand_attn_case(rng):
    # acceptance.cpp:216-248 shape distribution, smaller
    b = int(rng.integers(1, 4)); m = int(rng.integers(1, 70)); heads = int(rng.integers(1, 9))
    gd = int(rng.choice([4, 8, 16, 32]))
    d = heads * gd
    divs = [g for g in range(1, heads + 1) if heads % g == 0]
    groups = int(rng.choice(divs))
    rank = int(rng.integers(1, min(64, d // groups) + 1))
    return b, m, heads, d, groups, rank


def test_restatement_bitexact_attention_random(restatement, reference):
    rng = np.random.default_rng(4242)
    for t in range(25):
        b, m, heads, d, groups, rank = _rand_attn_case(rng)
        a = oracle.rand_attn(reference, d, groups, rank, 100000 + t * 631)
        x = reference.random((b, m, d), 50000 + t)
        plan = abi.TilePlan(int(rng.choice([8, 16, 32])), int(rng.choice([4, 8, 16])), 64, 1 << 22)
        assert np.array_equal(restatement.attention(x, a, heads, plan),
                              reference.attention(x, a, heads, plan)), t


def test_restatement_bitexact_ffn_random(restatement, reference):
    rng = np.random.default_rng(77)
    for t in range(25):
        b = int(rng.integers(1, 4)); m = int(rng.integers(1, 40)); d = int(rng.integers(4, 48))
        df = int(rng.integers(8, 96)); rank = int(rng.integers(1, min(d, df) + 1))
        f = oracle.rand_ffn(reference, d, df, rank, 300000 + t * 97, t % 4)
        x = reference.random((b, m, d), 70000 + t)
        plan = abi.TilePlan(int(rng.choice([8, 16])), 16, int(rng.choice([16, 32, 64])), 1 << 22)
        for v in (1, 2):
            assert np.array_equal(restatement.ffn(v, x, f, plan), reference.ffn(v, x, f, plan)), (t, v)


@pytest.mark.parametrize("mode", [abi.MODE_FLASH_V1, abi.MODE_FLASH_V2])
@pytest.mark.parametrize("pre_ln", [False, True])
def test_restatement_bitexact_model(restatement, reference, mode, pre_ln):
    layers = [oracle.rand_layer(reference, 48, 144, 4, 2 if i else 4, 6, 800000 + i * 1013, 10, 12)
              for i in range(3)]
    x = reference.random((2, 21, 48), 90000)
    assert np.array_equal(restatement.run_model(x, layers, mode, PLAN, pre_ln),
                          reference.run_model(x, layers, mode, PLAN, pre_ln))


def test_flash_modes_bitwise_equal_in_reference(reference):
    # ffn_v1 and ffn_v2 are bitwise equal in the reference
    f = oracle.rand_ffn(reference, 40, 100, 9, 5, abi.ACT_GELU_ERF)
    x = reference.random((2, 30, 40), 6)
    assert np.array_equal(reference.ffn(1, x, f, PLAN), reference.ffn(2, x, f, PLAN))


def test_streaming_matches_dense_twin_reference(reference):
    # acceptance criterion 4 (kKernelTol = 1e-4) on a few cases
    for t in range(4):
        a = oracle.rand_attn(reference, 64, 4, 8, 7 + t)
        x = reference.random((2, 40, 64), 9 + t)
        got = reference.attention(x, a, 8, PLAN)
        ref = reference.dense_attention_twin(x, a, 8)
        assert np.abs(got - ref).max() <= 1e-4


GEOMS = [abi.Geometry(b, m, d, df, h, g, r, 1)
         for (b, m, d, df, h, g, r) in [(1, 128, 768, 3072, 12, 12, 64), (2, 64, 128, 512, 4, 4, 16),
                                        (1, 8, 32, 64, 2, 2, 4), (8, 128, 768, 3072, 12, 1, 32),
                                        (32, 512, 768, 3072, 12, 12, 32)]]


@pytest.mark.parametrize("geom", GEOMS)
def test_closed_forms_match_reference(restatement, reference, geom):
    for f in range(8):
        assert restatement.lib.fo_expected_bytes(f, geom) == reference.expected_bytes(f, geom)


@pytest.mark.parametrize("kind", [abi.KERNEL_ATTENTION, abi.KERNEL_FFN_V1, abi.KERNEL_FFN_V2])
def test_working_set_matches_reference(restatement, reference, kind):
    import ctypes as C
    for plan in [abi.TilePlan(16, 16, 64, 131072), abi.TilePlan(16, 16, 32, 1 << 20),
                 abi.TilePlan(64, 4, 16, 4096), abi.TilePlan(0, 16, 16, 1 << 20)]:
        for geom in GEOMS:
            st_ref, b_ref = reference.validate_tile_plan(plan, kind, geom)
            st = C.c_int()
            b = restatement.lib.fo_tile_working_set(plan, kind, geom, C.byref(st))
            assert st.value == st_ref
            if st_ref == 0:
                assert b == b_ref
