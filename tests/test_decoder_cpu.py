"""CPU: decoder closed forms bit-exact against the
compiled reference (planner.cpp:123-141), including its error behaviour."""
import itertools

import pytest

from paper_2508_01506_b200 import abi

L = abi.lib()


def _mine(which, g, t=0):
    b = abi._sz(0)
    if which == 0:
        st = L.fsvd_decoder_kv_cache_bytes(g, b)
    elif which == 1:
        st = L.fsvd_decoder_prefill_bytes(g, b)
    else:
        st = L.fsvd_decoder_decode_step_bytes(g, t, b)
    return st, b.value


def test_decoder_closed_forms_match_reference(reference):
    n = 0
    for B, M, d, H, r, layers in itertools.product((1, 3, 32), (1, 17, 512), (64, 768), (4, 12),
                                                    (1, 8, 64), (0, 1, 12)):
        g = abi.Geometry(B, M, d, 4 * d, H, H, r, layers)
        for which in (0, 1):
            ref = reference.decoder_bytes(which, g)
            assert _mine(which, g) == ref, (which, B, M, d, H, r, layers)
        for t in (0, 1, M // 2 + 1, M, M + 1):
            assert _mine(2, g, t) == reference.decoder_bytes(2, g, t), (t, B, M, r, layers)
            n += 1
    assert n > 300


def test_decoder_closed_form_errors():
    g = abi.Geometry(2, 16, 64, 256, 4, 4, 8, 0)
    st, _ = _mine(0, g)
    assert st == abi.ERR_CONFIG and b"at least one layer" in L.fsvd_last_error()
    g = abi.Geometry(2, 16, 64, 256, 4, 4, 8, 2)
    st, _ = _mine(2, g, 17)
    assert st == abi.ERR_CONFIG and b"[1, seq_len]" in L.fsvd_last_error()
    g = abi.Geometry(2, 16, 64, 256, 4, 4, 17, 2)
    st, _ = _mine(1, g)
    assert st == abi.ERR_RANK
    # SURVEY cfg2 numbers: 12 layers, B 32, M 512, r 32
    g = abi.Geometry(32, 512, 768, 3072, 12, 12, 32, 12)
    assert _mine(0, g) == (0, 4 * 2 * 12 * 32 * 512 * 32)


def test_decoder_entry_points_validate_before_the_device():
    """Argument errors surface with the reference's kinds before any device
    work (no GPU needed): zero extents are ShapeErrors, missing arguments
    ConfigErrors."""
    import ctypes as C
    sz = abi._sz
    b = sz()
    st = L.fsvd_decoder_prefill(None, 1, 0, 2, 4, None, None, None, 8, None, 0, None)
    assert st == abi.ERR_SHAPE or st == abi.ERR_CONFIG
    st = L.fsvd_decoder_prefill(None, 1, 0, 0, 4, None, None, None, 8, None, 0, None)
    assert st == abi.ERR_SHAPE and b"at least 1" in L.fsvd_last_error()
    st = L.fsvd_decoder_step(None, 1, 0, 2, 0, None, None, None, 8, None, 0, None)
    assert st == abi.ERR_CONFIG and b"null" in L.fsvd_last_error()
    assert L.fsvd_decoder_graph_step(None, 0, None) == abi.ERR_CONFIG
    assert L.fsvd_kv_cache_bytes(None, 2, 8, C.byref(b)) == abi.ERR_CONFIG
    assert L.fsvd_decoder_workspace_bytes(None, 1, 2, 8, 0, C.byref(b)) == abi.ERR_CONFIG
    g = C.c_void_p()
    st = L.fsvd_decoder_graph_create(None, 1, 0, 2, None, None, None, 8, None, 0, C.byref(g))
    assert st == abi.ERR_CONFIG
    L.fsvd_decoder_graph_destroy(None)  # NULL is a no-op


def test_factorizer_entry_points_validate_before_the_device():
    import ctypes as C
    assert L.fsvd_factor_rank_r_batch(None, 1) == abi.ERR_CONFIG
    assert L.fsvd_factor_rank_r_batch(None, 0) in (abi.OK, abi.ERR_CUDA)  # empty batch
    r, pr, fr = abi._sz(0), abi._sz(0), abi._sz(0)
    assert L.fsvd_factorize_layers(None, 0, 12, r, pr, fr, None) == abi.ERR_CONFIG
