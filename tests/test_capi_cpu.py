"""CPU: the C-ABI library loads, exports every declared symbol, and its host
logic (meter, plan validation, closed forms, shape/config errors) behaves like
the reference.  No compute calls are made here."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2508_01506_b200 import abi
from helpers import Meter, header_functions

L = abi.lib()


def test_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 40
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(abi.EXPORTED), set(names) ^ set(abi.EXPORTED)
    assert L.fsvd_abi_version() == 1


def test_no_cpu_fallback_without_device():
    if L.fsvd_device_available():
        pytest.skip("GPU present")
    ora = oracle.Restatement()
    layer = oracle.rand_layer(ora, 32, 64, 4, 2, 4, 1)
    x = ora.random((1, 8, 32), 2)
    out = np.zeros_like(x)
    from paper_2508_01506_b200.model import layer_descs
    st = L.fsvd_run_model(abi.fptr(x), 1, 8, 32, layer_descs([layer]), 1, abi.MODE_FLASH_V1,
                          abi.TilePlan.default(), 0, b"layer", abi.F32, None, abi.fptr(out))
    assert st == abi.ERR_CUDA
    assert b"no CPU fallback" in L.fsvd_last_error()
    assert not out.any()


# ------------------------------------------------------------------ meter
def test_meter_classes_peak_and_regions():
    m = Meter()
    ids = []
    for tag, cls, b in [("a", abi.TRANSIENT, 100), ("b", abi.TRANSIENT, 50), ("x", abi.EXCLUDED, 7)]:
        i = C.c_uint64()
        abi.check(L.fsvd_meter_alloc(m.h, tag.encode(), cls, b, C.byref(i)))
        ids.append(i.value)
    assert m.peak == 150 and m.current == 150 and m.excluded == 7
    abi.check(L.fsvd_meter_free(m.h, ids[0]))
    assert m.current == 50 and m.peak == 150
    L.fsvd_meter_reset_peak(m.h)
    assert m.peak == 50
    # double free -> AccountingError (memtier.cpp:31-34)
    abi.check(L.fsvd_meter_free(m.h, ids[1]))
    assert L.fsvd_meter_free(m.h, ids[1]) == abi.ERR_ACCOUNTING


def test_meter_pins_idempotent_and_mismatch():
    m = Meter()
    abi.check(L.fsvd_meter_pin(m.h, b"w", 64))
    abi.check(L.fsvd_meter_pin(m.h, b"w", 64))
    assert m.persistent == 64
    assert L.fsvd_meter_pin(m.h, b"w", 65) == abi.ERR_ACCOUNTING  # memtier.cpp:55-58
    assert m.persistent == 64


def test_meter_region_imbalance_latched():
    m = Meter()
    e = C.c_size_t()
    abi.check(L.fsvd_meter_region_begin(m.h, b"r", C.byref(e)))
    i = C.c_uint64()
    abi.check(L.fsvd_meter_alloc(m.h, b"leak", abi.TRANSIENT, 8, C.byref(i)))
    abi.check(L.fsvd_meter_region_end(m.h, b"r", e.value))
    assert L.fsvd_meter_assert_clean(m.h) == abi.ERR_ACCOUNTING
    assert b"region \"r\" ended with 8" in L.fsvd_last_error()


def test_meter_event_log_replays():
    # tests/test_memtier.cpp:17-60 replay oracle: events reproduce the counters
    m = Meter()
    rng = np.random.default_rng(3)
    live = []
    for step in range(200):
        if live and rng.random() < 0.4:
            abi.check(L.fsvd_meter_free(m.h, live.pop(int(rng.integers(len(live))))))
        else:
            i = C.c_uint64()
            abi.check(L.fsvd_meter_alloc(m.h, b"t%d" % step, int(rng.integers(3)),
                                         int(rng.integers(1, 1000)), C.byref(i)))
            live.append(i.value)
    cur = {0: 0, 1: 0, 2: 0}
    peak = 0
    for kind, cls, tag, b, _ in m.events():
        if kind == abi_ev("ALLOC"):
            cur[cls] += b
        elif kind == abi_ev("FREE"):
            cur[cls] -= b
        peak = max(peak, cur[0])
    assert cur[0] == m.current and cur[2] == m.excluded and peak == m.peak


def abi_ev(name):
    return {"ALLOC": 0, "FREE": 1, "PIN": 2, "REGION_BEGIN": 3, "REGION_END": 4}[name]


# ------------------------------------------------------------------ closed forms
GEOMS = [abi.Geometry(b, m, d, df, h, g, r, 1)
         for (b, m, d, df, h, g, r) in [(1, 128, 768, 3072, 12, 12, 64), (2, 64, 128, 512, 4, 4, 16),
                                        (8, 128, 768, 3072, 12, 12, 64), (2, 16, 32, 64, 4, 2, 8)]]


@pytest.mark.parametrize("geom", GEOMS)
def test_expected_bytes_match_reference(reference, geom):
    for f in range(8):
        b = C.c_size_t()
        abi.check(L.fsvd_expected_bytes(f, geom, C.byref(b)))
        assert b.value == reference.expected_bytes(f, geom)


def test_validate_tile_plan_matches_reference(reference):
    for kind in range(3):
        for plan in [abi.TilePlan(16, 16, 64, 131072), abi.TilePlan(16, 16, 32, 1 << 20),
                     abi.TilePlan(128, 128, 128, 1 << 16), abi.TilePlan(16, 0, 16, 1 << 20)]:
            for g in GEOMS:
                b = C.c_size_t()
                st = L.fsvd_validate_tile_plan(plan, kind, g, C.byref(b))
                st_ref, b_ref = reference.validate_tile_plan(plan, kind, g)
                assert st == st_ref
                if st == 0:
                    assert b.value == b_ref


def test_budget_error_names_largest_buffer():
    # memtier.cpp:178-187; cfg1 FFN at fr=384 fails the default plan
    g = abi.Geometry(1, 128, 768, 3072, 1, 1, 384, 1)
    b = C.c_size_t()
    assert L.fsvd_validate_tile_plan(abi.TilePlan.default(), abi.KERNEL_FFN_V1, g,
                                     C.byref(b)) == abi.ERR_BUDGET
    msg = L.fsvd_last_error().decode()
    assert "250112 bytes exceeds budget 131072" in msg and '"v1_panel" (98304 bytes)' in msg
    assert b.value == 250112


def test_flash_layer_closed_forms():
    # encoder.cpp:333-345; test_encoder.cpp:255-263 golden (d=32 df=64 G=2 r=8 B=2 M=16)
    g = abi.Geometry(2, 16, 32, 64, 4, 2, 8, 1)
    assert L.fsvd_flash_layer_peak_transient_bytes(g) == 6144
    assert L.fsvd_flash_layer_persistent_bytes(g) == 11264


# ------------------------------------------------------------------ host-API checks (pre-device)
def test_host_api_shape_and_config_errors():
    ora = oracle.Restatement()
    a = oracle.rand_attn(ora, 32, 2, 4, 1)
    x = ora.random((1, 8, 32), 2)
    out = np.zeros_like(x)
    plan = abi.TilePlan(16, 16, 64, 1 << 20)
    # width mismatch -> ShapeError (attention.cpp:50-51)
    x2 = ora.random((1, 8, 16), 2)
    st = L.fsvd_flash_svd_attention(abi.fptr(x2), 1, 8, 16, a.desc(), 4, plan, abi.F32, None, b"a",
                                    abi.fptr(out), 1, 8, 32)
    assert st == abi.ERR_SHAPE
    # heads not dividing d -> ConfigError (attention.cpp:52-53)
    st = L.fsvd_flash_svd_attention(abi.fptr(x), 1, 8, 32, a.desc(), 5, plan, abi.F32, None, b"a",
                                    abi.fptr(out), 1, 8, 32)
    assert st == abi.ERR_CONFIG
    # groups not covering heads -> ConfigError (attention.cpp:209-210)
    a3 = oracle.rand_attn(ora, 32, 4, 4, 1)
    st = L.fsvd_flash_svd_attention(abi.fptr(x), 1, 8, 32, a3.desc(), 2, plan, abi.F32, None, b"a",
                                    abi.fptr(out), 1, 8, 32)
    assert st == abi.ERR_CONFIG
    # output not shaped like the input -> ShapeError
    st = L.fsvd_flash_svd_attention(abi.fptr(x), 1, 8, 32, a.desc(), 4, plan, abi.F32, None, b"a",
                                    abi.fptr(out), 1, 7, 32)
    assert st == abi.ERR_SHAPE
    # budget -> BudgetError (memtier.cpp:178)
    st = L.fsvd_flash_svd_attention(abi.fptr(x), 1, 8, 32, a.desc(), 4, abi.TilePlan(16, 16, 64, 100),
                                    abi.F32, None, b"a", abi.fptr(out), 1, 8, 32)
    assert st == abi.ERR_BUDGET
    # FFN rank mismatch -> ConfigError (ffn.cpp:47-48)
    f = oracle.rand_ffn(ora, 32, 64, 4, 3)
    bad = abi.FfnDesc(f.up.desc(), abi.LinearDesc(64, 5, 32, f.down.desc().u, f.down.desc().v,
                                                  f.down.desc().bias), 0)
    st = L.fsvd_ffn(1, abi.fptr(x), 1, 8, 32, bad, plan, abi.F32, None, b"f", abi.fptr(out), 1, 8, 32)
    assert st == abi.ERR_CONFIG
    st = L.fsvd_ffn(3, abi.fptr(x), 1, 8, 32, f.desc(), plan, abi.F32, None, b"f", abi.fptr(out),
                    1, 8, 32)
    assert st == abi.ERR_CONFIG


def test_run_model_rejects_aliased_output():
    ora = oracle.Restatement()
    layer = oracle.rand_layer(ora, 32, 64, 4, 2, 4, 1)
    x = ora.random((1, 8, 32), 2)
    from paper_2508_01506_b200.model import layer_descs
    st = L.fsvd_run_model(abi.fptr(x), 1, 8, 32, layer_descs([layer]), 1, abi.MODE_FLASH_V1,
                          abi.TilePlan.default(), 0, b"layer", abi.F32, None, abi.fptr(x))
    assert st == abi.ERR_CONFIG  # encoder.cpp:266-267


def test_layer_validation_errors():
    ora = oracle.Restatement()
    layer = oracle.rand_layer(ora, 32, 64, 4, 2, 4, 1)
    d = layer.desc()
    d.heads = 3
    p = C.c_void_p()
    assert L.fsvd_layer_pack_create(C.byref(d), abi.BF16, 0, C.byref(p)) == abi.ERR_CONFIG
    d = layer.desc()
    d.ffn.down.rank = 5
    assert L.fsvd_layer_pack_create(C.byref(d), abi.BF16, 0, C.byref(p)) == abi.ERR_CONFIG


def test_flops_and_io_closed_forms_match_reference(reference):
    """planner.cpp:60-98 flops_exact / io_bytes, bit-exact, all modes, with the
    reference's geometry errors."""
    import itertools
    n = 0
    for B, M, d, H, G, r in itertools.product((1, 32), (1, 128, 512), (64, 768), (4, 12), (1, 4),
                                              (1, 8, 16)):
        if d % H or d % G:
            continue
        g = abi.Geometry(B, M, d, 4 * d, H, G, r, 1)
        for mode in range(4):
            f, fi, fo = C.c_uint64(), C.c_uint64(), C.c_uint64()
            st = L.fsvd_flops_exact(g, mode, C.byref(f))
            rf = C.c_ulonglong()
            rst = reference.lib.ref_flops_exact_checked(g, mode, C.byref(rf))
            assert st == rst and (st or f.value == rf.value), (B, M, d, H, G, r, mode)
            st = L.fsvd_io_bytes(g, mode, C.byref(fi), C.byref(fo))
            ri, ro = C.c_ulonglong(), C.c_ulonglong()
            rst = reference.lib.ref_io_bytes(g, mode, C.byref(ri), C.byref(ro))
            assert st == rst and (st or (fi.value, fo.value) == (ri.value, ro.value))
            n += 1
    assert n > 200
