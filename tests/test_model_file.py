"""FSVD1 model files: the container reader's errors
match the reference reader byte for byte (proj/tests/test_encoder.cpp:472-551
fixtures, and oracle/_ref's read_tensor_file on the same bytes), models
written by the reference's own save_model assemble into the same layers, and
(GPU) run bit-identically to packs built from the arrays directly."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

import oracle
from paper_2508_01506_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
GOOD = bytes([
    0x46, 0x53, 0x56, 0x44, 0x01, 0x00, 0x00, 0x00,
    0x01, 0x00, 0x00, 0x00, 0x01, 0x00, 0x77, 0x00,
    0x02, 0x02, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00,
    0x00, 0x02, 0x00, 0x00, 0x00, 0x00, 0x00, 0x00,
    0x00, 0x00, 0x00, 0xC0, 0x3F, 0x00, 0x00, 0x00,
    0xC0, 0x00, 0x00, 0x80, 0x3E, 0x00, 0x00, 0x40,
    0x40,
])


def _mut(at, value):
    b = bytearray(GOOD)
    b[at] = value
    return bytes(b)


def _zero_extent():
    b = bytearray(GOOD)
    b[17:25] = bytes(8)
    return bytes(b)


# (case, bytes, expected FormatError offset) -- test_encoder.cpp:509-551
MALFORMED = [
    ("truncated", GOOD[:-2], 47),
    ("magic", _mut(0, 0x58), 0),
    ("version", _mut(4, 0x02), 4),
    ("dtype", _mut(15, 0x07), 15),
    ("rank", _mut(16, 0x00), 16),
    ("zero_extent", _zero_extent(), 17),
    ("trailing", GOOD + bytes([0xAA, 0xBB, 0xCC]), 49),
]


def _probe(path):
    L = abi.lib()
    n = C.c_size_t()
    g = abi.Geometry()
    st = L.fsvd_model_file_probe(path.encode(), C.byref(n), C.byref(g))
    return st, L.fsvd_last_error().decode(), L.fsvd_last_error_offset(), n.value, g


def test_hand_built_fixture_parses(tmp_path):
    p = tmp_path / "fixture.fsvd"
    p.write_bytes(GOOD)
    st, msg, _, _, _ = _probe(str(p))
    # the container is valid; "w" is not a layer tensor, so assembly refuses it
    assert st == abi.ERR_CONFIG and "unrecognized tensor name: w" in msg


@pytest.mark.parametrize("case,data,offset", MALFORMED, ids=[m[0] for m in MALFORMED])
def test_malformed_offsets_match_reference_contract(tmp_path, case, data, offset):
    p = tmp_path / f"{case}.fsvd"
    p.write_bytes(data)
    st, msg, off, _, _ = _probe(str(p))
    assert st == abi.ERR_FORMAT, msg
    assert off == offset and f"(at byte {offset})" in msg


@pytest.mark.parametrize("case,data,offset", MALFORMED, ids=[m[0] for m in MALFORMED])
def test_malformed_offsets_match_reference_reader(tmp_path, reference, case, data, offset):
    p = tmp_path / f"{case}.fsvd"
    p.write_bytes(data)
    assert reference.lib.ref_read_error_offset(str(p).encode()) == offset
    assert _probe(str(p))[2] == offset


def _ref_model(tmp_path, reference, layers, name="m.fsvd"):
    from paper_2508_01506_b200.model import layer_descs
    path = str(tmp_path / name)
    descs = layer_descs(layers)
    st = reference.lib.ref_save_model(path.encode(), descs, len(layers))
    assert st == 0, reference.lib.ref_last_error()
    return path


def test_reference_written_model_assembles(tmp_path, reference):
    from paper_2508_01506_b200.model import random_layer
    rng = np.random.default_rng(0)
    layers = [random_layer(64, 128, 4, 2, 8, 24, 40, rng, activation=a) for a in (0, 1)]
    path = _ref_model(tmp_path, reference, layers)
    st, msg, _, n, g = _probe(path)
    assert st == abi.OK, msg
    assert (n, g.layers, g.d_model, g.d_ff, g.heads, g.groups, g.rank) == (2, 2, 64, 128, 4, 2, 8)


def test_missing_and_duplicate_tensors(tmp_path, reference):
    from paper_2508_01506_b200.model import random_layer
    rng = np.random.default_rng(1)
    path = _ref_model(tmp_path, reference, [random_layer(32, 64, 2, 2, 4, 8, 8, rng)])
    data = open(path, "rb").read()
    # rebuild the record list, drop "layer.0.ffn.up.b", then duplicate "layer.0.heads"
    recs, off = [], 12
    count = struct.unpack_from("<I", data, 8)[0]
    for _ in range(count):
        nl = struct.unpack_from("<H", data, off)[0]
        name = data[off + 2:off + 2 + nl].decode()
        nd = data[off + 3 + nl]
        ext = struct.unpack_from(f"<{nd}Q", data, off + 4 + nl)
        size = 4 + nl + 8 * nd + 4 * int(np.prod(ext))
        recs.append((name, data[off:off + size]))
        off += size

    def write(rs, fn):
        q = tmp_path / fn
        q.write_bytes(b"FSVD" + struct.pack("<II", 1, len(rs)) + b"".join(r for _, r in rs))
        return str(q)
    st, msg, *_ = _probe(write([r for r in recs if r[0] != "layer.0.ffn.up.b"], "miss.fsvd"))
    assert st == abi.ERR_CONFIG and "missing tensor: layer.0.ffn.up.b" in msg
    heads = [r for r in recs if r[0] == "layer.0.heads"]
    st, msg, *_ = _probe(write(recs + heads, "dup.fsvd"))
    assert st == abi.ERR_CONFIG and "duplicate tensor name: layer.0.heads" in msg
    st, msg, *_ = _probe(str(tmp_path / "does_not_exist.fsvd"))
    assert st == abi.ERR_IO


def _records(path):
    """(name, ndarray) list of an FSVD1 file, in file order."""
    data = open(path, "rb").read()
    out, off = [], 12
    for _ in range(struct.unpack_from("<I", data, 8)[0]):
        nl = struct.unpack_from("<H", data, off)[0]
        name = data[off + 2:off + 2 + nl].decode()
        nd = data[off + 3 + nl]
        ext = struct.unpack_from(f"<{nd}Q", data, off + 4 + nl)
        at = off + 4 + nl + 8 * nd
        n = int(np.prod(ext))
        out.append((name, np.frombuffer(data, "<f4", n, at).reshape(ext)))
        off = at + 4 * n
    return out


def _write_records(recs, path):
    body = b""
    for name, a in recs:
        nb = name.encode()
        body += struct.pack("<H", len(nb)) + nb + bytes([0, a.ndim])
        body += struct.pack(f"<{a.ndim}Q", *a.shape) + np.ascontiguousarray(a, "<f4").tobytes()
    with open(path, "wb") as f:
        f.write(b"FSVD" + struct.pack("<II", 1, len(recs)) + body)
    return path


# EncoderLayer::validate() checks (encoder.cpp:156-221) a file can violate
# while the container is well formed: the loader must refuse each with the
# reference's error kind and message instead of reading past a short tensor.
BAD_SHAPES = [
    ("ffn_up_bias_short", "layer.0.ffn.up.b", lambda a: a[:1], "ffn up bias"),
    ("ffn_down_bias_short", "layer.0.ffn.down.b", lambda a: a[:3], "ffn down bias"),
    ("ln1_beta_short", "layer.0.ln1.beta", lambda a: a[:1], "ln1.beta"),
    ("ln2_beta_2d", "layer.0.ln2.beta", lambda a: a.reshape(1, -1), "ln2.beta"),
    ("ln2_gamma_short", "layer.0.ln2.gamma", lambda a: a[:-1], "ln2.gamma"),
    ("out_bias_short", "layer.0.attn.out.bias", lambda a: a[:1], "out_proj bias"),
    ("out_v_rank", "layer.0.attn.out.V", lambda a: a[:-1], "out_proj V"),
    ("up_v_rank", "layer.0.ffn.up.V", lambda a: a[:-1], "ffn up V"),
    ("down_v_rank", "layer.0.ffn.down.V", lambda a: a[:-1], "ffn down V"),
    ("down_u_rows", "layer.0.ffn.down.U", lambda a: a[:-1], "ffn down U"),
    ("attn_bias_short", "layer.0.attn.k.head.1.b", lambda a: a[:-1], "attention factor bias"),
    ("attn_v_2d_flat", "layer.0.attn.v.head.0.V", lambda a: a.reshape(-1), "attention factor V"),
    ("attn_u_rank", "layer.0.attn.q.head.1.U", lambda a: a[:, :-1], "attention factor U"),
]


@pytest.mark.parametrize("case,name,edit,what", BAD_SHAPES, ids=[b[0] for b in BAD_SHAPES])
def test_layer_shape_checks_match_reference(tmp_path, reference, case, name, edit, what):
    from paper_2508_01506_b200.model import random_layer
    rng = np.random.default_rng(3)
    path = _ref_model(tmp_path, reference, [random_layer(32, 64, 4, 2, 4, 8, 8, rng)])
    recs = [(n, edit(a) if n == name else a) for n, a in _records(path)]
    assert any(n == name for n, _ in recs)
    bad = _write_records(recs, str(tmp_path / f"{case}.fsvd"))
    n = C.c_size_t()
    ref_st = reference.lib.ref_load_model(bad.encode(), C.byref(n))
    ref_msg = reference.lib.ref_last_error().decode()
    st, msg, *_ = _probe(bad)
    assert ref_st == abi.ERR_SHAPE and what in ref_msg, ref_msg
    assert (st, msg) == (ref_st, ref_msg)


def test_rank_mismatch_is_config_error_like_reference(tmp_path, reference):
    from paper_2508_01506_b200.model import random_layer
    rng = np.random.default_rng(4)
    path = _ref_model(tmp_path, reference, [random_layer(32, 64, 4, 2, 4, 8, 8, rng)])
    recs = [(n, a[:, :-1] if n == "layer.0.ffn.down.U" else a) for n, a in _records(path)]
    bad = _write_records(recs, str(tmp_path / "rank.fsvd"))
    n = C.c_size_t()
    ref_st = reference.lib.ref_load_model(bad.encode(), C.byref(n))
    st, msg, *_ = _probe(bad)
    assert ref_st == abi.ERR_CONFIG
    assert (st, msg) == (ref_st, reference.lib.ref_last_error().decode())


def test_rewritten_model_roundtrips(tmp_path, reference):
    """_records/_write_records reproduce the reference writer's bytes."""
    from paper_2508_01506_b200.model import random_layer
    rng = np.random.default_rng(5)
    path = _ref_model(tmp_path, reference, [random_layer(32, 64, 4, 2, 4, 8, 8, rng)])
    again = _write_records(_records(path), str(tmp_path / "again.fsvd"))
    assert open(path, "rb").read() == open(again, "rb").read()


def test_committed_golden_model_assembles():
    st, msg, _, n, g = _probe(os.path.join(HERE, "golden", "tiny_model.fsvd"))
    assert st == abi.OK, msg
    assert n == 2 and g.d_model == 32 and g.heads == 4


@pytest.mark.gpu
def test_loaded_model_runs_like_array_packs(tmp_path, reference):
    import torch
    from paper_2508_01506_b200.model import layer_descs, random_layer, round_layer_bf16
    L = abi.lib()
    rng = np.random.default_rng(2)
    layers = [round_layer_bf16(random_layer(256, 512, 4, 4, 32, 64, 128, rng)) for _ in range(2)]
    path = _ref_model(tmp_path, reference, layers)
    loaded = (C.c_void_p * 2)()
    n = C.c_size_t()
    abi.check(L.fsvd_model_load(path.encode(), abi.BF16, 0, loaded, 2, C.byref(n)))
    assert n.value == 2
    descs = layer_descs(layers)
    direct = (C.c_void_p * 2)()
    for i in range(2):
        p = C.c_void_p()
        abi.check(L.fsvd_layer_pack_create(C.byref(descs[i]), abi.BF16, 0, C.byref(p)))
        direct[i] = p.value
    B, M = 2, 130
    ws = C.c_size_t()
    abi.check(L.fsvd_workspace_bytes(direct, 2, B, M, abi.MODE_FLASH_V2, C.byref(ws)))
    work = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
    x = torch.randn((B, M, 256), generator=torch.Generator().manual_seed(7)).to(torch.bfloat16).cuda()
    outs = []
    for packs in (loaded, direct):
        o = torch.empty_like(x)
        abi.check(L.fsvd_model_fwd(packs, 2, abi.MODE_FLASH_V2, 0, B, M, C.c_void_p(x.data_ptr()),
                                   C.c_void_p(o.data_ptr()), C.c_void_p(work.data_ptr()), ws.value,
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    for i in range(2):
        L.fsvd_layer_pack_destroy(C.c_void_p(loaded[i]))
        L.fsvd_layer_pack_destroy(C.c_void_p(direct[i]))
