"""GPU: decoder rows -- causal prefill and decode steps on
the rank-space KV cache.

Oracle: causality means that, layer by layer, the output at position i is
the ENCODER layer's output on the prefix [0, i] of that layer's (causal)
inputs, at its last row.  The oracle restatement (pinned to the reference,
tests/test_oracle.py) is run that way, one prefix per position per layer.  bf16 policy: <= 2e-2 relative (max|got - ref| / max|ref|) with
bf16-rounded inputs and factors on both sides.
"""
import numpy as np
import pytest

import oracle
from paper_2508_01506_b200 import abi
from paper_2508_01506_b200.decoder import Decoder
from paper_2508_01506_b200.model import bf16_round, round_layer_bf16

import helpers as H

pytestmark = pytest.mark.gpu
PLAN = abi.TilePlan(16, 16, 64, 1 << 22)


@pytest.fixture(scope="module")
def L():
    lib = abi.lib()
    if not lib.fsvd_device_available():
        pytest.fail("GPU tests need an sm_100 device: " + lib.fsvd_last_error().decode())
    return lib


@pytest.fixture(scope="module")
def ora():
    return oracle.Restatement()


def _layers(ora, n=2, d=256, df=1024, heads=4, r=32, fr=128, seed=300):
    return [round_layer_bf16(oracle.rand_layer(ora, d, df, heads, heads, r, seed + 7 * i, fr, fr))
            for i in range(n)]


def _causal_ref(ora, x, layers, pre_ln):
    """[B, M, d] causal stack output: per layer, row i = encoder layer on rows [0, i]."""
    h = np.ascontiguousarray(x, np.float32)
    for lay in layers:
        nxt = np.empty_like(h)
        for i in range(h.shape[1]):
            nxt[:, i] = ora.run_model(np.ascontiguousarray(h[:, :i + 1]), [lay], abi.MODE_FLASH_V2,
                                      PLAN, pre_ln)[:, -1]
        h = nxt
    return h


@pytest.mark.parametrize("pre_ln", [False, True])
def test_causal_prefill_equals_prefix_encoder(L, ora, pre_ln):
    import torch
    layers = _layers(ora)
    B, M, d = 2, 200, 256
    x = bf16_round(ora.random((B, M, d), 41))
    dec = Decoder(layers, B, 256, pre_ln)
    got = dec.prefill(torch.from_numpy(x).cuda().to(torch.bfloat16)).float().cpu().numpy()
    ref = _causal_ref(ora, x, layers, pre_ln)
    for i in (0, 1, 5, 63, 64, 127, 128, 129, 160, 199):
        assert H.rel_err(got[:, i], ref[:, i]) <= H.TOL_BF16, (i, H.rel_err(got[:, i], ref[:, i]))
    assert H.rel_err(got, ref) <= H.TOL_BF16
    dec.close()


def test_decode_wide_ffn_rank(L, ora):
    """FFN rank 512 (> 384: sliced feature stream, split per feature block in
    decode): prefill + steps equal the causal reference."""
    import torch
    layers = _layers(ora, n=1, fr=512, seed=700)
    B, P, S, d = 2, 60, 6, 256
    x = bf16_round(ora.random((B, P + S, d), 43))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    dec = Decoder(layers, B, 128, False)
    pre = dec.prefill(xd[:, :P].contiguous()).float().cpu().numpy()
    steps = np.stack([dec.step(xd[:, P + k].contiguous()).float().cpu().numpy() for k in range(S)], 1)
    ref = _causal_ref(ora, x, layers, False)
    assert H.rel_err(pre, ref[:, :P]) <= H.TOL_BF16
    assert H.rel_err(steps, ref[:, P:]) <= H.TOL_BF16
    dec.close()


def test_decode_heterogeneous_layer_ranks(L, ora):
    """Layers with different per-head ranks (16 then 64: the second layer's
    cache row is 4x wider): every layer's cache is sized from its own pack,
    so prefill + steps still equal the causal reference."""
    import torch
    layers = [round_layer_bf16(oracle.rand_layer(ora, 256, 1024, 4, 4, r, 900 + r, 128, 128))
              for r in (16, 64)]
    B, P, S, d = 2, 70, 4, 256
    x = bf16_round(ora.random((B, P + S, d), 44))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    dec = Decoder(layers, B, 96, False)
    assert dec.caches[1].numel() == 4 * dec.caches[0].numel()
    pre = dec.prefill(xd[:, :P].contiguous()).float().cpu().numpy()
    steps = np.stack([dec.step(xd[:, P + k].contiguous()).float().cpu().numpy() for k in range(S)], 1)
    ref = _causal_ref(ora, x, layers, False)
    assert H.rel_err(pre, ref[:, :P]) <= H.TOL_BF16
    assert H.rel_err(steps, ref[:, P:]) <= H.TOL_BF16
    dec.close()


@pytest.mark.parametrize("pre_ln", [False, True])
def test_decode_steps_equal_prefix_encoder(L, ora, pre_ln):
    """prefill 100 tokens, then 40 single-token steps across the 128 tile
    boundary; each step's output is the prefix encoder's last row, and the
    steps agree with one causal prefill over all 140 tokens."""
    import torch
    layers = _layers(ora, seed=500)
    B, P, S, d = 3, 100, 40, 256
    x = bf16_round(ora.random((B, P + S, d), 42))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    dec = Decoder(layers, B, 160, pre_ln)
    dec.prefill(xd[:, :P].contiguous())
    steps = []
    for k in range(S):
        steps.append(dec.step(xd[:, P + k].contiguous()).float().cpu().numpy())
    steps = np.stack(steps, axis=1)
    ref = _causal_ref(ora, x, layers, pre_ln)[:, P:]
    for k in (0, 1, 27, 28, 29, 39):
        assert H.rel_err(steps[:, k], ref[:, k]) <= H.TOL_BF16, (k, H.rel_err(steps[:, k], ref[:, k]))
    full = Decoder(layers, B, 160, pre_ln)
    allp = full.prefill(xd).float().cpu().numpy()[:, P:]
    assert H.rel_err(steps, allp) <= H.TOL_BF16
    dec.close()
    full.close()


@pytest.mark.parametrize("pre_ln", [False, True])
def test_graph_decode_equals_direct_steps(L, ora, pre_ln):
    """The captured decode step (position read on the device, split count
    sized for max_seq) replays to the same bits as direct steps."""
    import torch
    layers = _layers(ora, seed=600)
    B, P, S, d = 2, 60, 12, 256
    x = bf16_round(ora.random((B, P + S, d), 44))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    outs = []
    for graph in (False, True):
        dec = Decoder(layers, B, 700, pre_ln, graph=graph)
        dec.prefill(xd[:, :P].contiguous())
        outs.append(np.stack([dec.step(xd[:, P + k].contiguous()).float().cpu().numpy()
                              for k in range(S)], axis=1))
        dec.close()
    # direct steps size the cache splits by the live length, the graph by
    # max_seq: the fp32 merge order differs, so agreement is to rounding
    assert H.rel_err(outs[1], outs[0]) <= 1e-2
    ref = _causal_ref(ora, x, layers, pre_ln)[:, P:]
    assert H.rel_err(outs[1], ref) <= H.TOL_BF16


def test_decode_long_cache_uses_split_combine(L, ora):
    """B=1, 12 heads, 1500 cached tokens: the decode kernel splits the cache
    over CTAs and merges the partial softmax states."""
    import torch
    layers = _layers(ora, n=1, d=768, df=1536, heads=12, r=32, fr=128, seed=700)
    B, P, d = 1, 1500, 768
    x = bf16_round(ora.random((B, P + 1, d), 43))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    dec = Decoder(layers, B, 2048, False)
    dec.prefill(xd[:, :P].contiguous())
    got = dec.step(xd[:, P].contiguous()).float().cpu().numpy()
    # one layer: the causal output of the last position is the encoder's on the whole prefix
    ref = ora.run_model(x, layers, abi.MODE_FLASH_V2, PLAN)[:, -1]
    assert H.rel_err(got, ref) <= H.TOL_BF16
    dec.close()


def test_decoder_errors(L, ora):
    import torch
    layers = _layers(ora, n=1)
    dec = Decoder(layers, 2, 16)
    with pytest.raises(abi.FsvdError) as e:
        dec.prefill(torch.zeros((2, 17, 256), dtype=torch.bfloat16, device="cuda"))
    assert e.value.status == abi.ERR_CONFIG
    dec.pos = 16
    with pytest.raises(abi.FsvdError) as e:
        dec.step(torch.zeros((2, 256), dtype=torch.bfloat16, device="cuda"))
    assert e.value.status == abi.ERR_CONFIG and "below max_seq" in str(e.value)
    dec.close()
