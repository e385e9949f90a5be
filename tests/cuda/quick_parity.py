"""Quick GPU parity sweep (developer tool): every host-API op vs the oracle."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import bf16_round, layer_descs, round_layer_bf16  # noqa: E402

L = abi.lib()
print("device available:", L.fsvd_device_available(), L.fsvd_last_error())
ora = oracle.Restatement()
plan = abi.TilePlan(16, 16, 64, 1 << 22)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def run(name, d, df, H, G, r, pr, fr, B, M, dtype, seed=1):
    layer = oracle.rand_layer(ora, d, df, H, G, r, seed, proj_rank=pr, ffn_rank=fr)
    x = ora.random((B, M, d), seed + 5)
    if dtype == abi.BF16:
        round_layer_bf16(layer)
        x = bf16_round(x)
    res = {}
    t0 = time.time()
    # attention
    ref = ora.attention(x, layer.attn, H, plan)
    out = np.zeros_like(x)
    abi.check(L.fsvd_flash_svd_attention(abi.fptr(x), B, M, d, layer.attn.desc(), H, plan, dtype,
                                         None, b"attn", abi.fptr(out), B, M, d))
    res["attn"] = rel(out, ref)
    ctx = ref.copy() if dtype == abi.F32 else bf16_round(ref)
    ref = ora.outproj(ctx, layer.out_proj)
    out = np.zeros_like(x)
    abi.check(L.fsvd_lowrank_output_projection(abi.fptr(ctx), B, M, d, layer.out_proj.desc(), dtype,
                                               None, b"attn", abi.fptr(out), B, M, d))
    res["outproj"] = rel(out, ref)
    for v in (1, 2):
        ref = ora.ffn(v, x, layer.ffn, plan)
        out = np.zeros_like(x)
        abi.check(L.fsvd_ffn(v, abi.fptr(x), B, M, d, layer.ffn.desc(), plan, dtype, None, b"ffn",
                             abi.fptr(out), B, M, d))
        res[f"ffn_v{v}"] = rel(out, ref)
    for mode in (abi.MODE_FLASH_V1, abi.MODE_FLASH_V2):
        ref = ora.run_model(x, [layer], mode, plan)
        out = np.zeros_like(x)
        abi.check(L.fsvd_run_model(abi.fptr(x), B, M, d, layer_descs([layer]), 1, mode, plan, 0,
                                   b"layer", dtype, None, abi.fptr(out)))
        res[f"layer_m{mode}"] = rel(out, ref)
    print(f"{name:28s} dtype={'bf16' if dtype else 'f32 '} " +
          " ".join(f"{k}={v:.2e}" for k, v in res.items()) + f"  ({time.time()-t0:.1f}s)", flush=True)
    return res


cases = [
    ("tiny-odd", 48, 96, 4, 2, 5, 7, 9, 2, 33),
    ("bert-head r32 fr128", 256, 512, 4, 4, 32, 64, 128, 2, 130),
    ("bert-base r32 fr384", 768, 3072, 12, 12, 32, 384, 384, 1, 128),
    ("r16 fr192 grouped", 512, 1024, 8, 2, 16, 96, 192, 2, 200),
    ("r64 fr256", 512, 2048, 8, 8, 64, 256, 256, 1, 257),
]
for c in cases:
    for dt in (abi.F32, abi.BF16):
        try:
            run(*c, dt)
        except Exception as e:  # keep sweeping
            print(f"{c[0]:28s} dtype={dt} FAILED: {e}", flush=True)
