"""Device-timed throughput of the non-headline BASELINE.json configs.

  cfg3  BERT-Large (d=1024, 16 heads, d_ff 4096), seq 4096, r=32, pr=fr=512,
        FlashSVD-FFN V2, B in {1, 8}: tokens/s, per-sublayer times, workspace
        bytes against the dense-reconstruction baseline (peak-memory stress).
  cfg4  BERT-Base seq 1024, B=16: the rank sweep r in {8,16,32,64} x
        fr in {128..1024} (pr = min(r G, d)), tokens/s and the FFN kernel's
        algorithmic TFLOP/s -- the tensor-pipe vs HBM crossover of SURVEY 8(d).

Every number: fsvd_model_fwd / fsvd_ffn_fwd through the C ABI, bf16,
device-resident inputs, CUDA events on the launching stream, L2 flushed
(256 MiB write) between timed steps.  One JSON object per line.

  python tools/config_bench.py --cfg 3 4 --out profiles/r01_config_bench.jsonl
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.model import layer_descs, random_layer  # noqa: E402


def flops_per_token_layer(d, df, g, r, pr, fr, m):
    """SURVEY 8(d) algorithmic FLOP per token per layer."""
    return 2 * d * 3 * g * r + 6 * r * d + 4 * m * d + 4 * d * pr + 2 * fr * (2 * d + 2 * df)


def run(L, torch, d, df, H, r, pr, fr, B, M, layers, mode, steps=10, warmup=3):
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    rng = np.random.default_rng(7)
    lay = random_layer(d, df, H, H, r, pr, fr, rng)
    descs = layer_descs([lay])
    p = C.c_void_p()
    abi.check(L.fsvd_layer_pack_create(C.byref(descs[0]), abi.BF16, 0, C.byref(p)))
    tc = L.fsvd_layer_pack_uses_tensor_cores(p)
    parr = (C.c_void_p * layers)(*([p.value] * layers))  # same factors in every layer
    wsb = C.c_size_t()
    abi.check(L.fsvd_workspace_bytes_ln(parr, layers, B, M, mode, 0, C.byref(wsb)))
    work = torch.empty(wsb.value, dtype=torch.uint8, device=dev)
    x = torch.randn((B, M, d), device=dev).to(torch.bfloat16)
    out = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    T = B * M

    def fwd():
        abi.check(L.fsvd_model_fwd(parr, layers, mode, 0, B, M, C.c_void_p(x.data_ptr()),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(work.data_ptr()),
                                   wsb.value, sp))

    def timed(fn, n, flush_l2):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(n):
            if flush_l2:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        return tot / n

    ms = timed(fwd, steps, True)
    assert torch.isfinite(out.float()).all().item()
    variant = 2 if mode == abi.MODE_FLASH_V2 else 1
    ffn_out = torch.empty_like(x)
    mem_ws = wsb.value
    # the sublayer entry points run the unfused schedules (their transients
    # exceed the compact layer workspace): a scratch of their own
    work = torch.empty(max(wsb.value, T * (4 * H * 64 + 4 * fr + 2 * df) * 2), dtype=torch.uint8,
                       device=dev)
    wsb = C.c_size_t(work.numel())
    ffn_ms = timed(lambda: abi.check(L.fsvd_ffn_fwd(
        p, variant, B, M, C.c_void_p(x.data_ptr()), C.c_void_p(ffn_out.data_ptr()),
        C.c_void_p(work.data_ptr()), C.c_size_t(wsb.value), sp)), steps, False)
    attn_ms = timed(lambda: abi.check(L.fsvd_attention_fwd(
        p, B, M, C.c_void_p(x.data_ptr()), C.c_void_p(ffn_out.data_ptr()),
        C.c_void_p(work.data_ptr()), C.c_size_t(wsb.value), sp)), steps, False)
    ffn_flops = T * 2 * fr * (2 * d + 2 * df)
    model_flops = T * layers * flops_per_token_layer(d, df, H, r, pr, fr, M)
    es = 2
    dense_ws = 2 * T * d * es + max(3 * d, df) * T * es  # Q/K/V or hidden materialized
    L.fsvd_layer_pack_destroy(p)
    return {"d": d, "d_ff": df, "heads": H, "r": r, "pr": pr, "fr": fr, "batch": B, "seq": M,
            "layers": layers, "mode": "flash_v2" if mode == abi.MODE_FLASH_V2 else "flash_v1",
            "tensor_cores": bool(tc), "ms_per_forward": round(ms, 4),
            "tokens_per_s": round(T / (ms * 1e-3), 1),
            "model_tflops": round(model_flops / (ms * 1e-3) / 1e12, 1),
            "ffn_ms": round(ffn_ms, 4), "ffn_tflops": round(ffn_flops / (ffn_ms * 1e-3) / 1e12, 1),
            "attention_ms": round(attn_ms, 4),
            "workspace_mib": round(mem_ws / 2**20, 1),
            "activation_mib": round((mem_ws + T * d * es) / 2**20, 1),
            "activation_mib_out_of_place": round((mem_ws + 2 * T * d * es) / 2**20, 1),
            # dense-reconstruction schedules counted like bench.py: in place (one
            # batch buffer) and out of place (input + output)
            "naive_lowrank_reconstruction_mib": round((dense_ws + T * d * es) / 2**20, 1),
            "naive_lowrank_reconstruction_mib_out_of_place": round((dense_ws + 2 * T * d * es) / 2**20, 1),
            "dense_with_scores_mib": round((dense_ws + T * d * es + B * H * M * M * es) / 2**20, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="+", default=[3, 4])
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--batches", default="1,8", help="cfg3 batch sizes")
    ap.add_argument("--modes", default="v2,v1", help="cfg3 FFN variants")
    args = ap.parse_args()
    import torch
    L = abi.lib()
    if not L.fsvd_device_available():
        raise SystemExit("no sm_100 device: " + L.fsvd_last_error().decode())
    rows = []
    if 3 in args.cfg:
        modes = {"v2": abi.MODE_FLASH_V2, "v1": abi.MODE_FLASH_V1}
        for B in [int(v) for v in args.batches.split(",")]:
            for mode in [modes[m] for m in args.modes.split(",")]:
                rows.append(dict(cfg=3, **run(L, torch, 1024, 4096, 16, 32, 512, 512, B, 4096, 24,
                                              mode, args.steps)))
                print(json.dumps(rows[-1]), flush=True)
    if 4 in args.cfg:
        for r in (8, 16, 32, 64):
            pr = min(r * 12, 768)
            for fr in (128, 256, 384, 512, 768, 1024):
                rows.append(dict(cfg=4, **run(L, torch, 768, 3072, 12, r, pr, fr, 16, 1024, 12,
                                              abi.MODE_FLASH_V2, args.steps)))
                print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for row in rows:
                f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
