"""Decode throughput of the decoder rows on the cfg2
model (12 BERT-Base-sized layers, r 32, pr = fr = 384, bf16, random factors):
prefill CONTEXT tokens for BATCH sequences, then time STEPS single-token
decode steps (CUDA events on the launch stream, after warm-up).  Reports
tokens/s, ms per step, the rank-space cache size against the dense K/V
cache the same model would need, and the decode attention kernel's share.
Prints one JSON line."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200.decoder import Decoder  # noqa: E402
from paper_2508_01506_b200.model import random_layer  # noqa: E402


def main():
    B = int(os.environ.get("BATCH", "32"))
    CTX = int(os.environ.get("CONTEXT", "512"))
    STEPS = int(os.environ.get("STEPS", "64"))
    LAYERS = int(os.environ.get("LAYERS", "12"))
    rng = np.random.default_rng(0)
    layers = [random_layer(768, 3072, 12, 12, 32, 384, 384, rng) for _ in range(LAYERS)]
    graph = os.environ.get("GRAPH", "1") == "1"
    dec = Decoder(layers, B, CTX + STEPS + 8, graph=graph)
    x = torch.randn((B, CTX, 768), device="cuda").to(torch.bfloat16)
    toks = torch.randn((STEPS + 8, B, 768), device="cuda").to(torch.bfloat16)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    dec.prefill(x)  # warm-up (first launches, tensor maps, module load)
    torch.cuda.synchronize()
    t0.record()
    dec.prefill(x)
    t1.record()
    torch.cuda.synchronize()
    prefill_ms = t0.elapsed_time(t1)
    for k in range(4):  # warm-up steps
        dec.step(toks[k].contiguous())
    torch.cuda.synchronize()
    n0 = abi.lib().fsvd_kernel_launch_count()
    import time
    t0.record()
    c0 = time.perf_counter()
    for k in range(STEPS):
        dec.step(toks[4 + k].contiguous())
    issue_ms = (time.perf_counter() - c0) * 1e3 / STEPS
    t1.record()
    torch.cuda.synchronize()
    launches = abi.lib().fsvd_kernel_launch_count() - n0
    ms = t0.elapsed_time(t1) / STEPS
    cache = sum(c.numel() for c in dec.caches)
    dense_cache = LAYERS * B * (CTX + STEPS + 8) * 2 * 768 * 2
    # bytes the decode attention kernels read per step (K and V rows of every
    # layer at the mean context of the timed steps)
    ctx_mean = CTX + 4 + STEPS / 2
    attn_bytes = LAYERS * B * ctx_mean * 2 * 12 * 32 * 2
    print(json.dumps({
        "metric": "decode_tokens_per_s", "value": round(B / (ms * 1e-3), 1), "unit": "tokens/s",
        "ms_per_step": round(ms, 4), "host_issue_ms_per_step": round(issue_ms, 4), "batch": B, "context": CTX, "steps": STEPS,
        "layers": LAYERS, "prefill_ms": round(prefill_ms, 3),
        "prefill_tokens_per_s": round(B * CTX / (prefill_ms * 1e-3), 1),
        "kv_cache_mib": round(cache / 2**20, 2), "dense_kv_cache_mib": round(dense_cache / 2**20, 2),
        "attn_cache_bytes_per_step": int(attn_bytes), "gpu_launches_per_step": launches / STEPS,
        "cuda_graph": graph,
        "dtype": "bf16", "data": "synthetic (random factors, random bf16 tokens)"}))


if __name__ == "__main__":
    main()
