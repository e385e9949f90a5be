"""GPU framework baseline for the headline workload (cfg2: 12 BERT-Base-sized
layers, r = 32, pr = fr = 384, B = 32, M = 512, bf16): the same low-rank
encoder written in plain PyTorch on the same B200 -- cuBLAS GEMMs, torch SDPA
(cuDNN) attention, separate GELU / residual / LayerNorm ops -- in the two
schedules the reference names:

  naive_lowrank : Q/K/V, the out-projection and the FFN weights reconstructed
                  per call from the factors (dense-reconstruction semantics,
                  attention.cpp:271-292, ffn.cpp:220-255)
  lowrank       : factor-by-factor GEMMs (x U) V, the [T, d_ff] hidden
                  materialised (the unfused reference FFN V1 schedule)

Reports tokens/s (CUDA events, L2 flushed between steps like bench.py) and
the peak activation memory (torch.cuda.max_memory_allocated above the
weights and the input).  Prints one JSON line per schedule.  Test/measure
infrastructure only."""
import json
import math
import os
import sys

import torch
import torch.nn.functional as F

B, M, D, H, DF, R, FR = 32, 512, 768, 12, 3072, 32, 384
LAYERS = int(os.environ.get("LAYERS", "12"))
dev = torch.device("cuda")
bf = torch.bfloat16


def factors(i, o, r):
    return (torch.randn(i, r, device=dev) / math.sqrt(i)).to(bf), \
        (torch.randn(r, o, device=dev) / math.sqrt(r)).to(bf), (torch.randn(o, device=dev) * .02).to(bf)


def make_layer():
    g = D // H
    return dict(
        q=[factors(D, g, R) for _ in range(H)], k=[factors(D, g, R) for _ in range(H)],
        v=[factors(D, g, R) for _ in range(H)], o=factors(D, D, FR),
        up=factors(D, DF, FR), dn=factors(DF, D, FR),
        ln1=(torch.ones(D, device=dev, dtype=bf), torch.zeros(D, device=dev, dtype=bf)),
        ln2=(torch.ones(D, device=dev, dtype=bf), torch.zeros(D, device=dev, dtype=bf)))


def layer_fwd(L, x, schedule):
    T = x.shape[0] * x.shape[1]
    xf = x.reshape(T, D)
    if schedule == "naive_lowrank":
        W = {n: torch.cat([u @ v for (u, v, _) in L[n]], dim=1) for n in ("q", "k", "v")}
        bq = {n: torch.cat([b for (_, _, b) in L[n]]) for n in ("q", "k", "v")}
        q, k, v = (xf @ W[n] + bq[n] for n in ("q", "k", "v"))
        wo = L["o"][0] @ L["o"][1]
        w_in = L["up"][0] @ L["up"][1]
        w_out = L["dn"][0] @ L["dn"][1]
    else:
        q, k, v = (torch.cat([(xf @ u) @ vv + bb for (u, vv, bb) in L[n]], dim=1)
                   for n in ("q", "k", "v"))
    sh = lambda t: t.view(B, M, H, D // H).transpose(1, 2)  # noqa: E731
    ctx = F.scaled_dot_product_attention(sh(q), sh(k), sh(v)).transpose(1, 2).reshape(T, D)
    if schedule == "naive_lowrank":
        att = ctx @ wo + L["o"][2]
    else:
        att = (ctx @ L["o"][0]) @ L["o"][1] + L["o"][2]
    h1 = F.layer_norm(xf + att, (D,), *L["ln1"])
    if schedule == "naive_lowrank":
        hid = F.gelu(h1 @ w_in + L["up"][2])
        ffn = hid @ w_out + L["dn"][2]
    else:
        hid = F.gelu((h1 @ L["up"][0]) @ L["up"][1] + L["up"][2])
        ffn = (hid @ L["dn"][0]) @ L["dn"][1] + L["dn"][2]
    return F.layer_norm(h1 + ffn, (D,), *L["ln2"]).view(B, M, D)


def peak_activation_mib(schedule="naive_lowrank", n_layers=LAYERS, seed=0):
    """One forward of the torch schedule; returns the peak allocation above the
    weights and the input (torch.cuda.max_memory_allocated), in MiB.  bench.py
    calls this in its own run (rank 0) for the memory comparison."""
    torch.manual_seed(seed)
    layers = [make_layer() for _ in range(n_layers)]
    x = torch.randn(B, M, D, device=dev).to(bf)
    with torch.no_grad():
        y = x
        for L in layers:  # warm (cuBLAS / SDPA workspaces are allocated here)
            y = layer_fwd(L, y, schedule)
        del y
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        y = x
        for L in layers:
            y = layer_fwd(L, y, schedule)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
    del layers, x, y
    torch.cuda.empty_cache()
    return peak / 2**20


def main():
    torch.manual_seed(0)
    layers = [make_layer() for _ in range(LAYERS)]
    x = torch.randn(B, M, D, device=dev).to(bf)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for schedule in ("naive_lowrank", "lowrank"):
        with torch.no_grad():
            for _ in range(3):
                y = x
                for L in layers:
                    y = layer_fwd(L, y, schedule)
            torch.cuda.synchronize()
            base = torch.cuda.memory_allocated()
            torch.cuda.reset_peak_memory_stats()
            y = x
            for L in layers:
                y = layer_fwd(L, y, schedule)
            torch.cuda.synchronize()
            peak = torch.cuda.max_memory_allocated() - base
            times = []
            for _ in range(10):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                y = x
                for L in layers:
                    y = layer_fwd(L, y, schedule)
                b.record()
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
        ms = sorted(times)[len(times) // 2]
        print(json.dumps({"baseline": "torch " + schedule, "tokens_per_s": round(B * M / (ms * 1e-3), 1),
                          "ms_per_forward": round(ms, 3), "layers": LAYERS,
                          "peak_activation_mib_above_weights_and_input": round(peak / 2**20, 1),
                          "attention": "torch SDPA (cuDNN / flash backends)", "dtype": "bf16"}))


if __name__ == "__main__":
    main()
