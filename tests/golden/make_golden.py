"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref, built from /root/reference by
oracle/Makefile):  python tests/golden/make_golden.py

Every case draws its inputs with the reference's own seeded generator
(oracle::random_tensor, tests/support/oracles.hpp:80-87) and the
acceptance-style factor synthesis (acceptance.cpp:62-128), runs the reference
kernel, and stores the output.  The first values of the generator stream are
stored too, which pins the generator itself.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2508_01506_b200 import abi  # noqa: E402

# (name, kind, d, df, heads, groups, rank, pr, fr, B, M, seed, extra)
CASES = [
    ("attn_g2_r5", "attn", 48, 0, 4, 2, 5, 0, 0, 2, 33, 101, {}),
    ("attn_g1_r7", "attn", 48, 0, 6, 1, 7, 0, 0, 1, 17, 102, {}),
    ("attn_per_head_r8", "attn", 64, 0, 4, 4, 8, 0, 0, 3, 20, 103, {}),
    ("outproj_r6", "outproj", 40, 0, 1, 1, 0, 6, 0, 2, 9, 104, {}),
    ("ffn_v1_gelu", "ffn1", 32, 80, 1, 1, 0, 0, 12, 2, 19, 105, {"act": 0}),
    ("ffn_v2_tanh", "ffn2", 32, 80, 1, 1, 0, 0, 12, 2, 19, 106, {"act": 1}),
    ("ffn_v1_relu", "ffn1", 24, 64, 1, 1, 0, 0, 5, 1, 7, 107, {"act": 2}),
    ("ffn_v2_identity", "ffn2", 24, 64, 1, 1, 0, 0, 5, 1, 7, 108, {"act": 3}),
    ("layer_v1_post", "layer", 48, 96, 4, 4, 8, 8, 8, 2, 16, 109, {"mode": 2, "pre": 0}),
    ("layer_v2_pre", "layer", 48, 96, 4, 2, 6, 10, 12, 2, 16, 110, {"mode": 3, "pre": 1}),
    ("model2_v1", "model", 32, 64, 4, 2, 4, 8, 8, 1, 24, 111, {"mode": 2, "pre": 0, "layers": 2}),
]
PLAN = abi.TilePlan(16, 16, 64, 1 << 20)


def make_case(ref, c):
    name, kind, d, df, H, G, r, pr, fr, B, M, seed, extra = c
    x = ref.random((B, M, d), seed + 7)
    if kind == "attn":
        a = oracle.rand_attn(ref, d, G, r, seed * 631)
        return x, ref.attention(x, a, H, PLAN)
    if kind == "outproj":
        lin = oracle.rand_linear(ref, d, d, pr, seed * 97)
        return x, ref.outproj(x, lin)
    if kind in ("ffn1", "ffn2"):
        f = oracle.rand_ffn(ref, d, df, fr, seed * 97, extra["act"])
        return x, ref.ffn(1 if kind == "ffn1" else 2, x, f, PLAN)
    n = extra.get("layers", 1)
    layers = [oracle.rand_layer(ref, d, df, H, G, r, seed * 1013 + 17 * i, pr, fr) for i in range(n)]
    return x, ref.run_model(x, layers, extra["mode"], PLAN, pre_ln=bool(extra["pre"]))


def main():
    ref = oracle.Reference()
    out = {"gaussian_seed5": ref.random((64,), 5, 1.0), "gaussian_seed9_sd02": ref.random((64,), 9, 0.02)}
    for c in CASES:
        x, y = make_case(ref, c)
        out[c[0]] = y
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


def make_tiny_model(path=os.path.join(HERE, "tiny_model.fsvd")):
    """tiny_model.fsvd: two BERT-like layers (d=32, H=G=4, r=4, pr=8, fr=16;
    GELU-erf then GELU-tanh) written by the reference's own save_model."""
    from paper_2508_01506_b200.model import layer_descs, random_layer
    ref = oracle.Reference()
    rng = np.random.default_rng(123)
    layers = [random_layer(32, 64, 4, 4, 4, 8, 16, rng),
              random_layer(32, 64, 4, 4, 4, 8, 16, rng, activation=1)]
    assert ref.lib.ref_save_model(path.encode(), layer_descs(layers), 2) == 0
    if os.path.exists(path + ".json"):
        os.remove(path + ".json")


if __name__ == "__main__":
    main()
    make_tiny_model()
