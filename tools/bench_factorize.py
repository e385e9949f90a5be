"""Times the device factorizer on BERT-Base: 12 dense
layers (d 768, d_ff 3072, 12 heads, r 32 -> pr = fr = 384) factorized by one
fsvd_factorize_layers call (host arrays in, host factors out: the timed region
includes every copy), against the compiled reference's factorization of ONE
layer (factorize_attention + three factor_rank_r, svd.cpp / factorize.cpp)
on this host's cores, scaled x12.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_01506_b200 import abi  # noqa: E402
from paper_2508_01506_b200 import factorize as F  # noqa: E402


def dense_layer(d, df, seed):
    rng = np.random.default_rng(seed)
    n = lambda *s, sc=1.0: (rng.standard_normal(s) * sc).astype(np.float32)  # noqa: E731
    return F.DenseLayerWeights(n(d, d, sc=d ** -.5), n(d, sc=.02), n(d, d, sc=d ** -.5),
                               n(d, sc=.02), n(d, d, sc=d ** -.5), n(d, sc=.02),
                               n(d, d, sc=d ** -.5), n(d, sc=.02), n(d, df, sc=d ** -.5),
                               n(df, sc=.02), n(df, d, sc=d ** -.5), n(d, sc=.02))


def main():
    d, df, heads, r, layers = 768, 3072, 12, 32, int(os.environ.get("LAYERS", "12"))
    dense = [dense_layer(d, df, 10 + l) for l in range(layers)]
    L = abi.lib()
    F.factorize_layers(dense[:1], heads, rank=r)  # warm-up (context, module load)
    t0 = time.perf_counter()
    out = F.factorize_layers(dense, heads, rank=r)
    gpu_s = time.perf_counter() - t0
    line = {"metric": "bert_base_factorization_seconds", "layers": layers, "gpu_s": round(gpu_s, 3),
            "sweeps": L.fsvd_last_factor_sweeps(),
            "matrices": layers * (3 * heads + 3), "ranks": {"r": r, "pr": 384, "fr": 384}}
    if os.environ.get("REF", "1") == "1":
        sys.path.insert(0, ROOT)
        import oracle
        if oracle.Reference.available():
            ref = oracle.Reference()
            w = dense[0]
            t0 = time.perf_counter()
            ru, rv, _ = ref.factorize_attention([w.wq, w.wk, w.wv], [w.bq, w.bk, w.bv], heads, r)
            t_attn = time.perf_counter() - t0
            err = float(np.abs(out[0].attn.u - ru).max())
            t1 = time.perf_counter()
            for mat, lin in ((w.wo, out[0].out_proj), (w.w_in, out[0].ffn.up),
                             (w.w_out, out[0].ffn.down)):
                u, v = ref.factor_rank_r(mat, lin.rank)
                err = max(err, float(np.abs(lin.u - u).max()), float(np.abs(lin.v - v).max()))
            t_lin = time.perf_counter() - t1
            line["reference_one_layer_s"] = round(t_attn + t_lin, 2)
            line["reference_model_s_est"] = round(layers * (t_attn + t_lin), 1)
            line["reference_threads"] = os.cpu_count()
            line["max_abs_diff_vs_reference_layer0"] = err
            line["speedup_est"] = round(layers * (t_attn + t_lin) / gpu_s, 1)
    print(json.dumps(line))


if __name__ == "__main__":
    main()
