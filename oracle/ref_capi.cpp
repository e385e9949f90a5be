// ref_capi.cpp -- C entry points into the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libfsvd_ref.so.  It only converts the flat C descriptors of
// include/fsvd_b200.h into the reference's own types and calls the
// reference's public API; no arithmetic lives here.  Used by tests/ to pin
// the C restatement (oracle/fsvd_oracle.c) and the GPU path, and by bench.py
// as the reference CPU arm (cpu_baseline kind "reference").
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "flashsvd/attention.hpp"
#include "flashsvd/encoder.hpp"
#include "flashsvd/model_io.hpp"
#include "flashsvd/factorize.hpp"
#include "flashsvd/ffn.hpp"
#include "flashsvd/memtier.hpp"
#include "flashsvd/planner.hpp"
#include "fsvd_b200.h"
#include "support/oracles.hpp"

using namespace flashsvd;

namespace {

thread_local std::string g_err;

struct MeterStats {
  size_t peak_transient, persistent, events;
};

Tensor vec(const float* p, size_t n) {
  return Tensor({n}, std::vector<float>(p, p + n));
}
Tensor mat(const float* p, size_t r, size_t c) {
  return Tensor({r, c}, std::vector<float>(p, p + r * c));
}
FactorizedLinear linear(const fsvd_linear_desc& d) {
  FactorizedLinear f;
  f.u = mat(d.u, d.in_dim, d.rank);
  f.v = mat(d.v, d.rank, d.out_dim);
  f.bias = vec(d.bias, d.out_dim);
  return f;
}
AttentionFactorSet attn_set(const fsvd_attn_desc& a) {
  AttentionFactorSet s;
  s.d_model = a.d_model;
  s.groups = a.groups;
  s.rank = a.rank;
  const size_t gd = a.d_model / a.groups;
  for (size_t m = 0; m < 3; ++m) {
    auto& dst = m == 0 ? s.q : m == 1 ? s.k : s.v;
    for (size_t g = 0; g < a.groups; ++g) {
      FactorizedLinear f;
      f.u = mat(a.u + (m * a.groups + g) * a.d_model * a.rank, a.d_model, a.rank);
      f.v = mat(a.v + (m * a.groups + g) * a.rank * gd, a.rank, gd);
      f.bias = vec(a.bias + (m * a.groups + g) * gd, gd);
      dst.push_back(std::move(f));
    }
  }
  return s;
}
FfnFactors ffn_set(const fsvd_ffn_desc& d) {
  FfnFactors f;
  f.up = linear(d.up);
  f.down = linear(d.down);
  f.activation = static_cast<Activation>(d.activation);
  return f;
}
// The descriptor's optional parts (include/fsvd_b200.h): factorized attention
// when attn.u is set, factorized FFN when ffn.up.u is set, dense weights when
// L.dense is set -- the reference EncoderLayer's optionals.
EncoderLayer layer_of(const fsvd_layer_desc& L) {
  EncoderLayer e;
  e.heads = L.heads;
  if (L.attn.u) {
    e.attn_factors = attn_set(L.attn);
    e.out_proj = linear(L.out_proj);
  }
  if (L.ffn.up.u) e.ffn_factors = ffn_set(L.ffn);
  const size_t d = L.attn.d_model;
  if (L.dense) {
    const fsvd_dense_layer& w = *L.dense;
    const size_t df = w.d_ff;
    e.attn_dense = DenseAttentionWeights{mat(w.wq, d, d), vec(w.bq, d), mat(w.wk, d, d),
                                         vec(w.bk, d),    mat(w.wv, d, d), vec(w.bv, d),
                                         mat(w.wo, d, d), vec(w.bo, d)};
    e.ffn_dense = DenseFfnWeights{mat(w.w_in, d, df), vec(w.b_in, df), mat(w.w_out, df, d),
                                  vec(w.b_out, d), static_cast<Activation>(L.ffn.activation)};
  }
  e.ln1.gamma = vec(L.ln1_gamma, d);
  e.ln1.beta = vec(L.ln1_beta, d);
  e.ln1.eps = L.ln1_eps;
  e.ln2.gamma = vec(L.ln2_gamma, d);
  e.ln2.beta = vec(L.ln2_beta, d);
  e.ln2.eps = L.ln2_eps;
  return e;
}
TilePlan plan_of(const fsvd_tile_plan* p) {
  TilePlan t;
  if (p) {
    t.bm = p->bm;
    t.br = p->br;
    t.bdf = p->bdf;
    t.sram_budget_bytes = p->sram_budget_bytes;
  }
  return t;
}
void stats(const MemoryMeter& m, size_t* out3) {
  if (!out3) return;
  out3[0] = m.peak_transient_bytes();
  out3[1] = m.persistent_bytes();
  out3[2] = m.events().size();
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.kind()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// tests/support/oracles.hpp:80-87 (the reference's canonical input generator)
void ref_random_fill(float* out, size_t n, uint64_t seed, double stddev) {
  Tensor t = oracle::random_tensor({n}, seed, stddev);
  std::memcpy(out, t.data(), n * sizeof(float));
}

int ref_flash_svd_attention(const float* x, size_t b, size_t m, const fsvd_attn_desc* a,
                            size_t heads, const fsvd_tile_plan* plan, float* out,
                            size_t* meter3) {
  return guard([&] {
    const size_t d = a->d_model;
    Tensor xt({b, m, d}, std::vector<float>(x, x + b * m * d));
    Tensor o({b, m, d});
    MemoryMeter meter;
    flash_svd_attention(xt, attn_set(*a), heads, plan_of(plan), meter, "attn", o);
    meter.assert_clean();
    std::memcpy(out, o.data(), o.numel() * sizeof(float));
    stats(meter, meter3);
  });
}

int ref_dense_attention_twin(const float* x, size_t b, size_t m, const fsvd_attn_desc* a,
                             size_t heads, float* out) {
  return guard([&] {
    const size_t d = a->d_model;
    AttentionFactorSet s = attn_set(*a);
    Tensor xt({b, m, d}, std::vector<float>(x, x + b * m * d));
    Tensor o({b, m, d});
    Tensor bias[3] = {Tensor({d}), Tensor({d}), Tensor({d})};
    for (int w = 0; w < 3; ++w) std::memcpy(bias[w].data(), a->bias + w * d, d * sizeof(float));
    MemoryMeter meter;
    dense_attention(xt, reconstruct_attention(s, Qkv::Q), bias[0],
                    reconstruct_attention(s, Qkv::K), bias[1],
                    reconstruct_attention(s, Qkv::V), bias[2], heads, meter, o);
    std::memcpy(out, o.data(), o.numel() * sizeof(float));
  });
}

int ref_lowrank_output_projection(const float* ctx, size_t b, size_t m,
                                  const fsvd_linear_desc* p, float* out, size_t* meter3) {
  return guard([&] {
    const size_t d = p->in_dim;
    Tensor ct({b, m, d}, std::vector<float>(ctx, ctx + b * m * d));
    Tensor o({b, m, p->out_dim});
    MemoryMeter meter;
    lowrank_output_projection(ct, linear(*p), meter, "attn", o);
    std::memcpy(out, o.data(), o.numel() * sizeof(float));
    stats(meter, meter3);
  });
}

int ref_ffn(int variant, const float* x, size_t b, size_t m, size_t d, const fsvd_ffn_desc* f,
            const fsvd_tile_plan* plan, float* out, size_t* meter3) {
  return guard([&] {
    Tensor xt({b, m, d}, std::vector<float>(x, x + b * m * d));
    Tensor o({b, m, d});
    MemoryMeter meter;
    FfnFactors ff = ffn_set(*f);
    if (variant == 1)
      ffn_v1(xt, ff, plan_of(plan), meter, "ffn", o);
    else if (variant == 2)
      ffn_v2(xt, ff, plan_of(plan), meter, "ffn", o);
    else if (variant == 0)
      ffn_dense(xt, reconstruct(ff.up), ff.up.bias, reconstruct(ff.down), ff.down.bias,
                ff.activation, meter, o);
    else
      ffn_naive_lowrank(xt, ff, meter, o);
    std::memcpy(out, o.data(), o.numel() * sizeof(float));
    stats(meter, meter3);
  });
}

// mode: fsvd_run_mode; Dense runs on dense_equivalent() of the layers.
int ref_run_model(const float* x, size_t b, size_t m, const fsvd_layer_desc* layers,
                  size_t n_layers, int mode, const fsvd_tile_plan* plan, int pre_ln,
                  float* out, size_t* meter3) {
  return guard([&] {
    const size_t d = layers[0].attn.d_model;
    std::vector<EncoderLayer> ls;
    for (size_t i = 0; i < n_layers; ++i) {
      EncoderLayer e = layer_of(layers[i]);
      // a factor-only layer in Dense mode runs its dense twin (the C-ABI's
      // documented extension); a layer carrying dense weights uses them
      ls.push_back(mode == FSVD_MODE_DENSE && !e.attn_dense ? dense_equivalent(e) : std::move(e));
    }
    Tensor xt({b, m, d}, std::vector<float>(x, x + b * m * d));
    Tensor o({b, m, d});
    MemoryMeter meter;
    LayerRunOptions opts;
    opts.pre_layer_norm = pre_ln != 0;
    run_model(xt, ls, static_cast<RunMode>(mode), plan_of(plan), meter, o, opts);
    meter.assert_clean();
    std::memcpy(out, o.data(), o.numel() * sizeof(float));
    stats(meter, meter3);
  });
}

int ref_run_layer(const float* x, size_t b, size_t m, const fsvd_layer_desc* L, int mode,
                  const fsvd_tile_plan* plan, int pre_ln, float* out, size_t* meter3) {
  return guard([&] {
    const size_t d = L->attn.d_model;
    EncoderLayer e = layer_of(*L);
    if (mode == FSVD_MODE_DENSE && !e.attn_dense) e = dense_equivalent(e);
    Tensor xt({b, m, d}, std::vector<float>(x, x + b * m * d));
    Tensor o({b, m, d});
    MemoryMeter meter;
    LayerRunOptions opts;
    opts.pre_layer_norm = pre_ln != 0;
    run_layer(xt, e, static_cast<RunMode>(mode), plan_of(plan), meter, o, opts);
    meter.assert_clean();
    std::memcpy(out, o.data(), o.numel() * sizeof(float));
    stats(meter, meter3);
  });
}

int ref_validate_tile_plan(const fsvd_tile_plan* plan, int kind, const fsvd_geometry* g,
                           size_t* bytes) {
  return guard([&] {
    Geometry geo{g->batch, g->seq_len, g->d_model, g->d_ff, g->heads, g->groups, g->rank,
                 g->layers};
    *bytes = validate_tile_plan(plan_of(plan), static_cast<KernelKind>(kind), geo);
  });
}

size_t ref_expected_bytes(int formula, const fsvd_geometry* g) {
  Geometry geo{g->batch, g->seq_len, g->d_model, g->d_ff, g->heads, g->groups, g->rank,
               g->layers};
  return expected_bytes(static_cast<FormulaId>(formula), geo);
}

// planner.cpp:60-79 (uniform-rank FLOP count used by the reference bench)
// planner.cpp:89-98
int ref_io_bytes(const fsvd_geometry* g, int mode, unsigned long long* in, unsigned long long* out) {
  return guard([&] {
    Geometry geo{g->batch, g->seq_len, g->d_model, g->d_ff, g->heads, g->groups, g->rank,
                 g->layers};
    IoBytes io = io_bytes(geo, static_cast<RunMode>(mode));
    *in = io.in;
    *out = io.out;
  });
}
int ref_flops_exact_checked(const fsvd_geometry* g, int mode, unsigned long long* f) {
  return guard([&] {
    Geometry geo{g->batch, g->seq_len, g->d_model, g->d_ff, g->heads, g->groups, g->rank,
                 g->layers};
    *f = flops_exact(geo, static_cast<RunMode>(mode));
  });
}
unsigned long long ref_flops_exact(const fsvd_geometry* g, int mode) {
  Geometry geo{g->batch, g->seq_len, g->d_model, g->d_ff, g->heads, g->groups, g->rank,
               g->layers};
  return flops_exact(geo, static_cast<RunMode>(mode));
}

// FSVD1 (model_io.hpp): writes the layers with the reference's own
// save_model (canonical names, JSON sidecar at <path>.json).
int ref_save_model(const char* path, const fsvd_layer_desc* layers, size_t n_layers) {
  return guard([&] {
    std::vector<EncoderLayer> ls;
    for (size_t i = 0; i < n_layers; ++i) ls.push_back(layer_of(layers[i]));
    save_model(path, ls);
  });
}
// model_io.cpp:268-345 load_model (assemble + EncoderLayer::validate);
// returns the reference's status and the number of layers assembled.
int ref_load_model(const char* path, size_t* n_layers) {
  return guard([&] {
    std::vector<EncoderLayer> ls = load_model(path);
    if (n_layers) *n_layers = ls.size();
  });
}

// Byte offset of the FormatError the reference reader raises for `path`
// (-1: the container parsed; -2: another error).
long long ref_read_error_offset(const char* path) {
  try {
    read_tensor_file(path);
    return -1;
  } catch (const FormatError& e) {
    return static_cast<long long>(e.byte_offset());
  } catch (...) {
    return -2;
  }
}

// planner.cpp:123-141 -- decoder closed forms; which 0 kv cache, 1 prefill,
// 2 decode step at t.  Returns the reference's status (0 ok).
int ref_decoder_bytes(int which, const fsvd_geometry* g, size_t t, size_t* out) {
  return guard([&] {
    Geometry geo{g->batch, g->seq_len, g->d_model, g->d_ff, g->heads, g->groups, g->rank,
                 g->layers};
    *out = which == 0 ? decoder_kv_cache_bytes(geo)
                      : which == 1 ? decoder_prefill_bytes(geo) : decoder_decode_step_bytes(geo, t);
  });
}
// svd.cpp:412-456 -- leading-r even-split factors of a row-major m x n matrix.
int ref_factor_rank_r(const float* a, size_t m, size_t n, size_t r, float* u, float* v) {
  return guard([&] {
    LowRankPair p = factor_rank_r(mat(a, m, n), r);
    std::memcpy(u, p.u.data(), m * r * sizeof(float));
    std::memcpy(v, p.v.data(), r * n * sizeof(float));
  });
}
// svd.cpp:260-302 -- full thin SVD (float outputs; p = min(m, n)).
int ref_svd(const float* a, size_t m, size_t n, float* u, float* s, float* vt) {
  return guard([&] {
    SvdResult f = svd(mat(a, m, n));
    const size_t p = f.s.size();
    std::memcpy(u, f.u.data(), m * p * sizeof(float));
    std::memcpy(s, f.s.data(), p * sizeof(float));
    std::memcpy(vt, f.vt.data(), p * n * sizeof(float));
  });
}
// factorize.cpp:21-64 -- per-group factors written in the fsvd_attn_desc
// layout: u [3][G][d][r], v [3][G][r][d/G], bias [3][G][d/G].
int ref_factorize_attention(const float* wq, const float* bq, const float* wk, const float* bk,
                            const float* wv, const float* bv, size_t d, size_t groups,
                            size_t rank, float* u, float* v, float* bias) {
  return guard([&] {
    AttentionFactorSet s = factorize_attention(mat(wq, d, d), vec(bq, d), mat(wk, d, d),
                                               vec(bk, d), mat(wv, d, d), vec(bv, d), groups,
                                               rank);
    const size_t gd = d / groups;
    for (size_t m = 0; m < 3; ++m)
      for (size_t g = 0; g < groups; ++g) {
        const FactorizedLinear& f = (m == 0 ? s.q : m == 1 ? s.k : s.v)[g];
        const size_t i = m * groups + g;
        std::memcpy(u + i * d * rank, f.u.data(), d * rank * sizeof(float));
        std::memcpy(v + i * rank * gd, f.v.data(), rank * gd * sizeof(float));
        std::memcpy(bias + i * gd, f.bias.data(), gd * sizeof(float));
      }
  });
}

}  // extern "C"
