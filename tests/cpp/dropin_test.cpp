// dropin_test.cpp -- the C++ drop-in (include/flashsvd_b200/flashsvd_b200.hpp)
// used exactly as a reference-side caller would: reference types, reference
// MemoryMeter, reference signatures.  Every case runs the reference's own CPU
// function and flashsvd::b200's GPU function on identical inputs and checks
//   * outputs: rel = max|got - ref| / max|ref| <= 1e-4 (fp32 policy) or
//     <= 2e-2 (bf16 policy, inputs pre-rounded to bf16 on both sides);
//   * the meter: identical peak transient, persistent bytes and event log;
//   * the error contract: same exception type for bad inputs.
// Built by tests/cpp/Makefile against the reference objects in oracle/_ref
// (test infrastructure); run by tests/test_gpu_dropin.py on the GPU box.
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "flashsvd/attention.hpp"
#include "flashsvd/encoder.hpp"
#include "flashsvd/factorize.hpp"
#include "flashsvd/ffn.hpp"
#include "flashsvd_b200/flashsvd_b200.hpp"
#include "support/oracles.hpp"

using namespace flashsvd;

namespace {

int g_fail = 0, g_pass = 0;

void report(const std::string& name, bool ok, const std::string& detail) {
  std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.c_str());
  (ok ? g_pass : g_fail)++;
}

float bf16_round(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}
void round_tensor(Tensor& t) {
  for (std::size_t i = 0; i < t.numel(); ++i) t.at(i) = bf16_round(t.at(i));
}

double rel(const Tensor& got, const Tensor& ref) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < ref.numel(); ++i) {
    num = std::max(num, std::abs(double(got.at(i)) - double(ref.at(i))));
    den = std::max(den, std::abs(double(ref.at(i))));
  }
  return den > 0 ? num / den : num;
}

// Acceptance-style factor synthesis (U ~ N(0, 1/sqrt(in)), V ~ N(0, 1/sqrt(r)),
// bias ~ N(0, 0.02), LN gamma = 1 + N(0, 0.1)), seeded like acceptance.cpp.
FactorizedLinear lin(std::size_t in, std::size_t out, std::size_t r, uint64_t seed) {
  FactorizedLinear f;
  f.u = oracle::random_tensor({in, r}, seed, 1.0 / std::sqrt(double(in)));
  f.v = oracle::random_tensor({r, out}, seed + 1, 1.0 / std::sqrt(double(r)));
  f.bias = oracle::random_tensor({out}, seed + 2, 0.02);
  return f;
}
AttentionFactorSet attn_set(std::size_t d, std::size_t G, std::size_t r, uint64_t seed) {
  AttentionFactorSet s;
  s.d_model = d;
  s.groups = G;
  s.rank = r;
  for (int m = 0; m < 3; ++m)
    for (std::size_t g = 0; g < G; ++g) {
      auto& dst = m == 0 ? s.q : m == 1 ? s.k : s.v;
      dst.push_back(lin(d, d / G, r, seed));
      seed += 3;
    }
  return s;
}
FfnFactors ffn_set(std::size_t d, std::size_t df, std::size_t r, uint64_t seed, Activation a) {
  FfnFactors f;
  f.up = lin(d, df, r, seed);
  f.down = lin(df, d, r, seed + 10);
  f.activation = a;
  return f;
}
EncoderLayer layer_of(std::size_t d, std::size_t df, std::size_t H, std::size_t G, std::size_t r,
                      std::size_t pr, std::size_t fr, uint64_t seed) {
  EncoderLayer l;
  l.heads = H;
  l.attn_factors = attn_set(d, G, r, seed);
  l.out_proj = lin(d, d, pr, seed + 500);
  l.ffn_factors = ffn_set(d, df, fr, seed + 600, Activation::GeluErf);
  auto norm = [&](uint64_t s) {
    LayerNormParams p;
    p.gamma = oracle::random_tensor({d}, s, 0.1);
    for (std::size_t i = 0; i < d; ++i) p.gamma.at(i) += 1.0f;
    p.beta = oracle::random_tensor({d}, s + 1, 0.02);
    return p;
  };
  l.ln1 = norm(seed + 700);
  l.ln2 = norm(seed + 710);
  return l;
}
void round_linear(FactorizedLinear& f) {
  round_tensor(f.u);
  round_tensor(f.v);
  round_tensor(f.bias);
}
void round_layer(EncoderLayer& l) {
  for (auto* v : {&l.attn_factors->q, &l.attn_factors->k, &l.attn_factors->v})
    for (auto& f : *v) round_linear(f);
  round_linear(*l.out_proj);
  round_linear(l.ffn_factors->up);
  round_linear(l.ffn_factors->down);
  for (auto* t : {&l.ln1.gamma, &l.ln1.beta, &l.ln2.gamma, &l.ln2.beta}) round_tensor(*t);
}

std::string meter_diff(const MemoryMeter& a, const MemoryMeter& b) {
  if (a.peak_transient_bytes() != b.peak_transient_bytes())
    return "peak " + std::to_string(a.peak_transient_bytes()) + " vs " +
           std::to_string(b.peak_transient_bytes());
  if (a.persistent_bytes() != b.persistent_bytes())
    return "persistent " + std::to_string(a.persistent_bytes()) + " vs " +
           std::to_string(b.persistent_bytes());
  const auto ea = a.events(), eb = b.events();
  if (ea.size() != eb.size())
    return "event count " + std::to_string(ea.size()) + " vs " + std::to_string(eb.size());
  for (std::size_t i = 0; i < ea.size(); ++i)
    if (ea[i].kind != eb[i].kind || ea[i].tag != eb[i].tag || ea[i].bytes != eb[i].bytes ||
        (ea[i].kind == MeterEventKind::Alloc && ea[i].cls != eb[i].cls))
      return "event " + std::to_string(i) + " (" + ea[i].tag + " vs " + eb[i].tag + ")";
  try {
    b.assert_clean();
  } catch (const Error& e) {
    return std::string("assert_clean: ") + e.what();
  }
  return "";
}

void compare(const std::string& name, double tol, const std::function<void(MemoryMeter&, Tensor&)>& ref,
             const std::function<void(MemoryMeter&, Tensor&)>& got, Tensor out_ref, Tensor out_got) {
  MemoryMeter mr, mg;
  ref(mr, out_ref);
  got(mg, out_got);
  const double e = rel(out_got, out_ref);
  const std::string md = meter_diff(mr, mg);
  char buf[160];
  std::snprintf(buf, sizeof(buf), "rel=%.3e tol=%.0e peak=%zu persistent=%zu %s", e, tol,
                mg.peak_transient_bytes(), mg.persistent_bytes(), md.c_str());
  report(name, std::isfinite(e) && e <= tol && md.empty(), buf);
}

template <typename E>
void expect_throw(const std::string& name, const std::function<void()>& fn) {
  try {
    fn();
  } catch (const E&) {
    report(name, true, "");
    return;
  } catch (const std::exception& e) {
    report(name, false, std::string("wrong exception: ") + e.what());
    return;
  }
  report(name, false, "no exception");
}

}  // namespace

int main() {
  const TilePlan plan{16, 16, 32, 1u << 22};
  struct Shape {
    const char* name;
    std::size_t d, df, H, G, r, pr, fr, B, M;
  };
  const Shape shapes[] = {
      {"tiny-grouped", 48, 96, 4, 2, 5, 7, 9, 2, 33},
      {"bert-head-r32", 256, 512, 4, 4, 32, 64, 128, 2, 130},
      {"bert-base-cfg1", 768, 3072, 12, 12, 32, 384, 384, 1, 128},
  };
  for (const fsvd_dtype dt : {FSVD_F32, FSVD_BF16}) {
    b200::set_precision(dt);
    const double tol = dt == FSVD_F32 ? 1e-4 : 2e-2;
    const std::string sfx = dt == FSVD_F32 ? " [f32]" : " [bf16]";
    for (const Shape& s : shapes) {
      EncoderLayer l = layer_of(s.d, s.df, s.H, s.G, s.r, s.pr, s.fr, 800000 + s.d);
      Tensor x = oracle::random_tensor({s.B, s.M, s.d}, 90000 + s.M, 1.0);
      if (dt == FSVD_BF16) {
        round_layer(l);
        round_tensor(x);
      }
      const Tensor shape_like({s.B, s.M, s.d});
      const std::string n = std::string(s.name) + sfx;
      compare("flash_svd_attention " + n, tol,
              [&](MemoryMeter& m, Tensor& o) {
                flash_svd_attention(x, *l.attn_factors, s.H, plan, m, "attn", o);
              },
              [&](MemoryMeter& m, Tensor& o) {
                b200::flash_svd_attention(x, *l.attn_factors, s.H, plan, m, "attn", o);
              },
              shape_like, shape_like);
      compare("lowrank_output_projection " + n, tol,
              [&](MemoryMeter& m, Tensor& o) { lowrank_output_projection(x, *l.out_proj, m, "o", o); },
              [&](MemoryMeter& m, Tensor& o) {
                b200::lowrank_output_projection(x, *l.out_proj, m, "o", o);
              },
              shape_like, shape_like);
      compare("ffn_v1 " + n, tol,
              [&](MemoryMeter& m, Tensor& o) { ffn_v1(x, *l.ffn_factors, plan, m, "ffn", o); },
              [&](MemoryMeter& m, Tensor& o) { b200::ffn_v1(x, *l.ffn_factors, plan, m, "ffn", o); },
              shape_like, shape_like);
      compare("ffn_v2 " + n, tol,
              [&](MemoryMeter& m, Tensor& o) { ffn_v2(x, *l.ffn_factors, plan, m, "ffn", o); },
              [&](MemoryMeter& m, Tensor& o) { b200::ffn_v2(x, *l.ffn_factors, plan, m, "ffn", o); },
              shape_like, shape_like);
      for (const RunMode mode : {RunMode::FlashV1, RunMode::FlashV2})
        for (const bool pre : {false, true}) {
          LayerRunOptions opts;
          opts.pre_layer_norm = pre;
          compare(std::string("run_layer ") + mode_name(mode) + (pre ? " pre-LN " : " post-LN ") + n,
                  tol,
                  [&](MemoryMeter& m, Tensor& o) { run_layer(x, l, mode, plan, m, o, opts); },
                  [&](MemoryMeter& m, Tensor& o) { b200::run_layer(x, l, mode, plan, m, o, opts); },
                  shape_like, shape_like);
        }
      std::vector<EncoderLayer> model{l, layer_of(s.d, s.df, s.H, s.G, s.r, s.pr, s.fr, 801013)};
      if (dt == FSVD_BF16) round_layer(model[1]);
      compare(std::string("run_model x2 ") + n, tol,
              [&](MemoryMeter& m, Tensor& o) { run_model(x, model, RunMode::FlashV2, plan, m, o); },
              [&](MemoryMeter& m, Tensor& o) {
                b200::run_model(x, model, RunMode::FlashV2, plan, m, o);
              },
              shape_like, shape_like);
    }
  }

  // factorization (svd.cpp / factorize.cpp): device factors vs the reference's
  // own Jacobi, 1e-5 absolute (test_tensor.cpp:276-287's bar)
  {
    auto maxdiff = [](const Tensor& a, const Tensor& b) {
      double d = 0.0;
      for (std::size_t i = 0; i < a.numel(); ++i)
        d = std::max(d, std::abs(double(a.at(i)) - double(b.at(i))));
      return d;
    };
    for (const auto& c : std::vector<std::array<std::size_t, 3>>{
             {8, 8, 3}, {40, 8, 4}, {8, 40, 4}, {96, 96, 48}, {300, 64, 32}}) {
      Tensor a = oracle::random_tensor({c[0], c[1]}, 77 + c[0] + c[1], 1.0);
      LowRankPair ref = factor_rank_r(a, c[2]);
      LowRankPair got = b200::factor_rank_r(a, c[2]);
      const double du = maxdiff(got.u, ref.u), dv = maxdiff(got.v, ref.v);
      report("factor_rank_r " + std::to_string(c[0]) + "x" + std::to_string(c[1]) + " r" +
                 std::to_string(c[2]),
             du < 1e-5 && dv < 1e-5, "du=" + std::to_string(du) + " dv=" + std::to_string(dv));
    }
    const std::size_t d = 64, G = 4, r = 8;
    Tensor wq = oracle::random_tensor({d, d}, 11, 0.125), wk = oracle::random_tensor({d, d}, 12, 0.125),
           wv = oracle::random_tensor({d, d}, 13, 0.125), bq = oracle::random_tensor({d}, 14, 0.02),
           bk = oracle::random_tensor({d}, 15, 0.02), bv = oracle::random_tensor({d}, 16, 0.02);
    AttentionFactorSet ref = factorize_attention(wq, bq, wk, bk, wv, bv, G, r);
    AttentionFactorSet got = b200::factorize_attention(wq, bq, wk, bk, wv, bv, G, r);
    double worst = 0.0;
    for (std::size_t g = 0; g < G; ++g)
      for (const auto* pr : {&ref.q, &ref.k, &ref.v}) {
        const auto& gg = pr == &ref.q ? got.q : pr == &ref.k ? got.k : got.v;
        worst = std::max({worst, maxdiff(gg[g].u, (*pr)[g].u), maxdiff(gg[g].v, (*pr)[g].v),
                          maxdiff(gg[g].bias, (*pr)[g].bias)});
      }
    report("factorize_attention 64/G4/r8", worst < 1e-5, "max=" + std::to_string(worst));
    Tensor w = oracle::random_tensor({48, 80}, 21, 0.1);
    expect_throw<RankError>("factor_rank_r rank 0 -> RankError",
                            [&] { (void)b200::factor_rank_r(w, 0); });
    expect_throw<RankError>("factor_rank_r rank > min -> RankError",
                            [&] { (void)b200::factor_rank_r(w, 49); });
    expect_throw<ConfigError>("factorize_attention groups 5 -> ConfigError",
                              [&] { (void)b200::factorize_attention(wq, bq, wk, bk, wv, bv, 5, 2); });
  }

  // error contract (errors.hpp): same exception types as the reference
  b200::set_precision(FSVD_F32);
  EncoderLayer l = layer_of(48, 96, 4, 2, 5, 7, 9, 5);
  Tensor x = oracle::random_tensor({2, 9, 48}, 1, 1.0);
  MemoryMeter m;
  Tensor bad({2, 9, 40});
  expect_throw<ShapeError>("attention out shape mismatch -> ShapeError", [&] {
    b200::flash_svd_attention(x, *l.attn_factors, 4, plan, m, "a", bad);
  });
  expect_throw<ConfigError>("heads % groups -> ConfigError", [&] {
    Tensor o({2, 9, 48});
    b200::flash_svd_attention(x, *l.attn_factors, 3, plan, m, "a", o);
  });
  expect_throw<BudgetError>("tile plan over budget -> BudgetError", [&] {
    Tensor o({2, 9, 48});
    b200::ffn_v2(x, *l.ffn_factors, TilePlan{16, 16, 64, 1024}, m, "f", o);
  });
  expect_throw<ConfigError>("ffn up/down rank mismatch -> ConfigError", [&] {
    FfnFactors f = *l.ffn_factors;
    f.down = lin(96, 48, 4, 9);
    Tensor o({2, 9, 48});
    b200::ffn_v1(x, f, plan, m, "f", o);
  });
  expect_throw<ConfigError>("run_layer out aliases x -> ConfigError", [&] {
    b200::run_layer(x, l, RunMode::FlashV1, plan, m, x);
  });

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
