/*
 * fsvd_oracle.c -- plain-C restatement of the reference FlashSVD path.
 *
 * TEST INFRASTRUCTURE ONLY (see fsvd_oracle.h).  Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * Arithmetic is kept in the reference's exact order: every GEMM accumulates
 * its k terms in ascending order onto a zero or preloaded bias, exactly like
 * gemm_acc_ld (attention.cpp:19-31) / gemm_accumulate (tensor.cpp:32-46).
 * Build with -ffp-contract=off so no FMA contraction changes rounding.
 */
#include "fsvd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- */
/* tests/support/oracles.hpp:50-87 -- mt19937_64 + Box-Muller        */
/* ---------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} fo_gauss;

static void mt_seed(fo_gauss* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
  g->have_spare = 0;
  g->spare = 0.0;
}

static uint64_t mt_next(fo_gauss* g) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  if (g->idx >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[i + 1] & 0x7FFFFFFFULL);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[i + 1] & 0x7FFFFFFFULL);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (g->mt[311] & 0xFFFFFFFF80000000ULL) | (g->mt[0] & 0x7FFFFFFFULL);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag[x & 1ULL];
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

static double uniform01(fo_gauss* g) {
  return (double)(mt_next(g) >> 11) * (1.0 / 9007199254740992.0);
}

static double gauss_next(fo_gauss* g, double stddev) {
  if (g->have_spare) {
    g->have_spare = 0;
    return g->spare * stddev;
  }
  double u1, u2;
  do {
    u1 = uniform01(g);
  } while (u1 <= 1.0e-300);
  u2 = uniform01(g);
  const double mag = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586476925286766559 * u2;
  g->spare = mag * sin(ang);
  g->have_spare = 1;
  return mag * cos(ang) * stddev;
}

void fo_random_fill(float* out, size_t n, uint64_t seed, double stddev) {
  fo_gauss* g = (fo_gauss*)malloc(sizeof(fo_gauss));
  mt_seed(g, seed);
  for (size_t i = 0; i < n; ++i) out[i] = (float)gauss_next(g, stddev);
  free(g);
}

/* ---------------------------------------------------------------- */
/* Elementwise semantics (tensor.cpp:64-102, ffn.cpp:16-24)            */
/* ---------------------------------------------------------------- */
static float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f)); }
static float gelu_tanh(float x) {
  const float c = 0.79788456080286535588f;
  float inner = c * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(inner));
}
static float apply_act(float v, int act) {
  switch (act) {
    case FSVD_ACT_GELU_ERF: return gelu_erf(v);
    case FSVD_ACT_GELU_TANH: return gelu_tanh(v);
    case FSVD_ACT_RELU: return v > 0.0f ? v : 0.0f;
    default: return v;
  }
}
/* std::max(a, b) == (a < b) ? b : a */
static float fmax_std(float a, float b) { return (a < b) ? b : a; }

static void layer_norm_row(const float* x, float* y, size_t n, const float* gamma,
                           const float* beta, float eps) {
  float mean = 0.0f;
  for (size_t j = 0; j < n; ++j) mean += x[j];
  mean /= (float)n;
  float var = 0.0f;
  for (size_t j = 0; j < n; ++j) {
    float d = x[j] - mean;
    var += d * d;
  }
  var /= (float)n;
  float inv = 1.0f / sqrtf(var + eps);
  for (size_t j = 0; j < n; ++j) y[j] = gamma[j] * ((x[j] - mean) * inv) + beta[j];
}

/* attention.cpp:19-31: C += A * B with leading dimensions, k ascending. */
static void gemm_acc_ld(const float* a, size_t lda, const float* b, size_t ldb, float* c,
                        size_t ldc, size_t m, size_t k, size_t n) {
  for (size_t i = 0; i < m; ++i) {
    float* ci = c + i * ldc;
    const float* ai = a + i * lda;
    for (size_t kk = 0; kk < k; ++kk) {
      const float av = ai[kk];
      const float* bk = b + kk * ldb;
      for (size_t j = 0; j < n; ++j) ci[j] += av * bk[j];
    }
  }
}

/* attention.cpp:34-45: c = a * b^T */
static void gemm_nt(const float* a, const float* b, float* c, size_t m, size_t k, size_t n) {
  for (size_t i = 0; i < m; ++i) {
    const float* ai = a + i * k;
    for (size_t j = 0; j < n; ++j) {
      const float* bj = b + j * k;
      float acc = 0.0f;
      for (size_t d = 0; d < k; ++d) acc += ai[d] * bj[d];
      c[i * n + j] = acc;
    }
  }
}

/* ---------------------------------------------------------------- */
/* memtier.cpp:125-212 -- working sets and closed forms               */
/* ---------------------------------------------------------------- */
size_t fo_tile_working_set(const fsvd_tile_plan* plan, int kind, const fsvd_geometry* g,
                           int* status) {
  *status = 0;
  if (plan->bm == 0 || plan->br == 0 || plan->bdf == 0) {
    *status = FSVD_ERR_CONFIG;
    return 0;
  }
  const size_t bm = plan->bm, br = plan->br, bdf = plan->bdf;
  const size_t gd = g->d_model / g->groups, r = g->rank;
  size_t floats = 0;
  if (kind == FSVD_KERNEL_ATTENTION) {
    floats = bm * gd + br * gd + br * gd + bm * br + bm * br + bm * gd +
             (bm > br ? bm : br) * gd + bm + bm + gd;
  } else if (kind == FSVD_KERNEL_FFN_V1) {
    floats = bm * bdf + bm * r + bm * r + r * bdf + bdf * r + bdf;
  } else {
    floats = bm * bdf + bm * r + bm * r + bm * r + r * bdf + bdf * r + bdf + g->d_model;
  }
  const size_t bytes = 4 * floats;
  if (bytes > plan->sram_budget_bytes) *status = FSVD_ERR_BUDGET;
  return bytes;
}

size_t fo_expected_bytes(int id, const fsvd_geometry* g) {
  const size_t b = g->batch, m = g->seq_len, da = g->d_model, df = g->d_ff, h = g->heads,
               gr = g->groups, r = g->rank;
  switch (id) {
    case FSVD_FORMULA_DENSE_ATTN: return 4 * (3 * b * m * da + b * h * m * m);
    case FSVD_FORMULA_FLASH_ATTN_DENSE_QKV: return 4 * (3 * b * m * da);
    case FSVD_FORMULA_FLASH_SVD_ATTN: return 4 * (3 * h * b * m * r);
    case FSVD_FORMULA_GROUPED_ATTN: return 4 * (3 * gr * b * m * r);
    case FSVD_FORMULA_FFN_DENSE:
    case FSVD_FORMULA_FFN_NAIVE_LOWRANK: return 4 * (b * m * df);
    case FSVD_FORMULA_FFN_V1: return 4 * (2 * b * m * r);
    default: return 0;
  }
}

size_t fo_flash_layer_peak_transient_bytes(const fsvd_geometry* g) {
  return 4 * 3 * g->groups * g->batch * g->seq_len * g->rank;
}
size_t fo_flash_layer_persistent_bytes(const fsvd_geometry* g) {
  return 4 * g->rank * (7 * g->d_model + 2 * g->d_ff);
}

/* ---------------------------------------------------------------- */
/* attention.cpp:202-269 + online_softmax_head :92-137                */
/* ---------------------------------------------------------------- */
int fo_flash_svd_attention(const float* x, size_t batch, size_t seq,
                           const fsvd_attn_desc* set, size_t heads,
                           const fsvd_tile_plan* plan, float* out) {
  const size_t d = set->d_model, groups = set->groups, rank = set->rank;
  if (heads == 0 || d % heads != 0) return FSVD_ERR_CONFIG;
  if (groups == 0 || heads % groups != 0) return FSVD_ERR_CONFIG;
  {
    fsvd_geometry g = {batch, seq, d, 1, heads, heads, 1, 1};
    int st;
    fo_tile_working_set(plan, FSVD_KERNEL_ATTENTION, &g, &st);
    if (st) return st;
  }
  const size_t dh = d / heads, gd = d / groups, hpg = heads / groups;
  const size_t bm = plan->bm, br = plan->br;

  /* projection phase :228-247 -- P[mat][g][b][m][r] = X_b * U[mat][g] */
  const size_t pn = groups * batch * seq * rank;
  float* proj = (float*)calloc(3 * pn, sizeof(float));
  for (size_t mat = 0; mat < 3; ++mat)
    for (size_t g = 0; g < groups; ++g)
      for (size_t b = 0; b < batch; ++b)
        gemm_acc_ld(x + b * seq * d, d, set->u + (mat * groups + g) * d * rank, rank,
                    proj + mat * pn + ((g * batch + b) * seq) * rank, rank, seq, d, rank);

  const float scale = 1.0f / sqrtf((float)dh);
  float* q = (float*)malloc(bm * dh * sizeof(float));
  float* k = (float*)malloc(br * dh * sizeof(float));
  float* v = (float*)malloc(br * dh * sizeof(float));
  float* score = (float*)malloc(bm * br * sizeof(float));
  float* prob = (float*)malloc(bm * br * sizeof(float));
  float* acc = (float*)malloc(bm * dh * sizeof(float));
  float* row_max = (float*)malloc(bm * sizeof(float));
  float* row_sum = (float*)malloc(bm * sizeof(float));

  for (size_t b = 0; b < batch; ++b)
    for (size_t h = 0; h < heads; ++h) {
      const size_t g = h / hpg;
      const size_t head_col = (h % hpg) * dh;
      /* load lambda :254-264: bias preload, then rank accumulate */
#define FO_LOAD(which, row0, rows, dest)                                                  \
  do {                                                                                    \
    const float* prows = proj + (which) * pn + ((g * batch + b) * seq + (row0)) * rank;   \
    const float* bias = set->bias + ((which) * groups + g) * gd + head_col;              \
    for (size_t i_ = 0; i_ < (rows); ++i_) memcpy((dest) + i_ * dh, bias, sizeof(float) * dh); \
    gemm_acc_ld(prows, rank, set->v + ((which) * groups + g) * rank * gd + head_col, gd, \
                (dest), dh, (rows), rank, dh);                                            \
  } while (0)
      float* out_base = out + b * seq * d + h * dh;
      for (size_t m0 = 0; m0 < seq; m0 += bm) {
        const size_t mlen = (bm < seq - m0) ? bm : seq - m0;
        FO_LOAD(0, m0, mlen, q);
        for (size_t i = 0; i < mlen * dh; ++i) q[i] *= scale;
        memset(acc, 0, mlen * dh * sizeof(float));
        for (size_t i = 0; i < mlen; ++i) {
          row_sum[i] = 0.0f;
          row_max[i] = -INFINITY;
        }
        for (size_t n0 = 0; n0 < seq; n0 += br) {
          const size_t nlen = (br < seq - n0) ? br : seq - n0;
          FO_LOAD(1, n0, nlen, k);
          FO_LOAD(2, n0, nlen, v);
          gemm_nt(q, k, score, mlen, dh, nlen);
          for (size_t i = 0; i < mlen; ++i) {
            const float* srow = score + i * nlen;
            float tile_max = srow[0];
            for (size_t j = 1; j < nlen; ++j) tile_max = fmax_std(tile_max, srow[j]);
            const float m_new = fmax_std(row_max[i], tile_max);
            const float alpha = expf(row_max[i] - m_new);
            float* prow = prob + i * nlen;
            float part = 0.0f;
            for (size_t j = 0; j < nlen; ++j) {
              prow[j] = expf(srow[j] - m_new);
              part += prow[j];
            }
            row_sum[i] = row_sum[i] * alpha + part;
            float* arow = acc + i * dh;
            for (size_t dd = 0; dd < dh; ++dd) arow[dd] *= alpha;
            row_max[i] = m_new;
          }
          gemm_acc_ld(prob, nlen, v, dh, acc, dh, mlen, nlen, dh);
        }
        for (size_t i = 0; i < mlen; ++i) {
          float* orow = out_base + (m0 + i) * d;
          const float inv = 1.0f / row_sum[i];
          for (size_t dd = 0; dd < dh; ++dd) orow[dd] = acc[i * dh + dd] * inv;
        }
      }
#undef FO_LOAD
    }
  free(q); free(k); free(v); free(score); free(prob); free(acc); free(row_max); free(row_sum);
  free(proj);
  return 0;
}

/* attention.cpp:366-391 */
int fo_lowrank_output_projection(const float* ctx, size_t batch, size_t seq,
                                 const fsvd_linear_desc* proj, float* out) {
  const size_t d = proj->in_dim, rank = proj->rank;
  if (proj->out_dim != d) return FSVD_ERR_SHAPE;
  float* p = (float*)calloc(batch * seq * rank, sizeof(float));
  for (size_t b = 0; b < batch; ++b) {
    gemm_acc_ld(ctx + b * seq * d, d, proj->u, rank, p + b * seq * rank, rank, seq, d, rank);
    float* orow = out + b * seq * d;
    for (size_t i = 0; i < seq; ++i) memcpy(orow + i * d, proj->bias, sizeof(float) * d);
    gemm_acc_ld(p + b * seq * rank, rank, proj->v, d, orow, d, seq, rank, d);
  }
  free(p);
  return 0;
}

/* ffn.cpp:84-104 -- z += act(p * V_up[:, blk] + b_up[blk]) * U_down[blk, :] */
static void stream_feature_blocks(const float* p, size_t rows, const fsvd_ffn_desc* f,
                                  size_t bdf, float* h, float* v1_panel, float* u2_panel,
                                  float* z) {
  const size_t rank = f->up.rank, d_ff = f->up.out_dim;
  for (size_t f0 = 0; f0 < d_ff; f0 += bdf) {
    const size_t flen = (bdf < d_ff - f0) ? bdf : d_ff - f0;
    for (size_t kk = 0; kk < rank; ++kk)
      memcpy(v1_panel + kk * flen, f->up.v + kk * d_ff + f0, sizeof(float) * flen);
    memcpy(u2_panel, f->down.u + f0 * rank, sizeof(float) * flen * rank);
    memset(h, 0, rows * flen * sizeof(float));
    gemm_acc_ld(p, rank, v1_panel, flen, h, flen, rows, rank, flen);
    for (size_t i = 0; i < rows; ++i)
      for (size_t j = 0; j < flen; ++j)
        h[i * flen + j] = apply_act(h[i * flen + j] + f->up.bias[f0 + j], f->activation);
    gemm_acc_ld(h, flen, u2_panel, rank, z, rank, rows, flen, rank);
  }
}

/* ffn.cpp:118-185 (both variants produce identical bits; V2 recomputes the
 * rank projection per tile exactly as V1 computes it globally). */
int fo_ffn(int variant, const float* x, size_t batch, size_t seq, size_t width,
           const fsvd_ffn_desc* f, const fsvd_tile_plan* plan, float* out) {
  const size_t d = width;
  if (f->up.in_dim != d || f->down.out_dim != d) return FSVD_ERR_SHAPE;
  if (f->up.out_dim != f->down.in_dim) return FSVD_ERR_SHAPE;
  if (f->up.rank != f->down.rank) return FSVD_ERR_CONFIG;
  const size_t rank = f->up.rank;
  {
    fsvd_geometry g = {batch, seq, d, f->up.out_dim, 1, 1, rank, 1};
    int st;
    fo_tile_working_set(plan, variant == 2 ? FSVD_KERNEL_FFN_V2 : FSVD_KERNEL_FFN_V1, &g, &st);
    if (st) return st;
  }
  const size_t bm = plan->bm, bdf = plan->bdf;
  float* h = (float*)malloc(bm * bdf * sizeof(float));
  float* v1p = (float*)malloc(rank * bdf * sizeof(float));
  float* u2p = (float*)malloc(bdf * rank * sizeof(float));
  float* ptile = (float*)malloc(bm * rank * sizeof(float));
  float* z = (float*)malloc(bm * rank * sizeof(float));
  for (size_t b = 0; b < batch; ++b)
    for (size_t m0 = 0; m0 < seq; m0 += bm) {
      const size_t mlen = (bm < seq - m0) ? bm : seq - m0;
      memset(ptile, 0, bm * rank * sizeof(float));
      memset(z, 0, bm * rank * sizeof(float));
      gemm_acc_ld(x + (b * seq + m0) * d, d, f->up.u, rank, ptile, rank, mlen, d, rank);
      stream_feature_blocks(ptile, mlen, f, bdf, h, v1p, u2p, z);
      for (size_t i = 0; i < mlen; ++i) {
        float* orow = out + (b * seq + m0 + i) * d;
        memcpy(orow, f->down.bias, sizeof(float) * d);
        gemm_acc_ld(z + i * rank, rank, f->down.v, d, orow, d, 1, rank, d);
      }
    }
  free(h); free(v1p); free(u2p); free(ptile); free(z);
  return 0;
}

void fo_residual_norm(const float* a, const float* b, size_t rows, size_t d,
                      const float* gamma, const float* beta, float eps, float* dst) {
  float* sum = (float*)malloc(d * sizeof(float));
  for (size_t i = 0; i < rows; ++i) {
    const float* ar = a + i * d;
    const float* br = b + i * d;
    for (size_t j = 0; j < d; ++j) sum[j] = ar[j] + br[j];
    layer_norm_row(sum, dst + i * d, d, gamma, beta, eps);
  }
  free(sum);
}

/* encoder.cpp:224-260 */
int fo_run_layer(const float* x, size_t batch, size_t seq, const fsvd_layer_desc* L,
                 int mode, const fsvd_tile_plan* plan, int pre_ln, float* out) {
  const size_t d = L->attn.d_model, n = batch * seq * d, rows = batch * seq;
  const int variant = (mode == FSVD_MODE_FLASH_V2) ? 2 : 1;
  float* ctx = (float*)calloc(n, sizeof(float));
  float* branch = (float*)calloc(n, sizeof(float));
  float* resid = (float*)calloc(n, sizeof(float));
  int st = 0;
  if (!pre_ln) {
    if ((st = fo_flash_svd_attention(x, batch, seq, &L->attn, L->heads, plan, ctx))) goto done;
    if ((st = fo_lowrank_output_projection(ctx, batch, seq, &L->out_proj, branch))) goto done;
    fo_residual_norm(x, branch, rows, d, L->ln1_gamma, L->ln1_beta, L->ln1_eps, resid);
    if ((st = fo_ffn(variant, resid, batch, seq, d, &L->ffn, plan, branch))) goto done;
    fo_residual_norm(resid, branch, rows, d, L->ln2_gamma, L->ln2_beta, L->ln2_eps, out);
  } else {
    float* normed = (float*)calloc(n, sizeof(float));
    for (size_t i = 0; i < rows; ++i)
      layer_norm_row(x + i * d, normed + i * d, d, L->ln1_gamma, L->ln1_beta, L->ln1_eps);
    st = fo_flash_svd_attention(normed, batch, seq, &L->attn, L->heads, plan, ctx);
    if (!st) st = fo_lowrank_output_projection(ctx, batch, seq, &L->out_proj, branch);
    if (!st) {
      for (size_t i = 0; i < n; ++i) resid[i] = x[i] + branch[i];
      for (size_t i = 0; i < rows; ++i)
        layer_norm_row(resid + i * d, normed + i * d, d, L->ln2_gamma, L->ln2_beta, L->ln2_eps);
      st = fo_ffn(variant, normed, batch, seq, d, &L->ffn, plan, branch);
    }
    if (!st)
      for (size_t i = 0; i < n; ++i) out[i] = resid[i] + branch[i];
    free(normed);
  }
done:
  free(ctx); free(branch); free(resid);
  return st;
}

/* encoder.cpp:262-293 */
int fo_run_model(const float* x, size_t batch, size_t seq, const fsvd_layer_desc* layers,
                 size_t n_layers, int mode, const fsvd_tile_plan* plan, int pre_ln,
                 float* out) {
  const size_t d = n_layers ? layers[0].attn.d_model : 0;
  if (n_layers == 0) return FSVD_ERR_CONFIG;
  const size_t n = batch * seq * d;
  if (n_layers == 1) return fo_run_layer(x, batch, seq, &layers[0], mode, plan, pre_ln, out);
  float* ping = (float*)malloc(n * sizeof(float));
  float* pong = (float*)malloc(n * sizeof(float));
  const float* cur = x;
  int st = 0;
  for (size_t i = 0; i < n_layers && !st; ++i) {
    float* dst = (i + 1 == n_layers) ? out : (i % 2 == 0 ? ping : pong);
    st = fo_run_layer(cur, batch, seq, &layers[i], mode, plan, pre_ln, dst);
    cur = dst;
  }
  free(ping); free(pong);
  return st;
}
