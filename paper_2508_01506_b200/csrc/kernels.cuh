// kernels.cuh -- host launchers of every device kernel in the library.
//
// Tensor-core kernels (bf16 storage, fp32 accumulate, tcgen05 + TMA):
//   K1 gemm_bf16          low-rank projection GEMMs with fused epilogues
//   K2 attn_rankspace     FlashSVD attention (rank-space online softmax)
//   K3 ffn_stream         FlashSVD-FFN feature-block stream (V1 middle)
//   K4 ffn_fused          FlashSVD-FFN V2, fully fused per 128-row tile
//   K5 resid_layernorm    residual + LayerNorm row kernel
//   K6 gemm_ln            projection GEMM with residual + LayerNorm epilogue
// SIMT kernels (fp32 policy and shapes outside the tensor-core tiling):
//   simt_gemm, simt_attention, simt_ffn_stream, resid_layernorm (fp32)
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fsvd {

using bf16 = __nv_bfloat16;

enum Act : int { ACT_GELU_ERF = 0, ACT_GELU_TANH = 1, ACT_RELU = 2, ACT_NONE = 3 };

// ---- K1: C[M,N] = A[M,K] * B[N,K]^T (+ bias[N]) (act) (+ resid[M,N]) ---------
// A, B, C, resid bf16 row-major with leading dims; bias fp32 or null.
// C = A B^T (+ bias) (act) (+ resid, [M, N] with leading dimension ldr)
void gemm_bf16(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, bf16* C, int64_t ldc,
               int M, int N, int K, const float* bias, int act, cudaStream_t s,
               const bf16* resid = nullptr, int64_t ldr = 0);
bool gemm_bf16_supported(int M, int N, int K, int64_t lda, int64_t ldb, int64_t ldc);
// Split output: columns [0, split_n) of C = A B^T + bias go to C (pitch ldc),
// columns [split_n, N) to C2 (pitch ldc2).  split_n % 64 == 0.  The QKV
// projection uses it to put Qt (which K2 overwrites with its rank-space output)
// and the [P_k | P_v] chunk (dead after K2) in separate workspace regions.
void gemm_bf16_split(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, bf16* C,
                     int64_t ldc, int split_n, bf16* C2, int64_t ldc2, int M, int N, int K,
                     const float* bias, cudaStream_t s);

// ---- split planes (fp32 policy on the tensor cores) ---------------------------
// An fp32 matrix v is held as three bf16 matrices of the same shape, stored
// one after the other: hi = bf16(v), mid = bf16(v - hi), lo = bf16(v - hi -
// mid) (|v - hi - mid - lo| <= 2^-24 |v|, fp32 resolution).  A product runs
// as six bf16 MMA passes into one fp32 accumulator -- every plane pair of
// order <= 2: hi*hi, hi*mid, mid*hi, hi*lo, lo*hi, mid*mid -- leaving out
// terms below 2^-23 of the product.  A [rows, cols] matrix occupies
// 6*rows*cols bytes; plane stride = rows * leading dimension.
struct Planes {
  const bf16* hi;
  const bf16* mid;
  const bf16* lo;
};
struct PlanesOut {
  bf16* hi;
  bf16* mid;
  bf16* lo;
};
constexpr int kPlanes = 3;
// K1 in the split-plane form: C = A B^T (+ bias) (act) (+ resid), every
// matrix as planes with the same leading dimension in every plane.
void gemm_x3(const Planes& A, int64_t lda, const Planes& B, int64_t ldb, const PlanesOut& C,
             int64_t ldc, int M, int N, int K, const float* bias, int act, cudaStream_t s,
             const Planes* resid = nullptr, int64_t ldr = 0);
// fp32 <-> planes at the API boundary; row kernels between the GEMMs (planes.cu)
void split_planes(const float* src, const PlanesOut& y, int64_t n, cudaStream_t s);
void merge_planes(const Planes& a, float* dst, int64_t n, cudaStream_t s);
// y = LN(a (+ b)) * gamma + beta, rows of width d; in place allowed for d <= 2048
void ln_planes(const Planes& a, const Planes* b, const float* gamma, const float* beta, float eps,
               const PlanesOut& y, int rows, int d, cudaStream_t s, int pitch = 0);
void add_planes(const Planes& a, const Planes& b, const PlanesOut& y, int64_t n, cudaStream_t s);
// Host fp32 rows [rows, d] (staged on the device) <-> device activations
// [rows, pitch] in storage form 0 bf16, 1 fp32, 2 split planes; the padding
// columns d..pitch are written as zeros.
void rows_to_device(const float* src, int rows, int d, int pitch, int form, void* dst,
                    cudaStream_t s);
void rows_from_device(const void* src, int rows, int d, int pitch, int form, float* dst,
                      cudaStream_t s);

// ---- K6: y = LN(resid + bf16(A[T,K] * B[N,K]^T + bias)) * gamma + beta --------
// One CTA per 128 complete rows; N <= 768, K <= 512, multiples of 64.
// sum_out (optional, [T, N]): also store the un-normalised resid + A*B^T + bias
// (the pre-LN residual stream).
void gemm_ln_bf16(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, const float* bias,
                  const bf16* resid, const float* gamma, const float* beta, float eps, bf16* y,
                  int T, int N, int K, cudaStream_t s, bf16* sum_out = nullptr,
                  int seq_tiles = 0);
bool gemm_ln_supported(int N, int K);
// The same operation on a CTA pair (gemm_ln2_tc.cu, cta_group::2, 256 rows per
// cluster); returns false (nothing launched) outside its range.  gemm_ln_bf16
// uses it when gemm_ln_pair_enabled() (FSVD_LN_PAIR=1, opt-in).
bool gemm_ln_pair_bf16(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, const float* bias,
                       const bf16* resid, const float* gamma, const float* beta, float eps, bf16* y,
                       int T, int N, int K, cudaStream_t s, bf16* sum_out, int seq_tiles);
bool gemm_ln_pair_enabled();

// ---- K2: rank-space FlashSVD attention --------------------------------------
// out[t, h*rp : (h+1)*rp] = softmax(Qt_h K_g^T) V_g for each (sequence, head),
// reading Qt / K / V as rank-width column blocks of one [T, qkv_cols] buffer:
// head h's Qt at q_off + h*rp, group g's K at k_off + g*rp and V at v_off + g*rp.
// Scores must already be scaled into the log2 domain.
struct AttnTcArgs {
  const bf16* qkv;
  int64_t ldq;
  int qkv_cols;
  int q_off, k_off, v_off;
  int batch, seq, heads, groups, rank_pad;
  bf16* out;
  int64_t ldo;
  bool causal = false;  // decoder prefill: key j visible to query i iff j <= i
  // split planes (fp32 policy): qkv and out each hold three planes (qkv plane
  // stride batch*seq*ldq, out plane stride out_ps elements); the kernel runs
  // its X3 form (six bf16 passes per product)
  bool planes = false;
  int64_t out_ps = 0;
  // K / V in their own region ([T, kv_cols], pitch ldkv; k_off / v_off are
  // then column offsets in it); null: they sit in qkv.  out may alias the Qt
  // columns of qkv: an item reads its Qt tile before it writes its output
  // there, and no other item reads those cells.
  const bf16* kv = nullptr;
  int64_t ldkv = 0;
  int kv_cols = 0;
};
void attn_rankspace_bf16(const AttnTcArgs& a, cudaStream_t s);

// ---- decoder: rank-space KV cache (decode.cu) ------------------------------------
struct DecodeArgs {
  const bf16* qkv;  // [batch, ldq] projection rows of the new tokens
  int64_t ldq;
  int q_off;
  const bf16* cache;  // [batch, max_seq, 2*groups*rank_pad]
  int max_seq, batch, heads, groups, rank_pad;
  int len;     // cached tokens attended (new token included)
  int splits;  // decode_splits(batch, heads, len)
  float* part;  // splits > 1: [batch*heads, splits, rank_pad + 2]
  bf16* out;
  int64_t ldo;
  const int* pos_dev = nullptr;  // non-null: len = *pos_dev + 1 (graph replay)
};
int decode_splits(int batch, int heads, int len);
void set_device_int(int* p, int v, cudaStream_t s);
size_t decode_partial_bytes(int batch, int heads, int rank_pad, int max_len);
void attn_decode_bf16(const DecodeArgs& a, cudaStream_t s);
void kv_store_bf16(const bf16* src, int64_t lds, int c0, int width, int batch, int rows_per_b,
                   bf16* cache, int max_seq, int pos0, const int* pos_dev, cudaStream_t s);
bool attn_rankspace_supported(int rank_pad);

// ---- K3 / K4: FlashSVD-FFN -----------------------------------------------------
struct FfnTcArgs {
  int T, d_model, d_ff, rank_pad;
  const bf16* x;       // [T, d_model]          (V2 input)
  const bf16* up_u_t;  // [fr][d_model]          U_up^T
  const bf16* up_v_t;  // [d_ff][fr]             V_up^T
  const float* up_b;   // [d_ff]
  const bf16* dn_u_t;  // [fr][d_ff]             U_down^T
  const bf16* dn_v_t;  // [d_model][fr]          V_down^T
  const float* dn_b;   // [d_model]
  int act;
  const bf16* p_in;    // [T, fr]   (V1: P = X U_up)
  bf16* z_out;         // [T, fr]   (V1: Z)
  bf16* out;           // [T, d_model] (V2)
  // V2 only: when ln_g != null, out = LN(x + ffn(x)) * ln_g + ln_b (post-LN
  // residual + LayerNorm fused into the epilogue; d_model <= 768).
  const float* ln_g;
  const float* ln_b;
  float ln_eps;
  // V1 only: split_blocks > 0 spreads the d_ff feature blocks of each row
  // tile over ceil(blocks / split_blocks) CTAs, each writing an fp32 partial
  // Z to z_part[split][T][rank_pad] (z_out unused); sum with z_partial_sum.
  int split_blocks = 0;
  float* z_part = nullptr;
  // V2: 128-row tiles per sequence (seq / 128 when seq % 128 == 0, else 0).
  // The fused kernel starts each tile's feature-block and K-chunk loops at an
  // offset set by the tile's position inside its sequence, so concurrent CTAs
  // read different weight boxes (all CTAs streaming the same boxes at once
  // hot-spot the L2); a row's summation order depends only on where it sits
  // in its sequence, so results stay independent of the batch position.
  int seq_tiles = 0;
  // V2 without LN only: out = resid + ffn(x) (pre-LN layers)
  const bf16* resid = nullptr;
  // V2 with LN (pre-LN layer chaining): the LN residual is ln_resid instead of
  // x, and the un-normalised ln_resid + ffn(x) is also stored to sum_out
  const bf16* ln_resid = nullptr;
  bf16* sum_out = nullptr;
  // V1 stream in split planes (fp32 policy): P, V_up^T, U_down^T and Z each
  // hold three stacked planes (plane stride = rows x leading dimension); K3
  // runs its X3 form
  bool planes = false;
};
void ffn_stream_bf16(const FfnTcArgs& a, cudaStream_t s);   // V1 middle: P -> Z
void z_partial_sum_bf16(const float* part, int splits, int64_t n, bf16* z, cudaStream_t s);
void ffn_fused_bf16(const FfnTcArgs& a, cudaStream_t s);    // V2: X -> out
// V2 on a CTA pair (cta_group::2, 256 rows per cluster): half the weight bytes
// per SM; d_model, d_ff, rank_pad multiples of 128, rank_pad <= 384.
void ffn_fused_pair_bf16(const FfnTcArgs& a, cudaStream_t s);
bool ffn_pair_supported(int d_model, int d_ff, int rank_pad);
bool ffn_tc_supported(int d_model, int d_ff, int rank_pad);
// FFN rank padding (ffn_tc.cu): <= 384 -> multiple of 64 (V2 fused / K3 with Z
// resident); above -> n slices of ffn_wide_slice() columns (K3 only, V1 chain)
constexpr int kFfnMaxRankPad = 1536;
int ffn_rank_pad(int fr);
int ffn_wide_slice(int rank_pad);
// K3 for rank_pad > 384 on a cluster of rank_pad / slice CTAs sharing each
// hidden block over DSMEM (ffn_wide_tc.cu); split_blocks must be 0.
bool ffn_wide_cluster_supported(const FfnTcArgs& a);
void ffn_wide_cluster_bf16(const FfnTcArgs& a, cudaStream_t s);

// ---- K5: y = LN(a (+ b)) * gamma + beta, rows of width d ---------------------
// pitch > d: rows are stored with pitch columns (zero-padded model dimension);
// statistics over the first d, all pitch columns written.
void resid_layernorm_bf16(const bf16* a, const bf16* b, const float* gamma, const float* beta,
                          float eps, bf16* y, int rows, int d, cudaStream_t s, int pitch = 0);
void resid_layernorm_f32(const float* a, const float* b, const float* gamma, const float* beta,
                         float eps, float* y, int rows, int d, cudaStream_t s, int pitch = 0);
void add_bf16(const bf16* a, const bf16* b, bf16* y, int64_t n, cudaStream_t s);
void add_f32(const float* a, const float* b, float* y, int64_t n, cudaStream_t s);

// ---- SIMT kernels (templated on storage T = float or bf16, fp32 accumulate) --
// C[M,N] = A[M,K] * B[K,N] (+bias) (act), row-major with leading dims.
template <typename T>
void simt_gemm(const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, int M,
               int N, int K, const float* bias, int act, cudaStream_t s);

struct AttnSimtArgs {
  const void* P;     // [T][3][G][r] projected activations (row stride 3*G*r)
  const void* v;     // [3][G][r][gd]
  const float* bias; // [3][d]
  int batch, seq, heads, groups, rank, d_model;
  void* ctx;         // [T, d]
};
template <typename T>
void simt_attention(const AttnSimtArgs& a, cudaStream_t s);

struct FfnSimtArgs {
  const void* p;     // [T, r]
  const void* up_v;  // [r][d_ff]
  const float* up_b; // [d_ff]
  const void* dn_u;  // [d_ff][r]
  void* z;           // [T, r]
  int T, rank, d_ff, act;
};
template <typename T>
void simt_ffn_stream(const FfnSimtArgs& a, cudaStream_t s);
// ffn_v2 dataflow on CUDA cores: P and Z stay in shared memory (16-row tiles).
template <typename T>
void simt_ffn_fused(const T* x, const T* up_u, const T* up_v, const float* up_b, const T* dn_u,
                    const T* dn_v, const float* dn_b, T* out, int Tn, int d, int rank, int d_ff,
                    int act, cudaStream_t s);

template <typename T>
void convert_f32(const float* src, T* dst, int64_t n, cudaStream_t s);
template <typename T>
void to_f32(const T* src, float* dst, int64_t n, cudaStream_t s);

uint64_t launch_count();

}  // namespace fsvd
