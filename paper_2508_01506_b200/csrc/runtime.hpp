// runtime.hpp -- device factor packs, the activation buffer planner and the
// device-side encoder schedule (everything between the C ABI and kernels).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

#include "../../include/fsvd_b200.h"
#include "errors.hpp"
#include "kernels.cuh"

namespace fsvd {

// One encoder layer resident in HBM, in the layouts its kernels consume.
//   Tensor-core (bf16) layouts are K-major transposes padded with zeros:
//     wqkv_t [3*G*rp][d]   vq_t/vv_t [H][dh][rp]   vk [H][rp][dh]
//     uo_t [prp][d]  vo_t [d][prp]  uup_t [frp][d]  vup_t [df][frp]
//     udn_t [frp][df]  vdn_t [d][frp]
//   SIMT layouts are the reference orientation (x * W):
//     wqkv [d][3*G*r]  attn_v [3][G][r][gd]  uo [d][pr]  vo [pr][d] ...
struct Pack {
  fsvd_dtype dtype = FSVD_BF16;
  int es = 2;  // bytes per stored element
  // d: model dimension of the device layouts (the callers' dr rounded up to
  // 64 on the tensor-core path, zero-padded); df likewise (rounded up to 8)
  int d = 0, dr = 0, df = 0, H = 1, G = 1, r = 0, pr = 0, fr = 0, dh = 0, gd = 0, act = 0;
  float eps1 = 1e-5f, eps2 = 1e-5f;
  int rp = 0, prp = 0, frp = 0;
  bool has_attn = false, has_out = false, has_ffn = false, has_ln = false, dense = false;
  bool attn_tc = false, out_tc = false, ffn_tc = false;
  bool ffn_wide = false;  // frp > 384: sliced K3, V2 runs the V1 chain (ffn_tc.cu)
  // fp32 policy on the tensor cores (planes.cu): every weight below is stored
  // as split planes (the *_lo arrays hold the lo planes of the tensor-core
  // layouts), device activations are split planes, and the layer runs K1 / K2 /
  // K3 in their X3 form.  All-or-nothing per pack: a pack whose shapes leave
  // the tensor-core tiling runs the fp32 SIMT kernels instead.
  bool x3 = false;
  const void *wproj_lo = nullptr, *wvc_lo = nullptr, *uo_t_lo = nullptr, *vo_t_lo = nullptr,
             *wov_lo = nullptr, *uup_t_lo = nullptr, *vup_t_lo = nullptr, *udn_t_lo = nullptr,
             *vdn_t_lo = nullptr;
  void* mem = nullptr;
  size_t bytes = 0;
  // attention, tensor-core path (folded rank-space form, see attn_tc.cu):
  //   wproj_t [(H+2G)*rp][d]  rows: Qt of every head (U_q V_q V_k^T s), U_k, U_v
  //   bproj   [(H+2G)*rp]     Qt bias s b_q V_k^T, zeros for P_k / P_v
  //   wvc_t   [d][H*rp]       block-diagonal V_v (rank space -> head width)
  //   bv      [d]
  const void* wproj_t = nullptr;
  const float* bproj = nullptr;
  const void* wvc_t = nullptr;
  const float* bv = nullptr;
  int qkv_cols = 0;  // (H + 2G) * rp
  // attention, SIMT path (reference layouts)
  const void *wqkv = nullptr, *attn_v = nullptr;
  const float* attn_b = nullptr;
  // output projection: low-rank factors (drop-in lowrank_output_projection) and,
  // on the tensor-core path, the folded rank-space form used inside a layer:
  //   wov_t [d][H*rp] = (blockdiag(V_v) U_o V_o)^T,  bov = b_v U_o V_o + b_o
  const void *uo_t = nullptr, *vo_t = nullptr, *uo = nullptr, *vo = nullptr;
  const float* bo = nullptr;
  const void* wov_t = nullptr;
  const float* bov = nullptr;
  // FFN
  const void *uup_t = nullptr, *vup_t = nullptr, *udn_t = nullptr, *vdn_t = nullptr;
  const void *uup = nullptr, *vup = nullptr, *udn = nullptr, *vdn = nullptr;
  const float *bup = nullptr, *bdn = nullptr;
  // LayerNorms
  const float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
  // dense twin / materializing baselines (tensor-core path only); the Q rows
  // carry the softmax scale s = log2(e)/sqrt(dh)
  const void *dqkv_t = nullptr;   // [3d][d]   dense W_q|W_k|W_v transposed
  const float* dqkv_b = nullptr;  // [3*H*dhp] (Dense mode, padded head layout)
  const float* nqkv_b = nullptr;  // [3d] q|k|v biases of the naive low-rank rebuild
  const void *wpn_t = nullptr;    // [3*G*rp][d] U_q|U_k|U_v transposed (naive low-rank)
  const void *dvbd_t = nullptr;   // [3d][3*G*rp] block-diagonal V (naive low-rank)
  // Dense mode (encoder.cpp:99-105, 136-139) from the layer's dense weights,
  // else the dense twin of its factors: head width padded to dhp in
  // {16, 32, 64} so K2 runs it as a rank-space kernel with r = dhp:
  //   dqkv_t [3*H*dhp][d] (Q rows scaled by s, zero pad rows), dqkv_b,
  //   do_t [d][H*dhp] = W_o^T (zero pad columns), din_t [df][d], dout_t [d][df]
  int dhp = 0, ddf = 0, dact = 0;
  const void *do_t = nullptr, *din_t = nullptr, *dout_t = nullptr;
  const float *dbo = nullptr, *dbin = nullptr, *dbout = nullptr;
  const void *dqkv_lo = nullptr, *do_lo = nullptr, *din_lo = nullptr, *dout_lo = nullptr,
             *wpn_lo = nullptr, *dvbd_lo = nullptr;

  ~Pack();
};

struct PackRequest {
  const fsvd_attn_desc* attn = nullptr;
  size_t heads = 0;
  const fsvd_linear_desc* out_proj = nullptr;
  const fsvd_ffn_desc* ffn = nullptr;
  const float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
  float eps1 = 1e-5f, eps2 = 1e-5f;
  size_t d_model = 0;
  bool dense = false;  // also build the Dense-mode weights (and the naive low-rank ones)
  const fsvd_dense_layer* dense_w = nullptr;  // the layer's own dense weights, if any
  int dense_act = 0;  // the dense FFN's activation when the layer has no FFN factors
};

Pack* build_pack(const PackRequest& req, fsvd_dtype dtype);

// encoder.cpp:156-222 for the flat descriptor (throws Error).
void validate_layer(const fsvd_layer_desc& L);
// encoder.cpp:27-35 for a run mode; dense_twin_ok lets a factor-only layer
// run Dense mode as its dense twin (the C-ABI's documented extension).
void check_mode_weights(const fsvd_layer_desc& L, int mode, bool dense_twin_ok);

// Activation buffer planner: bytes of device workspace one layer needs for
// T = batch*seq tokens in the given mode (two [T, d] scratch buffers + the
// rank-sized transient region, aliased across sublayers).
// workspace of a [B, M] batch through layer_fwd (full attention); max over
// pre/post-LN without the flag
size_t layer_workspace_bytes(const Pack& p, size_t B, size_t M, int mode);
size_t layer_workspace_bytes(const Pack& p, size_t B, size_t M, int mode, bool pre_ln);
size_t op_transient_elems(const Pack& p, int op, int mode);  // op: 0 attn, 1 out, 2 ffn

// Device schedule (async on `s`).  x and out may alias in layer_fwd.
void attention_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* ctx,
                   void* trans, cudaStream_t s);
void outproj_fwd(const Pack& p, int mode, size_t B, size_t M, const void* ctx, void* out,
                 void* trans, cudaStream_t s);
size_t ffn_block_workspace_bytes(const Pack& p, size_t B, size_t M, int mode);
void ffn_block_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* out,
                   void* ws, size_t ws_bytes, cudaStream_t s);
void ffn_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* out, void* trans,
             cudaStream_t s);
// Attention variant of a layer run: the encoder's full attention, or the
// decoder rows (f4) on a layer's rank-space KV cache [B, max_seq, 2*G*rp].
struct AttnMode {
  enum Kind { Full, Prefill, Decode } kind = Full;
  void* cache = nullptr;
  size_t max_seq = 0;
  size_t pos = 0;  // Decode: position of the new token (keys 0..pos)
  // Decode under graph capture: the position is read from pos_dev at run
  // time, and the split count / partial buffers are sized for max_seq.
  const int* pos_dev = nullptr;
};
// Pre-LN layer chaining (model loops): `next` = the following layer, whose
// LN1 this layer applies in its FFN epilogue (the normalised rows land in the
// workspace A region); `ln1_done` = this layer's LN1 was applied that way.
struct LayerLink {
  const Pack* next = nullptr;
  bool ln1_done = false;
};
void layer_fwd(const Pack& p, int mode, bool pre_ln, size_t B, size_t M, const void* x, void* out,
               void* ws, size_t ws_bytes, cudaStream_t s, const AttnMode& am = AttnMode{},
               const LayerLink& link = LayerLink{});
// n layers in place (x -> out, out may equal x), pre-LN layers chained
// through LayerLink where both sides run the fused schedule.
void model_layers_fwd(const Pack* const* packs, size_t n, int mode, bool pre_ln, size_t B, size_t M,
                      const void* x, void* out, void* ws, size_t ws_bytes, cudaStream_t s);
// Whether pre-LN layer p may apply q's LN1 in its FFN epilogue (T rows).
bool pre_ln_link_ok(const Pack& p, const Pack& q, int mode, size_t T);
// Decoder: workspace for prefill of up to max_seq tokens and for decode steps.
size_t decoder_workspace_bytes(const Pack& p, size_t B, size_t max_seq, bool pre_ln);
size_t kv_cache_bytes(const Pack& p, size_t B, size_t max_seq);
void check_decoder_pack(const Pack& p);

uint16_t f32_to_bf16_bits(float f);

}  // namespace fsvd

struct fsvd_layer_pack {
  fsvd::Pack* p;
};
