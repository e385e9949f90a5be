/*
 * fsvd_b200.h -- C-ABI boundary of the B200-native FlashSVD streaming encoder.
 *
 * This is the drop-in boundary for the reference's low-rank operator API
 * (/root/reference/proj/include/flashsvd/{attention,ffn,encoder,memtier}.hpp).
 * Every entry point below names the reference interface it replaces.  The
 * C++ drop-in headers under include/flashsvd/ re-expose the reference
 * signatures on top of these functions; Python (ctypes), cgo or JNI bind the
 * same symbols directly.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross this ABI.
 *   - Host tensors are fp32, row-major, in the reference's orientation
 *     (x * W: U is in x r, V is r x out, factorize.hpp:11-21).
 *   - Device activations are row-major [batch, seq, d_model] in the pack's
 *     dtype (bf16 or fp32).
 *   - Status codes map 1:1 onto flashsvd::ErrorKind (errors.hpp:11-21), with
 *     FSVD_ERR_CUDA added for device failures.  Exceptions never cross the
 *     ABI; the message of the last failure on the calling thread is returned
 *     by fsvd_last_error().
 *   - There is no CPU fallback: every compute entry point launches sm_100a
 *     kernels and fails with FSVD_ERR_CUDA when no usable device exists.
 */
#ifndef FSVD_B200_H
#define FSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define FSVD_ABI_VERSION 1

/* errors.hpp:11-21 (ErrorKind), in declaration order, offset by one. */
typedef enum fsvd_status {
  FSVD_OK = 0,
  FSVD_ERR_SHAPE = 1,
  FSVD_ERR_RANK = 2,
  FSVD_ERR_CONFIG = 3,
  FSVD_ERR_BUDGET = 4,
  FSVD_ERR_ACCOUNTING = 5,
  FSVD_ERR_FORMAT = 6,
  FSVD_ERR_NUMERIC = 7,
  FSVD_ERR_INFEASIBLE = 8,
  FSVD_ERR_IO = 9,
  FSVD_ERR_CUDA = 10
} fsvd_status;

/* Storage / arithmetic precision policy of a factor pack and its kernels.
 * FSVD_F32 : fp32 storage, fp32 FMA accumulate (<= 1e-4 parity mode).
 * FSVD_BF16: bf16 storage, tcgen05 bf16 MMA, fp32 accumulate (<= 2e-2). */
typedef enum fsvd_dtype { FSVD_F32 = 0, FSVD_BF16 = 1 } fsvd_dtype;

/* ffn.hpp:13 */
typedef enum fsvd_activation {
  FSVD_ACT_GELU_ERF = 0,
  FSVD_ACT_GELU_TANH = 1,
  FSVD_ACT_RELU = 2,
  FSVD_ACT_IDENTITY = 3
} fsvd_activation;

/* encoder.hpp:21 */
typedef enum fsvd_run_mode {
  FSVD_MODE_DENSE = 0,
  FSVD_MODE_NAIVE_LOWRANK = 1,
  FSVD_MODE_FLASH_V1 = 2,
  FSVD_MODE_FLASH_V2 = 3
} fsvd_run_mode;

/* memtier.hpp:159 */
typedef enum fsvd_kernel_kind {
  FSVD_KERNEL_ATTENTION = 0,
  FSVD_KERNEL_FFN_V1 = 1,
  FSVD_KERNEL_FFN_V2 = 2
} fsvd_kernel_kind;

/* memtier.hpp:169-178 (FormulaId) */
typedef enum fsvd_formula {
  FSVD_FORMULA_DENSE_ATTN = 0,
  FSVD_FORMULA_FLASH_ATTN_DENSE_QKV = 1,
  FSVD_FORMULA_FLASH_SVD_ATTN = 2,
  FSVD_FORMULA_GROUPED_ATTN = 3,
  FSVD_FORMULA_FFN_DENSE = 4,
  FSVD_FORMULA_FFN_NAIVE_LOWRANK = 5,
  FSVD_FORMULA_FFN_V1 = 6,
  FSVD_FORMULA_FFN_V2 = 7
} fsvd_formula;

/* memtier.hpp:152-157 (TilePlan). */
typedef struct fsvd_tile_plan {
  size_t bm, br, bdf, sram_budget_bytes;
} fsvd_tile_plan;

/* geometry.hpp:11-20 */
typedef struct fsvd_geometry {
  size_t batch, seq_len, d_model, d_ff, heads, groups, rank, layers;
} fsvd_geometry;

/* FactorizedLinear (factorize.hpp:13-21): w (in x out) ~ u (in x r) v (r x out). */
typedef struct fsvd_linear_desc {
  size_t in_dim, rank, out_dim;
  const float* u;    /* [in_dim][rank]  */
  const float* v;    /* [rank][out_dim] */
  const float* bias; /* [out_dim]       */
} fsvd_linear_desc;

/* AttentionFactorSet (factorize.hpp:28-40), groups stored contiguously:
 *   u    [3][groups][d_model][rank]          (q, k, v)
 *   v    [3][groups][rank][d_model/groups]
 *   bias [3][groups][d_model/groups] == [3][d_model]                         */
typedef struct fsvd_attn_desc {
  size_t d_model, groups, rank;
  const float* u;
  const float* v;
  const float* bias;
} fsvd_attn_desc;

/* FfnFactors (ffn.hpp:17-21) */
typedef struct fsvd_ffn_desc {
  fsvd_linear_desc up;   /* d_model -> d_ff */
  fsvd_linear_desc down; /* d_ff -> d_model */
  fsvd_activation activation;
} fsvd_ffn_desc;

struct fsvd_dense_layer; /* dense weights, defined below */

/* EncoderLayer (encoder.hpp:49-67).  Like the reference, a layer carries
 * factorized weights, dense weights, or both:
 *   - factorized attention: attn.u != NULL (with out_proj); attn.d_model is
 *     d_model in every case;
 *   - factorized FFN: ffn.up.u != NULL; ffn.activation is also the dense
 *     FFN's activation;
 *   - dense weights (DenseAttentionWeights + DenseFfnWeights): dense != NULL.
 * RunMode::Dense uses the dense weights (encoder.cpp:27-35 check_mode_weights);
 * the flash / naive modes need the factors.  Device packs built with dense=1
 * from a factor-only layer get the dense twin instead (dense_equivalent,
 * encoder.cpp:295-331). */
typedef struct fsvd_layer_desc {
  size_t heads;
  fsvd_attn_desc attn;
  fsvd_linear_desc out_proj;
  fsvd_ffn_desc ffn;
  const float* ln1_gamma; const float* ln1_beta; float ln1_eps;
  const float* ln2_gamma; const float* ln2_beta; float ln2_eps;
  const struct fsvd_dense_layer* dense; /* NULL: no dense weights */
} fsvd_layer_desc;

/* ------------------------------------------------------------------ */
/* Library / errors                                                    */
/* ------------------------------------------------------------------ */
int fsvd_abi_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* fsvd_last_error(void);
/* 1 if an sm_100 device is usable, else 0 (message in fsvd_last_error). */
int fsvd_device_available(void);

/* ------------------------------------------------------------------ */
/* MemoryMeter (memtier.hpp:45-146, memtier.cpp:8-116)                  */
/* Byte meter of the two-tier model.  4 B/element reference accounting  */
/* plus a separate device high-water of the real (bf16/fp32) bytes.     */
/* ------------------------------------------------------------------ */
typedef struct fsvd_meter fsvd_meter;
typedef enum fsvd_alloc_class {
  FSVD_TRANSIENT = 0, FSVD_PERSISTENT = 1, FSVD_EXCLUDED = 2
} fsvd_alloc_class;
typedef enum fsvd_event_kind {
  FSVD_EV_ALLOC = 0, FSVD_EV_FREE = 1, FSVD_EV_PIN = 2,
  FSVD_EV_REGION_BEGIN = 3, FSVD_EV_REGION_END = 4
} fsvd_event_kind;

fsvd_status fsvd_meter_create(fsvd_meter** out);
void fsvd_meter_destroy(fsvd_meter* m);
fsvd_status fsvd_meter_alloc(fsvd_meter* m, const char* tag, fsvd_alloc_class cls,
                             size_t bytes, uint64_t* id);
fsvd_status fsvd_meter_free(fsvd_meter* m, uint64_t id);
fsvd_status fsvd_meter_pin(fsvd_meter* m, const char* tag, size_t bytes);
fsvd_status fsvd_meter_region_begin(fsvd_meter* m, const char* name, size_t* entry);
fsvd_status fsvd_meter_region_end(fsvd_meter* m, const char* name, size_t entry);
size_t fsvd_meter_current_transient(const fsvd_meter* m);
size_t fsvd_meter_peak_transient(const fsvd_meter* m);
size_t fsvd_meter_persistent(const fsvd_meter* m);
size_t fsvd_meter_current_excluded(const fsvd_meter* m);
void fsvd_meter_reset_peak(fsvd_meter* m);
fsvd_status fsvd_meter_assert_clean(const fsvd_meter* m);
size_t fsvd_meter_event_count(const fsvd_meter* m);
fsvd_status fsvd_meter_event(const fsvd_meter* m, size_t index, int* kind, int* cls,
                             size_t* bytes, uint64_t* id, char* tag, size_t tag_cap);
/* Real device bytes: activation arena high-water and factor-pack bytes
 * observed by operations run against this meter. */
size_t fsvd_meter_device_peak_bytes(const fsvd_meter* m);
size_t fsvd_meter_device_persistent_bytes(const fsvd_meter* m);

/* ------------------------------------------------------------------ */
/* Closed forms and plan validation (host only, no device needed)      */
/* ------------------------------------------------------------------ */
/* memtier.cpp:170-189: working-set bytes, FSVD_ERR_BUDGET / _CONFIG. */
fsvd_status fsvd_validate_tile_plan(const fsvd_tile_plan* plan, fsvd_kernel_kind kind,
                                    const fsvd_geometry* geom, size_t* bytes);
/* memtier.cpp:191-212 */
fsvd_status fsvd_expected_bytes(fsvd_formula id, const fsvd_geometry* geom, size_t* bytes);
/* planner.cpp:60-79 (flops_exact): algorithmic FLOP of one layer in `mode`
 * (uniform rank: rank = proj_rank = ffn_rank). */
fsvd_status fsvd_flops_exact(const fsvd_geometry* geom, fsvd_run_mode mode, uint64_t* flops);
/* planner.cpp:89-98 (io_bytes): fp32 activation + weight bytes in / out. */
fsvd_status fsvd_io_bytes(const fsvd_geometry* geom, fsvd_run_mode mode, uint64_t* in_bytes,
                          uint64_t* out_bytes);
/* encoder.cpp:333-345 */
size_t fsvd_flash_layer_peak_transient_bytes(const fsvd_geometry* geom);
size_t fsvd_flash_layer_persistent_bytes(const fsvd_geometry* geom);
size_t fsvd_flash_layer_bound_bytes(const fsvd_geometry* geom);

/* ------------------------------------------------------------------ */
/* Device factor packs (weights resident in HBM, kernel layouts)        */
/* ------------------------------------------------------------------ */
typedef struct fsvd_layer_pack fsvd_layer_pack;
/* Uploads one fully factorized layer.  Validates like
 * EncoderLayer::validate (encoder.cpp:156-222).  When dense != 0 the dense
 * twin (encoder.cpp:295-331) is also built so FSVD_MODE_DENSE can run. */
fsvd_status fsvd_layer_pack_create(const fsvd_layer_desc* layer, fsvd_dtype dtype,
                                   int dense, fsvd_layer_pack** out);
void fsvd_layer_pack_destroy(fsvd_layer_pack* p);
size_t fsvd_layer_pack_device_bytes(const fsvd_layer_pack* p);
/* 1 if this pack runs the tcgen05 tensor-core kernels, 0 if the SIMT
 * kernels (fp32 policy or shapes outside the tensor-core tiling). */
int fsvd_layer_pack_uses_tensor_cores(const fsvd_layer_pack* p);
/* Row pitch (elements) of this pack's device activations: d_model rounded up
 * to 64 when the layer runs on the tensor cores (the padding columns are
 * zero and stay zero), d_model otherwise.  Device-API buffers ([T, pitch])
 * use it; the host API pads and unpads itself.  fp32 packs on the tensor
 * cores store activations as split bf16 planes (hi [T, pitch], then lo). */
size_t fsvd_layer_pack_row_pitch(const fsvd_layer_pack* p);

/* Pack cache of the host drop-ins (fsvd_flash_svd_attention ...
 * fsvd_run_model): their device packs are kept per (device, dtype, content
 * hash of every factor / bias / LayerNorm array), so repeated calls on the
 * same layers -- the reference's run_model loop, commands.cpp:289-307 -- do
 * not rebuild or re-upload them; a changed value rebuilds.  LRU, capped at
 * FSVD_PACK_CACHE_MB (default 2048, 0 disables). */
fsvd_status fsvd_pack_cache_stats(size_t* entries, size_t* bytes, uint64_t* hits,
                                  uint64_t* misses);
fsvd_status fsvd_pack_cache_clear(void);

/* ------------------------------------------------------------------ */
/* FSVD1 model files (model_io.hpp:14-30, written by the reference's     */
/* save_model): container validation with byte offsets, assembly by the  */
/* canonical tensor names, upload as device factor packs.                */
/* ------------------------------------------------------------------ */
/* Host only: parses and assembles `path`; fills the geometry of layer 0
 * (layers = count).  FSVD_ERR_FORMAT carries the offending byte offset in
 * fsvd_last_error_offset(). */
fsvd_status fsvd_model_file_probe(const char* path, size_t* n_layers, fsvd_geometry* geom);
/* Loads every layer into packs[0 .. n_layers) (capacity >= layer count);
 * packs == NULL only reports n_layers. */
fsvd_status fsvd_model_load(const char* path, fsvd_dtype dtype, int dense,
                            fsvd_layer_pack** packs, size_t capacity, size_t* n_layers);
/* Byte offset of the last FSVD_ERR_FORMAT on this thread. */
size_t fsvd_last_error_offset(void);

/* ------------------------------------------------------------------ */
/* Device factorization: svd.cpp factor_rank_r,     */
/* factorize.cpp factorize_linear / factorize_attention, ffn.cpp         */
/* factorize_ffn, model_io.cpp synth_model's factorization step.  Host    */
/* pointers, synchronous; all matrices of a call are factorized in one   */
/* batched device run (fp64 one-sided block Jacobi).                     */
/* ------------------------------------------------------------------ */
/* svd.cpp:412-456 (factor_rank_r): a row-major m x n -> u (m x r), v (r x n),
 * even sqrt(sigma) split, largest-|.| entry of each u column positive.
 * FSVD_ERR_RANK: r == 0 or r > min(m, n). */
fsvd_status fsvd_factor_rank_r(const float* a, size_t m, size_t n, size_t rank, float* u,
                               float* v);
typedef struct fsvd_factor_job {
  const float* a; /* row-major m x n */
  size_t m, n, rank;
  float* u; /* m x rank */
  float* v; /* rank x n */
} fsvd_factor_job;
fsvd_status fsvd_factor_rank_r_batch(const fsvd_factor_job* jobs, size_t count);
/* factorize.cpp:21-64 (factorize_attention): w* are d x d (in x out), b* d.
 * Outputs in the fsvd_attn_desc layout: u [3][G][d][r], v [3][G][r][d/G],
 * bias [3][G][d/G] (q, k, v order).  FSVD_ERR_CONFIG: groups does not divide
 * d; FSVD_ERR_RANK: rank 0 or > d/groups. */
fsvd_status fsvd_factorize_attention(const float* wq, const float* bq, const float* wk,
                                     const float* bk, const float* wv, const float* bv,
                                     size_t d_model, size_t groups, size_t rank, float* u,
                                     float* v, float* bias);
/* One dense encoder layer (encoder.hpp:32-47 DenseAttentionWeights /
 * DenseFfnWeights), weights (in x out) row-major. */
typedef struct fsvd_dense_layer {
  size_t d_model, d_ff;
  const float *wq, *bq, *wk, *bk, *wv, *bv; /* d x d, d */
  const float *wo, *bo;                     /* d x d, d */
  const float *w_in, *b_in;                 /* d x d_ff, d_ff */
  const float *w_out, *b_out;               /* d_ff x d, d */
} fsvd_dense_layer;
/* Caller-owned outputs of one layer, in the fsvd_layer_desc layouts. */
typedef struct fsvd_factor_buffers {
  float *attn_u, *attn_v, *attn_b; /* [3][G][d][r], [3][G][r][d/G], [3][G][d/G] */
  float *out_u, *out_v, *out_b;    /* d x pr, pr x d, d */
  float *up_u, *up_v, *up_b;       /* d x fr, fr x d_ff, d_ff */
  float *down_u, *down_v, *down_b; /* d_ff x fr, fr x d, d */
} fsvd_factor_buffers;
/* synth_model's factorization step (model_io.cpp:486-533) for n_layers dense
 * layers in one batched device run.  Zero ranks resolve as the reference:
 * rank -> d/groups, proj_rank -> min(rank*groups, d), ffn_rank ->
 * min(proj_rank, d, d_ff) (model_io.cpp:489-499); the resolved values are
 * written back through the pointers.  out == NULL only resolves and checks
 * the ranks (size the buffers, then call again). */
fsvd_status fsvd_factorize_layers(const fsvd_dense_layer* layers, size_t n_layers,
                                  size_t groups, size_t* rank, size_t* proj_rank,
                                  size_t* ffn_rank, const fsvd_factor_buffers* out);
/* Jacobi sweeps the last factorization call ran (max over its matrices). */
int fsvd_last_factor_sweeps(void);

/* ------------------------------------------------------------------ */
/* Decoder rows: rank-space KV cache, causal        */
/* prefill and single-token decode steps on the flash tensor-core path. */
/* planner.cpp:123-141 closed forms; PAPER.md "Decoder Memory Cost      */
/* Analysis".  The cache of one layer is [batch, max_seq, 2*G*rp] bf16   */
/* (per token: G rank-space key blocks P_k, then G value blocks P_v).    */
/* Causal semantics: layer by layer, the output at position i is the    */
/* encoder layer's output on the prefix [0, i] of its inputs, last row   */
/* (tests pin exactly that).                                              */
/* ------------------------------------------------------------------ */
/* planner.cpp:123-127: 4 * 2 * layers * B * M * r (FSVD_ERR_CONFIG on an
 * invalid geometry or layers == 0). */
fsvd_status fsvd_decoder_kv_cache_bytes(const fsvd_geometry* geom, size_t* bytes);
/* planner.cpp:129-132: cache + 4 * (3 B M r + 2 B M r). */
fsvd_status fsvd_decoder_prefill_bytes(const fsvd_geometry* geom, size_t* bytes);
/* planner.cpp:134-141: step t in [1, seq_len]:
 * 4 * (2 * layers * B r t + B r (t - 1) + 5 B r). */
fsvd_status fsvd_decoder_decode_step_bytes(const fsvd_geometry* geom, size_t t, size_t* bytes);
/* Device bytes of one layer's cache. */
fsvd_status fsvd_kv_cache_bytes(const fsvd_layer_pack* pack, size_t batch, size_t max_seq,
                                size_t* bytes);
/* Workspace for prefills of up to max_seq tokens and for decode steps. */
fsvd_status fsvd_decoder_workspace_bytes(const fsvd_layer_pack* const* packs, size_t n_layers,
                                         size_t batch, size_t max_seq, int pre_ln,
                                         size_t* bytes);
/* Causal forward of x [batch, seq, d] (seq <= max_seq) through every layer;
 * fills rows [0, seq) of kv_caches[l] (device, one per layer).  x == out
 * allowed.  Async on `stream`. */
fsvd_status fsvd_decoder_prefill(const fsvd_layer_pack* const* packs, size_t n_layers,
                                 int pre_ln, size_t batch, size_t seq, const void* x, void* out,
                                 void* const* kv_caches, size_t max_seq, void* ws,
                                 size_t ws_bytes, void* stream);
/* One new token per sequence at position pos (< max_seq; rows [0, pos) of
 * every cache must hold the earlier tokens): x, out [batch, d]; appends row
 * pos to every cache and attends keys [0, pos]. */
fsvd_status fsvd_decoder_step(const fsvd_layer_pack* const* packs, size_t n_layers, int pre_ln,
                              size_t batch, size_t pos, const void* x, void* out,
                              void* const* kv_caches, size_t max_seq, void* ws, size_t ws_bytes,
                              void* stream);
/* The decode step of fixed buffers (x, out [batch, d], caches, workspace)
 * captured once into a CUDA graph; each replay takes the position as an
 * argument (read on the device), so a serving loop pays one graph launch per
 * token instead of ~11 kernel launches per layer. */
typedef struct fsvd_decoder_graph fsvd_decoder_graph;
fsvd_status fsvd_decoder_graph_create(const fsvd_layer_pack* const* packs, size_t n_layers,
                                      int pre_ln, size_t batch, const void* x, void* out,
                                      void* const* kv_caches, size_t max_seq, void* ws,
                                      size_t ws_bytes, fsvd_decoder_graph** graph);
fsvd_status fsvd_decoder_graph_step(fsvd_decoder_graph* graph, size_t pos, void* stream);
void fsvd_decoder_graph_destroy(fsvd_decoder_graph* graph);

/* ------------------------------------------------------------------ */
/* Device-resident async API (device pointers, cudaStream_t as void*)   */
/* ------------------------------------------------------------------ */
/* Bytes of workspace fsvd_model_fwd needs for this batch shape; the
 * activation buffer planner sizes it by rank, not by hidden width. */
fsvd_status fsvd_workspace_bytes(const fsvd_layer_pack* const* packs, size_t n_layers,
                                 size_t batch, size_t seq, fsvd_run_mode mode,
                                 size_t* bytes);
/* Exact requirement of one layer ordering: pre_ln = 0 (post-LN, the
 * reference default, fused LayerNorm epilogues) or 1.  fsvd_workspace_bytes
 * returns the larger of the two. */
fsvd_status fsvd_workspace_bytes_ln(const fsvd_layer_pack* const* packs, size_t n_layers,
                                    size_t batch, size_t seq, fsvd_run_mode mode, int pre_ln,
                                    size_t* bytes);
/* attention.cpp:202-269 (flash_svd_attention): x, ctx [batch, seq, d]. */
fsvd_status fsvd_attention_fwd(const fsvd_layer_pack* p, size_t batch, size_t seq,
                               const void* x, void* ctx, void* workspace,
                               size_t workspace_bytes, void* stream);
/* attention.cpp:366-391 (lowrank_output_projection) */
fsvd_status fsvd_outproj_fwd(const fsvd_layer_pack* p, size_t batch, size_t seq,
                             const void* ctx, void* out, void* workspace,
                             size_t workspace_bytes, void* stream);
/* ffn.cpp:118-156 (variant 1) and ffn.cpp:158-185 (variant 2) */
fsvd_status fsvd_ffn_fwd(const fsvd_layer_pack* p, int variant, size_t batch, size_t seq,
                         const void* x, void* out, void* workspace,
                         size_t workspace_bytes, void* stream);
/* Post-LN FFN sublayer: out = LN2(x + ffn(x)), the second half of run_layer
 * (encoder.cpp:245-256; ffn_v1 / ffn_v2 then residual_norm).  On the tensor
 * cores this is one kernel for variant 2 (K4 with its LayerNorm epilogue). */
fsvd_status fsvd_ffn_block_workspace_bytes(const fsvd_layer_pack* p, int variant, size_t batch,
                                           size_t seq, size_t* bytes);
fsvd_status fsvd_ffn_block_fwd(const fsvd_layer_pack* p, int variant, size_t batch, size_t seq,
                               const void* x, void* out, void* workspace,
                               size_t workspace_bytes, void* stream);
/* encoder.cpp:224-260 (run_layer).  x and out may alias. */
fsvd_status fsvd_layer_fwd(const fsvd_layer_pack* p, fsvd_run_mode mode, int pre_ln,
                           size_t batch, size_t seq, const void* x, void* out,
                           void* workspace, size_t workspace_bytes, void* stream);
/* encoder.cpp:262-293 (run_model).  x and out may alias. */
fsvd_status fsvd_model_fwd(const fsvd_layer_pack* const* packs, size_t n_layers,
                           fsvd_run_mode mode, int pre_ln, size_t batch, size_t seq,
                           const void* x, void* out, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Serving loop over host memory: runs n_batches forwards of [batch, seq, d]
 * bf16 activations read from x_host[i] and written to out_host[i] (pinned host
 * buffers; the same pointer may repeat).  Host->device copies, the forward and
 * device->host copies of consecutive batches overlap on three streams through
 * two device slots; everything is ordered before the caller's `stream`, so an
 * event recorded on it after the call covers all copies.  workspace must hold
 * fsvd_stream_workspace_bytes(). */
fsvd_status fsvd_stream_workspace_bytes(const fsvd_layer_pack* const* packs, size_t n_layers,
                                        size_t batch, size_t seq, fsvd_run_mode mode,
                                        size_t* bytes);
fsvd_status fsvd_model_fwd_stream(const fsvd_layer_pack* const* packs, size_t n_layers,
                                  fsvd_run_mode mode, int pre_ln, size_t batch, size_t seq,
                                  size_t n_batches, const void* const* x_host,
                                  void* const* out_host, void* workspace, size_t workspace_bytes,
                                  void* stream);

/* ------------------------------------------------------------------ */
/* Host API: behavioural drop-ins for the reference free functions.     */
/* fp32 host in/out, synchronous; H2D -> kernels -> D2H inside.  Shapes, */
/* tile plans and meter pins/regions/transients are checked and charged */
/* exactly as the reference does (4 B/element).  meter may be NULL.      */
/* ------------------------------------------------------------------ */
/* attention.hpp:18-21 */
fsvd_status fsvd_flash_svd_attention(const float* x, size_t batch, size_t seq,
                                     size_t width, const fsvd_attn_desc* set,
                                     size_t heads, const fsvd_tile_plan* plan,
                                     fsvd_dtype dtype, fsvd_meter* meter,
                                     const char* pin_prefix, float* out,
                                     size_t out_batch, size_t out_seq, size_t out_width);
/* attention.hpp:49-51 */
fsvd_status fsvd_lowrank_output_projection(const float* ctx, size_t batch, size_t seq,
                                           size_t width, const fsvd_linear_desc* proj,
                                           fsvd_dtype dtype, fsvd_meter* meter,
                                           const char* pin_prefix, float* out,
                                           size_t out_batch, size_t out_seq,
                                           size_t out_width);
/* ffn.hpp:33-34 (variant 1) and ffn.hpp:40-41 (variant 2) */
fsvd_status fsvd_ffn(int variant, const float* x, size_t batch, size_t seq, size_t width,
                     const fsvd_ffn_desc* f, const fsvd_tile_plan* plan, fsvd_dtype dtype,
                     fsvd_meter* meter, const char* pin_prefix, float* out,
                     size_t out_batch, size_t out_seq, size_t out_width);
/* encoder.hpp:83-85 */
fsvd_status fsvd_run_layer(const float* x, size_t batch, size_t seq, size_t width,
                           const fsvd_layer_desc* layer, fsvd_run_mode mode,
                           const fsvd_tile_plan* plan, int pre_ln, const char* meter_prefix,
                           fsvd_dtype dtype, fsvd_meter* meter, float* out);
/* encoder.hpp:90-92 */
fsvd_status fsvd_run_model(const float* x, size_t batch, size_t seq, size_t width,
                           const fsvd_layer_desc* layers, size_t n_layers,
                           fsvd_run_mode mode, const fsvd_tile_plan* plan, int pre_ln,
                           const char* meter_prefix, fsvd_dtype dtype, fsvd_meter* meter,
                           float* out);

/* ------------------------------------------------------------------ */
/* Instrumentation                                                     */
/* ------------------------------------------------------------------ */
/* Number of kernels this library launched since load (all streams). */
uint64_t fsvd_kernel_launch_count(void);
/* Name of the kernel that dominated the last fsvd_model_fwd schedule. */
const char* fsvd_kernel_name(int kernel_id);

/* ------------------------------------------------------------------ */
/* Kernel test hooks: one tensor-core kernel on caller device buffers   */
/* (bf16 row-major, fp32 vectors), asynchronous on `stream`.  Used by   */
/* the per-kernel numerics tests against a torch fp32 reference.        */
/* ------------------------------------------------------------------ */
/* K1: C[M,N] = A[M,K] B[N,K]^T (+ bias) (act) */
fsvd_status fsvd_test_gemm(const void* A, size_t lda, const void* B, size_t ldb, void* C,
                           size_t ldc, size_t M, size_t N, size_t K, const float* bias,
                           fsvd_activation act, int use_act, void* stream);
/* K6: y = LN(resid + bf16(A B^T + bias)) * gamma + beta */
fsvd_status fsvd_test_gemm_ln(const void* A, size_t lda, const void* B, size_t ldb,
                              const float* bias, const void* resid, const float* gamma,
                              const float* beta, float eps, void* y, size_t T, size_t N,
                              size_t K, void* stream);
/* K2: out[t, h*rp:(h+1)*rp] = softmax2(Qt_h K_g^T) V_g per sequence, rank
 * space; qkv [batch*seq, cols] holds head h's Qt at q_off + h*rp, group g's K
 * at k_off + g*rp and V at v_off + g*rp; scores are in the log2 domain. */
fsvd_status fsvd_test_attention(const void* qkv, size_t cols, size_t q_off, size_t k_off,
                                size_t v_off, size_t batch, size_t seq, size_t heads,
                                size_t groups, size_t rank_pad, void* out, size_t ldo,
                                void* stream);
/* K5: y = LN(a (+ b)) * gamma + beta */
fsvd_status fsvd_test_resid_layernorm(const void* a, const void* b, const float* gamma,
                                      const float* beta, float eps, void* y, size_t rows,
                                      size_t d, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* FSVD_B200_H */
