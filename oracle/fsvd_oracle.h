/*
 * fsvd_oracle.h -- CPU restatement of the FlashSVD reference path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this; the product library never links
 * or calls it.  Every function restates the reference C++ algorithm in plain
 * C, loop order for loop order, so that (compiled with -ffp-contract=off, as
 * the reference build in oracle/Makefile is) it is bit-identical to
 * /root/reference/proj/src.  Parity pinning: tests/test_oracle.py checks this
 * restatement bit-for-bit against the compiled reference (oracle/_ref) and
 * against the committed golden vectors in tests/golden/.
 */
#ifndef FSVD_ORACLE_H
#define FSVD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "fsvd_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* tests/support/oracles.hpp:50-87: mt19937_64 + Box-Muller with a spare. */
void fo_random_fill(float* out, size_t n, uint64_t seed, double stddev);

/* attention.cpp:202-269 (+ online_softmax_head :92-137).  0 on success,
 * else an fsvd_status code (shape/config/budget checks as the reference). */
int fo_flash_svd_attention(const float* x, size_t batch, size_t seq,
                           const fsvd_attn_desc* set, size_t heads,
                           const fsvd_tile_plan* plan, float* out);
/* attention.cpp:366-391 */
int fo_lowrank_output_projection(const float* ctx, size_t batch, size_t seq,
                                 const fsvd_linear_desc* proj, float* out);
/* ffn.cpp:118-156 (variant 1) and :158-185 (variant 2) */
int fo_ffn(int variant, const float* x, size_t batch, size_t seq, size_t width,
           const fsvd_ffn_desc* f, const fsvd_tile_plan* plan, float* out);
/* encoder.cpp:38-50 (residual_norm via tensor.cpp:88-102) */
void fo_residual_norm(const float* a, const float* b, size_t rows, size_t d,
                      const float* gamma, const float* beta, float eps, float* dst);
/* encoder.cpp:224-260; mode is FSVD_MODE_FLASH_V1 or FSVD_MODE_FLASH_V2. */
int fo_run_layer(const float* x, size_t batch, size_t seq, const fsvd_layer_desc* layer,
                 int mode, const fsvd_tile_plan* plan, int pre_ln, float* out);
/* encoder.cpp:262-293 */
int fo_run_model(const float* x, size_t batch, size_t seq, const fsvd_layer_desc* layers,
                 size_t n_layers, int mode, const fsvd_tile_plan* plan, int pre_ln,
                 float* out);

/* memtier.cpp:191-212 */
size_t fo_expected_bytes(int formula, const fsvd_geometry* g);
/* memtier.cpp:125-189: returns working-set bytes; *status = 0 / BUDGET / CONFIG */
size_t fo_tile_working_set(const fsvd_tile_plan* plan, int kind, const fsvd_geometry* g,
                           int* status);
/* encoder.cpp:333-345 */
size_t fo_flash_layer_peak_transient_bytes(const fsvd_geometry* g);
size_t fo_flash_layer_persistent_bytes(const fsvd_geometry* g);

#ifdef __cplusplus
}
#endif
#endif
