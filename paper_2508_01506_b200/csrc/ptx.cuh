// ptx.cuh -- thin inline-PTX layer for sm_100a: mbarrier, TMA, tcgen05/TMEM.
//
// Everything the tensor-core kernels need from the Blackwell execution model
// is wrapped here once: mbarrier phase waits, TMA tile loads/stores, TMEM
// allocation, UMMA shared-memory / instruction descriptors, tcgen05.mma and
// commit, and TMEM->register loads.  Compile with
// -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace fsvd {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Blocks until the phase with the given parity has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// One non-blocking probe of the phase (test_wait: returns at once).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// For a warp that idles through a long phase (e.g. a tail-only producer
// waiting out the whole main loop): polls with a sleep in between, so it
// takes no issue slots or shared-memory cycles from the warps doing the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: a kernel launched with launch_pdl() may start
// while its predecessor on the stream drains.  pdl_trigger() lets the next
// kernel be scheduled; pdl_wait() blocks until the predecessor grid has
// completed and its memory is visible -- every kernel calls it after its
// prologue (barriers, TMEM, descriptor prefetch) and before any global access.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------- CTA timeline (trace builds)
// FSVD_TRACE only: thread 0 of every CTA stamps %globaltimer (ns, comparable
// across SMs) at kernel entry, after pdl_wait and at exit, plus its SM id,
// into a per-translation-unit array copied out by fsvd_debug_cta_times_<tu>.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------------- fences
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 2-D tile load: box at (c0 = inner coordinate, c1 = outer coordinate).
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(const CUtensorMap* map, uint64_t* bar,
                                                 void* dst, int32_t c0, int32_t c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0,
                                             int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
// 3-D store: box {c0, c1, c2} (innermost first); rows past a dimension's
// extent are clipped, so a [batch, seq, cols] map never writes a short
// sequence's tail into the next sequence
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int32_t c0,
                                             int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_u32(const CUtensorMap* map, uint32_t src, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
}
// 1-D bulk copies (contiguous bytes, 16-byte aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- TMEM
// Warp-wide: allocates ncols (power of two >= 32) columns, writes the base
// address into *smem_dst.
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst) {
  static_assert(NCOLS >= 32 && NCOLS <= 512 && (NCOLS & (NCOLS - 1)) == 0, "bad TMEM cols");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOLS)
               : "memory");
}

// ---------------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor (tcgen05 "version 1"):
//   [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version=1,
//   [49,52) base offset (0: tiles are aligned to the swizzle repeat),
//   [61,64) layout: 0 none, 2 SW128, 4 SW64, 6 SW32.
enum Swizzle : uint32_t { SW_NONE = 0, SW128 = 2, SW64 = 4, SW32 = 6 };

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes,
                                              uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout & 7) << 61;
  return d;
}
// K-major operand whose rows are `row_bytes` (= swizzle width) long, packed
// densely: 8-row core groups are 8*row_bytes apart.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t row_bytes) {
  const uint32_t layout = row_bytes == 128 ? SW128 : row_bytes == 64 ? SW64 : SW32;
  return smem_desc(saddr, 16, 8 * row_bytes, layout);
}
// MN-major operand: rows (one per K index) are `row_bytes` long = the whole
// MN extent (<= swizzle width); 8-K-row groups are 8*row_bytes apart.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t saddr, uint32_t row_bytes) {
  const uint32_t layout = row_bytes == 128 ? SW128 : row_bytes == 64 ? SW64 : SW32;
  return smem_desc(saddr, 16, 8 * row_bytes, layout);
}

// Cheap descriptor construction inside MMA issue loops: the constant fields
// are computed once (desc_hi_*), only the 14-bit start address varies.
__device__ __forceinline__ uint64_t desc_hi_kmajor(uint32_t row_bytes) {
  return desc_kmajor(0, row_bytes);
}
__device__ __forceinline__ uint64_t desc_hi_mnmajor(uint32_t row_bytes) {
  return desc_mnmajor(0, row_bytes);
}
__device__ __forceinline__ uint64_t desc_at(uint64_t hi, uint32_t saddr) {
  return hi | static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
}

// Instruction descriptor, kind::f16 with BF16 inputs and FP32 accumulate.
//   [4,6) c_format=1 (F32), [7,10) a_format=1 (BF16), [10,13) b_format=1,
//   [15] a_major, [16] b_major (0 = K-major, 1 = MN-major),
//   [17,23) N>>3, [24,29) M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn = 0,
                                                  uint32_t b_mn = 0) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}
// kind::tf32 (fp32 storage read as TF32).
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N, uint32_t a_mn = 0,
                                                  uint32_t b_mn = 0) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by ONE thread.
__device__ __forceinline__ void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T: A (M x K bf16, two per 32-bit column,
// row m in lane m) read from TMEM, B from shared memory.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrives on an mbarrier once all previously issued tcgen05 ops of this
// thread have completed (implicit before_thread_sync fence).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- TMEM -> registers
// 32 lanes x 32 bit, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a),
               "r"(b)
               : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
               : "=r"(a), "=r"(b)
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
// Cluster of two CTAs on one TPC: the even CTA (rank 0) issues M = 256 MMAs
// whose A rows come half from each CTA's shared memory and whose B (N) is
// split between them; each CTA's TMEM holds its own 128 rows.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// Copies `bytes` of this CTA's shared memory into another CTA of the cluster
// (async proxy); the bytes complete on the destination CTA's mbarrier.
// dst and bar are shared::cluster addresses (mapa_shared).
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst, const void* src, uint32_t bytes,
                                                  uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "r"(smem_u32(src)), "r"(bytes), "r"(bar)
      : "memory");
}
// Arrives on the barrier at this offset in every CTA of `mask` once this
// thread's prior (cta_group::1) MMAs have completed.
__device__ __forceinline__ void mma_commit_multicast(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// Shared::cluster address of `local` in the CTA of rank `cta`.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// Remote arrive with no memory ordering (signals that carry no generic-proxy
// data, e.g. "TMEM region drained"): skips the release fence, which would
// also wait for this thread's in-flight global loads.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA load issued by either CTA of the pair; the transaction bytes complete on
// the LEADER's barrier (rank bit of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst) {
  static_assert(NCOLS >= 32 && NCOLS <= 512 && (NCOLS & (NCOLS - 1)) == 0, "bad TMEM cols");
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_free_pair(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOLS)
               : "memory");
}
__device__ __forceinline__ void mma_bf16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrives on the barrier at this offset in every CTA of `mask` once the
// pair's prior MMAs have completed.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ---------------------------------------------------------------- packing / smem
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// x rounded to bf16 (RNE) and widened back: the hi plane of a split value;
// x - bf16_round_f(x) is its lo plane (split planes, fp32 policy).
__device__ __forceinline__ float bf16_round_f(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
__device__ __forceinline__ void st_shared_v4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
// Byte offset of the 16-byte chunk `chunk` of row `row` inside a tile whose
// rows are `row_bytes` long and swizzled with the matching TMA/UMMA pattern
// (Swizzle<log2(row_bytes/16),4,3>): chunk index XOR (row / (128/row_bytes)) % (row_bytes/16).
__device__ __forceinline__ uint32_t swz_offset(uint32_t row, uint32_t chunk, uint32_t row_bytes) {
  const uint32_t nchunks = row_bytes >> 4;  // 8, 4 or 2
  const uint32_t line = (row * row_bytes) >> 7;  // 128-byte line index
  const uint32_t x = line & (nchunks - 1);
  return row * row_bytes + ((chunk ^ x) << 4);
}

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.79788456080286535588f;
  const float inner = c * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(inner));
}
// Tensor-core epilogue activations: one MUFU op each, error far below the bf16
// rounding applied right after.  GELU-erf writes erf(x/sqrt2) as tanh of an odd
// polynomial fitted for minimax error on [0, 6] (|GELU error| <= 2.6e-5 with an
// exact tanh; z is clamped so the polynomial stays increasing and tanh
// saturates beyond |x| = 5).  GELU-tanh uses the hardware tanh.approx.
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_erf_fast(float x) {
  const float z = fminf(x * x, 25.0f);
  const float p = fmaf(z, fmaf(z, -3.51516791e-4f, 3.70056460e-2f), 7.97507884e-1f);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(x * p), hx);
}
// Packed-pair forms (FMUL2 / FFMA2 on sm_100): same math, half the issue.
__device__ __forceinline__ float2 gelu_erf_fast2(float2 x) {
  float2 z = __fmul2_rn(x, x);
  z.x = fminf(z.x, 25.0f);
  z.y = fminf(z.y, 25.0f);
  float2 p = __ffma2_rn(z, make_float2(-3.51516791e-4f, -3.51516791e-4f),
                        make_float2(3.70056460e-2f, 3.70056460e-2f));
  p = __ffma2_rn(z, p, make_float2(7.97507884e-1f, 7.97507884e-1f));
  const float2 u = __fmul2_rn(x, p);
  const float2 t = make_float2(tanh_approx(u.x), tanh_approx(u.y));
  const float2 hx = __fmul2_rn(x, make_float2(0.5f, 0.5f));
  return __ffma2_rn(hx, t, hx);
}
__device__ __forceinline__ float2 gelu_tanh_fast2(float2 x) {
  const float2 x2 = __fmul2_rn(x, x);
  const float2 in = __fmul2_rn(
      __ffma2_rn(__fmul2_rn(x, make_float2(0.044715f, 0.044715f)), x2, x),
      make_float2(0.79788456080286535588f, 0.79788456080286535588f));
  const float2 t = make_float2(tanh_approx(in.x), tanh_approx(in.y));
  const float2 hx = __fmul2_rn(x, make_float2(0.5f, 0.5f));
  return __ffma2_rn(hx, t, hx);
}
__device__ __forceinline__ float gelu_tanh_fast(float x) {
  const float inner = 0.79788456080286535588f * fmaf(0.044715f * x, x * x, x);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(inner), hx);
}
__device__ __forceinline__ float apply_act(float v, int act) {
  switch (act) {
    case 0: return gelu_erf(v);
    case 1: return gelu_tanh(v);
    case 2: return v > 0.0f ? v : 0.0f;
    default: return v;
  }
}
// Applies the activation to a register chunk (no bias).
// v += b, then the activation, on packed pairs.
template <int N>
__device__ __forceinline__ void bias_act_chunk2(float (&v)[N], const float (&b)[N], int act) {
#pragma unroll
  for (int j = 0; j < N; j += 2) {
    float2 t = __fadd2_rn(make_float2(v[j], v[j + 1]), make_float2(b[j], b[j + 1]));
    if (act == 0) t = gelu_erf_fast2(t);
    else if (act == 1) t = gelu_tanh_fast2(t);
    else if (act == 2) t = make_float2(fmaxf(t.x, 0.0f), fmaxf(t.y, 0.0f));
    v[j] = t.x;
    v[j + 1] = t.y;
  }
}
template <int N>
__device__ __forceinline__ void act_chunk(float (&v)[N], int act) {
  switch (act) {
    case 0:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = gelu_erf_fast(v[j]);
      break;
    case 1:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = gelu_tanh_fast(v[j]);
      break;
    case 2:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = fmaxf(v[j], 0.0f);
      break;
    default:
      break;
  }
}
// fp32 policy (split planes): the activations at full precision (erff /
// tanhf, tensor.cpp:64-74) -- the MUFU forms above are bf16-grade.
template <int N>
__device__ __forceinline__ void bias_act_chunk2_exact(float (&v)[N], const float (&b)[N], int act) {
#pragma unroll
  for (int j = 0; j < N; ++j) v[j] = apply_act(v[j] + b[j], act);
}
template <int N>
__device__ __forceinline__ void bias_act_chunk_exact(float (&v)[N], const float* bias, int valid,
                                                     int act) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    if (bias != nullptr && j < valid) v[j] += __ldg(bias + j);
    v[j] = apply_act(v[j], act);
  }
}
// Loads bias[0..N) into registers (float4 when all N columns are in range).
template <int N>
__device__ __forceinline__ void load_bias(float (&b)[N], const float* bias, int valid) {
  if (valid >= N) {
#pragma unroll
    for (int j = 0; j < N; j += 4) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(bias + j));
      b[j] = t.x; b[j + 1] = t.y; b[j + 2] = t.z; b[j + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) b[j] = j < valid ? __ldg(bias + j) : 0.0f;
  }
}
// Adds bias[0..N) (float4 loads, bias 16-byte aligned; `valid` columns are in
// range) and applies the activation to a 32-wide register chunk.  The switch
// is hoisted out of the element loop so each variant is a straight-line body.
template <int N>
__device__ __forceinline__ void bias_act_chunk(float (&v)[N], const float* bias, int valid,
                                               int act) {
  if (bias != nullptr) {
    if (valid >= N) {
#pragma unroll
      for (int j = 0; j < N; j += 4) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + j));
        v[j] += b.x; v[j + 1] += b.y; v[j + 2] += b.z; v[j + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j < valid) v[j] += __ldg(bias + j);
    }
  }
  switch (act) {
    case 0:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = gelu_erf_fast(v[j]);
      break;
    case 1:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = gelu_tanh_fast(v[j]);
      break;
    case 2:
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = fmaxf(v[j], 0.0f);
      break;
    default:
      break;
  }
}

}  // namespace ptx
}  // namespace fsvd
