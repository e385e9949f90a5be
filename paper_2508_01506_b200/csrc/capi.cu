// capi.cu -- the extern "C" boundary (include/fsvd_b200.h).
//
// Exceptions never cross this file's entry points: every call is wrapped in
// guard(), which maps fsvd::Error kinds 1:1 onto fsvd_status and stores the
// message for fsvd_last_error().
//
// The host API (fsvd_flash_svd_attention ... fsvd_run_model) is the
// behavioural drop-in for the reference free functions: it performs the
// reference's shape / plan checks with the same error kinds, charges the
// meter with the same pins, regions and transient tags at 4 B/element
// (attention.cpp:216-233, :375-379; ffn.cpp:123-128, :163-165;
// encoder.cpp:224-293), then uploads, runs the device schedule and
// downloads.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fsvd_b200.h"
#include "common.cuh"
#include "factorize.hpp"
#include "meter.hpp"
#include "model_file.hpp"
#include "runtime.hpp"

struct fsvd_meter {
  fsvd::Meter m;
};
struct fsvd_decoder_graph {
  cudaGraphExec_t exec = nullptr;
  int* pos_dev = nullptr;
  size_t max_seq = 0;
  ~fsvd_decoder_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (pos_dev) cudaFree(pos_dev);
  }
};

namespace fsvd {
namespace {

thread_local std::string g_last_error;

template <typename F>
fsvd_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return FSVD_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<fsvd_status>(static_cast<int>(e.kind));
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return FSVD_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return FSVD_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FSVD_ERR_CUDA;
  }
}

// tensor.cpp: every extent of a reference tensor is >= 1 (ShapeError otherwise)
void check_extents(size_t batch, size_t seq) {
  if (batch == 0 || seq == 0) fail(Kind::Shape, "tensor extent must be at least 1");
}

void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(Kind::Cuda, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                         "); this library has no CPU fallback");
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) fail(Kind::Cuda, "device is not sm_100 (Blackwell B200)");
}

// ------------------------------------------------------------- plan checks
// memtier.cpp:125-189 (working set in fp32 elements, BudgetError names the
// largest buffer).
size_t working_set(const fsvd_tile_plan& plan, int kind, const fsvd_geometry& g,
                   bool throw_on_budget) {
  if (plan.bm == 0 || plan.br == 0 || plan.bdf == 0)
    fail(Kind::Config, "tile dimensions must be positive");
  if (g.groups == 0 || g.d_model % g.groups != 0) fail(Kind::Config, "groups must divide d_model");
  const size_t bm = plan.bm, br = plan.br, bdf = plan.bdf, gd = g.d_model / g.groups,
               r = g.rank;
  struct Buf {
    const char* name;
    size_t n;
  };
  std::vector<Buf> bufs;
  bufs.reserve(10);
  if (kind == FSVD_KERNEL_ATTENTION)
    bufs = {{"q_tile", bm * gd},   {"k_tile", br * gd},     {"v_tile", br * gd},
            {"score_tile", bm * br}, {"prob_tile", bm * br}, {"out_acc", bm * gd},
            {"load_stage", std::max(bm, br) * gd}, {"row_max", bm}, {"row_sum", bm},
            {"bias_row", gd}};
  else if (kind == FSVD_KERNEL_FFN_V1)
    bufs = {{"h_tile", bm * bdf}, {"p_row_tile", bm * r}, {"z_acc_tile", bm * r},
            {"v1_panel", r * bdf}, {"u2_panel", bdf * r}, {"bias_slice", bdf}};
  else if (kind == FSVD_KERNEL_FFN_V2)
    bufs = {{"h_tile", bm * bdf},  {"p_tile", bm * r},     {"p_row_tile", bm * r},
            {"z_acc_tile", bm * r}, {"v1_panel", r * bdf}, {"u2_panel", bdf * r},
            {"bias_slice", bdf},    {"out_row", g.d_model}};
  else
    fail(Kind::Config, "unknown kernel kind");
  size_t total = 0;
  const Buf* largest = &bufs[0];
  for (const Buf& b : bufs) {
    total += b.n;
    if (b.n > largest->n) largest = &b;
  }
  const size_t bytes = 4 * total;
  if (throw_on_budget && bytes > plan.sram_budget_bytes)
    fail(Kind::Budget, "tile working set " + std::to_string(bytes) + " bytes exceeds budget " +
                           std::to_string(plan.sram_budget_bytes) + "; largest buffer is \"" +
                           largest->name + "\" (" + std::to_string(4 * largest->n) + " bytes)");
  return bytes;
}

fsvd_tile_plan plan_or_default(const fsvd_tile_plan* p) {
  if (p) return *p;
  return fsvd_tile_plan{16, 16, 64, 131072};
}

size_t expected(int id, const fsvd_geometry& g) {
  const size_t b = g.batch, m = g.seq_len, da = g.d_model, df = g.d_ff, h = g.heads,
               gr = g.groups, r = g.rank;
  switch (id) {
    case FSVD_FORMULA_DENSE_ATTN: return 4 * (3 * b * m * da + b * h * m * m);
    case FSVD_FORMULA_FLASH_ATTN_DENSE_QKV: return 4 * (3 * b * m * da);
    case FSVD_FORMULA_FLASH_SVD_ATTN: return 4 * (3 * h * b * m * r);
    case FSVD_FORMULA_GROUPED_ATTN: return 4 * (3 * gr * b * m * r);
    case FSVD_FORMULA_FFN_DENSE:
    case FSVD_FORMULA_FFN_NAIVE_LOWRANK: return 4 * (b * m * df);
    case FSVD_FORMULA_FFN_V1: return 4 * (2 * b * m * r);
    case FSVD_FORMULA_FFN_V2: return 0;
  }
  fail(Kind::Config, "unknown formula id");
}

// ------------------------------------------------------------- host staging
// Device copies of a host fp32 activation in the pack dtype, plus the
// workspace.  The buffers are cached per (host thread, device) and only grow,
// so a repeated synchronous call does no cudaMalloc / cudaFree.

struct ScratchSet {
  void* p[2] = {nullptr, nullptr};  // 0: arena (in / out / workspace), 1: fp32 staging
  size_t cap[2] = {0, 0};
  int device = -1;
  ~ScratchSet() {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return;
    if (device >= 0) cudaSetDevice(device);
    for (void* q : p)
      if (q) cudaFree(q);
    if (cur >= 0) cudaSetDevice(cur);
  }
};

void* scratch(int slot, size_t bytes) {
  thread_local std::map<int, std::unique_ptr<ScratchSet>> sets;
  int dev = 0;
  FSVD_CUDA_CHECK(cudaGetDevice(&dev));
  std::unique_ptr<ScratchSet>& ss = sets[dev];
  if (!ss) {
    ss = std::make_unique<ScratchSet>();
    ss->device = dev;
  }
  if (bytes > ss->cap[slot]) {
    if (ss->p[slot]) {
      FSVD_CUDA_CHECK(cudaDeviceSynchronize());
      cudaFree(ss->p[slot]);
      ss->p[slot] = nullptr;
      ss->cap[slot] = 0;
    }
    FSVD_CUDA_CHECK(cudaMalloc(&ss->p[slot], bytes));
    ss->cap[slot] = bytes;
  }
  return ss->p[slot];
}

// Host fp32 [rows, d] <-> device activations [rows, pack.d] in the pack's
// storage form: bf16, fp32 (CUDA-core fp32 packs) or split planes (fp32 on the
// tensor cores); the tensor-core layouts pad d up to pack.d with zero columns.
int storage_form(const Pack& p) { return p.x3 ? 2 : (p.dtype == FSVD_BF16 ? 0 : 1); }

// Pageable host <-> device copies for the drop-ins.  A pageable cudaMemcpy
// runs at 7-15 GB/s on the B200 hosts (D2H the slower); instead the bytes go
// through two pinned 8 MiB chunks: host threads copy chunk k into one while
// the DMA engine moves chunk k-1 out of the other (51 GB/s), so a 50 MB
// activation crosses in ~2 ms each way instead of 3.5 / 7 ms.
// A few persistent host threads for the drop-ins' bulk host work (chunk
// memcpys, content hashes): run(job) calls job(part, parts) on every member
// and the caller, and returns when all are done.  One job at a time.
class HostTeam {
 public:
  static HostTeam& get() {
    static HostTeam t;
    return t;
  }
  size_t parts() const { return workers_.size() + 1; }
  void run(const std::function<void(size_t, size_t)>& job) {
    std::lock_guard<std::mutex> one(run_mu_);
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &job;
      pending_ = workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    job(0, parts());
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return pending_ == 0; });
  }
  // memcpy of n bytes split over the team
  void copy(void* dst, const void* src, size_t n) {
    if (n < (size_t(1) << 20)) {
      std::memcpy(dst, src, n);
      return;
    }
    run([=](size_t i, size_t np) {
      np = std::min<size_t>(np, 8);  // more copy threads measured slower
      if (i >= np) return;
      const size_t step = (n / np + 63) & ~size_t(63);
      const size_t o = std::min(n, i * step), e = std::min(n, o + step);
      if (e > o) std::memcpy(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o, e - o);
    });
  }

 private:
  HostTeam() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    const size_t nw = std::min<size_t>(15, hw - 1);
    for (size_t w = 0; w < nw; ++w)
      workers_.emplace_back([this, w] {
        uint64_t seen = 0;
        for (;;) {
          const std::function<void(size_t, size_t)>* job;
          {
            std::unique_lock<std::mutex> g(mu_);
            cv_.wait(g, [&] { return gen_ != seen || stop_; });
            if (stop_) return;
            seen = gen_;
            job = job_;
          }
          (*job)(w + 1, workers_.size() + 1);
          std::lock_guard<std::mutex> g(mu_);
          if (--pending_ == 0) done_.notify_one();
        }
      });
  }
  ~HostTeam() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t, size_t)>* job_ = nullptr;
  size_t pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct PinnedChunks {
  static constexpr size_t kChunk = size_t(8) << 20;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int device = -1;
};
std::mutex g_pinned_mu;  // one staged copy at a time per process

PinnedChunks& pinned_chunks() {
  static std::map<int, PinnedChunks> per_dev;
  int dev = 0;
  FSVD_CUDA_CHECK(cudaGetDevice(&dev));
  PinnedChunks& pc = per_dev[dev];
  if (pc.buf[0] == nullptr) {
    for (int i = 0; i < 2; ++i) {
      FSVD_CUDA_CHECK(cudaHostAlloc(&pc.buf[i], PinnedChunks::kChunk, cudaHostAllocDefault));
      FSVD_CUDA_CHECK(cudaEventCreateWithFlags(&pc.ev[i], cudaEventDisableTiming));
    }
    pc.device = dev;
  }
  return pc;
}

void staged_h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_pinned_mu);
  PinnedChunks& pc = pinned_chunks();
  const size_t nch = (n + PinnedChunks::kChunk - 1) / PinnedChunks::kChunk;
  for (size_t k = 0; k < nch; ++k) {
    const int b = static_cast<int>(k & 1);
    const size_t o = k * PinnedChunks::kChunk, len = std::min(PinnedChunks::kChunk, n - o);
    FSVD_CUDA_CHECK(cudaEventSynchronize(pc.ev[b]));  // the last DMA from this chunk is out
    HostTeam::get().copy(pc.buf[b], static_cast<const uint8_t*>(src) + o, len);
    FSVD_CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + o, pc.buf[b], len,
                                    cudaMemcpyHostToDevice, s));
    FSVD_CUDA_CHECK(cudaEventRecord(pc.ev[b], s));
  }
}

void staged_d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(g_pinned_mu);
  PinnedChunks& pc = pinned_chunks();
  const size_t nch = (n + PinnedChunks::kChunk - 1) / PinnedChunks::kChunk;
  auto dma = [&](size_t k) {
    const int b = static_cast<int>(k & 1);
    const size_t o = k * PinnedChunks::kChunk, len = std::min(PinnedChunks::kChunk, n - o);
    FSVD_CUDA_CHECK(cudaMemcpyAsync(pc.buf[b], static_cast<const uint8_t*>(src) + o, len,
                                    cudaMemcpyDeviceToHost, s));
    FSVD_CUDA_CHECK(cudaEventRecord(pc.ev[b], s));
  };
  if (nch > 0) dma(0);
  for (size_t k = 0; k < nch; ++k) {
    const int b = static_cast<int>(k & 1);
    const size_t o = k * PinnedChunks::kChunk, len = std::min(PinnedChunks::kChunk, n - o);
    if (k + 1 < nch) dma(k + 1);  // into the other chunk (its host copy finished last round)
    FSVD_CUDA_CHECK(cudaEventSynchronize(pc.ev[b]));
    HostTeam::get().copy(static_cast<uint8_t*>(dst) + o, pc.buf[b], len);
  }
}

void upload(const float* host, size_t rows, const Pack& p, void* dev, cudaStream_t s) {
  const size_t n = rows * p.dr;
  float* tmp = static_cast<float*>(scratch(1, n * 4));
  staged_h2d(tmp, host, n * 4, s);
  rows_to_device(tmp, static_cast<int>(rows), p.dr, p.d, storage_form(p), dev, s);
}
void download(const void* dev, size_t rows, const Pack& p, float* host, cudaStream_t s) {
  const size_t n = rows * p.dr;
  float* tmp = static_cast<float*>(scratch(1, n * 4));
  rows_from_device(dev, static_cast<int>(rows), p.dr, p.d, storage_form(p), tmp, s);
  staged_d2h(host, tmp, n * 4, s);
  FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
}

// Runs fn(x_dev, out_dev, trans_dev, stream) on the cached device arena for
// `rows` activation rows of width pack.dr in and out, and reports the arena
// to the meter's device high-water.
template <typename F>
void run_on_device(const float* x, size_t rows, float* out, const Pack& pack, size_t trans_bytes,
                   Meter* meter, F&& fn) {
  require_device();
  const size_t bytes = (rows * pack.d * pack.es + 255) & ~size_t(255);
  uint8_t* base = static_cast<uint8_t*>(scratch(0, 2 * bytes + trans_bytes + 256));
  cudaStream_t s = nullptr;
  upload(x, rows, pack, base, s);
  fn(base, base + bytes, base + 2 * bytes, s);
  FSVD_CUDA_CHECK(cudaGetLastError());
  download(base + bytes, rows, pack, out, s);
  if (meter) meter->note_device(2 * bytes + trans_bytes, pack.bytes);
}

// ------------------------------------------------------------- pack cache
// The host drop-ins receive fp32 factors on every call (the reference's
// signatures, encoder.hpp:83-92), and the reference's own bench loop calls
// run_model again and again on the same layers (commands.cpp:289-307).  A
// pack (fp64 folds on the host, bf16 / fp32 device layouts, H2D) is therefore
// cached per (device, dtype, content): the key is a 64-bit hash of every
// factor, bias and LayerNorm array plus the geometry, computed over the host
// threads in parallel.  An unchanged layer costs one read of its host arrays;
// any changed value -- even written in place at the same address -- rebuilds.
// LRU, capped at FSVD_PACK_CACHE_MB (default 2048; 0 disables the cache).
struct Span {
  const void* p;
  size_t n;
};

inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull, kP2 = 0xC2B2AE3D27D4EB4Full,
                   kP3 = 0x165667B19E3779F9ull;

uint64_t hash_bytes(const uint8_t* p, size_t n, uint64_t seed) {
  uint64_t a[4] = {seed + kP1 + kP2, seed + kP2, seed, seed - kP1};
  size_t i = 0;
  for (; i + 32 <= n; i += 32)
    for (int l = 0; l < 4; ++l) {
      uint64_t w;
      std::memcpy(&w, p + i + 8 * l, 8);
      a[l] = rotl64(a[l] + w * kP2, 31) * kP1;
    }
  uint64_t h = rotl64(a[0], 1) + rotl64(a[1], 7) + rotl64(a[2], 12) + rotl64(a[3], 18) + n;
  for (; i < n; ++i) h = rotl64(h ^ (p[i] * kP3), 11) * kP1;
  h ^= h >> 33;
  h *= kP2;
  h ^= h >> 29;
  h *= kP3;
  h ^= h >> 32;
  return h;
}

uint64_t hash_spans(const std::vector<Span>& spans) {
  constexpr size_t kChunk = size_t(1) << 20;
  std::vector<Span> chunks;
  for (const Span& sp : spans) {
    if (sp.n == 0 || sp.p == nullptr) {
      chunks.push_back({nullptr, 0});  // still contributes its position
      continue;
    }
    for (size_t o = 0; o < sp.n; o += kChunk)
      chunks.push_back({static_cast<const uint8_t*>(sp.p) + o, std::min(kChunk, sp.n - o)});
  }
  std::vector<uint64_t> hs(chunks.size());
  auto work = [&](size_t w, size_t nw) {
    for (size_t i = w; i < chunks.size(); i += nw)
      hs[i] = chunks[i].p ? hash_bytes(static_cast<const uint8_t*>(chunks[i].p), chunks[i].n, i)
                          : kP3 + i;
  };
  if (chunks.size() <= 2)
    work(0, 1);
  else
    HostTeam::get().run(work);  // persistent threads: no spawn per call
  uint64_t h = kP1 ^ chunks.size();
  for (uint64_t x : hs) h = rotl64(h ^ (x * kP2), 27) * kP1 + kP3;
  return h;
}

uint64_t hash_request(const PackRequest& q, fsvd_dtype dt) {
  std::vector<uint64_t> hdr = {static_cast<uint64_t>(dt), q.heads, q.d_model,
                               static_cast<uint64_t>(q.dense)};
  uint32_t e1, e2;
  std::memcpy(&e1, &q.eps1, 4);
  std::memcpy(&e2, &q.eps2, 4);
  hdr.push_back((uint64_t(e1) << 32) | e2);
  std::vector<Span> spans;
  auto lin = [&](const fsvd_linear_desc* l) {
    if (!l) {
      hdr.insert(hdr.end(), {0, 0, 0});
      return;
    }
    hdr.insert(hdr.end(), {l->in_dim, l->rank, l->out_dim});
    spans.push_back({l->u, 4 * l->in_dim * l->rank});
    spans.push_back({l->v, 4 * l->rank * l->out_dim});
    spans.push_back({l->bias, 4 * l->out_dim});
  };
  if (q.attn) {
    const fsvd_attn_desc& a = *q.attn;
    hdr.insert(hdr.end(), {1, a.d_model, a.groups, a.rank});
    spans.push_back({a.u, 4 * 3 * a.groups * a.d_model * a.rank});
    spans.push_back({a.v, 4 * 3 * a.rank * a.d_model});
    spans.push_back({a.bias, 4 * 3 * a.d_model});
  } else {
    hdr.push_back(0);
  }
  lin(q.out_proj);
  if (q.ffn) {
    hdr.insert(hdr.end(), {2, static_cast<uint64_t>(q.ffn->activation)});
    lin(&q.ffn->up);
    lin(&q.ffn->down);
  } else {
    hdr.push_back(0);
  }
  if (q.dense_w) {
    const fsvd_dense_layer& w = *q.dense_w;
    const size_t d = w.d_model, df = w.d_ff;
    hdr.insert(hdr.end(), {3, d, df, static_cast<uint64_t>(q.dense_act)});
    for (const float* m : {w.wq, w.wk, w.wv, w.wo}) spans.push_back({m, 4 * d * d});
    for (const float* b : {w.bq, w.bk, w.bv, w.bo, w.b_out}) spans.push_back({b, 4 * d});
    spans.push_back({w.w_in, 4 * d * df});
    spans.push_back({w.b_in, 4 * df});
    spans.push_back({w.w_out, 4 * df * d});
  } else {
    hdr.push_back(0);
  }
  for (const float* v : {q.ln1g, q.ln1b, q.ln2g, q.ln2b}) {
    hdr.push_back(v != nullptr);
    if (v) spans.push_back({v, 4 * q.d_model});
  }
  spans.insert(spans.begin(), Span{hdr.data(), hdr.size() * sizeof(uint64_t)});
  return hash_spans(spans);
}

struct PackCache {
  struct Entry {
    std::shared_ptr<Pack> pack;
    uint64_t tick;
  };
  std::mutex mu;
  std::map<std::pair<int, uint64_t>, Entry> map;
  size_t bytes = 0;
  uint64_t tick = 0, hits = 0, misses = 0;
  size_t cap() const {
    const char* e = std::getenv("FSVD_PACK_CACHE_MB");
    return (e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) : 2048) << 20;
  }
};
PackCache& pack_cache() {
  static PackCache* c = new PackCache();  // leaked: outlives static destructors
  return *c;
}

std::shared_ptr<Pack> cached_pack(const PackRequest& q, fsvd_dtype dt) {
  PackCache& c = pack_cache();
  const size_t cap = c.cap();
  if (cap == 0) return std::shared_ptr<Pack>(build_pack(q, dt));
  int dev = 0;
  FSVD_CUDA_CHECK(cudaGetDevice(&dev));
  const std::pair<int, uint64_t> key{dev, hash_request(q, dt)};
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.map.find(key);
    if (it != c.map.end()) {
      it->second.tick = ++c.tick;
      ++c.hits;
      return it->second.pack;
    }
    ++c.misses;
  }
  std::shared_ptr<Pack> p(build_pack(q, dt));
  std::lock_guard<std::mutex> lk(c.mu);
  auto ins = c.map.emplace(key, PackCache::Entry{p, ++c.tick});
  if (ins.second) c.bytes += p->bytes;
  while (c.bytes > cap && c.map.size() > 1) {  // evict least recently used
    auto lru = c.map.begin();
    for (auto it = c.map.begin(); it != c.map.end(); ++it)
      if (it->second.tick < lru->second.tick) lru = it;
    if (lru->first == key) break;
    c.bytes -= lru->second.pack->bytes;
    c.map.erase(lru);
  }
  return ins.first->second.pack;
}

// Pack request of one layer descriptor: each representation only if present.
PackRequest request_of(const fsvd_layer_desc& L, bool dense) {
  PackRequest q;
  if (L.attn.u) {
    q.attn = &L.attn;
    q.out_proj = &L.out_proj;
  }
  if (L.ffn.up.u) q.ffn = &L.ffn;
  q.heads = L.heads;
  q.ln1g = L.ln1_gamma;
  q.ln1b = L.ln1_beta;
  q.ln2g = L.ln2_gamma;
  q.ln2b = L.ln2_beta;
  q.eps1 = L.ln1_eps;
  q.eps2 = L.ln2_eps;
  q.d_model = L.attn.d_model;
  q.dense = dense;
  q.dense_w = dense ? L.dense : nullptr;
  q.dense_act = static_cast<int>(L.ffn.activation);
  return q;
}

std::shared_ptr<Pack> pack_attention(const fsvd_attn_desc& a, size_t heads, fsvd_dtype dt) {
  PackRequest q;
  q.attn = &a;
  q.heads = heads;
  q.d_model = a.d_model;
  return cached_pack(q, dt);
}

void check_dtype(fsvd_dtype dt) {
  if (dt != FSVD_F32 && dt != FSVD_BF16) fail(Kind::Config, "unknown dtype");
}

// ---- reference-equivalent sublayers (checks + meter + device) ----------------
void check_attention_io(size_t width, size_t d_model, size_t heads, size_t ob, size_t om,
                        size_t ow, size_t b, size_t m) {
  // attention.cpp:47-56
  if (width != d_model) fail(Kind::Shape, "input feature width does not match the projections");
  if (heads == 0 || d_model % heads != 0) fail(Kind::Config, "heads must divide d_model");
  if (ob != b || om != m || ow != width)
    fail(Kind::Shape, "attention output must be shaped like the input");
}

void host_attention(const float* x, size_t B, size_t M, size_t W, const fsvd_attn_desc& a,
                    size_t heads, const fsvd_tile_plan& plan, fsvd_dtype dt, Meter* meter,
                    const std::string& pfx, float* out, size_t ob, size_t om, size_t ow) {
  check_dtype(dt);
  check_attention_io(W, a.d_model, heads, ob, om, ow, B, M);
  if (a.groups == 0 || heads % a.groups != 0)
    fail(Kind::Config, "factor groups must evenly cover the heads");
  if (B == 0 || M == 0) fail(Kind::Shape, "tensor extent must be at least 1");
  const size_t d = a.d_model, G = a.groups, r = a.rank, gd = d / G;
  fsvd_geometry geo{B, M, d, 1, heads, heads, 1, 1};
  working_set(plan, FSVD_KERNEL_ATTENTION, geo, true);
  static const char* names[3] = {"q", "k", "v"};
  if (meter)
    for (int mat = 0; mat < 3; ++mat)
      for (size_t g = 0; g < G; ++g)
        meter->pin(pfx + "." + names[mat] + ".g" + std::to_string(g) + ".v", 4 * r * gd);
  MeterScope region(meter, "flash_svd_attention");
  MeterBuffer pq(meter, "p_q", MeterClass::Transient, G * B * M * r);
  MeterBuffer pk(meter, "p_k", MeterClass::Transient, G * B * M * r);
  MeterBuffer pv(meter, "p_v", MeterClass::Transient, G * B * M * r);
  require_device();
  auto pack = pack_attention(a, heads, dt);
  const size_t trans = B * M * op_transient_elems(*pack, 0, FSVD_MODE_FLASH_V1) * pack->es;
  run_on_device(x, B * M, out, *pack, trans, meter,
                [&](void* xd, void* od, void* td, cudaStream_t s) {
                  attention_fwd(*pack, FSVD_MODE_FLASH_V1, B, M, xd, od, td, s);
                });
}

void host_outproj(const float* ctx, size_t B, size_t M, size_t W, const fsvd_linear_desc& o,
                  fsvd_dtype dt, Meter* meter, const std::string& pfx, float* out, size_t ob,
                  size_t om, size_t ow) {
  check_dtype(dt);
  // attention.cpp:369-372
  if (W != o.in_dim) fail(Kind::Shape, "context width does not match the projection factors");
  if (ob != B || om != M || ow != W || o.out_dim != W)
    fail(Kind::Shape, "output projection must preserve the activation shape");
  const size_t d = o.in_dim, r = o.rank;
  if (meter) {
    meter->pin(pfx + ".out.u", 4 * d * r);
    meter->pin(pfx + ".out.v", 4 * r * o.out_dim);
  }
  MeterScope region(meter, "lowrank_output_projection");
  MeterBuffer p(meter, "p_out", MeterClass::Transient, B * M * r);
  require_device();
  PackRequest q;
  q.out_proj = &o;
  q.d_model = d;
  std::shared_ptr<Pack> pack = cached_pack(q, dt);
  const size_t trans = B * M * op_transient_elems(*pack, 1, FSVD_MODE_FLASH_V1) * pack->es;
  run_on_device(ctx, B * M, out, *pack, trans, meter,
                [&](void* xd, void* od, void* td, cudaStream_t s) {
                  outproj_fwd(*pack, FSVD_MODE_FLASH_V1, B, M, xd, od, td, s);
                });
}

void check_ffn_io(size_t W, const fsvd_ffn_desc& f, size_t ob, size_t om, size_t ow, size_t B,
                  size_t M) {
  // ffn.cpp:40-50
  if (f.up.in_dim != W || f.down.out_dim != W)
    fail(Kind::Shape, "ffn factor dims do not match the activation width");
  if (f.up.out_dim != f.down.in_dim) fail(Kind::Shape, "ffn up/down widths do not chain");
  if (f.up.rank != f.down.rank) fail(Kind::Config, "ffn factor pairs must share one rank");
  if (ob != B || om != M || ow != W) fail(Kind::Shape, "ffn output must be shaped like input");
}

void host_ffn(int variant, const float* x, size_t B, size_t M, size_t W, const fsvd_ffn_desc& f,
              const fsvd_tile_plan& plan, fsvd_dtype dt, Meter* meter, const std::string& pfx,
              float* out, size_t ob, size_t om, size_t ow) {
  check_dtype(dt);
  if (variant != 1 && variant != 2) fail(Kind::Config, "ffn variant must be 1 or 2");
  check_ffn_io(W, f, ob, om, ow, B, M);
  const size_t d = W, df = f.up.out_dim, r = f.up.rank;
  fsvd_geometry geo{B, M, d, df, 1, 1, r, 1};
  working_set(plan, variant == 1 ? FSVD_KERNEL_FFN_V1 : FSVD_KERNEL_FFN_V2, geo, true);
  if (meter) {  // ffn.cpp:64-70
    meter->pin(pfx + ".up.u", 4 * d * r);
    meter->pin(pfx + ".up.v", 4 * r * df);
    meter->pin(pfx + ".down.u", 4 * df * r);
    meter->pin(pfx + ".down.v", 4 * r * d);
  }
  MeterScope region(meter, variant == 1 ? "ffn_v1" : "ffn_v2");
  std::unique_ptr<MeterBuffer> pm, zm;
  if (variant == 1) {
    pm = std::make_unique<MeterBuffer>(meter, "p_mid", MeterClass::Transient, B * M * r);
    zm = std::make_unique<MeterBuffer>(meter, "z_mid", MeterClass::Transient, B * M * r);
  }
  require_device();
  PackRequest q;
  q.ffn = &f;
  q.d_model = d;
  std::shared_ptr<Pack> pack = cached_pack(q, dt);
  const int mode = variant == 1 ? FSVD_MODE_FLASH_V1 : FSVD_MODE_FLASH_V2;
  const size_t trans = B * M * op_transient_elems(*pack, 2, mode) * pack->es;
  run_on_device(x, B * M, out, *pack, trans, meter,
                [&](void* xd, void* od, void* td, cudaStream_t s) {
                  ffn_fwd(*pack, mode, B, M, xd, od, td, s);
                });
  zm.reset();
  pm.reset();
}

// Meter sequence of one layer (encoder.cpp:224-260) for every run mode; the
// device work runs separately on the whole model (layer_fwd).
void meter_layer(Meter* meter, const fsvd_layer_desc& L, int mode, const fsvd_tile_plan& plan,
                 bool pre_ln, const std::string& pfx, size_t B, size_t M) {
  const size_t d = L.attn.d_model, n = B * M * d, G = L.attn.groups ? L.attn.groups : 1,
               r = L.attn.rank, gd = d / G,
               df = L.ffn.up.u ? L.ffn.up.out_dim : (L.dense ? L.dense->d_ff : 0),
               fr = L.ffn.up.rank, pr = L.out_proj.rank, H = L.heads;
  MeterBuffer ctx(meter, pfx + ".attn_ctx", MeterClass::Excluded, n);
  MeterBuffer branch(meter, pfx + ".sublayer_out", MeterClass::Excluded, n);
  MeterBuffer resid(meter, pfx + ".resid", MeterClass::Excluded, n);
  std::unique_ptr<MeterBuffer> normed;
  if (pre_ln) normed = std::make_unique<MeterBuffer>(meter, pfx + ".norm_in", MeterClass::Excluded, n);
  {
    MeterScope sub(meter, pfx + ".attn");
    if (mode == FSVD_MODE_DENSE) {
      MeterScope rg(meter, "dense_attention");
      MeterBuffer q(meter, "q_full", MeterClass::Transient, n);
      MeterBuffer k(meter, "k_full", MeterClass::Transient, n);
      MeterBuffer v(meter, "v_full", MeterClass::Transient, n);
      MeterBuffer sc(meter, "scores", MeterClass::Transient, B * H * M * M);
    } else if (mode == FSVD_MODE_NAIVE_LOWRANK) {
      fsvd_geometry geo{B, M, d, 1, H, H, 1, 1};
      working_set(plan, FSVD_KERNEL_ATTENTION, geo, true);
      MeterScope rg(meter, "naive_lowrank_attention");
      MeterBuffer q(meter, "q_full", MeterClass::Transient, n);
      MeterBuffer k(meter, "k_full", MeterClass::Transient, n);
      MeterBuffer v(meter, "v_full", MeterClass::Transient, n);
    } else {
      fsvd_geometry geo{B, M, d, 1, H, H, 1, 1};
      working_set(plan, FSVD_KERNEL_ATTENTION, geo, true);
      static const char* names[3] = {"q", "k", "v"};
      if (meter)
        for (int mat = 0; mat < 3; ++mat)
          for (size_t g = 0; g < G; ++g)
            meter->pin(pfx + ".attn." + names[mat] + ".g" + std::to_string(g) + ".v", 4 * r * gd);
      {
        MeterScope rg(meter, "flash_svd_attention");
        MeterBuffer pq(meter, "p_q", MeterClass::Transient, G * B * M * r);
        MeterBuffer pk(meter, "p_k", MeterClass::Transient, G * B * M * r);
        MeterBuffer pv(meter, "p_v", MeterClass::Transient, G * B * M * r);
      }
      if (meter) {
        meter->pin(pfx + ".attn.out.u", 4 * d * pr);
        meter->pin(pfx + ".attn.out.v", 4 * pr * d);
      }
      MeterScope rg(meter, "lowrank_output_projection");
      MeterBuffer p(meter, "p_out", MeterClass::Transient, B * M * pr);
    }
  }
  {
    MeterScope sub(meter, pfx + ".ffn");
    if (mode == FSVD_MODE_DENSE || mode == FSVD_MODE_NAIVE_LOWRANK) {
      MeterScope rg(meter, mode == FSVD_MODE_DENSE ? "ffn_dense" : "ffn_naive_lowrank");
      MeterBuffer h(meter, "hidden", MeterClass::Transient, B * M * df);
    } else {
      const bool v1 = mode == FSVD_MODE_FLASH_V1;
      fsvd_geometry geo{B, M, d, df, 1, 1, fr, 1};
      working_set(plan, v1 ? FSVD_KERNEL_FFN_V1 : FSVD_KERNEL_FFN_V2, geo, true);
      if (meter) {
        meter->pin(pfx + ".ffn.up.u", 4 * d * fr);
        meter->pin(pfx + ".ffn.up.v", 4 * fr * df);
        meter->pin(pfx + ".ffn.down.u", 4 * df * fr);
        meter->pin(pfx + ".ffn.down.v", 4 * fr * d);
      }
      MeterScope rg(meter, v1 ? "ffn_v1" : "ffn_v2");
      if (v1) {
        MeterBuffer pm(meter, "p_mid", MeterClass::Transient, B * M * fr);
        MeterBuffer zm(meter, "z_mid", MeterClass::Transient, B * M * fr);
      }
    }
  }
}

void check_mode(int mode) {
  if (mode < FSVD_MODE_DENSE || mode > FSVD_MODE_FLASH_V2) fail(Kind::Config, "unknown run mode");
}

void host_run_model(const float* x, size_t B, size_t M, size_t W, const fsvd_layer_desc* layers,
                    size_t n_layers, int mode, const fsvd_tile_plan& plan, bool pre_ln,
                    const std::string& prefix, fsvd_dtype dt, Meter* meter, float* out,
                    bool single_layer_api) {
  check_dtype(dt);
  check_mode(mode);
  if (B == 0 || M == 0 || W == 0) fail(Kind::Shape, "run_model: x must be (batch, seq, d_model)");
  if (x == out) fail(Kind::Config, "run_model: out must be a distinct tensor");
  if (n_layers == 0) {
    std::memcpy(out, x, sizeof(float) * B * M * W);
    return;
  }
  for (size_t i = 0; i < n_layers; ++i) {
    validate_layer(layers[i]);
    check_mode_weights(layers[i], mode, true);
    if (layers[i].attn.d_model != W) fail(Kind::Shape, "run_layer: x must be (batch, seq, d_model)");
  }
  // meter: encoder.cpp:274-292 (ping/pong only for more than one layer)
  {
    std::unique_ptr<MeterBuffer> ping, pong;
    if (!single_layer_api && n_layers > 1) {
      ping = std::make_unique<MeterBuffer>(meter, prefix + ".interlayer.0", MeterClass::Excluded, B * M * W);
      pong = std::make_unique<MeterBuffer>(meter, prefix + ".interlayer.1", MeterClass::Excluded, B * M * W);
    }
    for (size_t i = 0; i < n_layers; ++i) {
      const std::string pfx = single_layer_api ? prefix : prefix + "." + std::to_string(i);
      meter_layer(meter, layers[i], mode, plan, pre_ln, pfx, B, M);
    }
  }
  // device
  require_device();
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::shared_ptr<Pack>> packs;
  size_t ws = 0, pack_bytes = 0;
  for (size_t i = 0; i < n_layers; ++i) {
    const PackRequest q =
        request_of(layers[i], mode == FSVD_MODE_DENSE || mode == FSVD_MODE_NAIVE_LOWRANK);
    packs.emplace_back(cached_pack(q, dt));
    if (q.dense && !packs.back()->dense)
      fail(Kind::Config, "dense / naive_lowrank modes run on the tensor cores only: head width "
                         "<= 64, d_model and d_ff multiples of 8");
    ws = std::max(ws, layer_workspace_bytes(*packs.back(), B, M, mode, pre_ln != 0));
    pack_bytes += packs.back()->bytes;
    if (packs.back()->x3 != packs[0]->x3)
      fail(Kind::Config, "fp32 policy: every layer must fit the tensor-core tiling, or none");
  }
  for (const auto& q : packs)
    if (q->d != packs[0]->d)
      fail(Kind::Config, "every layer must use the same device layout (tensor-core tiling)");
  static const bool prof = std::getenv("FSVD_DROPIN_PROFILE") != nullptr;  // developer timing
  const auto t1 = std::chrono::steady_clock::now();
  run_on_device(x, B * M, out, *packs[0], ws, nullptr,
                [&](void* xd, void* od, void* td, cudaStream_t s) {
                  std::vector<const Pack*> pp;
                  for (auto& p : packs) pp.push_back(p.get());
                  if (prof) {
                    FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
                    std::fprintf(stderr, "[dropin] upload %.2f ms\n",
                                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
                  }
                  const auto t2 = std::chrono::steady_clock::now();
                  model_layers_fwd(pp.data(), n_layers, mode, pre_ln, B, M, xd, od, td, ws, s);
                  if (prof) {
                    FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
                    std::fprintf(stderr, "[dropin] forward %.2f ms\n",
                                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t2).count());
                  }
                });
  if (prof)
    std::fprintf(stderr, "[dropin] packs (hash) %.2f ms, total after packs %.2f ms\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
  if (meter) meter->note_device(2 * B * M * W * packs[0]->es + ws, pack_bytes);
}

}  // namespace
}  // namespace fsvd

namespace fsvd {
namespace {
// factorize.cpp:25-39: geometry checks of factorize_attention.
void check_attention_factoring(size_t d, size_t groups, size_t rank) {
  if (groups == 0 || d % groups != 0) fail(Kind::Config, "groups must divide d_model");
  if (rank == 0) fail(Kind::Rank, "rank must be at least 1");
  if (rank > d / groups) fail(Kind::Rank, "rank exceeds per-group width d_model/groups");
}
// factorize.cpp:52-62: column block g of each projection -> one job.
void attention_jobs(const float* const w[3], size_t d, size_t groups, size_t rank, float* u,
                    float* v, std::vector<FactorJob>& js) {
  const size_t gd = d / groups;
  for (size_t m = 0; m < 3; ++m)
    for (size_t g = 0; g < groups; ++g) {
      const size_t i = m * groups + g;
      js.push_back({w[m] + g * gd, d, d, gd, rank, u + i * d * rank, v + i * rank * gd});
    }
}
void copy_attention_bias(const float* const b[3], size_t d, float* bias) {
  for (size_t m = 0; m < 3; ++m) std::memcpy(bias + m * d, b[m], d * sizeof(float));
}
}  // namespace
}  // namespace fsvd

using namespace fsvd;

extern "C" {

int fsvd_abi_version(void) { return FSVD_ABI_VERSION; }
const char* fsvd_last_error(void) { return g_last_error.c_str(); }
int fsvd_device_available(void) {
  return guard([] { require_device(); }) == FSVD_OK ? 1 : 0;
}

// ---------------------------------------------------------------- meter
fsvd_status fsvd_meter_create(fsvd_meter** out) {
  return guard([&] {
    if (!out) fail(Kind::Config, "null out pointer");
    *out = new fsvd_meter();
  });
}
void fsvd_meter_destroy(fsvd_meter* m) { delete m; }
fsvd_status fsvd_meter_alloc(fsvd_meter* m, const char* tag, fsvd_alloc_class cls, size_t bytes,
                             uint64_t* id) {
  return guard([&] {
    const uint64_t h = m->m.alloc(tag ? tag : "", static_cast<MeterClass>(cls), bytes);
    if (id) *id = h;
  });
}
fsvd_status fsvd_meter_free(fsvd_meter* m, uint64_t id) {
  return guard([&] { m->m.free(id); });
}
fsvd_status fsvd_meter_pin(fsvd_meter* m, const char* tag, size_t bytes) {
  return guard([&] { m->m.pin(tag ? tag : "", bytes); });
}
fsvd_status fsvd_meter_region_begin(fsvd_meter* m, const char* name, size_t* entry) {
  return guard([&] {
    const size_t e = m->m.region_begin(name ? name : "");
    if (entry) *entry = e;
  });
}
fsvd_status fsvd_meter_region_end(fsvd_meter* m, const char* name, size_t entry) {
  return guard([&] { m->m.region_end(name ? name : "", entry); });
}
size_t fsvd_meter_current_transient(const fsvd_meter* m) { return m->m.current_transient(); }
size_t fsvd_meter_peak_transient(const fsvd_meter* m) { return m->m.peak_transient(); }
size_t fsvd_meter_persistent(const fsvd_meter* m) { return m->m.persistent(); }
size_t fsvd_meter_current_excluded(const fsvd_meter* m) { return m->m.current_excluded(); }
void fsvd_meter_reset_peak(fsvd_meter* m) { m->m.reset_peak(); }
fsvd_status fsvd_meter_assert_clean(const fsvd_meter* m) {
  return guard([&] { m->m.assert_clean(); });
}
size_t fsvd_meter_event_count(const fsvd_meter* m) { return m->m.event_count(); }
fsvd_status fsvd_meter_event(const fsvd_meter* m, size_t index, int* kind, int* cls, size_t* bytes,
                             uint64_t* id, char* tag, size_t tag_cap) {
  return guard([&] {
    if (index >= m->m.event_count()) fail(Kind::Config, "event index out of range");
    const MeterEventRec e = m->m.event(index);
    if (kind) *kind = static_cast<int>(e.kind);
    if (cls) *cls = static_cast<int>(e.cls);
    if (bytes) *bytes = e.bytes;
    if (id) *id = e.id;
    if (tag && tag_cap) {
      std::strncpy(tag, e.tag.c_str(), tag_cap - 1);
      tag[tag_cap - 1] = 0;
    }
  });
}
size_t fsvd_meter_device_peak_bytes(const fsvd_meter* m) { return m->m.device_peak(); }
size_t fsvd_meter_device_persistent_bytes(const fsvd_meter* m) { return m->m.device_persistent(); }

// ---------------------------------------------------------------- closed forms
fsvd_status fsvd_validate_tile_plan(const fsvd_tile_plan* plan, fsvd_kernel_kind kind,
                                    const fsvd_geometry* geom, size_t* bytes) {
  size_t b = 0;
  fsvd_status st = guard([&] {
    if (!plan || !geom) fail(Kind::Config, "null argument");
    b = working_set(*plan, kind, *geom, false);
    if (bytes) *bytes = b;
    working_set(*plan, kind, *geom, true);
  });
  return st;
}
fsvd_status fsvd_expected_bytes(fsvd_formula id, const fsvd_geometry* geom, size_t* bytes) {
  return guard([&] {
    if (!geom || !bytes) fail(Kind::Config, "null argument");
    *bytes = expected(id, *geom);
  });
}
namespace {
// geometry.hpp:24-34
void validate_geometry(const fsvd_geometry& g) {
  if (g.batch == 0 || g.seq_len == 0 || g.d_model == 0 || g.d_ff == 0)
    fail(Kind::Config, "geometry extents must be positive");
  if (g.heads == 0 || g.d_model % g.heads != 0) fail(Kind::Config, "heads must divide d_model");
  if (g.groups == 0 || g.d_model % g.groups != 0) fail(Kind::Config, "groups must divide d_model");
  if (g.rank == 0) fail(Kind::Rank, "rank must be at least 1");
  if (g.rank > g.d_model / g.groups) fail(Kind::Rank, "rank exceeds per-group width d_model/groups");
}
uint64_t gemm_flops(uint64_t m, uint64_t k, uint64_t n) { return 2 * m * k * n; }
}  // namespace

fsvd_status fsvd_flops_exact(const fsvd_geometry* geom, fsvd_run_mode mode, uint64_t* flops) {
  return guard([&] {
    if (!geom || !flops) fail(Kind::Config, "null argument");
    check_mode(mode);
    const fsvd_geometry& g = *geom;
    validate_geometry(g);
    const uint64_t bm = (uint64_t)g.batch * g.seq_len, m = g.seq_len, da = g.d_model,
                   df = g.d_ff, h = g.heads, gr = g.groups, r = g.rank, dh = da / h;
    const uint64_t score_value = g.batch * h * (gemm_flops(m, dh, m) + gemm_flops(m, m, dh));
    if (mode == FSVD_MODE_DENSE) {
      *flops = 4 * gemm_flops(bm, da, da) + score_value + gemm_flops(bm, da, df) +
               gemm_flops(bm, df, da);
      return;
    }
    *flops = 3 * gr * gemm_flops(bm, da, r) + 3 * gr * gemm_flops(bm, r, da / gr) + score_value +
             gemm_flops(bm, da, r) + gemm_flops(bm, r, da) + gemm_flops(bm, da, r) +
             gemm_flops(bm, r, df) + gemm_flops(bm, df, r) + gemm_flops(bm, r, da);
  });
}
fsvd_status fsvd_io_bytes(const fsvd_geometry* geom, fsvd_run_mode mode, uint64_t* in_bytes,
                          uint64_t* out_bytes) {
  return guard([&] {
    if (!geom || !in_bytes || !out_bytes) fail(Kind::Config, "null argument");
    check_mode(mode);
    validate_geometry(*geom);
    const uint64_t bm = (uint64_t)geom->batch * geom->seq_len, da = geom->d_model,
                   df = geom->d_ff, r = geom->rank;
    *out_bytes = 4 * 2 * bm * da;
    *in_bytes = mode == FSVD_MODE_DENSE ? 4 * (3 * bm * da + 2 * bm * df)
                                        : 4 * (4 * bm * r + 3 * r * da + 2 * r * df);
  });
}
size_t fsvd_flash_layer_peak_transient_bytes(const fsvd_geometry* g) {
  return 4 * 3 * g->groups * g->batch * g->seq_len * g->rank;
}
size_t fsvd_flash_layer_persistent_bytes(const fsvd_geometry* g) {
  return 4 * g->rank * (7 * g->d_model + 2 * g->d_ff);
}
size_t fsvd_flash_layer_bound_bytes(const fsvd_geometry* g) {
  const size_t c = std::max<size_t>(3 * g->groups, 7);
  return 4 * c * g->rank * (g->batch * g->seq_len + g->d_model + g->d_ff);
}

// ---------------------------------------------------------------- packs
fsvd_status fsvd_layer_pack_create(const fsvd_layer_desc* layer, fsvd_dtype dtype, int dense,
                                   fsvd_layer_pack** out) {
  return guard([&] {
    if (!layer || !out) fail(Kind::Config, "null argument");
    check_dtype(dtype);
    validate_layer(*layer);
    require_device();
    const PackRequest q = request_of(*layer, dense != 0);
    std::unique_ptr<Pack> p(build_pack(q, dtype));
    *out = new fsvd_layer_pack{p.release()};
  });
}
void fsvd_layer_pack_destroy(fsvd_layer_pack* p) {
  if (p) {
    delete p->p;
    delete p;
  }
}
size_t fsvd_layer_pack_device_bytes(const fsvd_layer_pack* p) { return p ? p->p->bytes : 0; }
size_t fsvd_layer_pack_row_pitch(const fsvd_layer_pack* p) {
  return p ? static_cast<size_t>(p->p->d) : 0;
}
int fsvd_layer_pack_uses_tensor_cores(const fsvd_layer_pack* p) {
  return p && ((p->p->attn_tc && p->p->out_tc && p->p->ffn_tc) || p->p->x3) ? 1 : 0;
}

// ---------------------------------------------------------------- device API
fsvd_status fsvd_workspace_bytes(const fsvd_layer_pack* const* packs, size_t n_layers,
                                 size_t batch, size_t seq, fsvd_run_mode mode, size_t* bytes) {
  return guard([&] {
    if (!bytes) fail(Kind::Config, "null argument");
    check_mode(mode);
    size_t ws = 0;
    for (size_t i = 0; i < n_layers; ++i)
      ws = std::max(ws, layer_workspace_bytes(*packs[i]->p, batch, seq, mode));
    *bytes = ws;
  });
}
fsvd_status fsvd_workspace_bytes_ln(const fsvd_layer_pack* const* packs, size_t n_layers,
                                    size_t batch, size_t seq, fsvd_run_mode mode, int pre_ln,
                                    size_t* bytes) {
  return guard([&] {
    if (!bytes) fail(Kind::Config, "null argument");
    check_mode(mode);
    size_t ws = 0;
    for (size_t i = 0; i < n_layers; ++i)
      ws = std::max(ws, layer_workspace_bytes(*packs[i]->p, batch, seq, mode, pre_ln != 0));
    *bytes = ws;
  });
}
fsvd_status fsvd_attention_fwd(const fsvd_layer_pack* p, size_t batch, size_t seq, const void* x,
                               void* ctx, void* ws, size_t ws_bytes, void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    const size_t need = batch * seq * op_transient_elems(*p->p, 0, FSVD_MODE_FLASH_V1) * p->p->es;
    if (ws_bytes < need) fail(Kind::Config, "workspace too small for attention");
    attention_fwd(*p->p, FSVD_MODE_FLASH_V1, batch, seq, x, ctx, ws, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_outproj_fwd(const fsvd_layer_pack* p, size_t batch, size_t seq, const void* ctx,
                             void* out, void* ws, size_t ws_bytes, void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    const size_t need = batch * seq * op_transient_elems(*p->p, 1, FSVD_MODE_FLASH_V1) * p->p->es;
    if (ws_bytes < need) fail(Kind::Config, "workspace too small for the output projection");
    outproj_fwd(*p->p, FSVD_MODE_FLASH_V1, batch, seq, ctx, out, ws, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_ffn_fwd(const fsvd_layer_pack* p, int variant, size_t batch, size_t seq,
                         const void* x, void* out, void* ws, size_t ws_bytes, void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    if (variant != 1 && variant != 2) fail(Kind::Config, "ffn variant must be 1 or 2");
    const int mode = variant == 1 ? FSVD_MODE_FLASH_V1 : FSVD_MODE_FLASH_V2;
    const size_t need = batch * seq * op_transient_elems(*p->p, 2, mode) * p->p->es;
    if (ws_bytes < need) fail(Kind::Config, "workspace too small for the FFN");
    ffn_fwd(*p->p, mode, batch, seq, x, out, ws, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_ffn_block_workspace_bytes(const fsvd_layer_pack* p, int variant, size_t batch,
                                           size_t seq, size_t* bytes) {
  return guard([&] {
    if (!p || !bytes) fail(Kind::Config, "null argument");
    if (variant != 1 && variant != 2) fail(Kind::Config, "ffn variant must be 1 or 2");
    *bytes = ffn_block_workspace_bytes(*p->p, batch, seq,
                                       variant == 1 ? FSVD_MODE_FLASH_V1 : FSVD_MODE_FLASH_V2);
  });
}
fsvd_status fsvd_ffn_block_fwd(const fsvd_layer_pack* p, int variant, size_t batch, size_t seq,
                               const void* x, void* out, void* ws, size_t ws_bytes, void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    if (variant != 1 && variant != 2) fail(Kind::Config, "ffn variant must be 1 or 2");
    ffn_block_fwd(*p->p, variant == 1 ? FSVD_MODE_FLASH_V1 : FSVD_MODE_FLASH_V2, batch, seq, x,
                  out, ws, ws_bytes, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_layer_fwd(const fsvd_layer_pack* p, fsvd_run_mode mode, int pre_ln, size_t batch,
                           size_t seq, const void* x, void* out, void* ws, size_t ws_bytes,
                           void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    check_mode(mode);
    layer_fwd(*p->p, mode, pre_ln != 0, batch, seq, x, out, ws, ws_bytes,
              static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_model_fwd(const fsvd_layer_pack* const* packs, size_t n_layers,
                           fsvd_run_mode mode, int pre_ln, size_t batch, size_t seq,
                           const void* x, void* out, void* ws, size_t ws_bytes, void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    check_mode(mode);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n_layers == 0) {
      if (x != out) fail(Kind::Config, "model_fwd with no layers needs x == out or a copy");
      return;
    }
    std::vector<const Pack*> pp;
    for (size_t i = 0; i < n_layers; ++i) pp.push_back(packs[i]->p);
    model_layers_fwd(pp.data(), n_layers, mode, pre_ln != 0, batch, seq, x, out, ws, ws_bytes, s);
  });
}

namespace {
size_t stream_slot_bytes(const fsvd_layer_pack* const* packs, size_t batch, size_t seq) {
  const Pack& p0 = *packs[0]->p;
  return (batch * seq * p0.d * p0.es + 255) & ~size_t(255);
}
// Internal copy streams and events of the serving loop (one set per thread).
struct StreamSet {
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t h2d[2], comp[2], d2h[2], entry = nullptr;
  int device = -1;
  ~StreamSet() {
    if (in) {
      cudaStreamDestroy(in);
      cudaStreamDestroy(out);
      for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(h2d[i]);
        cudaEventDestroy(comp[i]);
        cudaEventDestroy(d2h[i]);
      }
      cudaEventDestroy(entry);
    }
  }
};
StreamSet& stream_set() {
  // one set per (host thread, device): a thread that switches devices keeps
  // each device's streams instead of leaking them
  thread_local std::map<int, std::unique_ptr<StreamSet>> sets;
  int dev = 0;
  FSVD_CUDA_CHECK(cudaGetDevice(&dev));
  std::unique_ptr<StreamSet>& slot = sets[dev];
  if (!slot) {
    auto ss = std::make_unique<StreamSet>();
    FSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&ss->in, cudaStreamNonBlocking));
    FSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&ss->out, cudaStreamNonBlocking));
    FSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ss->entry, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      FSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ss->h2d[i], cudaEventDisableTiming));
      FSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ss->comp[i], cudaEventDisableTiming));
      FSVD_CUDA_CHECK(cudaEventCreateWithFlags(&ss->d2h[i], cudaEventDisableTiming));
    }
    ss->device = dev;
    slot = std::move(ss);
  }
  return *slot;
}
}  // namespace

fsvd_status fsvd_pack_cache_stats(size_t* entries, size_t* bytes, uint64_t* hits,
                                  uint64_t* misses) {
  return guard([&] {
    PackCache& c = pack_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (entries) *entries = c.map.size();
    if (bytes) *bytes = c.bytes;
    if (hits) *hits = c.hits;
    if (misses) *misses = c.misses;
  });
}

fsvd_status fsvd_pack_cache_clear(void) {
  return guard([&] {
    PackCache& c = pack_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.map.clear();
    c.bytes = 0;
  });
}

fsvd_status fsvd_model_file_probe(const char* path, size_t* n_layers, fsvd_geometry* geom) {
  return guard([&] {
    if (!path) fail(Kind::Config, "null argument");
    std::unique_ptr<ModelFile> mf = read_model_file(path);
    if (n_layers) *n_layers = mf->layers.size();
    if (geom) {
      *geom = fsvd_geometry{};
      geom->layers = mf->layers.size();
      if (!mf->layers.empty()) {
        const fsvd_layer_desc& d = mf->layers[0].desc;
        geom->d_model = d.attn.d_model;
        geom->d_ff = d.ffn.up.out_dim;
        geom->heads = d.heads;
        geom->groups = d.attn.groups;
        geom->rank = d.attn.rank;
      }
    }
  });
}
fsvd_status fsvd_model_load(const char* path, fsvd_dtype dtype, int dense,
                            fsvd_layer_pack** packs, size_t capacity, size_t* n_layers) {
  return guard([&] {
    if (!path) fail(Kind::Config, "null argument");
    check_dtype(dtype);
    std::unique_ptr<ModelFile> mf = read_model_file(path);
    if (n_layers) *n_layers = mf->layers.size();
    if (!packs) return;
    if (capacity < mf->layers.size())
      fail(Kind::Config, "pack capacity " + std::to_string(capacity) + " < " +
                             std::to_string(mf->layers.size()) + " layers in the file");
    require_device();
    std::vector<std::unique_ptr<fsvd_layer_pack>> made;
    for (const ModelFile::Layer& L : mf->layers) {
      fsvd_layer_pack* p = nullptr;
      const fsvd_status st = fsvd_layer_pack_create(&L.desc, dtype, dense, &p);
      if (st != FSVD_OK) throw Error(static_cast<Kind>(st), fsvd_last_error());
      made.emplace_back(p);
    }
    for (size_t i = 0; i < made.size(); ++i) packs[i] = made[i].release();
  });
}
size_t fsvd_last_error_offset(void) { return format_error_offset(); }

// ------------------------------------------------------------ factorization
fsvd_status fsvd_factor_rank_r(const float* a, size_t m, size_t n, size_t rank, float* u,
                               float* v) {
  return guard([&] {
    check_factor_job(m, n, rank);
    require_device();
    factor_rank_r_batch({FactorJob{a, n, m, n, rank, u, v}});
  });
}
fsvd_status fsvd_factor_rank_r_batch(const fsvd_factor_job* jobs, size_t count) {
  return guard([&] {
    if (count && !jobs) fail(Kind::Config, "null argument");
    std::vector<FactorJob> js;
    for (size_t i = 0; i < count; ++i) {
      check_factor_job(jobs[i].m, jobs[i].n, jobs[i].rank);
      js.push_back({jobs[i].a, jobs[i].n, jobs[i].m, jobs[i].n, jobs[i].rank, jobs[i].u, jobs[i].v});
    }
    require_device();
    factor_rank_r_batch(js);
  });
}


fsvd_status fsvd_factorize_attention(const float* wq, const float* bq, const float* wk,
                                     const float* bk, const float* wv, const float* bv,
                                     size_t d_model, size_t groups, size_t rank, float* u,
                                     float* v, float* bias) {
  return guard([&] {
    if (!wq || !bq || !wk || !bk || !wv || !bv || !u || !v || !bias)
      fail(Kind::Config, "null argument");
    if (d_model == 0) fail(Kind::Shape, "attention projections must be square d_model x d_model");
    check_attention_factoring(d_model, groups, rank);
    require_device();
    const float* w[3] = {wq, wk, wv};
    const float* b[3] = {bq, bk, bv};
    std::vector<FactorJob> js;
    attention_jobs(w, d_model, groups, rank, u, v, js);
    factor_rank_r_batch(js);
    copy_attention_bias(b, d_model, bias);
  });
}

fsvd_status fsvd_factorize_layers(const fsvd_dense_layer* layers, size_t n_layers,
                                  size_t groups, size_t* rank, size_t* proj_rank,
                                  size_t* ffn_rank, const fsvd_factor_buffers* out) {
  return guard([&] {
    if (!layers || n_layers == 0) fail(Kind::Config, "synth_model: need at least one layer");
    if (!rank || !proj_rank || !ffn_rank) fail(Kind::Config, "null argument");
    const size_t d = layers[0].d_model, df = layers[0].d_ff;
    for (size_t l = 0; l < n_layers; ++l)
      if (layers[l].d_model != d || layers[l].d_ff != df || d == 0 || df == 0)
        fail(Kind::Shape, "every layer must share a nonzero d_model / d_ff");
    // model_io.cpp:482-499: zero knobs resolve to the matched defaults
    if (groups == 0 || d % groups != 0) fail(Kind::Config, "groups must divide d_model");
    const size_t r = *rank == 0 ? d / groups : *rank;
    const size_t pr = *proj_rank == 0 ? std::min(r * groups, d) : *proj_rank;
    const size_t fr = *ffn_rank == 0 ? std::min(pr, std::min(d, df)) : *ffn_rank;
    check_attention_factoring(d, groups, r);
    if (pr > d) fail(Kind::Rank, "proj_rank exceeds d_model");
    if (fr > std::min(d, df)) fail(Kind::Rank, "ffn_rank exceeds min(d_model, d_ff)");
    check_factor_job(d, d, pr);
    check_factor_job(d, df, fr);
    *rank = r;
    *proj_rank = pr;
    *ffn_rank = fr;
    if (!out) return;
    require_device();
    std::vector<FactorJob> js;
    for (size_t l = 0; l < n_layers; ++l) {
      const fsvd_dense_layer& L = layers[l];
      const fsvd_factor_buffers& o = out[l];
      const float* w[3] = {L.wq, L.wk, L.wv};
      for (const float* p : {L.wq, L.bq, L.wk, L.bk, L.wv, L.bv, L.wo, L.bo, L.w_in, L.b_in,
                             L.w_out, L.b_out})
        if (!p) fail(Kind::Config, "null dense weight");
      for (float* p : {o.attn_u, o.attn_v, o.attn_b, o.out_u, o.out_v, o.out_b, o.up_u, o.up_v,
                       o.up_b, o.down_u, o.down_v, o.down_b})
        if (!p) fail(Kind::Config, "null output buffer");
      attention_jobs(w, d, groups, r, o.attn_u, o.attn_v, js);
      js.push_back({L.wo, d, d, d, pr, o.out_u, o.out_v});
      js.push_back({L.w_in, df, d, df, fr, o.up_u, o.up_v});
      js.push_back({L.w_out, d, df, d, fr, o.down_u, o.down_v});
    }
    factor_rank_r_batch(js);
    for (size_t l = 0; l < n_layers; ++l) {
      const fsvd_dense_layer& L = layers[l];
      const fsvd_factor_buffers& o = out[l];
      const float* b[3] = {L.bq, L.bk, L.bv};
      copy_attention_bias(b, d, o.attn_b);
      std::memcpy(o.out_b, L.bo, d * sizeof(float));
      std::memcpy(o.up_b, L.b_in, df * sizeof(float));
      std::memcpy(o.down_b, L.b_out, d * sizeof(float));
    }
  });
}
int fsvd_last_factor_sweeps(void) { return last_factor_sweeps(); }

// ------------------------------------------------------------ decoder rows
namespace {
// geometry.hpp:24-34 (Geometry::validate) + planner.cpp:41-43 (require_layers)
void validate_decoder_geometry(const fsvd_geometry& g) {
  if (g.batch == 0 || g.seq_len == 0 || g.d_model == 0 || g.d_ff == 0)
    fail(Kind::Config, "geometry extents must be positive");
  if (g.heads == 0 || g.d_model % g.heads != 0) fail(Kind::Config, "heads must divide d_model");
  if (g.groups == 0 || g.d_model % g.groups != 0) fail(Kind::Config, "groups must divide d_model");
  if (g.rank == 0) fail(Kind::Rank, "rank must be at least 1");
  if (g.rank > g.d_model / g.groups) fail(Kind::Rank, "rank exceeds per-group width d_model/groups");
  if (g.layers == 0) fail(Kind::Config, "decoder needs at least one layer");
}
size_t kv_closed(const fsvd_geometry& g) {
  validate_decoder_geometry(g);
  return 4 * 2 * g.layers * g.batch * g.seq_len * g.rank;
}
void check_decoder_call(const fsvd_layer_pack* const* packs, size_t n_layers,
                        void* const* caches, size_t batch, size_t max_seq) {
  if (!packs || n_layers == 0 || !caches) fail(Kind::Config, "null argument");
  if (batch == 0 || max_seq == 0) fail(Kind::Config, "batch and max_seq must be positive");
  for (size_t i = 0; i < n_layers; ++i) {
    if (!packs[i] || !caches[i]) fail(Kind::Config, "null layer pack or cache");
    check_decoder_pack(*packs[i]->p);
  }
}
}  // namespace

fsvd_status fsvd_decoder_kv_cache_bytes(const fsvd_geometry* geom, size_t* bytes) {
  return guard([&] {
    if (!geom || !bytes) fail(Kind::Config, "null argument");
    *bytes = kv_closed(*geom);
  });
}
fsvd_status fsvd_decoder_prefill_bytes(const fsvd_geometry* geom, size_t* bytes) {
  return guard([&] {
    if (!geom || !bytes) fail(Kind::Config, "null argument");
    const size_t bmr = geom->batch * geom->seq_len * geom->rank;
    *bytes = kv_closed(*geom) + 4 * (3 * bmr + 2 * bmr);
  });
}
fsvd_status fsvd_decoder_decode_step_bytes(const fsvd_geometry* geom, size_t t, size_t* bytes) {
  return guard([&] {
    if (!geom || !bytes) fail(Kind::Config, "null argument");
    validate_decoder_geometry(*geom);
    if (t < 1 || t > geom->seq_len) fail(Kind::Config, "decode step must lie in [1, seq_len]");
    const size_t br = geom->batch * geom->rank;
    *bytes = 4 * (2 * geom->layers * br * t + br * (t - 1) + 5 * br);
  });
}
fsvd_status fsvd_kv_cache_bytes(const fsvd_layer_pack* pack, size_t batch, size_t max_seq,
                                size_t* bytes) {
  return guard([&] {
    if (!pack || !bytes) fail(Kind::Config, "null argument");
    check_decoder_pack(*pack->p);
    *bytes = kv_cache_bytes(*pack->p, batch, max_seq);
  });
}
fsvd_status fsvd_decoder_workspace_bytes(const fsvd_layer_pack* const* packs, size_t n_layers,
                                         size_t batch, size_t max_seq, int pre_ln,
                                         size_t* bytes) {
  return guard([&] {
    if (!packs || n_layers == 0 || !bytes) fail(Kind::Config, "null argument");
    size_t ws = 0;
    for (size_t i = 0; i < n_layers; ++i) {
      check_decoder_pack(*packs[i]->p);
      ws = std::max(ws, decoder_workspace_bytes(*packs[i]->p, batch, max_seq, pre_ln != 0));
    }
    *bytes = ws;
  });
}
fsvd_status fsvd_decoder_prefill(const fsvd_layer_pack* const* packs, size_t n_layers,
                                 int pre_ln, size_t batch, size_t seq, const void* x, void* out,
                                 void* const* kv_caches, size_t max_seq, void* ws,
                                 size_t ws_bytes, void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    check_decoder_call(packs, n_layers, kv_caches, batch, max_seq);
    if (seq == 0 || seq > max_seq) fail(Kind::Config, "prefill length must lie in [1, max_seq]");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    bool done = false;  // pre-LN chaining as in model_layers_fwd (runtime.cu)
    for (size_t i = 0; i < n_layers; ++i) {
      AttnMode am;
      am.kind = AttnMode::Prefill;
      am.cache = kv_caches[i];
      am.max_seq = max_seq;
      am.pos = 0;
      LayerLink lk;
      lk.ln1_done = done;
      if (pre_ln && i + 1 < n_layers &&
          pre_ln_link_ok(*packs[i]->p, *packs[i + 1]->p, FSVD_MODE_FLASH_V2, batch * seq))
        lk.next = packs[i + 1]->p;
      layer_fwd(*packs[i]->p, FSVD_MODE_FLASH_V2, pre_ln != 0, batch, seq, i == 0 ? x : out, out,
                ws, ws_bytes, s, am, lk);
      done = lk.next != nullptr;
    }
  });
}
fsvd_status fsvd_decoder_graph_create(const fsvd_layer_pack* const* packs, size_t n_layers,
                                      int pre_ln, size_t batch, const void* x, void* out,
                                      void* const* kv_caches, size_t max_seq, void* ws,
                                      size_t ws_bytes, fsvd_decoder_graph** graph) {
  return guard([&] {
    check_extents(batch, 1);
    check_decoder_call(packs, n_layers, kv_caches, batch, max_seq);
    if (!graph || !x || !out || !ws) fail(Kind::Config, "null argument");
    require_device();
    auto g = std::make_unique<fsvd_decoder_graph>();
    g->max_seq = max_seq;
    FSVD_CUDA_CHECK(cudaMalloc(&g->pos_dev, sizeof(int)));
    FSVD_CUDA_CHECK(cudaMemset(g->pos_dev, 0, sizeof(int)));
    cudaStream_t cs = nullptr;
    FSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t gr = nullptr;
    FSVD_CUDA_CHECK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    try {
      for (size_t i = 0; i < n_layers; ++i) {
        AttnMode am;
        am.kind = AttnMode::Decode;
        am.cache = kv_caches[i];
        am.max_seq = max_seq;
        am.pos_dev = g->pos_dev;
        layer_fwd(*packs[i]->p, FSVD_MODE_FLASH_V2, pre_ln != 0, batch, 1, i == 0 ? x : out, out,
                  ws, ws_bytes, cs, am);
      }
    } catch (...) {
      cudaStreamEndCapture(cs, &gr);
      if (gr) cudaGraphDestroy(gr);
      cudaStreamDestroy(cs);
      throw;
    }
    FSVD_CUDA_CHECK(cudaStreamEndCapture(cs, &gr));
    const cudaError_t ie = cudaGraphInstantiate(&g->exec, gr, 0);
    cudaGraphDestroy(gr);
    cudaStreamDestroy(cs);
    FSVD_CUDA_CHECK(ie);
    *graph = g.release();
  });
}
fsvd_status fsvd_decoder_graph_step(fsvd_decoder_graph* graph, size_t pos, void* stream) {
  return guard([&] {
    if (!graph) fail(Kind::Config, "null argument");
    if (pos >= graph->max_seq) fail(Kind::Config, "decode position must be below max_seq");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    set_device_int(graph->pos_dev, static_cast<int>(pos), s);
    FSVD_CUDA_CHECK(cudaGraphLaunch(graph->exec, s));
  });
}
void fsvd_decoder_graph_destroy(fsvd_decoder_graph* graph) { delete graph; }
fsvd_status fsvd_decoder_step(const fsvd_layer_pack* const* packs, size_t n_layers, int pre_ln,
                              size_t batch, size_t pos, const void* x, void* out,
                              void* const* kv_caches, size_t max_seq, void* ws, size_t ws_bytes,
                              void* stream) {
  return guard([&] {
    check_extents(batch, 1);
    check_decoder_call(packs, n_layers, kv_caches, batch, max_seq);
    if (pos >= max_seq) fail(Kind::Config, "decode position must be below max_seq");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (size_t i = 0; i < n_layers; ++i) {
      AttnMode am;
      am.kind = AttnMode::Decode;
      am.cache = kv_caches[i];
      am.max_seq = max_seq;
      am.pos = pos;
      layer_fwd(*packs[i]->p, FSVD_MODE_FLASH_V2, pre_ln != 0, batch, 1, i == 0 ? x : out, out,
                ws, ws_bytes, s, am);
    }
  });
}

fsvd_status fsvd_stream_workspace_bytes(const fsvd_layer_pack* const* packs, size_t n_layers,
                                        size_t batch, size_t seq, fsvd_run_mode mode,
                                        size_t* bytes) {
  return guard([&] {
    if (!bytes || !packs || n_layers == 0) fail(Kind::Config, "null argument");
    check_mode(mode);
    size_t ws = 0;
    for (size_t i = 0; i < n_layers; ++i)
      ws = std::max(ws, layer_workspace_bytes(*packs[i]->p, batch, seq, mode));
    *bytes = ws + 2 * stream_slot_bytes(packs, batch, seq) + 256;
  });
}

fsvd_status fsvd_model_fwd_stream(const fsvd_layer_pack* const* packs, size_t n_layers,
                                  fsvd_run_mode mode, int pre_ln, size_t batch, size_t seq,
                                  size_t n_batches, const void* const* x_host,
                                  void* const* out_host, void* ws, size_t ws_bytes,
                                  void* stream) {
  return guard([&] {
    check_extents(batch, seq);
    check_mode(mode);
    if (!packs || n_layers == 0 || (n_batches && (!x_host || !out_host)))
      fail(Kind::Config, "null argument");
    require_device();
    size_t need = 0;
    for (size_t i = 0; i < n_layers; ++i)
      need = std::max(need, layer_workspace_bytes(*packs[i]->p, batch, seq, mode, pre_ln != 0));
    const size_t slot = stream_slot_bytes(packs, batch, seq);
    if (ws_bytes < need + 2 * slot + 256)
      fail(Kind::Config, "workspace too small: need " + std::to_string(need + 2 * slot + 256) +
                             " bytes (fsvd_stream_workspace_bytes)");
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
    uint8_t* dev[2] = {base, base + slot};
    void* model_ws = base + 2 * slot;
    const size_t bytes = batch * seq * packs[0]->p->d * packs[0]->p->es;
    cudaStream_t sc = static_cast<cudaStream_t>(stream);
    StreamSet& ss = stream_set();
    std::vector<const Pack*> pp;
    for (size_t l = 0; l < n_layers; ++l) pp.push_back(packs[l]->p);
    // The copy streams start behind everything already queued on the
    // caller's stream (e.g. a previous call's forward or D2H still using the
    // same workspace slots).
    FSVD_CUDA_CHECK(cudaEventRecord(ss.entry, sc));
    FSVD_CUDA_CHECK(cudaStreamWaitEvent(ss.in, ss.entry, 0));
    FSVD_CUDA_CHECK(cudaStreamWaitEvent(ss.out, ss.entry, 0));
    for (size_t i = 0; i < n_batches; ++i) {
      const int k = static_cast<int>(i & 1);
      // slot k is free once batch i-2 has been copied out of it
      if (i >= 2) FSVD_CUDA_CHECK(cudaStreamWaitEvent(ss.in, ss.d2h[k], 0));
      FSVD_CUDA_CHECK(cudaMemcpyAsync(dev[k], x_host[i], bytes, cudaMemcpyHostToDevice, ss.in));
      FSVD_CUDA_CHECK(cudaEventRecord(ss.h2d[k], ss.in));
      FSVD_CUDA_CHECK(cudaStreamWaitEvent(sc, ss.h2d[k], 0));
      model_layers_fwd(pp.data(), n_layers, mode, pre_ln != 0, batch, seq, dev[k], dev[k], model_ws,
                       ws_bytes - (static_cast<uint8_t*>(model_ws) - static_cast<uint8_t*>(ws)), sc);
      FSVD_CUDA_CHECK(cudaEventRecord(ss.comp[k], sc));
      FSVD_CUDA_CHECK(cudaStreamWaitEvent(ss.out, ss.comp[k], 0));
      FSVD_CUDA_CHECK(cudaMemcpyAsync(out_host[i], dev[k], bytes, cudaMemcpyDeviceToHost, ss.out));
      FSVD_CUDA_CHECK(cudaEventRecord(ss.d2h[k], ss.out));
    }
    // the caller's stream covers every copy
    for (size_t i = n_batches >= 2 ? n_batches - 2 : 0; i < n_batches; ++i)
      FSVD_CUDA_CHECK(cudaStreamWaitEvent(sc, ss.d2h[i & 1], 0));
  });
}

// ---------------------------------------------------------------- host API
fsvd_status fsvd_flash_svd_attention(const float* x, size_t batch, size_t seq, size_t width,
                                     const fsvd_attn_desc* set, size_t heads,
                                     const fsvd_tile_plan* plan, fsvd_dtype dtype,
                                     fsvd_meter* meter, const char* pin_prefix, float* out,
                                     size_t ob, size_t om, size_t ow) {
  return guard([&] {
    if (!x || !set || !out) fail(Kind::Config, "null argument");
    host_attention(x, batch, seq, width, *set, heads, plan_or_default(plan), dtype,
                   meter ? &meter->m : nullptr, pin_prefix ? pin_prefix : "attn", out, ob, om, ow);
  });
}
fsvd_status fsvd_lowrank_output_projection(const float* ctx, size_t batch, size_t seq,
                                           size_t width, const fsvd_linear_desc* proj,
                                           fsvd_dtype dtype, fsvd_meter* meter,
                                           const char* pin_prefix, float* out, size_t ob,
                                           size_t om, size_t ow) {
  return guard([&] {
    if (!ctx || !proj || !out) fail(Kind::Config, "null argument");
    host_outproj(ctx, batch, seq, width, *proj, dtype, meter ? &meter->m : nullptr,
                 pin_prefix ? pin_prefix : "attn", out, ob, om, ow);
  });
}
fsvd_status fsvd_ffn(int variant, const float* x, size_t batch, size_t seq, size_t width,
                     const fsvd_ffn_desc* f, const fsvd_tile_plan* plan, fsvd_dtype dtype,
                     fsvd_meter* meter, const char* pin_prefix, float* out, size_t ob, size_t om,
                     size_t ow) {
  return guard([&] {
    if (!x || !f || !out) fail(Kind::Config, "null argument");
    host_ffn(variant, x, batch, seq, width, *f, plan_or_default(plan), dtype,
             meter ? &meter->m : nullptr, pin_prefix ? pin_prefix : "ffn", out, ob, om, ow);
  });
}
fsvd_status fsvd_run_layer(const float* x, size_t batch, size_t seq, size_t width,
                           const fsvd_layer_desc* layer, fsvd_run_mode mode,
                           const fsvd_tile_plan* plan, int pre_ln, const char* meter_prefix,
                           fsvd_dtype dtype, fsvd_meter* meter, float* out) {
  return guard([&] {
    if (!x || !layer || !out) fail(Kind::Config, "null argument");
    if (x == out) fail(Kind::Config, "run_layer: out must be a distinct tensor");
    host_run_model(x, batch, seq, width, layer, 1, mode, plan_or_default(plan), pre_ln != 0,
                   meter_prefix ? meter_prefix : "layer", dtype, meter ? &meter->m : nullptr, out,
                   true);
  });
}
fsvd_status fsvd_run_model(const float* x, size_t batch, size_t seq, size_t width,
                           const fsvd_layer_desc* layers, size_t n_layers, fsvd_run_mode mode,
                           const fsvd_tile_plan* plan, int pre_ln, const char* meter_prefix,
                           fsvd_dtype dtype, fsvd_meter* meter, float* out) {
  return guard([&] {
    if (!x || (!layers && n_layers) || !out) fail(Kind::Config, "null argument");
    const std::string pfx = meter_prefix ? meter_prefix : "layer";
    if (n_layers == 1)
      host_run_model(x, batch, seq, width, layers, 1, mode, plan_or_default(plan), pre_ln != 0,
                     pfx + ".0", dtype, meter ? &meter->m : nullptr, out, true);
    else
      host_run_model(x, batch, seq, width, layers, n_layers, mode, plan_or_default(plan),
                     pre_ln != 0, pfx, dtype, meter ? &meter->m : nullptr, out, false);
  });
}

uint64_t fsvd_kernel_launch_count(void) { return launch_count(); }

fsvd_status fsvd_test_gemm(const void* A, size_t lda, const void* B, size_t ldb, void* C,
                           size_t ldc, size_t M, size_t N, size_t K, const float* bias,
                           fsvd_activation act, int use_act, void* stream) {
  return guard([&] {
    require_device();
    if (!gemm_bf16_supported((int)M, (int)N, (int)K, lda, ldb, ldc))
      fail(Kind::Config, "gemm: unsupported shape");
    gemm_bf16(static_cast<const bf16*>(A), lda, static_cast<const bf16*>(B), ldb,
              static_cast<bf16*>(C), ldc, (int)M, (int)N, (int)K, bias,
              use_act ? static_cast<int>(act) : ACT_NONE, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_test_gemm_ln(const void* A, size_t lda, const void* B, size_t ldb,
                              const float* bias, const void* resid, const float* gamma,
                              const float* beta, float eps, void* y, size_t T, size_t N,
                              size_t K, void* stream) {
  return guard([&] {
    require_device();
    if (!gemm_ln_supported((int)N, (int)K)) fail(Kind::Config, "gemm_ln: unsupported shape");
    gemm_ln_bf16(static_cast<const bf16*>(A), lda, static_cast<const bf16*>(B), ldb, bias,
                 static_cast<const bf16*>(resid), gamma, beta, eps, static_cast<bf16*>(y), (int)T,
                 (int)N, (int)K, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_test_attention(const void* qkv, size_t cols, size_t q_off, size_t k_off,
                                size_t v_off, size_t batch, size_t seq, size_t heads,
                                size_t groups, size_t rank_pad, void* out, size_t ldo,
                                void* stream) {
  return guard([&] {
    require_device();
    if (!attn_rankspace_supported((int)rank_pad) || heads % groups != 0)
      fail(Kind::Config, "attention: unsupported shape");
    AttnTcArgs a;
    a.qkv = static_cast<const bf16*>(qkv);
    a.ldq = (int64_t)cols;
    a.qkv_cols = (int)cols;
    a.q_off = (int)q_off;
    a.k_off = (int)k_off;
    a.v_off = (int)v_off;
    a.batch = (int)batch;
    a.seq = (int)seq;
    a.heads = (int)heads;
    a.groups = (int)groups;
    a.rank_pad = (int)rank_pad;
    a.out = static_cast<bf16*>(out);
    a.ldo = (int64_t)ldo;
    attn_rankspace_bf16(a, static_cast<cudaStream_t>(stream));
  });
}
fsvd_status fsvd_test_resid_layernorm(const void* a, const void* b, const float* gamma,
                                      const float* beta, float eps, void* y, size_t rows,
                                      size_t d, void* stream) {
  return guard([&] {
    require_device();
    resid_layernorm_bf16(static_cast<const bf16*>(a), static_cast<const bf16*>(b), gamma, beta,
                         eps, static_cast<bf16*>(y), (int)rows, (int)d,
                         static_cast<cudaStream_t>(stream));
  });
}

const char* fsvd_kernel_name(int id) {
  switch (id) {
    case 0: return "k_gemm_bf16";
    case 1: return "k_attn_rankspace";
    case 2: return "k_ffn_stream";
    case 3: return "k_ffn_fused";
    case 4: return "k_resid_ln";
    default: return "";
  }
}

}  // extern "C"
