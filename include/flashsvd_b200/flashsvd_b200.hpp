// flashsvd_b200.hpp -- C++ drop-in for the reference's streaming operator API.
//
// Header-only.  Compiled against the reference's own headers
// (/root/reference/proj/include/flashsvd/*.hpp: Tensor, AttentionFactorSet,
// FactorizedLinear, FfnFactors, EncoderLayer, TilePlan, MemoryMeter) and
// linked with libfsvd_b200.so, it re-exposes the reference signatures in
// namespace flashsvd::b200:
//
//   flash_svd_attention        attention.hpp:18-21
//   lowrank_output_projection  attention.hpp:49-51
//   ffn_v1 / ffn_v2            ffn.hpp:33-34, 40-41
//   run_layer / run_model      encoder.hpp:83-85, 90-92
//
// Behaviour follows the reference contract: same shape/config/budget checks
// and exception types (errors.hpp), caller-owned tensors, synchronous return.
// The device work goes through the C-ABI host drop-ins (include/fsvd_b200.h),
// which charge a mirror meter exactly like the reference does; its event log
// (allocs, frees, pins, regions, 4 B/element) is replayed onto the caller's
// flashsvd::MemoryMeter, so peaks, pins and region balance read the same as
// after a reference call.
//
// Precision policy: fp32 storage + fp32 arithmetic (the <= 1e-4 parity mode)
// by default; set_precision(FSVD_BF16) selects the bf16 tensor-core kernels.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "flashsvd/attention.hpp"
#include "flashsvd/encoder.hpp"
#include "flashsvd/errors.hpp"
#include "flashsvd/factorize.hpp"
#include "flashsvd/ffn.hpp"
#include "flashsvd/memtier.hpp"
#include "flashsvd/tensor.hpp"
#include "fsvd_b200.h"

namespace flashsvd {
namespace b200 {

namespace detail {

inline fsvd_dtype& precision() {
  static thread_local fsvd_dtype p = FSVD_F32;
  return p;
}

// fsvd_status -> the reference's exception taxonomy (errors.hpp:11-68).
[[noreturn]] inline void raise(fsvd_status st, const std::string& msg) {
  switch (st) {
    case FSVD_ERR_SHAPE: throw ShapeError(msg);
    case FSVD_ERR_RANK: throw RankError(msg);
    case FSVD_ERR_CONFIG: throw ConfigError(msg);
    case FSVD_ERR_BUDGET: throw BudgetError(msg);
    case FSVD_ERR_ACCOUNTING: throw AccountingError(msg);
    case FSVD_ERR_FORMAT: throw FormatError(0, msg);
    case FSVD_ERR_NUMERIC: throw NumericError(msg);
    case FSVD_ERR_INFEASIBLE: throw InfeasibleError(msg);
    case FSVD_ERR_IO: throw IoError(msg);
    default: throw std::runtime_error("fsvd_b200 device error: " + msg);
  }
}
inline void check(fsvd_status st) {
  if (st != FSVD_OK) raise(st, fsvd_last_error());
}
// Status of a metered call: the message is captured before the meter replay
// (which makes successful C-ABI calls of its own) and raised after it.
struct Result {
  fsvd_status st;
  std::string msg;
  explicit Result(fsvd_status s) : st(s), msg(s == FSVD_OK ? "" : fsvd_last_error()) {}
  void raise_if_failed() const {
    if (st != FSVD_OK) raise(st, msg);
  }
};

// Mirror meter whose event log is replayed onto the caller's meter.
class MirrorMeter {
 public:
  MirrorMeter() { check(fsvd_meter_create(&m_)); }
  ~MirrorMeter() { fsvd_meter_destroy(m_); }
  MirrorMeter(const MirrorMeter&) = delete;
  MirrorMeter& operator=(const MirrorMeter&) = delete;
  fsvd_meter* get() { return m_; }

  // Replays every event in order: allocs/frees keep their pairing, pins are
  // idempotent by tag, region begin/end nest as RAII regions do.
  void replay(MemoryMeter& meter) {
    std::unordered_map<std::uint64_t, MeterHandle> handles;
    std::vector<std::unique_ptr<MeterRegion>> regions;
    const std::size_t n = fsvd_meter_event_count(m_);
    char tag[512];
    for (std::size_t i = 0; i < n; ++i) {
      int kind = 0, cls = 0;
      std::size_t bytes = 0;
      std::uint64_t id = 0;
      check(fsvd_meter_event(m_, i, &kind, &cls, &bytes, &id, tag, sizeof(tag)));
      switch (kind) {
        case FSVD_EV_ALLOC:
          handles[id] = meter.alloc(tag, static_cast<AllocClass>(cls), bytes);
          break;
        case FSVD_EV_FREE:
          meter.free(handles.at(id));
          handles.erase(id);
          break;
        case FSVD_EV_PIN: meter.pin_persistent(tag, bytes); break;
        case FSVD_EV_REGION_BEGIN:
          regions.push_back(std::make_unique<MeterRegion>(meter.scoped_region(tag)));
          break;
        case FSVD_EV_REGION_END:
          if (!regions.empty()) regions.pop_back();
          break;
        default: break;
      }
    }
  }

 private:
  fsvd_meter* m_ = nullptr;
};

// Contiguous fp32 packs of the reference containers (fsvd_b200.h layouts).
struct LinearPack {
  fsvd_linear_desc d{};
  explicit LinearPack(const FactorizedLinear& f) {
    d.in_dim = f.in_dim();
    d.rank = f.rank();
    d.out_dim = f.out_dim();
    d.u = f.u.data();
    d.v = f.v.data();
    d.bias = f.bias.data();
  }
};

struct AttnPack {
  std::vector<float> u, v, bias;
  fsvd_attn_desc d{};
  explicit AttnPack(const AttentionFactorSet& s) {
    const std::size_t G = s.groups, r = s.rank, dm = s.d_model, gd = G ? dm / G : 0;
    if (s.q.size() != G || s.k.size() != G || s.v.size() != G)
      throw ShapeError("attention factor set: expected one factor per group");
    u.reserve(3 * G * dm * r);
    v.reserve(3 * G * r * gd);
    bias.reserve(3 * dm);
    for (Qkv m : {Qkv::Q, Qkv::K, Qkv::V})
      for (const FactorizedLinear& f : s.matrix(m)) {
        if (f.u.numel() != dm * r || f.v.numel() != r * gd || f.bias.numel() != gd)
          throw ShapeError("attention factor: expected U (d, r), V (r, d/groups), bias (d/groups)");
        u.insert(u.end(), f.u.data(), f.u.data() + f.u.numel());
        v.insert(v.end(), f.v.data(), f.v.data() + f.v.numel());
        bias.insert(bias.end(), f.bias.data(), f.bias.data() + f.bias.numel());
      }
    d.d_model = dm;
    d.groups = G;
    d.rank = r;
    d.u = u.data();
    d.v = v.data();
    d.bias = bias.data();
  }
};

struct FfnPack {
  fsvd_ffn_desc d{};
  explicit FfnPack(const FfnFactors& f) {
    d.up = LinearPack(f.up).d;
    d.down = LinearPack(f.down).d;
    d.activation = static_cast<fsvd_activation>(static_cast<int>(f.activation));
  }
};

// One EncoderLayer: whichever of its representations it carries (encoder.hpp:
// 49-67) -- factorized attention + output projection, factorized FFN, dense
// weights -- after the reference's own EncoderLayer::validate().
struct LayerPack {
  std::unique_ptr<AttnPack> attn;
  fsvd_dense_layer dense{};
  fsvd_layer_desc d{};
  explicit LayerPack(const EncoderLayer& l) {
    l.validate();
    d.heads = l.heads;
    d.attn.d_model = l.d_model();
    if (l.attn_factors) {
      attn = std::make_unique<AttnPack>(*l.attn_factors);
      d.attn = attn->d;
      d.out_proj = LinearPack(*l.out_proj).d;
    }
    if (l.ffn_factors) d.ffn = FfnPack(*l.ffn_factors).d;
    if (l.attn_dense && l.ffn_dense) {
      const DenseAttentionWeights& a = *l.attn_dense;
      const DenseFfnWeights& f = *l.ffn_dense;
      dense = fsvd_dense_layer{l.d_model(), f.b_in.numel(), a.wq.data(), a.bq.data(),
                               a.wk.data(), a.bk.data(), a.wv.data(), a.bv.data(),
                               a.wo.data(), a.bo.data(), f.w_in.data(), f.b_in.data(),
                               f.w_out.data(), f.b_out.data()};
      d.dense = &dense;
      if (!l.ffn_factors) d.ffn.activation = static_cast<fsvd_activation>(static_cast<int>(f.activation));
    }
    d.ln1_gamma = l.ln1.gamma.data();
    d.ln1_beta = l.ln1.beta.data();
    d.ln1_eps = l.ln1.eps;
    d.ln2_gamma = l.ln2.gamma.data();
    d.ln2_beta = l.ln2.beta.data();
    d.ln2_eps = l.ln2.eps;
  }
};

// encoder.cpp:27-35 (check_mode_weights), same exception and message: the
// drop-in runs Dense mode only on a layer's own dense weights, like the
// reference (the C-ABI alone also offers the dense twin of a factor-only layer).
inline void check_mode_weights(const EncoderLayer& layer, RunMode mode) {
  if (mode == RunMode::Dense) {
    if (!layer.attn_dense || !layer.ffn_dense)
      throw ConfigError("dense mode needs dense weights on both sublayers");
  } else if (!layer.attn_factors || !layer.out_proj || !layer.ffn_factors) {
    throw ConfigError(std::string(mode_name(mode)) +
                      " mode needs factorized weights on both sublayers");
  }
}

inline fsvd_tile_plan plan_of(const TilePlan& p) {
  return fsvd_tile_plan{p.bm, p.br, p.bdf, p.sram_budget_bytes};
}

// Extents of a rank-3 tensor (zeros when the rank differs, so the C-ABI
// raises the reference's ShapeError).
struct Dims {
  std::size_t b = 0, m = 0, w = 0;
  explicit Dims(const Tensor& t) {
    if (t.ndim() == 3) {
      b = t.extent(0);
      m = t.extent(1);
      w = t.extent(2);
    }
  }
};

}  // namespace detail

// Selects the precision policy of subsequent calls on this thread.
inline void set_precision(fsvd_dtype dtype) { detail::precision() = dtype; }
inline fsvd_dtype precision() { return detail::precision(); }

// attention.hpp:18-21
inline void flash_svd_attention(const Tensor& x, const AttentionFactorSet& set, std::size_t heads,
                                const TilePlan& plan, MemoryMeter& meter,
                                const std::string& pin_prefix, Tensor& out) {
  detail::AttnPack pk(set);
  detail::MirrorMeter mm;
  const detail::Dims xi(x), oi(out);
  const fsvd_tile_plan tp = detail::plan_of(plan);
  const detail::Result st(fsvd_flash_svd_attention(
      x.data(), xi.b, xi.m, xi.w, &pk.d, heads, &tp, detail::precision(), mm.get(),
      pin_prefix.c_str(), out.data(), oi.b, oi.m, oi.w));
  mm.replay(meter);
  st.raise_if_failed();
}

// attention.hpp:49-51
inline void lowrank_output_projection(const Tensor& ctx, const FactorizedLinear& proj,
                                      MemoryMeter& meter, const std::string& pin_prefix,
                                      Tensor& out) {
  const detail::LinearPack pk(proj);
  detail::MirrorMeter mm;
  const detail::Dims xi(ctx), oi(out);
  const detail::Result st(fsvd_lowrank_output_projection(
      ctx.data(), xi.b, xi.m, xi.w, &pk.d, detail::precision(), mm.get(), pin_prefix.c_str(),
      out.data(), oi.b, oi.m, oi.w));
  mm.replay(meter);
  st.raise_if_failed();
}

namespace detail {
inline void ffn(int variant, const Tensor& x, const FfnFactors& f, const TilePlan& plan,
                MemoryMeter& meter, const std::string& pin_prefix, Tensor& out) {
  const FfnPack pk(f);
  MirrorMeter mm;
  const Dims xi(x), oi(out);
  const fsvd_tile_plan tp = plan_of(plan);
  const Result st(fsvd_ffn(variant, x.data(), xi.b, xi.m, xi.w, &pk.d, &tp, precision(),
                                  mm.get(), pin_prefix.c_str(), out.data(), oi.b, oi.m, oi.w));
  mm.replay(meter);
  st.raise_if_failed();
}
}  // namespace detail

// ffn.hpp:33-34
inline void ffn_v1(const Tensor& x, const FfnFactors& f, const TilePlan& plan,
                   MemoryMeter& meter, const std::string& pin_prefix, Tensor& out) {
  detail::ffn(1, x, f, plan, meter, pin_prefix, out);
}
// ffn.hpp:40-41
inline void ffn_v2(const Tensor& x, const FfnFactors& f, const TilePlan& plan,
                   MemoryMeter& meter, const std::string& pin_prefix, Tensor& out) {
  detail::ffn(2, x, f, plan, meter, pin_prefix, out);
}

// encoder.hpp:90-92
inline void run_model(const Tensor& x, const std::vector<EncoderLayer>& layers, RunMode mode,
                      const TilePlan& plan, MemoryMeter& meter, Tensor& out,
                      const LayerRunOptions& opts = {}) {
  if (x.ndim() != 3) throw ShapeError("run_model: x must be (batch, seq, d_model)");
  if (static_cast<const void*>(&out) == static_cast<const void*>(&x))
    throw ConfigError("run_model: out must be a distinct tensor");
  if (!out.same_shape(x)) throw ShapeError("run_model: out shape must match x");
  if (layers.empty()) {
    std::copy(x.data(), x.data() + x.numel(), out.data());
    return;
  }
  std::vector<detail::LayerPack> packs;
  packs.reserve(layers.size());
  for (const EncoderLayer& l : layers) {
    packs.emplace_back(l);
    detail::check_mode_weights(l, mode);
  }
  std::vector<fsvd_layer_desc> descs;
  for (const auto& p : packs) descs.push_back(p.d);
  detail::MirrorMeter mm;
  const detail::Dims xi(x);
  const fsvd_tile_plan tp = detail::plan_of(plan);
  const detail::Result st(fsvd_run_model(
      x.data(), xi.b, xi.m, xi.w, descs.data(), descs.size(),
      static_cast<fsvd_run_mode>(static_cast<int>(mode)), &tp, opts.pre_layer_norm ? 1 : 0,
      opts.meter_prefix.c_str(), detail::precision(), mm.get(), out.data()));
  mm.replay(meter);
  st.raise_if_failed();
}

// encoder.hpp:83-85
inline void run_layer(const Tensor& x, const EncoderLayer& layer, RunMode mode,
                      const TilePlan& plan, MemoryMeter& meter, Tensor& out,
                      const LayerRunOptions& opts = {}) {
  detail::LayerPack pk(layer);
  detail::check_mode_weights(layer, mode);
  if (x.ndim() != 3 || x.shape()[2] != layer.d_model())
    throw ShapeError("run_layer: x must be (batch, seq, d_model)");
  if (static_cast<const void*>(&out) == static_cast<const void*>(&x))
    throw ConfigError("run_layer: out must be a distinct tensor");
  if (!out.same_shape(x)) throw ShapeError("run_layer: out shape must match x");
  detail::MirrorMeter mm;
  const detail::Dims xi(x);
  const fsvd_tile_plan tp = detail::plan_of(plan);
  const detail::Result st(fsvd_run_layer(
      x.data(), xi.b, xi.m, xi.w, &pk.d, static_cast<fsvd_run_mode>(static_cast<int>(mode)), &tp,
      opts.pre_layer_norm ? 1 : 0, opts.meter_prefix.c_str(), detail::precision(), mm.get(),
      out.data()));
  mm.replay(meter);
  st.raise_if_failed();
}

// ------------------------------------------------------------ factorization
// svd.cpp:412-456: leading-r even-split factors on the device (fp64 Jacobi).
inline LowRankPair factor_rank_r(const Tensor& a, std::size_t r) {
  if (a.ndim() != 2) throw ShapeError("factorization input must be 2-D");
  const std::size_t m = a.shape()[0], n = a.shape()[1];
  LowRankPair out{Tensor({m, r == 0 ? 1 : r}), Tensor({r == 0 ? 1 : r, n})};
  detail::check(fsvd_factor_rank_r(a.data(), m, n, r, out.u.data(), out.v.data()));
  return out;
}

// factorize.cpp:10-17
inline FactorizedLinear factorize_linear(const Tensor& w, const Tensor& bias, std::size_t rank) {
  if (w.shape().size() != 2) throw ShapeError("factorize_linear expects a matrix");
  if (bias.shape().size() != 1 || bias.shape()[0] != w.shape()[1])
    throw ShapeError("bias length must match the output dimension");
  LowRankPair pair = b200::factor_rank_r(w, rank);
  return FactorizedLinear{std::move(pair.u), std::move(pair.v), bias};
}

// ffn.cpp:108-116 -- both matrices in one device run
inline FfnFactors factorize_ffn(const Tensor& w_in, const Tensor& b_in, const Tensor& w_out,
                                const Tensor& b_out, std::size_t rank, Activation act) {
  for (const Tensor* w : {&w_in, &w_out})
    if (w->shape().size() != 2) throw ShapeError("factorize_linear expects a matrix");
  if (b_in.shape().size() != 1 || b_in.shape()[0] != w_in.shape()[1] ||
      b_out.shape().size() != 1 || b_out.shape()[0] != w_out.shape()[1])
    throw ShapeError("bias length must match the output dimension");
  FfnFactors f;
  f.up = FactorizedLinear{Tensor({w_in.shape()[0], rank ? rank : 1}),
                          Tensor({rank ? rank : 1, w_in.shape()[1]}), b_in};
  f.down = FactorizedLinear{Tensor({w_out.shape()[0], rank ? rank : 1}),
                            Tensor({rank ? rank : 1, w_out.shape()[1]}), b_out};
  fsvd_factor_job jobs[2] = {
      {w_in.data(), w_in.shape()[0], w_in.shape()[1], rank, f.up.u.data(), f.up.v.data()},
      {w_out.data(), w_out.shape()[0], w_out.shape()[1], rank, f.down.u.data(), f.down.v.data()}};
  detail::check(fsvd_factor_rank_r_batch(jobs, 2));
  f.activation = act;
  return f;
}

// factorize.cpp:21-64 -- all 3*groups blocks in one device run
inline AttentionFactorSet factorize_attention(const Tensor& wq, const Tensor& bq, const Tensor& wk,
                                              const Tensor& bk, const Tensor& wv, const Tensor& bv,
                                              std::size_t groups, std::size_t rank) {
  const Tensor* weights[3] = {&wq, &wk, &wv};
  const Tensor* biases[3] = {&bq, &bk, &bv};
  const std::size_t d = wq.shape().size() == 2 ? wq.shape()[0] : 0;
  for (int i = 0; i < 3; ++i) {
    const Tensor& w = *weights[i];
    if (w.shape().size() != 2 || w.shape()[0] != d || w.shape()[1] != d)
      throw ShapeError("attention projections must be square d_model x d_model");
    if (biases[i]->shape().size() != 1 || biases[i]->shape()[0] != d)
      throw ShapeError("attention bias length must be d_model");
  }
  const std::size_t gd = groups && d % groups == 0 ? d / groups : 1, rr = rank ? rank : 1;
  std::vector<float> u(3 * std::max<std::size_t>(groups, 1) * d * rr),
      v(3 * std::max<std::size_t>(groups, 1) * rr * gd), b(3 * d);
  detail::check(fsvd_factorize_attention(wq.data(), bq.data(), wk.data(), bk.data(), wv.data(),
                                         bv.data(), d, groups, rank, u.data(), v.data(),
                                         b.data()));
  AttentionFactorSet set;
  set.d_model = d;
  set.groups = groups;
  set.rank = rank;
  std::vector<FactorizedLinear>* out[3] = {&set.q, &set.k, &set.v};
  for (std::size_t m = 0; m < 3; ++m)
    for (std::size_t g = 0; g < groups; ++g) {
      const std::size_t i = m * groups + g;
      FactorizedLinear f{Tensor({d, rank}), Tensor({rank, gd}), Tensor({gd})};
      std::copy(u.begin() + i * d * rank, u.begin() + (i + 1) * d * rank, f.u.data());
      std::copy(v.begin() + i * rank * gd, v.begin() + (i + 1) * rank * gd, f.v.data());
      std::copy(b.begin() + i * gd, b.begin() + (i + 1) * gd, f.bias.data());
      out[m]->push_back(std::move(f));
    }
  return set;
}

}  // namespace b200
}  // namespace flashsvd
