// model_file.cu -- FSVD1 model container -> factorized layer descriptors.
//
// lets compressed checkpoints written by the
// reference (save_model, model_io.hpp:14-30 / model_io.cpp) run on the
// device path.  Host-only code.
//
// Container (little-endian, unpadded): "FSVD", u32 version = 1, u32 count,
// then per tensor u16 name length, name bytes, u8 dtype (0 = f32), u8 ndim
// (1..8), u64 extents, f32 payload.  Malformed input raises a Format error
// whose byte offset follows the reference reader's contract
// (model_io.cpp:66-151): the first unreadable byte, or the file size when a
// field runs past the end, or the end of the last record for trailing bytes.
//
// Assembly follows the canonical tensor names of the reference writer:
//   layer.<i>.heads | ln{1,2}.{gamma,beta,eps} | ffn.act
//   layer.<i>.attn.{q,k,v}.head.<g>.{U,V,b} | attn.out.{U,V,bias}
//   layer.<i>.ffn.{up,down}.{U,V,b}
// Dense-only layers (attn.q.W ...) are rejected: the device path runs
// factorized layers (the dense twin is rebuilt from the factors on request).
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "model_file.hpp"

namespace fsvd {

size_t& format_error_offset() {
  static thread_local size_t off = 0;
  return off;
}

namespace {

[[noreturn]] void format_fail(size_t at, const std::string& what) {
  format_error_offset() = at;
  fail(Kind::Format, what + " (at byte " + std::to_string(at) + ")");
}

constexpr size_t kMaxNdim = 8;

class Reader {
 public:
  Reader(const std::vector<uint8_t>& b) : b_(b) {}
  size_t off() const { return off_; }
  void skip(size_t n) { off_ += n; }
  void need(size_t n, const char* what) {
    if (b_.size() - off_ < n) format_fail(b_.size(), std::string("file truncated in ") + what);
  }
  uint64_t uint(int bytes, const char* what) {
    need(static_cast<size_t>(bytes), what);
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(b_[off_ + i]) << (8 * i);
    off_ += static_cast<size_t>(bytes);
    return v;
  }
  uint8_t byte_at() const { return b_[off_]; }
  const uint8_t* ptr() const { return b_.data() + off_; }

 private:
  const std::vector<uint8_t>& b_;
  size_t off_ = 0;
};

struct Record {
  std::vector<size_t> shape;
  std::vector<float> data;
  size_t numel() const { return data.size(); }
};

std::map<std::string, Record> parse(const std::vector<uint8_t>& bytes) {
  Reader r(bytes);
  r.need(4, "magic");
  if (std::memcmp(bytes.data(), "FSVD", 4) != 0) format_fail(0, "bad magic, not an FSVD file");
  r.skip(4);
  const size_t version_at = r.off();
  if (r.uint(4, "version") != 1) format_fail(version_at, "unsupported container version");
  const uint64_t count = r.uint(4, "tensor count");
  std::map<std::string, Record> out;
  std::vector<std::string> order;
  for (uint64_t t = 0; t < count; ++t) {
    const size_t name_len = static_cast<size_t>(r.uint(2, "name length"));
    r.need(name_len, "name");
    std::string name(reinterpret_cast<const char*>(r.ptr()), name_len);
    r.skip(name_len);
    r.need(1, "dtype");
    if (r.byte_at() != 0) format_fail(r.off(), "unsupported dtype for tensor " + name);
    r.skip(1);
    r.need(1, "tensor rank");
    const size_t ndim = r.byte_at();
    if (ndim == 0 || ndim > kMaxNdim) format_fail(r.off(), "bad tensor rank for " + name);
    r.skip(1);
    Record rec;
    size_t numel = 1;
    for (size_t i = 0; i < ndim; ++i) {
      const size_t at = r.off();
      const uint64_t e = r.uint(8, "extent");
      if (e == 0) format_fail(at, "zero extent in " + name);
      if (e > (SIZE_MAX / sizeof(float)) / numel) format_fail(at, "extent overflow in " + name);
      rec.shape.push_back(static_cast<size_t>(e));
      numel *= static_cast<size_t>(e);
    }
    r.need(sizeof(float) * numel, "tensor payload");
    rec.data.resize(numel);
    std::memcpy(rec.data.data(), r.ptr(), sizeof(float) * numel);
    r.skip(sizeof(float) * numel);
    // duplicates are a model (assembly) error in the reference, not a format one
    if (!out.emplace(name, std::move(rec)).second) order.push_back(name);
  }
  if (r.off() != bytes.size()) format_fail(r.off(), "trailing bytes after the last tensor");
  if (!order.empty()) fail(Kind::Config, "duplicate tensor name: " + order.front());
  return out;
}

size_t layer_index(const std::string& name) {
  if (name.rfind("layer.", 0) != 0) return SIZE_MAX;
  const size_t dot = name.find('.', 6);
  if (dot == std::string::npos || dot == 6) return SIZE_MAX;
  const std::string digits = name.substr(6, dot - 6);
  if (digits.find_first_not_of("0123456789") != std::string::npos) return SIZE_MAX;
  return static_cast<size_t>(std::stoul(digits));
}

class Assembler {
 public:
  explicit Assembler(std::map<std::string, Record>&& m) : m_(std::move(m)) {}
  bool has(const std::string& n) const { return m_.count(n) != 0; }
  Record& get(const std::string& n) {
    auto it = m_.find(n);
    if (it == m_.end()) fail(Kind::Config, "model file is missing tensor: " + n);
    return it->second;
  }
  float scalar(const std::string& n) {
    Record& t = get(n);
    if (t.numel() != 1) fail(Kind::Shape, n + " must hold a single value");
    return t.data[0];
  }
  size_t count(const std::string& n, const char* what) {
    const float v = scalar(n);
    if (!(v >= 1.0f) || v != static_cast<float>(static_cast<size_t>(v)))
      fail(Kind::Config, std::string(what) + " must be a positive integer");
    return static_cast<size_t>(v);
  }

 private:
  std::map<std::string, Record> m_;
};

fsvd_linear_desc linear(Record& u, Record& v, Record& b) {
  if (u.shape.size() != 2 || v.shape.size() != 2)
    fail(Kind::Shape, "factor halves must be matrices");
  fsvd_linear_desc d{};
  d.in_dim = u.shape[0];
  d.rank = u.shape[1];
  d.out_dim = v.shape[1];
  d.u = u.data.data();
  d.v = v.data.data();
  d.bias = b.data.data();
  return d;
}

}  // namespace

std::unique_ptr<ModelFile> read_model_file(const std::string& path) {
  format_error_offset() = 0;
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(Kind::Io, "cannot open model file: " + path);
  std::vector<uint8_t> bytes;
  uint8_t buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) bytes.insert(bytes.end(), buf, buf + n);
  const bool err = std::ferror(f) != 0;
  std::fclose(f);
  if (err) fail(Kind::Io, "cannot read model file: " + path);

  std::map<std::string, Record> recs = parse(bytes);
  size_t layers = 0;
  for (const auto& kv : recs) {
    const size_t i = layer_index(kv.first);
    if (i == SIZE_MAX) fail(Kind::Config, "unrecognized tensor name: " + kv.first);
    layers = std::max(layers, i + 1);
  }
  auto mf = std::make_unique<ModelFile>();
  Assembler a(std::move(recs));
  mf->layers.resize(layers);
  for (size_t i = 0; i < layers; ++i) {
    const std::string p = "layer." + std::to_string(i) + ".";
    ModelFile::Layer& L = mf->layers[i];
    fsvd_layer_desc& d = L.desc;
    d = fsvd_layer_desc{};
    d.heads = a.count(p + "heads", "heads");
    d.ln1_gamma = a.get(p + "ln1.gamma").data.data();
    d.ln1_beta = a.get(p + "ln1.beta").data.data();
    d.ln1_eps = a.scalar(p + "ln1.eps");
    d.ln2_gamma = a.get(p + "ln2.gamma").data.data();
    d.ln2_beta = a.get(p + "ln2.beta").data.data();
    d.ln2_eps = a.scalar(p + "ln2.eps");
    const float act = a.scalar(p + "ffn.act");
    if (!(act == 0.0f || act == 1.0f || act == 2.0f || act == 3.0f))
      fail(Kind::Config, "bad activation code in model file");
    if (!a.has(p + "attn.q.head.0.U") || !a.has(p + "ffn.up.U"))
      fail(Kind::Config, "layer " + std::to_string(i) +
                             " has no factorized attention / FFN; the device path runs "
                             "factorized layers");
    size_t G = 0;
    while (a.has(p + "attn.q.head." + std::to_string(G) + ".U")) ++G;
    Record& q0 = a.get(p + "attn.q.head.0.U");
    if (q0.shape.size() != 2) fail(Kind::Shape, "attention factor U must be a matrix");
    const size_t dm = q0.shape[0], r = q0.shape[1];
    const char* names[3] = {"q", "k", "v"};
    for (int m = 0; m < 3; ++m)
      for (size_t g = 0; g < G; ++g) {
        const std::string gp = p + "attn." + names[m] + ".head." + std::to_string(g) + ".";
        Record& u = a.get(gp + "U");
        Record& v = a.get(gp + "V");
        Record& b = a.get(gp + "b");
        if (u.shape.size() != 2 || u.shape[0] != dm || u.shape[1] != r)
          fail(Kind::Shape, gp + "U: expected shape (d, r)");
        if (v.shape.size() != 2 || v.shape[0] != r || v.shape[1] * G != dm)
          fail(Kind::Shape, gp + "V: expected shape (r, d/groups)");
        if (b.numel() * G != dm) fail(Kind::Shape, gp + "b: expected d/groups values");
        L.attn_u.insert(L.attn_u.end(), u.data.begin(), u.data.end());
        L.attn_v.insert(L.attn_v.end(), v.data.begin(), v.data.end());
        L.attn_b.insert(L.attn_b.end(), b.data.begin(), b.data.end());
      }
    d.attn.d_model = dm;
    d.attn.groups = G;
    d.attn.rank = r;
    d.attn.u = L.attn_u.data();
    d.attn.v = L.attn_v.data();
    d.attn.bias = L.attn_b.data();
    d.out_proj = linear(a.get(p + "attn.out.U"), a.get(p + "attn.out.V"),
                        a.get(p + "attn.out.bias"));
    d.ffn.up = linear(a.get(p + "ffn.up.U"), a.get(p + "ffn.up.V"), a.get(p + "ffn.up.b"));
    d.ffn.down =
        linear(a.get(p + "ffn.down.U"), a.get(p + "ffn.down.V"), a.get(p + "ffn.down.b"));
    d.ffn.activation = static_cast<fsvd_activation>(static_cast<int>(act));
    if (a.get(p + "ln1.gamma").numel() != dm || a.get(p + "ln2.gamma").numel() != dm)
      fail(Kind::Shape, "layer norm parameters must have d_model values");
    validate_layer(d);
  }
  mf->keep = std::make_shared<Assembler>(std::move(a));
  return mf;
}

ModelFile::~ModelFile() = default;

}  // namespace fsvd
