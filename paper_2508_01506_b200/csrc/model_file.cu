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

// EncoderLayer::validate()'s shape checks (encoder.cpp:14-25), same messages.
void check_vec(const Record& t, size_t n, const char* what) {
  if (t.shape.size() != 1 || t.numel() != n)
    fail(Kind::Shape, std::string(what) + ": expected a length-" + std::to_string(n) + " vector");
}

void check_mat(const Record& t, size_t rows, size_t cols, const char* what) {
  if (t.shape.size() != 2 || t.shape[0] != rows || t.shape[1] != cols)
    fail(Kind::Shape, std::string(what) + ": expected shape (" + std::to_string(rows) + ", " +
                          std::to_string(cols) + ")");
}

size_t mat_cols(const Record& t) { return t.shape.size() == 2 ? t.shape[1] : 0; }

fsvd_linear_desc linear(Record& u, Record& v, Record& b) {
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
    // model_io.cpp:288-337 (assemble): the same lookups in the same order ...
    d.heads = a.count(p + "heads", "heads");
    Record& g1 = a.get(p + "ln1.gamma");
    Record& b1 = a.get(p + "ln1.beta");
    d.ln1_eps = a.scalar(p + "ln1.eps");
    Record& g2 = a.get(p + "ln2.gamma");
    Record& b2 = a.get(p + "ln2.beta");
    d.ln2_eps = a.scalar(p + "ln2.eps");
    const float act = a.scalar(p + "ffn.act");
    if (!(act == 0.0f || act == 1.0f || act == 2.0f || act == 3.0f))
      fail(Kind::Config, "bad activation code in model file");
    const bool attn_dense = a.has(p + "attn.q.W");
    if (attn_dense)
      for (const char* n : {"attn.q.W", "attn.q.b", "attn.k.W", "attn.k.b", "attn.v.W",
                            "attn.v.b", "attn.out.W", "attn.out.b"})
        a.get(p + n);
    const bool attn_fact = a.has(p + "attn.q.head.0.U");
    size_t G = 0;
    std::vector<Record*> qkv[3];
    const char* names[3] = {"q", "k", "v"};
    Record *ou = nullptr, *ov = nullptr, *ob = nullptr;
    size_t r = 0;
    if (attn_fact) {
      while (a.has(p + "attn.q.head." + std::to_string(G) + ".U")) ++G;
      for (int m = 0; m < 3; ++m)
        for (size_t g = 0; g < G; ++g) {
          const std::string gp = p + "attn." + names[m] + ".head." + std::to_string(g) + ".";
          qkv[m].push_back(&a.get(gp + "U"));
          qkv[m].push_back(&a.get(gp + "V"));
          qkv[m].push_back(&a.get(gp + "b"));
        }
      if (qkv[0][0]->shape.size() != 2) fail(Kind::Shape, "attention factor U must be a matrix");
      r = qkv[0][0]->shape[1];
      ou = &a.get(p + "attn.out.U");
      ov = &a.get(p + "attn.out.V");
      ob = &a.get(p + "attn.out.bias");
    }
    const bool ffn_dense = a.has(p + "ffn.in.W");
    if (ffn_dense)
      for (const char* n : {"ffn.in.W", "ffn.in.b", "ffn.out.W", "ffn.out.b"}) a.get(p + n);
    const bool ffn_fact = a.has(p + "ffn.up.U");
    Record *uu = nullptr, *uv = nullptr, *ub = nullptr, *du = nullptr, *dv = nullptr,
           *db = nullptr;
    if (ffn_fact) {
      uu = &a.get(p + "ffn.up.U");
      uv = &a.get(p + "ffn.up.V");
      ub = &a.get(p + "ffn.up.b");
      du = &a.get(p + "ffn.down.U");
      dv = &a.get(p + "ffn.down.V");
      db = &a.get(p + "ffn.down.b");
    }
    // ... then EncoderLayer::validate() (encoder.cpp:156-215), check by check.
    const size_t dm = g1.numel();  // d_model() = ln1.gamma.numel()
    if (dm == 0) fail(Kind::Shape, "layer norm parameters are empty");
    check_vec(g1, dm, "ln1.gamma");
    check_vec(b1, dm, "ln1.beta");
    check_vec(g2, dm, "ln2.gamma");
    check_vec(b2, dm, "ln2.beta");
    if (d.heads == 0 || dm % d.heads != 0) fail(Kind::Config, "heads must divide d_model");
    if (!attn_dense && !attn_fact) fail(Kind::Config, "layer has no attention weights");
    if (!ffn_dense && !ffn_fact) fail(Kind::Config, "layer has no FFN weights");
    if (attn_fact) {
      if (qkv[0][0]->shape[0] != dm) fail(Kind::Shape, "attention factors d_model mismatch");
      if (G == 0 || dm % G != 0) fail(Kind::Config, "groups must divide d_model");
      if (d.heads % G != 0) fail(Kind::Config, "groups must divide heads");
      const size_t gd = dm / G;
      for (size_t g = 0; g < G; ++g)
        for (int m = 0; m < 3; ++m) {
          check_mat(*qkv[m][3 * g], dm, r, "attention factor U");
          check_mat(*qkv[m][3 * g + 1], r, gd, "attention factor V");
          check_vec(*qkv[m][3 * g + 2], gd, "attention factor bias");
        }
      const size_t pr = mat_cols(*ou);
      check_mat(*ou, dm, pr, "out_proj U");
      check_mat(*ov, pr, dm, "out_proj V");
      check_vec(*ob, dm, "out_proj bias");
    }
    if (attn_dense) {
      for (const char* n : {"attn.q.W", "attn.k.W", "attn.v.W", "attn.out.W"})
        check_mat(a.get(p + n), dm, dm, "attention weight");
      for (const char* n : {"attn.q.b", "attn.k.b", "attn.v.b", "attn.out.b"})
        check_vec(a.get(p + n), dm, "attention bias");
    }
    // d_ff(): the factor's out_dim, else the dense input bias length
    const size_t df = ffn_fact ? mat_cols(*uv) : a.get(p + "ffn.in.b").numel();
    if (ffn_fact) {
      const size_t fr = mat_cols(*uu);
      if (fr != mat_cols(*du)) fail(Kind::Config, "FFN up/down factor ranks differ");
      check_mat(*uu, dm, fr, "ffn up U");
      check_mat(*uv, fr, df, "ffn up V");
      check_vec(*ub, df, "ffn up bias");
      check_mat(*du, df, fr, "ffn down U");
      check_mat(*dv, fr, dm, "ffn down V");
      check_vec(*db, dm, "ffn down bias");
    }
    if (ffn_dense) {
      check_mat(a.get(p + "ffn.in.W"), dm, df, "ffn input weight");
      check_vec(a.get(p + "ffn.in.b"), df, "ffn input bias");
      check_mat(a.get(p + "ffn.out.W"), df, dm, "ffn output weight");
      check_vec(a.get(p + "ffn.out.b"), dm, "ffn output bias");
    }
    if (!attn_fact || !ffn_fact)
      fail(Kind::Config, "layer " + std::to_string(i) +
                             " has no factorized attention / FFN; the device path runs "
                             "factorized layers");
    d.ln1_gamma = g1.data.data();
    d.ln1_beta = b1.data.data();
    d.ln2_gamma = g2.data.data();
    d.ln2_beta = b2.data.data();
    for (int m = 0; m < 3; ++m)
      for (size_t g = 0; g < G; ++g) {
        // fsvd_attn_desc layout: u [3, G, d, r], v [3, G, r, d/G], bias [3, d]
        L.attn_u.insert(L.attn_u.end(), qkv[m][3 * g]->data.begin(), qkv[m][3 * g]->data.end());
        L.attn_v.insert(L.attn_v.end(), qkv[m][3 * g + 1]->data.begin(),
                        qkv[m][3 * g + 1]->data.end());
        L.attn_b.insert(L.attn_b.end(), qkv[m][3 * g + 2]->data.begin(),
                        qkv[m][3 * g + 2]->data.end());
      }
    d.attn.d_model = dm;
    d.attn.groups = G;
    d.attn.rank = r;
    d.attn.u = L.attn_u.data();
    d.attn.v = L.attn_v.data();
    d.attn.bias = L.attn_b.data();
    d.out_proj = linear(*ou, *ov, *ob);
    d.ffn.up = linear(*uu, *uv, *ub);
    d.ffn.down = linear(*du, *dv, *db);
    d.ffn.activation = static_cast<fsvd_activation>(static_cast<int>(act));
    validate_layer(d);
  }
  mf->keep = std::make_shared<Assembler>(std::move(a));
  return mf;
}

ModelFile::~ModelFile() = default;

}  // namespace fsvd
