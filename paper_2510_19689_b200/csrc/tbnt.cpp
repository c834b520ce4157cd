// tbnt.cpp — native reader of the reference's .tbnt model stream and the
// cold-start path (stream -> verified params -> packed device weights).
//
// Stream layout (the weight-layout contract of reference model/io.py:43-57):
//   "TBNT" | u16 LE version (1) | 3 x [u32 LE length | payload] | u32 LE CRC-32C
//   payload 0: metadata JSON {model_version, config{...}, param_order[...],
//              param_shapes{name: [dims]}};  payload 1: f64 LE mean || var;
//   payload 2: f64 LE parameters concatenated in param_order.
// Validation order and error classes follow load_model (io.py:60-112):
// short stream / missing section -> TRUNCATED, bad magic / trailing bytes /
// bad metadata / size mismatches -> FORMAT, other version -> FORMAT_VERSION,
// CRC mismatch -> CHECKSUM, ModelConfig / TabNetModel invariants -> CONFIG.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tabnet_b200.h"
#include "tbn_internal.h"

namespace {

tbn_status err(tbn_status st, const std::string& msg) {
  tbn::set_last_error(msg);
  return st;
}

// ---- a small JSON reader (RFC 8259 values; enough for json.dumps output) ----
struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  double num = 0.0;
  bool integral = false;      // the token had no fraction / exponent
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JParser {
 public:
  JParser(const char* s, size_t n) : p_(s), e_(s + n) {}
  bool parse(JVal* out) {
    ws();
    if (!value(out, 0)) return false;
    ws();
    return p_ == e_;
  }

 private:
  const char* p_;
  const char* e_;
  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if ((size_t)(e_ - p_) < n || std::memcmp(p_, w, n) != 0) return false;
    p_ += n;
    return true;
  }
  static void utf8(std::string* s, uint32_t cp) {
    if (cp < 0x80) {
      s->push_back((char)cp);
    } else if (cp < 0x800) {
      s->push_back((char)(0xC0 | (cp >> 6)));
      s->push_back((char)(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      s->push_back((char)(0xE0 | (cp >> 12)));
      s->push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
      s->push_back((char)(0x80 | (cp & 0x3F)));
    } else {
      s->push_back((char)(0xF0 | (cp >> 18)));
      s->push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
      s->push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
      s->push_back((char)(0x80 | (cp & 0x3F)));
    }
  }
  bool hex4(uint32_t* v) {
    if (e_ - p_ < 4) return false;
    *v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p_++;
      *v <<= 4;
      if (c >= '0' && c <= '9') *v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') *v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') *v |= (uint32_t)(c - 'A' + 10);
      else return false;
    }
    return true;
  }
  bool string(std::string* s) {
    if (p_ >= e_ || *p_ != '"') return false;
    ++p_;
    while (p_ < e_ && *p_ != '"') {
      const unsigned char c = (unsigned char)*p_++;
      if (c < 0x20) return false;
      if (c != '\\') {
        s->push_back((char)c);
        continue;
      }
      if (p_ >= e_) return false;
      const char esc = *p_++;
      switch (esc) {
        case '"': s->push_back('"'); break;
        case '\\': s->push_back('\\'); break;
        case '/': s->push_back('/'); break;
        case 'b': s->push_back('\b'); break;
        case 'f': s->push_back('\f'); break;
        case 'n': s->push_back('\n'); break;
        case 'r': s->push_back('\r'); break;
        case 't': s->push_back('\t'); break;
        case 'u': {
          uint32_t cp;
          if (!hex4(&cp)) return false;
          if (cp >= 0xD800 && cp < 0xDC00 && e_ - p_ >= 6 && p_[0] == '\\' && p_[1] == 'u') {
            const char* save = p_;
            p_ += 2;
            uint32_t lo;
            if (hex4(&lo) && lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else p_ = save;
          }
          utf8(s, cp);
          break;
        }
        default: return false;
      }
    }
    if (p_ >= e_) return false;
    ++p_;
    return true;
  }
  bool number(JVal* v) {
    const char* s = p_;
    if (p_ < e_ && *p_ == '-') ++p_;
    if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) return false;
    while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    bool integral = true;
    if (p_ < e_ && *p_ == '.') {
      integral = false;
      ++p_;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
      integral = false;
      ++p_;
      if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    v->kind = JVal::NUM;
    v->integral = integral;
    v->num = std::strtod(std::string(s, p_).c_str(), nullptr);
    return true;
  }
  bool value(JVal* v, int depth) {
    if (depth > 64 || p_ >= e_) return false;
    ws();
    if (p_ >= e_) return false;
    const char c = *p_;
    if (c == '{') {
      ++p_;
      v->kind = JVal::OBJ;
      ws();
      if (p_ < e_ && *p_ == '}') { ++p_; return true; }
      for (;;) {
        ws();
        std::string k;
        if (!string(&k)) return false;
        ws();
        if (p_ >= e_ || *p_ != ':') return false;
        ++p_;
        JVal item;
        if (!value(&item, depth + 1)) return false;
        // duplicate keys: the last one wins, as in Python's json
        bool replaced = false;
        for (auto& kv : v->obj)
          if (kv.first == k) { kv.second = std::move(item); replaced = true; break; }
        if (!replaced) v->obj.emplace_back(std::move(k), std::move(item));
        ws();
        if (p_ < e_ && *p_ == ',') { ++p_; continue; }
        if (p_ < e_ && *p_ == '}') { ++p_; return true; }
        return false;
      }
    }
    if (c == '[') {
      ++p_;
      v->kind = JVal::ARR;
      ws();
      if (p_ < e_ && *p_ == ']') { ++p_; return true; }
      for (;;) {
        JVal item;
        if (!value(&item, depth + 1)) return false;
        v->arr.push_back(std::move(item));
        ws();
        if (p_ < e_ && *p_ == ',') { ++p_; continue; }
        if (p_ < e_ && *p_ == ']') { ++p_; return true; }
        return false;
      }
    }
    if (c == '"') {
      v->kind = JVal::STR;
      return string(&v->str);
    }
    if (lit("true")) { v->kind = JVal::BOOL; v->b = true; return true; }
    if (lit("false")) { v->kind = JVal::BOOL; v->b = false; return true; }
    if (lit("null")) { v->kind = JVal::NUL; return true; }
    if (lit("NaN")) { v->kind = JVal::NUM; v->num = NAN; return true; }          // Python json extensions
    if (lit("Infinity")) { v->kind = JVal::NUM; v->num = INFINITY; return true; }
    if (lit("-Infinity")) { v->kind = JVal::NUM; v->num = -INFINITY; return true; }
    return number(v);
  }
};

uint32_t rd_u32(const uint8_t* p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24); }
uint16_t rd_u16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }

}  // namespace

struct tbn_tbnt {
  tbn_config cfg{};
  double lambda_sparse = 1e-3;
  int64_t seed = 0;
  std::string model_version;
  std::vector<std::string> names;          // param_order
  std::vector<std::vector<int64_t>> shapes;
  std::vector<size_t> offsets;             // element offsets into flat
  std::vector<double> flat;                // aligned copy of payload 2
  std::vector<double> mean, var;
};

namespace {

// ModelConfig(**meta["config"]) (config.py:9-41): keyword names are the
// dataclass fields; an unknown or missing required key is a TypeError in the
// reference, i.e. ModelFormatError("bad metadata section") here.
tbn_status read_config(const JVal& c, tbn_tbnt* t) {
  if (c.kind != JVal::OBJ) return err(TBN_ERR_FORMAT, "bad metadata section: config is not an object");
  static const char* known[] = {"feature_count", "n_classes", "n_d", "n_a", "n_steps",
                                "lambda_sparse", "gamma", "seed"};
  for (const auto& kv : c.obj) {
    bool ok = false;
    for (const char* k : known) ok |= kv.first == k;
    if (!ok) return err(TBN_ERR_FORMAT, "bad metadata section: unexpected config key '" + kv.first + "'");
    if (kv.second.kind != JVal::NUM && kv.second.kind != JVal::BOOL)
      return err(TBN_ERR_FORMAT, "bad metadata section: config '" + kv.first + "' is not a number");
  }
  auto num = [&](const char* k, double dflt, bool* present) -> double {
    const JVal* v = c.get(k);
    *present = v != nullptr;
    if (!v) return dflt;
    return v->kind == JVal::BOOL ? (v->b ? 1.0 : 0.0) : v->num;
  };
  bool has = false;
  const double fc = num("feature_count", 0, &has);
  if (!has) return err(TBN_ERR_FORMAT, "bad metadata section: config lacks 'feature_count'");
  const double nc = num("n_classes", 2, &has), nd = num("n_d", 8, &has), na = num("n_a", 8, &has),
               ns = num("n_steps", 3, &has), ls = num("lambda_sparse", 1e-3, &has),
               gm = num("gamma", 1.3, &has), sd = num("seed", 0, &has);
  // ModelConfig.__post_init__ (config.py:29-41) -> ConfigurationError
  if (!(fc >= 1)) return err(TBN_ERR_CONFIG, "feature_count must be >= 1");
  if (!(nc >= 2)) return err(TBN_ERR_CONFIG, "n_classes must be >= 2");
  if (!(nd >= 1) || !(na >= 1)) return err(TBN_ERR_CONFIG, "n_d and n_a must be >= 1");
  if (!(ns >= 1)) return err(TBN_ERR_CONFIG, "n_steps must be >= 1");
  if (ls < 0) return err(TBN_ERR_CONFIG, "lambda_sparse must be >= 0");
  if (gm < 1.0) return err(TBN_ERR_CONFIG, "gamma must be >= 1");
  for (double v : {fc, nc, nd, na, ns})
    if (v != std::floor(v) || v > 1e9) return err(TBN_ERR_FORMAT, "bad metadata section: non-integer shape field");
  t->cfg.feature_count = (int32_t)fc;
  t->cfg.n_classes = (int32_t)nc;
  t->cfg.n_d = (int32_t)nd;
  t->cfg.n_a = (int32_t)na;
  t->cfg.n_steps = (int32_t)ns;
  t->cfg.flags = 0;
  t->cfg.gamma = gm;
  t->lambda_sparse = ls;
  t->seed = (int64_t)sd;
  return TBN_OK;
}

tbn_status parse(const uint8_t* s, size_t n, tbn_tbnt* t) {
  if (!s && n) return err(TBN_ERR_FORMAT, "null stream");
  if (n < 10) return err(TBN_ERR_TRUNCATED, "stream shorter than header");
  if (std::memcmp(s, "TBNT", 4) != 0) return err(TBN_ERR_FORMAT, "bad magic bytes");
  const uint16_t version = rd_u16(s + 4);
  if (version != 1)
    return err(TBN_ERR_FORMAT_VERSION, "format version " + std::to_string(version) + " not supported (expected 1)");
  size_t off = 6;
  const uint8_t* sec[3];
  size_t len[3];
  for (int i = 0; i < 3; ++i) {
    if (off + 4 > n - 4) return err(TBN_ERR_TRUNCATED, "section header missing");
    len[i] = rd_u32(s + off);
    off += 4;
    if (off + len[i] > n - 4) return err(TBN_ERR_TRUNCATED, "section payload incomplete");
    sec[i] = s + off;
    off += len[i];
  }
  if (off + 4 != n) return err(TBN_ERR_FORMAT, "unexpected trailing bytes");
  if (tbn_crc32c(s, off, 0) != rd_u32(s + off)) return err(TBN_ERR_CHECKSUM, "CRC-32C mismatch");

  JVal meta;
  JParser jp(reinterpret_cast<const char*>(sec[0]), len[0]);
  if (!jp.parse(&meta) || meta.kind != JVal::OBJ) return err(TBN_ERR_FORMAT, "bad metadata section: invalid JSON");
  const JVal* cfg = meta.get("config");
  const JVal* order = meta.get("param_order");
  const JVal* shapes = meta.get("param_shapes");
  const JVal* mv = meta.get("model_version");
  if (!cfg) return err(TBN_ERR_FORMAT, "bad metadata section: 'config'");
  tbn_status st = read_config(*cfg, t);
  if (st != TBN_OK) return st;
  if (!order || order->kind != JVal::ARR) return err(TBN_ERR_FORMAT, "bad metadata section: 'param_order'");
  if (!shapes || shapes->kind != JVal::OBJ) return err(TBN_ERR_FORMAT, "bad metadata section: 'param_shapes'");

  // normalization stats (payload 1): 2F little-endian float64
  const int64_t F = t->cfg.feature_count;
  if (len[1] % 8 != 0 || (int64_t)(len[1] / 8) != 2 * F)
    return err(TBN_ERR_FORMAT, "normalization stats size mismatch");
  t->mean.resize(F);
  t->var.resize(F);
  std::memcpy(t->mean.data(), sec[1], F * 8);
  std::memcpy(t->var.data(), sec[1] + F * 8, F * 8);

  // parameters (payload 2), param_order x param_shapes
  if (len[2] % 8 != 0) return err(TBN_ERR_FORMAT, "parameter section size mismatch");
  const size_t total = len[2] / 8;
  t->flat.resize(total);
  if (total) std::memcpy(t->flat.data(), sec[2], total * 8);
  size_t pos = 0;
  for (const JVal& nm : order->arr) {
    if (nm.kind != JVal::STR) return err(TBN_ERR_FORMAT, "bad metadata section: param name");
    const JVal* sh = shapes->get(nm.str);
    if (!sh || sh->kind != JVal::ARR) return err(TBN_ERR_FORMAT, "bad metadata section: no shape for " + nm.str);
    std::vector<int64_t> dims;
    size_t size = 1;
    for (const JVal& d : sh->arr) {
      if (d.kind != JVal::NUM || d.num < 0 || d.num != std::floor(d.num) || d.num > 1e12)
        return err(TBN_ERR_FORMAT, "bad metadata section: shape of " + nm.str);
      dims.push_back((int64_t)d.num);
      size *= (size_t)d.num;
    }
    if (pos + size > total) return err(TBN_ERR_FORMAT, "parameter section size mismatch");
    t->names.push_back(nm.str);
    t->shapes.push_back(dims);
    t->offsets.push_back(pos);
    pos += size;
  }
  if (pos != total) return err(TBN_ERR_FORMAT, "parameter section size mismatch");
  // TabNetModel.__post_init__ (network.py:110-114)
  if (!mv || mv->kind != JVal::STR) return err(TBN_ERR_FORMAT, "bad metadata section: 'model_version'");
  t->model_version = mv->str;
  if (t->model_version.empty()) return err(TBN_ERR_CONFIG, "model_version must be non-empty");
  for (double v : t->var)
    if (!(v > 0)) return err(TBN_ERR_CONFIG, "normalization variances must be > 0");
  return TBN_OK;
}

}  // namespace

extern "C" {

tbn_status tbn_tbnt_parse(const uint8_t* data, size_t n, tbn_tbnt** out) {
  if (!out) return err(TBN_ERR_FORMAT, "null output");
  *out = nullptr;
  std::unique_ptr<tbn_tbnt> t(new tbn_tbnt());
  const tbn_status st = parse(data, n, t.get());
  if (st != TBN_OK) return st;
  *out = t.release();
  return TBN_OK;
}

void tbn_tbnt_free(tbn_tbnt* t) { delete t; }

tbn_status tbn_tbnt_info(const tbn_tbnt* t, tbn_config* cfg, double* lambda_sparse, int64_t* seed,
                         const char** model_version, int32_t* n_params) {
  if (!t) return err(TBN_ERR_FORMAT, "null handle");
  if (cfg) *cfg = t->cfg;
  if (lambda_sparse) *lambda_sparse = t->lambda_sparse;
  if (seed) *seed = t->seed;
  if (model_version) *model_version = t->model_version.c_str();
  if (n_params) *n_params = (int32_t)t->names.size();
  return TBN_OK;
}

tbn_status tbn_tbnt_param(const tbn_tbnt* t, int32_t i, const char** name, int32_t* ndim, int64_t* dims,
                          const double** data) {
  if (!t || i < 0 || i >= (int32_t)t->names.size()) return err(TBN_ERR_FORMAT, "parameter index out of range");
  if (name) *name = t->names[i].c_str();
  const auto& sh = t->shapes[i];
  if (ndim) *ndim = (int32_t)sh.size();
  if (dims)
    for (size_t d = 0; d < sh.size() && d < 8; ++d) dims[d] = sh[d];
  if (data) *data = t->flat.data() + t->offsets[i];
  return TBN_OK;
}

tbn_status tbn_tbnt_norm(const tbn_tbnt* t, const double** mean, const double** var) {
  if (!t) return err(TBN_ERR_FORMAT, "null handle");
  if (mean) *mean = t->mean.data();
  if (var) *var = t->var.data();
  return TBN_OK;
}

tbn_status tbn_model_create_from_tbnt(const uint8_t* data, size_t n, int32_t precision, int32_t device,
                                      int32_t cfg_flags, int32_t head_column, tbn_model** out) {
  if (!out) return err(TBN_ERR_CONFIG, "null output");
  *out = nullptr;
  tbn_tbnt t;
  tbn_status st = parse(data, n, &t);
  if (st != TBN_OK) return st;
  tbn_config cfg = t.cfg;
  std::vector<const char*> names;
  std::vector<const double*> vals;
  std::vector<int64_t> sizes;
  std::vector<double> head_w, head_b;
  const bool regression = (cfg_flags & TBN_CFG_REGRESSION) != 0;
  if (regression && (head_column < 0 || head_column >= cfg.n_classes))
    return err(TBN_ERR_CONFIG, "head_column outside the stored head");
  for (size_t i = 0; i < t.names.size(); ++i) {
    size_t size = 1;
    for (int64_t d : t.shapes[i]) size *= (size_t)d;
    const double* v = t.flat.data() + t.offsets[i];
    if (regression && t.names[i] == "head_W") {     // TabNetRegressor: one column of the head
      const int64_t C = cfg.n_classes, ND = cfg.n_d;
      if ((int64_t)size != ND * C) return err(TBN_ERR_CONFIG, "head_W shape");
      head_w.resize(ND);
      for (int64_t k = 0; k < ND; ++k) head_w[k] = v[k * C + head_column];
      v = head_w.data();
      size = (size_t)ND;
    } else if (regression && t.names[i] == "head_b") {
      if ((int64_t)size != cfg.n_classes) return err(TBN_ERR_CONFIG, "head_b shape");
      head_b.assign(1, v[head_column]);
      v = head_b.data();
      size = 1;
    }
    names.push_back(t.names[i].c_str());
    vals.push_back(v);
    sizes.push_back((int64_t)size);
  }
  if (regression) {
    cfg.n_classes = 1;
    cfg.flags |= TBN_CFG_REGRESSION;
  }
  return tbn_model_create(&cfg, names.data(), vals.data(), sizes.data(), (int32_t)names.size(), t.mean.data(),
                          t.var.data(), precision, device, out);
}

}  // extern "C"
