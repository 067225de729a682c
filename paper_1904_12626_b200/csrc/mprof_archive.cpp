// The profile archive of the drop-in C++ API (reference archive.hpp:12-58;
// SPEC.md io module, ProfileArchive / write_profile / read_profile):
// JSON with "inf" for +infinity, -1 for undefined indexes and floats at
// shortest round-trip precision (std::to_chars), so write -> read is the
// identity on every field. The schema matches paper_1904_12626_b200/archive.py
// (the Python mirror reads what this writes and the other way round).
// Host-only code: the archive is a format, not a kernel.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "mprof/archive.hpp"

namespace mprof {

// ---- accessors (archive.hpp:36-43) ---------------------------------------------
Index ProfileArchive::window() const {
  return profile ? profile->window : (multi ? multi->window : 0);
}
Index ProfileArchive::exclusion_zone() const {
  return profile ? profile->exclusion_zone : (multi ? multi->exclusion_zone : 0);
}
Index ProfileArchive::profile_size() const {
  return profile ? profile->size() : (multi ? multi->size() : 0);
}
double ProfileArchive::coverage() const { return profile ? profile->coverage : 1.0; }
Index ProfileArchive::data_len_a() const {
  if (profile) return profile->data_len;
  if (multi) return multi->data_len;
  return data_a ? data_a->size() : 0;
}
Index ProfileArchive::data_len_b() const { return profile ? profile->data_len_b : 0; }
Index ProfileArchive::data_dims() const {
  if (profile) return profile->data_dims;
  if (multi) return multi->data_dims;
  return data_a ? data_a->dims() : 0;
}
bool ProfileArchive::is_ab() const { return profile && profile->join_kind == JoinKind::ab; }

namespace {

// ---- writer ---------------------------------------------------------------------
class Out {
 public:
  void key(const char* k) {
    sep();
    quoted(k);
    s_ += ':';
    first_ = true;  // the value follows without a comma
  }
  void str(const std::string& v) {
    sepv();
    quoted(v);
  }
  void quoted(const std::string& v) {
    s_ += '"';
    for (char c : v) {
      switch (c) {
        case '"': s_ += "\\\""; break;
        case '\\': s_ += "\\\\"; break;
        case '\n': s_ += "\\n"; break;
        case '\t': s_ += "\\t"; break;
        case '\r': s_ += "\\r"; break;
        default:
          if ((unsigned char)c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof(b), "\\u%04x", (unsigned)c);
            s_ += b;
          } else {
            s_ += c;
          }
      }
    }
    s_ += '"';
  }
  void num(double v) {
    sepv();
    if (std::isinf(v) && v > 0) {
      s_ += "\"inf\"";
      return;
    }
    if (!std::isfinite(v)) throw IoError("archive: NaN / -inf have no encoding");
    char b[32];
    auto r = std::to_chars(b, b + sizeof(b), v);  // shortest round-trip form
    s_.append(b, r.ptr);
    // keep floats recognisable as floats (1.0 not 1), as Python's repr does
    if (std::string_view(b, r.ptr - b).find_first_of(".eEn") == std::string_view::npos) s_ += ".0";
  }
  void num(Index v) {
    sepv();
    s_ += std::to_string(v);
  }
  void boolean(bool v) {
    sepv();
    s_ += v ? "true" : "false";
  }
  void null() {
    sepv();
    s_ += "null";
  }
  void begin(char c) {
    sepv();
    s_ += c;
    first_ = true;
  }
  void end(char c) {
    s_ += c;
    first_ = false;
  }
  template <typename T>
  void vec(const std::vector<T>& v) {
    begin('[');
    for (const T& x : v) num(x);
    end(']');
  }
  template <typename T>
  void mat(const std::vector<std::vector<T>>& m) {
    begin('[');
    for (const auto& r : m) vec(r);
    end(']');
  }
  std::string take() { return std::move(s_); }

 private:
  void sep() {
    if (!first_) s_ += ',';
    first_ = false;
  }
  void sepv() { sep(); }
  std::string s_;
  bool first_ = true;
};

void series(Out& o, const std::optional<MultiTimeSeries>& d) {
  if (!d) return o.null();
  if (d->dims() == 1) return o.vec(d->dim(0).values());
  o.begin('[');
  for (Index k = 0; k < d->dims(); ++k) o.vec(d->dim(k).values());
  o.end(']');
}

// ---- parser (a small recursive-descent JSON reader) -------------------------------
struct J;
using JP = std::shared_ptr<J>;
struct J {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0.0;
  bool integral = false;
  long long inum = 0;
  std::string s;
  std::vector<JP> arr;
  std::map<std::string, JP> obj;
};

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  JP parse() {
    JP v = value();
    ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* why) {
    throw IoError(std::string("corrupt archive: ") + why + " at offset " + std::to_string(p_));
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\t' || t_[p_] == '\r'))
      ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  JP value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end");
    auto v = std::make_shared<J>();
    const char c = t_[p_];
    if (c == '{') {
      v->kind = J::Obj;
      ++p_;
      ws();
      if (p_ < t_.size() && t_[p_] == '}') { ++p_; return v; }
      for (;;) {
        ws();
        if (p_ >= t_.size() || t_[p_] != '"') fail("object key expected");
        std::string k = string();
        ws();
        if (p_ >= t_.size() || t_[p_++] != ':') fail("':' expected");
        v->obj[k] = value();
        ws();
        if (p_ < t_.size() && t_[p_] == ',') { ++p_; continue; }
        if (p_ < t_.size() && t_[p_] == '}') { ++p_; break; }
        fail("',' or '}' expected");
      }
    } else if (c == '[') {
      v->kind = J::Arr;
      ++p_;
      ws();
      if (p_ < t_.size() && t_[p_] == ']') { ++p_; return v; }
      for (;;) {
        v->arr.push_back(value());
        ws();
        if (p_ < t_.size() && t_[p_] == ',') { ++p_; continue; }
        if (p_ < t_.size() && t_[p_] == ']') { ++p_; break; }
        fail("',' or ']' expected");
      }
    } else if (c == '"') {
      v->kind = J::Str;
      v->s = string();
    } else if (lit("true")) {
      v->kind = J::Bool;
      v->b = true;
    } else if (lit("false")) {
      v->kind = J::Bool;
    } else if (lit("null")) {
      v->kind = J::Null;
    } else {
      v->kind = J::Num;
      const size_t s = p_;
      while (p_ < t_.size() && std::strchr("+-0123456789.eE", t_[p_])) ++p_;
      if (p_ == s) fail("value expected");
      const char* b = t_.data() + s;
      const char* e = t_.data() + p_;
      if (std::from_chars(b, e, v->num).ptr != e) fail("bad number");
      v->integral = std::string_view(b, e - b).find_first_of(".eE") == std::string_view::npos;
      if (v->integral && std::from_chars(b, e, v->inum).ptr != e) fail("bad integer");
    }
    return v;
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < t_.size() && t_[p_] != '"') {
      char c = t_[p_++];
      if (c == '\\') {
        if (p_ >= t_.size()) fail("bad escape");
        const char e = t_[p_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (p_ + 4 > t_.size()) fail("bad \\u escape");
            unsigned cp = 0;
            std::from_chars(t_.data() + p_, t_.data() + p_ + 4, cp, 16);
            p_ += 4;
            if (cp < 0x80) {
              out += (char)cp;
            } else if (cp < 0x800) {
              out += (char)(0xC0 | (cp >> 6));
              out += (char)(0x80 | (cp & 0x3F));
            } else {
              out += (char)(0xE0 | (cp >> 12));
              out += (char)(0x80 | ((cp >> 6) & 0x3F));
              out += (char)(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (p_ >= t_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
  const std::string& t_;
  size_t p_ = 0;
};

[[noreturn]] void bad(const std::string& what) { throw IoError("corrupt archive: " + what); }

const JP& field(const J& o, const char* k) {
  static const JP none = std::make_shared<J>();
  auto it = o.obj.find(k);
  return it == o.obj.end() ? none : it->second;
}
bool present(const J& o, const char* k) {
  auto it = o.obj.find(k);
  return it != o.obj.end() && it->second->kind != J::Null;
}
double dnum(const J& v, const char* what) {
  if (v.kind == J::Str && v.s == "inf") return kInf;
  if (v.kind != J::Num) bad(std::string(what) + " is not a number");
  return v.num;
}
Index inum(const J& v, const char* what) {
  if (v.kind != J::Num || !v.integral) bad(std::string(what) + " is not an integer");
  return v.inum;
}
std::string sval(const J& o, const char* k) {
  const JP& v = field(o, k);
  if (v->kind == J::Null) return {};
  if (v->kind != J::Str) bad(std::string(k) + " is not a string");
  return v->s;
}
std::vector<double> dvec(const J& v, const char* what) {
  if (v.kind != J::Arr) bad(std::string(what) + " is not an array");
  std::vector<double> out;
  out.reserve(v.arr.size());
  for (const JP& e : v.arr) out.push_back(dnum(*e, what));
  return out;
}
std::vector<Index> ivec(const J& v, const char* what) {
  if (v.kind != J::Arr) bad(std::string(what) + " is not an array");
  std::vector<Index> out;
  out.reserve(v.arr.size());
  for (const JP& e : v.arr) out.push_back(inum(*e, what));
  return out;
}
template <typename T, typename F>
std::vector<std::vector<T>> mat(const J& v, const char* what, F row) {
  if (v.kind != J::Arr) bad(std::string(what) + " is not an array");
  std::vector<std::vector<T>> out;
  for (const JP& r : v.arr) out.push_back(row(*r, what));
  return out;
}

std::optional<MultiTimeSeries> series_from(const J& v) {
  if (v.kind == J::Null) return std::nullopt;
  if (v.kind != J::Arr) bad("embedded data is not an array");
  std::vector<TimeSeries> dims;
  try {
    if (!v.arr.empty() && v.arr.front()->kind == J::Arr) {
      for (const JP& r : v.arr) dims.emplace_back(dvec(*r, "data"));
    } else {
      dims.emplace_back(dvec(v, "data"));
    }
    return MultiTimeSeries(std::move(dims));
  } catch (const ParameterError& e) {
    bad(std::string("embedded data: ") + e.what());
  }
}

Mode mode_of(const std::string& name) {
  const std::optional<Mode> m = mode_from_name(name);
  if (!m) bad("unknown mode '" + name + "'");
  return *m;
}

}  // namespace

std::string archive_to_json(const ProfileArchive& ar) {
  Out o;
  o.begin('{');
  o.key("schema_version"); o.num((Index)ProfileArchive::kSchemaVersion);
  o.key("mode"); o.str(mode_name(ar.mode));
  o.key("join_kind"); o.str(ar.is_ab() ? "ab" : "self");
  o.key("window"); o.num(ar.window());
  o.key("exclusion_zone"); o.num(ar.exclusion_zone());
  o.key("ez_fraction"); o.num(ar.ez_fraction);
  o.key("coverage"); o.num(ar.coverage());
  o.key("seed"); o.num((Index)(ar.profile ? (Index)ar.profile->seed : 0));
  o.key("data_len"); o.num(ar.data_len_a());
  o.key("data_len_b"); o.num(ar.data_len_b());
  o.key("data_dims"); o.num(ar.data_dims());
  o.key("profile_size"); o.num(ar.profile_size());
  if (ar.profile) {
    const MatrixProfile& p = *ar.profile;
    if (p.index.size() != p.values.size()) throw IoError("archive: profile index / values differ");
    o.key("profile_mode"); o.str(mode_name(p.mode));
    o.key("values"); o.vec(p.values);
    o.key("index"); o.vec(p.index);
    o.key("left_index");
    if (p.has_left_right()) o.vec(p.left_index); else o.null();
    o.key("right_index");
    if (p.has_left_right()) o.vec(p.right_index); else o.null();
  } else {
    o.key("values"); o.null();
    o.key("index"); o.null();
    o.key("left_index"); o.null();
    o.key("right_index"); o.null();
  }
  o.key("multi");
  if (ar.multi) {
    const MultiMatrixProfile& m = *ar.multi;
    o.begin('{');
    o.key("values"); o.mat(m.values);
    o.key("index"); o.mat(m.index);
    o.key("dim_order"); o.mat(m.dim_order);
    o.key("window"); o.num(m.window);
    o.key("exclusion_zone"); o.num(m.exclusion_zone);
    o.key("must_dims"); o.vec(m.must_dims);
    o.key("exc_dims"); o.vec(m.exc_dims);
    o.key("data_len"); o.num(m.data_len);
    o.key("data_dims"); o.num(m.data_dims);
    o.end('}');
  } else {
    o.null();
  }
  o.key("data_a"); series(o, ar.data_a);
  o.key("data_b"); series(o, ar.data_b);
  o.key("name_a"); o.str(ar.name_a);
  o.key("name_b"); o.str(ar.name_b);
  o.key("source_a"); o.str(ar.source_a);
  o.key("source_b"); o.str(ar.source_b);
  o.key("extra");
  o.begin('{');
  if (ar.motif) {
    o.key("motif");
    o.begin('{');
    o.key("pairs");
    o.begin('[');
    for (const MotifPair& mp : ar.motif->pairs) {
      o.begin('{');
      o.key("anchor"); o.num(mp.anchor);
      o.key("pair"); o.num(mp.pair);
      o.key("distance"); o.num(mp.distance);
      o.key("neighbors"); o.vec(mp.neighbors);
      o.end('}');
    }
    o.end(']');
    o.key("window"); o.num(ar.motif->window);
    o.key("radius"); o.num(ar.motif->radius);
    o.key("exclusion_zone"); o.num(ar.motif->exclusion_zone);
    o.end('}');
  }
  if (ar.discord) {
    o.key("discord");
    o.begin('{');
    o.key("index");
    o.begin('[');
    for (const auto& d : ar.discord->discords) o.num(d.first);
    o.end(']');
    o.key("distance");
    o.begin('[');
    for (const auto& d : ar.discord->discords) o.num(d.second);
    o.end(']');
    o.key("exclusion_zone"); o.num(ar.discord->exclusion_zone);
    o.key("truncated"); o.boolean(ar.discord->truncated);
    o.end('}');
  }
  if (ar.chain) {
    o.key("chain");
    o.begin('{');
    o.key("chains"); o.mat(ar.chain->chains);
    o.key("best_chain"); o.vec(ar.chain->best_chain);
    o.key("count"); o.num(ar.chain->count);
    o.end('}');
  }
  if (ar.fluss) {
    const FlussResult& f = *ar.fluss;
    o.key("fluss");
    o.begin('{');
    o.key("arc_counts"); o.vec(f.arc_counts);
    o.key("cac"); o.vec(f.cac);
    o.key("segments"); o.vec(f.segments);
    o.key("min_value"); o.num(f.min_value);
    o.key("min_index"); o.num(f.min_index);
    o.key("truncated"); o.boolean(f.truncated);
    o.key("window"); o.num(f.window);
    o.key("exclusion_factor"); o.num(f.exclusion_factor);
    o.end('}');
  }
  o.end('}');
  o.end('}');
  return o.take();
}

ProfileArchive archive_from_json(const std::string& text) {
  const JP root = Parser(text).parse();
  const J& d = *root;
  if (d.kind != J::Obj) bad("top level is not an object");
  if (!present(d, "schema_version") ||
      inum(*field(d, "schema_version"), "schema_version") != ProfileArchive::kSchemaVersion)
    throw IoError("unsupported archive schema_version (expected " +
                  std::to_string(ProfileArchive::kSchemaVersion) + ")");
  ProfileArchive ar;
  ar.mode = mode_of(sval(d, "mode"));
  if (present(d, "ez_fraction")) ar.ez_fraction = dnum(*field(d, "ez_fraction"), "ez_fraction");
  if (present(d, "values")) {
    MatrixProfile p;
    p.values = dvec(*field(d, "values"), "values");
    p.index = ivec(*field(d, "index"), "index");
    const Index size = inum(*field(d, "profile_size"), "profile_size");
    if ((Index)p.values.size() != size || p.index.size() != p.values.size())
      bad("profile length mismatch");
    if (present(d, "left_index")) {
      p.left_index = ivec(*field(d, "left_index"), "left_index");
      p.right_index = ivec(*field(d, "right_index"), "right_index");
      if (p.left_index.size() != p.values.size() || p.right_index.size() != p.values.size())
        bad("left/right length mismatch");
    }
    p.window = inum(*field(d, "window"), "window");
    p.exclusion_zone = inum(*field(d, "exclusion_zone"), "exclusion_zone");
    p.mode = present(d, "profile_mode") ? mode_of(sval(d, "profile_mode")) : ar.mode;
    const std::string jk = sval(d, "join_kind");
    if (jk != "self" && jk != "ab") bad("join_kind must be self or ab");
    p.join_kind = jk == "ab" ? JoinKind::ab : JoinKind::self;
    p.coverage = dnum(*field(d, "coverage"), "coverage");
    p.seed = (std::uint64_t)inum(*field(d, "seed"), "seed");
    p.data_len = inum(*field(d, "data_len"), "data_len");
    p.data_len_b = inum(*field(d, "data_len_b"), "data_len_b");
    p.data_dims = inum(*field(d, "data_dims"), "data_dims");
    ar.profile = std::move(p);
  }
  if (present(d, "multi")) {
    const J& m = *field(d, "multi");
    MultiMatrixProfile mm;
    mm.values = mat<double>(*field(m, "values"), "multi.values", dvec);
    mm.index = mat<Index>(*field(m, "index"), "multi.index", ivec);
    mm.dim_order = mat<Index>(*field(m, "dim_order"), "multi.dim_order", ivec);
    mm.window = inum(*field(m, "window"), "multi.window");
    mm.exclusion_zone = inum(*field(m, "exclusion_zone"), "multi.exclusion_zone");
    mm.must_dims = ivec(*field(m, "must_dims"), "multi.must_dims");
    mm.exc_dims = ivec(*field(m, "exc_dims"), "multi.exc_dims");
    mm.data_len = inum(*field(m, "data_len"), "multi.data_len");
    mm.data_dims = inum(*field(m, "data_dims"), "multi.data_dims");
    ar.multi = std::move(mm);
  }
  ar.data_a = series_from(*field(d, "data_a"));
  ar.data_b = series_from(*field(d, "data_b"));
  ar.name_a = sval(d, "name_a");
  ar.name_b = sval(d, "name_b");
  ar.source_a = sval(d, "source_a");
  ar.source_b = sval(d, "source_b");
  if (present(d, "extra")) {
    const J& x = *field(d, "extra");
    if (present(x, "motif")) {
      const J& m = *field(x, "motif");
      MotifSet ms;
      const J& pairs = *field(m, "pairs");
      if (pairs.kind != J::Arr) bad("motif.pairs is not an array");
      for (const JP& e : pairs.arr) {
        MotifPair mp;
        mp.anchor = inum(*field(*e, "anchor"), "motif.anchor");
        mp.pair = inum(*field(*e, "pair"), "motif.pair");
        mp.distance = dnum(*field(*e, "distance"), "motif.distance");
        mp.neighbors = ivec(*field(*e, "neighbors"), "motif.neighbors");
        ms.pairs.push_back(std::move(mp));
      }
      ms.window = inum(*field(m, "window"), "motif.window");
      ms.radius = dnum(*field(m, "radius"), "motif.radius");
      ms.exclusion_zone = inum(*field(m, "exclusion_zone"), "motif.exclusion_zone");
      ar.motif = std::move(ms);
    }
    if (present(x, "discord")) {
      const J& q = *field(x, "discord");
      DiscordSet ds;
      const std::vector<Index> idx = ivec(*field(q, "index"), "discord.index");
      const std::vector<double> dist = dvec(*field(q, "distance"), "discord.distance");
      if (idx.size() != dist.size()) bad("discord index / distance lengths differ");
      for (size_t k = 0; k < idx.size(); ++k) ds.discords.emplace_back(idx[k], dist[k]);
      ds.exclusion_zone = inum(*field(q, "exclusion_zone"), "discord.exclusion_zone");
      ds.truncated = field(q, "truncated")->kind == J::Bool && field(q, "truncated")->b;
      ar.discord = std::move(ds);
    }
    if (present(x, "chain")) {
      const J& c = *field(x, "chain");
      ChainSet cs;
      cs.chains = mat<Index>(*field(c, "chains"), "chain.chains", ivec);
      cs.best_chain = ivec(*field(c, "best_chain"), "chain.best_chain");
      cs.count = inum(*field(c, "count"), "chain.count");
      ar.chain = std::move(cs);
    }
    if (present(x, "fluss")) {
      const J& f = *field(x, "fluss");
      FlussResult fr;
      fr.arc_counts = ivec(*field(f, "arc_counts"), "fluss.arc_counts");
      fr.cac = dvec(*field(f, "cac"), "fluss.cac");
      fr.segments = ivec(*field(f, "segments"), "fluss.segments");
      fr.min_value = dnum(*field(f, "min_value"), "fluss.min_value");
      fr.min_index = inum(*field(f, "min_index"), "fluss.min_index");
      fr.truncated = field(f, "truncated")->kind == J::Bool && field(f, "truncated")->b;
      fr.window = inum(*field(f, "window"), "fluss.window");
      fr.exclusion_factor = dnum(*field(f, "exclusion_factor"), "fluss.exclusion_factor");
      ar.fluss = std::move(fr);
    }
  }
  return ar;
}

void write_profile(const ProfileArchive& archive, const std::string& path) {
  const std::string text = archive_to_json(archive);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw IoError("cannot write " + path);
  f << text;
  if (!f) throw IoError("write failed: " + path);
}

ProfileArchive read_profile(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot read " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return archive_from_json(ss.str());
}

namespace {
std::string g6(double v) {  // printf %.6g, as the Python mirror's {:.6g}
  char b[32];
  std::snprintf(b, sizeof(b), "%.6g", v);
  return b;
}
}  // namespace

std::string render_profile_block(const ProfileArchive& ar) {
  std::string out = "Matrix profile (" + std::string(mode_name(ar.mode)) + ", " +
                    (ar.is_ab() ? "AB-join" : "self-join") + ")\n";
  out += "Profile size = " + std::to_string(ar.profile_size()) + "\n";
  out += "Window size = " + std::to_string(ar.window()) + "\n";
  out += "Exclusion zone = " + std::to_string(ar.exclusion_zone()) + "\n";
  out += "Coverage = " + g6(ar.coverage()) + "\n";
  if (ar.profile) {
    const MatrixProfile& p = *ar.profile;
    Index i_min = -1, i_max = -1;
    for (Index i = 0; i < p.size(); ++i) {
      const double v = p.values[(size_t)i];
      if (!std::isfinite(v)) continue;
      if (i_min < 0 || v < p.values[(size_t)i_min]) i_min = i;
      if (i_max < 0 || v > p.values[(size_t)i_max]) i_max = i;
    }
    if (i_min >= 0) {  // 1-based positions (archive.hpp:51-54)
      out += "Min distance = " + g6(p.values[(size_t)i_min]) + " at " + std::to_string(i_min + 1) +
             " (nearest " + std::to_string(p.index[(size_t)i_min] + 1) + ")\n";
      out += "Max distance = " + g6(p.values[(size_t)i_max]) + " at " + std::to_string(i_max + 1) +
             "\n";
    }
  }
  return out;
}

std::string render_discord_block(const DiscordSet& ds) {
  std::string out = "Discords = " + std::to_string(ds.discords.size()) +
                    (ds.truncated ? " (fewer than requested)" : "") + "\n";
  out += "Exclusion zone = " + std::to_string(ds.exclusion_zone) + "\n";
  for (size_t k = 0; k < ds.discords.size(); ++k)
    out += "Discord " + std::to_string(k + 1) + " at " + std::to_string(ds.discords[k].first + 1) +
           " distance " + g6(ds.discords[k].second) + "\n";
  return out;
}

std::string render_fluss_block(const FlussResult& f, Index profile_size) {
  std::string out = "Profile size = " + std::to_string(profile_size) + "\n";
  out += "Window size = " + std::to_string(f.window) + "\n";
  out += "Segments = " + std::to_string(f.segments.size()) +
         (f.truncated ? " (fewer than requested)" : "") + "\n";
  for (size_t k = 0; k < f.segments.size(); ++k)
    out += "Regime change " + std::to_string(k + 1) + " at " + std::to_string(f.segments[k] + 1) +
           "\n";
  if (f.min_index >= 0)
    out += "Min CAC = " + g6(f.min_value) + " at " + std::to_string(f.min_index + 1) + "\n";
  return out;
}

}  // namespace mprof
