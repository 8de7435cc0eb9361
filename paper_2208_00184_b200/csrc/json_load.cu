// json_load.cu — graph and device documents parsed straight into the SoA
// arrays the device path uploads, without the reference's DOM + AoS detour
// (json_io.cpp:43-74 graph_from_json, :93-117 devices_from_json).
//
// Host code: a strict single-pass JSON reader (RFC 8259 grammar, UTF-8 validated, last
// duplicate key wins — nlohmann::json::parse semantics) that first validates the whole
// document (so syntax errors win over schema errors, as with json::parse), then reads
// the fields the reference reads, in the reference's order and with its error messages.
// Numbers follow nlohmann's typing: integer literals are int64 (negative) / uint64
// (positive) when they fit, else double; get<int64_t>() truncates doubles and wraps
// uint64 (static_cast), which is what the reference's number<T>() does.
#include <cmath>
#include <cstdlib>
#include <clocale>
#include <cstring>
#include <locale.h>
#include <string>
#include <unordered_map>
#include <vector>

#include "abi_util.cuh"
#include "results.h"

namespace dpb {
namespace {

struct Span {
  const char* b = nullptr;
  const char* e = nullptr;
  bool ok() const { return b != nullptr; }
};

struct Num {
  enum Kind { kInt, kUInt, kFloat } kind = kInt;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0.0;
  int64_t as_i64() const {
    return kind == kInt ? i : kind == kUInt ? static_cast<int64_t>(u) : static_cast<int64_t>(d);
  }
  int32_t as_i32() const {
    return kind == kInt ? static_cast<int32_t>(i) : kind == kUInt ? static_cast<int32_t>(u) : static_cast<int32_t>(d);
  }
  double as_f64() const { return kind == kInt ? static_cast<double>(i) : kind == kUInt ? static_cast<double>(u) : d; }
};

[[noreturn]] void syntax(const char* what) { fail(DP_E_PARSE_ERROR, "invalid JSON: %s", what); }

struct Reader {
  const char* p;
  const char* end;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < end && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  void expect(char c, const char* what) {
    if (!eat(c)) syntax(what);
  }
  // Validates a string starting at '"'; decodes it into *out when out != nullptr.
  void string(std::string* out) {
    if (p >= end || *p != '"') syntax("expected string");
    ++p;
    for (;;) {
      if (p >= end) syntax("unterminated string");
      const unsigned char c = static_cast<unsigned char>(*p);
      if (c == '"') {
        ++p;
        return;
      }
      if (c < 0x20) syntax("control character in string");
      if (c == '\\') {
        if (++p >= end) syntax("unterminated escape");
        const char x = *p++;
        uint32_t cp = 0;
        switch (x) {
          case '"': cp = '"'; break;
          case '\\': cp = '\\'; break;
          case '/': cp = '/'; break;
          case 'b': cp = '\b'; break;
          case 'f': cp = '\f'; break;
          case 'n': cp = '\n'; break;
          case 'r': cp = '\r'; break;
          case 't': cp = '\t'; break;
          case 'u': {
            cp = hex4();
            if (cp >= 0xD800 && cp <= 0xDBFF) {
              if (end - p < 6 || p[0] != '\\' || p[1] != 'u') syntax("unpaired surrogate");
              p += 2;
              const uint32_t lo = hex4();
              if (lo < 0xDC00 || lo > 0xDFFF) syntax("invalid surrogate pair");
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
              syntax("unpaired surrogate");
            }
            break;
          }
          default: syntax("invalid escape");
        }
        if (out) utf8(out, cp);
        continue;
      }
      // raw UTF-8 sequence (validated, RFC 3629)
      int len = c < 0x80 ? 1 : (c >> 5) == 0x6 ? 2 : (c >> 4) == 0xE ? 3 : (c >> 3) == 0x1E ? 4 : 0;
      if (!len || end - p < len) syntax("ill-formed UTF-8");
      uint32_t cp = len == 1 ? c : len == 2 ? (c & 0x1F) : len == 3 ? (c & 0x0F) : (c & 0x07);
      for (int k = 1; k < len; ++k) {
        const unsigned char cc = static_cast<unsigned char>(p[k]);
        if ((cc & 0xC0) != 0x80) syntax("ill-formed UTF-8");
        cp = (cp << 6) | (cc & 0x3F);
      }
      if ((len == 2 && cp < 0x80) || (len == 3 && cp < 0x800) || (len == 4 && (cp < 0x10000 || cp > 0x10FFFF)) ||
          (cp >= 0xD800 && cp <= 0xDFFF))
        syntax("ill-formed UTF-8");
      if (out) out->append(p, len);
      p += len;
    }
  }
  uint32_t hex4() {
    if (end - p < 4) syntax("truncated \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else syntax("invalid \\u escape");
    }
    return v;
  }
  static void utf8(std::string* o, uint32_t cp) {
    if (cp < 0x80) {
      o->push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      o->push_back(static_cast<char>(0xC0 | (cp >> 6)));
      o->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      o->push_back(static_cast<char>(0xE0 | (cp >> 12)));
      o->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      o->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      o->push_back(static_cast<char>(0xF0 | (cp >> 18)));
      o->push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      o->push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      o->push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }
  Num number() {
    const char* s = p;
    bool neg = false, frac = false;
    if (p < end && *p == '-') {
      neg = true;
      ++p;
    }
    if (p >= end || *p < '0' || *p > '9') syntax("invalid number");
    if (*p == '0') {
      ++p;
    } else {
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && *p == '.') {
      frac = true;
      ++p;
      if (p >= end || *p < '0' || *p > '9') syntax("invalid number");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      frac = true;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || *p < '0' || *p > '9') syntax("invalid number");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    std::string tok(s, p);
    Num n;
    if (!frac) {
      errno = 0;
      char* q = nullptr;
      if (neg) {
        const long long v = std::strtoll(tok.c_str(), &q, 10);
        if (errno == 0) {
          n.kind = Num::kInt;
          n.i = v;
          return n;
        }
      } else {
        const unsigned long long v = std::strtoull(tok.c_str(), &q, 10);
        if (errno == 0) {
          n.kind = Num::kUInt;
          n.u = v;
          return n;
        }
      }
    }
    n.kind = Num::kFloat;
    // the "C" locale whatever LC_NUMERIC says (nlohmann reads '.' under any locale)
    static const locale_t c_locale = newlocale(LC_ALL_MASK, "C", static_cast<locale_t>(0));
    n.d = strtod_l(tok.c_str(), nullptr, c_locale);
    return n;
  }
  void literal(const char* w) {
    const size_t k = std::strlen(w);
    if (static_cast<size_t>(end - p) < k || std::memcmp(p, w, k) != 0) syntax("invalid literal");
    p += k;
  }
  // Validates one value and returns its span.  Iterative (an explicit stack of open
  // containers), so nesting depth is bounded by memory only, as in json::parse.
  Span value() {
    ws();
    if (p >= end) syntax("unexpected end of input");
    Span s;
    s.b = p;
    std::vector<char> open;
    for (;;) {
      ws();
      if (p >= end) syntax("unexpected end of input");
      bool closed = true;  // a complete value was just read
      switch (*p) {
        case '{':
          ++p;
          if (!eat('}')) {
            open.push_back('{');
            ws();
            string(nullptr);
            expect(':', "expected ':'");
            closed = false;
          }
          break;
        case '[':
          ++p;
          if (!eat(']')) {
            open.push_back('[');
            closed = false;
          }
          break;
        case '"': string(nullptr); break;
        case 't': literal("true"); break;
        case 'f': literal("false"); break;
        case 'n': literal("null"); break;
        default: number(); break;
      }
      if (!closed) continue;
      // after a complete value: the next member / element, or close containers
      for (;;) {
        if (open.empty()) {
          s.e = p;
          return s;
        }
        if (open.back() == '{') {
          if (eat(',')) {
            ws();
            string(nullptr);
            expect(':', "expected ':'");
            break;
          }
          expect('}', "expected ',' or '}'");
        } else {
          if (eat(',')) break;
          expect(']', "expected ',' or ']'");
        }
        open.pop_back();
      }
    }
  }
};

// The kinds of a validated value, read from its first character.
inline bool is_object(Span s) { return s.ok() && *s.b == '{'; }
inline bool is_array(Span s) { return s.ok() && *s.b == '['; }
inline bool is_string(Span s) { return s.ok() && *s.b == '"'; }
inline bool is_null(Span s) { return s.ok() && *s.b == 'n'; }
inline bool is_number(Span s) { return s.ok() && (*s.b == '-' || (*s.b >= '0' && *s.b <= '9')); }

// Members of a validated object (last duplicate wins): calls f(key, value span).
template <typename F>
void members(Span obj, F f) {
  Reader r{obj.b + 1, obj.e};
  if (r.eat('}')) return;
  std::string key;
  do {
    r.ws();
    key.clear();
    r.string(&key);
    r.expect(':', "expected ':'");
    const Span v = r.value();
    f(key, v);
  } while (r.eat(','));
}

template <typename F>
void elements(Span arr, F f) {
  Reader r{arr.b + 1, arr.e};
  if (r.eat(']')) return;
  do f(r.value());
  while (r.eat(','));
}

Num num_of(Span s) {
  Reader r{s.b, s.e};
  return r.number();
}

// json_io.cpp:25-33 number<T>(): missing field / not a number.
Num field_number(const Span* v, const char* name, const char* context) {
  if (!v->ok()) fail(DP_E_PARSE_ERROR, "missing field '%s' in %s", name, context);
  if (!is_number(*v)) fail(DP_E_PARSE_ERROR, "field '%s' in %s must be a number", name, context);
  return num_of(*v);
}

// json_io.cpp:35-40
void check_schema_version(Span top, const char* context) {
  Span sv;
  members(top, [&](const std::string& k, Span v) {
    if (k == "schema_version") sv = v;
  });
  if (!sv.ok()) return;
  bool ok = false;
  if (is_number(sv)) {
    const Num n = num_of(sv);
    ok = n.kind != Num::kFloat && n.as_i32() == 1;
  }
  if (!ok) fail(DP_E_PARSE_ERROR, "unsupported schema_version in %s", context);
}

Span validated_document(const char* text, int64_t len) {
  if (!text || len < 0) fail(DP_E_ARGUMENT, "null JSON text");
  Reader r{text, text + len};
  const Span top = r.value();
  r.ws();
  if (r.p != r.end) syntax("unexpected trailing content");
  return top;
}

}  // namespace
}  // namespace dpb

using namespace dpb;

extern "C" {

int dp_graph_from_json(const char* text, int64_t len, dp_graph_out_t** out) {
  try {
    if (!out) fail(DP_E_ARGUMENT, "null output");
    const Span top = validated_document(text, len);
    if (!is_object(top)) fail(DP_E_PARSE_ERROR, "graph document must be an object");
    check_schema_version(top, "graph");
    Span nodes, edges;
    members(top, [&](const std::string& k, Span v) {
      if (k == "nodes") nodes = v;
      else if (k == "edges") edges = v;
    });
    if (!nodes.ok()) fail(DP_E_PARSE_ERROR, "missing field 'nodes' in graph");
    if (!is_array(nodes)) fail(DP_E_PARSE_ERROR, "field 'nodes' must be an array");
    std::vector<int64_t> id, w, mem;
    std::vector<int32_t> grp;
    std::unordered_map<std::string, int32_t> labels;
    bool any_group = false;
    std::string gname;
    elements(nodes, [&](Span nj) {
      Span f_id, f_w, f_mem, f_grp;
      if (is_object(nj)) {
        members(nj, [&](const std::string& k, Span v) {
          if (k == "id") f_id = v;
          else if (k == "compute_us") f_w = v;
          else if (k == "memory_bytes") f_mem = v;
          else if (k == "colocation_group") f_grp = v;
        });
      }
      id.push_back(field_number(&f_id, "id", "node").as_i64());
      w.push_back(field_number(&f_w, "compute_us", "node").as_i64());
      mem.push_back(field_number(&f_mem, "memory_bytes", "node").as_i64());
      int32_t label = -1;
      if (f_grp.ok() && !is_null(f_grp)) {
        if (!is_string(f_grp)) fail(DP_E_PARSE_ERROR, "field 'colocation_group' must be a string or null");
        gname.clear();
        Reader r{f_grp.b, f_grp.e};
        r.string(&gname);
        auto it = labels.emplace(gname, static_cast<int32_t>(labels.size())).first;
        label = it->second;
        any_group = true;
      }
      grp.push_back(label);
    });
    if (!edges.ok()) fail(DP_E_PARSE_ERROR, "missing field 'edges' in graph");
    if (!is_array(edges)) fail(DP_E_PARSE_ERROR, "field 'edges' must be an array");
    std::vector<int64_t> es, ed, eb;
    elements(edges, [&](Span ej) {
      Span f_s, f_d, f_b;
      if (is_object(ej)) {
        members(ej, [&](const std::string& k, Span v) {
          if (k == "src") f_s = v;
          else if (k == "dst") f_d = v;
          else if (k == "tensor_bytes") f_b = v;
        });
      }
      es.push_back(field_number(&f_s, "src", "edge").as_i64());
      ed.push_back(field_number(&f_d, "dst", "edge").as_i64());
      eb.push_back(field_number(&f_b, "tensor_bytes", "edge").as_i64());
    });
    dp_graph_out_t* g = new_graph_out(static_cast<int32_t>(id.size()), static_cast<int32_t>(es.size()));
    std::memcpy(g->node_id, id.data(), sizeof(int64_t) * id.size());
    std::memcpy(g->compute_us, w.data(), sizeof(int64_t) * w.size());
    std::memcpy(g->memory_bytes, mem.data(), sizeof(int64_t) * mem.size());
    if (g->group) {
      if (any_group) std::memcpy(g->group, grp.data(), sizeof(int32_t) * grp.size());
      else for (size_t i = 0; i < grp.size(); ++i) g->group[i] = -1;
    }
    std::memcpy(g->edge_src, es.data(), sizeof(int64_t) * es.size());
    std::memcpy(g->edge_dst, ed.data(), sizeof(int64_t) * ed.size());
    std::memcpy(g->edge_bytes, eb.data(), sizeof(int64_t) * eb.size());
    *out = g;
    return DP_OK;
  } catch (const DpFail& f) {
    set_last_error(f.code, f.msg);
    return f.code;
  } catch (const std::bad_alloc&) {
    set_last_error(DP_E_OUT_OF_MEMORY, "host allocation failed");
    return DP_E_OUT_OF_MEMORY;
  }
}

int dp_devices_from_json(const char* text, int64_t len, int32_t* count, int32_t* ids, int64_t* memory_bytes,
                         int32_t capacity, dp_comm_t* comm) {
  try {
    if (!count || !comm) fail(DP_E_ARGUMENT, "null output");
    const Span top = validated_document(text, len);
    // json_io.cpp:93-117
    if (!is_object(top)) fail(DP_E_PARSE_ERROR, "device document must be an object");
    check_schema_version(top, "devices");
    Span devices, cm;
    members(top, [&](const std::string& k, Span v) {
      if (k == "devices") devices = v;
      else if (k == "comm") cm = v;
    });
    if (!devices.ok()) fail(DP_E_PARSE_ERROR, "missing field 'devices' in device file");
    bool empty = true;
    if (is_array(devices)) elements(devices, [&](Span) { empty = false; });
    if (!is_array(devices) || empty) fail(DP_E_PARSE_ERROR, "field 'devices' must be a non-empty array");
    int32_t k = 0;
    elements(devices, [&](Span dj) {
      Span f_id, f_mem;
      if (is_object(dj)) {
        members(dj, [&](const std::string& key, Span v) {
          if (key == "id") f_id = v;
          else if (key == "memory_bytes") f_mem = v;
        });
      }
      const int32_t did = field_number(&f_id, "id", "device").as_i32();
      const int64_t m = field_number(&f_mem, "memory_bytes", "device").as_i64();
      if (m <= 0) fail(DP_E_PARSE_ERROR, "field 'memory_bytes' must be > 0 in device %d", did);
      if (k < capacity && ids && memory_bytes) {
        ids[k] = did;
        memory_bytes[k] = m;
      }
      ++k;
    });
    if (!cm.ok()) fail(DP_E_PARSE_ERROR, "missing field 'comm' in device file");
    Span f_k, f_b;
    if (is_object(cm)) {
      members(cm, [&](const std::string& key, Span v) {
        if (key == "k_us_per_byte") f_k = v;
        else if (key == "b_us") f_b = v;
      });
    }
    comm->k_us_per_byte = field_number(&f_k, "k_us_per_byte", "comm").as_f64();
    comm->b_us = field_number(&f_b, "b_us", "comm").as_f64();
    if (comm->k_us_per_byte < 0 || comm->b_us < 0) fail(DP_E_PARSE_ERROR, "comm coefficients must be non-negative");
    *count = k;
    return DP_OK;
  } catch (const DpFail& f) {
    set_last_error(f.code, f.msg);
    return f.code;
  }
}

}  // extern "C"
