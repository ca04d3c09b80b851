// SPDX-License-Identifier: MIT
#include "json.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "model.hpp"

namespace scn {

// ---------------------------------------------------------------- reader

namespace {
struct Reader {
  const char* p;
  const char* end;
  const char* begin;
  const char* prefix;
  [[noreturn]] void err(const std::string& what) {
    fail(SCENOPT_E_PARSE_ERROR, std::string(prefix) + "syntax error at byte " + std::to_string(p - begin) + ": " + what);
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(end - p) >= n && std::memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  void put_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (end - p < 4) err("truncated \\u escape");
    unsigned v = 0;
    for (int t = 0; t < 4; ++t, ++p) {
      const char c = *p;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
      else err("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    ++p;  // opening quote
    std::string out;
    while (true) {
      if (p >= end) err("unterminated string");
      const char c = *p++;
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) err("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= end) err("unterminated escape");
      const char e = *p++;
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (!lit("\\u")) err("unpaired surrogate");
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) err("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp < 0xE000) {
            err("unpaired surrogate");
          }
          put_utf8(out, cp);
          break;
        }
        default: err("bad escape");
      }
    }
    return out;
  }
  void number(JV& v) {
    const char* s = p;
    if (p < end && *p == '-') ++p;
    if (p >= end) err("truncated number");
    if (*p == '0') {
      ++p;
    } else if (*p >= '1' && *p <= '9') {
      while (p < end && *p >= '0' && *p <= '9') ++p;
    } else {
      err("invalid number");
    }
    bool frac = false;
    if (p < end && *p == '.') {
      frac = true;
      ++p;
      if (p >= end || *p < '0' || *p > '9') err("invalid number");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      frac = true;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || *p < '0' || *p > '9') err("invalid number");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (!frac) {
      int64_t iv = 0;
      const auto r = std::from_chars(s, p, iv);
      if (r.ec == std::errc() && r.ptr == p) {
        v.k = JV::Int;
        v.i = iv;
        return;
      }
    }
    double dv = 0.0;
    const auto r = std::from_chars(s, p, dv);
    if (r.ptr != p) err("invalid number");
    v.k = JV::Dbl;
    v.d = dv;  // out-of-range magnitudes saturate like strtod
  }
  void value(JV& v, int depth) {
    if (depth > 512) err("nesting too deep");
    ws();
    if (p >= end) err("unexpected end of input");
    const char c = *p;
    if (c == '{') {
      ++p;
      v.k = JV::Obj;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return;
      }
      while (true) {
        ws();
        if (p >= end || *p != '"') err("expected a string key");
        std::string key = str();
        ws();
        if (p >= end || *p != ':') err("expected ':'");
        ++p;
        v.o.emplace_back(std::move(key), JV{});
        value(v.o.back().second, depth + 1);
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return;
        }
        err("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      v.k = JV::Arr;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return;
      }
      while (true) {
        v.a.emplace_back();
        value(v.a.back(), depth + 1);
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return;
        }
        err("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.k = JV::Str;
      v.s = str();
      return;
    }
    if (lit("true")) {
      v.k = JV::Bool;
      v.b = true;
      return;
    }
    if (lit("false")) {
      v.k = JV::Bool;
      return;
    }
    if (lit("null")) return;
    if (c == '-' || (c >= '0' && c <= '9')) {
      number(v);
      return;
    }
    err("unexpected character");
  }
};

}  // namespace

JV parse_json(const std::string& text, const char* prefix) {
  Reader r{text.data(), text.data() + text.size(), text.data(), prefix};
  JV v;
  r.value(v, 0);
  r.ws();
  if (r.p != r.end) r.err("trailing characters");
  return v;
}

// ---------------------------------------------------------------- writer
// nlohmann's placement of a shortest digit string d1..dk with value
// 0.d1..dk x 10^n (dtoa_impl::format_buffer, min_exp -4, max_exp 15).
void put_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (v == 0.0) {
    out += std::signbit(v) ? "-0.0" : "0.0";
    return;
  }
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  std::string sci(buf, r.ptr);  // [-]d[.ddd]e[+-]xx
  if (sci[0] == '-') {
    out += '-';
    sci.erase(0, 1);
  }
  const size_t e = sci.find('e');
  std::string digits;
  for (size_t t = 0; t < e; ++t)
    if (sci[t] != '.') digits += sci[t];
  const int k = static_cast<int>(digits.size());
  const int n = std::stoi(sci.substr(e + 1)) + 1;
  if (k <= n && n <= 15) {
    out += digits;
    out.append(static_cast<size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, static_cast<size_t>(n));
    out += '.';
    out += digits.substr(static_cast<size_t>(n));
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append(static_cast<size_t>(-n), '0');
    out += digits;
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out += digits.substr(1);
    }
    out += 'e';
    int x = n - 1;
    out += x < 0 ? '-' : '+';
    if (x < 0) x = -x;
    if (x < 10) out += '0';
    out += std::to_string(x);
  }
}

void put_string(std::string& out, const std::string& s) {
  out += '"';
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char u[8];
          std::snprintf(u, sizeof u, "\\u%04x", static_cast<unsigned>(static_cast<unsigned char>(c)));
          out += u;
        } else {
          out += c;
        }
    }
  }
  out += '"';
}

void Writer::nl() {
  if (indent < 0) return;
  out += '\n';
  out.append(static_cast<size_t>(indent * depth), ' ');
}
void Writer::sep() {
  if (count.back()++ > 0) out += ',';
  nl();
}
void Writer::open(char c) {
  out += c;
  ++depth;
  count.push_back(0);
}
void Writer::close(char c) {
  --depth;
  if (count.back() > 0) nl();
  count.pop_back();
  out += c;
}
void Writer::key(const std::string& k) {
  sep();
  put_string(out, k);
  out += indent < 0 ? ":" : ": ";
}

// nlohmann dump of a DOM value; object members in sorted key order
// (std::map semantics: the last duplicate wins)
void dump_value(Writer& w, const JV& v) {
  switch (v.k) {
    case JV::Null: w.out += "null"; return;
    case JV::Bool: w.out += v.b ? "true" : "false"; return;
    case JV::Int: w.out += std::to_string(v.i); return;
    case JV::Dbl: put_double(w.out, v.d); return;
    case JV::Str: put_string(w.out, v.s); return;
    case JV::Arr:
      w.open('[');
      for (const JV& e : v.a) {
        w.sep();
        dump_value(w, e);
      }
      w.close(']');
      return;
    case JV::Obj: {
      std::vector<const std::pair<std::string, JV>*> m;
      for (const auto& kv : v.o) {
        bool replaced = false;
        for (auto& q : m)
          if (q->first == kv.first) {
            q = &kv;
            replaced = true;
          }
        if (!replaced) m.push_back(&kv);
      }
      std::sort(m.begin(), m.end(), [](const auto* a, const auto* b) { return a->first < b->first; });
      w.open('{');
      for (const auto* kv : m) {
        w.key(kv->first);
        dump_value(w, kv->second);
      }
      w.close('}');
      return;
    }
  }
}


}  // namespace scn
