// SPDX-License-Identifier: MIT
// Minimal JSON DOM reader and a writer with nlohmann::json's dump() layout
// (sorted object keys, indent or compact, its number placement). Used by the
// problem files (problem_io.cpp) and the experiment reports (experiment.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace scn {

struct JV {
  enum Kind : uint8_t { Null, Bool, Int, Dbl, Str, Arr, Obj } k = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<JV> a;
  std::vector<std::pair<std::string, JV>> o;  // insertion order; lookups take the last duplicate
  bool is_num() const { return k == Int || k == Dbl; }
  double num() const { return k == Int ? static_cast<double>(i) : d; }
  const JV* find(const char* key) const {
    for (size_t t = o.size(); t-- > 0;)
      if (o[t].first == key) return &o[t].second;
    return nullptr;
  }
};

// throws Error(SCENOPT_E_PARSE_ERROR, prefix + "syntax error at byte ...")
JV parse_json(const std::string& text, const char* prefix);
void put_double(std::string& out, double v);  // nlohmann float layout
void put_string(std::string& out, const std::string& s);

// Streaming writer with nlohmann dump(indent) layout; indent < 0 is compact.
struct Writer {
  std::string out;
  int indent = 2;
  int depth = 0;
  std::vector<int> count;  // elements written per open container
  void nl();
  void sep();  // before an element / member
  void open(char c);
  void close(char c);
  void key(const std::string& k);
  void elem() { sep(); }
};
void dump_value(Writer& w, const JV& v);

}  // namespace scn
