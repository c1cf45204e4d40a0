// Minimal JSON value + parser + writer (host side of the C ABI; no external deps).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace tofu {

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;  // insertion order preserved

  bool is_null() const { return kind == Null; }
  const Json* get(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json& at(const std::string& k) const;
  int64_t as_int() const;
  double as_num() const;
  const std::string& as_str() const;
};

Json json_parse(const std::string& text);

// Writer helpers
std::string json_quote(const std::string& s);
std::string json_num(double v);

}  // namespace tofu
