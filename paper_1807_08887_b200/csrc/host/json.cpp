#include "json.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.h"

namespace tofu {

const Json& Json::at(const std::string& k) const {
  const Json* v = get(k);
  if (!v) throw Error(TOFU_ERR_PARSE, "json: missing key '" + k + "'");
  return *v;
}
int64_t Json::as_int() const {
  if (kind != Num) throw Error(TOFU_ERR_PARSE, "json: expected number");
  return (int64_t)std::llround(num);
}
double Json::as_num() const {
  if (kind != Num) throw Error(TOFU_ERR_PARSE, "json: expected number");
  return num;
}
const std::string& Json::as_str() const {
  if (kind != Str) throw Error(TOFU_ERR_PARSE, "json: expected string");
  return str;
}

namespace {
struct P {
  const std::string& s;
  size_t i = 0;
  explicit P(const std::string& t) : s(t) {}
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
  }
  [[noreturn]] void err(const char* m) { throw Error(TOFU_ERR_PARSE, std::string("json: ") + m + " at " + std::to_string(i)); }
  Json value() {
    ws();
    if (i >= s.size()) err("unexpected end");
    char c = s[i];
    Json v;
    if (c == '{') {
      v.kind = Json::Obj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') { ++i; return v; }
      while (true) {
        ws();
        if (s[i] != '"') err("expected key");
        std::string k = string();
        ws();
        if (s[i] != ':') err("expected ':'");
        ++i;
        v.obj.emplace_back(k, value());
        ws();
        if (s[i] == ',') { ++i; continue; }
        if (s[i] == '}') { ++i; break; }
        err("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = Json::Arr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') { ++i; return v; }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (s[i] == ',') { ++i; continue; }
        if (s[i] == ']') { ++i; break; }
        err("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = Json::Str;
      v.str = string();
    } else if (s.compare(i, 4, "true") == 0) {
      v.kind = Json::Bool; v.b = true; i += 4;
    } else if (s.compare(i, 5, "false") == 0) {
      v.kind = Json::Bool; i += 5;
    } else if (s.compare(i, 4, "null") == 0) {
      i += 4;
    } else {
      char* end = nullptr;
      v.num = std::strtod(s.c_str() + i, &end);
      if (end == s.c_str() + i) err("bad value");
      v.kind = Json::Num;
      i = end - s.c_str();
    }
    return v;
  }
  std::string string() {
    ++i;  // opening quote
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        ++i;
        char e = s[i];
        if (e == 'n') out += '\n';
        else if (e == 't') out += '\t';
        else if (e == 'r') out += '\r';
        else if (e == 'u') {
          unsigned cp = std::strtoul(s.substr(i + 1, 4).c_str(), nullptr, 16);
          i += 4;
          if (cp < 0x80) out += (char)cp;
          else if (cp < 0x800) { out += (char)(0xC0 | (cp >> 6)); out += (char)(0x80 | (cp & 0x3F)); }
          else { out += (char)(0xE0 | (cp >> 12)); out += (char)(0x80 | ((cp >> 6) & 0x3F)); out += (char)(0x80 | (cp & 0x3F)); }
        } else out += e;
        ++i;
      } else {
        out += s[i++];
      }
    }
    if (i >= s.size()) err("unterminated string");
    ++i;
    return out;
  }
};
}  // namespace

Json json_parse(const std::string& text) {
  P p(text);
  Json v = p.value();
  p.ws();
  if (p.i != text.size()) p.err("trailing data");
  return v;
}

std::string json_quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') { o += '\\'; o += c; }
    else if (c == '\n') o += "\\n";
    else o += c;
  }
  return o + "\"";
}

std::string json_num(double v) {
  if (std::isfinite(v) && v == std::floor(v) && std::fabs(v) < 9e15) return std::to_string((long long)v);
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

}  // namespace tofu
