// json.hpp — minimal JSON reader for the topology / engine-config / fault documents.
// Objects keep key order (unknown-key rejection and stable dumps need it).
#pragma once
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace spray {

struct JsonError : std::runtime_error {
  explicit JsonError(const std::string& w) : std::runtime_error(w) {}
};

class Json {
 public:
  enum Kind { Null, Bool, Number, String, Array, Object };
  Kind kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  bool is_null() const { return kind == Null; }
  bool is_object() const { return kind == Object; }
  bool is_array() const { return kind == Array; }
  bool is_string() const { return kind == String; }
  bool is_number() const { return kind == Number; }
  bool contains(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return true;
    return false;
  }
  const Json& at(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw JsonError("missing key '" + k + "'");
  }
  const std::string& as_string() const {
    if (kind != String) throw JsonError("expected a string");
    return str;
  }
  double as_number() const {
    if (kind != Number) throw JsonError("expected a number");
    return num;
  }
  bool as_bool() const {
    if (kind != Bool) throw JsonError("expected a boolean");
    return b;
  }
  double number_or(const std::string& k, double d) const { return contains(k) ? at(k).as_number() : d; }
  std::string string_or(const std::string& k, const std::string& d) const {
    return contains(k) ? at(k).as_string() : d;
  }

  static Json parse(const std::string& text) {
    size_t i = 0;
    Json j = parse_value(text, i);
    skip_ws(text, i);
    if (i != text.size()) throw JsonError("trailing characters at offset " + std::to_string(i));
    return j;
  }

 private:
  static void skip_ws(const std::string& s, size_t& i) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
  }
  static Json parse_value(const std::string& s, size_t& i) {
    skip_ws(s, i);
    if (i >= s.size()) throw JsonError("unexpected end of document");
    const char c = s[i];
    Json j;
    if (c == '{') {
      j.kind = Object;
      ++i;
      skip_ws(s, i);
      if (i < s.size() && s[i] == '}') { ++i; return j; }
      for (;;) {
        skip_ws(s, i);
        if (i >= s.size() || s[i] != '"') throw JsonError("expected a key at offset " + std::to_string(i));
        std::string k = parse_string(s, i);
        skip_ws(s, i);
        if (i >= s.size() || s[i] != ':') throw JsonError("expected ':' at offset " + std::to_string(i));
        ++i;
        j.obj.emplace_back(std::move(k), parse_value(s, i));
        skip_ws(s, i);
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == '}') { ++i; return j; }
        throw JsonError("expected ',' or '}' at offset " + std::to_string(i));
      }
    }
    if (c == '[') {
      j.kind = Array;
      ++i;
      skip_ws(s, i);
      if (i < s.size() && s[i] == ']') { ++i; return j; }
      for (;;) {
        j.arr.push_back(parse_value(s, i));
        skip_ws(s, i);
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == ']') { ++i; return j; }
        throw JsonError("expected ',' or ']' at offset " + std::to_string(i));
      }
    }
    if (c == '"') {
      j.kind = String;
      j.str = parse_string(s, i);
      return j;
    }
    if (s.compare(i, 4, "true") == 0) { i += 4; j.kind = Bool; j.b = true; return j; }
    if (s.compare(i, 5, "false") == 0) { i += 5; j.kind = Bool; j.b = false; return j; }
    if (s.compare(i, 4, "null") == 0) { i += 4; return j; }
    const char* begin = s.c_str() + i;
    char* end = nullptr;
    const double v = std::strtod(begin, &end);
    if (end == begin) throw JsonError("unexpected character at offset " + std::to_string(i));
    i += static_cast<size_t>(end - begin);
    j.kind = Number;
    j.num = v;
    return j;
  }
  static std::string parse_string(const std::string& s, size_t& i) {
    std::string out;
    ++i;  // opening quote
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) break;
        switch (s[i]) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i + 4 >= s.size()) throw JsonError("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(s.substr(i + 1, 4).c_str(), nullptr, 16));
            if (cp < 0x80) out += static_cast<char>(cp);
            else if (cp < 0x800) { out += static_cast<char>(0xc0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3f)); }
            else { out += static_cast<char>(0xe0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 0x3f)); out += static_cast<char>(0x80 | (cp & 0x3f)); }
            i += 4;
            break;
          }
          default: out += s[i];
        }
        ++i;
      } else {
        out += s[i++];
      }
    }
    if (i >= s.size()) throw JsonError("unterminated string");
    ++i;
    return out;
  }
};

}  // namespace spray
