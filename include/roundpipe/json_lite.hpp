#pragma once
// Minimal strict JSON reader for the config files (objects, arrays, strings,
// numbers, true/false/null). The reference uses nlohmann/json for the same
// job (reference: proj/include/roundpipe/config_io.hpp:11); this repo has no
// vendored third-party headers, so the tiny subset it needs lives here.

#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace roundpipe {
namespace json_lite {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TypeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Value {
 public:
  enum class Type { Null, Bool, Number, String, Array, Object };

  Value() = default;
  Type type() const { return type_; }
  bool is_object() const { return type_ == Type::Object; }
  bool is_number() const { return type_ == Type::Number; }
  bool is_string() const { return type_ == Type::String; }

  double as_double() const {
    if (type_ != Type::Number) throw TypeError("expected a number");
    return num_;
  }
  int as_int() const { return static_cast<int>(as_double()); }
  bool as_bool() const {
    if (type_ != Type::Bool) throw TypeError("expected a boolean");
    return b_;
  }
  const std::string& as_string() const {
    if (type_ != Type::String) throw TypeError("expected a string");
    return str_;
  }
  bool contains(const std::string& key) const {
    return type_ == Type::Object && obj_.count(key) != 0;
  }
  const Value& at(const std::string& key) const {
    if (type_ != Type::Object) throw TypeError("expected an object");
    auto it = obj_.find(key);
    if (it == obj_.end()) throw TypeError("missing key '" + key + "'");
    return it->second;
  }
  const std::vector<Value>& items() const {
    if (type_ != Type::Array) throw TypeError("expected an array");
    return arr_;
  }

  static Value parse(const std::string& text) {
    std::size_t pos = 0;
    Value v = parse_value(text, pos, 0);
    skip_ws(text, pos);
    if (pos != text.size()) throw ParseError("trailing characters");
    return v;
  }

 private:
  Type type_ = Type::Null;
  bool b_ = false;
  double num_ = 0;
  std::string str_;
  std::vector<Value> arr_;
  std::map<std::string, Value> obj_;

  static void skip_ws(const std::string& s, std::size_t& p) {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\t' || s[p] == '\n' ||
                            s[p] == '\r'))
      ++p;
  }
  static void expect(const std::string& s, std::size_t& p, const char* lit) {
    for (const char* c = lit; *c; ++c, ++p)
      if (p >= s.size() || s[p] != *c) throw ParseError("bad literal");
  }
  static std::string parse_string(const std::string& s, std::size_t& p) {
    if (p >= s.size() || s[p] != '"') throw ParseError("expected string");
    ++p;
    std::string out;
    while (true) {
      if (p >= s.size()) throw ParseError("unterminated string");
      const char c = s[p++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20)
        throw ParseError("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (p >= s.size()) throw ParseError("bad escape");
      const char e = s[p++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          if (p + 4 > s.size()) throw ParseError("bad \\u escape");
          const unsigned cp =
              static_cast<unsigned>(std::stoul(s.substr(p, 4), nullptr, 16));
          p += 4;
          if (cp < 0x80) {
            out.push_back(static_cast<char>(cp));
          } else if (cp < 0x800) {
            out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          } else {
            out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
            out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
            out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
          }
          break;
        }
        default: throw ParseError("bad escape");
      }
    }
    return out;
  }
  static Value parse_value(const std::string& s, std::size_t& p, int depth) {
    if (depth > 64) throw ParseError("nesting too deep");
    skip_ws(s, p);
    if (p >= s.size()) throw ParseError("unexpected end of input");
    Value v;
    const char c = s[p];
    if (c == '{') {
      v.type_ = Type::Object;
      ++p;
      skip_ws(s, p);
      if (p < s.size() && s[p] == '}') { ++p; return v; }
      while (true) {
        skip_ws(s, p);
        std::string key = parse_string(s, p);
        skip_ws(s, p);
        if (p >= s.size() || s[p] != ':') throw ParseError("expected ':'");
        ++p;
        v.obj_[key] = parse_value(s, p, depth + 1);
        skip_ws(s, p);
        if (p < s.size() && s[p] == ',') { ++p; continue; }
        if (p < s.size() && s[p] == '}') { ++p; break; }
        throw ParseError("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.type_ = Type::Array;
      ++p;
      skip_ws(s, p);
      if (p < s.size() && s[p] == ']') { ++p; return v; }
      while (true) {
        v.arr_.push_back(parse_value(s, p, depth + 1));
        skip_ws(s, p);
        if (p < s.size() && s[p] == ',') { ++p; continue; }
        if (p < s.size() && s[p] == ']') { ++p; break; }
        throw ParseError("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.type_ = Type::String;
      v.str_ = parse_string(s, p);
    } else if (c == 't') {
      expect(s, p, "true");
      v.type_ = Type::Bool;
      v.b_ = true;
    } else if (c == 'f') {
      expect(s, p, "false");
      v.type_ = Type::Bool;
    } else if (c == 'n') {
      expect(s, p, "null");
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      // JSON number grammar, then strtod for the value
      std::size_t q = p;
      if (s[q] == '-') ++q;
      if (q >= s.size() || !(s[q] >= '0' && s[q] <= '9'))
        throw ParseError("bad number");
      if (s[q] == '0') ++q; else while (q < s.size() && s[q] >= '0' && s[q] <= '9') ++q;
      if (q < s.size() && s[q] == '.') {
        ++q;
        if (q >= s.size() || !(s[q] >= '0' && s[q] <= '9')) throw ParseError("bad number");
        while (q < s.size() && s[q] >= '0' && s[q] <= '9') ++q;
      }
      if (q < s.size() && (s[q] == 'e' || s[q] == 'E')) {
        ++q;
        if (q < s.size() && (s[q] == '+' || s[q] == '-')) ++q;
        if (q >= s.size() || !(s[q] >= '0' && s[q] <= '9')) throw ParseError("bad number");
        while (q < s.size() && s[q] >= '0' && s[q] <= '9') ++q;
      }
      v.type_ = Type::Number;
      v.num_ = std::strtod(s.substr(p, q - p).c_str(), nullptr);
      p = q;
    } else {
      throw ParseError("unexpected character");
    }
    return v;
  }
};

}  // namespace json_lite
}  // namespace roundpipe
