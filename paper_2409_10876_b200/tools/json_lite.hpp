// Minimal JSON reader for pactrec's phantom spec files (the reference uses
// nlohmann::json, absent here).  Parses RFC 8259 documents (objects, arrays,
// strings with escapes, numbers, true/false/null) into a tree; errors carry
// the byte offset.  Only what load_phantom_spec needs: lookups with defaults,
// required lookups and typed getters that raise one exception type.
#ifndef PACTREC_JSON_LITE_HPP
#define PACTREC_JSON_LITE_HPP

#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace jsonl {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Value {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = kNull;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // document order

  bool is_object() const { return kind == kObject; }
  bool is_array() const { return kind == kArray; }
  size_t size() const { return kind == kArray ? arr.size() : kind == kObject ? obj.size() : 0; }
  const Value* find(const std::string& key) const {
    if (kind != kObject) return nullptr;
    const Value* hit = nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) hit = &kv.second;  // last duplicate wins
    return hit;
  }
  bool contains(const std::string& key) const { return find(key) != nullptr; }
  double number(const std::string& what) const {
    if (kind != kNumber) throw Error(what + " must be a number");
    return num;
  }
  bool boolean(const std::string& what) const {
    if (kind != kBool) throw Error(what + " must be true or false");
    return b;
  }
  const Value& at(const std::string& key, const std::string& what) const {
    const Value* v = find(key);
    if (!v) throw Error("missing key '" + key + "' in " + what);
    return *v;
  }
  double number_or(const std::string& key, double dflt, const std::string& what) const {
    const Value* v = find(key);
    return v ? v->number(what + "." + key) : dflt;
  }
  bool bool_or(const std::string& key, bool dflt, const std::string& what) const {
    const Value* v = find(key);
    return v ? v->boolean(what + "." + key) : dflt;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& text) : s_(text) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;

  [[noreturn]] void fail(const std::string& why) const {
    throw Error("parse error at byte " + std::to_string(i_) + ": " + why);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r'))
      ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  bool word(const char* w) {
    size_t n = std::char_traits<char>::length(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end of input");
    Value v;
    const char c = s_[i_];
    if (c == '{') {
      ++i_;
      v.kind = Value::kObject;
      if (eat('}')) return v;
      do {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected a string key");
        std::string k = string();
        expect(':');
        v.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i_;
      v.kind = Value::kArray;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Value::kString;
      v.str = string();
    } else if (word("true")) {
      v.kind = Value::kBool;
      v.b = true;
    } else if (word("false")) {
      v.kind = Value::kBool;
    } else if (word("null")) {
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      v.kind = Value::kNumber;
      v.num = number();
    } else {
      fail(std::string("unexpected character '") + c + "'");
    }
    return v;
  }
  double number() {
    const size_t start = i_;
    auto digits = [&] {
      const size_t d0 = i_;
      while (i_ < s_.size() && s_[i_] >= '0' && s_[i_] <= '9') ++i_;
      if (i_ == d0) fail("malformed number");
    };
    if (s_[i_] == '-') ++i_;
    if (i_ < s_.size() && s_[i_] == '0')
      ++i_;
    else
      digits();
    if (i_ < s_.size() && s_[i_] == '.') {
      ++i_;
      digits();
    }
    if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
      ++i_;
      if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
      digits();
    }
    return std::strtod(s_.substr(start, i_ - start).c_str(), nullptr);
  }
  static void utf8(std::string& out, unsigned cp) {
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
    if (i_ + 4 > s_.size()) fail("short \\u escape");
    unsigned v = 0;
    for (int k = 0; k < 4; ++k) {
      const char h = s_[i_++];
      v <<= 4;
      if (h >= '0' && h <= '9') v |= h - '0';
      else if (h >= 'a' && h <= 'f') v |= h - 'a' + 10;
      else if (h >= 'A' && h <= 'F') v |= h - 'A' + 10;
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string string() {
    ++i_;  // opening quote
    std::string out;
    while (true) {
      if (i_ >= s_.size()) fail("unterminated string");
      const char c = s_[i_++];
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (i_ >= s_.size()) fail("unterminated escape");
      const char e = s_[i_++];
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
          if (cp >= 0xD800 && cp < 0xDC00 && i_ + 1 < s_.size() && s_[i_] == '\\' &&
              s_[i_ + 1] == 'u') {
            i_ += 2;
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace jsonl

#endif  // PACTREC_JSON_LITE_HPP
