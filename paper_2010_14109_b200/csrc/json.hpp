// Minimal JSON reader for graph documents and op descriptors (RFC 8259
// subset: objects, arrays, strings with escapes, numbers, true/false/null).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace oc {

struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  double num = 0;
  bool is_int = false;
  int64_t i = 0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;  // insertion order kept

  const JVal* get(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  int64_t geti(const std::string& k, int64_t dflt = 0) const {
    const JVal* v = get(k);
    if (!v || v->kind != NUM) return dflt;
    return v->is_int ? v->i : (int64_t)v->num;
  }
  double getd(const std::string& k, double dflt = 0) const {
    const JVal* v = get(k);
    if (!v || v->kind != NUM) return dflt;
    return v->num;
  }
  bool getb(const std::string& k, bool dflt = false) const {
    const JVal* v = get(k);
    if (!v || v->kind != BOOL) return dflt;
    return v->b;
  }
  std::string gets(const std::string& k, const std::string& dflt = "") const {
    const JVal* v = get(k);
    if (!v || v->kind != STR) return dflt;
    return v->s;
  }
};

class JParser {
 public:
  JParser(const char* p, size_t n) : p_(p), end_(p + n) {}
  bool parse(JVal& out, std::string& err) {
    try {
      ws();
      value(out);
      ws();
      if (p_ != end_) throw std::string("trailing characters");
      return true;
    } catch (const std::string& e) {
      err = e;
      return false;
    }
  }

 private:
  const char* p_;
  const char* end_;
  void ws() {
    while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  char peek() {
    if (p_ >= end_) throw std::string("unexpected end of input");
    return *p_;
  }
  void expect(char c) {
    if (peek() != c) throw std::string("expected '") + c + "'";
    ++p_;
  }
  void lit(const char* w) {
    for (const char* q = w; *q; ++q) {
      if (p_ >= end_ || *p_ != *q) throw std::string("bad literal");
      ++p_;
    }
  }
  void value(JVal& v) {
    char c = peek();
    if (c == '{') {
      v.kind = JVal::OBJ;
      ++p_;
      ws();
      if (peek() == '}') { ++p_; return; }
      for (;;) {
        ws();
        JVal k;
        if (peek() != '"') throw std::string("expected key string");
        str(k.s);
        ws();
        expect(':');
        ws();
        JVal val;
        value(val);
        v.obj.emplace_back(std::move(k.s), std::move(val));
        ws();
        if (peek() == ',') { ++p_; continue; }
        expect('}');
        return;
      }
    } else if (c == '[') {
      v.kind = JVal::ARR;
      ++p_;
      ws();
      if (peek() == ']') { ++p_; return; }
      for (;;) {
        ws();
        JVal e;
        value(e);
        v.arr.push_back(std::move(e));
        ws();
        if (peek() == ',') { ++p_; continue; }
        expect(']');
        return;
      }
    } else if (c == '"') {
      v.kind = JVal::STR;
      str(v.s);
    } else if (c == 't') {
      lit("true"); v.kind = JVal::BOOL; v.b = true;
    } else if (c == 'f') {
      lit("false"); v.kind = JVal::BOOL; v.b = false;
    } else if (c == 'n') {
      lit("null"); v.kind = JVal::NUL;
    } else {
      num(v);
    }
  }
  void str(std::string& out) {
    expect('"');
    while (true) {
      char c = peek();
      ++p_;
      if (c == '"') return;
      if ((unsigned char)c < 0x20) throw std::string("control character in string");
      if (c != '\\') { out.push_back(c); continue; }
      char e = peek();
      ++p_;
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
          if (end_ - p_ < 4) throw std::string("bad \\u escape");
          unsigned cp = (unsigned)strtoul(std::string(p_, 4).c_str(), nullptr, 16);
          p_ += 4;
          if (cp < 0x80) out.push_back((char)cp);
          else if (cp < 0x800) { out.push_back((char)(0xC0 | (cp >> 6))); out.push_back((char)(0x80 | (cp & 0x3F))); }
          else { out.push_back((char)(0xE0 | (cp >> 12))); out.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
                 out.push_back((char)(0x80 | (cp & 0x3F))); }
          break;
        }
        default: throw std::string("bad escape");
      }
    }
  }
  void num(JVal& v) {
    const char* s = p_;
    bool frac = false;
    if (p_ < end_ && *p_ == '-') ++p_;
    if (p_ >= end_ || !((*p_ >= '0' && *p_ <= '9'))) throw std::string("bad value");
    while (p_ < end_ && ((*p_ >= '0' && *p_ <= '9') || *p_ == '.' || *p_ == 'e' || *p_ == 'E' ||
                         *p_ == '+' || *p_ == '-')) {
      if (*p_ == '.' || *p_ == 'e' || *p_ == 'E') frac = true;
      ++p_;
    }
    std::string t(s, p_);
    v.kind = JVal::NUM;
    v.num = strtod(t.c_str(), nullptr);
    if (!frac) {
      v.is_int = true;
      v.i = strtoll(t.c_str(), nullptr, 10);
    }
  }
};

}  // namespace oc
