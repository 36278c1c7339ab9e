// A small JSON reader for the model-format files the HF loader parses (config.json, the
// safetensors header, tokenizer.json).  RFC 8259 values; strings are returned as UTF-8
// (\uXXXX escapes and surrogate pairs decoded).  Errors throw nc::Error(NC_ERR_FORMAT).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "nc_internal.hpp"

namespace nc {

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;   // in file order (tokenizer.json vocab order matters not)

  const Json *get(const std::string &k) const {
    if (kind != Obj) return nullptr;
    for (const auto &kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Json &at(const std::string &k) const {
    const Json *j = get(k);
    if (!j) fail(NC_ERR_FORMAT, "JSON: missing key '" + k + "'");
    return *j;
  }
  double number() const {
    if (kind != Num) fail(NC_ERR_FORMAT, "JSON: number expected");
    return num;
  }
  const std::string &string() const {
    if (kind != Str) fail(NC_ERR_FORMAT, "JSON: string expected");
    return str;
  }

  static Json parse(const char *p, size_t n) {
    Parser ps{p, p + n};
    ps.ws();
    Json j = ps.value(0);
    ps.ws();
    if (ps.p != ps.e) fail(NC_ERR_FORMAT, "JSON: trailing characters");
    return j;
  }

 private:
  struct Parser {
    const char *p, *e;
    void ws() {
      while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    [[noreturn]] void bad(const char *w) { fail(NC_ERR_FORMAT, std::string("JSON: ") + w); }
    char peek() { return p < e ? *p : '\0'; }
    void expect(char c) {
      if (p >= e || *p != c) bad("unexpected character");
      ++p;
    }
    static void utf8(std::string &o, uint32_t cp) {
      if (cp < 0x80) o += (char)cp;
      else if (cp < 0x800) { o += (char)(0xC0 | (cp >> 6)); o += (char)(0x80 | (cp & 63)); }
      else if (cp < 0x10000) {
        o += (char)(0xE0 | (cp >> 12)); o += (char)(0x80 | ((cp >> 6) & 63)); o += (char)(0x80 | (cp & 63));
      } else {
        o += (char)(0xF0 | (cp >> 18)); o += (char)(0x80 | ((cp >> 12) & 63));
        o += (char)(0x80 | ((cp >> 6) & 63)); o += (char)(0x80 | (cp & 63));
      }
    }
    uint32_t hex4() {
      if (e - p < 4) bad("short \\u escape");
      uint32_t v = 0;
      for (int i = 0; i < 4; ++i) {
        const char c = *p++;
        v <<= 4;
        if (c >= '0' && c <= '9') v |= c - '0';
        else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
        else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
        else bad("bad \\u escape");
      }
      return v;
    }
    std::string string() {
      expect('"');
      std::string o;
      while (true) {
        if (p >= e) bad("unterminated string");
        const char c = *p++;
        if (c == '"') break;
        if (c != '\\') { o += c; continue; }
        if (p >= e) bad("bad escape");
        const char x = *p++;
        switch (x) {
          case '"': o += '"'; break;
          case '\\': o += '\\'; break;
          case '/': o += '/'; break;
          case 'b': o += '\b'; break;
          case 'f': o += '\f'; break;
          case 'n': o += '\n'; break;
          case 'r': o += '\r'; break;
          case 't': o += '\t'; break;
          case 'u': {
            uint32_t cp = hex4();
            if (cp >= 0xD800 && cp < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
              p += 2;
              const uint32_t lo = hex4();
              if (lo < 0xDC00 || lo >= 0xE000) bad("bad surrogate pair");
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            }
            utf8(o, cp);
            break;
          }
          default: bad("bad escape");
        }
      }
      return o;
    }
    Json value(int depth) {
      if (depth > 256) bad("nesting too deep");
      Json j;
      const char c = peek();
      if (c == '{') {
        ++p;
        j.kind = Obj;
        ws();
        if (peek() == '}') { ++p; return j; }
        while (true) {
          ws();
          std::string k = string();
          ws();
          expect(':');
          ws();
          j.obj.emplace_back(std::move(k), value(depth + 1));
          ws();
          if (peek() == ',') { ++p; continue; }
          expect('}');
          return j;
        }
      }
      if (c == '[') {
        ++p;
        j.kind = Arr;
        ws();
        if (peek() == ']') { ++p; return j; }
        while (true) {
          ws();
          j.arr.push_back(value(depth + 1));
          ws();
          if (peek() == ',') { ++p; continue; }
          expect(']');
          return j;
        }
      }
      if (c == '"') { j.kind = Str; j.str = string(); return j; }
      if (e - p >= 4 && std::string(p, 4) == "true") { p += 4; j.kind = Bool; j.b = true; return j; }
      if (e - p >= 5 && std::string(p, 5) == "false") { p += 5; j.kind = Bool; return j; }
      if (e - p >= 4 && std::string(p, 4) == "null") { p += 4; return j; }
      // number
      const char *q = p;
      if (q < e && (*q == '-' || *q == '+')) ++q;
      while (q < e && ((*q >= '0' && *q <= '9') || *q == '.' || *q == 'e' || *q == 'E' || *q == '-' || *q == '+')) ++q;
      if (q == p) bad("value expected");
      j.kind = Num;
      j.num = std::strtod(std::string(p, q).c_str(), nullptr);
      p = q;
      return j;
    }
  };
};

}  // namespace nc
