#include "json.hpp"

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "freeride.hpp"

namespace freeride::json {

const Value* Value::find(const std::string& key) const {
  for (const auto& kv : o)
    if (kv.first == key) return &kv.second;
  return nullptr;
}

Value& Value::set(const std::string& key, Value v) {
  for (auto& kv : o)
    if (kv.first == key) return kv.second = std::move(v);
  o.emplace_back(key, std::move(v));
  return o.back().second;
}

Value& Value::push(Value v) {
  a.push_back(std::move(v));
  return a.back();
}

namespace {

struct Parser {
  const std::string& t;
  std::size_t p = 0;
  [[noreturn]] void fail(const std::string& what) const {
    throw SchemaError("$", "JSON parse error at byte " + std::to_string(p) + ": " + what);
  }
  void ws() {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < t.size() && t[p] == c) {
      ++p;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  std::string str() {
    ws();
    if (p >= t.size() || t[p] != '"') fail("expected a string");
    ++p;
    std::string out;
    while (p < t.size() && t[p] != '"') {
      char c = t[p++];
      if (c == '\\') {
        if (p >= t.size()) fail("bad escape");
        const char e = t[p++];
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
            if (p + 4 > t.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(t.substr(p, 4).c_str(), nullptr, 16));
            p += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (p >= t.size()) fail("unterminated string");
    ++p;
    return out;
  }
  Value value() {
    ws();
    if (p >= t.size()) fail("unexpected end");
    const char c = t[p];
    if (c == '{') {
      ++p;
      Value v = Value::object();
      if (eat('}')) return v;
      do {
        std::string k = str();
        expect(':');
        v.o.emplace_back(std::move(k), value());
      } while (eat(','));
      expect('}');
      return v;
    }
    if (c == '[') {
      ++p;
      Value v = Value::array();
      if (eat(']')) return v;
      do v.a.push_back(value());
      while (eat(','));
      expect(']');
      return v;
    }
    if (c == '"') return Value::string(str());
    if (t.compare(p, 4, "true") == 0) return p += 4, Value::boolean(true);
    if (t.compare(p, 5, "false") == 0) return p += 5, Value::boolean(false);
    if (t.compare(p, 4, "null") == 0) return p += 4, Value::null();
    const std::size_t b = p;
    bool integral = true;
    if (t[p] == '-') ++p;
    while (p < t.size() && std::isdigit(static_cast<unsigned char>(t[p]))) ++p;
    if (p < t.size() && (t[p] == '.' || t[p] == 'e' || t[p] == 'E')) {
      integral = false;
      ++p;
      while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '+' ||
                              t[p] == '-' || t[p] == 'e' || t[p] == 'E'))
        ++p;
    }
    if (p == b || (p == b + 1 && t[b] == '-')) fail("unexpected character");
    const std::string num = t.substr(b, p - b);
    if (integral) {
      errno = 0;
      const long long v = std::strtoll(num.c_str(), nullptr, 10);
      if (errno == 0) return Value::integer(v);
    }
    return Value::number(std::strtod(num.c_str(), nullptr));
  }
};

void dump_str(const std::string& s, std::string& out) {
  out += '"';
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", static_cast<unsigned>(c));
          out += buf;
        } else {
          out += c;
        }
    }
  }
  out += '"';
}

void dump_to(const Value& v, std::string& out) {
  switch (v.kind) {
    case Value::Kind::Null: out += "null"; break;
    case Value::Kind::Bool: out += v.b ? "true" : "false"; break;
    case Value::Kind::Int: out += std::to_string(v.i); break;
    case Value::Kind::Double: {
      if (!std::isfinite(v.d)) {
        out += "null";
        break;
      }
      char buf[40];
      std::snprintf(buf, sizeof(buf), "%.17g", v.d);
      std::string s(buf);
      if (s.find_first_of(".eE") == std::string::npos) s += ".0";  // stays a double on re-read
      out += s;
      break;
    }
    case Value::Kind::String: dump_str(v.s, out); break;
    case Value::Kind::Array:
      out += '[';
      for (std::size_t k = 0; k < v.a.size(); ++k) {
        if (k) out += ',';
        dump_to(v.a[k], out);
      }
      out += ']';
      break;
    case Value::Kind::Object:
      out += '{';
      for (std::size_t k = 0; k < v.o.size(); ++k) {
        if (k) out += ',';
        dump_str(v.o[k].first, out);
        out += ':';
        dump_to(v.o[k].second, out);
      }
      out += '}';
      break;
  }
}

}  // namespace

Value parse(const std::string& text) {
  Parser ps{text};
  Value v = ps.value();
  ps.ws();
  if (ps.p != text.size()) ps.fail("trailing characters");
  return v;
}

std::string dump(const Value& v) {
  std::string out;
  dump_to(v, out);
  return out;
}

const Value& need(const Value& obj, const std::string& key, const std::string& path) {
  if (obj.kind != Value::Kind::Object) throw SchemaError(path, "expected an object");
  const Value* v = obj.find(key);
  if (!v) throw SchemaError(path + "." + key, "missing key");
  return *v;
}

std::int64_t get_int(const Value& v, const std::string& path) {
  if (v.kind == Value::Kind::Int) return v.i;
  if (v.kind == Value::Kind::Double && std::floor(v.d) == v.d && std::fabs(v.d) < 9.0e15)
    return static_cast<std::int64_t>(v.d);
  throw SchemaError(path, "expected an integer");
}

double get_number(const Value& v, const std::string& path) {
  if (!v.is_number()) throw SchemaError(path, "expected a number");
  return v.as_double();
}

const std::string& get_string(const Value& v, const std::string& path) {
  if (v.kind != Value::Kind::String) throw SchemaError(path, "expected a string");
  return v.s;
}

bool get_bool(const Value& v, const std::string& path) {
  if (v.kind != Value::Kind::Bool) throw SchemaError(path, "expected a boolean");
  return v.b;
}

const std::vector<Value>& get_array(const Value& v, const std::string& path) {
  if (v.kind != Value::Kind::Array) throw SchemaError(path, "expected an array");
  return v.a;
}

}  // namespace freeride::json
