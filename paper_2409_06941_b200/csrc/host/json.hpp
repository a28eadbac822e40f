// Minimal JSON for the experiment config, the run-trace stream and reports
// (the reference binds nlohmann/json, which it does not ship: config.hpp:8,
// trace.hpp:6).  Objects keep insertion order so every document this library
// writes is byte-stable; integers round-trip exactly (int64), doubles are
// written with 17 significant digits.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace freeride::json {

struct Value {
  enum class Kind { Null, Bool, Int, Double, String, Array, Object };
  Kind kind = Kind::Null;
  bool b = false;
  std::int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::vector<std::pair<std::string, Value>> o;

  Value() = default;
  static Value null() { return Value(); }
  static Value boolean(bool v) { Value x; x.kind = Kind::Bool; x.b = v; return x; }
  static Value integer(std::int64_t v) { Value x; x.kind = Kind::Int; x.i = v; return x; }
  static Value number(double v) { Value x; x.kind = Kind::Double; x.d = v; return x; }
  static Value string(std::string v) { Value x; x.kind = Kind::String; x.s = std::move(v); return x; }
  static Value array() { Value x; x.kind = Kind::Array; return x; }
  static Value object() { Value x; x.kind = Kind::Object; return x; }

  bool is_null() const { return kind == Kind::Null; }
  bool is_number() const { return kind == Kind::Int || kind == Kind::Double; }
  double as_double() const { return kind == Kind::Int ? static_cast<double>(i) : d; }
  const Value* find(const std::string& key) const;
  Value& set(const std::string& key, Value v);   // object: append (or replace)
  Value& push(Value v);                          // array: append
};

// Throws freeride::SchemaError("$", ...) with the byte offset on malformed text.
Value parse(const std::string& text);
std::string dump(const Value& v);

// Typed accessors for schema checks: SchemaError(path) on a missing key or a
// wrong type (path like "$.pipeline.num_stages").
const Value& need(const Value& obj, const std::string& key, const std::string& path);
std::int64_t get_int(const Value& v, const std::string& path);
double get_number(const Value& v, const std::string& path);
const std::string& get_string(const Value& v, const std::string& path);
bool get_bool(const Value& v, const std::string& path);
const std::vector<Value>& get_array(const Value& v, const std::string& path);

}  // namespace freeride::json
