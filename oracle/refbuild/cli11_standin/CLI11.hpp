// CLI11.hpp STAND-IN — TEST INFRASTRUCTURE ONLY (oracle/refbuild).
//
// The reference's command-line tool (proj/tools/gwgrid_main.cpp) parses its
// arguments with CLI11, which the reference does not commit
// (proj/README.md:41-43) and this image does not have.  This is our own small
// parser for exactly the CLI11 calls that file makes — App, add_subcommand,
// require_subcommand, add_option (arithmetic, string, path, optional<T>,
// vector<T> with ->delimiter), add_flag, ->required, ->check(IsMember),
// parse / ParseError / exit, operator bool — with CLI11's conventions
// (--name value or --name=value, --help exits 0, any parse problem is a
// ParseError with a non-zero exit code), so that the UNMODIFIED tool builds
// where it lies (oracle/refbuild/Makefile -> oracle/_ref/gwgrid).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <limits>
#include <memory>
#include <optional>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& what, int code) : std::runtime_error(what), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};
class CallForHelp : public ParseError {
 public:
  CallForHelp() : ParseError("help requested", 0) {}
};

class IsMember {
 public:
  IsMember(std::initializer_list<const char*> values) {
    for (const char* v : values) set_.insert(v);
  }
  std::string operator()(const std::string& value) const {
    if (set_.count(value)) return {};
    std::string all;
    for (const std::string& v : set_) all += (all.empty() ? "" : ",") + v;
    return value + " not in {" + all + "}";
  }

 private:
  std::set<std::string> set_;
};

namespace detail {

template <class T>
bool convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
    return true;
  } else if constexpr (std::is_same_v<T, std::filesystem::path>) {
    out = s;
    return true;
  } else if constexpr (std::is_same_v<T, bool>) {
    if (s == "1" || s == "true") return out = true, true;
    if (s == "0" || s == "false") return out = false, true;
    return false;
  } else if constexpr (std::is_floating_point_v<T>) {
    if (s.empty()) return false;
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    if (end != s.c_str() + s.size()) return false;
    out = static_cast<T>(v);
    return true;
  } else if constexpr (std::is_unsigned_v<T>) {
    if (s.empty() || s[0] == '-') return false;
    char* end = nullptr;
    const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
    if (end != s.c_str() + s.size() || v > std::numeric_limits<T>::max()) return false;
    out = static_cast<T>(v);
    return true;
  } else {
    static_assert(std::is_integral_v<T>, "eli11 stand-in: unsupported option type");
    if (s.empty()) return false;
    char* end = nullptr;
    const long long v = std::strtoll(s.c_str(), &end, 10);
    if (end != s.c_str() + s.size() || v > std::numeric_limits<T>::max() ||
        v < std::numeric_limits<T>::min())
      return false;
    out = static_cast<T>(v);
    return true;
  }
}

template <class T>
struct is_vector : std::false_type {};
template <class T>
struct is_vector<std::vector<T>> : std::true_type {};
template <class T>
struct is_optional : std::false_type {};
template <class T>
struct is_optional<std::optional<T>> : std::true_type {};

}  // namespace detail

class Option {
 public:
  std::string name, description;
  bool is_flag = false, required_ = false, seen = false;
  char delimiter_ = '\0';
  std::vector<std::function<std::string(const std::string&)>> checks;
  std::function<bool(const std::vector<std::string>&)> store;

  Option* required(bool v = true) {
    required_ = v;
    return this;
  }
  Option* delimiter(char c) {
    delimiter_ = c;
    return this;
  }
  template <class V>
  Option* check(V validator) {
    checks.emplace_back([validator](const std::string& s) { return validator(s); });
    return this;
  }
  std::size_t count() const { return seen ? 1 : 0; }
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "")
      : description_(std::move(description)), name_(std::move(name)) {}

  template <class T>
  Option* add_option(const std::string& name, T& variable, const std::string& description = "") {
    Option* o = add(name, description);
    o->store = [&variable, o](const std::vector<std::string>& values) {
      if constexpr (detail::is_vector<T>::value) {
        variable.clear();
        for (const std::string& raw : values) {
          std::vector<std::string> parts;
          if (o->delimiter_ != '\0') {
            std::stringstream ss(raw);
            std::string item;
            while (std::getline(ss, item, o->delimiter_)) parts.push_back(item);
          } else {
            parts.push_back(raw);
          }
          for (const std::string& part : parts) {
            typename T::value_type v{};
            if (!detail::convert(part, v)) return false;
            variable.push_back(v);
          }
        }
        return !variable.empty();
      } else if constexpr (detail::is_optional<T>::value) {
        typename T::value_type v{};
        if (values.size() != 1 || !detail::convert(values[0], v)) return false;
        variable = v;
        return true;
      } else {
        return values.size() == 1 && detail::convert(values[0], variable);
      }
    };
    return o;
  }

  Option* add_flag(const std::string& name, bool& variable, const std::string& description = "") {
    Option* o = add(name, description);
    o->is_flag = true;
    o->store = [&variable](const std::vector<std::string>&) {
      variable = true;
      return true;
    };
    return o;
  }

  App* add_subcommand(const std::string& name, const std::string& description = "") {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }
  App* require_subcommand(int n = 1) {
    required_subcommands_ = n;
    return this;
  }

  explicit operator bool() const { return parsed_; }
  bool parsed() const { return parsed_; }

  void parse(int argc, const char* const* argv) {
    std::vector<std::string> args;
    for (int i = 1; i < argc; ++i) args.emplace_back(argv[i]);
    std::size_t pos = 0;
    parse_from(args, pos);
    if (pos != args.size()) throw ParseError("unexpected argument " + args[pos], 109);
  }

  int exit(const ParseError& e, std::ostream& out = std::cout, std::ostream& err = std::cerr) const {
    if (e.get_exit_code() == 0) {
      out << help();
      return 0;
    }
    err << e.what() << "\n" << "Run with --help for more information.\n";
    return e.get_exit_code();
  }

  std::string help() const {
    std::ostringstream os;
    os << description_ << "\nOptions:\n  -h,--help\n";
    for (const auto& o : options_) os << "  " << o->name << "  " << o->description << "\n";
    if (!subs_.empty()) os << "Subcommands:\n";
    for (const auto& s : subs_) os << "  " << s->name_ << "  " << s->description_ << "\n";
    return os.str();
  }

 private:
  Option* add(const std::string& name, const std::string& description) {
    options_.push_back(std::make_unique<Option>());
    options_.back()->name = name;
    options_.back()->description = description;
    return options_.back().get();
  }

  void parse_from(const std::vector<std::string>& args, std::size_t& pos) {
    parsed_ = true;
    int subcommands_seen = 0;
    while (pos < args.size()) {
      const std::string& tok = args[pos];
      if (tok == "-h" || tok == "--help") throw CallForHelp();
      if (tok.size() > 1 && tok[0] == '-') {
        std::string key = tok, inline_value;
        bool has_inline = false;
        const auto eq = tok.find('=');
        if (tok.rfind("--", 0) == 0 && eq != std::string::npos) {
          key = tok.substr(0, eq);
          inline_value = tok.substr(eq + 1);
          has_inline = true;
        }
        Option* o = find(key);
        if (!o) throw ParseError("The following argument was not expected: " + tok, 109);
        ++pos;
        std::vector<std::string> values;
        if (o->is_flag) {
          if (has_inline) throw ParseError(key + " takes no value", 109);
        } else if (has_inline) {
          values.push_back(inline_value);
        } else {
          if (pos >= args.size()) throw ParseError(key + ": 1 required value missing", 114);
          values.push_back(args[pos++]);
        }
        for (const std::string& v : values)
          for (const auto& chk : o->checks) {
            const std::string problem = chk(v);
            if (!problem.empty()) throw ParseError(key + ": " + problem, 105);
          }
        if (!o->store(values)) throw ParseError("Could not convert: " + key + " = " + (values.empty() ? "" : values[0]), 104);
        o->seen = true;
        continue;
      }
      App* sub = nullptr;
      for (const auto& s : subs_)
        if (s->name_ == tok) sub = s.get();
      if (!sub) break;  // a positional nobody takes: the caller reports it
      ++pos;
      ++subcommands_seen;
      sub->parse_from(args, pos);
    }
    for (const auto& o : options_)
      if (o->required_ && !o->seen) throw ParseError(o->name + " is required", 106);
    if (required_subcommands_ > 0 && subcommands_seen != required_subcommands_)
      throw ParseError("A subcommand is required", 106);
  }

  Option* find(const std::string& key) const {
    for (const auto& o : options_)
      if (o->name == key) return o.get();
    return nullptr;
  }

  std::string description_, name_;
  std::vector<std::unique_ptr<Option>> options_;
  std::vector<std::unique_ptr<App>> subs_;
  int required_subcommands_ = 0;
  bool parsed_ = false;
};

}  // namespace CLI
