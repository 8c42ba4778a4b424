// CLI11.hpp -- TEST INFRASTRUCTURE ONLY: the subset of CLI11 (not installed
// in this image) that the reference's own front end, proj/tools/binbatch_cli.cpp,
// uses, so that file builds unchanged against either the reference headers
// or the B200 drop-in.  Options are "--name value" / "--name=value" (short
// "-X value"), one subcommand, required options and simple validators;
// errors throw CLI::ParseError, which App::exit reports (exit code 106, or
// 0 for --help).
#pragma once
#include <charconv>
#include <cstdio>
#include <functional>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <sys/stat.h>
#include <type_traits>
#include <vector>

namespace CLI {

struct ParseError : std::runtime_error {
  int code;
  ParseError(const std::string& m, int c = 106) : std::runtime_error(m), code(c) {}
};

using Validator = std::function<std::string(const std::string&)>;  // "" = ok

inline const Validator PositiveNumber = [](const std::string& s) -> std::string {
  try {
    return std::stod(s) > 0 ? "" : "value must be positive: " + s;
  } catch (...) {
    return "not a number: " + s;
  }
};
inline const Validator ExistingFile = [](const std::string& s) -> std::string {
  struct stat st;
  return stat(s.c_str(), &st) == 0 && S_ISREG(st.st_mode) ? "" : "file does not exist: " + s;
};
inline Validator IsMember(std::vector<std::string> set) {
  return [set](const std::string& s) -> std::string {
    for (const auto& m : set)
      if (m == s) return "";
    return "not a member: " + s;
  };
}

namespace detail {
template <class T>
struct is_optional : std::false_type {};
template <class T>
struct is_optional<std::optional<T>> : std::true_type {};
template <class T>
struct is_vector : std::false_type {};
template <class T>
struct is_vector<std::vector<T>> : std::true_type {};

template <class T>
void convert(const std::string& s, T& out) {
  if constexpr (std::is_same_v<T, std::string>) {
    out = s;
  } else if constexpr (std::is_same_v<T, bool>) {
    out = s == "1" || s == "true";
  } else if constexpr (std::is_floating_point_v<T>) {
    size_t used = 0;
    out = static_cast<T>(std::stod(s, &used));
    if (used != s.size()) throw ParseError("not a number: " + s);
  } else {
    static_assert(std::is_integral_v<T>, "unsupported option type");
    auto r = std::from_chars(s.data(), s.data() + s.size(), out);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw ParseError("not an integer: " + s);
  }
}
}  // namespace detail

class Option {
 public:
  Option(std::string names, std::function<void(const std::string&)> set, std::function<std::string()> show)
      : set_(std::move(set)), show_(std::move(show)) {
    std::stringstream ss(names);
    for (std::string n; std::getline(ss, n, ',');) names_.push_back(n);
  }
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }
  Option* delimiter(char c) {
    delim_ = c;
    return this;
  }
  Option* capture_default_str() { return this; }
  bool matches(const std::string& n) const {
    for (const auto& m : names_)
      if (m == n) return true;
    return false;
  }
  void apply(const std::string& v) {
    if (!seen_ && reset_) reset_();
    std::vector<std::string> parts;
    if (delim_) {
      std::stringstream ss(v);
      for (std::string p; std::getline(ss, p, delim_);) parts.push_back(p);
    } else {
      parts.push_back(v);
    }
    for (const auto& p : parts) {
      for (const auto& c : checks_) {
        const std::string e = c(p);
        if (!e.empty()) throw ParseError(names_[0] + ": " + e);
      }
      set_(p);
    }
    seen_ = true;
  }
  std::string help() const { return names_[0]; }
  bool required_ = false, seen_ = false;
  std::vector<std::string> names_;
  std::function<void()> reset_;

 private:
  std::function<void(const std::string&)> set_;
  std::function<std::string()> show_;
  std::vector<Validator> checks_;
  char delim_ = 0;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  template <class T>
  Option* add_option(const std::string& names, T& var, const std::string& /*desc*/ = "") {
    auto set = [&var](const std::string& s) {
      if constexpr (detail::is_optional<T>::value) {
        typename T::value_type v{};
        detail::convert(s, v);
        var = v;
      } else if constexpr (detail::is_vector<T>::value) {
        typename T::value_type v{};
        detail::convert(s, v);
        var.push_back(v);
      } else {
        detail::convert(s, var);
      }
    };
    opts_.push_back(std::make_unique<Option>(names, set, [] { return std::string(); }));
    if constexpr (detail::is_vector<T>::value) opts_.back()->reset_ = [&var] { var.clear(); };  // given: replaces the default
    return opts_.back().get();
  }
  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  void require_subcommand(int n) { need_sub_ = n; }
  void fallthrough(bool = true) { fallthrough_ = true; }
  bool got_subcommand(const App* sub) const { return chosen_ == sub; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    App* cur = this;
    for (size_t i = 0; i < args.size(); ++i) {
      std::string a = args[i];
      if (a == "--help" || a == "-h") throw ParseError(usage(), 0);
      if (a.size() > 1 && a[0] == '-') {
        std::string val;
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
          val = a.substr(eq + 1);
          a = a.substr(0, eq);
        } else {
          if (i + 1 >= args.size()) throw ParseError(a + " needs a value");
          val = args[++i];
        }
        Option* o = cur->find(a);
        if (!o && cur != this && fallthrough_) o = find(a);
        if (!o) throw ParseError("unknown option " + a);
        o->apply(val);
        continue;
      }
      App* sub = nullptr;
      for (auto& s : subs_)
        if (s->name_ == a) sub = s.get();
      if (!sub || cur != this) throw ParseError("unexpected argument " + a);
      cur = chosen_ = sub;
    }
    if (need_sub_ && !chosen_) throw ParseError("a subcommand is required\n" + usage());
    for (App* app : {this, chosen_})
      if (app)
        for (auto& o : app->opts_)
          if (o->required_ && !o->seen_) throw ParseError(o->help() + " is required");
  }
  int exit(const ParseError& e) const {
    std::fprintf(e.code ? stderr : stdout, "%s\n", e.what());
    return e.code;
  }

 private:
  Option* find(const std::string& n) {
    for (auto& o : opts_)
      if (o->matches(n)) return o.get();
    return nullptr;
  }
  std::string usage() const {
    std::string u = desc_ + "\nsubcommands:";
    for (const auto& s : subs_) u += " " + s->name_;
    return u;
  }
  std::string desc_, name_;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
  App* chosen_ = nullptr;
  int need_sub_ = 0;
  bool fallthrough_ = false;
};

}  // namespace CLI
