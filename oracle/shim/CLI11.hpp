// Minimal stand-in for the CLI11 single header (oracle build only).
//
// CLI11 is vendored upstream under proj/vendor/ (git-ignored, proj/.gitignore:2)
// and is absent from /root/reference. This shim implements only the surface
// proj/src/cli.cpp touches (cli.cpp:120-132,297-405): App, add_subcommand,
// require_subcommand, add_option(name, T&, desc)->required(), parse on a
// reversed argv vector, parsed(), help(), ParseError::get_exit_code().
// It lets oracle/Makefile compile the reference's cli.cpp unmodified.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& msg, int code) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

namespace detail {

template <typename T>
struct is_optional : std::false_type {};
template <typename T>
struct is_optional<std::optional<T>> : std::true_type {};

template <typename T>
void convert(const std::string& s, T& out) {
  if constexpr (is_optional<T>::value) {
    typename T::value_type v{};
    convert(s, v);
    out = v;
  } else if constexpr (std::is_same_v<T, std::string>) {
    out = s;
  } else if constexpr (std::is_floating_point_v<T>) {
    std::size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw ParseError("bad number: " + s, 106);
    out = static_cast<T>(v);
  } else if constexpr (std::is_integral_v<T> && std::is_unsigned_v<T>) {
    std::size_t pos = 0;
    const unsigned long long v = std::stoull(s, &pos);
    if (pos != s.size()) throw ParseError("bad integer: " + s, 106);
    out = static_cast<T>(v);
  } else if constexpr (std::is_integral_v<T>) {
    std::size_t pos = 0;
    const long long v = std::stoll(s, &pos);
    if (pos != s.size()) throw ParseError("bad integer: " + s, 106);
    out = static_cast<T>(v);
  } else {
    static_assert(sizeof(T) == 0, "unsupported option type");
  }
}

}  // namespace detail

class Option {
 public:
  Option(std::vector<std::string> names, std::function<void(const std::string&)> setter)
      : names_(std::move(names)), setter_(std::move(setter)) {}
  Option* required(bool r = true) { required_ = r; return this; }
  bool matches(const std::string& n) const {
    for (const auto& x : names_)
      if (x == n) return true;
    return false;
  }
  const std::string& first_name() const { return names_.front(); }
  void set(const std::string& v) {
    try {
      setter_(v);
    } catch (const ParseError&) {
      throw;
    } catch (const std::exception&) {
      throw ParseError("could not convert '" + v + "' for " + first_name(), 106);
    }
    seen_ = true;
  }
  bool required_ = false;
  bool seen_ = false;

 private:
  std::vector<std::string> names_;
  std::function<void(const std::string&)> setter_;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}

  void require_subcommand(int n) { require_sub_ = n; }

  App* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }

  template <typename T>
  Option* add_option(const std::string& spec, T& target, const std::string& = "") {
    std::vector<std::string> names;
    std::string cur;
    for (char ch : spec + ",") {
      if (ch == ',') {
        if (!cur.empty()) names.push_back(cur);
        cur.clear();
      } else {
        cur += ch;
      }
    }
    opts_.push_back(std::make_unique<Option>(
        names, [&target](const std::string& v) { detail::convert(v, target); }));
    return opts_.back().get();
  }

  bool parsed() const { return parsed_; }

  std::string help() const {
    std::string h = desc_ + "\n";
    for (const auto& s : subs_) h += "  " + s->name_ + "  " + s->desc_ + "\n";
    return h;
  }

  // CLI11 convention: the argument vector arrives reversed (last arg first).
  void parse(std::vector<std::string>& rev) {
    std::vector<std::string> args(rev.rbegin(), rev.rend());
    std::size_t i = 0;
    if (!args.empty() && (args[0] == "-h" || args[0] == "--help"))
      throw ParseError("help", 0);
    if (args.empty()) {
      if (require_sub_ > 0) throw ParseError("a subcommand is required", 106);
      return;
    }
    App* sub = nullptr;
    for (auto& s : subs_)
      if (s->name_ == args[0]) sub = s.get();
    if (!sub) throw ParseError("unknown subcommand: " + args[0], 109);
    ++i;
    sub->parsed_ = true;
    while (i < args.size()) {
      std::string a = args[i++];
      if (a == "-h" || a == "--help") throw ParseError("help", 0);
      std::string value;
      bool inline_value = false;
      if (a.rfind("--", 0) == 0) {
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
          value = a.substr(eq + 1);
          a = a.substr(0, eq);
          inline_value = true;
        }
      }
      Option* opt = nullptr;
      for (auto& o : sub->opts_)
        if (o->matches(a)) opt = o.get();
      if (!opt) throw ParseError("unexpected argument: " + a, 109);
      if (!inline_value) {
        if (i >= args.size()) throw ParseError(a + " requires a value", 106);
        value = args[i++];
      }
      opt->set(value);
    }
    for (auto& o : sub->opts_)
      if (o->required_ && !o->seen_) throw ParseError(o->first_name() + " is required", 106);
  }

 private:
  std::string desc_;
  std::string name_;
  int require_sub_ = 0;
  bool parsed_ = false;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI
