// tests/cpp/stub/CLI11.hpp — TEST INFRASTRUCTURE ONLY.
//
// The reference's CLI (proj/tools/main.cpp:5) includes CLI11, a third-party
// single-header argument parser (version not pinned by the reference: no
// vendor copy, no lockfile) that is absent from this image.  This is a small
// restatement of the subset of its public API main.cpp calls — App,
// require_subcommand, add_subcommand, add_option(name, std::string&),
// add_flag(name, bool&), add_option_function<std::string>, parsed(), and the
// CLI11_PARSE macro — so that main.cpp compiles UNCHANGED and runs, both
// against the reference's own sources and against the B200 drop-in headers
// (tests/test_reference_callers.py).  Semantics kept: options take the next
// argument (or "--name=value"), flags take none, exactly one subcommand when
// required, unknown arguments are an error (exit code 109 like CLI11's
// ExtrasError), --help prints the descriptions and exits 0.
#pragma once

#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

namespace CLI {

struct ParseExit {
  int code;
};

class App {
 public:
  explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

  App* require_subcommand(int n) {
    require_ = n;
    return this;
  }

  App* add_subcommand(const std::string& name, const std::string& description) {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }

  App* add_option(const std::string& name, std::string& target, const std::string& description = "") {
    opts_.push_back({name, description, true, [&target](const std::string& v) { target = v; }});
    return this;
  }

  App* add_flag(const std::string& name, bool& target, const std::string& description = "") {
    opts_.push_back({name, description, false, [&target](const std::string&) { target = true; }});
    return this;
  }

  template <class T>
  App* add_option_function(const std::string& name, std::function<void(const T&)> fn,
                           const std::string& description = "") {
    opts_.push_back({name, description, true, [fn](const std::string& v) { fn(v); }});
    return this;
  }

  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    size_t i = 0;
    parse_into(args, i);
    if (i != args.size()) fail("The following argument was not expected: " + args[i]);
  }

 private:
  struct Opt {
    std::string name, desc;
    bool takes_value;
    std::function<void(const std::string&)> apply;
  };

  [[noreturn]] static void fail(const std::string& msg) {
    std::cerr << msg << "\nRun with --help for more information.\n";
    throw ParseExit{109};
  }

  void help() const {
    std::cout << desc_ << "\nUsage: " << (name_.empty() ? "d4orm" : name_) << " [OPTIONS]"
              << (subs_.empty() ? "" : " SUBCOMMAND") << "\n";
    for (const auto& o : opts_) std::cout << "  " << o.name << (o.takes_value ? " TEXT" : "") << "  " << o.desc << "\n";
    for (const auto& s : subs_) std::cout << "  " << s->name_ << "  " << s->desc_ << "\n";
    throw ParseExit{0};
  }

  void parse_into(const std::vector<std::string>& args, size_t& i) {
    parsed_ = true;
    int subs_seen = 0;
    while (i < args.size()) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") help();
      if (a.rfind("-", 0) == 0) {
        std::string key = a, val;
        const size_t eq = a.find('=');
        const bool inline_val = eq != std::string::npos;
        if (inline_val) key = a.substr(0, eq), val = a.substr(eq + 1);
        const Opt* hit = nullptr;
        for (const auto& o : opts_)
          if (o.name == key) hit = &o;
        if (!hit) return;  // not ours: the caller reports it
        ++i;
        if (hit->takes_value && !inline_val) {
          if (i >= args.size()) fail(key + " requires an argument");
          val = args[i++];
        }
        hit->apply(val);
        continue;
      }
      App* sub = nullptr;
      for (const auto& s : subs_)
        if (s->name_ == a) sub = s.get();
      if (!sub || subs_seen >= (require_ > 0 ? require_ : 1)) return;
      ++i;
      ++subs_seen;
      sub->parse_into(args, i);
    }
    if (require_ > 0 && subs_seen < require_) fail("A subcommand is required");
  }

  std::string desc_, name_;
  int require_ = 0;
  bool parsed_ = false;
  std::vector<Opt> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI

#define CLI11_PARSE(app, argc, argv)        \
  try {                                     \
    (app).parse((argc), (argv));            \
  } catch (const CLI::ParseExit& e__) {     \
    return e__.code;                        \
  }
