// Command-line layer of pactrec (the reference uses CLI11, absent here).
//
// Same user-visible contract as tools/pactrec.cpp's CLI11 set-up:
//   * a tree of subcommands, exactly one leaf selected per run;
//   * long options `--name value` / `--name=value`, boolean flags
//     `--name` / `--no-name`, vector options taking several values;
//   * precedence: command-line flag > PACT_<NAME> environment variable
//     (dashes -> underscores, upper case) > `--config` file > built-in default
//     (pactrec.cpp:26-28, 61-81);
//   * the config file is flat `key=value` (INI): `[recon.das]` sections or
//     dotted keys address subcommand options; a key for an option of the
//     selected command chain may also appear unsectioned; unknown keys are an
//     error (allow_config_extras(false));
//   * resolved() renders the final values of the selected chain in the same
//     format, loadable again with --config (the resolved_config.ini echo).
// Parse problems raise cli::ParseError (pactrec exits 2); --help raises
// cli::Help after printing the usage of the command reached so far (exit 0).
#ifndef PACTREC_CLI_ARGS_HPP
#define PACTREC_CLI_ARGS_HPP

#include <cctype>
#include <charconv>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace cli {

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Help {};

inline std::string env_name(const std::string& long_name) {
  std::string s = "PACT_";
  for (char c : long_name) s += c == '-' ? '_' : static_cast<char>(std::toupper(c));
  return s;
}

namespace conv {
inline void check_full(const char* b, const char* e, const std::string& opt, const std::string& v,
                       const char* what) {
  if (b == e || *e != '\0' || errno == ERANGE)
    throw ParseError("--" + opt + ": value '" + v + "' is not " + what);
}
inline void from(const std::string& v, int& out, const std::string& opt) {
  errno = 0;
  char* e = nullptr;
  const long x = std::strtol(v.c_str(), &e, 10);
  check_full(v.c_str(), e, opt, v, "an integer");
  if (x < INT32_MIN || x > INT32_MAX) throw ParseError("--" + opt + ": value '" + v + "' out of range");
  out = static_cast<int>(x);
}
inline void from(const std::string& v, uint64_t& out, const std::string& opt) {
  errno = 0;
  char* e = nullptr;
  if (!v.empty() && v[0] == '-') throw ParseError("--" + opt + ": value '" + v + "' is negative");
  out = std::strtoull(v.c_str(), &e, 10);
  check_full(v.c_str(), e, opt, v, "an unsigned integer");
}
inline void from(const std::string& v, double& out, const std::string& opt) {
  errno = 0;
  char* e = nullptr;
  out = std::strtod(v.c_str(), &e);
  check_full(v.c_str(), e, opt, v, "a number");
}
inline void from(const std::string& v, std::string& out, const std::string&) { out = v; }
inline void from(const std::string& v, bool& out, const std::string& opt) {
  std::string l;
  for (char c : v) l += static_cast<char>(std::tolower(c));
  if (l == "1" || l == "true" || l == "on" || l == "yes") out = true;
  else if (l == "0" || l == "false" || l == "off" || l == "no") out = false;
  else throw ParseError("--" + opt + ": value '" + v + "' is not a boolean");
}
inline std::string to(int v) { return std::to_string(v); }
inline std::string to(uint64_t v) { return std::to_string(v); }
inline std::string to(const std::string& v) { return v; }
inline std::string to(bool v) { return v ? "true" : "false"; }
inline std::string to(double v) {  // shortest text that reads back to the same double
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}
inline std::vector<std::string> split_list(const std::string& v) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : v) {
    if (c == ',' || std::isspace(static_cast<unsigned char>(c))) {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}
}  // namespace conv

enum class Source { kDefault, kConfig, kEnv, kCli };

struct Option {
  std::string name, desc, env, type, default_text;
  bool flag = false, vector = false;
  Source source = Source::kDefault;
  std::function<void(const std::string&)> set;  // one value (vector: appends)
  std::function<void()> clear;                  // vector: reset before a new source
  std::function<std::string()> get;
};

class Command {
 public:
  Command(std::string name, std::string desc, Command* parent)
      : name_(std::move(name)), desc_(std::move(desc)), parent_(parent) {}
  Command(const Command&) = delete;

  Command* add_subcommand(const std::string& name, const std::string& desc) {
    subs_.push_back(std::make_unique<Command>(name, desc, this));
    return subs_.back().get();
  }
  void require_subcommand() { need_sub_ = true; }

  template <typename T>
  Option& add(const std::string& name, T& var, const std::string& desc) {
    Option o;
    o.name = name;
    o.desc = desc;
    o.env = env_name(name);
    o.type = type_of(var);
    o.set = [&var, name](const std::string& v) { conv::from(v, var, name); };
    o.get = [&var] { return conv::to(var); };
    o.default_text = o.get();
    opts_.push_back(std::move(o));
    return opts_.back();
  }
  Option& add_flag(const std::string& name, bool& var, const std::string& desc) {
    Option& o = add(name, var, desc);
    o.flag = true;
    return o;
  }
  template <typename T>
  Option& add_vector(const std::string& name, std::vector<T>& var, const std::string& desc,
                     const std::string& env) {
    Option o;
    o.name = name;
    o.desc = desc;
    o.env = env;
    o.vector = true;
    o.type = type_of(T{}) + " ...";
    o.set = [&var, name](const std::string& v) {
      T x{};
      conv::from(v, x, name);
      var.push_back(x);
    };
    o.clear = [&var] { var.clear(); };
    o.get = [&var] {
      std::string s;
      for (size_t i = 0; i < var.size(); ++i) s += (i ? " " : "") + conv::to(var[i]);
      return s;
    };
    opts_.push_back(std::move(o));
    return opts_.back();
  }

  explicit operator bool() const { return selected_; }
  const std::string& name() const { return name_; }
  std::string path() const {
    if (!parent_ || !parent_->parent_) return parent_ ? name_ : std::string();
    return parent_->path() + "." + name_;
  }

 protected:
  friend class App;
  static std::string type_of(int) { return "INT"; }
  static std::string type_of(uint64_t) { return "UINT"; }
  static std::string type_of(double) { return "FLOAT"; }
  static std::string type_of(bool) { return "BOOL"; }
  static std::string type_of(const std::string&) { return "TEXT"; }

  Option* find(const std::string& n) {
    for (auto& o : opts_)
      if (o.name == n) return &o;
    return nullptr;
  }
  bool has_selected_sub() const {
    for (const auto& s : subs_)
      if (s->selected_) return true;
    return false;
  }
  Command* sub(const std::string& n) {
    for (auto& s : subs_)
      if (s->name_ == n) return s.get();
    return nullptr;
  }
  std::string usage_path() const { return parent_ ? parent_->usage_path() + " " + name_ : name_; }
  void print_help(std::ostream& os) const {
    os << desc_ << "\nUsage: " << usage_path() << " [OPTIONS]" << (subs_.empty() ? "" : " SUBCOMMAND")
       << "\n";
    if (!opts_.empty()) os << "\nOptions:\n";
    os << "  -h,--help              print this help and exit\n";
    for (const auto& o : opts_) {
      std::string lhs = "  --" + o.name + (o.flag ? ",--no-" + o.name : " " + o.type);
      if (lhs.size() < 40) lhs.resize(40, ' ');
      os << lhs << " " << o.desc;
      if (!o.vector) os << " [" << o.default_text << "]";
      if (!o.env.empty()) os << " (env: " << o.env << ")";
      os << "\n";
    }
    if (!subs_.empty()) {
      os << "\nSubcommands:\n";
      for (const auto& s : subs_) {
        std::string lhs = "  " + s->name_;
        if (lhs.size() < 24) lhs.resize(24, ' ');
        os << lhs << " " << s->desc_ << "\n";
      }
    }
  }

  std::string name_, desc_;
  Command* parent_;
  std::vector<std::unique_ptr<Command>> subs_;
  std::vector<Option> opts_;
  bool need_sub_ = false, selected_ = false;
};

class App : public Command {
 public:
  App(std::string name, std::string desc) : Command(std::move(name), std::move(desc), nullptr) {}

  /// Parses argv (tokens after argv[0]), then fills unset options from the
  /// environment and the config file.  Throws ParseError / Help.
  void parse(int argc, char** argv) {
    std::vector<std::string> tok(argv + 1, argv + argc);
    std::string config_path;
    Command* cur = this;
    selected_ = true;
    chain_ = {this};
    for (size_t i = 0; i < tok.size(); ++i) {
      const std::string& t = tok[i];
      if (t == "-h" || t == "--help") {
        cur->print_help(std::cout);
        throw Help{};
      }
      if (t.rfind("--", 0) == 0) {
        std::string key = t.substr(2), val;
        const size_t eq = key.find('=');
        const bool has_val = eq != std::string::npos;
        if (has_val) {
          val = key.substr(eq + 1);
          key = key.substr(0, eq);
        }
        if (key == "config") {
          if (!has_val) {
            if (i + 1 >= tok.size()) throw ParseError("--config requires a file argument");
            val = tok[++i];
          }
          config_path = val;
          continue;
        }
        bool negated = false;
        Option* o = lookup(key);
        if (!o && key.rfind("no-", 0) == 0) {
          o = lookup(key.substr(3));
          negated = o && o->flag;
          if (!negated) o = nullptr;
        }
        if (!o) throw ParseError("The following argument was not expected: " + t);
        if (o->flag) {
          if (has_val && negated) throw ParseError("--" + key + " does not take a value");
          o->set(has_val ? val : (negated ? "false" : "true"));
        } else if (o->vector) {
          if (o->source != Source::kCli) o->clear();
          if (has_val) {
            for (const auto& v : conv::split_list(val)) o->set(v);
          } else {
            size_t n = 0;
            while (i + 1 < tok.size() && tok[i + 1].rfind("--", 0) != 0 && !cur->sub(tok[i + 1])) {
              o->set(tok[++i]);
              ++n;
            }
            if (!n) throw ParseError(t + " requires at least one value");
          }
        } else {
          if (!has_val) {
            if (i + 1 >= tok.size()) throw ParseError(t + " requires a value");
            val = tok[++i];
          }
          o->set(val);
        }
        o->source = Source::kCli;
        continue;
      }
      Command* s = cur->sub(t);
      if (!s) throw ParseError("The following argument was not expected: " + t);
      s->selected_ = true;
      cur = s;
      chain_.push_back(s);
    }
    for (Command* c : chain_)
      if (c->need_sub_ && !c->has_selected_sub())
        throw ParseError(c == this ? std::string("A subcommand is required")
                                   : "A subcommand of '" + c->name_ + "' is required");
    for (Command* c : chain_)
      for (auto& o : c->opts_) {
        if (o.source != Source::kDefault || o.env.empty()) continue;
        const char* e = std::getenv(o.env.c_str());
        if (!e) continue;
        if (o.vector) {
          o.clear();
          for (const auto& v : conv::split_list(e)) o.set(v);
        } else {
          o.set(e);
        }
        o.source = Source::kEnv;
      }
    if (!config_path.empty()) apply_config(config_path);
  }

  /// The resolved configuration of the selected command chain (INI with the
  /// option descriptions as comments).
  std::string resolved() const {
    std::ostringstream os;
    for (const Command* c : chain_) {
      if (c->opts_.empty()) continue;
      const std::string p = c->path();
      if (!p.empty()) os << "\n[" << p << "]\n";
      for (const auto& o : c->opts_) {
        os << "# " << o.desc << "\n";
        std::string v = o.get();
        if (o.type == "TEXT" || o.vector) v = "\"" + v + "\"";
        os << o.name << "=" << v << "\n";
      }
    }
    return os.str();
  }

 private:
  std::vector<Command*> chain_;

  Option* lookup(const std::string& key) {
    for (auto it = chain_.rbegin(); it != chain_.rend(); ++it)
      if (Option* o = (*it)->find(key)) return o;
    return nullptr;
  }

  static std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
    while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
    return s.substr(a, b - a);
  }

  Command* command_at(const std::string& path) {
    Command* c = this;
    size_t a = 0;
    while (a < path.size()) {
      size_t b = path.find('.', a);
      if (b == std::string::npos) b = path.size();
      c = c->sub(path.substr(a, b - a));
      if (!c) return nullptr;
      a = b + 1;
    }
    return c;
  }

  void apply_config(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw ParseError("cannot open config file " + path);
    std::string line, section;
    int lineno = 0;
    while (std::getline(is, line)) {
      ++lineno;
      line = trim(line);
      if (line.empty() || line[0] == '#' || line[0] == ';') continue;
      if (line.front() == '[') {
        if (line.back() != ']') throw ParseError(path + ":" + std::to_string(lineno) + ": bad section");
        section = trim(line.substr(1, line.size() - 2));
        if (section == "default") section.clear();
        continue;
      }
      const size_t eq = line.find('=');
      if (eq == std::string::npos)
        throw ParseError(path + ":" + std::to_string(lineno) + ": expected key=value");
      std::string key = trim(line.substr(0, eq)), val = trim(line.substr(eq + 1));
      if (val.size() >= 2 && (val.front() == '"' || val.front() == '\'') && val.back() == val.front())
        val = val.substr(1, val.size() - 2);
      std::string where = section;
      const size_t dot = key.rfind('.');
      if (dot != std::string::npos) {
        where += (where.empty() ? "" : ".") + key.substr(0, dot);
        key = key.substr(dot + 1);
      }
      Command* c = command_at(where);
      Option* o = nullptr;
      if (!c) throw ParseError("INI was not able to parse " + (where.empty() ? key : where + "." + key));
      if (where.empty()) {
        o = lookup(key);  // flat file: the selected chain, deepest first
        if (!o) o = c->find(key);
      } else {
        o = c->find(key);
      }
      if (!o || key == "help")
        throw ParseError("INI was not able to parse " + (where.empty() ? key : where + "." + key));
      if (!c->selected_ && !where.empty()) continue;  // another subcommand's setting
      if (o->source != Source::kDefault) continue;
      if (o->vector) {
        o->clear();
        for (const auto& v : conv::split_list(val)) o->set(v);
      } else {
        o->set(val);
      }
      o->source = Source::kConfig;
    }
  }
};

}  // namespace cli

#endif  // PACTREC_CLI_ARGS_HPP
