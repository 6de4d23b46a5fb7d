// Minimal CLI11-compatible shim (the reference's vendor/CLI11.hpp is not
// shipped: proj/.gitignore:2).  Implements exactly the surface
// proj/tools/xigemm_bench.cpp uses so the reference's own evaluation CLI builds
// unchanged against this library: App (subcommands, require_subcommand,
// set_config [accepted, ignored], parse, parsed, exit), add_option for
// scalars / strings / vectors with ->delimiter(',') and ->check(PositiveNumber),
// and the ParseError / CallForHelp / ValidationError exceptions.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
    int code;
    Error(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct ParseError : Error {
    explicit ParseError(const std::string& m, int c = 2) : Error(m, c) {}
};
struct CallForHelp : ParseError {
    CallForHelp() : ParseError("help requested", 0) {}
};
struct ValidationError : ParseError {
    ValidationError(const std::string& name, const std::string& msg) : ParseError(name + ": " + msg, 2) {}
    explicit ValidationError(const std::string& msg) : ParseError(msg, 2) {}
};

struct Validator {
    std::function<std::string(const std::string&)> fn;  // "" = ok, else the error
};
inline const Validator PositiveNumber{[](const std::string& s) -> std::string {
    char* end = nullptr;
    const double v = std::strtod(s.c_str(), &end);
    return (end && *end == 0 && v > 0) ? "" : "value " + s + " not a positive number";
}};

namespace detail {
template <class T>
void convert(const std::string& s, T& out) {
    if constexpr (std::is_same_v<T, std::string>) {
        out = s;
    } else if constexpr (std::is_floating_point_v<T>) {
        out = static_cast<T>(std::stod(s));
    } else if constexpr (std::is_unsigned_v<T>) {
        out = static_cast<T>(std::stoull(s));
    } else {
        out = static_cast<T>(std::stoll(s));
    }
}
template <class T>
struct is_vector : std::false_type {};
template <class T>
struct is_vector<std::vector<T>> : std::true_type {};
}  // namespace detail

class Option {
  public:
    std::string name, desc;
    char delim = 0;
    std::vector<Validator> checks;
    std::function<void(const std::vector<std::string>&)> set;
    Option* check(const Validator& v) {
        checks.push_back(v);
        return this;
    }
    Option* delimiter(char c) {
        delim = c;
        return this;
    }
    void apply(const std::string& value) {
        std::vector<std::string> parts;
        if (delim) {
            std::stringstream ss(value);
            std::string p;
            while (std::getline(ss, p, delim)) parts.push_back(p);
        } else {
            parts.push_back(value);
        }
        for (const auto& p : parts)
            for (const auto& c : checks)
                if (auto err = c.fn(p); !err.empty()) throw ValidationError(name, err);
        try {
            set(parts);
        } catch (const std::logic_error&) {
            throw ValidationError(name, "could not convert " + value);
        }
    }
};

class App {
  public:
    explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
    App* add_subcommand(const std::string& name, const std::string& desc) {
        subs_.push_back(std::make_unique<App>(desc, name));
        return subs_.back().get();
    }
    template <class T>
    Option* add_option(const std::string& name, T& ref, const std::string& desc = "") {
        auto o = std::make_unique<Option>();
        o->name = name;
        o->desc = desc;
        T* p = &ref;
        o->set = [p](const std::vector<std::string>& vals) {
            if constexpr (detail::is_vector<T>::value) {
                p->clear();
                for (const auto& v : vals) {
                    typename T::value_type x{};
                    detail::convert(v, x);
                    p->push_back(x);
                }
            } else {
                detail::convert(vals.at(0), *p);
            }
        };
        opts_.push_back(std::move(o));
        return opts_.back().get();
    }
    void require_subcommand(int n) { require_ = n; }
    void set_config(const std::string&, const std::string&) {}
    bool parsed() const { return parsed_; }
    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        size_t i = 0;
        App* target = this;
        parsed_ = true;
        if (!subs_.empty()) {
            if (i < args.size() && (args[i] == "--help" || args[i] == "-h")) throw CallForHelp();
            if (i >= args.size()) {
                if (require_) throw ParseError("a subcommand is required");
            } else {
                target = nullptr;
                for (auto& s : subs_)
                    if (s->name_ == args[i]) target = s.get();
                if (!target) throw ParseError("unknown subcommand: " + args[i]);
                target->parsed_ = true;
                ++i;
            }
        }
        for (; i < args.size(); ++i) {
            std::string key = args[i], value;
            if (key == "--help" || key == "-h") throw CallForHelp();
            const auto eq = key.find('=');
            if (eq != std::string::npos) {
                value = key.substr(eq + 1);
                key = key.substr(0, eq);
            } else {
                if (i + 1 >= args.size()) throw ParseError(key + ": missing value");
                value = args[++i];
            }
            Option* o = nullptr;
            for (auto& x : target->opts_)
                if (x->name == key) o = x.get();
            if (!o) throw ParseError("unknown option " + key);
            o->apply(value);
        }
    }
    int exit(const Error& e) {
        if (dynamic_cast<const CallForHelp*>(&e)) {
            std::cout << desc_ << "\nsubcommands:";
            for (auto& s : subs_) std::cout << "\n  " << s->name_ << "  " << s->desc_;
            std::cout << "\n";
            return 0;
        }
        std::cerr << e.what() << "\n";
        return e.code;
    }

  private:
    std::string desc_, name_;
    int require_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<Option>> opts_;
    std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
