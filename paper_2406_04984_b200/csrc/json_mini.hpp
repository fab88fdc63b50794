// Minimal JSON value for the MEFT1 checkpoint header: parse, and dump compactly with object keys sorted (the
// layout nlohmann::json::dump() produces for the reference's header, so headers match byte for byte).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace meft_json {

struct ParseError : std::runtime_error {
    explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};

struct Value {
    enum Kind { Null, Bool, Int, Real, Str, Arr, Obj } kind = Null;
    bool b = false;
    std::int64_t i = 0;
    double r = 0.0;
    std::string s;
    std::vector<Value> a;
    std::map<std::string, Value> o;

    static Value integer(std::int64_t v) {
        Value x;
        x.kind = Int;
        x.i = v;
        return x;
    }
    static Value string(const std::string& v) {
        Value x;
        x.kind = Str;
        x.s = v;
        return x;
    }
    static Value boolean(bool v) {
        Value x;
        x.kind = Bool;
        x.b = v;
        return x;
    }
    static Value object() {
        Value x;
        x.kind = Obj;
        return x;
    }
    bool has(const std::string& k) const { return kind == Obj && o.count(k); }
    const Value& at(const std::string& k) const { return o.at(k); }
};

class Parser {
  public:
    explicit Parser(const std::string& text) : t_(text) {}
    Value parse() {
        Value v = value();
        ws();
        if (p_ != t_.size()) fail("trailing characters");
        return v;
    }

  private:
    [[noreturn]] void fail(const std::string& why) { throw ParseError("json: " + why + " at offset " + std::to_string(p_)); }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
    }
    bool eat(char c) {
        ws();
        if (p_ < t_.size() && t_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    std::string str() {
        expect('"');
        std::string out;
        while (p_ < t_.size() && t_[p_] != '"') {
            char c = t_[p_++];
            if (c == '\\') {
                if (p_ >= t_.size()) fail("bad escape");
                const char e = t_[p_++];
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
                        if (p_ + 4 > t_.size()) fail("bad \\u escape");
                        const unsigned cp = unsigned(std::stoul(t_.substr(p_, 4), nullptr, 16));
                        p_ += 4;
                        if (cp < 0x80) out += char(cp);
                        else if (cp < 0x800) {
                            out += char(0xC0 | (cp >> 6));
                            out += char(0x80 | (cp & 0x3F));
                        } else {
                            out += char(0xE0 | (cp >> 12));
                            out += char(0x80 | ((cp >> 6) & 0x3F));
                            out += char(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: fail("bad escape");
                }
            } else {
                out += c;
            }
        }
        if (p_ >= t_.size()) fail("unterminated string");
        ++p_;
        return out;
    }
    Value value() {
        ws();
        if (p_ >= t_.size()) fail("unexpected end");
        const char c = t_[p_];
        Value v;
        if (c == '{') {
            ++p_;
            v.kind = Value::Obj;
            if (eat('}')) return v;
            do {
                ws();
                std::string k = str();
                expect(':');
                v.o[k] = value();
            } while (eat(','));
            expect('}');
        } else if (c == '[') {
            ++p_;
            v.kind = Value::Arr;
            if (eat(']')) return v;
            do v.a.push_back(value());
            while (eat(','));
            expect(']');
        } else if (c == '"') {
            v.kind = Value::Str;
            v.s = str();
        } else if (t_.compare(p_, 4, "true") == 0) {
            p_ += 4;
            v = Value::boolean(true);
        } else if (t_.compare(p_, 5, "false") == 0) {
            p_ += 5;
            v = Value::boolean(false);
        } else if (t_.compare(p_, 4, "null") == 0) {
            p_ += 4;
        } else {
            const size_t s0 = p_;
            if (t_[p_] == '-') ++p_;
            bool real = false;
            while (p_ < t_.size() && (isdigit(static_cast<unsigned char>(t_[p_])) || t_[p_] == '.' || t_[p_] == 'e' ||
                                      t_[p_] == 'E' || t_[p_] == '+' || t_[p_] == '-')) {
                real |= (t_[p_] == '.' || t_[p_] == 'e' || t_[p_] == 'E');
                ++p_;
            }
            const std::string num = t_.substr(s0, p_ - s0);
            if (num.empty() || num == "-") fail("bad token");
            if (real) {
                v.kind = Value::Real;
                v.r = std::stod(num);
            } else {
                v.kind = Value::Int;
                v.i = std::stoll(num);
            }
        }
        return v;
    }
    const std::string& t_;
    size_t p_ = 0;
};

inline void dump_string(const std::string& s, std::string& out) {
    out += '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    out += buf;
                } else {
                    out += char(c);
                }
        }
    }
    out += '"';
}

inline void dump(const Value& v, std::string& out) {
    switch (v.kind) {
        case Value::Null: out += "null"; break;
        case Value::Bool: out += v.b ? "true" : "false"; break;
        case Value::Int: out += std::to_string(v.i); break;
        case Value::Real: {
            char buf[40];
            std::snprintf(buf, sizeof buf, "%.17g", v.r);
            std::string s = buf;
            if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
            out += s;
            break;
        }
        case Value::Str: dump_string(v.s, out); break;
        case Value::Arr: {
            out += '[';
            for (size_t k = 0; k < v.a.size(); ++k) {
                if (k) out += ',';
                dump(v.a[k], out);
            }
            out += ']';
            break;
        }
        case Value::Obj: {
            out += '{';
            bool first = true;
            for (const auto& kv : v.o) {
                if (!first) out += ',';
                first = false;
                dump_string(kv.first, out);
                out += ':';
                dump(kv.second, out);
            }
            out += '}';
            break;
        }
    }
}

inline std::string dump(const Value& v) {
    std::string s;
    dump(v, s);
    return s;
}

}  // namespace meft_json
