// Minimal JSON value for the MEFT1 checkpoint header: parse, and dump compactly with object keys sorted (the
// layout nlohmann::json::dump() produces for the reference's header, so headers match byte for byte).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
    unsigned hex4() {  // the 4 hex digits of a \u escape
        if (p_ + 4 > t_.size()) fail("bad \\u escape");
        unsigned v = 0;
        for (int i = 0; i < 4; ++i) {
            const char h = t_[p_++];
            v <<= 4;
            if (h >= '0' && h <= '9') v |= unsigned(h - '0');
            else if (h >= 'a' && h <= 'f') v |= unsigned(h - 'a' + 10);
            else if (h >= 'A' && h <= 'F') v |= unsigned(h - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
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
                        unsigned cp = hex4();
                        if (cp >= 0xD800 && cp <= 0xDBFF) {  // high surrogate: must pair with \uDC00-\uDFFF
                            if (p_ + 2 > t_.size() || t_[p_] != '\\' || t_[p_ + 1] != 'u')
                                fail("unpaired UTF-16 surrogate");
                            p_ += 2;
                            const unsigned lo = hex4();
                            if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired UTF-16 surrogate");
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                            fail("unpaired UTF-16 surrogate");
                        }
                        if (cp < 0x80) {
                            out += char(cp);
                        } else if (cp < 0x800) {
                            out += char(0xC0 | (cp >> 6));
                            out += char(0x80 | (cp & 0x3F));
                        } else if (cp < 0x10000) {
                            out += char(0xE0 | (cp >> 12));
                            out += char(0x80 | ((cp >> 6) & 0x3F));
                            out += char(0x80 | (cp & 0x3F));
                        } else {
                            out += char(0xF0 | (cp >> 18));
                            out += char(0x80 | ((cp >> 12) & 0x3F));
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
            if (real) {  // strtod, not stod: subnormals (e.g. 5e-324) are valid JSON numbers, not range errors
                v.kind = Value::Real;
                char* end = nullptr;
                v.r = std::strtod(num.c_str(), &end);
                if (end != num.c_str() + num.size()) fail("bad number");
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

// Reals as nlohmann/json writes them (the reference's checkpoint headers): the shortest digit string that reads
// back to the same double, laid out by its rules -- fixed notation for decimal exponents in (-4, 15] ("0.001",
// "100.0", "1.5"), otherwise d[.ddd]e+XX with at least two exponent digits ("1e-05"); non-finite values are null.
inline void dump_real(double x, std::string& out) {
    if (!std::isfinite(x)) {
        out += "null";
        return;
    }
    if (x == 0.0) {
        out += std::signbit(x) ? "-0.0" : "0.0";
        return;
    }
    char buf[40];
    int prec = 1;
    for (; prec <= 17; ++prec) {  // shortest %.{p-1}e that round-trips
        std::snprintf(buf, sizeof buf, "%.*e", prec - 1, x);
        if (std::strtod(buf, nullptr) == x) break;
    }
    // buf = [-]d[.ddd]e(+|-)XX: collect the digits and the decimal exponent
    std::string digits;
    const char* q = buf;
    if (*q == '-') {
        out += '-';
        ++q;
    }
    for (; *q && *q != 'e'; ++q)
        if (*q != '.') digits += *q;
    const int e10 = std::atoi(q + 1);
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = int(digits.size());
    const int n = e10 + 1;  // x = 0.digits * 10^n
    if (k <= n && n <= 15) {
        out += digits + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(size_t(-n), '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[8];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
}

inline void dump(const Value& v, std::string& out) {
    switch (v.kind) {
        case Value::Null: out += "null"; break;
        case Value::Bool: out += v.b ? "true" : "false"; break;
        case Value::Int: out += std::to_string(v.i); break;
        case Value::Real: dump_real(v.r, out); break;
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
