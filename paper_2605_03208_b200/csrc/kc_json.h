// kc_json.h -- minimal JSON reader/writer for the kc-snapshot/1 metadata files
// (dispatch.json, memory_regions.json, capture_log.json).  Product path only.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

namespace kcj {

struct Value {
    enum Type { Null, Bool, Num, Str, Arr, Obj } t = Null;
    bool b = false;
    double d = 0.0;
    bool is_int = false;
    long long i = 0;
    unsigned long long u = 0;
    std::string s;
    std::vector<Value> a;
    std::vector<std::pair<std::string, Value>> o;

    const Value* get(const char* k) const {
        if (t != Obj) return nullptr;
        for (auto& kv : o)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
    unsigned long long as_u64(unsigned long long dflt = 0) const {
        if (t == Num) return is_int ? u : (unsigned long long)d;
        return dflt;
    }
    std::string as_str(const char* dflt = "") const { return t == Str ? s : std::string(dflt); }
};

class Parser {
   public:
    explicit Parser(const std::string& text) : p_(text.c_str()), end_(text.c_str() + text.size()) {}
    bool parse(Value& v) {
        ws();
        if (!value(v)) return false;
        ws();
        return p_ == end_;
    }

   private:
    const char* p_;
    const char* end_;
    void ws() {
        while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\t' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* w) {
        size_t n = 0;
        while (w[n]) ++n;
        if ((size_t)(end_ - p_) < n) return false;
        for (size_t i = 0; i < n; ++i)
            if (p_[i] != w[i]) return false;
        p_ += n;
        return true;
    }
    bool str(std::string& out) {
        if (p_ >= end_ || *p_ != '"') return false;
        ++p_;
        while (p_ < end_ && *p_ != '"') {
            char c = *p_++;
            if (c == '\\') {
                if (p_ >= end_) return false;
                char e = *p_++;
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (end_ - p_ < 4) return false;
                        unsigned cp = 0;
                        for (int k = 0; k < 4; ++k) {
                            char h = *p_++;
                            cp <<= 4;
                            if (h >= '0' && h <= '9') cp |= h - '0';
                            else if (h >= 'a' && h <= 'f') cp |= h - 'a' + 10;
                            else if (h >= 'A' && h <= 'F') cp |= h - 'A' + 10;
                            else return false;
                        }
                        out += cp < 0x80 ? (char)cp : '?';
                        break;
                    }
                    default: out += e; break;
                }
            } else {
                out += c;
            }
        }
        if (p_ >= end_) return false;
        ++p_;
        return true;
    }
    bool value(Value& v) {
        ws();
        if (p_ >= end_) return false;
        char c = *p_;
        if (c == '{') {
            v.t = Value::Obj;
            ++p_;
            ws();
            if (p_ < end_ && *p_ == '}') { ++p_; return true; }
            for (;;) {
                ws();
                std::string k;
                if (!str(k)) return false;
                ws();
                if (p_ >= end_ || *p_ != ':') return false;
                ++p_;
                Value x;
                if (!value(x)) return false;
                v.o.emplace_back(std::move(k), std::move(x));
                ws();
                if (p_ < end_ && *p_ == ',') { ++p_; continue; }
                if (p_ < end_ && *p_ == '}') { ++p_; return true; }
                return false;
            }
        }
        if (c == '[') {
            v.t = Value::Arr;
            ++p_;
            ws();
            if (p_ < end_ && *p_ == ']') { ++p_; return true; }
            for (;;) {
                Value x;
                if (!value(x)) return false;
                v.a.push_back(std::move(x));
                ws();
                if (p_ < end_ && *p_ == ',') { ++p_; continue; }
                if (p_ < end_ && *p_ == ']') { ++p_; return true; }
                return false;
            }
        }
        if (c == '"') { v.t = Value::Str; return str(v.s); }
        if (lit("true")) { v.t = Value::Bool; v.b = true; return true; }
        if (lit("false")) { v.t = Value::Bool; v.b = false; return true; }
        if (lit("null")) { v.t = Value::Null; return true; }
        // number
        const char* s = p_;
        bool neg = false, frac = false;
        if (*p_ == '-') { neg = true; ++p_; }
        while (p_ < end_ && ((*p_ >= '0' && *p_ <= '9') || *p_ == '.' || *p_ == 'e' || *p_ == 'E' || *p_ == '+' ||
                             *p_ == '-')) {
            if (*p_ == '.' || *p_ == 'e' || *p_ == 'E') frac = true;
            ++p_;
        }
        if (p_ == s) return false;
        std::string num(s, p_);
        v.t = Value::Num;
        v.d = strtod(num.c_str(), nullptr);
        if (!frac) {
            v.is_int = true;
            if (neg) { v.i = strtoll(num.c_str(), nullptr, 10); v.u = (unsigned long long)v.i; }
            else { v.u = strtoull(num.c_str(), nullptr, 10); v.i = (long long)v.u; }
        }
        return true;
    }
};

inline bool read_file(const std::string& path, std::string& out) {
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) return false;
    char buf[1 << 16];
    size_t n;
    while ((n = fread(buf, 1, sizeof buf, f)) > 0) out.append(buf, n);
    fclose(f);
    return true;
}

inline std::string esc(const std::string& s) {
    std::string o;
    for (char c : s) {
        if (c == '"' || c == '\\') { o += '\\'; o += c; }
        else if ((unsigned char)c < 0x20) { char b[8]; snprintf(b, sizeof b, "\\u%04x", c); o += b; }
        else o += c;
    }
    return o;
}

}  // namespace kcj
