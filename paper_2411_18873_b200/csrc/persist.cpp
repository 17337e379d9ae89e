// Persistence in the reference's on-disk formats, so a forest
// trained on the device round-trips through the reference's own loader and back:
//   model JSON       "etune-model-v1"   EnergyModel::to_json / from_json  energy_model.cpp:259-336
//   samples JSONL    one object a line  save/load_energy_samples          energy_model.cpp:372-420
//   device profile   "etune-profile-v1"  device_profile_to_json / from_json device.cpp:44-110
// The reference serialises with nlohmann::json (object keys in sorted order, doubles
// as the shortest round-trip decimal in nlohmann's layout: "1.0", "0.001", "1e-06");
// the writer below follows that layout, and the parser reads numbers with strtod like
// nlohmann's lexer, so every double survives bit for bit.  Host code only: these are
// the data formats either side of the device path, not part of it.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "etune_internal.hpp"

namespace etune_b200 {
void set_error(const std::string& msg);
}

namespace {

using etune_b200::set_error;

constexpr const char* kModelVersion = "etune-model-v1";        // energy_model.hpp:11
constexpr const char* kFeatureSchema = "etune-features-v1";    // features.hpp:12
constexpr const char* kProfileVersion = "etune-profile-v1";    // device.hpp:8
constexpr int kFeatureDim = 16;

// ------------------------------------------------------------------ writer
void append_exponent(std::string& s, int e) {
    s += 'e';
    if (e < 0) {
        s += '-';
        e = -e;
    } else {
        s += '+';
    }
    if (e < 10) {
        s += '0';
        s += char('0' + e);
    } else {
        s += std::to_string(e);
    }
}

// ------------------------------------------------------------------ Grisu2
// Third-party notice: the double-to-text routine below restates the algorithm (and, where the
// output must match byte for byte, the cached-power table and rounding conditions) of
// nlohmann::json 3.11.3's dtoa_impl, which is distributed under the MIT License:
//   Copyright (c) 2013-2022 Niels Lohmann <https://nlohmann.me>; the Grisu2 implementation in
//   dtoa_impl is based on Florian Loitsch's reference code.  Permission is hereby granted, free
//   of charge, to any person obtaining a copy of this software and associated documentation files
//   (the "Software"), to deal in the Software without restriction, including without limitation
//   the rights to use, copy, modify, merge, publish, distribute, sublicense, and/or sell copies of
//   the Software, and to permit persons to whom the Software is furnished to do so, subject to
//   the following conditions: The above copyright notice and this permission notice shall be
//   included in all copies or substantial portions of the Software.  THE SOFTWARE IS PROVIDED
//   "AS IS", WITHOUT WARRANTY OF ANY KIND, EXPRESS OR IMPLIED.
// nlohmann::json 3.11.3 (the reference's pinned JSON library, nlohmann/json.hpp
// dtoa_impl) prints doubles with Grisu2 (Loitsch, "Printing Floating-Point Numbers
// Quickly and Accurately with Integers", PLDI 2010): digits of a value inside the
// rounding interval [m-, m+], computed in 64-bit fixed point after scaling by a
// cached power of ten so the binary exponent lies in [-60, -32].  Grisu2 is not
// always shortest (e.g. -0.42472286838491913 where 16 digits would round-trip), so
// byte parity with the reference needs this exact variant, restated here.
struct DiyFp {
    uint64_t f;
    int e;
};
DiyFp diy_mul(DiyFp x, DiyFp y) {  // upper 64 bits of the 128-bit product, rounded half up
    const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f + (static_cast<unsigned __int128>(1) << 63);
    return {uint64_t(p >> 64), x.e + y.e + 64};
}
DiyFp diy_normalize(DiyFp x) {
    while ((x.f >> 63) == 0) {
        x.f <<= 1;
        --x.e;
    }
    return x;
}
struct CachedPow {
    uint64_t f;
    int e, k;
};
// 10^k for k = -300, -292, ..., 324: 64-bit significand rounded to nearest and binary
// exponent (generated from exact rational arithmetic)
constexpr CachedPow kCachedPowers[] = {
    {0xAB70FE17C79AC6CA, -1060, -300}, {0xFF77B1FCBEBCDC4F, -1034, -292}, {0xBE5691EF416BD60C, -1007, -284},
    {0x8DD01FAD907FFC3C, -980, -276}, {0xD3515C2831559A83, -954, -268}, {0x9D71AC8FADA6C9B5, -927, -260},
    {0xEA9C227723EE8BCB, -901, -252}, {0xAECC49914078536D, -874, -244}, {0x823C12795DB6CE57, -847, -236},
    {0xC21094364DFB5637, -821, -228}, {0x9096EA6F3848984F, -794, -220}, {0xD77485CB25823AC7, -768, -212},
    {0xA086CFCD97BF97F4, -741, -204}, {0xEF340A98172AACE5, -715, -196}, {0xB23867FB2A35B28E, -688, -188},
    {0x84C8D4DFD2C63F3B, -661, -180}, {0xC5DD44271AD3CDBA, -635, -172}, {0x936B9FCEBB25C996, -608, -164},
    {0xDBAC6C247D62A584, -582, -156}, {0xA3AB66580D5FDAF6, -555, -148}, {0xF3E2F893DEC3F126, -529, -140},
    {0xB5B5ADA8AAFF80B8, -502, -132}, {0x87625F056C7C4A8B, -475, -124}, {0xC9BCFF6034C13053, -449, -116},
    {0x964E858C91BA2655, -422, -108}, {0xDFF9772470297EBD, -396, -100}, {0xA6DFBD9FB8E5B88F, -369, -92},
    {0xF8A95FCF88747D94, -343, -84}, {0xB94470938FA89BCF, -316, -76}, {0x8A08F0F8BF0F156B, -289, -68},
    {0xCDB02555653131B6, -263, -60}, {0x993FE2C6D07B7FAC, -236, -52}, {0xE45C10C42A2B3B06, -210, -44},
    {0xAA242499697392D3, -183, -36}, {0xFD87B5F28300CA0E, -157, -28}, {0xBCE5086492111AEB, -130, -20},
    {0x8CBCCC096F5088CC, -103, -12}, {0xD1B71758E219652C, -77, -4}, {0x9C40000000000000, -50, 4},
    {0xE8D4A51000000000, -24, 12}, {0xAD78EBC5AC620000, 3, 20}, {0x813F3978F8940984, 30, 28},
    {0xC097CE7BC90715B3, 56, 36}, {0x8F7E32CE7BEA5C70, 83, 44}, {0xD5D238A4ABE98068, 109, 52},
    {0x9F4F2726179A2245, 136, 60}, {0xED63A231D4C4FB27, 162, 68}, {0xB0DE65388CC8ADA8, 189, 76},
    {0x83C7088E1AAB65DB, 216, 84}, {0xC45D1DF942711D9A, 242, 92}, {0x924D692CA61BE758, 269, 100},
    {0xDA01EE641A708DEA, 295, 108}, {0xA26DA3999AEF774A, 322, 116}, {0xF209787BB47D6B85, 348, 124},
    {0xB454E4A179DD1877, 375, 132}, {0x865B86925B9BC5C2, 402, 140}, {0xC83553C5C8965D3D, 428, 148},
    {0x952AB45CFA97A0B3, 455, 156}, {0xDE469FBD99A05FE3, 481, 164}, {0xA59BC234DB398C25, 508, 172},
    {0xF6C69A72A3989F5C, 534, 180}, {0xB7DCBF5354E9BECE, 561, 188}, {0x88FCF317F22241E2, 588, 196},
    {0xCC20CE9BD35C78A5, 614, 204}, {0x98165AF37B2153DF, 641, 212}, {0xE2A0B5DC971F303A, 667, 220},
    {0xA8D9D1535CE3B396, 694, 228}, {0xFB9B7CD9A4A7443C, 720, 236}, {0xBB764C4CA7A44410, 747, 244},
    {0x8BAB8EEFB6409C1A, 774, 252}, {0xD01FEF10A657842C, 800, 260}, {0x9B10A4E5E9913129, 827, 268},
    {0xE7109BFBA19C0C9D, 853, 276}, {0xAC2820D9623BF429, 880, 284}, {0x80444B5E7AA7CF85, 907, 292},
    {0xBF21E44003ACDD2D, 933, 300}, {0x8E679C2F5E44FF8F, 960, 308}, {0xD433179D9C8CB841, 986, 316},
    {0x9E19DB92B4E31BA9, 1013, 324},
};
constexpr int kAlpha = -60, kGamma = -32;

CachedPow cached_power(int e) {  // alpha <= c.e + e + 64 <= gamma
    const int f = kAlpha - e - 1;
    const int k = (f * 78913) / (1 << 18) + int(f > 0);  // ceil(f * log10(2))
    const int index = (300 + k + 7) / 8;
    return kCachedPowers[index];
}

int largest_pow10(uint32_t n, uint32_t* pow10) {
    uint32_t p = 1;
    int d = 1;
    while (d < 10 && n / p >= 10) {
        p *= 10;
        ++d;
    }
    *pow10 = p;
    return d;
}

void grisu_round(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        buf[len - 1]--;
        rest += ten_k;
    }
}

// v > 0 finite -> digits in buf[0, len) and decimal exponent: v ~= digits * 10^exp
void grisu2(double v, char* buf, int* len, int* dexp) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const uint64_t E = bits >> 52, F = bits & ((uint64_t(1) << 52) - 1);
    const DiyFp w0 = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F + (uint64_t(1) << 52), int(E) - 1075};
    const bool closer = F == 0 && E > 1;  // the lower neighbour is half as far
    DiyFp mp = diy_normalize(DiyFp{2 * w0.f + 1, w0.e - 1});
    DiyFp mm = closer ? DiyFp{4 * w0.f - 1, w0.e - 2} : DiyFp{2 * w0.f - 1, w0.e - 1};
    mm.f <<= (mm.e - mp.e);
    mm.e = mp.e;
    const DiyFp w = diy_normalize(w0);
    const CachedPow c = cached_power(mp.e);
    const DiyFp cm{c.f, c.e};
    const DiyFp W = diy_mul(w, cm), Wm = diy_mul(mm, cm), Wp = diy_mul(mp, cm);
    const DiyFp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
    *dexp = -c.k;
    // digit generation
    uint64_t delta = Mp.f - Mm.f;
    uint64_t dist = Mp.f - W.f;
    const int sh = -Mp.e;
    const uint64_t one = uint64_t(1) << sh;
    uint32_t p1 = uint32_t(Mp.f >> sh);
    uint64_t p2 = Mp.f & (one - 1);
    uint32_t pow10;
    int n = largest_pow10(p1, &pow10);
    int L = 0;
    while (n > 0) {
        buf[L++] = char('0' + p1 / pow10);
        p1 %= pow10;
        --n;
        const uint64_t rest = (uint64_t(p1) << sh) + p2;
        if (rest <= delta) {
            *dexp += n;
            grisu_round(buf, L, dist, delta, rest, uint64_t(pow10) << sh);
            *len = L;
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        buf[L++] = char('0' + (p2 >> sh));
        p2 &= one - 1;
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    *dexp -= m;
    grisu_round(buf, L, dist, delta, p2, one);
    *len = L;
}

// nlohmann::detail::to_chars layout over the Grisu2 digits: decimal
// notation while the decimal point lies in (-4, 15], ".0" on integral values,
// otherwise d.ddde+XX with at least two exponent digits; non-finite -> null.
void put_double(std::string& s, double v) {
    if (!std::isfinite(v)) {
        s += "null";
        return;
    }
    if (std::signbit(v)) {
        s += '-';
        v = -v;
    }
    if (v == 0.0) {
        s += "0.0";
        return;
    }
    char buf[32];
    int k = 0, dexp = 0;
    grisu2(v, buf, &k, &dexp);
    const std::string digits(buf, size_t(k));
    const int n = k + dexp;  // value = 0.digits * 10^n
    constexpr int kMinExp = -4, kMaxExp = 15;
    if (k <= n && n <= kMaxExp) {
        s += digits;
        s.append(size_t(n - k), '0');
        s += ".0";
    } else if (0 < n && n <= kMaxExp) {
        s += digits.substr(0, size_t(n));
        s += '.';
        s += digits.substr(size_t(n));
    } else if (kMinExp < n && n <= 0) {
        s += "0.";
        s.append(size_t(-n), '0');
        s += digits;
    } else {
        s += digits[0];
        if (k > 1) {
            s += '.';
            s += digits.substr(1);
        }
        append_exponent(s, n - 1);
    }
}

void put_string(std::string& s, const std::string& v) {
    s += '"';
    for (unsigned char c : v) {
        switch (c) {
        case '"': s += "\\\""; break;
        case '\\': s += "\\\\"; break;
        case '\b': s += "\\b"; break;
        case '\f': s += "\\f"; break;
        case '\n': s += "\\n"; break;
        case '\r': s += "\\r"; break;
        case '\t': s += "\\t"; break;
        default:
            if (c < 0x20) {
                char u[8];
                std::snprintf(u, sizeof(u), "\\u%04x", unsigned(c));
                s += u;
            } else {
                s += char(c);
            }
        }
    }
    s += '"';
}

// ------------------------------------------------------------------ parser
struct JVal;
using JObj = std::map<std::string, JVal>;
using JArr = std::vector<JVal>;
struct JVal {
    enum Kind { Null, Bool, Int, UInt, Float, Str, Arr, Obj } kind = Null;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0.0;
    std::string s;
    std::shared_ptr<JArr> a;
    std::shared_ptr<JObj> o;
};

struct JsonError {
    std::string what;
};

class Parser {
public:
    Parser(const char* p, size_t n) : p_(p), e_(p + n) {}
    JVal document() {
        JVal v = value();
        ws();
        if (p_ != e_) fail("unexpected trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const std::string& m) { throw JsonError{m}; }
    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (size_t(e_ - p_) >= n && std::memcmp(p_, w, n) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }
    JVal value() {
        ws();
        if (p_ >= e_) fail("unexpected end of input");
        JVal v;
        const char c = *p_;
        if (c == '{') {
            ++p_;
            v.kind = JVal::Obj;
            v.o = std::make_shared<JObj>();
            ws();
            if (p_ < e_ && *p_ == '}') {
                ++p_;
                return v;
            }
            for (;;) {
                ws();
                if (p_ >= e_ || *p_ != '"') fail("expected object key");
                std::string k = str();
                ws();
                if (p_ >= e_ || *p_ != ':') fail("expected ':'");
                ++p_;
                (*v.o)[k] = value();
                ws();
                if (p_ < e_ && *p_ == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < e_ && *p_ == '}') {
                    ++p_;
                    return v;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            ++p_;
            v.kind = JVal::Arr;
            v.a = std::make_shared<JArr>();
            ws();
            if (p_ < e_ && *p_ == ']') {
                ++p_;
                return v;
            }
            for (;;) {
                v.a->push_back(value());
                ws();
                if (p_ < e_ && *p_ == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < e_ && *p_ == ']') {
                    ++p_;
                    return v;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = JVal::Str;
            v.s = str();
            return v;
        }
        if (lit("true")) {
            v.kind = JVal::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = JVal::Bool;
            return v;
        }
        if (lit("null")) return v;
        return number();
    }
    std::string str() {
        ++p_;  // opening quote
        std::string out;
        while (p_ < e_ && *p_ != '"') {
            const unsigned char c = static_cast<unsigned char>(*p_++);
            if (c < 0x20) fail("control character in string");
            if (c != '\\') {
                out += char(c);
                continue;
            }
            if (p_ >= e_) fail("bad escape");
            const char x = *p_++;
            switch (x) {
            case '"': out += '"'; break;
            case '\\': out += '\\'; break;
            case '/': out += '/'; break;
            case 'b': out += '\b'; break;
            case 'f': out += '\f'; break;
            case 'n': out += '\n'; break;
            case 'r': out += '\r'; break;
            case 't': out += '\t'; break;
            case 'u': {
                auto hex4 = [&]() -> unsigned {
                    if (e_ - p_ < 4) fail("bad \\u escape");
                    unsigned cp = 0;
                    for (int q = 0; q < 4; ++q) {
                        const char h = *p_++;
                        cp <<= 4;
                        if (h >= '0' && h <= '9') cp |= unsigned(h - '0');
                        else if (h >= 'a' && h <= 'f') cp |= unsigned(h - 'a' + 10);
                        else if (h >= 'A' && h <= 'F') cp |= unsigned(h - 'A' + 10);
                        else fail("bad \\u escape");
                    }
                    return cp;
                };
                unsigned cp = hex4();
                if (cp >= 0xD800 && cp <= 0xDBFF) {
                    if (!(e_ - p_ >= 2 && p_[0] == '\\' && p_[1] == 'u')) fail("unpaired surrogate");
                    p_ += 2;
                    const unsigned lo = hex4();
                    if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired surrogate");
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                    fail("unpaired surrogate");
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
        }
        if (p_ >= e_) fail("unterminated string");
        ++p_;
        return out;
    }
    // RFC 8259 number; integers stay integers (int64, then uint64), everything else is
    // strtod of the token, like nlohmann's lexer
    JVal number() {
        const char* b = p_;
        bool is_float = false;
        if (p_ < e_ && *p_ == '-') ++p_;
        if (p_ >= e_) fail("bad number");
        if (*p_ == '0') {
            ++p_;
        } else if (*p_ >= '1' && *p_ <= '9') {
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        } else {
            fail("unexpected character");
        }
        if (p_ < e_ && *p_ == '.') {
            is_float = true;
            ++p_;
            if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) fail("bad number");
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
            is_float = true;
            ++p_;
            if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
            if (p_ >= e_ || !(*p_ >= '0' && *p_ <= '9')) fail("bad number");
            while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
        }
        const std::string tok(b, p_);
        JVal v;
        if (!is_float) {
            errno = 0;
            if (tok[0] == '-') {
                const long long x = std::strtoll(tok.c_str(), nullptr, 10);
                if (errno == 0) {
                    v.kind = JVal::Int;
                    v.i = x;
                    return v;
                }
            } else {
                const unsigned long long x = std::strtoull(tok.c_str(), nullptr, 10);
                if (errno == 0) {
                    if (x <= uint64_t(INT64_MAX)) {
                        v.kind = JVal::Int;
                        v.i = int64_t(x);
                    } else {
                        v.kind = JVal::UInt;
                        v.u = x;
                    }
                    return v;
                }
            }
        }
        v.kind = JVal::Float;
        v.d = std::strtod(tok.c_str(), nullptr);
        return v;
    }
    const char* p_;
    const char* e_;
};

const JVal& at(const JVal& o, const char* key) {
    if (o.kind != JVal::Obj) throw JsonError{"type must be object"};
    auto it = o.o->find(key);
    if (it == o.o->end()) throw JsonError{std::string("key '") + key + "' not found"};
    return it->second;
}
const JVal* find(const JVal& o, const char* key) {
    if (o.kind != JVal::Obj) return nullptr;
    auto it = o.o->find(key);
    return it == o.o->end() ? nullptr : &it->second;
}
double as_double(const JVal& v) {
    switch (v.kind) {
    case JVal::Int: return double(v.i);
    case JVal::UInt: return double(v.u);
    case JVal::Float: return v.d;
    default: throw JsonError{"type must be number"};
    }
}
int64_t as_int(const JVal& v) {
    switch (v.kind) {
    case JVal::Int: return v.i;
    case JVal::UInt: return int64_t(v.u);
    case JVal::Float: return int64_t(v.d);
    default: throw JsonError{"type must be number"};
    }
}
uint64_t as_u64(const JVal& v) {
    switch (v.kind) {
    case JVal::Int: return uint64_t(v.i);
    case JVal::UInt: return v.u;
    case JVal::Float: return uint64_t(v.d);
    default: throw JsonError{"type must be number"};
    }
}
// j.value(key, default) for a string member
std::string str_or(const JVal& o, const char* key, const std::string& dflt) {
    const JVal* v = find(o, key);
    if (!v) return dflt;
    if (v->kind != JVal::Str) throw JsonError{"type must be string"};
    return v->s;
}

etune_status fail(etune_status st, const std::string& m) {
    set_error(m);
    return st;
}

etune_status emit(const std::string& text, char* out, int64_t cap, int64_t* out_len) {
    if (out_len) *out_len = int64_t(text.size());
    if (!out) return ETUNE_OK;  // length query
    if (cap < int64_t(text.size()) + 1)
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "output buffer too small: need " + std::to_string(text.size() + 1));
    std::memcpy(out, text.data(), text.size());
    out[text.size()] = '\0';
    return ETUNE_OK;
}

}  // namespace

extern "C" {

etune_status etune_model_to_json(const int32_t* feature, const double* threshold, const int32_t* left,
                                 const int32_t* right, const double* value, const int64_t* tree_offsets,
                                 int64_t num_trees, const etune_boost_params* params, double base_score,
                                 double reference_energy_mj, char* out, int64_t cap, int64_t* out_len) {
    if (num_trees < 0 || !tree_offsets || !params) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad model arguments");
    const int64_t nn = tree_offsets[num_trees];
    if (nn > 0 && (!feature || !threshold || !left || !right || !value))
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "null node arrays");
    // keys in sorted order (nlohmann::json objects are std::map), compact dump()
    std::string s;
    s.reserve(size_t(64 + 96 * nn));
    s += "{\"base_score\":";
    put_double(s, base_score);
    s += ",\"feature_schema\":";
    put_string(s, kFeatureSchema);
    s += ",\"model_version\":";
    put_string(s, kModelVersion);
    s += ",\"params\":{\"learning_rate\":";
    put_double(s, params->learning_rate);
    s += ",\"max_depth\":" + std::to_string(params->max_depth);
    s += ",\"min_leaf_weight\":";
    put_double(s, params->min_leaf_weight);
    s += ",\"num_trees\":" + std::to_string(params->num_trees);
    s += ",\"reg_lambda\":";
    put_double(s, params->reg_lambda);
    s += "},\"reference_energy_mj\":";
    put_double(s, reference_energy_mj);
    s += ",\"trees\":[";
    for (int64_t t = 0; t < num_trees; ++t) {
        if (t) s += ',';
        s += '[';
        for (int64_t i = tree_offsets[t]; i < tree_offsets[t + 1]; ++i) {
            if (i > tree_offsets[t]) s += ',';
            s += "{\"f\":" + std::to_string(feature[i]) + ",\"l\":" + std::to_string(left[i]) +
                 ",\"r\":" + std::to_string(right[i]) + ",\"t\":";
            put_double(s, threshold[i]);
            s += ",\"v\":";
            put_double(s, value[i]);
            s += '}';
        }
        s += ']';
    }
    s += "]}";
    return emit(s, out, cap, out_len);
}

etune_status etune_model_from_json(const char* text, int64_t len, etune_model_host* m) {
    if (!text || len < 0 || !m) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    std::memset(m, 0, sizeof(*m));
    JVal j;
    try {
        j = Parser(text, size_t(len)).document();
    } catch (const JsonError& e) {
        return fail(ETUNE_ERR_IO, "unreadable model file: " + e.what);
    }
    std::vector<int32_t> fe, le, ri;
    std::vector<double> th, va;
    std::vector<int64_t> off{0};
    try {
        const std::string version = str_or(j, "model_version", "");
        if (version != kModelVersion)
            return fail(ETUNE_ERR_VERSION_MISMATCH, "model version '" + version + "' is not supported");
        const std::string schema = str_or(j, "feature_schema", "");
        if (schema != kFeatureSchema)
            return fail(ETUNE_ERR_VERSION_MISMATCH, "model feature schema '" + schema + "' does not match " +
                                                        std::string(kFeatureSchema));
        const JVal& p = at(j, "params");
        m->params.num_trees = int32_t(as_int(at(p, "num_trees")));
        m->params.max_depth = int32_t(as_int(at(p, "max_depth")));
        m->params.learning_rate = as_double(at(p, "learning_rate"));
        m->params.min_leaf_weight = as_double(at(p, "min_leaf_weight"));
        m->params.reg_lambda = as_double(at(p, "reg_lambda"));
        m->base_score = as_double(at(j, "base_score"));
        m->reference_energy_mj = as_double(at(j, "reference_energy_mj"));
        const JVal& trees = at(j, "trees");
        if (trees.kind != JVal::Arr) throw JsonError{"trees must be an array"};
        for (const JVal& tj : *trees.a) {
            if (tj.kind != JVal::Arr) throw JsonError{"tree must be an array"};
            if (tj.a->empty()) return fail(ETUNE_ERR_IO, "model file contains an empty tree");
            for (const JVal& n : *tj.a) {
                fe.push_back(int32_t(as_int(at(n, "f"))));
                th.push_back(as_double(at(n, "t")));
                le.push_back(int32_t(as_int(at(n, "l"))));
                ri.push_back(int32_t(as_int(at(n, "r"))));
                va.push_back(as_double(at(n, "v")));
            }
            off.push_back(int64_t(fe.size()));
        }
    } catch (const JsonError& e) {
        return fail(ETUNE_ERR_IO, "unreadable model file: " + e.what);
    }
    const size_t nn = fe.size();
    m->num_trees = int64_t(off.size()) - 1;
    m->num_nodes = int64_t(nn);
    m->feature = static_cast<int32_t*>(std::malloc(4 * nn + 4));
    m->left = static_cast<int32_t*>(std::malloc(4 * nn + 4));
    m->right = static_cast<int32_t*>(std::malloc(4 * nn + 4));
    m->threshold = static_cast<double*>(std::malloc(8 * nn + 8));
    m->value = static_cast<double*>(std::malloc(8 * nn + 8));
    m->tree_offsets = static_cast<int64_t*>(std::malloc(8 * off.size()));
    if (!m->feature || !m->left || !m->right || !m->threshold || !m->value || !m->tree_offsets) {
        etune_model_host_free(m);
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "out of host memory");
    }
    std::memcpy(m->feature, fe.data(), 4 * nn);
    std::memcpy(m->left, le.data(), 4 * nn);
    std::memcpy(m->right, ri.data(), 4 * nn);
    std::memcpy(m->threshold, th.data(), 8 * nn);
    std::memcpy(m->value, va.data(), 8 * nn);
    std::memcpy(m->tree_offsets, off.data(), 8 * off.size());
    return ETUNE_OK;
}

void etune_model_host_free(etune_model_host* m) {
    if (!m) return;
    std::free(m->feature);
    std::free(m->left);
    std::free(m->right);
    std::free(m->threshold);
    std::free(m->value);
    std::free(m->tree_offsets);
    std::memset(m, 0, sizeof(*m));
}

etune_status etune_samples_to_jsonl(const double* features, const double* measured_mj, const double* normalized,
                                    int64_t n, char* out, int64_t cap, int64_t* out_len) {
    if (n < 0 || (n > 0 && (!features || !measured_mj || !normalized)))
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad sample arrays");
    std::string s;
    s.reserve(size_t(n) * 420);
    for (int64_t i = 0; i < n; ++i) {  // energy_model.cpp:376-381: one compact object per line
        s += "{\"features\":[";
        for (int k = 0; k < kFeatureDim; ++k) {
            if (k) s += ',';
            put_double(s, features[i * kFeatureDim + k]);
        }
        s += "],\"measured_energy_mj\":";
        put_double(s, measured_mj[i]);
        s += ",\"normalized_energy\":";
        put_double(s, normalized[i]);
        s += "}\n";
    }
    return emit(s, out, cap, out_len);
}

etune_status etune_samples_from_jsonl(const char* text, int64_t len, etune_samples_host* out) {
    if (!text || len < 0 || !out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    std::memset(out, 0, sizeof(*out));
    std::vector<double> f, mm, nz;
    const char* p = text;
    const char* e = text + len;
    int line_no = 0;
    while (p < e) {  // std::getline: lines end at '\n'; empty lines are skipped
        const char* q = static_cast<const char*>(std::memchr(p, '\n', size_t(e - p)));
        if (!q) q = e;
        ++line_no;
        const std::string ln = "line " + std::to_string(line_no);
        if (q > p) {
            JVal j;
            try {
                j = Parser(p, size_t(q - p)).document();
            } catch (const JsonError& er) {
                return fail(ETUNE_ERR_IO, "bad JSONL at " + ln + ": " + er.what);
            }
            try {
                const JVal& fv = at(j, "features");
                const size_t w = fv.kind == JVal::Arr ? fv.a->size() : 0;
                if (fv.kind != JVal::Arr || w != size_t(kFeatureDim))
                    return fail(ETUNE_ERR_SCHEMA_MISMATCH, ln + ": feature vector width " + std::to_string(w) +
                                                               " != " + std::to_string(kFeatureDim));
                for (int k = 0; k < kFeatureDim; ++k) f.push_back(as_double((*fv.a)[size_t(k)]));
                const double me = as_double(at(j, "measured_energy_mj"));
                const JVal* nv = find(j, "normalized_energy");
                const double ne = nv ? as_double(*nv) : 0.0;
                if (!(me > 0.0)) return fail(ETUNE_ERR_NON_POSITIVE_ENERGY, ln + ": measured energy must be positive");
                mm.push_back(me);
                nz.push_back(ne);
            } catch (const JsonError& er) {
                return fail(ETUNE_ERR_IO, "bad JSONL at " + ln + ": " + er.what);
            }
        }
        p = q + 1;
    }
    const size_t n = mm.size();
    out->n = int64_t(n);
    out->features = static_cast<double*>(std::malloc(8 * f.size() + 8));
    out->measured_energy_mj = static_cast<double*>(std::malloc(8 * n + 8));
    out->normalized_energy = static_cast<double*>(std::malloc(8 * n + 8));
    if (!out->features || !out->measured_energy_mj || !out->normalized_energy) {
        etune_samples_host_free(out);
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "out of host memory");
    }
    std::memcpy(out->features, f.data(), 8 * f.size());
    std::memcpy(out->measured_energy_mj, mm.data(), 8 * n);
    std::memcpy(out->normalized_energy, nz.data(), 8 * n);
    return ETUNE_OK;
}

void etune_samples_host_free(etune_samples_host* s) {
    if (!s) return;
    std::free(s->features);
    std::free(s->measured_energy_mj);
    std::free(s->normalized_energy);
    std::memset(s, 0, sizeof(*s));
}

etune_status etune_measurement_log_to_jsonl(const etune_log_record* r, int64_t n, char* out, int64_t cap,
                                            int64_t* out_len) {
    if (n < 0 || (n > 0 && !r)) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad record array");
    std::string s;
    s.reserve(size_t(n) * 200);
    for (int64_t i = 0; i < n; ++i) {
        const etune_log_record& x = r[i];
        s += "{\"avg_power_w\":";
        put_double(s, x.m.avg_power_w);
        s += ",\"backend\":";
        put_string(s, std::string(x.backend, strnlen(x.backend, sizeof(x.backend))));
        s += ",\"candidate_id\":" + std::to_string(x.m.candidate_id);
        s += ",\"energy_mj\":";
        put_double(s, x.m.energy_mj);
        s += ",\"iterations\":" + std::to_string(x.m.iterations);
        s += ",\"latency_ms\":";
        put_double(s, x.m.latency_ms);
        s += ",\"timestamp\":";
        put_string(s, std::string(x.timestamp, strnlen(x.timestamp, sizeof(x.timestamp))));
        s += "}\n";
    }
    return emit(s, out, cap, out_len);
}

etune_status etune_measurement_log_from_jsonl(const char* text, int64_t len, etune_log_record** out, int64_t* n) {
    if (!text || len < 0 || !out || !n) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    *out = nullptr;
    *n = 0;
    std::vector<etune_log_record> recs;
    const char* p = text;
    const char* e = text + len;
    int line_no = 0;
    while (p < e) {
        const char* q = static_cast<const char*>(std::memchr(p, '\n', size_t(e - p)));
        if (!q) q = e;
        ++line_no;
        const std::string ln = "line " + std::to_string(line_no);
        if (q > p) {
            etune_log_record x;
            std::memset(&x, 0, sizeof(x));
            try {
                const JVal j = Parser(p, size_t(q - p)).document();
                x.m.candidate_id = as_u64(at(j, "candidate_id"));
                x.m.latency_ms = as_double(at(j, "latency_ms"));
                x.m.avg_power_w = as_double(at(j, "avg_power_w"));
                x.m.energy_mj = as_double(at(j, "energy_mj"));
                const JVal* it = find(j, "iterations");
                x.m.iterations = it ? as_int(*it) : 0;
                x.m.feasible = 1;
                const std::string be = str_or(j, "backend", ""), ts = str_or(j, "timestamp", "");
                std::memcpy(x.backend, be.data(), std::min(be.size(), sizeof(x.backend) - 1));
                std::memcpy(x.timestamp, ts.data(), std::min(ts.size(), sizeof(x.timestamp) - 1));
            } catch (const JsonError& er) {
                return fail(ETUNE_ERR_IO, "bad measurement log at " + ln + ": " + er.what);
            }
            // energy_mj = avg_power_w x latency_ms within 1e-9 relative
            const double want = x.m.avg_power_w * x.m.latency_ms;
            if (!(std::fabs(x.m.energy_mj - want) <= 1e-9 * std::fabs(want)))
                return fail(ETUNE_ERR_CONSISTENCY, "measurement log " + ln + ": energy_mj != avg_power_w * latency_ms");
            recs.push_back(x);
        }
        p = q + 1;
    }
    *n = int64_t(recs.size());
    *out = static_cast<etune_log_record*>(std::malloc(sizeof(etune_log_record) * recs.size() + 1));
    if (!*out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "out of host memory");
    if (!recs.empty()) std::memcpy(*out, recs.data(), sizeof(etune_log_record) * recs.size());
    return ETUNE_OK;
}

void etune_measurement_log_free(etune_log_record* r) { std::free(r); }

etune_status etune_device_profile_to_json(const etune_device_config* d, const char* name, char* out, int64_t cap,
                                          int64_t* out_len) {
    if (!d) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null device config");
    // dump(2): sorted keys, two-space indent, trailing newline (device.cpp:44-62)
    std::string s = "{\n";
    auto key = [&](const char* k, bool first) {
        if (!first) s += ",\n";
        s += "  ";
        put_string(s, k);
        s += ": ";
    };
    key("base_throughput_flops_per_s_per_sm", true);
    put_double(s, d->base_throughput_flops_per_s_per_sm);
    key("constant_power_w", false);
    put_double(s, d->constant_power_w);
    key("dynamic_energy_per_flop_nj", false);
    put_double(s, d->dynamic_energy_per_flop_nj);
    key("dynamic_energy_per_glb_access_nj", false);
    put_double(s, d->dynamic_energy_per_glb_access_nj);
    key("dynamic_energy_per_shared_access_nj", false);
    put_double(s, d->dynamic_energy_per_shared_access_nj);
    key("latency_floor_ms", false);
    put_double(s, d->latency_floor_ms);
    key("mem_bandwidth_elems_per_s", false);
    put_double(s, d->mem_bandwidth_elems_per_s);
    key("name", false);
    put_string(s, name ? name : "a100-like");
    key("noise_sigma_rel", false);
    put_double(s, d->noise_sigma_rel);
    key("num_sms", false);
    s += std::to_string(d->num_sms);
    key("profile_version", false);
    put_string(s, kProfileVersion);
    key("rng_seed", false);
    s += std::to_string(d->rng_seed);
    key("sampler_hz", false);
    put_double(s, d->sampler_hz);
    key("static_power_per_sm_w", false);
    put_double(s, d->static_power_per_sm_w);
    key("warmup_s", false);
    put_double(s, d->warmup_s);
    s += "\n}\n";
    return emit(s, out, cap, out_len);
}

etune_status etune_device_profile_from_json(const char* text, int64_t len, etune_device_config* d, char* name,
                                            int64_t name_cap) {
    if (!text || len < 0 || !d) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    JVal j;
    try {
        j = Parser(text, size_t(len)).document();
    } catch (const JsonError& e) {
        return fail(ETUNE_ERR_PARSE, "bad device profile JSON: " + e.what);
    }
    etune_device_config o;
    std::memset(&o, 0, sizeof(o));
    std::string nm = "a100-like";
    try {
        const std::string version = str_or(j, "profile_version", "");
        if (version != kProfileVersion)
            return fail(ETUNE_ERR_VERSION_MISMATCH, "device profile version '" + version +
                                                        "' is not supported (expected " +
                                                        std::string(kProfileVersion) + ")");
        nm = str_or(j, "name", nm);
        o.num_sms = int32_t(as_int(at(j, "num_sms")));
        o.constant_power_w = as_double(at(j, "constant_power_w"));
        o.static_power_per_sm_w = as_double(at(j, "static_power_per_sm_w"));
        o.dynamic_energy_per_flop_nj = as_double(at(j, "dynamic_energy_per_flop_nj"));
        o.dynamic_energy_per_glb_access_nj = as_double(at(j, "dynamic_energy_per_glb_access_nj"));
        o.dynamic_energy_per_shared_access_nj = as_double(at(j, "dynamic_energy_per_shared_access_nj"));
        o.base_throughput_flops_per_s_per_sm = as_double(at(j, "base_throughput_flops_per_s_per_sm"));
        o.mem_bandwidth_elems_per_s = as_double(at(j, "mem_bandwidth_elems_per_s"));
        o.latency_floor_ms = as_double(at(j, "latency_floor_ms"));
        o.sampler_hz = as_double(at(j, "sampler_hz"));
        o.warmup_s = as_double(at(j, "warmup_s"));
        o.noise_sigma_rel = as_double(at(j, "noise_sigma_rel"));
        o.rng_seed = as_u64(at(j, "rng_seed"));
    } catch (const JsonError& e) {
        return fail(ETUNE_ERR_PARSE, "bad device profile JSON: " + e.what);
    }
    // DeviceConfig::validate (device.cpp:12-38)
    auto pos = [&](double v, const char* f) -> bool {
        if (!(v > 0.0)) {
            set_error(std::string("device profile field '") + f + "' must be positive");
            return false;
        }
        return true;
    };
    if (o.num_sms < 1) return fail(ETUNE_ERR_VALIDATION, "num_sms must be >= 1");
    if (!pos(o.constant_power_w, "constant_power_w") || !pos(o.static_power_per_sm_w, "static_power_per_sm_w") ||
        !pos(o.dynamic_energy_per_flop_nj, "dynamic_energy_per_flop_nj") ||
        !pos(o.dynamic_energy_per_glb_access_nj, "dynamic_energy_per_glb_access_nj") ||
        !pos(o.dynamic_energy_per_shared_access_nj, "dynamic_energy_per_shared_access_nj") ||
        !pos(o.base_throughput_flops_per_s_per_sm, "base_throughput_flops_per_s_per_sm") ||
        !pos(o.mem_bandwidth_elems_per_s, "mem_bandwidth_elems_per_s") ||
        !pos(o.latency_floor_ms, "latency_floor_ms"))
        return ETUNE_ERR_VALIDATION;
    if (o.sampler_hz < 30.0 || o.sampler_hz > 50.0) return fail(ETUNE_ERR_VALIDATION, "sampler_hz must lie in [30, 50]");
    if (o.warmup_s < 0.0) return fail(ETUNE_ERR_VALIDATION, "warmup_s must be >= 0");
    if (o.noise_sigma_rel < 0.0) return fail(ETUNE_ERR_VALIDATION, "noise_sigma_rel must be >= 0");
    if (name) {
        if (name_cap < int64_t(nm.size()) + 1)
            return fail(ETUNE_ERR_INVALID_ARGUMENT, "name buffer too small: need " + std::to_string(nm.size() + 1));
        std::memcpy(name, nm.c_str(), nm.size() + 1);
    }
    *d = o;
    return ETUNE_OK;
}

}  // extern "C"
