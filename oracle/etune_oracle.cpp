// TEST INFRASTRUCTURE ONLY — see etune_oracle.h for the contract and pinning.
//
// Plain, single-threaded C-style C++ restatement of the reference hot path.
// Compiled -O2 -ffp-contract=off (oracle/Makefile) so double arithmetic is
// evaluated exactly in source order, as the reference's default-march build is.
#include "etune_oracle.h"

#include <algorithm>
#include <limits>
#include <atomic>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

thread_local std::string g_err;

enum Status {
    OK = 0,
    PARSE = 1,
    VALIDATION = 2,
    SPACE_EXHAUSTED = 3,
    ILLEGAL_SCHEDULE = 4,
    TOO_LARGE = 5,
    NON_POSITIVE_ENERGY = 6,
    INSUFFICIENT_DATA = 7,
    LENGTH_MISMATCH = 10,
    EMPTY_INPUT = 11,
};

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

// ------------------------------------------------------------------ opspec
// opspec.hpp:30-47 field order; opspec.cpp:65-93 validate; 103-117 nest.
struct Op {
    int64_t kind, batch, m, n, k, height, width, in_ch, out_ch, ks, stride, pad;
};
Op op_of(const int64_t* w) {
    Op o;
    std::memcpy(&o, w, sizeof(Op));
    return o;
}

int op_validate(const Op& o) {  // opspec.cpp:65-93
    if (o.kind == 0 || o.kind == 1) {
        if (o.batch < 1 || o.m < 1 || o.n < 1 || o.k < 1)
            return fail(VALIDATION, "matmul extents must all be >= 1");
        if (o.kind == 1 && o.m != 1) return fail(VALIDATION, "mv requires M == 1");
        return OK;
    }
    if (o.batch < 1 || o.height < 1 || o.width < 1 || o.in_ch < 1 || o.out_ch < 1 || o.ks < 1)
        return fail(VALIDATION, "conv extents must all be >= 1");
    if (o.stride < 1) return fail(VALIDATION, "conv stride must be >= 1");
    if (o.pad < 0) return fail(VALIDATION, "conv padding must be >= 0");
    const int64_t hs = o.height + 2 * o.pad - o.ks;
    const int64_t ws = o.width + 2 * o.pad - o.ks;
    if (hs < 0 || ws < 0 || hs % o.stride != 0 || ws % o.stride != 0)
        return fail(VALIDATION, "conv output extent must be a positive integer");
    return OK;
}

struct Nest {
    int64_t b, m, n, k;
};
Nest op_nest(const Op& o) {  // opspec.cpp:103-117
    if (o.kind == 2) {
        const int64_t oh = (o.height + 2 * o.pad - o.ks) / o.stride + 1;
        const int64_t ow = (o.width + 2 * o.pad - o.ks) / o.stride + 1;
        return {o.batch, oh * ow, o.out_ch, o.in_ch * o.ks * o.ks};
    }
    return {o.batch, o.m, o.n, o.k};
}

// ---------------------------------------------------------------- schedule
struct Tiling {
    int64_t blocks, threads, pt;
    bool operator==(const Tiling& t) const {
        return blocks == t.blocks && threads == t.threads && pt == t.pt;
    }
};
struct Sched {
    Tiling sp[3];
    int64_t k_tile, unroll, vec;
    int64_t grid() const { return sp[0].blocks * sp[1].blocks * sp[2].blocks; }
    int64_t block() const { return sp[0].threads * sp[1].threads * sp[2].threads; }
};
Sched sched_of(const int64_t* w) {
    Sched s;
    for (int d = 0; d < 3; ++d) s.sp[d] = {w[3 * d], w[3 * d + 1], w[3 * d + 2]};
    s.k_tile = w[9];
    s.unroll = w[10];
    s.vec = w[11];
    return s;
}
void sched_put(const Sched& s, int64_t* w) {
    for (int d = 0; d < 3; ++d) {
        w[3 * d] = s.sp[d].blocks;
        w[3 * d + 1] = s.sp[d].threads;
        w[3 * d + 2] = s.sp[d].pt;
    }
    w[9] = s.k_tile;
    w[10] = s.unroll;
    w[11] = s.vec;
}

bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int validate_schedule(const Op& o, const Sched& s) {  // schedule.cpp:26-61
    const Nest nest = op_nest(o);
    const int64_t ext[3] = {nest.b, nest.m, nest.n};
    for (int d = 0; d < 3; ++d) {
        const Tiling& t = s.sp[d];
        if (t.blocks < 1 || t.threads < 1 || t.pt < 1)
            return fail(ILLEGAL_SCHEDULE, "non-positive tile factor");
        if (t.blocks * t.threads * t.pt != ext[d])
            return fail(ILLEGAL_SCHEDULE, "tiling does not multiply to the extent");
    }
    if (s.k_tile < 1 || nest.k % s.k_tile != 0)
        return fail(ILLEGAL_SCHEDULE, "k_tile must divide the reduction extent");
    const int64_t block = s.block();
    if (block < 1 || block > 1024) return fail(ILLEGAL_SCHEDULE, "block size outside [1, 1024]");
    if (!pow2(s.unroll) || s.k_tile % s.unroll != 0)
        return fail(ILLEGAL_SCHEDULE, "unroll must be a power of two dividing k_tile");
    if ((s.vec != 1 && s.vec != 2 && s.vec != 4) || s.sp[2].pt % s.vec != 0)
        return fail(ILLEGAL_SCHEDULE, "vectorize must be in {1,2,4} and divide pt_n");
    return OK;
}

// ------------------------------------------------------------------- space
uint64_t fnv_word(uint64_t h, uint64_t v) {  // space.cpp:12-18
    for (int b = 0; b < 8; ++b) {
        h ^= (v >> (8 * b)) & 0xffu;
        h *= 1099511628211ull;
    }
    return h;
}
uint64_t cand_id(const Op& o, const Sched& s) {  // space.cpp:22-45
    uint64_t h = 14695981039346656037ull;
    const int64_t* ow = &o.kind;
    for (int i = 0; i < 12; ++i) h = fnv_word(h, static_cast<uint64_t>(ow[i]));
    for (int d = 0; d < 3; ++d) {
        h = fnv_word(h, static_cast<uint64_t>(s.sp[d].blocks));
        h = fnv_word(h, static_cast<uint64_t>(s.sp[d].threads));
        h = fnv_word(h, static_cast<uint64_t>(s.sp[d].pt));
    }
    h = fnv_word(h, static_cast<uint64_t>(s.k_tile));
    h = fnv_word(h, static_cast<uint64_t>(s.unroll));
    h = fnv_word(h, static_cast<uint64_t>(s.vec));
    return h;
}

std::vector<int64_t> divisors(int64_t e) {  // space.cpp:57-67
    std::vector<int64_t> out;
    for (int64_t d = 1; d * d <= e; ++d) {
        if (e % d == 0) {
            out.push_back(d);
            if (d != e / d) out.push_back(e / d);
        }
    }
    std::sort(out.begin(), out.end());
    return out;
}
std::vector<Tiling> dim_tilings(int64_t e) {  // space.cpp:69-78
    std::vector<Tiling> out;
    for (int64_t b : divisors(e)) {
        const int64_t rest = e / b;
        for (int64_t t : divisors(rest)) out.push_back({b, t, rest / t});
    }
    return out;
}
std::vector<int64_t> pow2_upto(int64_t cap) {  // space.cpp:82-87
    std::vector<int64_t> out;
    for (int64_t v = 1; v <= cap; v *= 2) out.push_back(v);
    if (out.empty()) out.push_back(1);
    return out;
}

struct Limits {
    int64_t max_block = 1024, max_unroll = 8, max_vec = 4;
};
Limits limits_of(const int64_t* w) {
    Limits l;
    if (w) {
        l.max_block = w[0];
        l.max_unroll = w[1];
        l.max_vec = w[2];
    }
    return l;
}

// ScheduleEnumerator, space.cpp:91-150: odometer, last position fastest.
struct Enumerator {
    Op op;
    Limits lim;
    std::vector<Tiling> til[3];
    std::vector<int64_t> kt, un, ve;
    size_t idx[6] = {0, 0, 0, 0, 0, 0};
    bool fresh = true, done = false;
    Enumerator(const Op& o, const Limits& l) : op(o), lim(l) {
        const Nest n = op_nest(o);
        til[0] = dim_tilings(n.b);
        til[1] = dim_tilings(n.m);
        til[2] = dim_tilings(n.n);
        kt = divisors(n.k);
        un = pow2_upto(std::max<int64_t>(1, l.max_unroll));
        ve = pow2_upto(std::min<int64_t>(4, std::max<int64_t>(1, l.max_vec)));
    }
    Sched cur() const {
        Sched s;
        for (int d = 0; d < 3; ++d) s.sp[d] = til[d][idx[d]];
        s.k_tile = kt[idx[3]];
        s.unroll = un[idx[4]];
        s.vec = ve[idx[5]];
        return s;
    }
    bool legal() const {  // space.cpp:116-125
        const Sched s = cur();
        if (s.block() > std::min<int64_t>(lim.max_block, 1024)) return false;
        if (s.k_tile % s.unroll != 0) return false;
        if (s.sp[2].pt % s.vec != 0) return false;
        return true;
    }
    bool advance() {
        const size_t sz[6] = {til[0].size(), til[1].size(), til[2].size(),
                              kt.size(), un.size(), ve.size()};
        for (int p = 5; p >= 0; --p) {
            if (++idx[p] < sz[p]) return true;
            idx[p] = 0;
        }
        return false;
    }
    bool next(Sched* out) {
        if (done) return false;
        if (fresh) {
            fresh = false;
            if (legal()) {
                *out = cur();
                return true;
            }
        }
        while (advance()) {
            if (legal()) {
                *out = cur();
                return true;
            }
        }
        done = true;
        return false;
    }
};

int64_t count_sched(const Op& o, const Limits& l, int64_t cap) {  // space.cpp:152-160
    Enumerator en(o, l);
    Sched s;
    int64_t c = 0;
    while (en.next(&s)) {
        if (++c == cap) break;
    }
    return c;
}

// --------------------------------------------------------------------- RNG
// std::mt19937_64 restated (64-bit MT: n=312, m=156, r=31, a=0xb5026f5aa96619e9,
// u=29 d=0x5555555555555555, s=17 b=0x71d67fffeda60000, t=37 c=0xfff7eee000000000,
// l=43, f=6364136223846793005).
struct Mt64 {
    uint64_t s[312];
    int i;
    explicit Mt64(uint64_t seed) {
        s[0] = seed;
        for (int k = 1; k < 312; ++k) s[k] = 6364136223846793005ull * (s[k - 1] ^ (s[k - 1] >> 62)) + k;
        i = 312;
    }
    void twist() {
        for (int k = 0; k < 312; ++k) {
            const uint64_t x = (s[k] & 0xffffffff80000000ull) | (s[(k + 1) % 312] & 0x7fffffffull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xb5026f5aa96619e9ull;
            s[k] = s[(k + 156) % 312] ^ xa;
        }
        i = 0;
    }
    uint64_t operator()() {
        if (i >= 312) twist();
        uint64_t y = s[i++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71d67fffeda60000ull;
        y ^= (y << 37) & 0xfff7eee000000000ull;
        y ^= y >> 43;
        return y;
    }
};

// libstdc++ uniform_int_distribution<size_t>(0, range-1) on a 64-bit engine:
// _S_nd<unsigned __int128> (Lemire, threshold (-range % range)).
template <typename G>
uint64_t lemire(G& g, uint64_t range) {
    unsigned __int128 prod = static_cast<unsigned __int128>(g()) * range;
    uint64_t low = static_cast<uint64_t>(prod);
    if (low < range) {
        const uint64_t thr = (0 - range) % range;
        while (low < thr) {
            prod = static_cast<unsigned __int128>(g()) * range;
            low = static_cast<uint64_t>(prod);
        }
    }
    return static_cast<uint64_t>(prod >> 64);
}
// uniform_int_distribution<size_t>(a, b)
template <typename G>
uint64_t uniform_ab(G& g, uint64_t a, uint64_t b) { return lemire(g, b - a + 1) + a; }

// uniform_real_distribution<double>(0,1) == generate_canonical<double,53>: one word.
template <typename G>
double canonical(G& g) {
    double r = static_cast<double>(g()) / 18446744073709551616.0;
    if (r >= 1.0) r = std::nextafter(1.0, 0.0);
    return r;
}

// -------------------------------------------------------------- counters
struct Counters {
    int64_t grid, block, flops, int_ops, glb_ld, glb_st, shared_ld, shared_st;
    double sm_eff;
    int64_t active;
};
Counters derive(const Op& o, const Sched& s, int num_sms) {  // counters.cpp:9-49
    const Nest nest = op_nest(o);
    const int64_t bt_b = s.sp[0].threads * s.sp[0].pt;
    const int64_t bt_m = s.sp[1].threads * s.sp[1].pt;
    const int64_t bt_n = s.sp[2].threads * s.sp[2].pt;
    Counters c;
    c.grid = s.grid();
    c.block = s.block();
    const int64_t steps = nest.k / s.k_tile;
    const int64_t outputs = nest.b * nest.m * nest.n;
    c.flops = 2 * outputs * nest.k;
    const int64_t tile = bt_b * s.k_tile * (bt_m + bt_n);
    c.glb_ld = c.grid * steps * tile;
    c.shared_st = c.glb_ld;
    c.shared_ld = c.grid * c.block * nest.k * s.sp[0].pt * (s.sp[1].pt + s.sp[2].pt);
    c.int_ops = c.shared_ld;
    c.glb_st = outputs;
    c.active = std::min<int64_t>(c.grid, num_sms);
    c.sm_eff = (static_cast<double>(c.active) / num_sms) *
               std::min(1.0, static_cast<double>(c.block) / 256.0);
    return c;
}

void features_of(const Op& o, const Sched& s, const Counters& c, double* f) {
    // features.cpp:15-46
    const Nest nest = op_nest(o);
    auto lg = [](int64_t v) { return std::log1p(static_cast<double>(v)); };
    int64_t levels = 8;
    for (int d = 0; d < 3; ++d)
        if (s.sp[d].pt > 1) ++levels;
    f[0] = lg(c.flops);
    f[1] = lg(c.int_ops);
    f[2] = lg(c.glb_ld);
    f[3] = lg(c.glb_st);
    f[4] = lg(c.shared_ld);
    f[5] = lg(c.shared_st);
    f[6] = static_cast<double>(s.vec);
    f[7] = static_cast<double>(s.unroll);
    f[8] = lg(levels);
    f[9] = lg(s.sp[2].pt);
    f[10] = lg(nest.k / s.k_tile);
    f[11] = lg(c.grid);
    f[12] = lg(c.block);
    f[13] = c.sm_eff;
    f[14] = lg(c.active);
    f[15] = static_cast<double>(c.flops) / static_cast<double>(c.glb_ld + c.glb_st + 1);
}

// ----------------------------------------------------------------- genetic
std::vector<int64_t> legal_unrolls(int64_t k_tile, const Limits& l) {  // genetic.cpp:11-19
    std::vector<int64_t> out;
    for (int64_t u = 1; u <= std::max<int64_t>(1, l.max_unroll); u *= 2)
        if (k_tile % u == 0) out.push_back(u);
    return out;
}
std::vector<int64_t> legal_vectors(int64_t ptn, const Limits& l) {  // genetic.cpp:21-29
    std::vector<int64_t> out;
    const int64_t cap = std::min<int64_t>(4, l.max_vec);
    for (int64_t v = 1; v <= std::max<int64_t>(1, cap); v *= 2)
        if (ptn % v == 0) out.push_back(v);
    return out;
}
template <typename T, typename G>
T pick_different(const std::vector<T>& opts, const T& avoid, G& g) {  // genetic.cpp:32-44
    if (opts.size() <= 1) return opts.empty() ? avoid : opts.front();
    std::vector<T> alt;
    for (const T& o : opts)
        if (!(o == avoid)) alt.push_back(o);
    if (alt.empty()) return avoid;
    return alt[uniform_ab(g, 0, alt.size() - 1)];
}

template <typename G>
Sched mutate_knob(const Op& o, const Sched& s, int knob, const Limits& l, G& g) {
    // genetic.cpp:60-87
    const Nest nest = op_nest(o);
    Sched out = s;
    const int64_t ext[3] = {nest.b, nest.m, nest.n};
    switch (knob) {
    case 0:
    case 1:
    case 2:
        out.sp[knob] = pick_different(dim_tilings(ext[knob]), s.sp[knob], g);
        break;
    case 3:
        out.k_tile = pick_different(divisors(nest.k), s.k_tile, g);
        break;
    case 4:
        out.unroll = pick_different(legal_unrolls(out.k_tile, l), s.unroll, g);
        break;
    case 5:
        out.vec = pick_different(legal_vectors(out.sp[2].pt, l), s.vec, g);
        break;
    }
    return out;
}

template <typename G>
int repair(const Op& o, Sched s, const Limits& l, G& g, Sched* out) {  // genetic.cpp:89-135
    const int64_t cap = std::min<int64_t>(l.max_block, 1024);
    const Nest nest = op_nest(o);
    const int64_t ext[3] = {nest.b, nest.m, nest.n};
    for (int a = 0; a < 64 && s.block() > cap; ++a) {
        int dim = 0;
        for (int i = 1; i < 3; ++i)
            if (s.sp[i].threads > s.sp[dim].threads) dim = i;
        const int64_t other = s.block() / s.sp[dim].threads;
        std::vector<Tiling> fit;
        for (const Tiling& t : dim_tilings(ext[dim]))
            if (t.threads * other <= cap) fit.push_back(t);
        if (fit.empty()) {
            s.sp[dim] = {ext[dim], 1, 1};
        } else {
            s.sp[dim] = fit[uniform_ab(g, 0, fit.size() - 1)];
        }
    }
    if (s.k_tile < 1 || nest.k % s.k_tile != 0) s.k_tile = pick_different(divisors(nest.k), int64_t{0}, g);
    {
        const auto u = legal_unrolls(s.k_tile, l);
        if (std::find(u.begin(), u.end(), s.unroll) == u.end()) s.unroll = u[uniform_ab(g, 0, u.size() - 1)];
    }
    {
        const auto v = legal_vectors(s.sp[2].pt, l);
        if (std::find(v.begin(), v.end(), s.vec) == v.end()) s.vec = v[uniform_ab(g, 0, v.size() - 1)];
    }
    const int st = validate_schedule(o, s);
    if (st) return st;
    *out = s;
    return OK;
}

// ------------------------------------------------------------------ forest
struct Forest {
    const int32_t* feature;
    const double* threshold;
    const int32_t* left;
    const int32_t* right;
    const double* value;
    const int64_t* off;
    int64_t num_trees;
    double base, lr;
};
double tree_eval(const Forest& F, int64_t t, const double* f) {  // energy_model.cpp:36-44
    const int64_t b = F.off[t];
    int node = 0;
    while (F.feature[b + node] >= 0) {
        node = f[F.feature[b + node]] < F.threshold[b + node] ? F.left[b + node] : F.right[b + node];
    }
    return F.value[b + node];
}
double predict(const Forest& F, const double* f) {  // energy_model.cpp:245-249
    double sum = 0.0;
    for (int64_t t = 0; t < F.num_trees; ++t) sum += tree_eval(F, t, f);
    const double p = F.base + F.lr * sum;
    return (1e-6 < p) ? p : 1e-6;  // std::max(kPredictionFloor, p)
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_op_validate(const int64_t* op) { return op_validate(op_of(op)); }

int orc_op_nest(const int64_t* op, int64_t* out4) {
    const Op o = op_of(op);
    if (int st = op_validate(o)) return st;
    const Nest n = op_nest(o);
    out4[0] = n.b;
    out4[1] = n.m;
    out4[2] = n.n;
    out4[3] = n.k;
    return OK;
}

int orc_validate_schedule(const int64_t* op, const int64_t* sched) {
    return validate_schedule(op_of(op), sched_of(sched));
}

int orc_candidate_ids(const int64_t* op, const int64_t* sched, int64_t n, uint64_t* out) {
    const Op o = op_of(op);
    for (int64_t i = 0; i < n; ++i) out[i] = cand_id(o, sched_of(sched + 12 * i));
    return OK;
}

int orc_count_schedules(const int64_t* op, const int64_t* limits, int64_t cap, int64_t* out) {
    const Op o = op_of(op);
    if (int st = op_validate(o)) return st;
    *out = count_sched(o, limits_of(limits), cap);
    return OK;
}

int orc_enumerate(const int64_t* op, const int64_t* limits, int64_t cap, int64_t* out_sched,
                  int64_t* out_n) {
    const Op o = op_of(op);
    if (int st = op_validate(o)) return st;
    Enumerator en(o, limits_of(limits));
    Sched s;
    int64_t n = 0;
    while (n < cap && en.next(&s)) sched_put(s, out_sched + 12 * n++);
    *out_n = n;
    return OK;
}

// ------------------------------------------------------- measurement (sim)
// The reference declares SimBackend / sim_true_power_and_latency / nvml_sim_measure
// (measure.hpp:29-60, 102-114) but ships no implementation; SPEC:314-322 fixes the
// formula: latency = max(compute, memory, floor), power = constant + static*active +
// dynamic_energy / latency.  This restatement (parity unpinned by the reference) fixes
// the operation order, and the sampler noise -- SPEC:327's multiplicative Gaussian -- is made
// bit-reproducible on any IEEE machine: a standard normal per sample by Marsaglia's polar method
// over splitmix64 words, with ln built from +, *, / only (det_log), no libm.  The
// device kernel (paper_2411_18873_b200/csrc/measure.cu) follows it operation by
// operation.  Constants: 1000 iterations / 2 s sample window, samples
// capped at 4096 per measurement.
namespace {
uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
// ln s for s in (0, 1) from IEEE +, *, / only: s = m 2^e, m in [sqrt(1/2), sqrt(2)),
// ln m = 2 atanh((m - 1) / (m + 1)) by the odd series to t^23 (Horner in t^2), ln s =
// e ln2_hi + (e ln2_lo + ln m) -- the device kernel evaluates the same operations
const double kLogC[12] = {0x1p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
double det_log(double s) {
    uint64_t b;
    std::memcpy(&b, &s, 8);
    int e = int((b >> 52) & 0x7ffu) - 1023;
    const uint64_t mb = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
    double m;
    std::memcpy(&m, &mb, 8);
    if (m > 0x1.6a09e667f3bcdp+0) {
        m = m * 0.5;
        e += 1;
    }
    const double t = (m - 1.0) / (m + 1.0);
    const double t2 = t * t;
    double q = kLogC[11];
    for (int i = 10; i >= 0; --i) q = q * t2 + kLogC[i];
    const double lm = (t * q) * 2.0;
    const double de = static_cast<double>(e);
    return de * 0x1.62e42feep-1 + (de * 0x1.a39ef35793c76p-33 + lm);
}
// standard normal j of the stream `key`: Marsaglia's polar method, attempt a from the words
// key + 64 j + 2a and + 2a + 1 (v = 2u - 1, exact); 0 after 32 rejections
double det_normal(uint64_t key, int64_t j) {
    for (int a = 0; a < 32; ++a) {
        const uint64_t h1 = splitmix(key + static_cast<uint64_t>(j) * 64u + static_cast<uint64_t>(2 * a));
        const uint64_t h2 = splitmix(key + static_cast<uint64_t>(j) * 64u + static_cast<uint64_t>(2 * a + 1));
        const double v1 = static_cast<double>(h1 >> 11) * 0x1p-52 - 1.0;
        const double v2 = static_cast<double>(h2 >> 11) * 0x1p-52 - 1.0;
        const double s = v1 * v1 + v2 * v2;
        if (s > 0.0 && s < 1.0) return v1 * std::sqrt((-2.0 * det_log(s)) / s);
    }
    return 0.0;
}
struct SimDev {
    double num_sms, constant, static_sm, e_flop, e_glb, e_shared, tput, bw, floor_ms, hz, warmup, sigma;
    uint64_t seed;
};
void sim_measure(const Counters& c, const SimDev& d, uint64_t id, double* out4) {
    const double active = static_cast<double>(c.active);
    const double compute_s = static_cast<double>(c.flops) / ((active * d.tput) * c.sm_eff);
    const double memory_s = static_cast<double>(c.glb_ld + c.glb_st) / d.bw;
    double lat_ms = (compute_s > memory_s ? compute_s : memory_s) * 1000.0;
    if (lat_ms < d.floor_ms) lat_ms = d.floor_ms;
    const double dyn_mj = ((static_cast<double>(c.flops) * d.e_flop + static_cast<double>(c.glb_ld + c.glb_st) * d.e_glb) +
                           static_cast<double>(c.shared_ld + c.shared_st) * d.e_shared) * 1e-6;
    const double power = (d.constant + d.static_sm * active) + dyn_mj / lat_ms;
    const double lat_s = lat_ms / 1000.0;
    const double want = std::ceil(2.0 / lat_s);
    const int64_t iters = want > 1000.0 ? static_cast<int64_t>(want) : 1000;
    double sf = std::floor(static_cast<double>(iters) * lat_s * d.hz);
    if (sf < 1.0) sf = 1.0;
    if (sf > 4096.0) sf = 4096.0;
    const int64_t S = static_cast<int64_t>(sf);
    double avg = power;
    if (d.sigma != 0.0) {
        const uint64_t key = splitmix(d.seed ^ id);
        double sum = 0.0;
        for (int64_t j = 0; j < S; ++j) {
            const double z = det_normal(key, j);  // N(0, 1)
            sum += power * (1.0 + d.sigma * z);
        }
        avg = sum / static_cast<double>(S);
    }
    out4[0] = lat_ms;
    out4[1] = avg;
    out4[2] = avg * lat_ms;
    out4[3] = static_cast<double>(iters);
}
}  // namespace

/* dev13: num_sms, constant_w, static_per_sm_w, e_flop_nj, e_glb_nj, e_shared_nj,
 * throughput_flops_per_s_per_sm, bandwidth_elems_per_s, latency_floor_ms, sampler_hz,
 * warmup_s, noise_sigma_rel (doubles) ; seed separately.  out: n x {latency_ms,
 * avg_power_w, energy_mj, iterations}. */
int orc_sim_measure(const int64_t* op, const int64_t* sched, int64_t n, const double* dev12, uint64_t seed,
                    double* out) {
    const Op o = op_of(op);
    const SimDev d{dev12[0], dev12[1], dev12[2], dev12[3], dev12[4], dev12[5], dev12[6],
                   dev12[7], dev12[8], dev12[9], dev12[10], dev12[11], seed};
    const int sms = static_cast<int>(dev12[0]);
    for (int64_t i = 0; i < n; ++i) {
        const Sched s = sched_of(sched + 12 * i);
        if (int st = validate_schedule(o, s)) return st;
        sim_measure(derive(o, s, sms), d, cand_id(o, s), out + 4 * i);
    }
    return OK;
}

int orc_counters(const int64_t* op, const int64_t* sched, int64_t n, int num_sms, int64_t* out) {
    const Op o = op_of(op);
    for (int64_t i = 0; i < n; ++i) {
        const Sched s = sched_of(sched + 12 * i);
        if (int st = validate_schedule(o, s)) return st;
        const Counters c = derive(o, s, num_sms);
        int64_t* w = out + 10 * i;
        w[0] = c.grid;
        w[1] = c.block;
        w[2] = c.flops;
        w[3] = c.int_ops;
        w[4] = c.glb_ld;
        w[5] = c.glb_st;
        w[6] = c.shared_ld;
        w[7] = c.shared_st;
        std::memcpy(&w[8], &c.sm_eff, 8);
        w[9] = c.active;
    }
    return OK;
}

int orc_features(const int64_t* op, const int64_t* sched, int64_t n, int num_sms, double* out) {
    const Op o = op_of(op);
    for (int64_t i = 0; i < n; ++i) {
        const Sched s = sched_of(sched + 12 * i);
        if (int st = validate_schedule(o, s)) return st;
        features_of(o, s, derive(o, s, num_sms), out + 16 * i);
    }
    return OK;
}

int orc_mt64_words(uint64_t seed, int64_t n, uint64_t* out) {
    Mt64 g(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = g();
    return OK;
}
int orc_std_mt64_words(uint64_t seed, int64_t n, uint64_t* out) {
    std::mt19937_64 g(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = g();
    return OK;
}
uint64_t orc_lemire(uint64_t seed, int64_t draws, uint64_t range_size, uint64_t* out) {
    Mt64 g(seed);
    for (int64_t i = 0; i < draws; ++i) out[i] = uniform_ab(g, 0, range_size - 1);
    return g();  // next word: proves identical word consumption
}
uint64_t orc_std_uniform(uint64_t seed, int64_t draws, uint64_t range_size, uint64_t* out) {
    std::mt19937_64 g(seed);
    std::uniform_int_distribution<std::size_t> d(0, range_size - 1);
    for (int64_t i = 0; i < draws; ++i) out[i] = d(g);
    return g();
}
int orc_canonical(uint64_t seed, int64_t n, double* out) {
    Mt64 g(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = canonical(g);
    return OK;
}
int orc_std_canonical(uint64_t seed, int64_t n, double* out) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> d(0.0, 1.0);
    for (int64_t i = 0; i < n; ++i) out[i] = d(g);
    return OK;
}

int orc_sample_random(const int64_t* op, int64_t n, uint64_t seed, const int64_t* limits,
                      int64_t* out_sched, uint64_t* out_ids) {
    // space.cpp:170-251
    if (n < 1) return fail(VALIDATION, "sample_random requires n >= 1");
    const Op o = op_of(op);
    if (int st = op_validate(o)) return st;
    const Limits l = limits_of(limits);
    Mt64 g(seed);
    const int64_t mcap = std::max<int64_t>(2 * n, 4096);
    const int64_t counted = count_sched(o, l, mcap + 1);
    if (counted < n) return fail(SPACE_EXHAUSTED, "fewer legal schedules than requested");
    if (counted <= mcap) {
        std::vector<Sched> all;
        Enumerator en(o, l);
        Sched s;
        while (en.next(&s)) all.push_back(s);
        for (int64_t i = 0; i < n; ++i) {
            const uint64_t j = uniform_ab(g, static_cast<uint64_t>(i), all.size() - 1);
            std::swap(all[static_cast<size_t>(i)], all[j]);
            sched_put(all[static_cast<size_t>(i)], out_sched + 12 * i);
            out_ids[i] = cand_id(o, all[static_cast<size_t>(i)]);
        }
        return OK;
    }
    const Nest nest = op_nest(o);
    const std::vector<Tiling> til[3] = {dim_tilings(nest.b), dim_tilings(nest.m), dim_tilings(nest.n)};
    const std::vector<int64_t> kt = divisors(nest.k);
    const int64_t bcap = std::min<int64_t>(l.max_block, 1024);
    std::unordered_set<uint64_t> seen;
    int64_t attempts = 0, got = 0;
    const int64_t max_attempts = 10000 + n * 1000;
    while (got < n) {
        if (++attempts > max_attempts) return fail(SPACE_EXHAUSTED, "random sampling failed");
        Sched s;
        for (int d = 0; d < 3; ++d) s.sp[d] = til[d][uniform_ab(g, 0, til[d].size() - 1)];
        s.k_tile = kt[uniform_ab(g, 0, kt.size() - 1)];
        {
            std::vector<int64_t> legal;
            for (int64_t u = 1; u <= l.max_unroll && s.k_tile % u == 0; u *= 2) legal.push_back(u);
            s.unroll = legal[uniform_ab(g, 0, legal.size() - 1)];
        }
        {
            std::vector<int64_t> legal;
            for (int64_t v = 1; v <= std::min<int64_t>(4, l.max_vec) && s.sp[2].pt % v == 0; v *= 2)
                legal.push_back(v);
            s.vec = legal[uniform_ab(g, 0, legal.size() - 1)];
        }
        if (s.block() > bcap) continue;
        const uint64_t id = cand_id(o, s);
        if (!seen.insert(id).second) continue;
        sched_put(s, out_sched + 12 * got);
        out_ids[got] = id;
        ++got;
    }
    return OK;
}

}  // extern "C"

namespace {
// Counter-based word source of the opt-in counter reproduce mode (breed.cu CounterCursor): offspring
// i draws word_j = splitmix64(key_i + j) with key_i = splitmix64(seed ^ splitmix64(i)).
struct CounterGen {
    uint64_t key, j = 0;
    uint64_t operator()() { return splitmix(key + (j++)); }
};

// genetic.cpp:137-187 with the offspring's word source from `gen_of(i)` (the reference's one
// mt19937_64 stream, or a counter-based stream per offspring)
template <typename GenOf>
int reproduce_body(const int64_t* op, const int64_t* parent_sched, int64_t num_parents, int64_t n,
                   const double* rates, const int64_t* limits, int64_t* out_sched, uint64_t* out_ids,
                   uint64_t* out_lineage, int8_t* out_lineage_len, GenOf gen_of) {
    if (num_parents < 1) return fail(VALIDATION, "reproduce requires at least one parent");
    const Op o = op_of(op);
    const Limits l = limits_of(limits);
    const double mut = rates ? rates[0] : 0.85, cro = rates ? rates[1] : 0.10, cpy = rates ? rates[2] : 0.05;
    const double total = mut + cro + cpy;
    if (total <= 0.0) return fail(VALIDATION, "genetic rates must not all be zero");
    std::vector<Sched> par(static_cast<size_t>(num_parents));
    std::vector<uint64_t> pid(static_cast<size_t>(num_parents));
    for (int64_t p = 0; p < num_parents; ++p) {
        par[p] = sched_of(parent_sched + 12 * p);
        pid[p] = cand_id(o, par[p]);
    }
    for (int64_t i = 0; i < n; ++i) {
        auto& g = gen_of(i);
        const size_t bi = static_cast<size_t>(i) % par.size();
        const double u = canonical(g) * total;
        Sched s;
        if (u < mut) {
            const int knob = static_cast<int>(uniform_ab(g, 0, 5));
            s = mutate_knob(o, par[bi], knob, l, g);
            if (int st = repair(o, s, l, g, &s)) return st;
            out_lineage[2 * i] = pid[bi];
            out_lineage[2 * i + 1] = 0;
            out_lineage_len[i] = 1;
        } else if (u < mut + cro) {
            size_t pi = uniform_ab(g, 0, par.size() - 1);
            bool has_other = false;
            for (uint64_t x : pid)
                if (x != pid[bi]) has_other = true;
            while (has_other && pid[pi] == pid[bi]) pi = uniform_ab(g, 0, par.size() - 1);
            const uint64_t mask = g() & 63u;
            s = par[bi];
            const Sched& b = par[pi];
            if (mask & 1) s.sp[0] = b.sp[0];  // crossover_with_mask, genetic.cpp:48-58
            if (mask & 2) s.sp[1] = b.sp[1];
            if (mask & 4) s.sp[2] = b.sp[2];
            if (mask & 8) s.k_tile = b.k_tile;
            if (mask & 16) s.unroll = b.unroll;
            if (mask & 32) s.vec = b.vec;
            if (int st = repair(o, s, l, g, &s)) return st;
            out_lineage[2 * i] = pid[bi];
            out_lineage[2 * i + 1] = pid[pi];
            out_lineage_len[i] = 2;
        } else {
            s = par[bi];
            out_lineage[2 * i] = pid[bi];
            out_lineage[2 * i + 1] = 0;
            out_lineage_len[i] = 1;
        }
        sched_put(s, out_sched + 12 * i);
        out_ids[i] = cand_id(o, s);
    }
    return OK;
}
}  // namespace

extern "C" {

int orc_reproduce(const int64_t* op, const int64_t* parent_sched, int64_t num_parents, int64_t n,
                  const double* rates, uint64_t seed, const int64_t* limits, int64_t* out_sched,
                  uint64_t* out_ids, uint64_t* out_lineage, int8_t* out_lineage_len) {
    Mt64 g(seed);  // ONE sequential stream for the whole generation (genetic.cpp:155)
    return reproduce_body(op, parent_sched, num_parents, n, rates, limits, out_sched, out_ids, out_lineage,
                          out_lineage_len, [&](int64_t) -> Mt64& { return g; });
}

/* The opt-in counter mode (etune_cu_reproduce_counter): the same decisions, each offspring on its own
 * counter-based stream.  Test infrastructure like every orc_* function. */
int orc_reproduce_counter(const int64_t* op, const int64_t* parent_sched, int64_t num_parents, int64_t n,
                          const double* rates, uint64_t seed, const int64_t* limits, int64_t* out_sched,
                          uint64_t* out_ids, uint64_t* out_lineage, int8_t* out_lineage_len) {
    CounterGen g{0};
    return reproduce_body(op, parent_sched, num_parents, n, rates, limits, out_sched, out_ids, out_lineage,
                          out_lineage_len, [&](int64_t i) -> CounterGen& {
                              g = CounterGen{splitmix(seed ^ splitmix(static_cast<uint64_t>(i)))};
                              return g;
                          });
}

int orc_predict(const int32_t* feature, const double* threshold, const int32_t* left,
                const int32_t* right, const double* value, const int64_t* tree_offsets,
                int64_t num_trees, double base_score, double learning_rate, const double* feats,
                int64_t n, double* out) {
    const Forest F{feature, threshold, left, right, value, tree_offsets, num_trees, base_score, learning_rate};
    for (int64_t i = 0; i < n; ++i) out[i] = predict(F, feats + 16 * i);
    return OK;
}

int orc_energy_loss(double pred, double meas, double* out3) {  // energy_model.cpp:23-34
    if (!(meas > 0.0)) return fail(NON_POSITIVE_ENERGY, "measured energy must be positive");
    const double diff = pred - meas;
    out3[0] = diff * diff / meas;
    out3[1] = 2.0 * diff / meas;
    out3[2] = 2.0 / meas;
    return OK;
}

int orc_train(const double* feats, const double* energy, int64_t n64, int num_trees, int max_depth,
              double lr, double min_leaf_weight, double lambda, int32_t* o_feature, double* o_thr,
              int32_t* o_left, int32_t* o_right, double* o_value, int64_t* o_off, double* o_base,
              double* o_ref, double* o_loss) {
    // energy_model.cpp:173-243 (+ TreeBuilder 48-169)
    if (n64 < 2) return fail(INSUFFICIENT_DATA, "training needs at least 2 samples");
    double reference = INFINITY;
    for (int64_t i = 0; i < n64; ++i) {
        if (!(energy[i] > 0.0)) return fail(NON_POSITIVE_ENERGY, "training sample with non-positive energy");
        reference = std::min(reference, energy[i]);
    }
    const int n = static_cast<int>(n64);
    std::vector<double> target(n);
    for (int i = 0; i < n; ++i) target[i] = energy[i] / reference;
    double inv = 0.0;
    for (double y : target) inv += 1.0 / y;
    const double base = static_cast<double>(n) / inv;
    auto F = [&](int i, int f) { return feats[16 * static_cast<int64_t>(i) + f]; };
    std::vector<std::vector<int>> sorted(16);
    for (int f = 0; f < 16; ++f) {
        sorted[f].resize(n);
        for (int i = 0; i < n; ++i) sorted[f][i] = i;
        std::stable_sort(sorted[f].begin(), sorted[f].end(), [&](int a, int b) { return F(a, f) < F(b, f); });
    }
    std::vector<double> pred(n, base), grad(n), hess(n);
    auto mean_loss = [&]() {
        double t = 0.0;
        for (int i = 0; i < n; ++i) {
            const double d = pred[i] - target[i];
            t += d * d / target[i];
        }
        return t / static_cast<double>(n);
    };
    if (o_loss) o_loss[0] = mean_loss();
    int64_t node_base = 0;
    for (int round = 0; round < num_trees; ++round) {
        for (int i = 0; i < n; ++i) {
            const double d = pred[i] - target[i];
            grad[i] = 2.0 * d / target[i];
            hess[i] = 2.0 / target[i];
        }
        // ---- TreeBuilder::build
        struct Node {
            int feature = -1;
            double thr = 0.0;
            int left = -1, right = -1;
            double value = 0.0;
        };
        struct Stat {
            double g = 0.0, h = 0.0;
        };
        struct Best {
            double gain = 0.0;
            int feature = -1;
            double thr = 0.0;
        };
        auto obj = [&](const Stat& s) { return s.g * s.g / (s.h + lambda); };
        std::vector<Node> nodes(1);
        std::vector<int> node_of(n, 0);
        std::vector<Stat> stats(1);
        for (int i = 0; i < n; ++i) {
            stats[0].g += grad[i];
            stats[0].h += hess[i];
        }
        std::vector<int> frontier = {0};
        for (int depth = 0; depth < max_depth && !frontier.empty(); ++depth) {
            const size_t nn = nodes.size();
            std::vector<Best> best(nn);
            std::vector<Stat> run(nn);
            std::vector<double> prev(nn, 0.0);
            std::vector<char> has_prev(nn, 0), active(nn, 0);
            for (int id : frontier) active[id] = 1;
            for (int f = 0; f < 16; ++f) {
                for (int id : frontier) {
                    run[id] = Stat{};
                    has_prev[id] = 0;
                }
                for (int idx : sorted[f]) {
                    const int id = node_of[idx];
                    if (!active[id]) continue;
                    const double v = F(idx, f);
                    Stat& r = run[id];
                    if (has_prev[id] && v > prev[id]) {
                        const Stat& tot = stats[id];
                        const Stat right{tot.g - r.g, tot.h - r.h};
                        if (r.h >= min_leaf_weight && right.h >= min_leaf_weight) {
                            const double gain = 0.5 * (obj(r) + obj(right) - obj(tot));
                            Best& b = best[id];
                            if (gain > 1e-12 && gain > b.gain) {
                                b.gain = gain;
                                b.feature = f;
                                b.thr = 0.5 * (prev[id] + v);
                            }
                        }
                    }
                    r.g += grad[idx];
                    r.h += hess[idx];
                    prev[id] = v;
                    has_prev[id] = 1;
                }
            }
            std::vector<int> next;
            for (int id : frontier) {
                const Best& b = best[id];
                if (b.feature < 0) continue;
                nodes[id].feature = b.feature;
                nodes[id].thr = b.thr;
                nodes[id].left = static_cast<int>(nodes.size());
                nodes[id].right = nodes[id].left + 1;
                nodes.push_back(Node{});
                nodes.push_back(Node{});
                stats.resize(nodes.size());
                next.push_back(nodes[id].left);
                next.push_back(nodes[id].right);
            }
            if (next.empty()) break;
            for (int i = 0; i < n; ++i) {
                int id = node_of[i];
                const Node& nd = nodes[id];
                if (nd.feature < 0) continue;
                id = F(i, nd.feature) < nd.thr ? nd.left : nd.right;
                node_of[i] = id;
                stats[id].g += grad[i];
                stats[id].h += hess[i];
            }
            frontier = std::move(next);
        }
        for (size_t id = 0; id < nodes.size(); ++id) {
            if (nodes[id].feature >= 0) continue;
            nodes[id].value = -stats[id].g / (stats[id].h + lambda);
        }
        // ---- emit + update predictions (energy_model.cpp:234-240)
        o_off[round] = node_base;
        for (size_t id = 0; id < nodes.size(); ++id) {
            o_feature[node_base + id] = nodes[id].feature;
            o_thr[node_base + id] = nodes[id].thr;
            o_left[node_base + id] = nodes[id].left;
            o_right[node_base + id] = nodes[id].right;
            o_value[node_base + id] = nodes[id].value;
        }
        for (int i = 0; i < n; ++i) {
            int node = 0;
            while (nodes[node].feature >= 0)
                node = F(i, nodes[node].feature) < nodes[node].thr ? nodes[node].left : nodes[node].right;
            pred[i] += lr * nodes[node].value;
        }
        node_base += static_cast<int64_t>(nodes.size());
        if (o_loss) o_loss[round + 1] = mean_loss();
    }
    o_off[num_trees] = node_base;
    *o_base = base;
    *o_ref = reference;
    return OK;
}

int orc_snr_db(const double* pred, const double* meas, int64_t n, double* out) {
    // energy_model.cpp:352-370
    if (n == 0) return fail(EMPTY_INPUT, "snr_db requires non-empty input");
    double signal = 0.0, error = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (!(meas[i] > 0.0)) return fail(NON_POSITIVE_ENERGY, "snr_db requires positive measurements");
        signal += meas[i] * meas[i];
        const double d = pred[i] - meas[i];
        error += d * d;
    }
    if (error <= 0.0) {
        *out = 100.0;
        return OK;
    }
    *out = std::min(100.0, 10.0 * std::log10(signal / error));
    return OK;
}

int orc_topk(const double* score, int64_t n, int64_t k, int64_t* out_idx) {
    if (k < 0 || k > n) return fail(VALIDATION, "k outside [0, n]");
    std::vector<int64_t> idx(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return score[a] < score[b]; });
    for (int64_t i = 0; i < k; ++i) out_idx[i] = idx[i];
    return OK;
}

int orc_score_threads(const int64_t* op, const int64_t* sched, int64_t n, int num_sms,
                      const int32_t* feature, const double* threshold, const int32_t* left,
                      const int32_t* right, const double* value, const int64_t* tree_offsets,
                      int64_t num_trees, double base_score, double learning_rate, int threads,
                      double* out_pred) {
    const Op o = op_of(op);
    const Forest F{feature, threshold, left, right, value, tree_offsets, num_trees, base_score, learning_rate};
    if (threads < 1) threads = 1;
    std::atomic<int> bad{0};
    auto work = [&](int64_t lo, int64_t hi) {
        double f[16];
        for (int64_t i = lo; i < hi; ++i) {
            const Sched s = sched_of(sched + 12 * i);
            if (validate_schedule(o, s)) {
                bad = 1;
                return;
            }
            features_of(o, s, derive(o, s, num_sms), f);
            out_pred[i] = predict(F, f);
        }
    };
    std::vector<std::thread> pool;
    const int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
    return bad ? fail(ILLEGAL_SCHEDULE, "illegal schedule in population") : OK;
}

}  // extern "C"

// ---------------------------------------------------------- Algorithm 1 (search)
// CPU restatement of the search loop (the reference has no
// code) built from the restated primitives above, step for step what
// paper_2411_18873_b200/csrc/search.cpp does on the device.  cfg_i: M, generation_size,
// k_init_fifths, max_rounds, patience, inverted, num_trees, max_depth, latency_only
// (run_latency_only); cfg_d: mu_db,
// improve_rel, mutation, crossover, copy, learning_rate, min_leaf_weight, reg_lambda.
// Reports: rep_i n x {round, k_before, k_after, measured, cumulative, best_id},
// rep_d n x {snr_db, best_latency_ms, best_energy_mj, best_power_w}.
extern "C" int orc_run_search(const int64_t* op, const int64_t* limits, const double* dev12, uint64_t dev_seed,
                              const int64_t* cfg_i, const double* cfg_d, uint64_t seed, int64_t max_reports,
                              int64_t* rep_i, double* rep_d, int64_t* n_reports, int64_t* out_parents,
                              int64_t* n_parents) {
    const int64_t M = cfg_i[0], G = cfg_i[1];
    int k5 = int(cfg_i[2]);
    const int64_t max_rounds = cfg_i[3], patience = cfg_i[4], inverted = cfg_i[5];
    const int trees = int(cfg_i[6]), depth = int(cfg_i[7]);
    const bool latency_only = cfg_i[8] != 0;
    const double mu = cfg_d[0], improve = cfg_d[1], rates[3] = {cfg_d[2], cfg_d[3], cfg_d[4]};
    const double lr = cfg_d[5], mlw = cfg_d[6], lam = cfg_d[7];
    const int sms = int(dev12[0]);
    using VI = std::vector<int64_t>;
    using VD = std::vector<double>;
    auto sched_rows = [](const VI& all, const VI& idx) {
        VI out(idx.size() * 12);
        for (size_t j = 0; j < idx.size(); ++j)
            std::copy(all.begin() + 12 * idx[j], all.begin() + 12 * idx[j] + 12, out.begin() + 12 * j);
        return out;
    };
    VD feats, energy;  // accumulated samples
    const size_t cap_nodes = size_t(std::max(trees, 1)) * ((size_t(1) << (depth + 1)) - 1);
    std::vector<int32_t> fe(cap_nodes), le(cap_nodes), ri(cap_nodes);
    VD th(cap_nodes), va(cap_nodes), loss(size_t(trees) + 1);
    std::vector<int64_t> off(size_t(trees) + 1);
    double base = 0, ref = 0;
    auto retrain = [&]() {
        return orc_train(feats.data(), energy.data(), int64_t(energy.size()), trees, depth, lr, mlw, lam, fe.data(),
                         th.data(), le.data(), ri.data(), va.data(), off.data(), &base, &ref, loss.data());
    };
    bool have_best = false;
    uint64_t best_id = 0;
    double best_lat = 0, best_en = 0, best_pow = 0;
    int64_t cumulative = 0, stall = 0, nrep = 0;
    auto update_best = [&](const VI& s, const VD& m4) -> bool {
        const int64_t n = int64_t(s.size() / 12);
        std::vector<uint64_t> ids(static_cast<size_t>(n));
        orc_candidate_ids(op, s.data(), n, ids.data());
        const double before = have_best ? best_en : std::numeric_limits<double>::infinity();
        for (int64_t i = 0; i < n; ++i) {
            const double l = m4[4 * i], p = m4[4 * i + 1], e = m4[4 * i + 2];
            const bool better = !have_best || e < best_en ||
                                (e == best_en && (l < best_lat || (l == best_lat && ids[i] < best_id)));
            if (better) {
                have_best = true;
                best_en = e;
                best_lat = l;
                best_id = ids[i];
                best_pow = p;
            }
        }
        return best_en < before * (1.0 - improve);
    };
    // run_latency_only: best = lowest latency (then id) of the rounds' fastest candidates,
    // whose energy is measured for the report
    auto update_best_latency = [&](const VI& s1) -> bool {
        VD m1(4);
        orc_sim_measure(op, s1.data(), 1, dev12, dev_seed, m1.data());
        uint64_t id = 0;
        orc_candidate_ids(op, s1.data(), 1, &id);
        const double before = have_best ? best_lat : std::numeric_limits<double>::infinity();
        if (!have_best || m1[0] < best_lat || (m1[0] == best_lat && id < best_id)) {
            have_best = true;
            best_lat = m1[0];
            best_pow = m1[1];
            best_en = m1[2];
            best_id = id;
        }
        return best_lat < before * (1.0 - improve);
    };
    auto report = [&](int64_t round, int kb, double snr, int64_t measured) {
        if (nrep < max_reports) {
            int64_t* ri = rep_i + 6 * nrep;
            double* rd = rep_d + 4 * nrep;
            ri[0] = round;
            ri[1] = kb;
            ri[2] = k5;
            ri[3] = measured;
            ri[4] = cumulative;
            std::memcpy(&ri[5], &best_id, 8);
            rd[0] = snr;
            rd[1] = best_lat;
            rd[2] = best_en;
            rd[3] = best_pow;
        }
        ++nrep;
    };
    // initial round
    VI pop(size_t(G) * 12);
    std::vector<uint64_t> pid(static_cast<size_t>(G));
    if (int st = orc_sample_random(op, G, seed, limits, pop.data(), pid.data())) return st;
    VD m4(size_t(G) * 4);
    if (int st = orc_sim_measure(op, pop.data(), G, dev12, dev_seed, m4.data())) return st;
    VD lat(static_cast<size_t>(G));
    for (int64_t i = 0; i < G; ++i) lat[i] = m4[4 * i];
    VI idx(static_cast<size_t>(M));
    orc_topk(lat.data(), G, M, idx.data());
    VI mg = sched_rows(pop, idx);
    if (latency_only) {
        VI par = mg;
        cumulative = 1;
        update_best_latency(VI(mg.begin(), mg.begin() + 12));
        report(0, k5, std::numeric_limits<double>::quiet_NaN(), 1);
        for (int64_t r = 1; r <= max_rounds && stall < patience; ++r) {
            const int64_t np = int64_t(par.size() / 12);
            VI off_s(size_t(G) * 12);
            std::vector<uint64_t> oid(static_cast<size_t>(G)), lin(size_t(G) * 2);
            std::vector<int8_t> ll(static_cast<size_t>(G));
            if (int st = orc_reproduce(op, par.data(), np, G, rates, seed + uint64_t(r), limits, off_s.data(),
                                       oid.data(), lin.data(), ll.data()))
                return st;
            orc_sim_measure(op, off_s.data(), G, dev12, dev_seed, m4.data());
            for (int64_t i = 0; i < G; ++i) lat[i] = m4[4 * i];
            orc_topk(lat.data(), G, M, idx.data());
            mg = sched_rows(off_s, idx);
            const int64_t npar = (M + 1) / 2;  // the ceil(M/2) fastest
            par.assign(mg.begin(), mg.begin() + 12 * npar);
            cumulative += 1;
            const bool improved = update_best_latency(VI(mg.begin(), mg.begin() + 12));
            stall = improved ? 0 : stall + 1;
            report(r, k5, std::numeric_limits<double>::quiet_NaN(), 1);
        }
        *n_reports = nrep;
        *n_parents = int64_t(par.size() / 12);
        if (out_parents) std::copy(par.begin(), par.end(), out_parents);
        return OK;
    }
    VD mm(size_t(M) * 4);
    orc_sim_measure(op, mg.data(), M, dev12, dev_seed, mm.data());
    feats.resize(size_t(M) * 16);
    orc_features(op, mg.data(), M, sms, feats.data());
    for (int64_t i = 0; i < M; ++i) energy.push_back(mm[4 * i + 2]);
    if (int st = retrain()) return st;
    VI par = mg;
    cumulative = M;
    update_best(mg, mm);
    report(0, k5, std::numeric_limits<double>::quiet_NaN(), M);
    for (int64_t r = 1; r <= max_rounds && stall < patience; ++r) {
        const int64_t np = int64_t(par.size() / 12);
        VI off_s(size_t(G) * 12);
        std::vector<uint64_t> oid(static_cast<size_t>(G)), lin(size_t(G) * 2);
        std::vector<int8_t> ll(static_cast<size_t>(G));
        if (int st = orc_reproduce(op, par.data(), np, G, rates, seed + uint64_t(r), limits, off_s.data(), oid.data(),
                                   lin.data(), ll.data()))
            return st;
        orc_sim_measure(op, off_s.data(), G, dev12, dev_seed, m4.data());
        for (int64_t i = 0; i < G; ++i) lat[i] = m4[4 * i];
        orc_topk(lat.data(), G, M, idx.data());
        mg = sched_rows(off_s, idx);
        VD f(size_t(M) * 16), pred(static_cast<size_t>(M));
        orc_features(op, mg.data(), M, sms, f.data());
        orc_predict(fe.data(), th.data(), le.data(), ri.data(), va.data(), off.data(), trees, base, lr, f.data(), M,
                    pred.data());
        int64_t km = (int64_t(k5) * M + 4) / 5;
        if (km < 1) km = 1;
        VI sel(static_cast<size_t>(km));
        orc_topk(pred.data(), M, km, sel.data());
        VI sg = sched_rows(mg, sel);
        VD sm(size_t(km) * 4), psel(static_cast<size_t>(km)), mnorm(static_cast<size_t>(km));
        orc_sim_measure(op, sg.data(), km, dev12, dev_seed, sm.data());
        for (int64_t i = 0; i < km; ++i) {
            psel[i] = pred[sel[i]];
            mnorm[i] = sm[4 * i + 2] / ref;
        }
        double snr = 0.0;
        if (int st = orc_snr_db(psel.data(), mnorm.data(), km, &snr)) return st;
        const int64_t npar = (M + 1) / 2;
        VI pidx(static_cast<size_t>(npar));
        orc_topk(pred.data(), M, npar, pidx.data());
        par = sched_rows(mg, pidx);
        const size_t old = feats.size();
        feats.resize(old + size_t(km) * 16);
        orc_features(op, sg.data(), km, sms, feats.data() + old);
        for (int64_t i = 0; i < km; ++i) energy.push_back(sm[4 * i + 2]);
        if (int st = retrain()) return st;
        const int kb = k5;
        const bool poor = inverted ? !(snr < mu) : (snr < mu);
        k5 = poor ? std::min(5, k5 + 1) : std::max(0, k5 - 1);
        cumulative += km;
        const bool improved = update_best(sg, sm);
        stall = improved ? 0 : stall + 1;
        report(r, kb, snr, km);
    }
    *n_reports = nrep;
    const int64_t np = int64_t(par.size() / 12);
    *n_parents = np;
    if (out_parents) std::copy(par.begin(), par.end(), out_parents);
    return OK;
}
