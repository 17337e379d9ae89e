// reproduce() for large generations on the whole GPU, bit-exact with the reference's ONE
// sequential std::mt19937_64 stream (genetic.cpp:137-187).
//
// Offspring i starts at word o_i of the stream and consumes c(i, o_i) words, a function of
// the words at o_i.. and of the base parent parents[i % P]; o_{i+1} = o_i + c(i, o_i) is a
// sequential chain.  breed_kernel walks it on one CTA (243 ns per offspring).
// Here the chain is cut into blocks of S offspring and resolved block-parallel:
//
//   est   c(i, .) at 4 counter-generated word positions per offspring: the mean and variance
//         of the words each block consumes (any uniform 64-bit source has the same consumption
//         law).  Only window placement depends on it; results never do.
//   plan  block b's start o_{bS} lies within +-5 sd of the estimated prefix with overwhelming
//         probability: a window [lo_b, lo_b + W_b) of candidate starts, cut into chunks of
//         kWc starts (one "item" each).
//   win   ONE launch: the CTA that draws ticket 0 generates the reference's word stream
//         (mt19937_64(seed)) into HBM, 156 words per dependent step, publishing its progress;
//         every other CTA takes the next item, waits until the words it may read exist, and
//         walks EVERY start of its chunk through the block at once.  Walks that land on the same
//         word at the same offspring are identical from then on and are merged (a tagged
//         atomicMax in a shared hash, confirmed by comparing positions); the live set thins like
//         coalescing random walks (~W/45 left after 2048 steps) and is compacted every step.
//         The stream the walkers read is staged in a shared-memory ring that slides along the
//         chunk's mean path (cp.async, far ahead of use).  Output: the end position of every
//         start, the merge forest, and the live walkers' positions every Q offspring.
//   chain one thread follows the true chain across blocks, one lookup per block
//         (o_{(b+1)S} = end_b[o_{bS} - lo_b]); a start outside its window, or a walk that met an
//         illegal schedule or left the words its item waited for, is walked exactly on the spot.
//   emit  one thread per Q-offspring sub-block: its true start from the merge forest and the
//         snapshots, then the Q offspring evaluated at their true offsets -> genomes, partners.
//
// Every emitted child is breed_body() evaluated at its true word offset — the speculation
// (windows, merges) only decides where the true offsets are found, never what the children
// are.  When the stream does not fit its buffer the chain kernel leaves `done` = 0 and the
// single-CTA breed_kernel launched after it produces the generation.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "breed_core.cuh"
#include "etune_internal.hpp"
#include "kernels.hpp"
#include "mt64.cuh"

namespace etune_b200 {

namespace {

using namespace breedcore;

constexpr int kQ = 64;                  // offspring per emitted sub-block
constexpr int kWinT = 256;              // threads per window CTA (>= 156: the generator)
constexpr int kWc = 2048;               // starts per window item (chunk-local u16 walker ids)
constexpr int kRing = 2560;             // stream words staged per window CTA (slot p % kRing)
constexpr int kRingMargin = 256;        // the ring starts this many words behind the chunk's mean path
constexpr int kEpoch = 16;              // steps per epoch: claims, merges, ring slide, compaction once per epoch
static_assert(kQ % kEpoch == 0, "snapshots fall on epoch ends");
constexpr int kHash = 4096;             // merge hash slots (>= the live positions' span)
constexpr int kWcap = 16 * kWc;         // window starts per block at most
constexpr int kEstK = 4;                // consumption samples per offspring
constexpr int kEstThreads = 256;
constexpr int kGenCols = 156;           // mt19937_64: x[k+312] = x[k+156] ^ twist(x[k], x[k+1])
static_assert(kWinT >= kGenCols, "the generator runs one column per thread");
constexpr uint32_t kFateUnknown = 0xffffffffu;
constexpr uint32_t kFateIllegal = 0xfffffffeu;
constexpr uint32_t kGone = 0xffffffffu;  // pos[] of a walker that met a fate

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

struct ParHdr {
    unsigned long long L;          // stream words generated
    unsigned long long progress;   // words generated so far (the generator publishes it)
    unsigned long long snap_used;  // snapshot pool entries reserved
    int32_t status;                // 0 ok; 1 does not fit: the single-CTA chain produces the generation
    int32_t nres;                  // blocks the chain resolved (blocks past an illegal child are not)
    int32_t done;                  // the parallel path produced the generation (breed_kernel exits)
    int32_t other;                 // has_other
    int32_t items;                 // window items
    uint32_t ticket;               // window CTAs started
};

struct BlockWin {
    uint32_t lo, W, woff, ioff;  // window start, size, offset in the per-start arrays, first item
    uint32_t need;               // words this block's items may read
    float mean;                  // estimated words per offspring in this block
    uint32_t pad[2];
};

// Cursor over the generated stream in HBM with the first four words prefetched (an
// evaluation's words are consecutive, so one round trip covers nearly every offspring).
struct GCursor {
    const uint64_t* w;
    uint64_t p, hi, base;
    uint64_t c0, c1, c2, c3;
    bool ok;
    __device__ __forceinline__ GCursor(const uint64_t* s, uint64_t start, uint64_t h)
        : w(s), p(start), hi(h), base(start), ok(true) {
        // the stream buffer is padded by 8 words past its capacity, so these loads stay in bounds
        c0 = __ldg(s + start);
        c1 = __ldg(s + start + 1);
        c2 = __ldg(s + start + 2);
        c3 = __ldg(s + start + 3);
    }
    __device__ __forceinline__ uint64_t next() {
        if (p >= hi) {
            ok = false;
            return 0;
        }
        const uint64_t k = p - base;
        uint64_t x;
        if (k == 0) x = c0;
        else if (k == 1) x = c1;
        else if (k == 2) x = c2;
        else if (k == 3) x = c3;
        else x = __ldg(w + p);
        ++p;
        return x;
    }
};

// Cursor of the window walkers: the shared ring when the word is staged there, else L2
// (ld.cg: the stream is written during this launch, so nothing goes through L1).
struct RCursor {
    const uint64_t* ring;
    const uint64_t* w;
    int64_t base, vhi;  // the ring holds words [base, vhi) (vhi <= base + kRing: copies landed)
    uint64_t p, hi;
    bool ok;
    __device__ __forceinline__ uint64_t next() {
        if (p >= hi) {
            ok = false;
            return 0;
        }
        const int64_t q = int64_t(p);
        const uint64_t x = (q >= base && q < vhi) ? ring[uint32_t(p) % kRing] : __ldcg(w + p);
        ++p;
        return x;
    }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// exclusive block scan of one u32 per thread (blockDim multiple of 32, <= 1024); ends with a barrier
__device__ __forceinline__ uint32_t block_scan_u32(uint32_t v, uint32_t* total, uint32_t* ws) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
        if (lane >= s) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t y = lane < nw ? ws[lane] : 0u;
        for (int s = 1; s < 32; s <<= 1) {
            const uint32_t z = __shfl_up_sync(0xffffffffu, y, s);
            if (lane >= s) y += z;
        }
        if (lane < nw) ws[lane] = y;  // inclusive
    }
    __syncthreads();
    const uint32_t before = wid > 0 ? ws[wid - 1] : 0u;
    *total = ws[nw - 1];
    __syncthreads();
    return before + x - v;
}

// has_other (genetic.cpp:172-174): some parent id differs from the first; header reset
__global__ void breed_other_kernel(const uint64_t* __restrict__ pid, int64_t np, ParHdr* hdr) {
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const uint64_t id0 = __ldg(pid);
    int diff = 0;
    for (int64_t j = threadIdx.x; j < np; j += blockDim.x) diff |= __ldg(pid + j) != id0;
    if (__syncthreads_or(diff) && threadIdx.x == 0) s = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        hdr->other = s;
        hdr->status = 0;
        hdr->done = 0;
        hdr->nres = 0;
        hdr->snap_used = 0;
        hdr->progress = 0;
        hdr->ticket = 0;
        hdr->items = 0;
    }
}

// per block: sum over its offspring of the sample mean and variance of the words consumed
__global__ void __launch_bounds__(kEstThreads) breed_est_kernel(const uint8_t* __restrict__ gplan,
                                                                const uint64_t* __restrict__ par,
                                                                const uint64_t* __restrict__ pid, int64_t np, int64_t n,
                                                                int S, double mut, double mutcro, double total,
                                                                uint64_t seed, const ParHdr* __restrict__ hdr,
                                                                double2* __restrict__ est) {
    __shared__ double rm[kEstThreads / 32], rv[kEstThreads / 32];
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(gplan);
    const BreedConst K{gplan, par, pid, np, mut, mutcro, total, hdr->other};
    const int64_t i0 = int64_t(blockIdx.x) * S;
    const int64_t i1 = imin64(n, i0 + S);
    double sm = 0.0, sv = 0.0;
    const uint64_t key0 = splitmix64(seed ^ 0x6a09e667f3bcc909ull);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        double a = 0.0, a2 = 0.0;
        for (int s = 0; s < kEstK; ++s) {
            CounterCursor c{splitmix64(key0 + uint64_t(i) * kEstK + uint64_t(s)), 0, true};
            (void)breed_body(K, H, i, c, 0);
            const double w = double(c.p);
            a += w;
            a2 += w * w;
        }
        sm += a / kEstK;
        sv += (a2 - a * a / kEstK) / (kEstK - 1);
    }
    for (int s = 16; s > 0; s >>= 1) {
        sm += __shfl_xor_sync(0xffffffffu, sm, s);
        sv += __shfl_xor_sync(0xffffffffu, sv, s);
    }
    if ((threadIdx.x & 31) == 0) {
        rm[threadIdx.x >> 5] = sm;
        rv[threadIdx.x >> 5] = sv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0, v = 0.0;
        for (int w = 0; w < kEstThreads / 32; ++w) {
            m += rm[w];
            v += rv[w];
        }
        est[blockIdx.x] = make_double2(m, v);
    }
}

// windows from the prefix sums of the block estimates; items; the stream length to generate
__global__ void __launch_bounds__(1024) breed_plan_kernel(const double2* __restrict__ est, int B, int S, int64_t n,
                                                          uint64_t cap, double sd_mult, BlockWin* __restrict__ win,
                                                          ParHdr* hdr) {
    __shared__ double cm[1024], cv[1024];
    __shared__ uint32_t cw[1024], ci[1024];
    __shared__ unsigned long long s_need;
    const int per = (B + 1023) / 1024;
    const int b0 = threadIdx.x * per, b1 = min(B, b0 + per);
    double m = 0.0, v = 0.0;
    for (int b = b0; b < b1; ++b) {
        m += est[b].x;
        v += est[b].y;
    }
    cm[threadIdx.x] = m;
    cv[threadIdx.x] = v;
    if (threadIdx.x == 0) s_need = 0;
    __syncthreads();
    if (threadIdx.x == 0) {  // 1024 partial sums: serial exclusive scan
        double am = 0.0, av = 0.0;
        for (int t = 0; t < 1024; ++t) {
            const double x = cm[t], y = cv[t];
            cm[t] = am;
            cv[t] = av;
            am += x;
            av += y;
        }
    }
    __syncthreads();
    m = cm[threadIdx.x];
    v = cv[threadIdx.x];
    uint32_t wsum = 0, isum = 0;
    unsigned long long need = 0;
    for (int b = b0; b < b1; ++b) {
        uint64_t lo = 0, W = 1;
        const uint64_t floor_b = uint64_t(int64_t(b) * S);  // every offspring draws >= 1 word
        if (b > 0) {
            const double h = sd_mult * sqrt(v * (1.0 + 1.0 / kEstK)) + 8.0;
            const double l = floor(m - h);
            lo = l > double(floor_b) ? uint64_t(l) : floor_b;
            const uint64_t hi = uint64_t(ceil(m + h));
            W = hi >= lo ? hi - lo + 1 : 1;
            if (W > uint64_t(kWcap)) {  // keep the centre; the chain walks a miss exactly
                const uint64_t c = uint64_t(m);
                lo = c > uint64_t(kWcap / 2) ? c - uint64_t(kWcap / 2) : 0;
                if (lo < floor_b) lo = floor_b;
                W = kWcap;
            }
        }
        const double bm = est[b].x, bv = est[b].y;
        const int64_t nb = imin64(S, n - int64_t(b) * S);
        const unsigned long long e =
            (unsigned long long)(lo + W) + (unsigned long long)(ceil(bm + 10.0 * sqrt(bv) + 64.0));
        need = e > need ? e : need;
        win[b].lo = uint32_t(lo);
        win[b].W = uint32_t(W);
        win[b].need = uint32_t(e < 0xfffffff0ull ? e : 0xfffffff0ull);
        win[b].mean = float(bm / double(nb));
        m += est[b].x;
        v += est[b].y;
        wsum += uint32_t(W);
        isum += uint32_t((W + kWc - 1) / kWc);
    }
    atomicMax(&s_need, need);
    cw[threadIdx.x] = wsum;
    ci[threadIdx.x] = isum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0, c = 0;
        for (int t = 0; t < 1024; ++t) {
            const uint32_t x = cw[t], y = ci[t];
            cw[t] = a;
            ci[t] = c;
            a += x;
            c += y;
        }
        const unsigned long long L = ((s_need + 311) / 312) * 312;
        if (L > cap || L >= 0xfffffff0ull) hdr->status = 1;  // does not fit: breed_kernel produces it
        hdr->L = L;
        hdr->items = int32_t(c);
    }
    __syncthreads();
    uint32_t off = cw[threadIdx.x], io = ci[threadIdx.x];
    for (int b = b0; b < b1; ++b) {
        win[b].woff = off;
        win[b].ioff = io;
        off += win[b].W;
        io += (win[b].W + kWc - 1) / kWc;
    }
}

// The generator: mt19937_64(seed) words [0, L) into HBM.  With x[0..312) the seeded state and
// half-block m = x[156 m, 156 m + 156), column j of half m is
//   x[156 m + j] = x[156 (m-1) + j] ^ twist(x[156 (m-2) + j], x[156 (m-2) + j + 1])
// (x[156 (m-2) + 156] = x[156 (m-1)]), and stream word k = temper(x[312 + k]): 156 threads advance
// one half-block per barrier; progress is published every 32 half-blocks.
__device__ void generate_stream(uint64_t seed, uint64_t L, uint64_t* __restrict__ stream, ParHdr* hdr,
                                uint64_t* hb /* >= 4 x 160 + 312 words */) {
    const int j = threadIdx.x;
    uint64_t* seeded = hb + 4 * 160;
    if (j == 0) mt64::seed_state(seeded, seed);
    __syncthreads();
    uint64_t* H = hb;  // ring of four half-blocks, 160 entries each
    if (j < kGenCols) {
        H[0 * 160 + j] = seeded[j];
        H[1 * 160 + j] = seeded[kGenCols + j];
    }
    __syncthreads();
    const uint64_t halves = L / kGenCols;
    for (uint64_t m = 2; m < halves + 2; ++m) {
        const bool publish = ((m - 1) & 31) == 0 || m + 1 == halves + 2;
        if (j < kGenCols) {
            const uint64_t* h2 = H + ((m - 2) & 3) * 160;
            const uint64_t* h1 = H + ((m - 1) & 3) * 160;
            const uint64_t cur = h2[j];
            const uint64_t nxt = j + 1 < kGenCols ? h2[j + 1] : h1[0];
            const uint64_t x = mt64::twist1(cur, nxt, h1[j]);
            H[(m & 3) * 160 + j] = x;
            __stcg(stream + (m - 2) * kGenCols + j, mt64::temper(x));
            if (publish) __threadfence();
        }
        __syncthreads();
        if (publish && j == 0) atomicExch(&hdr->progress, (unsigned long long)((m - 1) * kGenCols));
    }
}

// the generator alone (diagnostic split: ETUNE_BREED_PAR_SPLITGEN)
__global__ void __launch_bounds__(256) breed_gen_kernel(uint64_t seed, uint64_t* __restrict__ stream, ParHdr* hdr) {
    __shared__ uint64_t hb[4 * 160 + 312];
    if (hdr->status) return;
    generate_stream(seed, hdr->L, stream, hdr, hb);
}

__device__ __forceinline__ void wait_words(ParHdr* hdr, unsigned long long need) {
    if (threadIdx.x == 0) {
        const volatile unsigned long long* pr = &hdr->progress;
        while (*pr < need) __nanosleep(256);
        __threadfence();
    }
    __syncthreads();
}

// The walkers' evaluator: ONLY the number of words an offspring consumes, for the uniform base parent
// of this step, from the first six words at its offset, as straight-line code (no per-walker
// switch / loops, so a warp stays converged).  It follows breed_body() decision by decision —
// coin, knob or partner, pick_other / pick_pow2 or the crossover mask, then repair_schedule's
// single tiling re-pick and the unroll / vectorize redraws — and answers 0 ("slow") wherever the
// reference could draw differently: any Lemire draw that might be rejected (conservatively:
// low product < range), a crossover partner with the base's id, a re-pick that cannot fit, or
// more than six words.  Slow walkers are evaluated by breed_body itself.
struct StepBase {       // the base parent parents[i % P] of this step
    uint32_t m4, m5;    // 1 + its unroll / vectorize log2 caps (the tilings' and K's counts are in H)
    uint64_t g, id;
};

struct Words6 {
    uint64_t w0, w1, w2, w3, w4, w5;
    __device__ __forceinline__ uint64_t at(uint32_t s) const {  // s in [2, 5]
        uint64_t r = w2;
        r = s == 3 ? w3 : r;
        r = s == 4 ? w4 : r;
        r = s == 5 ? w5 : r;
        return r;
    }
};

__device__ __forceinline__ StepBase step_base(const PlanHdr& H, const uint8_t* P, uint64_t g, uint64_t id) {
    StepBase B;
    B.g = g;
    B.id = id;
    const Genome x = genome_unpack(B.g);
    const TilingRec* til2 = at<TilingRec>(P, H.off_til[2]);
    const int64_t* divk = at<int64_t>(P, H.off_divk);
    B.m4 = uint32_t(min(H.max_unroll_log2, ctz64(divk[x.k]))) + 1;
    B.m5 = uint32_t(min(H.max_vec_log2, ctz64(int64_t(til2[x.t2].pt)))) + 1;
    return B;
}

// The coin of genetic.cpp:162 (uniform_real_distribution<double>(0,1) * total, exactly as
// breed_body computes it) is monotone in the word w0, so "u < x" is "w0 < T(x)": the two cuts
// (mutation, mutation + crossover) are found once per CTA by bisection on w0 and the walkers
// compare integers.
__device__ __forceinline__ double coin_u(uint64_t w0, double total) {
    const double coin = __dmul_rn(__ull2double_rn(w0), 0x1p-64);
    return __dmul_rn(coin < 1.0 ? coin : 0x1.fffffffffffffp-1, total);
}
struct CoinCut {
    uint64_t t_mc, t_m;  // u < mutcro iff all_mc or w0 < t_mc; u < mut iff all_m or w0 < t_m
    int all_mc, all_m;
};
__device__ void coin_cut(double x, double total, uint64_t* t, int* all) {
    if (coin_u(~0ull, total) < x) {
        *all = 1;
        *t = ~0ull;
        return;
    }
    uint64_t lo = 0, hi = ~0ull;  // coin_u(hi) >= x
    while (lo < hi) {
        const uint64_t mid = lo + ((hi - lo) >> 1);
        if (coin_u(mid, total) >= x) hi = mid;
        else lo = mid + 1;
    }
    *all = 0;
    *t = lo;
}

__device__ __forceinline__ uint32_t fast_words(const BreedConst& K, const PlanHdr& H, const StepBase& B,
                                               const CoinCut& C, const Words6& w) {
    if (!(C.all_mc || w.w0 < C.t_mc)) return 1u;  // copy
    Genome x = genome_unpack(B.g);
    uint32_t s;
    if (C.all_m || w.w0 < C.t_m) {  // mutate_knob (genetic.cpp:60-87)
        if (w.w1 * 6ull < 6ull) return 0u;
        const uint32_t knob = uint32_t(__umul64hi(w.w1, 6ull));
        uint32_t m = uint32_t(H.nt[0]), a = x.t0;
        m = knob == 1 ? uint32_t(H.nt[1]) : m;
        a = knob == 1 ? x.t1 : a;
        m = knob == 2 ? uint32_t(H.nt[2]) : m;
        a = knob == 2 ? x.t2 : a;
        m = knob == 3 ? uint32_t(H.ndk) : m;
        a = knob == 3 ? x.k : a;
        m = knob == 4 ? B.m4 : m;
        a = knob == 4 ? x.u : a;
        m = knob == 5 ? B.m5 : m;
        a = knob == 5 ? x.v : a;
        const bool pow2 = knob >= 4;
        uint32_t nv;
        if (m <= 1) {  // no alternative: no draw
            nv = pow2 ? 0u : a;
            s = 2;
        } else {
            const bool outside = pow2 && a > m - 1;  // pick_pow2 with the current value off the list
            const uint64_t rng = outside ? m : m - 1;
            if (w.w2 * rng < rng) return 0u;
            const uint32_t j = uint32_t(__umul64hi(w.w2, rng));
            nv = outside ? j : (j < a ? j : j + 1);
            s = 3;
        }
        x.t0 = knob == 0 ? nv : x.t0;
        x.t1 = knob == 1 ? nv : x.t1;
        x.t2 = knob == 2 ? nv : x.t2;
        x.k = knob == 3 ? nv : x.k;
        x.u = knob == 4 ? nv : x.u;
        x.v = knob == 5 ? nv : x.v;
    } else {  // crossover (genetic.cpp:168-180)
        const uint64_t np = uint64_t(K.np);
        if (w.w1 * np < np) return 0u;
        const uint64_t pi = __umul64hi(w.w1, np);
        if (K.has_other && __ldg(K.pid + pi) == B.id) return 0u;  // the partner redraw loop
        const uint32_t mask = uint32_t(w.w2 & 63u);
        const Genome y = genome_unpack(__ldg(K.par + pi));
        x.t0 = (mask & 1u) ? y.t0 : x.t0;
        x.t1 = (mask & 2u) ? y.t1 : x.t1;
        x.t2 = (mask & 4u) ? y.t2 : x.t2;
        x.k = (mask & 8u) ? y.k : x.k;
        x.u = (mask & 16u) ? y.u : x.u;
        x.v = (mask & 32u) ? y.v : x.v;
        s = 3;
    }
    // repair_schedule (genetic.cpp:89-135)
    const TilingRec* til0 = at<TilingRec>(K.P, H.off_til[0]);
    const TilingRec* til1 = at<TilingRec>(K.P, H.off_til[1]);
    const TilingRec* til2 = at<TilingRec>(K.P, H.off_til[2]);
    const uint64_t th0 = til0[x.t0].threads, th1 = til1[x.t1].threads, th2 = til2[x.t2].threads;
    const int64_t cap = H.block_cap;
    if (int64_t(th0 * th1 * th2) > cap) {  // one re-pick of the dimension with the most threads
        int dim = 0;
        uint64_t tm = th0;
        if (th1 > tm) { dim = 1; tm = th1; }
        if (th2 > tm) { dim = 2; tm = th2; }
        const uint64_t other = dim == 0 ? th1 * th2 : (dim == 1 ? th0 * th2 : th0 * th1);
        if (int64_t(other) > cap) return 0u;  // no tiling fits: {extent,1,1} and another round
        const int64_t lim = int64_t(uint32_t(cap) / uint32_t(other));  // cap <= 1024, other <= cap here
        const uint8_t* F = K.P + (dim == 0 ? H.off_fit[0] : (dim == 1 ? H.off_fit[1] : H.off_fit[2]));
        const int ntv = reinterpret_cast<const FitHeader*>(F)->ntv;
        const uint32_t* tv = reinterpret_cast<const uint32_t*>(F + sizeof(FitHeader));
        const uint32_t* start = tv + ntv;
        const uint16_t* list = reinterpret_cast<const uint16_t*>(start + ntv + 1);
        int lo = 0, hi = ntv;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (int64_t(tv[mid]) <= lim) lo = mid + 1;
            else hi = mid;
        }
        const uint32_t fit = lo > 0 ? start[lo] - start[lo - 1] : 0u;
        if (fit == 0) return 0u;
        const uint64_t wd = w.at(s);
        if (wd * uint64_t(fit) < uint64_t(fit)) return 0u;
        const uint32_t t = list[start[lo - 1] + uint32_t(__umul64hi(wd, uint64_t(fit)))];
        x.t0 = dim == 0 ? t : x.t0;
        x.t1 = dim == 1 ? t : x.t1;
        x.t2 = dim == 2 ? t : x.t2;
        ++s;
    }
    const int64_t* divk = at<int64_t>(K.P, H.off_divk);
    const uint32_t cu = uint32_t(min(H.max_unroll_log2, ctz64(divk[x.k])));
    if (x.u > cu) {
        const uint64_t wd = w.at(s);
        if (wd * uint64_t(cu + 1) < uint64_t(cu + 1)) return 0u;
        ++s;
    }
    const uint32_t cv = uint32_t(min(H.max_vec_log2, ctz64(int64_t(til2[x.t2].pt))));
    if (x.v > cv) {
        if (s > 5) return 0u;
        const uint64_t wd = w.at(s);
        if (wd * uint64_t(cv + 1) < uint64_t(cv + 1)) return 0u;
        ++s;
    }
    return s;
}

// one window item: every start of a chunk walked through its block at once, merged as walks meet.
// One barrier round per epoch of kEpoch steps (not per step): inside an epoch each thread moves its
// own walkers; at the epoch's end the claim words (tagged with the time, so a stale or early claim
// can only hide a merge -- the walks then stay separate, still exact -- never fake one) merge the
// walks standing on the same word, and the live list is compacted.
__global__ void __launch_bounds__(kWinT, 3)
    breed_win_kernel(const uint8_t* __restrict__ gplan, uint32_t plan_pre, const uint64_t* __restrict__ par,
                     const uint64_t* __restrict__ pid, int64_t np, int64_t n, int S, int B, double mut, double mutcro,
                     double total, uint64_t seed, uint64_t* __restrict__ stream, ParHdr* hdr,
                     const BlockWin* __restrict__ win, uint32_t* __restrict__ endpos, uint16_t* __restrict__ gparent,
                     uint16_t* __restrict__ gmtime, uint2* __restrict__ snapidx, uint64_t* __restrict__ pool,
                     unsigned long long pool_cap, int gen_here, int prof, int check, unsigned long long* err) {
    // dynamic smem: [ring u64[kRing] | claims u32[kHash] | pos u32[kWc] | live u16[2][kWc] |
    //                parent u16[kWc] | plan prefix (header, tilings, divisors of K, repair tables)]
    extern __shared__ int4 wsm[];
    uint64_t* ring = reinterpret_cast<uint64_t*>(wsm);
    uint32_t* claims = reinterpret_cast<uint32_t*>(ring + kRing);
    uint32_t* pos = claims + kHash;
    uint16_t* live0 = reinterpret_cast<uint16_t*>(pos + kWc);
    uint16_t* live1 = live0 + kWc;
    uint16_t* parent = live1 + kWc;
    uint8_t* splan = reinterpret_cast<uint8_t*>(parent + kWc);
    __shared__ uint32_t ws[32];
    __shared__ uint32_t s_ticket, s_base;
    __shared__ int s_item_b;
    if (hdr->status) return;
    if (threadIdx.x == 0) s_ticket = atomicAdd(&hdr->ticket, 1u);
    __syncthreads();
    const uint32_t ticket = s_ticket;
    unsigned long long t_start = 0;
    if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    if (ticket == 0) {  // this CTA is running: the generator the others wait on
        if (gen_here) generate_stream(seed, hdr->L, stream, hdr, ring);
        if (prof && threadIdx.x == 0) {
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            printf("GEN %llu %llu\n", t_start, t_end);
        }
        return;
    }
    const int item = int(ticket) - 1;
    if (item >= hdr->items) return;
    if (threadIdx.x == 0) {  // the block owning this item: last b with ioff <= item
        int lo = 0, hi = B;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (int(win[mid].ioff) <= item) lo = mid;
            else hi = mid;
        }
        s_item_b = lo;
    }
    for (uint32_t q = threadIdx.x; q < (plan_pre >> 4); q += blockDim.x)
        reinterpret_cast<int4*>(splan)[q] = __ldg(reinterpret_cast<const int4*>(gplan) + q);
    __syncthreads();
    const int b = s_item_b;
    const BlockWin bw = win[b];
    const int chunk = item - int(bw.ioff);
    const uint32_t c0 = uint32_t(chunk) * kWc;
    const uint32_t Wn = min(uint32_t(kWc), bw.W - c0);  // starts in this chunk
    const uint32_t lo = bw.lo + c0;                      // first start position of the chunk
    const uint32_t woff = bw.woff + c0;
    const int64_t i0 = int64_t(b) * S;
    const int nb = int(imin64(S, n - i0));
    const int nsub = S / kQ;
    const uint64_t hiw = bw.need;  // the words this item waits for; beyond them a walk is "unknown"
    const double mean = double(bw.mean) > 0.0 ? double(bw.mean) : 0.0;

    for (int j = threadIdx.x; j < kHash; j += blockDim.x) claims[j] = 0u;
    for (uint32_t w = threadIdx.x; w < Wn; w += blockDim.x) {
        pos[w] = lo + w;
        parent[w] = uint16_t(w);
        gparent[woff + w] = uint16_t(w);
        live0[w] = uint16_t(w);
    }
    // the ring holds words [base_t, base_t + kRing) (slot p % kRing), base_t on the chunk's mean
    // path, slid once per epoch (see the epoch loop for when the slid-in words may be read)
    const uint64_t mfix = uint64_t(mean * 4294967296.0);  // words per offspring, 32.32 fixed point
    auto base_at = [&](int s) -> int64_t {
        return (int64_t(lo) + int64_t((mfix * uint64_t(s)) >> 32) - kRingMargin) & ~int64_t(1);
    };
    wait_words(hdr, hiw);
    int64_t base = base_at(0);
    for (int q = threadIdx.x; q < kRing; q += blockDim.x) {
        const int64_t p = base + q;
        if (p >= 0 && uint64_t(p) < hiw) ring[uint32_t(p) % kRing] = __ldcg(stream + p);
    }
    __syncthreads();
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(splan);
    const BreedConst K{splan, par, pid, np, mut, mutcro, total, hdr->other};
    uint16_t* cur = live0;
    uint16_t* nxt = live1;
    uint32_t nlive = Wn;
    unsigned long long t_ready = 0, evals = 0, gloads = 0, ck_sb = 0, ck_a = 0, ck_bar = 0, ck_b = 0;
    const int nep = (nb + kEpoch - 1) / kEpoch;  // epochs (profile averages are per epoch)
    if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
    // Epochs of kEpoch steps: every walker of a thread advances through the epoch's steps with no
    // barrier in between (its position is read and written by its owner only); claims, merges,
    // the ring slide, compaction and snapshots happen once per epoch.  Walkers that coalesced
    // inside an epoch are merged at its end -- from then on they are the same walk, and gmtime
    // records the merge as of the epoch's last step (the emit follows merges at steps < tq).
    __shared__ StepBase sbase[2][kEpoch];  // the epoch's base parents, prepared once per step
    __shared__ CoinCut s_cut;
    if (threadIdx.x == 0) {
        coin_cut(mutcro, total, &s_cut.t_mc, &s_cut.all_mc);
        coin_cut(mut, total, &s_cut.t_m, &s_cut.all_m);
    }
    if (threadIdx.x < kEpoch && int(threadIdx.x) < nb) {
        const int64_t q = (i0 + threadIdx.x) % np;  // base parent of offspring i (genetic.cpp:160)
        sbase[0][threadIdx.x] = step_base(*reinterpret_cast<const PlanHdr*>(splan), splan, __ldg(par + q),
                                          __ldg(pid + q));
    }
    __syncthreads();
    const CoinCut CC = s_cut;
    uint32_t* P0 = pos;  // one buffer: during an epoch only a walker's owner touches its position
    int f = 0;
    for (int t = 0; t < nb; t += kEpoch, ++f) {
        const int te = min(nb, t + kEpoch);
        // ring words landed and visible: the slide issued at the end of epoch e is waited for at the
        // end of epoch e + 1 and crosses that epoch's last barrier, so epoch f reads below
        // base_{(f-1)E} + kRing (the initial fill covers base_0 + kRing)
        const int64_t vhi = base_at(f >= 2 ? (f - 1) * kEpoch : 0) + kRing;
        const int64_t fhi = vhi < int64_t(hiw) ? vhi : int64_t(hiw);
        // a contiguous share of the live list per thread (order-preserving compaction below)
        const uint32_t per = (nlive + kWinT - 1) / kWinT;
        const uint32_t a0 = min(nlive, threadIdx.x * per), a1 = min(nlive, a0 + per);
        const StepBase* sb = sbase[f & 1];
        long long ck0 = prof ? clock64() : 0;
        for (int st = t; st < te && a0 < a1; ++st) {
            const StepBase SB = sb[st - t];
            const int64_t i = i0 + st;
            for (uint32_t a = a0; a < a1; ++a) {
                const uint32_t w = cur[a];
                if (parent[w] != w) continue;  // merged at an earlier epoch
                const uint32_t p0 = P0[w];
                if (p0 == kGone) continue;
                uint32_t fw = 0;
                if (int64_t(p0) >= base && int64_t(p0) + 6 <= fhi) {
                    const uint32_t r0 = p0 % kRing;  // slots r0 .. r0 + 5, wrapping once at most
                    auto slot = [&](uint32_t d) { const uint32_t r = r0 + d; return r < kRing ? r : r - kRing; };
                    const Words6 wv{ring[r0], ring[slot(1)], ring[slot(2)], ring[slot(3)], ring[slot(4)], ring[slot(5)]};
                    fw = fast_words(K, H, SB, CC, wv);
                }
                if (prof) {
                    ++evals;
                    if (fw == 0) ++gloads;
                }
                if (fw == 0 || check) {
                    RCursor c{ring, stream, base, vhi, p0, hiw, true};
                    const Child ch = breed_body(K, H, i, c, p0);
                    if (fw != 0 && uint64_t(p0) + fw != c.p)  // diagnostic: the fast count disagrees
                        atomicMin(err, (static_cast<unsigned long long>(i) << 8) | unsigned(ETUNE_ERR_CONSISTENCY));
                    if (ch.words == kUnknown || ch.words == kIllegal) {
                        endpos[woff + w] = ch.words == kIllegal ? kFateIllegal : kFateUnknown;
                        P0[w] = kGone;
                        continue;
                    }
                    fw = uint32_t(c.p - p0);
                }
                P0[w] = p0 + fw;
            }
        }
        // claims at the epoch's end: the lowest walker on a word (hash slot, tagged by the time)
        const uint32_t tkey = uint32_t(te) << 16;
        for (uint32_t a = a0; a < a1; ++a) {
            const uint32_t w = cur[a];
            if (parent[w] != w) continue;
            const uint32_t p1 = P0[w];
            if (p1 != kGone) atomicMax(claims + (p1 & (kHash - 1)), tkey | (0xffffu - w));
        }
        if (threadIdx.x < kEpoch && te + int(threadIdx.x) < nb) {  // the next epoch's base parents
            const int64_t q = (i0 + te + threadIdx.x) % np;
            sbase[(f + 1) & 1][threadIdx.x] = step_base(H, splan, __ldg(par + q), __ldg(pid + q));
        }
        long long ck1 = prof ? clock64() : 0;
        __syncthreads();
        long long ck2 = prof ? clock64() : 0;
        if (prof) { ck_a += uint64_t(ck1 - ck0); ck_bar += uint64_t(ck2 - ck1); }
        // slide the ring along the mean path (the words entering it are read epochs later)
        const int64_t nbase = base_at(te);
        if (nbase > base) {
            for (int64_t p = base + kRing + 2 * int64_t(threadIdx.x); p < nbase + kRing; p += 2 * blockDim.x)
                if (p >= 0 && uint64_t(p) < hiw) cp_async16(ring + uint32_t(p) % kRing, stream + p);
            base = nbase;
        }
        cp_async_commit();
        cp_async_wait<1>();
        uint32_t keep = 0;
        for (uint32_t a = a0; a < a1; ++a) {
            const uint32_t w = cur[a];
            if (parent[w] != w) continue;
            const uint32_t p1 = P0[w];
            if (p1 == kGone) continue;
            const uint32_t k = claims[p1 & (kHash - 1)];
            const uint32_t ww = 0xffffu - (k & 0xffffu);
            // the winner claimed at this time and stands on the same word: the same walk from here
            if ((k >> 16) == uint32_t(te) && ww != w && P0[ww] == p1) {
                parent[w] = uint16_t(ww);
                gparent[woff + w] = uint16_t(ww);
                gmtime[woff + w] = uint16_t(te - 1);
                continue;
            }
            ++keep;
        }
        if (prof) ck_b += uint64_t(clock64() - ck2);
        const bool snap = (te % kQ) == 0 && te < nb;
        {
            uint32_t tot;
            uint32_t o = block_scan_u32(keep, &tot, ws);  // (ends with a barrier)
            for (uint32_t a = a0; a < a1; ++a) {
                const uint32_t w = cur[a];
                if (parent[w] != w || P0[w] == kGone) continue;
                nxt[o++] = uint16_t(w);
            }
            __syncthreads();
            uint16_t* sw = cur;
            cur = nxt;
            nxt = sw;
            nlive = tot;
            if (snap) {  // snapshot of the live walkers (w ascending) at time te
                if (threadIdx.x == 0) {
                    const unsigned long long ob = atomicAdd(&hdr->snap_used, (unsigned long long)tot);
                    s_base = (ob + tot <= pool_cap) ? uint32_t(ob) : 0xffffffffu;
                    snapidx[size_t(item) * nsub + te / kQ] = make_uint2(s_base, tot);
                }
                __syncthreads();
                const uint32_t sb = s_base;
                if (sb != 0xffffffffu)
                    for (uint32_t a = threadIdx.x; a < tot; a += blockDim.x) {
                        const uint32_t w = cur[a];
                        pool[sb + a] = ((unsigned long long)w << 32) | P0[w];
                    }
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    if (prof) {
        __shared__ unsigned long long s_ev, s_gl;
        if (threadIdx.x == 0) s_ev = s_gl = 0;
        __syncthreads();
        atomicAdd(&s_ev, evals);
        atomicAdd(&s_gl, gloads);
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t_end;
            unsigned smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            printf("ITEM %d %d %u %u %llu %llu %llu %llu %llu %u %llu %llu %llu %llu\n", item, b, Wn, smid, t_start, t_ready,
                   t_end, s_ev, s_gl, nlive, ck_sb / nep, ck_a / nep, ck_bar / nep, ck_b / nep);
        }
    }
    const uint32_t* pf = pos;  // positions at time nb
    for (uint32_t a = threadIdx.x; a < nlive; a += blockDim.x) {
        const uint32_t w = cur[a];
        if (parent[w] == w && pf[w] != kGone) endpos[woff + w] = pf[w];
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < Wn; w += blockDim.x) {
        uint32_t r = w;
        while (parent[r] != r) r = parent[r];
        if (r != w) endpos[woff + w] = endpos[woff + r];
    }
}

// exact evaluation of offspring [ia, ie) from word offset p (children from emit_from on);
// returns the offset after the last one; *st: 0 ok, 1 the stream ran out, 2 illegal child
__device__ uint64_t walk_emit(const BreedConst& K, const PlanHdr& H, const uint64_t* stream, uint64_t L, int64_t ia,
                              int64_t ie, int64_t emit_from, uint64_t p, uint64_t* out, int32_t* partner,
                              unsigned long long* err, int* st) {
    for (int64_t i = ia; i < ie; ++i) {
        GCursor c(stream, p, L);
        const Child ch = breed_body(K, H, i, c, p);
        if (ch.words == kIllegal) {
            atomicMin(err, (static_cast<unsigned long long>(i) << 8) | unsigned(ETUNE_ERR_ILLEGAL_SCHEDULE));
            *st = 2;
            return p;
        }
        if (ch.words == kUnknown) {
            *st = 1;
            return p;
        }
        if (i >= emit_from) {
            out[i] = ch.g;
            if (partner) partner[i] = ch.partner;
        }
        p = c.p;
    }
    *st = 0;
    return p;
}

// the true chain across blocks: one lookup per block, exact walks where a window missed
__global__ void __launch_bounds__(32) breed_chain_kernel(const uint8_t* __restrict__ gplan, const uint64_t* __restrict__ par,
                                                         const uint64_t* __restrict__ pid, int64_t np, int64_t n, int S,
                                                         int B, double mut, double mutcro, double total,
                                                         const uint64_t* __restrict__ stream, ParHdr* hdr,
                                                         const BlockWin* __restrict__ win,
                                                         const uint32_t* __restrict__ endpos,
                                                         uint32_t* __restrict__ starts, uint8_t* __restrict__ walked,
                                                         uint64_t* __restrict__ out, int32_t* __restrict__ partner,
                                                         unsigned long long* err) {
    if (threadIdx.x != 0 || hdr->status) return;
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(gplan);
    const BreedConst K{gplan, par, pid, np, mut, mutcro, total, hdr->other};
    const uint64_t L = hdr->L;
    uint64_t p = 0;
    BlockWin nx = win[0];
    for (int b = 0; b < B; ++b) {
        const BlockWin bw = nx;
        if (b + 1 < B) nx = win[b + 1];
        starts[b] = uint32_t(p);
        const uint64_t rel = p - bw.lo;
        const uint32_t e = (p >= bw.lo && rel < bw.W) ? endpos[bw.woff + rel] : kFateUnknown;
        if (e < kFateIllegal) {
            walked[b] = 0;
            p = e;
            continue;
        }
        // outside the window, or the walk from here met an illegal schedule / left its words
        walked[b] = 1;
        const int64_t i0 = int64_t(b) * S, i1 = imin64(n, i0 + S);
        int st = 0;
        p = walk_emit(K, H, stream, L, i0, i1, i0, p, out, partner, err, &st);
        if (st == 2) {  // the reference throws here; children before it are written
            hdr->nres = b;
            hdr->done = 1;
            return;
        }
        if (st == 1) {  // stream exhausted: the single-CTA chain produces the generation
            hdr->status = 1;
            return;
        }
    }
    hdr->nres = B;
    hdr->done = 1;
}

// one thread per Q-offspring sub-block of a block the chain resolved by lookup
__global__ void __launch_bounds__(128) breed_emit_kernel(const uint8_t* __restrict__ gplan, const uint64_t* __restrict__ par,
                                                         const uint64_t* __restrict__ pid, int64_t np, int64_t n, int S,
                                                         int B, double mut, double mutcro, double total,
                                                         const uint64_t* __restrict__ stream, const ParHdr* __restrict__ hdr,
                                                         const BlockWin* __restrict__ win,
                                                         const uint16_t* __restrict__ gparent,
                                                         const uint16_t* __restrict__ gmtime,
                                                         const uint2* __restrict__ snapidx,
                                                         const uint64_t* __restrict__ pool,
                                                         const uint32_t* __restrict__ starts,
                                                         const uint8_t* __restrict__ walked, uint64_t* __restrict__ out,
                                                         int32_t* __restrict__ partner, unsigned long long* err) {
    const int nsub = S / kQ;
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= int64_t(B) * nsub) return;
    if (hdr->status || !hdr->done) return;
    const int b = int(g / nsub), k = int(g % nsub);
    if (b >= hdr->nres || walked[b]) return;
    const int64_t i0 = int64_t(b) * S;
    const int64_t ia = i0 + int64_t(k) * kQ;
    if (ia >= n) return;
    const int64_t ie = imin64(n, imin64(ia + kQ, i0 + S));
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(gplan);
    const BreedConst K{gplan, par, pid, np, mut, mutcro, total, hdr->other};
    const BlockWin bw = win[b];
    const uint32_t w0 = starts[b] - bw.lo;  // the true start's index in the window
    const uint32_t chunk = w0 / kWc;
    const uint32_t item = bw.ioff + chunk;
    const uint32_t coff = bw.woff + chunk * kWc;
    uint64_t p = starts[b];
    int kk = k;
    for (; kk > 0; --kk) {  // latest snapshot at or before this sub-block holding the true walk
        const uint2 si = snapidx[size_t(item) * nsub + kk];
        if (si.x == 0xffffffffu) continue;
        const uint32_t tq = uint32_t(kk) * kQ;  // merges at steps < tq are in effect
        uint32_t w = w0 - chunk * kWc;
        for (;;) {
            const uint32_t pw = gparent[coff + w];
            if (pw == w || gmtime[coff + w] >= tq) break;
            w = pw;
        }
        uint32_t lo2 = 0, hi2 = si.y;  // binary search of w in the snapshot (w ascending)
        while (lo2 < hi2) {
            const uint32_t mid = (lo2 + hi2) >> 1;
            if (uint32_t(pool[si.x + mid] >> 32) < w) lo2 = mid + 1;
            else hi2 = mid;
        }
        if (lo2 < si.y && uint32_t(pool[si.x + lo2] >> 32) == w) {
            p = uint32_t(pool[si.x + lo2]);
            break;
        }
    }
    int st = 0;
    (void)walk_emit(K, H, stream, hdr->L, i0 + int64_t(kk) * kQ, ie, ia, p, out, partner, err, &st);
}

// diagnostic (ETUNE_BREED_PAR_PROF): latency of one offspring evaluation on one thread, words from
// shared memory and from L2, after the generation (the stream's first 8192 words)
__global__ void breed_lat_kernel(const uint8_t* __restrict__ gplan, uint32_t plan_pre, const uint64_t* __restrict__ par,
                                 const uint64_t* __restrict__ pid, int64_t np, double mut, double mutcro, double total,
                                 const uint64_t* __restrict__ stream, const ParHdr* __restrict__ hdr) {
    extern __shared__ int4 lsm[];
    uint64_t* words = reinterpret_cast<uint64_t*>(lsm);
    uint8_t* splan = reinterpret_cast<uint8_t*>(words + 8192);
    for (int q = threadIdx.x; q < 8192; q += blockDim.x) words[q] = stream[q];
    for (uint32_t q = threadIdx.x; q < (plan_pre >> 4); q += blockDim.x)
        reinterpret_cast<int4*>(splan)[q] = reinterpret_cast<const int4*>(gplan)[q];
    __syncthreads();
    if (threadIdx.x != 0) return;
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(splan);
    const BreedConst K{splan, par, pid, np, mut, mutcro, total, hdr->other};
    uint64_t p = 0, acc = 0;
    long long c0 = clock64();
    int64_t i = 0;
    for (; i < 2000 && p < 8000; ++i) {
        RCursor c{words, stream, 0, 8192, p, 8192, true};
        const Child ch = breed_body(K, H, i, c, p);
        acc ^= ch.g;
        p = c.p;
    }
    long long c1 = clock64();
    uint64_t p2 = 0;
    int64_t i2 = 0;
    for (; i2 < 2000 && p2 < 8000; ++i2) {
        GCursor c(stream, p2, 8192);
        const Child ch = breed_body(K, H, i2, c, p2);
        acc ^= ch.g;
        p2 = c.p;
    }
    long long c2 = clock64();
    printf("LAT smem %.1f cycles/offspring (%lld), L2 %.1f cycles/offspring, acc %llx\n", double(c1 - c0) / double(i),
           (long long)i, double(c2 - c1) / double(i2), (unsigned long long)acc);
}

struct ParLayout {
    ParHdr* hdr;
    double2* est;
    BlockWin* win;
    uint32_t* starts;
    uint8_t* walked;
    uint64_t* stream;
    uint32_t* endpos;
    uint16_t* gparent;
    uint16_t* gmtime;
    uint2* snapidx;
    uint64_t* pool;
    size_t bytes, words, pool_cap, items_max;
};

ParLayout par_layout(char* w, int64_t n, int S) {
    const int64_t B = (n + S - 1) / S;
    ParLayout l{};
    l.words = size_t(n) * 8 + (size_t(1) << 17);
    l.items_max = size_t(B) * (kWcap / kWc);
    l.pool_cap = size_t(B) * kWcap / 2 + 65536;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char* p = w ? w + off : nullptr;
        off = (off + bytes + 255) & ~size_t(255);
        return p;
    };
    l.hdr = reinterpret_cast<ParHdr*>(take(sizeof(ParHdr)));
    l.est = reinterpret_cast<double2*>(take(size_t(B) * sizeof(double2)));
    l.win = reinterpret_cast<BlockWin*>(take(size_t(B) * sizeof(BlockWin)));
    l.starts = reinterpret_cast<uint32_t*>(take(size_t(B) * 4));
    l.walked = reinterpret_cast<uint8_t*>(take(size_t(B)));
    l.stream = reinterpret_cast<uint64_t*>(take((l.words + 8) * 8));
    l.endpos = reinterpret_cast<uint32_t*>(take(size_t(B) * kWcap * 4));
    l.gparent = reinterpret_cast<uint16_t*>(take(size_t(B) * kWcap * 2));
    l.gmtime = reinterpret_cast<uint16_t*>(take(size_t(B) * kWcap * 2));
    l.snapidx = reinterpret_cast<uint2*>(take(l.items_max * (S / kQ) * sizeof(uint2)));
    l.pool = reinterpret_cast<uint64_t*>(take(l.pool_cap * 8));
    l.bytes = off;
    return l;
}

}  // namespace

size_t breed_par_bytes(int64_t n, int S, size_t* stream_words, size_t* pool_cap) {
    const ParLayout l = par_layout(nullptr, n, S);
    *stream_words = l.words;
    *pool_cap = l.pool_cap;
    return l.bytes;
}

int breed_par_block(int64_t n) {
    // offspring per block: enough blocks to fill the GPU, long enough to amortise the windows
    int S = 256;
    while (S < 2048 && int64_t(S) * 256 < n) S <<= 1;
    return S;
}

cudaError_t launch_breed_par(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint64_t* d_par,
                             const uint64_t* d_pid, int64_t np, int64_t n, double mut, double cro, double cpy,
                             uint64_t seed, uint64_t* d_out, int32_t* d_partner, void* d_work, int S, double sd_mult,
                             size_t words_cap, int split_gen, uint32_t plan_pre, int32_t** d_done) {
    (void)plan_bytes;
    const double mutcro = mut + cro;   // genetic.cpp:169, evaluated like the reference
    const double total = mutcro + cpy; // genetic.cpp:150
    const int B = int((n + S - 1) / S);
    const ParLayout l = par_layout(static_cast<char*>(d_work), n, S);
    *d_done = &l.hdr->done;
    cudaError_t e;
    breed_other_kernel<<<1, 1024, 0, c.stream>>>(d_pid, np, l.hdr);
    breed_est_kernel<<<B, kEstThreads, 0, c.stream>>>(d_plan, d_par, d_pid, np, n, S, mut, mutcro, total, seed, l.hdr,
                                                      l.est);
    const size_t cap = words_cap > 0 && words_cap < l.words ? words_cap : l.words;
    breed_plan_kernel<<<1, 1024, 0, c.stream>>>(l.est, B, S, n, uint64_t(cap), sd_mult, l.win, l.hdr);
    const size_t win_dyn = size_t(kRing) * 8 + size_t(kHash) * 4 + size_t(kWc) * (4 + 4 + 2) + plan_pre;
    static_assert(size_t(kRing) >= 4 * 160 + 312, "the generator's half-blocks live in the ring");
    e = cudaFuncSetAttribute(breed_win_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(win_dyn));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(breed_win_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    const bool split = split_gen & 1;
    const int prof = (split_gen >> 1) & 1;  // diagnostic: per-item timing printed by the device
    if (prof) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, breed_win_kernel, kWinT, win_dyn);
        std::printf("WIN smem %zu B (plan prefix %u), %d CTAs/SM\n", win_dyn, plan_pre, occ);
    }
    if (split) breed_gen_kernel<<<1, 256, 0, c.stream>>>(seed, l.stream, l.hdr);
    // grid: every possible item + the generator; CTAs beyond the plan's items exit at once
    breed_win_kernel<<<unsigned(l.items_max + 1), kWinT, win_dyn, c.stream>>>(
        d_plan, plan_pre, d_par, d_pid, np, n, S, B, mut, mutcro, total, seed, l.stream, l.hdr, l.win, l.endpos, l.gparent,
        l.gmtime, l.snapidx, l.pool, (unsigned long long)l.pool_cap, split ? 0 : 1, prof, (split_gen >> 2) & 1, c.d_err);
    if (prof) {
        cudaFuncSetAttribute(breed_lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(8192 * 8 + plan_pre));
        breed_lat_kernel<<<1, 32, 8192 * 8 + plan_pre, c.stream>>>(d_plan, plan_pre, d_par, d_pid, np, mut, mutcro,
                                                                    total, l.stream, l.hdr);
    }
    breed_chain_kernel<<<1, 32, 0, c.stream>>>(d_plan, d_par, d_pid, np, n, S, B, mut, mutcro, total, l.stream, l.hdr,
                                                l.win, l.endpos, l.starts, l.walked, d_out, d_partner, c.d_err);
    const int64_t subs = int64_t(B) * (S / kQ);
    breed_emit_kernel<<<int((subs + 127) / 128), 128, 0, c.stream>>>(
        d_plan, d_par, d_pid, np, n, S, B, mut, mutcro, total, l.stream, l.hdr, l.win, l.gparent, l.gmtime, l.snapidx,
        l.pool, l.starts, l.walked, d_out, d_partner, c.d_err);
    note_launches(6);
    return cudaGetLastError();
}

}  // namespace etune_b200
