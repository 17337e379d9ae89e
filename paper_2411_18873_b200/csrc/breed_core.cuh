// The per-offspring decision code of reproduce() (genetic.cpp:137-187) shared by every
// device reproduce path: the single-CTA chain (breed.cu), the block-parallel exact path
// (breed_par.cu) and the opt-in counter mode.  breed_body() evaluates ONE offspring at a
// word offset of whatever word source the cursor reads; it is the reference's
// mutate_knob / crossover_with_mask / repair_schedule / validate_schedule sequence on the
// 8-byte genome, consuming the words in exactly the reference's order.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "etune_internal.hpp"

namespace etune_b200 {
namespace breedcore {

constexpr uint16_t kUnknown = 0;      // evaluation needs words beyond the available stream
constexpr uint16_t kIllegal = 0xffff; // repair produced an illegal schedule (reference throws)

template <typename T>
__device__ __forceinline__ const T* at(const uint8_t* base, uint32_t off) {
    return reinterpret_cast<const T*>(base + off);
}

// uniform_int_distribution<size_t>(0, r-1)(rng) of libstdc++ (GCC 13) on a 64-bit
// engine: Lemire's multiply-shift with the (-r % r) rejection threshold.
template <typename Cur>
__device__ __forceinline__ uint64_t lemire(Cur& c, uint64_t r) {
    uint64_t x = c.next();
    uint64_t lo = x * r;
    uint64_t hi = __umul64hi(x, r);
    if (lo < r) {
        const uint64_t thr = (0ull - r) % r;
        while (lo < thr && c.ok) {
            x = c.next();
            lo = x * r;
            hi = __umul64hi(x, r);
        }
    }
    return hi;
}

__device__ __forceinline__ int ctz64(int64_t v) { return __ffsll(static_cast<long long>(v)) - 1; }

struct BreedConst {
    const uint8_t* P;   // plan blob (shared memory when it fits)
    const uint64_t* par;
    const uint64_t* pid;
    int64_t np;
    double mut, mutcro, total;
    int has_other;
};

struct Child {
    uint64_t g;
    int32_t partner;
    uint16_t words;  // kUnknown / kIllegal / consumed count
};

// pick_different over options {0..m-1} (index space) avoiding index `a` that is one
// of them: alternatives are all options but `a`, in order (genetic.cpp:32-44).
template <typename Cur>
__device__ __forceinline__ uint32_t pick_other(Cur& c, uint32_t m, uint32_t a) {
    if (m <= 1) return a;
    const uint32_t j = uint32_t(lemire(c, m - 1));
    return j < a ? j : j + 1;
}

// pick_different over the power-of-two list {2^0..2^cap} avoiding 2^a (a may lie
// outside the list: then every option is an alternative) — legal_unrolls /
// legal_vectors in log2 form (genetic.cpp:11-29).
template <typename Cur>
__device__ __forceinline__ uint32_t pick_pow2(Cur& c, uint32_t cap, uint32_t a) {
    const uint32_t m = cap + 1;
    if (m <= 1) return 0;  // options.front() == 1
    if (a <= cap) {
        const uint32_t j = uint32_t(lemire(c, m - 1));
        return j < a ? j : j + 1;
    }
    return uint32_t(lemire(c, m));
}

// Counter-based word source (opt-in "counter" reproduce mode, etune_cu_reproduce_counter): offspring
// i draws its own stream word_j = splitmix64(key_i + j), key_i = splitmix64(seed ^ splitmix64(i)),
// so every offspring is independent of the others (one thread each) while consuming the words in
// exactly the reference's order and transforms (canonical, Lemire, masks).  Not the reference's
// mt19937_64 stream: its oracle is orc_reproduce_counter (oracle/etune_oracle.cpp).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

struct CounterCursor {
    uint64_t key;
    uint64_t p;  // words drawn
    bool ok;
    __device__ __forceinline__ uint64_t next() { return splitmix64(key + (p++)); }
};

template <typename Cur>
__device__ Child breed_body(const BreedConst& K, const PlanHdr& H, int64_t i, Cur& c, uint64_t start) {
    Child out{0, -1, kUnknown};
    const int64_t base = i % K.np;
    Genome x = genome_unpack(__ldg(K.par + base));
    const TilingRec* til[3] = {at<TilingRec>(K.P, H.off_til[0]), at<TilingRec>(K.P, H.off_til[1]),
                               at<TilingRec>(K.P, H.off_til[2])};
    const int64_t* divk = at<int64_t>(K.P, H.off_divk);
    // uniform_real_distribution<double>(0,1) = generate_canonical<double,53>: double(w) / 2^64,
    // clamped to nextafter(1, 0); then * total (genetic.cpp:162)
    const double coin = __dmul_rn(__ull2double_rn(c.next()), 0x1p-64);
    const double u = __dmul_rn(coin < 1.0 ? coin : 0x1.fffffffffffffp-1, K.total);
    bool repair = true;
    if (u < K.mut) {
        const uint32_t knob = uint32_t(lemire(c, 6));  // uniform_int_distribution<int>(0, 5)
        switch (knob) {
        case 0: x.t0 = pick_other(c, uint32_t(H.nt[0]), x.t0); break;
        case 1: x.t1 = pick_other(c, uint32_t(H.nt[1]), x.t1); break;
        case 2: x.t2 = pick_other(c, uint32_t(H.nt[2]), x.t2); break;
        case 3: x.k = pick_other(c, uint32_t(H.ndk), x.k); break;
        case 4: {
            const int cu = min(H.max_unroll_log2, ctz64(divk[x.k]));
            x.u = pick_pow2(c, uint32_t(cu), x.u);
            break;
        }
        default: {
            const int cv = min(H.max_vec_log2, ctz64(int64_t(til[2][x.t2].pt)));
            x.v = pick_pow2(c, uint32_t(cv), x.v);
            break;
        }
        }
    } else if (u < K.mutcro) {
        const uint64_t bid = __ldg(K.pid + base);
        int64_t pi = int64_t(lemire(c, uint64_t(K.np)));
        while (K.has_other && c.ok && __ldg(K.pid + pi) == bid) pi = int64_t(lemire(c, uint64_t(K.np)));
        const uint32_t mask = uint32_t(c.next() & 63u);
        const Genome y = genome_unpack(__ldg(K.par + pi));  // crossover_with_mask, genetic.cpp:48-58
        if (mask & 1u) x.t0 = y.t0;
        if (mask & 2u) x.t1 = y.t1;
        if (mask & 4u) x.t2 = y.t2;
        if (mask & 8u) x.k = y.k;
        if (mask & 16u) x.u = y.u;
        if (mask & 32u) x.v = y.v;
        out.partner = int32_t(pi);
    } else {
        repair = false;  // copy
    }
    if (repair && c.ok) {  // repair_schedule, genetic.cpp:89-135
        const int64_t cap = H.block_cap;
        uint32_t t[3] = {x.t0, x.t1, x.t2};
        for (int attempt = 0; attempt < 64 && c.ok; ++attempt) {
            const uint64_t th[3] = {til[0][t[0]].threads, til[1][t[1]].threads, til[2][t[2]].threads};
            const int64_t block = int64_t(th[0] * th[1] * th[2]);
            if (!(block > cap)) break;
            int dim = 0;
            if (th[1] > th[dim]) dim = 1;
            if (th[2] > th[dim]) dim = 2;
            const int64_t other = block / int64_t(th[dim]);
            // tilings with threads * other <= cap, in enumeration order: the precomputed
            // list for the largest distinct thread count <= cap / other
            const uint8_t* F = K.P + H.off_fit[dim];
            const int ntv = reinterpret_cast<const FitHeader*>(F)->ntv;
            const uint32_t* tv = reinterpret_cast<const uint32_t*>(F + sizeof(FitHeader));
            const uint32_t* start = tv + ntv;
            const uint16_t* list = reinterpret_cast<const uint16_t*>(start + ntv + 1);
            const int64_t lim = other > 0 ? cap / other : -1;
            int lo = 0, hi = ntv;  // number of distinct thread counts <= lim
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (int64_t(tv[mid]) <= lim) lo = mid + 1;
                else hi = mid;
            }
            const uint32_t fit = lo > 0 ? start[lo] - start[lo - 1] : 0u;
            if (fit == 0) {
                t[dim] = uint32_t(H.nt[dim] - 1);  // {extent, 1, 1}: the last tiling in enumeration order
            } else {
                const uint32_t r = uint32_t(lemire(c, fit));
                t[dim] = list[start[lo - 1] + r];
            }
        }
        x.t0 = t[0];
        x.t1 = t[1];
        x.t2 = t[2];
        // k_tile is a divisor of K by construction (genome index), so the k_tile branch never fires
        const uint32_t cu = uint32_t(min(H.max_unroll_log2, ctz64(divk[x.k])));
        if (x.u > cu) x.u = uint32_t(lemire(c, cu + 1));
        const uint32_t cv = uint32_t(min(H.max_vec_log2, ctz64(int64_t(til[2][x.t2].pt))));
        if (x.v > cv) x.v = uint32_t(lemire(c, cv + 1));
        const int64_t block =
            int64_t(uint64_t(til[0][x.t0].threads) * til[1][x.t1].threads * uint64_t(til[2][x.t2].threads));
        if (c.ok && (block < 1 || block > 1024)) {  // validate_schedule (schedule.cpp:26-61)
            out.words = kIllegal;
            return out;
        }
    }
    if (!c.ok) return out;
    out.g = genome_pack(x.t0, x.t1, x.t2, x.k, x.u, x.v);
    const uint64_t used = c.p - start;
    out.words = used < 0xfffeull ? uint16_t(used) : uint16_t(0xfffe);
    return out;
}

}  // namespace breedcore
}  // namespace etune_b200
