// Per-candidate scoring core shared by score_kernel (kernels.cu).  Written as a
// __host__ __device__ template only so that tests/cpp/score_core_test.cpp can check
// the forest compiler's tables on a CPU without a GPU; the product never calls it on
// the host (libetune_cuda.so has no host scoring path).
#pragma once

#include <cstdint>
#include <cstring>

#include "etune_internal.hpp"

#if !defined(__CUDACC__) && !defined(__forceinline__)
#define __forceinline__ inline
#endif
#if defined(__CUDACC__)
#define ETUNE_UNROLL _Pragma("unroll")
#else
#define ETUNE_UNROLL  // host builds (forest compiler, tests): plain loops
#endif

#if defined(__CUDA_ARCH__)
#define ETUNE_DMUL(a, b) __dmul_rn(a, b)
#define ETUNE_DADD(a, b) __dadd_rn(a, b)
#define ETUNE_FFS32(x) (__ffs(int(x)) - 1)
#define ETUNE_FFS64(x) (__ffsll((long long)(x)) - 1)
#else
#define ETUNE_DMUL(a, b) ((a) * (b))
#define ETUNE_DADD(a, b) ((a) + (b))
#define ETUNE_FFS32(x) (__builtin_ffs(int(x)) - 1)
#define ETUNE_FFS64(x) (__builtin_ffsll((long long)(x)) - 1)
#endif

namespace etune_b200 {

template <typename T>
__host__ __device__ __forceinline__ const T* blob_at(const uint8_t* base, uint32_t off) {
    return reinterpret_cast<const T*>(base + off);
}

// Class of every channel for one genome (see Channel in etune_internal.hpp), plus the
// tiling records the candidate id needs.
struct CandClasses {
    uint32_t c[kNumChannels];
    TilingRec r[3];
    Genome x;
};

__host__ __device__ __forceinline__ CandClasses candidate_classes(const uint8_t* S, const ScoreHdr& H, uint64_t g) {
    CandClasses o;
    o.x = genome_unpack(g);
    o.r[0] = blob_at<TilingRec>(S, H.off_til[0])[o.x.t0];
    o.r[1] = blob_at<TilingRec>(S, H.off_til[1])[o.x.t1];
    o.r[2] = blob_at<TilingRec>(S, H.off_til[2])[o.x.t2];
    const int nd1 = H.nd[1], nd2 = H.nd[2];
    uint32_t block = o.r[0].threads * o.r[1].threads * o.r[2].threads;
    block = block <= 1024u ? block : 1024u;
    const uint32_t gk = blob_at<uint16_t>(S, H.off_gridkey)[(o.r[0].db * nd1 + o.r[1].db) * nd2 + o.r[2].db];
    const uint32_t lv = (o.r[0].pt > 1) + (o.r[1].pt > 1) + (o.r[2].pt > 1);
    o.c[kChInt] = blob_at<uint8_t>(S, H.off_cls[kChInt])[o.r[1].dpt * nd2 + o.r[2].dpt];
    o.c[kChGlb] = blob_at<uint8_t>(S, H.off_cls[kChGlb])[o.r[1].dbt * nd2 + o.r[2].dbt];
    o.c[kChGrid] = blob_at<uint8_t>(S, H.off_cls[kChGrid])[gk];
    o.c[kChBlk] = blob_at<uint8_t>(S, H.off_cls[kChBlk])[block];
    // f13 = (active/sms) * min(1, block/256) (counters.cpp:44-47), exact IEEE product
    const double x13 = ETUNE_DMUL(blob_at<double>(S, H.off_grida)[gk], blob_at<double>(S, H.off_blockb)[block]);
    const double* f13 = blob_at<double>(S, H.off_f13);
    int lo = 0, hi = H.n13;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (f13[mid] <= x13) lo = mid + 1;
        else hi = mid;
    }
    o.c[kChEff] = uint32_t(lo);
    o.c[kChKuv] = blob_at<uint8_t>(S, H.off_cls[kChKuv])[(o.x.k * 16u + o.x.u) * 4u + o.x.v];
    o.c[kChLvp] = blob_at<uint8_t>(S, H.off_cls[kChLvp])[lv * nd2 + o.r[2].dpt];
    return o;
}

// Sum of leaf values over trees [0, ntrees) in tree order (energy_model.cpp:247).
// `trees` is warp-uniform (on the device: the kernel-parameter constant bank);
// channels a tree does not test are skipped by predication (no smem traffic).
// `cb` are the candidate's channel classes pre-scaled to byte offsets
// (class * sizeof(M)); table and leaf offsets in the records are byte offsets from
// the blob start, so each lookup is one add + one shared load.
// Shared-memory loads by 32-bit shared-window address on the device (one IADD per
// table lookup: record offset + pre-scaled class + blob base); host: plain pointers.
#if defined(__CUDA_ARCH__)
using SAddr = uint32_t;
__device__ __forceinline__ uint32_t lds32(SAddr a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint64_t lds64(SAddr a) {
    uint64_t v;
    asm("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double ldsf64(SAddr a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ SAddr blob_saddr(const uint8_t* S) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(S));
}
#else
using SAddr = const uint8_t*;
inline uint32_t lds32(SAddr a) { return *reinterpret_cast<const uint32_t*>(a); }
inline uint64_t lds64(SAddr a) { return *reinterpret_cast<const uint64_t*>(a); }
inline double ldsf64(SAddr a) { return *reinterpret_cast<const double*>(a); }
inline SAddr blob_saddr(const uint8_t* S) { return S; }
#endif

#if defined(__CUDA_ARCH__)
__device__ __forceinline__ double join_f64(uint32_t hi, uint32_t lo) { return __hiloint2double(int(hi), int(lo)); }
#else
inline double join_f64(uint32_t hi, uint32_t lo) {
    const uint64_t b = (uint64_t(hi) << 32) | lo;
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}
#endif

template <typename M>
__host__ __device__ __forceinline__ M lds_mask(SAddr a) {
    if constexpr (sizeof(M) == 4) return lds32(a);
    else return lds64(a);
}

// `cb[ch]` = blob base + class * sizeof(M): each lookup is one add + one shared load.
template <typename M>
__host__ __device__ __forceinline__ M tree_mask(const TreeRec& r, const SAddr* cb) {
    M m = ~M(0);
ETUNE_UNROLL
    for (int ch = 0; ch < kNumChannels; ++ch)
        if ((r.meta >> (24 + ch)) & 1u) m &= lds_mask<M>(cb[ch] + r.lut[ch]);
    return m;
}

// Exit leaf = lowest set bit of the mask; leaves are stored at the de Bruijn slot of
// their bit (forest.cpp), so the slot is (m & -m) * B >> (bits - log2 bits): integer
// ALU/FMA-pipe work instead of a BREV + FLO pair on the saturated XU pipe.
template <typename M>
__host__ __device__ __forceinline__ double leaf_value(SAddr base, const TreeRec& r, M m) {
    uint32_t slot;
    if constexpr (sizeof(M) == 4) {
        slot = (uint32_t(m & (0u - m)) * 0x077CB531u) >> 27;
    } else {
        slot = uint32_t((uint64_t(m & (0ull - m)) * 0x03f79d71b4ca8b09ull) >> 58);
    }
    const SAddr blk = base + ((r.meta & 0xffffffu) + slot * 4u);
    const uint32_t hi = lds32(blk);
    const uint32_t lo = lds32(blk + uint32_t(sizeof(M)) * 32u);  // low words follow the mbits high words
    return join_f64(hi, lo);
}

template <typename M>
__host__ __device__ __forceinline__ double forest_sum(const uint8_t* S, const ScoreHdr& H, const TreeRec* trees,
                                                      const uint32_t* c) {
    const SAddr base = blob_saddr(S);
    SAddr cb[kNumChannels];
ETUNE_UNROLL
    for (int ch = 0; ch < kNumChannels; ++ch) cb[ch] = base + c[ch] * uint32_t(sizeof(M));
    double sum = 0.0;
    int t = 0;
    const int nt = H.ntrees;
    // two trees per iteration: their table reads are independent (ILP)
    for (; t + 1 < nt; t += 2) {
        const TreeRec a = trees[t];
        const TreeRec b = trees[t + 1];
        const M ma = tree_mask<M>(a, cb);
        const M mb = tree_mask<M>(b, cb);
        const double va = leaf_value<M>(base, a, ma);
        const double vb = leaf_value<M>(base, b, mb);
        sum = ETUNE_DADD(sum, va);
        sum = ETUNE_DADD(sum, vb);
    }
    for (; t < nt; ++t) {
        const TreeRec a = trees[t];
        sum = ETUNE_DADD(sum, leaf_value<M>(base, a, tree_mask<M>(a, cb)));
    }
    return sum;
}

// Pair mode (32-bit masks): one 8-byte table load per used channel serves trees 2p and
// 2p+1; `cb8[ch]` = blob base + class * 8.  Sums stay in tree order.
__host__ __device__ __forceinline__ double leaf_value32(SAddr base, uint32_t off, uint32_t m) {
    const uint32_t slot = ((m & (0u - m)) * 0x077CB531u) >> 27;
    const SAddr blk = base + off + slot * 4u;
    return join_f64(lds32(blk), lds32(blk + 128u));
}

__host__ __device__ __forceinline__ double forest_sum_pairs(const uint8_t* S, const ScoreHdr& H, const PairRec* pairs,
                                                            const uint32_t* c) {
    const SAddr base = blob_saddr(S);
    SAddr cb[kNumChannels];
ETUNE_UNROLL
    for (int ch = 0; ch < kNumChannels; ++ch) cb[ch] = base + c[ch] * 8u;
    double sum = 0.0;
    const int np = H.npairs;
    for (int p = 0; p < np; ++p) {
        const PairRec r = pairs[p];
        uint64_t m = ~0ull;
ETUNE_UNROLL
        for (int ch = 0; ch < kNumChannels; ++ch)
            if ((r.meta_a >> (24 + ch)) & 1u) m &= lds64(cb[ch] + r.lut[ch]);
        const double va = leaf_value32(base, r.meta_a & 0xffffffu, uint32_t(m));
        sum = ETUNE_DADD(sum, va);
        if (r.meta_b >> 31) {
            const double vb = leaf_value32(base, r.meta_b & 0xffffffu, uint32_t(m >> 32));
            sum = ETUNE_DADD(sum, vb);
        }
    }
    return sum;
}

// Keyed form (KeyedHdr, etune_internal.hpp): sum of leaf values in tree order from the
// candidate's key-table row (one byte per tree, 16 trees per 16-byte load) and its Kuv
// class.  `row` is global memory on the device (read-only path), host memory in tests.
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ uint4 ld_row16(const uint8_t* row, int q) {
    return __ldg(reinterpret_cast<const uint4*>(row) + q);
}
// 32 bytes (one sector) per thread in one 256-bit load (sm_100: LDG.256)
struct RowOct {
    uint32_t w[8];
};
__device__ __forceinline__ RowOct ld_row32(const uint8_t* row, int o) {
    RowOct r;
    asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
          "=r"(r.w[7])
        : "l"(row + 32 * o));
    return r;
}
#else
struct RowQuad {
    uint32_t x, y, z, w;
};
inline RowQuad ld_row16(const uint8_t* row, int q) {
    RowQuad r;
    std::memcpy(&r, row + 16 * q, 16);
    return r;
}
struct RowOct {
    uint32_t w[8];
};
inline RowOct ld_row32(const uint8_t* row, int o) {
    RowOct r;
    std::memcpy(&r, row + 32 * o, 32);
    return r;
}
#endif

// tree t's leaf value from its row byte: Kuv trees AND their listed mask with the
// Kuv-class mask (both conflict-free rows), the others hold the slot itself.  All tree
// constants come from KeyedParams (the kernel-parameter bank on the device).
// `kc4` = Kuv class * 4; tree constants are immediates of the parameter bank
__host__ __device__ __forceinline__ double keyed_leaf(const KeyedParams& P, SAddr base, uint32_t kc4, uint32_t t,
                                                      uint32_t code) {
    uint32_t slot = code;
    if ((P.kuv_flags[t >> 5] >> (t & 31)) & 1u) {
        const uint32_t m = lds32(base + P.moff[t] + code * 4u) & lds32(base + P.koff[t] + kc4);
        slot = ((m & (0u - m)) * 0x077CB531u) >> 27;
    }
    const SAddr blk = base + P.off_leaves + t * 256u + slot * 4u;
    return join_f64(lds32(blk), lds32(blk + 128u));
}

// byte j of w (one PRMT on the device)
__host__ __device__ __forceinline__ uint32_t byte_of(uint32_t w, uint32_t j) {
#if defined(__CUDA_ARCH__)
    return __byte_perm(w, 0u, 0x4440u + j);
#else
    return (w >> (8 * j)) & 0xffu;
#endif
}

// 16 trees from one 16-byte row quad; FULL: no per-tree bound checks
template <bool FULL>
__host__ __device__ __forceinline__ double keyed_group(const KeyedParams& P, SAddr base, uint32_t kc4, uint32_t t0,
                                                       const uint32_t* w, double sum) {
ETUNE_UNROLL
    for (uint32_t j = 0; j < 16; ++j) {
        const uint32_t t = t0 + j;
        if (FULL || t < P.ntrees) sum = ETUNE_DADD(sum, keyed_leaf(P, base, kc4, t, byte_of(w[j >> 2], j & 3)));
    }
    return sum;
}

// Full form: 25 trees per 16-byte quad, slot j of a quad at bits [5j, 5j + 5) of its
// 128 bits (little-endian words; slots 6, 12 and 19 straddle two words); rows are padded to
// whole 32-byte sectors and read one sector per load, so 100 trees are two 256-bit loads.
// FULL: no bound checks in the quad.
__host__ __device__ __forceinline__ uint32_t funnel_r(uint32_t lo, uint32_t hi, uint32_t sh) {
#if defined(__CUDA_ARCH__)
    return __funnelshift_r(lo, hi, sh);
#else
    return sh ? (lo >> sh) | (hi << (32u - sh)) : lo;
#endif
}

template <bool FULL>
__host__ __device__ __forceinline__ double keyed_group5(const KeyedParams& P, SAddr base, uint32_t t0,
                                                        const uint32_t* w, double sum) {
ETUNE_UNROLL
    for (uint32_t j = 0; j < 25; ++j) {
        const uint32_t t = t0 + j;
        if (FULL || t < P.ntrees) {
            const uint32_t b = 5u * j, i = b >> 5, sh = b & 31u;
            const uint32_t slot = (sh <= 27u ? (w[i] >> sh) : funnel_r(w[i], w[i + 1], sh)) & 31u;
            const SAddr blk = base + P.off_leaves + t * 256u + slot * 4u;
            sum = ETUNE_DADD(sum, join_f64(lds32(blk), lds32(blk + 128u)));
        }
    }
    return sum;
}

__host__ __device__ __forceinline__ double keyed_sum5(const uint8_t* KB, const KeyedParams& P, const uint8_t* row) {
    const SAddr base = blob_saddr(KB);
    double sum = 0.0;
    const uint32_t T = P.ntrees;
    // rows are whole 32-byte sectors: two quads (50 trees) per 256-bit load
ETUNE_UNROLL
    for (uint32_t t0 = 0; t0 < uint32_t(kKeyedMaxTrees); t0 += 50) {
        if (t0 >= T) break;
        const RowOct r = ld_row32(row, int(t0 / 50));
        if (t0 + 25 <= T) sum = keyed_group5<true>(P, base, t0, r.w, sum);
        else sum = keyed_group5<false>(P, base, t0, r.w, sum);
        if (t0 + 25 >= T) break;
        if (t0 + 50 <= T) sum = keyed_group5<true>(P, base, t0 + 25, r.w + 4, sum);
        else sum = keyed_group5<false>(P, base, t0 + 25, r.w + 4, sum);
    }
    return sum;
}

__host__ __device__ __forceinline__ double keyed_sum(const uint8_t* KB, const KeyedParams& P, const uint8_t* row,
                                                     uint32_t kc) {
    const SAddr base = blob_saddr(KB);
    const uint32_t kc4 = kc * 4u;
    double sum = 0.0;
    const uint32_t T = P.ntrees;
    // fully unrolled over the kKeyedMaxTrees bound: every tree constant is an immediate
    // constant-bank operand; whole groups of 16 trees carry no per-tree bound check
ETUNE_UNROLL
    for (uint32_t t0 = 0; t0 < uint32_t(kKeyedMaxTrees); t0 += 16) {
        if (t0 >= T) break;
        const auto r = ld_row16(row, int(t0 >> 4));
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
        if (t0 + 16 <= T) sum = keyed_group<true>(P, base, kc4, t0, w, sum);
        else sum = keyed_group<false>(P, base, kc4, t0, w, sum);
    }
    return sum;
}

__host__ __device__ __forceinline__ uint32_t keyed_key(const KeyedHdr& K, const Genome& x) {
    return (x.t0 * uint32_t(K.nt[1]) + x.t1) * uint32_t(K.nt[2]) + x.t2;
}

// row of a candidate in the key table: per key, or per (key, Kuv class) in the full form
__host__ __device__ __forceinline__ uint32_t keyed_row_index(const KeyedParams& P, const KeyedHdr& K, const Genome& x,
                                                             uint32_t kc) {
    const uint32_t key = keyed_key(K, x);
    return P.kfull ? key * P.nkc + kc : key;
}

__host__ __device__ __forceinline__ double keyed_finish(const KeyedHdr& K, double sum) {
    const double p = ETUNE_DADD(K.base, ETUNE_DMUL(K.lr, sum));  // energy_model.cpp:248
    return (1e-6 < p) ? p : 1e-6;
}

__host__ __device__ __forceinline__ double finish_prediction(const ScoreHdr& H, double sum) {
    const double p = ETUNE_DADD(H.base, ETUNE_DMUL(H.lr, sum));  // energy_model.cpp:248
    return (1e-6 < p) ? p : 1e-6;                                // std::max(kPredictionFloor, p)
}

}  // namespace etune_b200
