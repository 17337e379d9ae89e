// Device helpers shared by the scoring kernels (kernels.cu, rowtab.cu): candidate_id's
// FNV-1a, the genome -> knob records decode, features_from_counters through the plan's
// tables, the reference tree walk, and the fused selection's bucket function.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "etune_internal.hpp"
#include "kernels.hpp"
#include "selbin.cuh"

namespace etune_b200 {


constexpr uint64_t kFnvPrime = 1099511628211ull;
constexpr uint64_t mulmod64(uint64_t a, uint64_t b) { return a * b; }
constexpr uint64_t kFnvPrime4 = mulmod64(mulmod64(kFnvPrime, kFnvPrime), mulmod64(kFnvPrime, kFnvPrime));


__device__ __forceinline__ void stage(const uint8_t* __restrict__ g, uint32_t bytes, int4* s) {
    const int4* src = reinterpret_cast<const int4*>(g);
    const uint32_t n16 = bytes >> 4;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) s[i] = __ldg(src + i);
}

__device__ __forceinline__ void report(unsigned long long* err, int64_t index, int code) {
    atomicMin(err, (static_cast<unsigned long long>(index) << 8) | static_cast<unsigned>(code));
}

// FNV-1a over one 8-byte little-endian word whose upper 4 bytes are zero (every
// schedule value is < 2^32): 4 byte steps, then the 4 zero bytes as one multiply.
__device__ __forceinline__ uint64_t fnv_small(uint64_t h, uint32_t v) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        h ^= (v >> (8 * b)) & 0xffu;
        h *= kFnvPrime;
    }
    return h * kFnvPrime4;
}

template <typename T>
__device__ __forceinline__ const T* at(const uint8_t* base, uint32_t off) {
    return reinterpret_cast<const T*>(base + off);
}

struct Knobs {
    TilingRec r[3];
    int64_t k_tile;
    uint32_t unroll, vec;
    uint32_t k;
};

__device__ __forceinline__ uint64_t candidate_hash(uint64_t prefix, const Knobs& c) {
    uint64_t h = prefix;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        h = fnv_small(h, c.r[d].blocks);
        h = fnv_small(h, c.r[d].threads);
        h = fnv_small(h, c.r[d].pt);
    }
    h = fnv_small(h, static_cast<uint32_t>(c.k_tile));
    h = fnv_small(h, c.unroll);
    h = fnv_small(h, c.vec);
    return h;
}

__device__ __forceinline__ Knobs load_knobs(const uint8_t* P, const PlanHdr& H, uint64_t g) {
    const Genome x = genome_unpack(g);
    Knobs c;
    c.r[0] = at<TilingRec>(P, H.off_til[0])[x.t0];
    c.r[1] = at<TilingRec>(P, H.off_til[1])[x.t1];
    c.r[2] = at<TilingRec>(P, H.off_til[2])[x.t2];
    c.k = x.k;
    c.k_tile = at<int64_t>(P, H.off_divk)[x.k];
    c.unroll = 1u << x.u;
    c.vec = 1u << x.v;
    return c;
}

// ---------------------------------------------------------------- features
// features_from_counters (features.cpp:15-46) through the plan's tables.
__device__ __forceinline__ void plan_features(const uint8_t* P, const PlanHdr& H, const Knobs& c, double f[16]) {
    const int nd1 = H.nd[1], nd2 = H.nd[2];
    const uint32_t block = c.r[0].threads * c.r[1].threads * c.r[2].threads;
    const uint32_t gk = at<uint16_t>(P, H.off_gridkey)[(c.r[0].db * nd1 + c.r[1].db) * nd2 + c.r[2].db];
    const GridRec gr = at<GridRec>(P, H.off_grid)[gk];
    const GlbRec gl = at<GlbRec>(P, H.off_glb2)[c.r[1].dbt * nd2 + c.r[2].dbt];
    const double lint = at<double>(P, H.off_int2)[c.r[1].dpt * nd2 + c.r[2].dpt];
    const BlockRec br = at<BlockRec>(P, H.off_block)[block <= 1024 ? block : 1024];
    const int lv = (c.r[0].pt > 1) + (c.r[1].pt > 1) + (c.r[2].pt > 1);
    f[0] = H.f0;
    f[1] = lint;
    f[2] = gl.lg_glb_ld;
    f[3] = H.f3;
    f[4] = lint;
    f[5] = gl.lg_glb_ld;
    f[6] = static_cast<double>(c.vec);
    f[7] = static_cast<double>(c.unroll);
    f[8] = at<double>(P, H.off_lvl)[lv];
    f[9] = at<double>(P, H.off_ptn)[c.r[2].dpt];
    f[10] = at<double>(P, H.off_steps)[c.k];
    f[11] = gr.lg_grid;
    f[12] = br.lg_block;
    f[13] = __dmul_rn(gr.a, br.b);
    f[14] = gr.lg_active;
    f[15] = gl.f15;
}


// RegressionTree::eval summed in tree order (energy_model.cpp:36-44, 245-249)
__device__ __forceinline__ double walk_forest(const PredictHdr& H, const int32_t* roots, const GNode* nodes,
                                              const double f[16]) {
    double sum = 0.0;
    for (int t = 0; t < H.ntrees; ++t) {
        int node = roots[t];
        int feature = nodes[node].feature;
        while (feature >= 0) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < 16; ++j) v = (j == feature) ? f[j] : v;
            node = v < nodes[node].thr ? nodes[node].left : nodes[node].right;
            feature = nodes[node].feature;
        }
        sum = __dadd_rn(sum, nodes[node].value);
    }
    const double p = __dadd_rn(H.base, __dmul_rn(H.lr, sum));
    return (1e-6 < p) ? p : 1e-6;
}


}  // namespace etune_b200
