// Internal layouts shared by the host planner (plan.cpp, forest.cpp) and the
// sm_100a kernels (*.cu).  Everything a kernel needs sits in one contiguous,
// 16-byte aligned "blob" that the kernel stages into shared memory once per CTA.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/etune_cuda.h"

#if !defined(__CUDACC__) && !defined(__host__)
#define __host__
#endif
#if !defined(__CUDACC__) && !defined(__device__)
#define __device__
#endif

namespace etune_b200 {

// ---------------------------------------------------------------- genome
// One candidate = 64 bits of knob indices into the plan's tables.
//   [ 0,16) tiling index, batch dim     [16,32) tiling index, m dim
//   [32,48) tiling index, n dim         [48,58) index of k_tile in divisors(K)
//   [58,62) log2(unroll)                [62,64) log2(vectorize)
constexpr int kTilingBits = 16;
constexpr int kKBits = 10;
constexpr int kUBits = 4;
constexpr int kVBits = 2;
constexpr uint32_t kMaxTilings = 1u << kTilingBits;
constexpr uint32_t kMaxKDivisors = 1u << kKBits;

struct Genome {
    uint32_t t0, t1, t2, k, u, v;
};

__host__ __device__ inline uint64_t genome_pack(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t k,
                                                uint32_t u, uint32_t v) {
    return uint64_t(t0) | (uint64_t(t1) << 16) | (uint64_t(t2) << 32) | (uint64_t(k) << 48) |
           (uint64_t(u) << 58) | (uint64_t(v) << 62);
}
__host__ __device__ inline Genome genome_unpack(uint64_t g) {
    Genome r;
    r.t0 = uint32_t(g) & 0xffffu;
    r.t1 = uint32_t(g >> 16) & 0xffffu;
    r.t2 = uint32_t(g >> 32) & 0xffffu;
    r.k = uint32_t(g >> 48) & 0x3ffu;
    r.u = uint32_t(g >> 58) & 0xfu;
    r.v = uint32_t(g >> 62) & 0x3u;
    return r;
}

// One ordered factorisation extent = blocks * threads * per_thread
// (enumerate_dim_tilings, space.cpp:69-78), plus divisor indices of the quantities
// the feature tables are keyed by.
struct TilingRec {
    uint32_t blocks, threads, pt;
    uint16_t db;   // index of `blocks` in divisors(extent)
    uint16_t dpt;  // index of `per_thread`
    uint16_t dbt;  // index of `block_tile` = threads * per_thread
    uint16_t pad;
};
static_assert(sizeof(TilingRec) == 20, "TilingRec layout");

struct GridRec {      // per distinct grid value g (a divisor of B*M*N)
    double lg_grid;   // log1p(g)              f11
    double lg_active; // log1p(min(g, sms))    f14
    double a;         // double(active)/sms    first factor of f13
};
struct GlbRec {       // per (block-tile m, block-tile n)
    double lg_glb_ld; // log1p(glb_ld)         f2, f5
    double f15;       // flops / (glb_ld + glb_st + 1)
};
struct BlockRec {     // per block size 0..1024
    double lg_block;  // log1p(block)          f12
    double b;         // min(1, block/256)     second factor of f13
};

// ------------------------------------------------------------- plan blob
struct PlanHdr {
    int64_t B, M, N, K;
    int64_t flops, glb_st;
    uint64_t fnv_prefix;  // FNV-1a state after the 12 operator words
    double f0, f3;        // log1p(flops), log1p(glb_st): constant over the op
    int32_t nt[3];        // tilings per dim
    int32_t nd[3];        // divisors of B, M, N
    int32_t ndk;          // divisors of K
    int32_t ngrid;        // distinct grid values
    int32_t num_sms;      // DeviceConfig::num_sms of the model (not the GPU)
    int32_t block_cap;    // min(max_block_threads, 1024)
    int32_t max_unroll_log2, max_vec_log2;  // enumeration limits
    uint32_t off_til[3];  // TilingRec[nt[d]]
    uint32_t off_divk;    // int64 k_tile values [ndk]
    uint32_t off_gridkey; // uint16 [nd0][nd1][nd2] -> grid index
    uint32_t off_grid;    // GridRec[ngrid]
    uint32_t off_int2;    // double [nd1][nd2] (by per-thread divisor idx) log1p(int_ops)
    uint32_t off_glb2;    // GlbRec [nd1][nd2] (by block-tile divisor idx)
    uint32_t off_block;   // BlockRec[1025]
    uint32_t off_ptn;     // double [nd2] log1p(pt_n)
    uint32_t off_steps;   // double [ndk] log1p(K / k_tile)
    uint32_t off_lvl;     // double [4] log1p(8..11)
    uint32_t total;
};

// ------------------------------------------------------------ score blob
// Per (plan, forest): rank bins + the forest partially evaluated for the op and
// laid out as perfect binary trees of 32-bit test words.
//
// Bins: every feature j gets a byte b' = 1 + #(effective thresholds on j <= x);
// a node test "f[j] < thr" becomes "b'_j < r'" and is evaluated branch-free as
//   x = prmt(pairlo, pairhi, w) (byte j replicated x4);  go_right = (x >= w)
// with w = r' << 24 | pair << 16 | (j & 7) * 0x1111  (see forest.cpp).
struct TreeMeta {
    int32_t node_base;  // index into nodes[] (uint32)
    int32_t leaf_base;  // index into leaves[] (double)
    int32_t depth;      // perfect depth after partial evaluation (0 = single leaf)
    int32_t pad;
};

struct ScoreHdr {
    int64_t K;
    uint64_t fnv_prefix;
    double base, lr;
    int32_t ntrees, max_depth;
    int32_t nt[3], nd[3], ndk, ngrid;
    int32_t n13;             // effective f13 boundaries (device binary search)
    uint8_t bconst[16];      // bins of features constant over the op (f0, f3, ...)
    uint32_t off_til[3];     // TilingRec
    uint32_t off_divk;       // int64 k values (ids)
    uint32_t off_gridkey;    // uint16
    uint32_t off_bgrid;      // uint16 per grid: f11 | f14 << 8
    uint32_t off_grida;      // double per grid
    uint32_t off_bint2;      // uint16 per (dpt1, dpt2): f1 | f4 << 8
    uint32_t off_bglb2;      // uint32 per (dbt1, dbt2): f2 | f5 << 8 | f15 << 16
    uint32_t off_bblock;     // uint8 per block 0..1024: f12
    uint32_t off_blockb;     // double per block 0..1024
    uint32_t off_bptn;       // uint8 per dpt2: f9
    uint32_t off_bsteps;     // uint8 per k: f10
    uint32_t off_small;      // uint8[32]: lvl[4] (f8), u[16] (f7), v[4] (f6), pad
    uint32_t off_f13;        // double[n13] boundaries
    uint32_t off_meta;       // TreeMeta[ntrees]
    uint32_t off_nodes;      // uint32
    uint32_t off_leaves;     // double
    uint32_t total;
};

// ------------------------------------------------------- generic predict blob
// EnergyModel::predict on arbitrary feature vectors: reference node order.
struct GNode {
    double thr;
    int32_t feature;  // -1 leaf
    int32_t left;     // absolute node index (leaf: unused)
    int32_t right;
    int32_t pad;
    double value;
};
static_assert(sizeof(GNode) == 32, "GNode layout");
struct PredictHdr {
    int32_t ntrees;
    int32_t nnodes;
    double base, lr;
    uint32_t off_roots;  // int32 root index per tree
    uint32_t off_nodes;  // GNode
    uint32_t total;
    uint32_t pad;
};

inline uint32_t align16(size_t x) { return uint32_t((x + 15) & ~size_t(15)); }

// Host-side status plumbing.
void set_error(const std::string& msg);
struct Status {
    etune_status code;
    std::string msg;
};

}  // namespace etune_b200
