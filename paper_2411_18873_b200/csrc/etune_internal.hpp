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
    uint32_t off_fit[3];  // repair tables per dim (FitTables below)
    uint32_t total;
};

// repair_schedule's "tilings whose threads fit" lists (genetic.cpp:101-110), per dim:
//   int32 ntv; int32 pad; uint32 tv[ntv] (distinct thread counts, ascending);
//   uint32 start[ntv + 1]; uint16 list[] where list[start[c] .. start[c+1]) are the
//   tiling indices with threads <= tv[c], in enumeration order.
struct FitHeader {
    int32_t ntv, pad;
};

// ------------------------------------------------------------ score blob
// Per (plan, forest).  Each feature is a function of one "channel key" of the
// candidate (e.g. glb_ld, f2/f5/f15, is keyed by the (block-tile m, block-tile n)
// divisor pair).  The host partitions every channel's key domain into classes of
// identical test outcomes over the whole forest, then stores per (tree, channel) a
// lookup table  class -> bitmask of the tree's leaves that stay reachable
// (QuickScorer: a node whose test goes right removes its left subtree's leaves).
// Device: mask = AND_c LUT[t][c][class_c]; exit leaf = lowest set bit; leaf values
// are the reference's doubles, summed in tree order (energy_model.cpp:247).
enum Channel : int {
    kChInt = 0,   // (dpt_m, dpt_n)          -> f1, f4 (int_ops = shared_ld)
    kChGlb = 1,   // (dbt_m, dbt_n)          -> f2, f5, f15 (glb_ld = shared_st)
    kChGrid = 2,  // grid index              -> f11, f14
    kChBlk = 3,   // block size 0..1024      -> f12
    kChEff = 4,   // f13 rank bin            -> f13 (sm_efficiency = a(grid) * b(block))
    kChKuv = 5,   // (k idx, log2 u, log2 v) -> f10, f7, f6
    kChLvp = 6,   // (levels, dpt_n)         -> f8, f9
    kNumChannels = 7
};

struct TreeRec {          // 32 bytes, read warp-uniformly (kernel-parameter constant bank)
    uint32_t lut[7];      // byte offset (from the blob start) of this tree's class->mask
                          // table per channel; only meaningful when the channel is used
    uint32_t meta;        // byte offset of the tree's leaf values (bits 0-23) | used-channel mask << 24
};
constexpr int kMaxParamTrees = 1000;  // 32000 B of kernel parameters (CUDA 12.1+: 32764 max)
// Pair mode (32-bit leaf masks): trees 2p and 2p+1 share one record and one 64-bit
// class->(mask_a | mask_b << 32) table per channel, so one 8-byte shared load serves
// both trees (one wavefront when the channel has <= 16 classes).
struct PairRec {          // 36 bytes
    uint32_t lut[7];      // byte offset of the pair's class->mask-pair table per channel
    uint32_t meta_a;      // leaf block of tree 2p (bits 0-23) | union of used channels << 24
    uint32_t meta_b;      // leaf block of tree 2p+1 (bits 0-23) | 1 << 31 when tree 2p+1 exists
};
static_assert(sizeof(PairRec) == 36, "PairRec layout");
union ForestParams {
    TreeRec rec[kMaxParamTrees];
    PairRec pair[kMaxParamTrees / 2];
};

struct ScoreHdr {
    int64_t K;
    uint64_t fnv_prefix;
    double base, lr;
    int32_t ntrees, mask_bits;   // 32 or 64
    int32_t nt[3], nd[3], ndk, ngrid, n13, npairs;  // npairs > 0: pair mode (PairRec records)
    uint32_t off_til[3];     // TilingRec
    uint32_t off_divk;       // int64 k values (ids)
    uint32_t off_gridkey;    // uint16 [nd0][nd1][nd2]
    uint32_t off_grida;      // double per grid: active/sms
    uint32_t off_blockb;     // double per block 0..1024: min(1, block/256)
    uint32_t off_f13;        // double[n13] effective f13 boundaries
    uint32_t off_cls[7];     // uint8 class tables per channel key (kChEff: none)
    uint32_t off_trees;      // TreeRec[ntrees] or PairRec[npairs]
    uint32_t off_lut;        // mask words (uint32 or uint64; pair mode: uint64 mask pairs)
    uint32_t off_leaves;     // double
    uint32_t total;
};

// --------------------------------------------------------- keyed score blob
// Every channel except Kuv is a function of the three tiling indices alone, so the
// forest compiler evaluates, per tiling triple ("key"), each tree's AND of its non-Kuv
// channel masks M_t(key) and stores one byte per (key, tree) in a key table in global
// memory (L2-resident, rows of `row_bytes`, 16-byte aligned):
//   trees that do not test Kuv: the exit leaf's de Bruijn slot of M_t(key) itself;
//   trees that do:              the index of M_t(key) in the tree's list of distinct
//                               masks (<= 256; lists packed, per-tree start in the
//                               kernel-parameter bank), ANDed on the device with the
//                               tree's Kuv-class mask.
// A candidate reads its row with 16-byte loads (16 trees each), so the per-tree work is
// one or three shared loads (+ the two leaf words) instead of one table load per channel.
// Full form (when the table stays <= 64 MB): one row per (key, Kuv class) holding every
// tree's exit slot as 5 bits, 25 per 16-byte quad (100 trees: 64-byte rows), so a tree costs
// only its leaf words.
// Blob (shared memory): header, divisors of K, Kuv class table, leaf blocks (32 hi + 32 lo
// words/tree) -- the full form stages only this prefix -- then tilings, packed mask lists,
// Kuv masks [tree][nkc].
struct KeyedHdr {
    int64_t K;
    uint64_t fnv_prefix;
    double base, lr;
    int32_t ntrees, row_bytes, nkc, pad0;
    int32_t nt[3], nd[3], ndk, pad1;
    uint32_t kuv_flags[4];  // bit t: tree t tests Kuv (ntrees <= 128)
    uint32_t off_til[3];
    uint32_t off_divk;
    uint32_t off_clskuv;   // uint8 [(k*16+u)*4+v] -> Kuv class
    uint32_t off_mlist;    // uint32: distinct non-Kuv masks of the Kuv trees, tree after tree
    uint32_t off_kuvtab;   // uint32 [tree][nkc]
    uint32_t off_leaves;   // per tree 32 high words then 32 low words, de Bruijn slots
    uint32_t total;
    uint32_t full_bytes;   // prefix the full form reads (header, divk, Kuv classes, leaves)
};
constexpr int kKeyedMaxTrees = 128;
struct KeyedParams {       // kernel parameter (constant bank: warp-uniform reads cost no shared-memory issue)
    uint32_t moff[kKeyedMaxTrees];  // byte offset of tree t's mask list from the blob start
    uint32_t koff[kKeyedMaxTrees];  // byte offset of tree t's Kuv-mask row ([tree][nkc]) from the blob start
    uint32_t kuv_flags[4];          // copy of KeyedHdr::kuv_flags (all zero in the full form)
    uint32_t off_kuvtab, off_leaves, nkc, ntrees;
    uint32_t kfull;                 // 1: rows per (key, Kuv class) of 5-bit exit slots (25 per quad)
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
