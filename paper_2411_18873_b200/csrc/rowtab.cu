// Row-table form of the cost model: the default scoring form, compiled on the device.
//
// Every feature of features_from_counters (features.cpp:15-46) is a function of the
// candidate's three spatial tilings ("key", e.g. glb_ld of the block tiles) except f6
// (vectorize), f7 (unroll) and f10 (log1p of K / k_tile), which depend on the reduction
// knobs (k_tile, unroll, vectorize) alone.  A tree's path (RegressionTree::eval,
// energy_model.cpp:36-44) only depends on which side of each threshold a feature falls,
// so two (k, u, v) triples whose f6 / f7 / f10 values pass exactly the same thresholds
// of the forest take the same path in every tree: they form one "Kuv class".  The
// prediction (energy_model.cpp:245-249) is therefore a pure function of the row
// (key, Kuv class), and there are far fewer rows than candidates (C2: 4704 keys x 21
// classes = 98,784 rows vs 2^20 candidates).
//
//   rowtab_classes_kernel  one CTA: the forest's thresholds on f6 / f7 / f10, each knob
//                          value's count of thresholds it does not fall below, the
//                          distinct attained count triples over the legal (k, u, v)
//                          -> Kuv class table [k][u][v] and one representative per class
//   rowtab_build_kernel    four lanes per row: the representative genome's features from
//                          the plan tables, the reference tree walk over the forest, the
//                          row's prediction (+ the lowest / highest order key for the
//                          fused selection's buckets)
//   score_rows_kernel      per candidate: genome -> row -> prediction (one 8-byte gather
//                          from the L2-resident table), candidate_id from the per-key FNV
//                          state, + the selection histogram
//
// Nothing is evaluated on the host: a model trained on the device is scorable without a
// host round trip, and the compile is three launches (tens of microseconds).  The row's
// prediction is computed by exactly the walk score_walk_kernel runs per candidate (same
// features, same doubles, tree-order sum, no FMA), so every form is bit-identical.
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <vector>

#include "etune_internal.hpp"
#include "kernels.hpp"
#include "pdl.cuh"
#include "plan_core.cuh"

namespace etune_b200 {

namespace {

constexpr int kClsT = 1024;
constexpr int kThrCache = 1024;  // thresholds per feature staged in shared memory
constexpr int kMaxJointWords = 2048;  // A10 * A7 * A6 <= 1024 * 16 * 3 bits

// Knob value domain of the Kuv channel: every (k_tile index, log2 unroll, log2 vec) a
// legal schedule can hold (validate_schedule, schedule.cpp:26-61: unroll a power of two
// dividing k_tile -- at most 2^15 in a genome -- and vectorize in {1, 2, 4}).
constexpr int kKuvU = 16;
constexpr int kKuvV = 3;

__device__ __forceinline__ int ctz64(int64_t x) { return x ? __ffsll(x) - 1 : 63; }

constexpr uint64_t kFnvP6 = kFnvPrime4 * kFnvPrime * kFnvPrime;  // six zero bytes
constexpr uint64_t kFnvP7 = kFnvP6 * kFnvPrime;

// candidate_id's last two words (space.cpp:43-44): unroll (a power of two <= 2^15: two non-zero
// bytes at most) and vectorize (one byte), from the state after k_tile
// fnv_small(h, v) (the four bytes of v, then the four zero bytes of the int64 word) with the zero
// bytes of a k_tile < 2^16 folded into one multiply by P^6
__device__ __forceinline__ uint64_t fnv_ktile(uint64_t h, uint32_t v) {
    h = (h ^ (v & 0xffu)) * kFnvPrime;
    h = (h ^ ((v >> 8) & 0xffu)) * kFnvPrime;
    if (v >> 16) {
        h = (h ^ ((v >> 16) & 0xffu)) * kFnvPrime;
        h = (h ^ (v >> 24)) * kFnvPrime;
        return h * kFnvPrime4;
    }
    return h * kFnvP6;
}

__device__ __forceinline__ uint64_t fnv_tail(uint64_t h, uint32_t u, uint32_t v) {
    const uint32_t unroll = 1u << u;
    h = (h ^ (unroll & 0xffu)) * kFnvPrime;
    h = (h ^ (unroll >> 8)) * kFnvPrime;
    h *= kFnvP6;
    h = (h ^ (1u << v)) * kFnvPrime;
    return h * kFnvP7;
}

// thresholds t of one feature with !(x < t): the tests x passes to the right
__device__ __forceinline__ int count_right(double x, const double* t, int n) {
    int c = 0;
    for (int i = 0; i < n; ++i) c += !(x < t[i]);
    return c;
}

struct ClsSmem {
    double thr[3][kThrCache];   // f10, f7, f6 thresholds
    int cnt[3];
    int A[3];                   // attained distinct counts per feature (k, u, v)
    int c10[1024], a10[1024], rep10[1024], f10[1024];
    int c7[kKuvU], a7[kKuvU], rep7[kKuvU], f7[kKuvU];
    int c6[4], a6[4], rep6[4], f6[4];
    uint32_t bits[kMaxJointWords];
    uint32_t pre[kMaxJointWords];
    uint32_t scan[32];
};

__global__ void __launch_bounds__(kClsT, 1) rowtab_classes_kernel(const uint8_t* __restrict__ P,
                                                                  const uint8_t* __restrict__ Q,
                                                                  double* __restrict__ gthr, int nnodes,
                                                                  RowTabMeta* __restrict__ meta,
                                                                  uint16_t* __restrict__ clskuv,
                                                                  uint32_t* __restrict__ crep) {
    extern __shared__ int4 dsm[];
    ClsSmem& S = *reinterpret_cast<ClsSmem*>(dsm);
    const int tid = threadIdx.x;
    pdl_wait();
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    const PredictHdr& QH = *reinterpret_cast<const PredictHdr*>(Q);
    const GNode* nodes = at<GNode>(Q, QH.off_nodes);
    const int64_t* divk = at<int64_t>(P, H.off_divk);
    const double* steps = at<double>(P, H.off_steps);  // f10 = log1p(K / k_tile) per k index
    const int ndk = H.ndk;
    if (tid < 3) S.cnt[tid] = 0;
    __syncthreads();
    // 1. the forest's thresholds on f10 / f7 / f6 (order within a list is irrelevant: only counts are used)
    for (int i = tid; i < nnodes; i += blockDim.x) {
        const int f = nodes[i].feature;
        const int s = f == 10 ? 0 : f == 7 ? 1 : f == 6 ? 2 : -1;
        if (s >= 0) gthr[size_t(s) * nnodes + atomicAdd(&S.cnt[s], 1)] = nodes[i].thr;
    }
    __syncthreads();
    const double* T[3];
    for (int s = 0; s < 3; ++s) {
        const int n = S.cnt[s];
        if (n <= kThrCache) {
            for (int i = tid; i < n; i += blockDim.x) S.thr[s][i] = gthr[size_t(s) * nnodes + i];
            T[s] = S.thr[s];
        } else {
            T[s] = gthr + size_t(s) * nnodes;
        }
    }
    __syncthreads();
    // 2. per knob value: how many of the feature's thresholds it passes to the right
    for (int k = tid; k < ndk; k += blockDim.x) S.c10[k] = count_right(steps[k], T[0], S.cnt[0]);
    if (tid < kKuvU) S.c7[tid] = count_right(double(1u << tid), T[1], S.cnt[1]);
    if (tid < kKuvV) S.c6[tid] = count_right(double(1u << tid), T[2], S.cnt[2]);
    __syncthreads();
    // 3. dense rank of each value's count among the distinct counts; the first value with
    //    each count represents its class
    for (int k = tid; k < ndk; k += blockDim.x) {
        bool first = true;
        for (int j = 0; j < k && first; ++j) first = S.c10[j] != S.c10[k];
        S.f10[k] = first;
    }
    if (tid < kKuvU) {
        bool first = true;
        for (int j = 0; j < tid && first; ++j) first = S.c7[j] != S.c7[tid];
        S.f7[tid] = first;
    }
    if (tid < kKuvV) {
        bool first = true;
        for (int j = 0; j < tid && first; ++j) first = S.c6[j] != S.c6[tid];
        S.f6[tid] = first;
    }
    __syncthreads();
    for (int k = tid; k < ndk; k += blockDim.x) {
        int a = 0;
        for (int j = 0; j < ndk; ++j) a += S.f10[j] && S.c10[j] < S.c10[k];
        S.a10[k] = a;
        if (S.f10[k]) S.rep10[a] = k;
    }
    if (tid < kKuvU) {
        int a = 0;
        for (int j = 0; j < kKuvU; ++j) a += S.f7[j] && S.c7[j] < S.c7[tid];
        S.a7[tid] = a;
        if (S.f7[tid]) S.rep7[a] = tid;
    }
    if (tid < kKuvV) {
        int a = 0;
        for (int j = 0; j < kKuvV; ++j) a += S.f6[j] && S.c6[j] < S.c6[tid];
        S.a6[tid] = a;
        if (S.f6[tid]) S.rep6[a] = tid;
    }
    if (tid == 0) {
        int a = 0, b = 0, d = 0;
        for (int k = 0; k < ndk; ++k) a += S.f10[k];
        for (int u = 0; u < kKuvU; ++u) b += S.f7[u];
        for (int v = 0; v < kKuvV; ++v) d += S.f6[v];
        S.A[0] = a;
        S.A[1] = b;
        S.A[2] = d;
    }
    __syncthreads();
    const int A10 = S.A[0], A7 = S.A[1], A6 = S.A[2];
    const int J = A10 * A7 * A6;
    const int words = (J + 31) >> 5;
    for (int w = tid; w < words; w += blockDim.x) S.bits[w] = 0u;
    __syncthreads();
    // 4. joint count triples attained by legal (k, u, v): one bit each
    const int ncombo = ndk * 64;
    for (int idx = tid; idx < ncombo; idx += blockDim.x) {
        const int k = idx >> 6, u = (idx >> 2) & 15, v = idx & 3;
        if (v < kKuvV && u <= ctz64(divk[k])) {
            const int j = (S.a10[k] * A7 + S.a7[u]) * A6 + S.a6[v];
            atomicOr(&S.bits[j >> 5], 1u << (j & 31));
        }
    }
    __syncthreads();
    // exclusive popcount prefix over the words (<= 2048 words: two per thread)
    {
        const int w0 = 2 * tid;
        const uint32_t p0 = w0 < words ? __popc(S.bits[w0]) : 0u;
        const uint32_t p1 = w0 + 1 < words ? __popc(S.bits[w0 + 1]) : 0u;
        const uint32_t mine = p0 + p1;
        uint32_t x = mine;
        for (int s = 1; s < 32; s <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
            if ((tid & 31) >= s) x += y;
        }
        if ((tid & 31) == 31) S.scan[tid >> 5] = x;
        __syncthreads();
        if (tid < 32) {
            uint32_t z = S.scan[tid];
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, z, s);
                if (tid >= s) z += y;
            }
            S.scan[tid] = z;  // inclusive per warp
        }
        __syncthreads();
        const uint32_t before = (tid >> 5) ? S.scan[(tid >> 5) - 1] : 0u;
        const uint32_t ex = before + x - mine;
        if (w0 < words) S.pre[w0] = ex;
        if (w0 + 1 < words) S.pre[w0 + 1] = ex + p0;
    }
    __syncthreads();
    // 5. class of every (k, u, v) and the representative knob values of every class
    for (int idx = tid; idx < ncombo; idx += blockDim.x) {
        const int k = idx >> 6, u = (idx >> 2) & 15, v = idx & 3;
        uint16_t cls = 0xffffu;
        if (v < kKuvV && u <= ctz64(divk[k])) {
            const int j = (S.a10[k] * A7 + S.a7[u]) * A6 + S.a6[v];
            cls = uint16_t(S.pre[j >> 5] + __popc(S.bits[j >> 5] & ((1u << (j & 31)) - 1u)));
        }
        clskuv[idx] = cls;
    }
    for (int j = tid; j < J; j += blockDim.x) {
        if ((S.bits[j >> 5] >> (j & 31)) & 1u) {
            const uint32_t cls = S.pre[j >> 5] + __popc(S.bits[j >> 5] & ((1u << (j & 31)) - 1u));
            const int i6 = j % A6, i7 = (j / A6) % A7, i10 = j / (A6 * A7);
            crep[cls] = (uint32_t(S.rep10[i10]) << 8) | (uint32_t(S.rep7[i7]) << 2) | uint32_t(S.rep6[i6]);
        }
    }
    if (tid == 0) {
        meta->nkc = int32_t(words ? S.pre[words - 1] + __popc(S.bits[words - 1]) : 0);
        meta->bounds[0] = ~0ull;
        meta->bounds[1] = 0ull;
        meta->nthr[0] = S.cnt[0];
        meta->nthr[1] = S.cnt[1];
        meta->nthr[2] = S.cnt[2];
        meta->rows = int64_t(H.nt[0]) * H.nt[1] * H.nt[2] * int64_t(meta->nkc);
    }
}

constexpr int kBuildT = 256;
// compact walk: L lanes per row (4 by default), tree t on lane t % L; the lanes' leaf values are added
// in tree order through shuffles, so the sum is the reference's sequential one (bit-identical), while
// a row's dependent node-load chain is L times shorter and the rows spread evenly over the SMs
constexpr int kBuildFS = 17;  // feature-vector stride in doubles (16 + 1: the lanes' reads spread over the banks)

__device__ __forceinline__ uint64_t order_key(double p) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(p));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Node of the build walk: 16 bytes in shared memory (vs the 32-byte GNode) so the forest and
// the per-thread feature vectors fit two CTAs per SM.  tv = threshold (interior) or leaf value;
// lr = left | right << 16 (absolute node indices, forests of < 65536 nodes).
struct CNode {
    double tv;
    uint32_t lr;
    int32_t feature;
};
static_assert(sizeof(CNode) == 16, "CNode layout");

// Per row: features of the row's representative genome, then RegressionTree::eval summed in tree
// order (energy_model.cpp:36-44, 245-249) -- the same comparisons, the same leaf doubles and the
// same DADD order as walk_forest / the reference.  COMPACT: nodes staged as CNode and the row's
// features in shared memory (one LDS per visited node), L lanes per row walking the trees
// round-robin; else one thread per row and the GNode walk over global memory (forests of >= 65536
// nodes or too large for shared memory).
template <bool COMPACT, int L>
__global__ void __launch_bounds__(kBuildT) rowtab_build_kernel(const uint8_t* __restrict__ P,
                                                               const uint8_t* __restrict__ Q, int nnodes,
                                                               RowTabMeta* __restrict__ meta,
                                                               const uint32_t* __restrict__ crep,
                                                               double* __restrict__ rowpred) {
    extern __shared__ int4 smem[];
    const PredictHdr& QH = *reinterpret_cast<const PredictHdr*>(Q);
    const int32_t* groots = at<int32_t>(Q, QH.off_roots);
    const GNode* gnodes = at<GNode>(Q, QH.off_nodes);
    const int ntrees = QH.ntrees;
    CNode* sn = reinterpret_cast<CNode*>(smem);
    int32_t* sroots = reinterpret_cast<int32_t*>(sn + nnodes);
    double* fs = reinterpret_cast<double*>(smem) + ((size_t(nnodes) * 16 + size_t(ntrees) * 4 + 15) / 16) * 2;
    if (COMPACT) {  // read-only forest: staged before the dependency wait (PDL)
        for (int i = threadIdx.x; i < nnodes; i += blockDim.x) {
            const GNode g = gnodes[i];
            CNode c;
            c.tv = g.feature >= 0 ? g.thr : g.value;
            c.lr = uint32_t(g.left & 0xffff) | (uint32_t(g.right & 0xffff) << 16);
            c.feature = g.feature;
            sn[i] = c;
        }
        for (int t = threadIdx.x; t < ntrees; t += blockDim.x) sroots[t] = groots[t];
        __syncthreads();
    }
    pdl_wait();
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    const TilingRec* T0 = at<TilingRec>(P, H.off_til[0]);
    const TilingRec* T1 = at<TilingRec>(P, H.off_til[1]);
    const TilingRec* T2 = at<TilingRec>(P, H.off_til[2]);
    const int64_t* divk = at<int64_t>(P, H.off_divk);
    const uint32_t nkc = uint32_t(meta->nkc);
    const uint32_t nt1 = uint32_t(H.nt[1]), nt2 = uint32_t(H.nt[2]);
    const int64_t rows = int64_t(H.nt[0]) * nt1 * nt2 * nkc;
    const double base = QH.base, lr = QH.lr;
    uint64_t lo = ~0ull, hi = 0ull;
    auto row_knobs = [&](int64_t r) {
        const uint32_t key = uint32_t(r / nkc), kc = uint32_t(r - int64_t(key) * nkc);
        const uint32_t t2 = key % nt2, q = key / nt2, t1 = q % nt1, t0 = q / nt1;
        const uint32_t rep = __ldg(crep + kc);
        Knobs c;
        c.r[0] = T0[t0];
        c.r[1] = T1[t1];
        c.r[2] = T2[t2];
        c.k = rep >> 8;
        c.k_tile = divk[c.k];
        c.unroll = 1u << ((rep >> 2) & 15u);
        c.vec = 1u << (rep & 3u);
        return c;
    };
    if (COMPACT) {
        const int l = threadIdx.x & (L - 1), g = threadIdx.x / L;
        const int lead = (threadIdx.x & 31) & ~(L - 1);  // the group's lane 0 within the warp
        double* myf = fs + g * kBuildFS;
        const int64_t step = int64_t(gridDim.x) * (kBuildT / L);
        const int64_t iters = (rows + step - 1) / step;  // warp-uniform trip count (shuffles below)
        for (int64_t it = 0; it < iters; ++it) {
            const int64_t r = it * step + int64_t(blockIdx.x) * (kBuildT / L) + g;
            const bool valid = r < rows;
            if (valid) {  // every lane computes the features, lane l stores those with j % L == l
                double f[16];
                plan_features(P, H, row_knobs(r), f);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if ((j & (L - 1)) == l) myf[j] = f[j];
            }
            __syncwarp();
            double sum = 0.0;
            for (int tb = 0; tb < ntrees; tb += L) {
                const int t = tb + l;
                double v = 0.0;
                if (valid && t < ntrees) {
                    CNode nd = sn[sroots[t]];
                    while (nd.feature >= 0) {
                        const double x = myf[nd.feature];
                        nd = sn[x < nd.tv ? (nd.lr & 0xffffu) : (nd.lr >> 16)];
                    }
                    v = nd.tv;
                }
#pragma unroll
                for (int q = 0; q < L; ++q) {  // trees tb .. tb + L - 1, in order
                    const double w = __shfl_sync(0xffffffffu, v, lead + q);
                    if (tb + q < ntrees) sum = __dadd_rn(sum, w);
                }
            }
            __syncwarp();  // the next row's features overwrite myf
            if (valid && l == 0) {
                const double s = __dadd_rn(base, __dmul_rn(lr, sum));
                const double p = (1e-6 < s) ? s : 1e-6;
                rowpred[r] = p;
                const uint64_t o = order_key(p);
                lo = o < lo ? o : lo;
                hi = o > hi ? o : hi;
            }
        }
    } else {
        for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows;
             r += int64_t(gridDim.x) * blockDim.x) {
            double f[16];
            plan_features(P, H, row_knobs(r), f);
            const double p = walk_forest(QH, groots, gnodes, f);
            rowpred[r] = p;
            const uint64_t o = order_key(p);
            lo = o < lo ? o : lo;
            hi = o > hi ? o : hi;
        }
    }
    for (int s = 16; s > 0; s >>= 1) {
        const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, s), b = __shfl_xor_sync(0xffffffffu, hi, s);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(reinterpret_cast<unsigned long long*>(&meta->bounds[0]), static_cast<unsigned long long>(lo));
        atomicMax(reinterpret_cast<unsigned long long*>(&meta->bounds[1]), static_cast<unsigned long long>(hi));
    }
}

// Per (key, k_tile index): candidate_id's FNV-1a state (space.cpp:22-45) after the 12 operator
// words, the key's three DimTiling records and k_tile; the score kernels hash only unroll and
// vectorize (fnv_tail).
__global__ void key_hash_kernel(const uint8_t* __restrict__ P, int64_t nkeys, uint64_t* __restrict__ out,
                                uint64_t* __restrict__ out_key) {
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    const TilingRec* T[3] = {at<TilingRec>(P, H.off_til[0]), at<TilingRec>(P, H.off_til[1]),
                             at<TilingRec>(P, H.off_til[2])};
    const int64_t* divk = at<int64_t>(P, H.off_divk);
    const uint32_t nt1 = uint32_t(H.nt[1]), nt2 = uint32_t(H.nt[2]);
    const int ndk = H.ndk;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < nkeys * ndk;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t key = q / ndk;
        const int k = int(q - key * ndk);
        const uint32_t t[3] = {uint32_t(key / (int64_t(nt1) * nt2)), uint32_t((key / nt2) % nt1),
                               uint32_t(key % nt2)};
        uint64_t h = H.fnv_prefix;
        for (int d = 0; d < 3; ++d) {
            const TilingRec r = T[d][t[d]];
            h = fnv_small(h, r.blocks);
            h = fnv_small(h, r.threads);
            h = fnv_small(h, r.pt);
        }
        out[q] = fnv_small(h, uint32_t(divk[k]));
        if (k == 0) out_key[key] = h;  // the state before k_tile, per key
    }
}

// ------------------------------------------------------------------- scoring
constexpr int kRowsT = 512;
constexpr int kRowsPer = 4;  // candidates per thread per pass (independent gathers in flight)

__global__ void __launch_bounds__(kRowsT) score_rows_kernel(const uint8_t* __restrict__ gplan,
                                                            const uint16_t* __restrict__ clskuv,
                                                            const RowTabMeta* __restrict__ meta,
                                                            const double* __restrict__ rowpred,
                                                            const uint64_t* __restrict__ khk,
                                                            const uint64_t* __restrict__ genome, int64_t n,
                                                            double* __restrict__ pred, uint64_t* __restrict__ ids,
                                                            const SelHist sel_in, int nodedup) {
    extern __shared__ uint32_t rsm[];  // Kuv class table [ndk][16][4] (u16 pairs), then k_tile low words [ndk]
    __shared__ uint32_t shist[kSelBins];
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(gplan);
    const int ndk = H.ndk;
    const uint32_t nt1 = uint32_t(H.nt[1]), nt2 = uint32_t(H.nt[2]);
    const int64_t* divk = at<int64_t>(gplan, H.off_divk);
    uint32_t* sdivk = rsm + ndk * 32;
    if (sel_in.hist)
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) shist[i] = 0u;
    for (int i = threadIdx.x; i < ndk; i += blockDim.x) sdivk[i] = uint32_t(divk[i]);
    pdl_wait();  // the class table, row table and bounds may come from the kernels just before
    const SelHist sel = sel_resolve(sel_in);
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(clskuv);
        for (int i = threadIdx.x; i < ndk * 32; i += blockDim.x) rsm[i] = __ldg(src + i);
    }
    const uint32_t nkc = uint32_t(meta->nkc);
    __syncthreads();
    const uint16_t* scls = reinterpret_cast<const uint16_t*>(rsm);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; base < n; base += kRowsPer * stride) {
        uint64_t g[kRowsPer];
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j) {
            const int64_t i = base + j * stride;
            g[j] = i < n ? __ldcs(genome + i) : 0ull;
        }
        uint32_t key[kRowsPer];
        double p[kRowsPer];
        uint64_t h[kRowsPer];
        // a thread's candidates are `stride` apart and share their base parent when P divides it: an
        // equal genome earlier in the pass gathers for it (3 bits per j: the source candidate or j)
        uint32_t dsrc = 0u;
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j) {
            const Genome x = genome_unpack(g[j]);
            key[j] = (x.t0 * nt1 + x.t1) * nt2 + x.t2;
            const uint32_t kc = min(uint32_t(scls[(x.k * 16u + x.u) * 4u + x.v]), nkc - 1u);  // in bounds for any genome
            uint32_t src = uint32_t(j);
#pragma unroll
            for (int q = j - 1; q >= 0; --q)
                if (!nodedup && g[q] == g[j]) src = uint32_t(q);
            dsrc |= src << (3 * j);
            const bool own = src == uint32_t(j) && base + j * stride < n;
            p[j] = own ? __ldg(rowpred + (size_t(key[j]) * nkc + kc)) : 0.0;
            h[j] = (ids && own) ? __ldg(khk + (size_t(key[j]) * ndk + x.k)) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j) {
            const int64_t i = base + j * stride;
            if (i >= n) break;
            const uint32_t src = (dsrc >> (3 * j)) & 7u;
#pragma unroll
            for (int q = 0; q < j; ++q)
                if (src == uint32_t(q)) {
                    p[j] = p[q];
                    h[j] = h[q];
                }
            pred[i] = p[j];  // plain store: stays in L2 for the selection filter that re-reads it
            if (sel.hist) atomicAdd(&shist[sel_bin(p[j], sel)], 1u);
            if (ids) {
                const Genome x = genome_unpack(g[j]);
                __stcs(reinterpret_cast<unsigned long long*>(ids) + i,
                       static_cast<unsigned long long>(fnv_tail(h[j], x.u, x.v)));
            }
        }
    }
    if (sel.hist) {
        __syncthreads();
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) {
            const uint32_t v = shist[i];
            if (v) atomicAdd(sel.hist + i, v);
        }
    }
}

// ------------------------------------------------------- rows in prediction order
// The fused selection walks the rows in prediction order, so the compile sorts them: a stable
// LSD radix sort (four 8-bit passes) on the top 32 bits of each row's order key relative to the
// lowest, then an exact fix-up of the (rare) runs whose truncated keys collide, by (full key,
// row).  Everything is sized on the device (meta->rows): no host synchronisation.
constexpr int kRsT = 512;
constexpr int kRsTile = 4096;  // items per tile

__device__ __forceinline__ int rs_shift32(const RowTabMeta* meta) {
    const uint64_t kmin = meta->bounds[0], kmax = meta->bounds[1];
    const uint64_t span = kmax > kmin ? kmax - kmin : 0ull;
    const int bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
    return bits > 32 ? bits - 32 : 0;
}

__global__ void rowtab_keys_kernel(const RowTabMeta* __restrict__ meta, const double* __restrict__ rowpred,
                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    pdl_wait();
    const int64_t R = meta->rows;
    const uint64_t kmin = meta->bounds[0];
    const int sh = rs_shift32(meta);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < R; r += int64_t(gridDim.x) * blockDim.x) {
        keys[r] = uint32_t((order_key(rowpred[r]) - kmin) >> sh);
        vals[r] = uint32_t(r);
    }
}

__device__ __forceinline__ void rs_agg_inc(uint32_t* bin, unsigned d, bool valid) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const unsigned peers = __match_any_sync(act, d);
    if ((__ffs(peers) - 1) == int(threadIdx.x & 31)) atomicAdd(&bin[d], unsigned(__popc(peers)));
}

// per tile: digit counts -> cnt[d * ntiles + t]
__global__ void __launch_bounds__(kRsT) rs_hist_kernel(const RowTabMeta* __restrict__ meta,
                                                      const uint32_t* __restrict__ keys, int shift, int ntiles,
                                                      uint32_t* __restrict__ cnt) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    pdl_wait();
    const int64_t R = meta->rows;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kRsTile;
    for (int r = 0; r < kRsTile / kRsT; ++r) {
        const int64_t i = base + r * kRsT + threadIdx.x;
        const bool v = i < R;
        rs_agg_inc(h, v ? (keys[i] >> shift) & 0xffu : 0u, v);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) cnt[int64_t(d) * ntiles + blockIdx.x] = h[d];
}

// one CTA per digit: exclusive scan of its tile counts in place, digit total -> tot[d]
__global__ void __launch_bounds__(256) rs_scan_kernel(uint32_t* __restrict__ cnt, int ntiles,
                                                     uint32_t* __restrict__ tot) {
    __shared__ uint32_t ws[8];
    __shared__ uint32_t carry;
    pdl_wait();
    const int d = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    uint32_t* row = cnt + int64_t(d) * ntiles;
    for (int b = 0; b < ntiles; b += 256) {
        const int i = b + tid;
        const uint32_t v = i < ntiles ? row[i] : 0u;
        uint32_t x = v;
        for (int s = 1; s < 32; s <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
            if (lane >= s) x += y;
        }
        if (lane == 31) ws[wid] = x;
        __syncthreads();
        uint32_t before = carry, all = carry;
        for (int w = 0; w < 8; ++w) {
            before += w < wid ? ws[w] : 0u;
            all += ws[w];
        }
        if (i < ntiles) row[i] = before + x - v;
        __syncthreads();
        if (tid == 0) carry = all;
        __syncthreads();
    }
    if (tid == 0) tot[d] = carry;
}

// stable scatter of one tile: digit base (scan of the 256 totals) + tile prefix + rank in tile
__global__ void __launch_bounds__(kRsT) rs_scatter_kernel(const RowTabMeta* __restrict__ meta,
                                                         const uint32_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin, int shift,
                                                         const uint32_t* __restrict__ cnt,
                                                         const uint32_t* __restrict__ tot, int ntiles,
                                                         uint32_t* __restrict__ kout, uint32_t* __restrict__ vout) {
    constexpr int W = kRsT / 32;
    __shared__ uint32_t base[256];
    __shared__ uint32_t gofs[256];
    __shared__ uint32_t wc[W][257];
    pdl_wait();
    const int64_t R = meta->rows;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 256) {  // exclusive scan of the digit totals (8 warps x 32)
        const uint32_t v = tot[tid];
        uint32_t x = v;
        for (int s = 1; s < 32; s <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
            if (lane >= s) x += y;
        }
        wc[0][tid] = x;  // inclusive within the warp; combined below
        base[tid] = 0;
    }
    __syncthreads();
    if (tid < 256) {
        uint32_t before = 0;
        for (int w = 0; w < (tid >> 5); ++w) before += wc[0][w * 32 + 31];
        gofs[tid] = before + wc[0][tid] - tot[tid] + cnt[int64_t(tid) * ntiles + blockIdx.x];
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    const int64_t tbase = int64_t(blockIdx.x) * kRsTile;
    for (int r = 0; r < kRsTile / kRsT; ++r) {
        for (int j = tid; j < W * 257; j += blockDim.x) (&wc[0][0])[j] = 0;
        __syncthreads();
        const int64_t i = tbase + r * kRsT + tid;
        const bool valid = i < R;
        uint32_t key = 0, val = 0;
        unsigned d = 256;
        if (valid) {
            key = kin[i];
            val = vin[i];
            d = (key >> shift) & 0xffu;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned wrank = __popc(peers & lt);
        if (valid && (__ffs(peers) - 1) == lane) wc[warp][d] = __popc(peers);
        __syncthreads();
        if (tid < 256) {
            uint32_t run = base[tid];
            for (int w = 0; w < W; ++w) {
                const uint32_t c = wc[w][tid];
                wc[w][tid] = run;
                run += c;
            }
            base[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = gofs[d] + wc[warp][d] + wrank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}

// After the radix sort on truncated keys, rows whose truncated keys collide but whose full keys
// are out of order are rare.  rowtab_inv_kernel (one thread per position) marks the start of
// every run of equal truncated keys that holds such an inversion; rowtab_runsort_kernel sorts
// only the marked runs by (full key, row) -- one thread per run, insertion sort.
__device__ __forceinline__ bool rs_after(const double* rowpred, uint32_t q, uint32_t r) {
    const uint64_t kq = order_key(rowpred[q]), kr = order_key(rowpred[r]);
    return kq > kr || (kq == kr && q > r);
}

__global__ void rowtab_inv_kernel(const RowTabMeta* __restrict__ meta, const double* __restrict__ rowpred,
                                  const uint32_t* __restrict__ k32, const uint32_t* __restrict__ srows,
                                  uint32_t* __restrict__ mark) {
    pdl_wait();
    const int64_t R = meta->rows;
    for (int64_t p = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < R; p += int64_t(gridDim.x) * blockDim.x) {
        if (k32[p - 1] != k32[p] || !rs_after(rowpred, srows[p - 1], srows[p])) continue;
        int64_t st = p - 1;
        while (st > 0 && k32[st - 1] == k32[p]) --st;
        atomicOr(mark + (st >> 5), 1u << (st & 31));
    }
}

__global__ void rowtab_runsort_kernel(const RowTabMeta* __restrict__ meta, const double* __restrict__ rowpred,
                                      const uint32_t* __restrict__ k32, uint32_t* __restrict__ srows,
                                      uint32_t* __restrict__ mark) {
    pdl_wait();
    const int64_t R = meta->rows;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < R; p += int64_t(gridDim.x) * blockDim.x) {
        if (!((mark[p >> 5] >> (p & 31)) & 1u)) continue;
        int64_t e = p + 1;
        while (e < R && k32[e] == k32[p]) ++e;
        for (int64_t i = p + 1; i < e; ++i) {
            const uint32_t r = srows[i];
            int64_t j = i - 1;
            while (j >= p && rs_after(rowpred, srows[j], r)) {
                srows[j + 1] = srows[j];
                --j;
            }
            srows[j + 1] = r;
        }
    }
}

// Dense rank ("group") of every row in prediction order: position p starts a new group when its
// full key differs from position p-1's.  Per tile of kRsTile positions: the group starts counted
// (rowtab_gcount_kernel), one CTA scans the tile counts (rowtab_gscan_kernel), then each tile
// assigns gid = groups started before it + its inclusive block scan - 1 and scatters
// rowgid[row] = gid (rowtab_gapply_kernel); meta->groups = the number of distinct predictions.
__device__ __forceinline__ uint32_t rs_newgroup(const double* rowpred, const uint32_t* srows, int64_t p) {
    return p == 0 || order_key(rowpred[srows[p - 1]]) != order_key(rowpred[srows[p]]) ? 1u : 0u;
}

__global__ void __launch_bounds__(kRsT) rowtab_gcount_kernel(const RowTabMeta* __restrict__ meta,
                                                            const double* __restrict__ rowpred,
                                                            const uint32_t* __restrict__ srows,
                                                            uint32_t* __restrict__ tcnt) {
    __shared__ uint32_t red[kRsT / 32];
    pdl_wait();
    const int64_t R = meta->rows;
    uint32_t c = 0;
    for (int r = 0; r < kRsTile / kRsT; ++r) {
        const int64_t p = int64_t(blockIdx.x) * kRsTile + r * kRsT + threadIdx.x;
        if (p < R) c += rs_newgroup(rowpred, srows, p);
    }
    for (int sft = 16; sft > 0; sft >>= 1) c += __shfl_xor_sync(0xffffffffu, c, sft);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kRsT / 32; ++w) t += red[w];
        tcnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) rowtab_gscan_kernel(RowTabMeta* __restrict__ meta, uint32_t* __restrict__ tcnt,
                                                           int ntiles) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    pdl_wait();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int b = 0; b < ntiles; b += 1024) {
        const int i = b + tid;
        const uint32_t v = i < ntiles ? tcnt[i] : 0u;
        uint32_t x = v;
        for (int sft = 1; sft < 32; sft <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, sft);
            if (lane >= sft) x += y;
        }
        if (lane == 31) ws[wid] = x;
        __syncthreads();
        uint32_t before = carry, all = carry;
        for (int w = 0; w < 32; ++w) {
            before += w < wid ? ws[w] : 0u;
            all += ws[w];
        }
        if (i < ntiles) tcnt[i] = before + x - v;  // exclusive
        __syncthreads();
        if (tid == 0) carry = all;
        __syncthreads();
    }
    if (tid == 0) meta->groups = int64_t(carry);
}

__global__ void __launch_bounds__(kRsT) rowtab_gapply_kernel(const RowTabMeta* __restrict__ meta,
                                                            const double* __restrict__ rowpred,
                                                            const uint32_t* __restrict__ srows,
                                                            const uint32_t* __restrict__ tcnt,
                                                            uint32_t* __restrict__ rowgid) {
    __shared__ uint32_t ws[kRsT / 32];
    __shared__ uint32_t carry;
    pdl_wait();
    const int64_t R = meta->rows;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = tcnt[blockIdx.x];
    __syncthreads();
    for (int r = 0; r < kRsTile / kRsT; ++r) {
        const int64_t p = int64_t(blockIdx.x) * kRsTile + r * kRsT + tid;
        const uint32_t v = p < R ? rs_newgroup(rowpred, srows, p) : 0u;
        uint32_t x = v;
        for (int sft = 1; sft < 32; sft <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, sft);
            if (lane >= sft) x += y;
        }
        if (lane == 31) ws[wid] = x;
        __syncthreads();
        uint32_t before = carry, all = carry;
        for (int w = 0; w < kRsT / 32; ++w) {
            before += w < wid ? ws[w] : 0u;
            all += ws[w];
        }
        if (p < R) rowgid[srows[p]] = before + x - 1u;  // inclusive count of group starts - 1
        __syncthreads();
        if (tid == 0) carry = all;
        __syncthreads();
    }
}

// The fused selection's one gather per candidate: {prediction, group} in a 16-byte row record.
__global__ void rowtab_pack_kernel(const RowTabMeta* __restrict__ meta, const double* __restrict__ rowpred,
                                   const uint32_t* __restrict__ rowgid, RowRec* __restrict__ rec) {
    pdl_wait();
    const int64_t R = meta->rows;
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < R; r += int64_t(gridDim.x) * blockDim.x) {
        RowRec x;
        x.pred = rowpred[r];
        x.gid = rowgid[r];
        x.pad = 0;
        rec[r] = x;
    }
}

// ------------------------------------------------ fused score + keep-the-best
// One cooperative grid.  A candidate's prediction is its row's, and its place in prediction order
// is its row's group g (the dense rank of the row's prediction: equal predictions, equal g), so
// the k best by (prediction, index) are the k smallest (g, index).  CTA b owns the contiguous
// candidates [b*per*T, (b+1)*per*T); thread t of it candidates base + j*T + t, j < per, so index
// order inside a CTA is (j, t) order.  Every candidate's g stays in shared memory across the
// grid barriers (nothing is re-read from HBM, and no per-candidate global atomic: copies of one
// parent share a row and would serialise in L2).
//   A   score: the thread's genomes are loaded first (coalesced, all in flight) and kept in shared
//       memory; genome -> row -> {prediction, g} (one 16-byte gather, all of a thread's gathers in
//       flight together) -> prediction out; a shared-memory histogram of g by segment (G / 4096
//       groups each) flushed with one atomic per non-empty segment (a warp's atomics on one line).
//   ids The candidate ids (per-key FNV state staged in shared memory by one bulk copy, then the
//       k_tile / unroll / vectorize bytes) are outputs only: they are computed between the arrive
//       and the wait of the split grid barriers, filling their release latency (j < 4 at barrier
//       1, j >= 4 at barrier 2).
//   B   (every CTA, after barrier 1) the segment b0 of the k-th candidate: one 16-byte load of the
//       counts per thread and a block scan.
//   C   (segments of <= 64 groups: G <= 2^18) the candidates below b0 (fewer than k) are appended
//       to a list; the CTA's candidates in b0 are compacted in index order and given their order
//       among the CTA's candidates of the same group (a stable multi-split); the CTA publishes
//       its count per group of b0 and adds it to the per-group totals.
//   D   (after barrier 2) a candidate of b0 in group offset q goes to position
//         before(b0) + (b0's candidates in groups < q) + (group q's candidates in CTAs before b)
//         + (its order in the CTA),
//       written when < k -- ties, thousands of copies of one parent in a bred population, are
//       placed by index without a sort; the list below b0 is ranked by counting.
//   Segments of more groups (G > 2^18): B2 radix-selects the k-th group g* (one barrier per 12
//   bits), C2 appends the candidates below g* and counts each CTA's ties at g*, D2 places the
//   ties by CTA prefix and ranks the list.
constexpr int kSRT = 1024;  // one CTA per SM: half the CTAs to synchronise and to stage tables
constexpr int kSRPer = 8;
constexpr int kSRMaxCtas = 1024;
constexpr int kSRMaxSeg = 4096;    // segment histogram bins (shared memory)
constexpr int kSRKeys = 64;        // groups per segment the exact crossing path (C/D) handles
constexpr int kSRIdsA = 0, kSRIdsB = 4, kSRIdsC = 8;  // ids: j < A in phase A, [A, B) at barrier 1, [B, C) at
                                                      // barrier 2, the rest in phase D's round trip
constexpr int kSRListCap = 8192;   // appended records (radix path: < k; crossing path: < k)
static_assert(kSRListCap >= kSelMaxK, "the tie path appends at most k records");
// dynamic shared memory: [R0: genome staging, later the ranked list + the CTA's crossing-segment
// candidates (64 KB) | g per candidate (u32, per*T) | segment histogram | Kuv classes | k_tile
// words | per-key FNV states when <= 64 KB]
constexpr uint32_t kSRR0 = 64 * 1024;

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// diagnostic (ETUNE_ROWSEL_TRACE): per-CTA globaltimer stamps, kSRTraceSlots slots per CTA
constexpr int kSRTraceSlots = 18;  // slot 15 holds the crossing segment's count, slot 16 the SM id: not times
#define SR_TRACE(slot) \
    do { \
        if (trace && threadIdx.x == 0) trace[blockIdx.x * kSRTraceSlots + (slot)] = globaltimer(); \
    } while (0)

constexpr int kSRLevels = 3;  // radix-select levels over the group index (<= 2^25 groups)
constexpr int kSRRep = 8;  // replicas of the appended list: the ranking CTAs read different L2 lines
struct RowSelWork {
    uint32_t nlist, pad[3];
    uint32_t gbar[2], gpad[2];           // split grid barriers 1 and 2: arrivals of this call
    uint32_t tot[kSRKeys][32];           // crossing segment: candidates per group offset (a line each)
    uint32_t tiecnt[kSRMaxCtas];
    uint32_t kcnt[kSRKeys][kSRMaxCtas];  // crossing segment: candidates per (group offset, CTA)
    uint32_t lvl[kSRLevels][kSRMaxSeg];  // candidates per bin of each radix-select level
    uint64_t lkey[kSRRep][kSRListCap];   // g << 32 | index of the appended records, kSRRep copies
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
        if (lane >= s) x += y;
    }
    return x;
}

// exclusive block scan of one u32 per thread (blockDim = kSRT); *total = block sum.  ws holds
// 33 words: the warp sums, scanned by warp 0 (no per-thread loop over the warps)
__device__ __forceinline__ uint32_t sr_block_scan(uint32_t v, uint32_t* ws, uint32_t* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t x = warp_incl_scan(v);
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = ws[lane], inc = warp_incl_scan(w);
        ws[lane] = inc - w;
        if (lane == 31) ws[32] = inc;
    }
    __syncthreads();
    const uint32_t before = ws[wid];
    *total = ws[32];
    __syncthreads();  // ws is reused by the next scan
    return before + x - v;
}

// exclusive block scan of five u32 lanes per thread (componentwise: a uint4 and a u32); ws5
// holds 5 x 33 words
__device__ __forceinline__ uint4 sr_block_scan5(uint4 v, uint32_t v5, uint32_t* ws5, uint4* total, uint32_t* ex5,
                                                uint32_t* total5) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t x0 = warp_incl_scan(v.x), x1 = warp_incl_scan(v.y), x2 = warp_incl_scan(v.z),
                   x3 = warp_incl_scan(v.w), x4 = warp_incl_scan(v5);
    if (lane == 31) {
        ws5[0 * 33 + wid] = x0;
        ws5[1 * 33 + wid] = x1;
        ws5[2 * 33 + wid] = x2;
        ws5[3 * 33 + wid] = x3;
        ws5[4 * 33 + wid] = x4;
    }
    __syncthreads();
    if (wid < 5) {  // warp c scans component c
        const uint32_t w = ws5[wid * 33 + lane], inc = warp_incl_scan(w);
        ws5[wid * 33 + lane] = inc - w;
        if (lane == 31) ws5[wid * 33 + 32] = inc;
    }
    __syncthreads();
    const uint4 r = make_uint4(ws5[0 * 33 + wid] + x0 - v.x, ws5[1 * 33 + wid] + x1 - v.y, ws5[2 * 33 + wid] + x2 - v.z,
                               ws5[3 * 33 + wid] + x3 - v.w);
    *ex5 = ws5[4 * 33 + wid] + x4 - v5;
    *total = make_uint4(ws5[0 * 33 + 32], ws5[1 * 33 + 32], ws5[2 * 33 + 32], ws5[3 * 33 + 32]);
    *total5 = ws5[4 * 33 + 32];
    __syncthreads();
    return r;
}

// smem histogram hs[0..nb) -> global g[0..nb), one atomic per non-empty bin
__device__ __forceinline__ void sr_flush(const uint32_t* hs, uint32_t* g, int nb) {
    for (int i = threadIdx.x; i < nb; i += kSRT) {
        const uint32_t v = hs[i];
        if (v) atomicAdd(g + i, v);
    }
}

// the bin holding the kk-th item (1-based) among nb <= kSRMaxSeg counters (one 16-byte load per
// thread; bins past nb read as zero: the work area keeps all kSRMaxSeg counters zero between
// calls): its index, the count before it and in it, identical in every thread
__device__ __forceinline__ void sr_cross(const uint32_t* g, uint32_t kk, uint32_t* ws, uint32_t* s_bin,
                                         uint32_t* s_before, uint32_t* s_cnt) {
    static_assert(kSRMaxSeg == 4 * kSRT, "one uint4 of counters per thread");
    const uint4 q = __ldcg(reinterpret_cast<const uint4*>(g) + threadIdx.x);
    const uint32_t c[4] = {q.x, q.y, q.z, q.w};
    uint32_t tot;
    uint32_t run = sr_block_scan(q.x + q.y + q.z + q.w, ws, &tot);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (c[i] && run < kk && run + c[i] >= kk) {
            *s_bin = uint32_t(threadIdx.x) * 4u + uint32_t(i);
            *s_before = run;
            *s_cnt = c[i];
        }
        run += c[i];
    }
    __syncthreads();
}

// one-dimensional bulk copy global -> shared (TMA, cp.async.bulk) completing on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// The m appended records (<= kSRListCap) get their output positions by counting: rank = records
// with a smaller (g, index).  CTA c ranks records [32c, 32c + 32): lane l of every warp owns
// record 32c + l, warp w compares it with the w-th 32nd of the list (broadcast shared loads,
// staged by one bulk copy), the partial counts are summed; rank < k goes to out[rank].
__device__ __forceinline__ void sr_rank_out(const RowSelWork* W, uint32_t m, uint32_t k, unsigned long long* xk,
                                            int64_t* out, uint64_t* mbar, uint32_t phase, uint32_t* part,
                                            unsigned long long* trace) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kW = kSRT / 32;
    if (blockIdx.x * 32u >= m) return;  // block-uniform: this CTA owns no record
    if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the list was written by generic stores
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the staging area was read generically
        bulk_g2s(xk, W->lkey[blockIdx.x % kSRRep], (m * 8u + 15u) & ~15u, mbar);
    }
    mbar_wait(mbar, phase);
    SR_TRACE(8);
    const uint32_t per = (m + kW - 1) / kW, j0 = warp * per, j1 = min(m, j0 + per);
    for (uint32_t r0 = blockIdx.x * 32u; r0 < m; r0 += gridDim.x * 32u) {
        const uint32_t r = r0 + lane;
        const unsigned long long mine = r < m ? xk[r] : ~0ull;
        uint32_t cnt = 0;
#pragma unroll 8
        for (uint32_t j = j0; j < j1; ++j) cnt += xk[j] < mine ? 1u : 0u;
        part[warp * 32 + lane] = cnt;
        __syncthreads();
        SR_TRACE(9);
        if (warp == 0) {
            uint32_t c = 0;
#pragma unroll
            for (int w = 0; w < kW; ++w) c += part[w * 32 + lane];
            if (r < m && c < k) out[c] = int64_t(uint32_t(mine));
        }
        __syncthreads();
    }
}

// CTA-aggregated append of each thread's records (one global atomic per CTA): take(j) / key(j)
template <typename Take, typename Key>
__device__ __forceinline__ void sr_append_block(RowSelWork* W, uint32_t* ws, uint32_t* s_base, int per, Take take,
                                                Key key) {
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kSRPer; ++j) cnt += (j < per && take(j)) ? 1u : 0u;
    uint32_t tot;
    uint32_t off = sr_block_scan(cnt, ws, &tot);
    if (threadIdx.x == 0) *s_base = tot ? atomicAdd(&W->nlist, tot) : 0u;
    __syncthreads();
    off += *s_base;
#pragma unroll
    for (int j = 0; j < kSRPer; ++j)
        if (j < per && take(j)) {
            if (off < uint32_t(kSRListCap)) {
                const uint64_t kv = key(j);
#pragma unroll
                for (int r = 0; r < kSRRep; ++r) W->lkey[r][off] = kv;
            }
            ++off;
        }
}

// Split grid barrier (the grid is co-resident: cooperative launch) on a per-barrier arrival
// counter.  arrive: the CTA's writes are ordered before its arrival (bar.sync, then a cumulative
// fence by the arriving thread); wait: spin with acquire loads until every CTA arrived.  Work
// placed between the two fills the barrier's release latency -- here, the candidate ids.  The
// counters return to zero between calls: barrier 2's in phase A of the next call (its arrivals
// come after barrier 1), barrier 1's by CTA 0 once barrier 2 (or the radix path's first
// barrier) has passed -- every CTA is past barrier 1 by then.
__device__ __forceinline__ void gbar_arrive(uint32_t* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
    }
}
__device__ __forceinline__ void gbar_wait(const uint32_t* bar) {
    if (threadIdx.x == 0) {
        uint32_t v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v >= gridDim.x) break;
            __nanosleep(32);
        }
    }
    __syncthreads();
}

// row-record gather with a selectable cache policy (diagnostic ETUNE_ROWSEL_GMODE, low 4 bits): 0
// ld.global.nc (L1 allocating), 1 ld.global.cg (L2 only; the default), 2 .nc.L1::no_allocate,
// 3 .nc.L1::evict_first; + 16: no in-thread row dedup (every candidate gathers its record).
// The table (1.5 MB for C2) does not fit L1 and ~7 K gathers per SM are in flight at once: bypassing L1
// measured 1.5 us per step faster than the L1-allocating load (profiles/r02z_gather_policy.txt).
__device__ __forceinline__ double2 ld_row(const RowRec* p, int mode) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 r;
    if (mode == 1) return __ldcg(q);
    if (mode == 2) {
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(q));
        return r;
    }
    if (mode == 3) {
        asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(q));
        return r;
    }
    return __ldg(q);
}

struct SRStatic {
    uint32_t ws[5 * 33];
    uint32_t part[kSRT];
    uint32_t wcount[kSRT / 32][kSRKeys + 1];  // multi-split: per (warp, group offset) counts (+1: no bank conflicts)
    uint32_t run[kSRKeys];                // the CTA's candidates per group offset of b0
    uint32_t ktot[kSRKeys];               // b0's candidates in group offsets < q (all CTAs)
    uint32_t kpre[kSRKeys];               // group offset q's candidates in the CTAs before this one
    uint32_t jw[kSRPer * 32];             // b0's candidates per (j, warp), then their offsets
    uint32_t lw[32];                      // candidates below b0 per warp, then their offsets
    uint32_t bin, before, cnt, base, mc;
    uint32_t fb, fl;                      // phase C fast path: b0 / below-b0 candidates of the CTA
    __align__(8) uint64_t mbar[kSRPer + 2];
};

// host-known plan scalars of the step kernel (kernel arguments: no dependent header loads)
struct SRPlan {
    uint32_t nt1, nt2, nkeys;
    int ndk;
    uint32_t off_divk;
    int khash_smem;
};

__global__ void __launch_bounds__(kSRT, 1) score_select_rows_kernel(
    const uint8_t* __restrict__ gplan, SRPlan PL, const uint16_t* __restrict__ clskuv,
    const RowTabMeta* __restrict__ meta, const RowRec* __restrict__ rowrec, const uint64_t* __restrict__ khash,
    const uint64_t* __restrict__ genome, int64_t n, int64_t k, int per, double* __restrict__ pred,
    uint64_t* __restrict__ ids, int64_t* __restrict__ out, RowSelWork* __restrict__ W,
    unsigned long long* __restrict__ trace, int only_a, int force_radix, int ids_a, int ids_b, int ids_c, int gmode) {
    namespace cg = cooperative_groups;
    SR_TRACE(0);
    extern __shared__ int4 dsm4[];
    uint8_t* dsm = reinterpret_cast<uint8_t*>(dsm4);
    __shared__ SRStatic S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t base = uint32_t(blockIdx.x) * uint32_t(per) * kSRT;  // n < 2^31
    // ---- A0: the thread's genomes first (coalesced, all in flight), then the tables
    uint64_t x0[kSRPer];
#pragma unroll
    for (int j = 0; j < kSRPer; ++j) {
        const uint32_t i = base + uint32_t(j) * kSRT + tid;
        x0[j] = (j < per && i < uint32_t(n)) ? __ldcs(genome + i) : ~0ull;
    }
    const int ndk = PL.ndk;
    const uint32_t nt1 = PL.nt1, nt2 = PL.nt2;
    uint64_t* sgen = reinterpret_cast<uint64_t*>(dsm);                    // R0
    uint32_t* sgg = reinterpret_cast<uint32_t*>(dsm + kSRR0);             // per * T
    uint32_t* hist = sgg + per * kSRT;                                    // kSRMaxSeg
    uint32_t* scls32 = hist + kSRMaxSeg;                                  // ndk * 32
    uint32_t* sdivk = scls32 + ndk * 32;                                  // ndk (rounded to 4)
    uint64_t* skh = reinterpret_cast<uint64_t*>(sdivk + ((ndk + 3) & ~3));  // 16-byte aligned
    const bool bulk = PL.khash_smem && ids;
    if (tid == 0) {  // per-key FNV states: one bulk copy (mbar kSRPer), needed only for the ids
        for (int j = 0; j < kSRPer + 2; ++j) mbar_init(&S.mbar[j]);
        mbar_fence_init();
        if (bulk) bulk_g2s(skh, khash, (PL.nkeys * 8u + 15u) & ~15u, &S.mbar[kSRPer]);
    }
    const RowTabMeta M = *meta;
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(clskuv);
        for (int i = tid; i < ndk * 32; i += kSRT) scls32[i] = __ldg(src + i);
        const int64_t* divk = at<int64_t>(gplan, PL.off_divk);
        for (int i = tid; i < ndk; i += kSRT) sdivk[i] = uint32_t(__ldg(divk + i));
        reinterpret_cast<uint4*>(hist)[tid] = make_uint4(0, 0, 0, 0);
        if (tid < kSRPer * 32) S.jw[tid] = 0u;  // phase C: only warps holding candidates at or below b0 write
        if (tid < 32) S.lw[tid] = 0u;
        if (tid == 0) S.fb = S.fl = 0u;
    }
    const uint32_t groups = uint32_t(M.groups);
    const int gbits = groups > 1 ? 32 - __clz(int(groups - 1)) : 0;
    const int segshift = gbits > 12 ? gbits - 12 : 0;  // level 0: <= 4096 segments of the group index
    const int nseg = int((groups + (1u << segshift) - 1) >> segshift);
    const uint32_t nkc = uint32_t(M.nkc);
    __syncthreads();
    SR_TRACE(17);
    const uint16_t* scls = reinterpret_cast<const uint16_t*>(scls32);
    // ---- A1: every gather of the thread in flight together; the genomes go to shared memory
    // A thread's candidates j share their base parent (i % P), so bred populations repeat rows inside a
    // thread (C2 bench population: 5.7 distinct genomes per 7): a candidate whose row an earlier one of
    // the thread already gathers is not gathered again; A2 copies the earlier candidate's record
    // (dsrc: 3 bits per j, the source candidate or j itself).  Absent candidates gather nothing.
    double p[kSRPer];
    uint32_t gq[kSRPer];
    uint32_t rw[kSRPer];
    uint32_t dsrc = 0u, absent = 0u;  // absent: bit j set when candidate j does not exist
    const bool dedup = !(gmode & 16);
#pragma unroll
    for (int j = 0; j < kSRPer; ++j) {
        if (j >= per) break;
        const uint64_t g = x0[j];
        sgen[j * kSRT + tid] = g;
        const bool v = g != ~0ull;
        const Genome x = genome_unpack(v ? g : 0ull);
        const uint32_t key = (x.t0 * nt1 + x.t1) * nt2 + x.t2;
        const uint32_t kc = min(uint32_t(scls[(x.k * 16u + x.u) * 4u + x.v]), nkc - 1u);
        rw[j] = v ? key * nkc + kc : 0xffffffffu;
        absent |= v ? 0u : 1u << j;
        uint32_t src = uint32_t(j);
#pragma unroll
        for (int q = j - 1; q >= 0; --q)
            if (dedup && rw[q] == rw[j]) src = uint32_t(q);  // the earliest match
        dsrc |= src << (3 * j);
        // the gather's predicate is known before it issues: no select on a loaded value serialises the
        // thread's gathers
        p[j] = 0.0;
        gq[j] = 0u;
        if (v && src == uint32_t(j)) {
            const double2 r = ld_row(rowrec + rw[j], gmode & 15);
            p[j] = r.x;
            gq[j] = uint32_t(__double_as_longlong(r.y));
        }
    }
    SR_TRACE(14);
    // candidate ids of the thread's candidates [j0, j1): computed inside the barriers' release
    // latency (they are outputs only; nothing in the kernel reads them)
    auto write_ids = [&](int j0, int j1) {
        if (!ids) return;
        if (bulk) mbar_wait(&S.mbar[kSRPer], 0);
        const bool full = int64_t(base) + int64_t(per) * kSRT <= n;  // block-uniform: no absent candidate
        auto one = [&](int j, const uint64_t* kh) {
            const uint64_t g = sgen[j * kSRT + tid];
            const Genome x = genome_unpack(full || g != ~0ull ? g : 0ull);  // an absent candidate reads key 0
            const uint32_t key = (x.t0 * nt1 + x.t1) * nt2 + x.t2;
            const uint64_t id = fnv_tail(fnv_ktile(kh[key], sdivk[x.k]), x.u, x.v);
            if (full || g != ~0ull)
                __stcs(reinterpret_cast<unsigned long long*>(ids) + (base + uint32_t(j) * kSRT + tid),
                       static_cast<unsigned long long>(id));
        };
        if (bulk) {
            for (int j = j0; j < j1; ++j) one(j, skh);
        } else {
            for (int j = j0; j < j1; ++j) one(j, khash);
        }
    };
    // ---- A2: outputs, histogram, g kept in shared memory; the thread's lowest g
    uint32_t gmin = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < kSRPer; ++j) {
        if (j >= per) break;
        {
            const uint32_t src = (dsrc >> (3 * j)) & 7u;  // a repeated row: the earlier candidate's record
#pragma unroll
            for (int q = 0; q < j; ++q)
                if (src == uint32_t(q)) {
                    p[j] = p[q];
                    gq[j] = gq[q];
                }
        }
        if ((absent >> j) & 1u) gq[j] = 0xffffffffu;  // no candidate
        sgg[j * kSRT + tid] = gq[j];
        gmin = min(gmin, gq[j]);
        if (gq[j] == 0xffffffffu) continue;
        const uint32_t i = base + uint32_t(j) * kSRT + tid;
        __stcs(pred + i, p[j]);
        atomicAdd(hist + (gq[j] >> segshift), 1u);
        if (j < ids_a) write_ids(j, j + 1);  // these ids overlap phase A's memory stalls
    }
    SR_TRACE(1);
    __syncthreads();
    // flush: segment i = r * T + t (a warp's atomics hit one line)
#pragma unroll
    for (int r = 0; r < kSRMaxSeg / kSRT; ++r) {
        const uint32_t v = hist[r * kSRT + tid];
        if (v) atomicAdd(W->lvl[0] + r * kSRT + tid, v);
    }
    // the per-group totals of the crossing segment are added after barrier 1 and read after
    // barrier 2: the previous call's are cleared here
    if (blockIdx.x == 0 && tid < kSRKeys) W->tot[tid][0] = 0u;
    if (blockIdx.x == 0 && tid == 0) W->gbar[1] = 0u;  // the previous call's barrier 2; this call's arrive after barrier 1
    SR_TRACE(2);
    if (only_a) {  // diagnostic: phase A alone (profilers cannot split a cooperative kernel)
        write_ids(min(per, ids_a), per);
        return;
    }
    const bool exact_path = segshift <= 6 && !force_radix;  // grid-uniform
    // ids of j < 4 inside barrier 1, of j >= 4 (R0's second half: untouched until after barrier 2)
    // inside barrier 2; the radix path writes them all at barrier 1
    static_assert(kSRR0 / 2 == 4 * kSRT * 8, "genomes of j >= 4 live in R0's second half");
    const int ja = min(per, ids_a), jsplit = exact_path ? max(ja, min(per, ids_b)) : per;
    const int jsplit2 = exact_path ? max(jsplit, min(per, ids_c)) : per;  // the rest in phase D's round trip
    gbar_arrive(&W->gbar[0]);
    write_ids(ja, jsplit);
    SR_TRACE(13);
    gbar_wait(&W->gbar[0]);
    SR_TRACE(3);
    // ---- B: the segment b0 of the k-th candidate (every CTA: one 16-byte load per thread)
    const uint32_t kk = uint32_t(k);
    sr_cross(W->lvl[0], kk, S.ws, &S.bin, &S.before, &S.cnt);
    const uint32_t b0 = S.bin, before0 = S.before;
    SR_TRACE(7);
    if (trace && tid == 0) {
        trace[blockIdx.x * kSRTraceSlots + 15] = S.cnt;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trace[blockIdx.x * kSRTraceSlots + 16] = smid;
    }
    // R0 after phase A: b0's candidates in the first half (the genomes of j < 4 there are done with
    // at barrier 1), the ranked list in the second (written after barrier 2, whose release latency
    // computes the ids of j >= 4 from the genomes still there)
    uint32_t* sb0 = reinterpret_cast<uint32_t*>(dsm);                              // R0, 32 KB
    unsigned long long* xk = reinterpret_cast<unsigned long long*>(dsm + kSRR0 / 2);  // R0, 32 KB
    auto gkey = [&](int j) { return (uint64_t(sgg[j * kSRT + tid]) << 32) | uint64_t(base + uint32_t(j) * kSRT + tid); };
    if (exact_path) {
        const uint32_t nq = 1u << segshift, qmask = nq - 1u;
        const unsigned lt = (1u << lane) - 1u;
        // ---- C: the candidates below b0 -> the list (fewer than k); b0's candidates compacted in
        //      index order (j, warp, lane).  Warp ballots per j, one warp scans the (j, warp) counts.
        // a warp none of whose candidates is at or below b0 (nearly all of them) skips C
        const bool wact = __any_sync(0xffffffffu, gmin != 0xffffffffu && (gmin >> segshift) <= b0);
        uint32_t mb = 0, ml = 0;  // per j: in b0 / below b0
        uint32_t lw = 0;
        if (wact) {
#pragma unroll
            for (int j = 0; j < kSRPer; ++j) {
                const uint32_t g = j < per ? gq[j] : 0xffffffffu;  // still in registers
                const uint32_t sg = g >> segshift;
                if (g != 0xffffffffu) {
                    if (sg < b0) ml |= 1u << j;
                    else if (sg == b0) mb |= 1u << j;
                }
            }
        }
        // fast path (the usual case: nothing below b0, at most 32 of the CTA's candidates in it):
        // unordered append to shared memory, then one warp sorts them by index, multi-splits them by
        // group and publishes the counts -- one block barrier instead of the ordered compaction's four
        if (mb) {
            const uint32_t nb = __popc(mb);
            uint32_t slot = atomicAdd(&S.fb, nb);
#pragma unroll
            for (int j = 0; j < kSRPer; ++j)
                if (((mb >> j) & 1u) && slot < 8192u) sb0[slot++] = (uint32_t(j * kSRT + tid) << 19) | (gq[j] & qmask);
        }
        if (ml) atomicAdd(&S.fl, __popc(ml));
        if (tid < kSRKeys) S.run[tid] = 0u;
        __syncthreads();
        const bool fast = S.fl == 0u && S.fb <= 64u;  // block-uniform
        uint32_t mc = S.fb;  // b0's candidates in sb0 (the ordered compaction recounts them)
        if (fast && warp == 0) {
            const uint32_t fbn = S.fb;  // lane l holds entries l and l + 32 (index in the high bits)
            uint32_t e0 = lane < int(fbn) ? sb0[lane] : 0xffffffffu;
            uint32_t e1 = lane + 32 < int(fbn) ? sb0[lane + 32] : 0xffffffffu;
            for (int kb = 2; kb <= 64; kb <<= 1)  // bitonic sort of the 64, ascending
                for (int jb = kb >> 1; jb > 0; jb >>= 1) {
                    if (jb == 32) {  // partners in the same lane (kb == 64: ascending)
                        const uint32_t lo = min(e0, e1), hi = max(e0, e1);
                        e0 = lo;
                        e1 = hi;
                    } else {
                        const uint32_t o0 = __shfl_xor_sync(0xffffffffu, e0, jb);
                        const uint32_t o1 = __shfl_xor_sync(0xffffffffu, e1, jb);
                        const bool lowside = (lane & jb) == 0;
                        const bool up0 = (lane & kb) == 0, up1 = ((lane + 32) & kb) == 0;
                        e0 = (lowside == up0) ? min(e0, o0) : max(e0, o0);
                        e1 = (lowside == up1) ? min(e1, o1) : max(e1, o1);
                    }
                }
            // stable multi-split of the sorted 64: order among the same group offset
            const bool v0 = lane < int(fbn), v1 = lane + 32 < int(fbn);
            const uint32_t q0 = v0 ? (e0 & 63u) : 64u, q1 = v1 ? (e1 & 63u) : 65u;
            const unsigned p0 = __match_any_sync(0xffffffffu, q0), l0 = p0 & lt;
            const unsigned p1 = __match_any_sync(0xffffffffu, q1), l1 = p1 & lt;
            if (v0 && l0 == 0) S.run[q0] = __popc(p0);
            __syncwarp();
            const uint32_t c0 = v1 ? S.run[q1] : 0u;  // the first half's count of e1's group
            __syncwarp();
            if (v0) sb0[lane] = e0 | (uint32_t(__popc(l0)) << 6);
            if (v1) sb0[lane + 32] = e1 | ((c0 + uint32_t(__popc(l1))) << 6);
            if (v1 && l1 == 0) S.run[q1] = c0 + __popc(p1);
            __syncwarp();
            for (int qq = lane; qq < int(nq); qq += 32) {
                const uint32_t r = S.run[qq];
                W->kcnt[qq][blockIdx.x] = r;
                if (r) atomicAdd(&W->tot[qq][0], r);
            }
        }
        if (wact && !fast) {
#pragma unroll
            for (int j = 0; j < kSRPer; ++j) {
                const unsigned bb = __ballot_sync(0xffffffffu, (mb >> j) & 1u);
                const unsigned bl = __ballot_sync(0xffffffffu, (ml >> j) & 1u);
                if (lane == 0) S.jw[j * 32 + warp] = __popc(bb);
                lw += __popc(bl);
            }
        }
        if (!fast) {  // block-uniform: the ordered compaction
        if (wact && lane == 0) S.lw[warp] = lw;
        if (tid < kSRKeys) S.run[tid] = 0u;
        __syncthreads();
        if (warp == 0) {
            uint32_t c[kSRPer], sum = 0;  // lane l: (j, warp) entries [8l, 8l + 8) in j-major order
#pragma unroll
            for (int i = 0; i < kSRPer; ++i) {
                c[i] = S.jw[kSRPer * lane + i];
                sum += c[i];
            }
            const uint32_t inc = warp_incl_scan(sum);
            uint32_t run = inc - sum;
#pragma unroll
            for (int i = 0; i < kSRPer; ++i) {
                S.jw[kSRPer * lane + i] = run;
                run += c[i];
            }
            const uint32_t l = S.lw[lane], li = warp_incl_scan(l);
            S.lw[lane] = li - l;
            const uint32_t lt_all = __shfl_sync(0xffffffffu, li, 31);
            if (lane == 31) {
                S.mc = inc;
                S.base = lt_all ? atomicAdd(&W->nlist, lt_all) : 0u;
            }
        }
        __syncthreads();
        mc = S.mc;
        uint32_t loff = S.base + S.lw[warp];
#pragma unroll
        for (int j = 0; j < kSRPer; ++j) {
            if (!wact) break;  // warp-uniform
            const unsigned bb = __ballot_sync(0xffffffffu, (mb >> j) & 1u);
            const unsigned bl = __ballot_sync(0xffffffffu, (ml >> j) & 1u);
            if ((mb >> j) & 1u)
                sb0[S.jw[j * 32 + warp] + __popc(bb & lt)] = (uint32_t(j * kSRT + tid) << 19) | (gq[j] & qmask);
            if ((ml >> j) & 1u) {
                const uint32_t off = loff + __popc(bl & lt);
                if (off < uint32_t(kSRListCap)) {
                    const uint64_t kv = gkey(j);
#pragma unroll
                    for (int r = 0; r < kSRRep; ++r) W->lkey[r][off] = kv;
                }
            }
            loff += __popc(bl);
        }
        __syncthreads();
        SR_TRACE(11);
        // stable multi-split: each b0 candidate's order among the CTA's candidates of its group
        if (mc <= 32) {  // block-uniform: one warp, records already in index order
            if (warp == 0) {
                const bool valid = lane < int(mc);
                const uint32_t e = valid ? sb0[lane] : 0u;
                const uint32_t q = valid ? (e & 63u) : 64u;
                const unsigned peers = __match_any_sync(0xffffffffu, q);
                const unsigned lower = peers & lt;
                if (valid) sb0[lane] = e | (uint32_t(__popc(lower)) << 6);
                if (valid && lower == 0) S.run[q] = __popc(peers);
            }
            __syncthreads();
        }
        for (uint32_t c0 = 0; mc > 32 && c0 < mc; c0 += kSRT) {
            for (int i = tid; i < (kSRT / 32) * (kSRKeys + 1); i += kSRT) (&S.wcount[0][0])[i] = 0u;
            __syncthreads();
            const uint32_t pidx = c0 + uint32_t(tid);
            const bool valid = pidx < mc;
            const uint32_t e = valid ? sb0[pidx] : 0u;
            const uint32_t q = valid ? (e & 63u) : 64u;
            const unsigned peers = __match_any_sync(0xffffffffu, q);
            const unsigned lower = peers & lt;
            if (valid && lower == 0) S.wcount[warp][q] = __popc(peers);
            __syncthreads();
            for (int qq = warp; qq < kSRKeys; qq += kSRT / 32) {  // warp per group offset: scan over the warps
                const uint32_t c = S.wcount[lane][qq], inc = warp_incl_scan(c), r = S.run[qq];
                S.wcount[lane][qq] = r + inc - c;
                __syncwarp();
                if (lane == 31) S.run[qq] = r + inc;
            }
            __syncthreads();
            if (valid) sb0[pidx] = e | ((S.wcount[warp][q] + __popc(lower)) << 6);  // 13-bit order
            __syncthreads();
        }
        SR_TRACE(12);
        if (tid < int(nq)) {
            const uint32_t r = S.run[tid];
            W->kcnt[tid][blockIdx.x] = r;
            if (r) atomicAdd(&W->tot[tid][0], r);
        }
        }  // ordered compaction
        SR_TRACE(4);
        gbar_arrive(&W->gbar[1]);
        write_ids(jsplit, jsplit2);
        gbar_wait(&W->gbar[1]);
        SR_TRACE(5);
        if (blockIdx.x == 0 && tid == 0) W->gbar[0] = 0u;  // every CTA is past barrier 1
        // nothing reads the list length or the level-0 counts after the barrier: reset them here
        if (blockIdx.x == 0 && tid == 0) W->nlist = 0u;
        for (int i = blockIdx.x * kSRT + tid; i < nseg; i += gridDim.x * kSRT) W->lvl[0][i] = 0u;
        // ---- D: b0's per-group totals (warp 0) and, per group the CTA holds, the CTAs before it.
        //      The loads go out first; the last candidates' ids fill their round trip.
        constexpr int kPre = 5;  // CTAs before this one per lane and group: the grid is <= 160 here
        uint32_t t0 = 0, t1 = 0, pa[kPre], pb[kPre];
        const int qa = warp, qb = warp + 32;
        const bool ha = qa < int(nq) && S.run[qa] != 0u, hb = qb < int(nq) && S.run[qb] != 0u;  // warp-uniform
        if (warp == 0) {
            t0 = lane < int(nq) ? __ldcg(&W->tot[lane][0]) : 0u;
            t1 = lane + 32 < int(nq) ? __ldcg(&W->tot[lane + 32][0]) : 0u;
        }
#pragma unroll
        for (int i = 0; i < kPre; ++i) {
            const uint32_t c = uint32_t(lane + 32 * i);
            pa[i] = (ha && c < blockIdx.x) ? __ldcg(&W->kcnt[qa][c]) : 0u;
            pb[i] = (hb && c < blockIdx.x) ? __ldcg(&W->kcnt[qb][c]) : 0u;
        }
        write_ids(jsplit2, per);
        if (warp == 0) {
            uint32_t inc = t0;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const uint32_t all0 = __shfl_sync(0xffffffffu, inc, 31);
            uint32_t inc1 = t1;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc1, o);
                if (lane >= o) inc1 += y;
            }
            S.ktot[lane] = inc - t0;
            S.ktot[lane + 32] = all0 + inc1 - t1;
        }
        if (ha || hb) {
            uint32_t sa = 0, sbb = 0;
#pragma unroll
            for (int i = 0; i < kPre; ++i) {
                sa += pa[i];
                sbb += pb[i];
            }
            for (uint32_t c = lane + 32 * kPre; c < blockIdx.x; c += 32) {  // grids beyond 160 CTAs
                if (ha) sa += __ldcg(&W->kcnt[qa][c]);
                if (hb) sbb += __ldcg(&W->kcnt[qb][c]);
            }
            for (int o = 16; o; o >>= 1) {
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
                sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
            }
            if (lane == 0) {
                if (ha) S.kpre[qa] = sa;
                if (hb) S.kpre[qb] = sbb;
            }
        }
        __syncthreads();
        for (uint32_t pidx = tid; pidx < mc; pidx += kSRT) {
            const uint32_t e = sb0[pidx];
            const uint32_t q = e & 63u, ord = (e >> 6) & 0x1fffu, loc = e >> 19;
            const uint32_t pos = before0 + S.ktot[q] + S.kpre[q] + ord;
            if (pos < kk) out[pos] = int64_t(base + loc);
        }
        if (before0) sr_rank_out(W, before0, kk, xk, out, &S.mbar[kSRPer + 1], 0, S.part, trace);
        SR_TRACE(6);
        return;
    }
    // ---- B2: radix select of the k-th candidate's group g* over the group index: at each level the
    //      bin holding the k-th candidate still in play (every CTA, identically), then -- until a bin
    //      is a single group -- the next 12 bits of g of the candidates in that bin, histogrammed per
    //      CTA and flushed (one grid barrier per level; two levels for up to 2^20 groups)
    uint32_t below = 0, kr = kk, P = 0;
    int Sc = segshift, nbc = nseg, L = 0;
    for (;; ++L) {
        if (L > 0) sr_cross(W->lvl[L], kr, S.ws, &S.bin, &S.before, &S.cnt);
        const uint32_t bin = L > 0 ? S.bin : b0;
        const uint32_t bef = L > 0 ? S.before : before0;
        below += bef;
        kr -= bef;
        P = (L == 0) ? bin : ((P << (nbc > 1 ? 31 - __clz(int(nbc)) : 0)) | bin);  // candidates with g >> Sc == P
        if (Sc == 0) break;
        const int Sn = Sc > 12 ? Sc - 12 : 0, nbn = 1 << (Sc - Sn);
        for (int i = tid; i < nbn; i += kSRT) hist[i] = 0u;
        __syncthreads();
        for (int j = 0; j < per; ++j) {
            const uint32_t g = sgg[j * kSRT + tid];
            if (g != 0xffffffffu && (g >> Sc) == P) atomicAdd(hist + ((g >> Sn) & uint32_t(nbn - 1)), 1u);
        }
        __syncthreads();
        sr_flush(hist, W->lvl[L + 1], nbn);
        cg::this_grid().sync();
        for (int i = blockIdx.x * kSRT + tid; i < nbc; i += gridDim.x * kSRT) W->lvl[L][i] = 0u;  // read by all
        Sc = Sn;
        nbc = nbn;
    }
    const uint32_t gstar = P;
    const uint32_t need = kk - below;  // >= 1 candidates at g* are taken, by index
    SR_TRACE(4);
    // ---- C2: the candidates below g* (fewer than k) are appended; each CTA counts its ties at g*
    sr_append_block(W, S.ws, &S.base, per, [&](int j) { return sgg[j * kSRT + tid] < gstar; }, gkey);
    uint32_t my_ties = 0;
    for (int j = 0; j < per; ++j) my_ties += sgg[j * kSRT + tid] == gstar;
    uint32_t cta_ties;
    sr_block_scan(my_ties, S.ws, &cta_ties);
    if (tid == 0) W->tiecnt[blockIdx.x] = cta_ties;
    cg::this_grid().sync();
    SR_TRACE(5);
    if (blockIdx.x == 0 && tid == 0) W->gbar[0] = 0u;  // every CTA is past barrier 1
    if (blockIdx.x == 0 && tid == 0) W->nlist = 0u;
    for (int i = blockIdx.x * kSRT + tid; i < nbc; i += gridDim.x * kSRT) W->lvl[L][i] = 0u;
    // ---- D2: output positions without a sort.  A tie's position is below + its rank among the ties
    //      by index: (ties of the CTAs before b) + its order in the CTA; ranks < need are written.
    //      The records below g* are ranked among themselves by counting.
    uint32_t tb = 0;
    for (uint32_t b2 = tid; b2 < blockIdx.x; b2 += kSRT) tb += __ldcg(W->tiecnt + b2);
    uint32_t tot_before;
    sr_block_scan(tb, S.ws, &tot_before);
    if (cta_ties && tot_before < need) {  // block-uniform
        uint32_t run = tot_before;
        for (int j = 0; j < per; ++j) {
            if (run >= need) break;  // block-uniform
            const bool tie = sgg[j * kSRT + tid] == gstar;
            uint32_t tot;
            const uint32_t o = sr_block_scan(tie ? 1u : 0u, S.ws, &tot);
            if (tie && run + o < need) out[below + run + o] = int64_t(base + uint32_t(j) * kSRT + tid);
            run += tot;
        }
    }
    if (below) sr_rank_out(W, below, kk, xk, out, &S.mbar[kSRPer + 1], 0, S.part, trace);
    SR_TRACE(6);
}

constexpr uint32_t kPlanSmemMax = 96 * 1024;

}  // namespace

int64_t rowtab_kuv_domain(const int64_t* divk, int ndk) {
    int64_t s = 0;
    for (int k = 0; k < ndk; ++k) {
        int z = 0;
        while (z < 15 && divk[k] % (int64_t(2) << z) == 0) ++z;
        s += int64_t(z + 1) * kKuvV;
    }
    return s;
}

size_t rowtab_scratch_bytes(int nnodes) { return size_t(3) * size_t(nnodes > 0 ? nnodes : 1) * sizeof(double); }

cudaError_t launch_key_hash(const LaunchCtx& c, const uint8_t* d_plan, int64_t nkeys, uint64_t* d_khk,
                            uint64_t* d_khash) {
    if (nkeys <= 0) return cudaSuccess;
    const int64_t want = (nkeys * 64 + 255) / 256;
    const int grid = int(want < int64_t(c.sm_count) * 4 ? want : int64_t(c.sm_count) * 4);
    key_hash_kernel<<<grid, 256, 0, c.stream>>>(d_plan, nkeys, d_khk, d_khash);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_rowtab_compile(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                                  const uint8_t* d_pred, uint32_t pred_bytes, int nnodes, int ndk, int64_t rows_cap,
                                  void* d_scratch, RowTabMeta* d_meta, uint16_t* d_clskuv, uint32_t* d_crep,
                                  double* d_rowpred) {
    (void)plan_bytes;
    (void)pred_bytes;
    if (ndk > 1024) return cudaErrorInvalidValue;
    static const cudaError_t attr =
        cudaFuncSetAttribute(rowtab_classes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(ClsSmem)));
    if (attr != cudaSuccess) return attr;
    cudaError_t e = launch_pdl(rowtab_classes_kernel, dim3(1), dim3(kClsT), sizeof(ClsSmem), c.stream, d_plan, d_pred,
                               static_cast<double*>(d_scratch), nnodes, d_meta, d_clskuv, d_crep);
    if (e != cudaSuccess) return e;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // compact walk: 16-byte nodes + roots + the threads' feature vectors in shared memory
    int ntrees = 0;
    const size_t node_bytes = size_t(nnodes) * 16;
    {  // the tree count is in the predict blob's header (host mirror not needed: bound by nnodes)
        ntrees = nnodes;  // roots region sized for the worst case (one node per tree)
    }
    // ETUNE_BUILD_LANES (diagnostic): lanes per row of the compact walk, 1 / 2 / 4 / 8 (default 4)
    static const int lanes = [] {
        const char* ev = std::getenv("ETUNE_BUILD_LANES");
        const int v = ev ? std::atoi(ev) : 4;
        return v == 1 || v == 2 || v == 8 ? v : 4;
    }();
    const int rows_cta = kBuildT / lanes;
    const size_t sm_c = ((node_bytes + size_t(ntrees) * 4 + 15) / 16) * 16 + size_t(kBuildFS) * rows_cta * 8;
    const bool compact = nnodes < 65536 && sm_c <= size_t(optin);
    int per_sm = 0;
    int64_t want = (rows_cap + kBuildT - 1) / kBuildT;
    if (compact) {
        want = (rows_cap + rows_cta - 1) / rows_cta;
        auto go = [&](auto kern) {
            cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm_c));
            if (e2 != cudaSuccess) return e2;
            e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBuildT, sm_c);
            if (e2 != cudaSuccess) return e2;
            if (per_sm < 1) return cudaErrorInvalidConfiguration;
            const int64_t cap = int64_t(c.sm_count) * per_sm;
            return launch_pdl(kern, dim3(int(want < cap ? (want > 0 ? want : 1) : cap)), dim3(kBuildT), sm_c, c.stream,
                              d_plan, d_pred, nnodes, d_meta, static_cast<const uint32_t*>(d_crep), d_rowpred);
        };
        e = lanes == 1 ? go(rowtab_build_kernel<true, 1>)
            : lanes == 2 ? go(rowtab_build_kernel<true, 2>)
            : lanes == 8 ? go(rowtab_build_kernel<true, 8>)
                         : go(rowtab_build_kernel<true, 4>);
    } else {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rowtab_build_kernel<false, 1>, kBuildT, 0);
        if (e != cudaSuccess) return e;
        const int64_t cap = int64_t(c.sm_count) * (per_sm > 0 ? per_sm : 1);
        e = launch_pdl(rowtab_build_kernel<false, 1>, dim3(int(want < cap ? (want > 0 ? want : 1) : cap)), dim3(kBuildT),
                       0, c.stream, d_plan, d_pred, nnodes, d_meta, static_cast<const uint32_t*>(d_crep), d_rowpred);
    }
    note_launches(2);
    return e;
}

cudaError_t launch_score_rows(const LaunchCtx& c, const uint8_t* d_plan, int ndk, const uint16_t* d_clskuv,
                              const RowTabMeta* d_meta, const double* d_rowpred, const uint64_t* d_khash,
                              const uint64_t* d_genome, int64_t n, double* d_pred, uint64_t* d_ids,
                              const SelHist& sel) {
    if (n <= 0) return cudaSuccess;
    const size_t sm = size_t(ndk) * 64 * 2 + size_t(ndk) * 4;
    if (sm > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(score_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score_rows_kernel, kRowsT, sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int64_t want = (n + int64_t(kRowsT) * kRowsPer - 1) / (int64_t(kRowsT) * kRowsPer);
    const int64_t cap = int64_t(c.sm_count) * per_sm;
    const int grid = int(want < cap ? want : cap);
    const char* nd = std::getenv("ETUNE_ROWS_NODEDUP");  // diagnostic, read every call
    const int nodedup = nd && nd[0] == '1' ? 1 : 0;
    e = launch_pdl(score_rows_kernel, dim3(grid), dim3(kRowsT), sm, c.stream, d_plan, d_clskuv, d_meta, d_rowpred,
                   d_khash, d_genome, n, d_pred, d_ids, sel, nodedup);
    note_launches(1);
    return e;
}

}  // namespace etune_b200

namespace etune_b200 {

size_t rowtab_sort_scratch_bytes(int64_t rows_cap) {  // (the row records are the caller's)
    const int64_t nt = (rows_cap + kRsTile - 1) / kRsTile;
    return size_t(rows_cap) * 16 + size_t(nt) * 256 * 4 + 256 * 4 + size_t(nt) * 4 + size_t((rows_cap + 31) / 32) * 4 +
           2048;
}

cudaError_t launch_rowtab_sort(const LaunchCtx& c, RowTabMeta* d_meta, const double* d_rowpred, int64_t rows_cap,
                               uint32_t* d_srows, uint32_t* d_rowgid, RowRec* d_rowrec, void* d_scratch) {
    if (rows_cap <= 0) return cudaSuccess;
    const int64_t nt64 = (rows_cap + kRsTile - 1) / kRsTile;
    const int nt = int(nt64);
    char* p = static_cast<char*>(d_scratch);
    uint32_t* k0 = reinterpret_cast<uint32_t*>(p);
    uint32_t* k1 = k0 + rows_cap;
    uint32_t* v1 = k1 + rows_cap;
    uint32_t* cnt = v1 + rows_cap;
    uint32_t* tot = cnt + size_t(nt) * 256;
    uint32_t* tcnt = tot + 256;
    uint32_t* mark = tcnt + nt;
    cudaError_t e = cudaMemsetAsync(mark, 0, size_t((rows_cap + 31) / 32) * 4, c.stream);
    if (e != cudaSuccess) return e;
    const int64_t want = (rows_cap + 255) / 256;
    const int grid = int(want < int64_t(c.sm_count) * 8 ? want : int64_t(c.sm_count) * 8);
    const RowTabMeta* cm = d_meta;
    e = launch_pdl(rowtab_keys_kernel, dim3(grid), dim3(256), 0, c.stream, cm, d_rowpred, k0, d_srows);
    uint32_t* kk[2] = {k0, k1};
    uint32_t* vv[2] = {d_srows, v1};
    int cur = 0;
    for (int shift = 0; shift < 32 && e == cudaSuccess; shift += 8) {  // four passes: the result ends in k0 / d_srows
        e = launch_pdl(rs_hist_kernel, dim3(nt), dim3(kRsT), 0, c.stream, cm, static_cast<const uint32_t*>(kk[cur]),
                       shift, nt, cnt);
        if (e == cudaSuccess) e = launch_pdl(rs_scan_kernel, dim3(256), dim3(256), 0, c.stream, cnt, nt, tot);
        if (e == cudaSuccess)
            e = launch_pdl(rs_scatter_kernel, dim3(nt), dim3(kRsT), 0, c.stream, cm,
                           static_cast<const uint32_t*>(kk[cur]), static_cast<const uint32_t*>(vv[cur]), shift,
                           static_cast<const uint32_t*>(cnt), static_cast<const uint32_t*>(tot), nt, kk[cur ^ 1],
                           vv[cur ^ 1]);
        cur ^= 1;
    }
    const uint32_t* ck0 = k0;
    const uint32_t* csr = d_srows;
    if (e == cudaSuccess)
        e = launch_pdl(rowtab_inv_kernel, dim3(grid), dim3(256), 0, c.stream, cm, d_rowpred, ck0, csr, mark);
    if (e == cudaSuccess)
        e = launch_pdl(rowtab_runsort_kernel, dim3(grid), dim3(256), 0, c.stream, cm, d_rowpred, ck0, d_srows, mark);
    if (e == cudaSuccess)
        e = launch_pdl(rowtab_gcount_kernel, dim3(nt), dim3(kRsT), 0, c.stream, cm, d_rowpred, csr, tcnt);
    if (e == cudaSuccess) e = launch_pdl(rowtab_gscan_kernel, dim3(1), dim3(1024), 0, c.stream, d_meta, tcnt, nt);
    if (e == cudaSuccess)
        e = launch_pdl(rowtab_gapply_kernel, dim3(nt), dim3(kRsT), 0, c.stream, cm, d_rowpred, csr,
                       static_cast<const uint32_t*>(tcnt), d_rowgid);
    if (e == cudaSuccess)
        e = launch_pdl(rowtab_pack_kernel, dim3(grid), dim3(256), 0, c.stream, cm, d_rowpred,
                       static_cast<const uint32_t*>(d_rowgid), d_rowrec);
    note_launches(1 + 12 + 6);
    return e;
}

size_t rowsel_work_bytes() { return sizeof(RowSelWork); }

cudaError_t launch_score_select_rows(const LaunchCtx& c, const uint8_t* d_plan, int ndk, int64_t nkeys,
                                     const int32_t* nt, uint32_t off_divk, const uint16_t* d_clskuv, const RowTabMeta* d_meta, const RowRec* d_rowrec,
                                     const uint64_t* d_khash, const uint64_t* d_genome, int64_t n, int64_t k,
                                     double* d_pred, uint64_t* d_ids, int64_t* d_idx, void* d_work) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    if (k > kSelMaxK || k > n || n >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    // [R0 | g per candidate | histogram | Kuv classes | k_tile words | per-key FNV states when <= 64 KB]
    const int khash_smem = nkeys * 8 <= 64 * 1024 ? 1 : 0;
    const size_t sm_fixed = size_t(kSRR0) + size_t(kSRMaxSeg) * 4 + size_t(ndk) * 128 + size_t((ndk + 3) & ~3) * 4 +
                            (khash_smem ? size_t((nkeys * 8 + 15) & ~int64_t(15)) : 0);
    SRPlan PL{};
    PL.nt1 = uint32_t(nt[1]);
    PL.nt2 = uint32_t(nt[2]);
    PL.nkeys = uint32_t(nkeys);
    PL.ndk = ndk;
    PL.off_divk = off_divk;
    PL.khash_smem = khash_smem;
    int optin = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // one CTA per SM: candidates per thread so that the grid covers n
    int64_t gmax = std::min<int64_t>(int64_t(c.sm_count), kSRMaxCtas);
    const int64_t per = (n + gmax * kSRT - 1) / (gmax * kSRT);
    if (per > kSRPer) return cudaErrorNotSupported;  // beyond the grid: the bucketed selection
    const size_t sm = sm_fixed + size_t(per) * kSRT * 4;
    if (sm + sizeof(SRStatic) + 1024 > size_t(optin)) return cudaErrorNotSupported;  // tables too large
    {  // the kernel's dynamic-smem ceiling only grows (contexts on several host threads share it)
        static std::mutex mu;
        static size_t attr_sm = 0;
        std::lock_guard<std::mutex> lock(mu);
        if (sm > attr_sm) {
            const cudaError_t e = cudaFuncSetAttribute(score_select_rows_kernel,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            if (e != cudaSuccess) return e;
            attr_sm = sm;
        }
    }
    const int64_t grid = (n + per * kSRT - 1) / (per * kSRT);
    int per_i = int(per);
    RowSelWork* W = static_cast<RowSelWork*>(d_work);
    // ETUNE_ROWSEL_TRACE=N (diagnostic): per-CTA globaltimer stamps of N back-to-back calls into a ring;
    // every N calls the ring is synchronised and summarised (min / median / max over CTAs and calls
    // of each phase boundary, relative to the earliest CTA start of the call)
    static const int want_trace = std::getenv("ETUNE_ROWSEL_TRACE") ? std::atoi(std::getenv("ETUNE_ROWSEL_TRACE")) : 0;
    static unsigned long long* trace = nullptr;
    static int trace_calls = 0;
    if (want_trace > 0 && !trace) {
        cudaMalloc(&trace, size_t(want_trace) * kSRMaxCtas * kSRTraceSlots * sizeof(unsigned long long));
        cudaMemset(trace, 0, size_t(want_trace) * kSRMaxCtas * kSRTraceSlots * sizeof(unsigned long long));
    }
    unsigned long long* tr = want_trace > 0 ? trace + size_t(trace_calls) * kSRMaxCtas * kSRTraceSlots : nullptr;
    // ETUNE_ROWSEL_ONLY_A=1 (diagnostic, results invalid): stop after the scoring phase so that a
    // profiler sees it as a kernel of its own
    static const int only_a = std::getenv("ETUNE_ROWSEL_ONLY_A") != nullptr ? 1 : 0;
    int oa = only_a;
    // ETUNE_ROWSEL_RADIX=1 (diagnostic, read every call): the radix-select path for any group count
    const char* fr = std::getenv("ETUNE_ROWSEL_RADIX");
    int force_radix = (fr && fr[0] == '1') ? 1 : 0;
    // which candidates' ids are computed where: j < ids_a inside phase A, ids_a <= j < ids_b inside barrier
    // 1's release, the rest inside barrier 2's (ETUNE_ROWSEL_IDS="a,b", diagnostic; b >= 4: R0 layout)
    int ids_a = kSRIdsA, ids_b = kSRIdsB, ids_c = kSRIdsC;
    if (const char* e = std::getenv("ETUNE_ROWSEL_IDS")) {
        if (std::sscanf(e, "%d,%d,%d", &ids_a, &ids_b, &ids_c) != 3) ids_a = kSRIdsA, ids_b = kSRIdsB, ids_c = kSRIdsC;
        if (ids_b < 4) ids_b = 4;
    }
    const char* gm = std::getenv("ETUNE_ROWSEL_GMODE");  // diagnostic, read every call
    int gmode = gm ? std::atoi(gm) : 1;
    void* args[] = {(void*)&d_plan,   (void*)&PL,       (void*)&d_clskuv, (void*)&d_meta, (void*)&d_rowrec,
                    (void*)&d_khash,  (void*)&d_genome, (void*)&n,    (void*)&k,        (void*)&per_i,
                    (void*)&d_pred,   (void*)&d_ids,    (void*)&d_idx,  (void*)&W,        (void*)&tr,
                    (void*)&oa,       (void*)&force_radix, (void*)&ids_a, (void*)&ids_b, (void*)&ids_c, (void*)&gmode};
    note_launches(1);
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(score_select_rows_kernel),
                                                      dim3(unsigned(grid)), dim3(kSRT), args, sm, c.stream);
    if (tr && e == cudaSuccess && ++trace_calls == want_trace) {
        trace_calls = 0;
        cudaStreamSynchronize(c.stream);
        std::vector<unsigned long long> h(size_t(want_trace) * kSRMaxCtas * kSRTraceSlots);
        cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
        constexpr int S = kSRTraceSlots;
        std::vector<double> v[S];
        for (int call = 0; call < want_trace; ++call) {
            const unsigned long long* t = h.data() + size_t(call) * kSRMaxCtas * S;
            unsigned long long t0 = ~0ull;
            for (int b = 0; b < int(grid); ++b) t0 = std::min(t0, t[b * S]);
            for (int b = 0; b < int(grid); ++b)
                for (int s = 0; s < S; ++s)
                    if (s != 15 && s != 16 && t[b * S + s] >= t0) v[s].push_back(double(t[b * S + s] - t0) * 1e-3);
        }
        std::fprintf(stderr, "rowsel: candidates in the crossing segment of the last call: %llu\n",
                     (unsigned long long)h[size_t(want_trace - 1) * kSRMaxCtas * S + 15]);
        static const char* names[S] = {"start", "A done", "flushed", "sync1", "appended", "sync2",
                                       "ranked", "crossed", "staged", "counted", "L-append", "compact",
                                       "msplit", "ids1 done", "A1 issued", "count", "smid", "prologue"};
        std::fprintf(stderr, "rowsel trace n=%lld grid=%lld per=%d over %d calls (us from the first CTA start):\n",
                     (long long)n, (long long)grid, per_i, want_trace);
        for (int s = 0; s < S; ++s) {
            if (v[s].empty()) continue;
            std::sort(v[s].begin(), v[s].end());
            std::fprintf(stderr, "  %-9s min %7.2f  p50 %7.2f  p90 %7.2f  max %7.2f\n", names[s], v[s].front(),
                         v[s][v[s].size() / 2], v[s][v[s].size() * 9 / 10], v[s].back());
        }
        // the same stamps per SM-id bucket of 16 (mean over the CTAs and calls): is a part of the chip slower?
        for (int s : {14, 1, 13}) {
            double sum[16] = {}, cnt[16] = {};
            for (int call = 0; call < want_trace; ++call) {
                const unsigned long long* t = h.data() + size_t(call) * kSRMaxCtas * S;
                unsigned long long t0 = ~0ull;
                for (int b = 0; b < int(grid); ++b) t0 = std::min(t0, t[b * S]);
                for (int b = 0; b < int(grid); ++b) {
                    if (t[b * S + s] < t0) continue;
                    const int q = int(t[b * S + 16] / 16) & 15;
                    sum[q] += double(t[b * S + s] - t0) * 1e-3;
                    cnt[q] += 1;
                }
            }
            std::fprintf(stderr, "  %-9s by smid/16:", names[s]);
            for (int q = 0; q < 16; ++q)
                if (cnt[q] > 0) std::fprintf(stderr, " %5.2f", sum[q] / cnt[q]);
            std::fprintf(stderr, "\n");
        }
        cudaMemset(trace, 0, h.size() * 8);
    }
    return e;
}

}  // namespace etune_b200
