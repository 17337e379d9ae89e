// Selection: the k lowest predictions under the total order (score asc, index asc).
//
// topk = ONE cooperative kernel (grid-wide barriers between phases, no host sync):
//   A. order-preserving 64-bit keys (cached in shared memory per CTA) + AND/OR of
//      all keys, i.e. which bits vary at all
//   B. MSB-first radix select of the exact k-th key T over the varying bits, 11-bit
//      digits: per-CTA shared histograms (warp-aggregated atomics, so thousands of
//      tied predictions - SURVEY H3 - do not serialise) -> global histogram -> every
//      CTA derives the same digit
//   C. per-CTA counts of key < T and key == T
//   D. stable compaction in index order: all keys < T plus the `need` lowest-index
//      keys == T -> exactly k (key, index) pairs
//   E. CTA 0 bitonic-sorts the k pairs by (key, index)  [k <= 4096]
// For k > 4096 the host follows with the stable LSD radix sort below (k is known on
// the host, so no synchronisation is needed to decide).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "kernels.hpp"
#include "pdl.cuh"
#include "selbin.cuh"

namespace etune_b200 {

namespace {

constexpr int kTile = 4096;        // items per tile (count/scatter, LSD sort)
constexpr int kBins = 2048;        // 11-bit digits
constexpr int kSmallSort = 4096;   // one-CTA bitonic bound

__device__ __forceinline__ uint64_t order_key(double x) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

constexpr int kCoopT = 1024;
constexpr int kMaxPasses = 7;             // 8 + 11-bit digits over <= 64 varying bits
constexpr int kSmemKeys = 24 * 1024;      // keys cached per CTA (192 KB)

struct TopkWork {
    unsigned long long cta_and[1024], cta_or[1024];         // phase A, one slot per CTA (no init)
    unsigned int hist[kMaxPasses][kBins];
    unsigned int cnt[2][1024];            // per-CTA (lt, eq) counts
};

// warp-aggregated shared atomic add of 1 to bin[d]
__device__ __forceinline__ void agg_inc(unsigned int* bin, unsigned d, bool valid) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const unsigned peers = __match_any_sync(act, d);
    if ((__ffs(peers) - 1) == int(threadIdx.x & 31)) atomicAdd(&bin[d], unsigned(__popc(peers)));
}

__device__ __forceinline__ unsigned block_sum(unsigned v, unsigned* red) {
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

// Exclusive scan across the warps of a block of one value per warp (`v` significant in
// lane 0 of each warp); returns the warp's exclusive prefix to every lane and the block
// total in *total.  Two barriers.
__device__ __forceinline__ unsigned warp_prefix(unsigned v, unsigned* buf, unsigned* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) buf[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const unsigned x = lane < nw ? buf[lane] : 0u;
        unsigned y = x;
        for (int s = 1; s < 32; s <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, y, s);
            if (lane >= s) y += t;
        }
        if (lane < nw) buf[32 + lane] = y - x;
        if (lane == 31) buf[64] = y;
    }
    __syncthreads();
    *total = buf[64];
    return buf[32 + warp];
}

// (key, index) compare-exchange for the in-register bitonic network
__device__ __forceinline__ void cmpx(unsigned long long& k, unsigned& i, unsigned long long pk, unsigned pi,
                                     bool keep_min) {
    const bool mine_less = k < pk || (k == pk && i < pi);
    if (mine_less != keep_min) {
        k = pk;
        i = pi;
    }
}

// Whole top-k in one cooperative launch (grid-wide barriers between phases).  Each CTA
// owns one contiguous chunk of the scores, caches its keys in shared memory (when they
// fit) and all CTAs derive identical radix decisions from the global histograms.
__global__ void __launch_bounds__(kCoopT, 1) topk_coop_kernel(const double* __restrict__ score, int64_t n, int64_t k,
                                                              TopkWork* __restrict__ w, uint64_t* __restrict__ sel_key,
                                                              uint32_t* __restrict__ sel_idx, int64_t* __restrict__ out,
                                                              int cache_keys, int final_sort) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ unsigned long long skeys[];
    __shared__ unsigned int h[kBins];
    __shared__ unsigned int red[32];
    __shared__ unsigned int scanbuf[72];
    __shared__ unsigned int s_pick[2];
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const int64_t chunk = (n + G - 1) / G;
    const int64_t lo = int64_t(b) * chunk;
    const int64_t hi = lo + chunk < n ? lo + chunk : n;
    const int64_t m = hi > lo ? hi - lo : 0;
    auto key_at = [&](int64_t j) -> uint64_t {  // j in [0, m)
        return cache_keys ? skeys[j] : order_key(score[lo + j]);
    };

    // ---- phase A: keys (+ cache) and which bits vary
    uint64_t a = ~0ull, o = 0ull;
    for (int64_t j = tid; j < m; j += blockDim.x) {
        const uint64_t key = order_key(score[lo + j]);
        if (cache_keys) skeys[j] = key;
        a &= key;
        o |= key;
    }
    for (int s = 16; s > 0; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    __shared__ unsigned long long ra[32], ro[32];
    if ((tid & 31) == 0) {
        ra[tid >> 5] = a;
        ro[tid >> 5] = o;
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 1; i < int(blockDim.x >> 5); ++i) {
            a &= ra[i];
            o |= ro[i];
        }
        w->cta_and[b] = ra[0] & a;
        w->cta_or[b] = ro[0] | o;
    }
    if (b == 0) {  // the rest of the work area is initialised here: no memsets before the launch
        unsigned int* hz = &w->hist[0][0];
        for (int i = tid; i < kMaxPasses * kBins; i += blockDim.x) hz[i] = 0u;
    }
    grid.sync();

    // ---- phase B: radix select of the exact k-th key T (MSB first, 11-bit digits)
    uint64_t andv = ~0ull, orv = 0ull;
    for (int i = tid; i < G; i += blockDim.x) {  // block-wide reduction of the per-CTA slots
        andv &= w->cta_and[i];
        orv |= w->cta_or[i];
    }
    for (int s = 16; s > 0; s >>= 1) {
        andv &= __shfl_xor_sync(0xffffffffu, andv, s);
        orv |= __shfl_xor_sync(0xffffffffu, orv, s);
    }
    __syncthreads();  // ra/ro reuse
    if ((tid & 31) == 0) {
        ra[tid >> 5] = andv;
        ro[tid >> 5] = orv;
    }
    __syncthreads();
    for (int i = 0; i < int(blockDim.x >> 5); ++i) {
        andv &= ra[i];
        orv |= ro[i];
    }
    const uint64_t varying = andv ^ orv;
    uint64_t prefix = andv;  // bits above `bit` fixed so far
    unsigned rem = unsigned(k);  // 1-based rank of T inside the current prefix group
    int bit = varying ? 64 - __clzll(static_cast<long long>(varying)) : 0;  // bits [0, bit) still open
    for (int pass = 0; bit > 0; ++pass) {
        const int dw = pass == 0 ? 8 : 11;  // narrow first digit: fewer global atomics
        const int width = bit >= dw ? dw : bit;
        const int sh = bit - width;
        const uint64_t himask = (bit >= 64) ? 0ull : (~0ull << bit);
        for (int i = tid; i < kBins; i += blockDim.x) h[i] = 0;
        __syncthreads();
        const int64_t mr = (m + blockDim.x - 1) / blockDim.x * blockDim.x;
        for (int64_t j = tid; j < mr; j += blockDim.x) {
            bool v = false;
            unsigned d = 0;
            if (j < m) {
                const uint64_t key = key_at(j);
                v = (key & himask) == (prefix & himask);
                d = unsigned(key >> sh) & ((1u << width) - 1u);
            }
            agg_inc(h, d, v);
        }
        __syncthreads();
        for (int i = tid; i < (1 << width); i += blockDim.x)
            if (h[i]) atomicAdd(&w->hist[pass][i], h[i]);
        grid.sync();
        // every CTA: pick the digit holding rank `rem` (identical result everywhere)
        const int nb = 1 << width;
        const int per = (nb + blockDim.x - 1) / blockDim.x;  // 1 or 2 bins per thread
        unsigned mine = 0;
        for (int q = 0; q < per; ++q) {
            const int i = tid * per + q;
            if (i < nb) mine += w->hist[pass][i];
        }
        // exclusive scan of `mine` over the block
        unsigned x = mine;
        for (int s = 1; s < 32; s <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, s);
            if ((tid & 31) >= s) x += y;
        }
        unsigned btot;
        const unsigned wbase = warp_prefix(__shfl_sync(0xffffffffu, x, 31), scanbuf, &btot);
        unsigned run = wbase + x - mine;  // exclusive
        for (int q = 0; q < per; ++q) {
            const int i = tid * per + q;
            if (i < nb) {
                const unsigned c = w->hist[pass][i];
                if (run < rem && run + c >= rem) {
                    s_pick[0] = unsigned(i);
                    s_pick[1] = rem - run;
                }
                run += c;
            }
        }
        __syncthreads();
        prefix = (prefix & himask) | (uint64_t(s_pick[0]) << sh);  // bits below sh: still open
        rem = s_pick[1];
        bit = sh;
        __syncthreads();
    }
    const uint64_t T = prefix;
    const unsigned need = rem;                // ties at T taken by ascending index
    // ---- phase C: per-CTA counts
    unsigned lt = 0, eq = 0;
    for (int64_t j = tid; j < m; j += blockDim.x) {
        const uint64_t key = key_at(j);
        lt += key < T;
        eq += key == T;
    }
    lt = block_sum(lt, red);
    eq = block_sum(eq, red);
    if (tid == 0) {
        w->cnt[0][b] = lt;
        w->cnt[1][b] = eq;
    }
    grid.sync();
    // ---- phase D: stable compaction in index order
    unsigned pl = 0, pe = 0;
    for (int i = tid; i < b; i += blockDim.x) {
        pl += w->cnt[0][i];
        pe += w->cnt[1][i];
    }
    pl = block_sum(pl, red);
    pe = block_sum(pe, red);
    const int lane = tid & 31;
    const unsigned ltm = (1u << lane) - 1u;
    const int64_t mr = (m + blockDim.x - 1) / blockDim.x * blockDim.x;
    for (int64_t j0 = 0; j0 < mr; j0 += blockDim.x) {
        const int64_t j = j0 + tid;
        uint64_t key = 0;
        bool isl = false, ise = false;
        if (j < m) {
            key = key_at(j);
            isl = key < T;
            ise = key == T;
        }
        const unsigned bl = __ballot_sync(0xffffffffu, isl), be = __ballot_sync(0xffffffffu, ise);
        // one scan of both counts packed in 16-bit halves (a block holds <= 1024 keys)
        unsigned tot;
        const unsigned x0 = warp_prefix(unsigned(__popc(bl)) | (unsigned(__popc(be)) << 16), scanbuf, &tot);
        const unsigned tl = tot & 0xffffu, te = tot >> 16;
        const unsigned xl = pl + (x0 & 0xffffu) + __popc(bl & ltm);
        const unsigned xe = pe + (x0 >> 16) + __popc(be & ltm);
        if (isl || (ise && xe < need)) {
            const unsigned pos = xl + (xe < need ? xe : need);
            sel_key[pos] = key;
            sel_idx[pos] = uint32_t(lo + j);
        }
        pl += tl;
        pe += te;
        __syncthreads();  // scan buffers reused by the next chunk
    }
    if (!final_sort) return;
    grid.sync();
    // ---- phase E: CTA 0 sorts the k pairs by (key, index) (bitonic, k <= kSmallSort)
    if (b != 0) return;
    int P = 1;
    while (P < int(k)) P <<= 1;
    if (P <= int(blockDim.x)) {
        // one pair per thread in registers: strides < 32 by warp shuffles, larger strides
        // through shared memory (15 exchanges for 1024 pairs instead of 55 smem stages)
        unsigned long long* xk = skeys;
        unsigned int* xi = reinterpret_cast<unsigned int*>(skeys + 1024);
        unsigned long long kk = tid < int(k) ? sel_key[tid] : ~0ull;
        unsigned ii = tid < int(k) ? sel_idx[tid] : 0xffffffffu;
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const bool up = (tid & size) == 0;
                const bool low = (tid & stride) == 0;  // the lower index of the pair
                unsigned long long pk;
                unsigned pi;
                if (stride >= 32) {
                    __syncthreads();
                    xk[tid] = kk;
                    xi[tid] = ii;
                    __syncthreads();
                    pk = xk[tid ^ stride];
                    pi = xi[tid ^ stride];
                } else {
                    pk = __shfl_xor_sync(0xffffffffu, kk, stride);
                    pi = __shfl_xor_sync(0xffffffffu, ii, stride);
                }
                if (tid < P) cmpx(kk, ii, pk, pi, up == low);
            }
        }
        if (tid < int(k)) out[tid] = ii;
        return;
    }
    unsigned long long* sk = skeys;
    unsigned int* si = reinterpret_cast<unsigned int*>(skeys + kSmallSort);
    for (int i = tid; i < P; i += blockDim.x) {
        sk[i] = i < int(k) ? sel_key[i] : ~0ull;
        si[i] = i < int(k) ? sel_idx[i] : 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool gt = (sk[i] > sk[j]) || (sk[i] == sk[j] && si[i] > si[j]);
                    if (gt == up) {
                        const unsigned long long tk = sk[i];
                        sk[i] = sk[j];
                        sk[j] = tk;
                        const unsigned ti = si[i];
                        si[i] = si[j];
                        si[j] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < int(k); i += blockDim.x) out[i] = si[i];
}

// ------------------------------------------------------- stable LSD radix sort
constexpr int kLsdT = 512;

// dn / dbits (nullable): item count and key bit length read from device memory (a sort whose
// size is only known on the device, e.g. the row table's rows); passes at or beyond dbits are
// skipped (the scatter copies its tile through so the ping-pong buffers stay consistent).
__global__ void __launch_bounds__(kLsdT) lsd_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                        uint32_t* __restrict__ hist, int ntiles,
                                                        const int64_t* __restrict__ dn,
                                                        const int32_t* __restrict__ dbits) {
    if (dbits && shift >= *dbits) return;
    if (dn) n = *dn;
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kTile;
    for (int r = 0; r < kTile / kLsdT; ++r) {
        const int64_t i = base + r * kLsdT + threadIdx.x;
        const bool v = i < n;
        agg_inc(h, v ? unsigned(keys[i] >> shift) & 0xffu : 0u, v);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[int64_t(d) * ntiles + blockIdx.x] = h[d];
}

// exclusive scan of hist[256][ntiles] in digit-major order: warp per digit row
__global__ void __launch_bounds__(1024) lsd_scan_kernel(uint32_t* __restrict__ hist, int ntiles, int shift,
                                                        const int32_t* __restrict__ dbits) {
    if (dbits && shift >= *dbits) return;
    __shared__ uint32_t tot[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = warp; d < 256; d += 32) {
        uint32_t run = 0;
        for (int b = 0; b < ntiles; b += 32) {
            const int i = b + lane;
            const uint32_t v = i < ntiles ? hist[int64_t(d) * ntiles + i] : 0u;
            uint32_t x = v;
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
                if (lane >= s) x += y;
            }
            if (i < ntiles) hist[int64_t(d) * ntiles + i] = run + x - v;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) tot[d] = run;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 digit totals
        uint32_t carry = 0;
        for (int b = 0; b < 256; b += 32) {
            const uint32_t v = tot[b + lane];
            uint32_t x = v;
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, s);
                if (lane >= s) x += y;
            }
            tot[b + lane] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    __syncthreads();
    for (int d = warp; d < 256; d += 32) {
        const uint32_t add = tot[d];
        for (int i = lane; i < ntiles; i += 32) hist[int64_t(d) * ntiles + i] += add;
    }
}

__global__ void __launch_bounds__(kLsdT) lsd_scatter_kernel(const uint64_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin, int64_t n, int shift,
                                                           const uint32_t* __restrict__ offs, int ntiles,
                                                           uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           const int64_t* __restrict__ dn,
                                                           const int32_t* __restrict__ dbits) {
    if (dn) n = *dn;
    if (dbits && shift >= *dbits) {  // skipped pass: carry the tile over unchanged
        for (int64_t i = int64_t(blockIdx.x) * kTile + threadIdx.x; i < n && i < int64_t(blockIdx.x + 1) * kTile;
             i += blockDim.x) {
            kout[i] = kin[i];
            vout[i] = vin[i];
        }
        return;
    }
    constexpr int W = kLsdT / 32;
    __shared__ uint32_t base[256];
    __shared__ uint32_t gofs[256];
    __shared__ uint32_t wc[W][257];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int d = tid; d < 256; d += blockDim.x) {
        base[d] = 0;
        gofs[d] = offs[int64_t(d) * ntiles + blockIdx.x];
    }
    const unsigned lt = (1u << lane) - 1u;
    const int64_t tbase = int64_t(blockIdx.x) * kTile;
    for (int r = 0; r < kTile / kLsdT; ++r) {
        for (int j = tid; j < W * 257; j += blockDim.x) (&wc[0][0])[j] = 0;
        __syncthreads();
        const int64_t i = tbase + r * kLsdT + tid;
        const bool valid = i < n;
        uint64_t key = 0;
        uint32_t val = 0;
        unsigned d = 256;
        if (valid) {
            key = kin[i];
            val = vin[i];
            d = unsigned(key >> shift) & 0xffu;
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

__global__ void widen_kernel(const uint32_t* __restrict__ vals, int64_t k, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < k; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = vals[i];
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// --------------------------------------------- fused selection (score_select)
// The score kernel has counted every prediction into kSelBins monotone buckets
// (kernels.cu sel_bin).  Bucket d* holds the k-th key: every key of a lower bucket
// is selected, the bucket itself is resolved exactly by one CTA.
struct SelWork {
    unsigned int hist[kSelBins];
    unsigned int nL, nB;  // appended below-bucket / in-bucket pairs
    unsigned int ticket;  // sel_rank_kernel: CTAs done
    unsigned int pad[61];
};
constexpr int kSelT = 512;          // filter CTA
constexpr int kFinT = 1024;         // finish CTA
constexpr int kSelCacheB = 8192;    // in-bucket pairs cached in the finish CTA's smem

struct SelLayout {
    SelWork* w;
    uint64_t* lk;  // [kSelMaxK]
    uint32_t* li;
    uint32_t* lr;  // rank counters of the below-bucket pairs
    uint64_t* bk;  // [n]
    uint32_t* bi;
    uint32_t* br;  // rank counters of the in-bucket pairs
};

__host__ __device__ inline size_t sel_al(size_t x) { return (x + 255) & ~size_t(255); }

SelLayout sel_layout(void* base, int64_t n) {
    char* p = static_cast<char*>(base);
    SelLayout L;
    L.w = reinterpret_cast<SelWork*>(p);
    p += sel_al(sizeof(SelWork));
    L.lk = reinterpret_cast<uint64_t*>(p);
    p += sel_al(8 * size_t(kSelMaxK));
    L.li = reinterpret_cast<uint32_t*>(p);
    p += sel_al(4 * size_t(kSelMaxK));
    L.lr = reinterpret_cast<uint32_t*>(p);
    p += sel_al(4 * size_t(kSelMaxK));
    L.bk = reinterpret_cast<uint64_t*>(p);
    p += sel_al(8 * size_t(n));
    L.bi = reinterpret_cast<uint32_t*>(p);
    p += sel_al(4 * size_t(n));
    L.br = reinterpret_cast<uint32_t*>(p);
    return L;
}

// Every CTA derives the same d* (the bucket holding rank k) from the global histogram,
// then classifies kFiltPer scores per thread (loads issued before the histogram scan,
// so their latency overlaps it).
constexpr int kFiltPer = 8;

__global__ void __launch_bounds__(kSelT) sel_filter_kernel(const double* __restrict__ score, int64_t n, int64_t k,
                                                           SelLayout L, const SelHist sel_in) {
    __shared__ unsigned int scanbuf[72];
    __shared__ unsigned int s_d;
    const int tid = threadIdx.x;
    static_assert(kSelBins == 2 * kSelT, "two bins per thread");
    const int64_t span = int64_t(kSelT) * kFiltPer;
    int64_t base = int64_t(blockIdx.x) * span;
    double v[kFiltPer];
#pragma unroll
    for (int r = 0; r < kFiltPer; ++r) {  // scores are written by the score kernel: after the wait
        v[r] = 0.0;
    }
    pdl_wait();
    const SelHist sel = sel_resolve(sel_in);  // device-resident bounds: written by an earlier kernel
#pragma unroll
    for (int r = 0; r < kFiltPer; ++r) {
        const int64_t j = base + r * kSelT + tid;
        if (j < n) v[r] = __ldcg(score + j);
    }
    const unsigned h0 = L.w->hist[2 * tid], h1 = L.w->hist[2 * tid + 1];
    const unsigned mine = h0 + h1;
    unsigned x = mine;
    for (int s = 1; s < 32; s <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, s);
        if ((tid & 31) >= s) x += y;
    }
    unsigned btot;
    const unsigned run = warp_prefix(__shfl_sync(0xffffffffu, x, 31), scanbuf, &btot) + x - mine;  // exclusive
    const unsigned kk = unsigned(k);
    if (run < kk && run + h0 >= kk) s_d = unsigned(2 * tid);
    else if (run + h0 < kk && run + mine >= kk) s_d = unsigned(2 * tid + 1);
    __syncthreads();
    const unsigned d = s_d;
    __shared__ unsigned s_base[2];
    for (;;) {
        // classify; takes are appended CTA-aggregated (one global atomic per list per
        // CTA), so thousands of tied predictions do not serialise on one counter
        uint64_t key[kFiltPer];
        unsigned tl = 0, tb = 0;
#pragma unroll
        for (int r = 0; r < kFiltPer; ++r) {
            const int64_t j = base + r * kSelT + tid;
            const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v[r]));
            key[r] = (bits >> 63) ? ~bits : (bits | 0x8000000000000000ull);
            unsigned bin = kSelBins;
            if (j < n) {
                if (key[r] < sel.kmin) {
                    bin = 0u;
                } else {
                    const uint64_t q = (key[r] - sel.kmin) >> sel.shift;
                    bin = q < uint64_t(kSelBins - 1) ? unsigned(q) : unsigned(kSelBins - 1);
                }
            }
            tl |= unsigned(bin < d) << r;
            tb |= unsigned(bin == d) << r;
        }
        if (__syncthreads_or(tl | tb)) {
            const unsigned c = unsigned(__popc(tl)) | (unsigned(__popc(tb)) << 16);
            unsigned x = c;
            for (int s = 1; s < 32; s <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, x, s);
                if ((tid & 31) >= s) x += y;
            }
            unsigned tot;
            const unsigned pre = warp_prefix(__shfl_sync(0xffffffffu, x, 31), scanbuf, &tot) + x - c;
            if (tid == 0) {
                s_base[0] = (tot & 0xffffu) ? atomicAdd(&L.w->nL, tot & 0xffffu) : 0u;
                s_base[1] = (tot >> 16) ? atomicAdd(&L.w->nB, tot >> 16) : 0u;
            }
            __syncthreads();
            unsigned pl = s_base[0] + (pre & 0xffffu), pb = s_base[1] + (pre >> 16);
#pragma unroll
            for (int r = 0; r < kFiltPer; ++r) {
                const uint32_t j = uint32_t(base + r * kSelT + tid);
                if ((tl >> r) & 1u) {
                    L.lk[pl] = key[r];
                    L.li[pl] = j;
                    L.lr[pl] = 0u;  // sel_rank_kernel accumulates into it
                    ++pl;
                }
                if ((tb >> r) & 1u) {
                    L.bk[pb] = key[r];
                    L.bi[pb] = j;
                    L.br[pb] = 0u;
                    ++pb;
                }
            }
        }
        base += int64_t(gridDim.x) * span;
        if (base >= n) break;
#pragma unroll
        for (int r = 0; r < kFiltPer; ++r) {
            const int64_t j = base + r * kSelT + tid;
            v[r] = j < n ? __ldcg(score + j) : 0.0;
        }
    }
}

// Candidate set C = below-bucket list ++ in-bucket list.  When it is small (the usual
// case) every element's rank in C under (key, index) is counted directly and
// out[rank] = index for rank < k.  Work units are tiles of kRankI items x kRankJ
// candidates spread over the whole GPU (each lane holds 4 items, each staged record
// is one broadcast shared load compared against all 4 by a 96-bit borrow chain);
// partial ranks go to the per-pair counters (zeroed by the filter) with atomics and the
// last CTA scatters.  |C| = 4096: 16.7 M compares.  Larger sets (heavy ties spilling
// the bucket) take sel_finish_kernel.
constexpr int kRankT = 512;
constexpr int kRankR = 4;                     // items per lane
constexpr unsigned kRankI = 32 * kRankR;      // items per tile
constexpr unsigned kRankJ = 512;              // candidates per tile
constexpr unsigned kRankCap = 8192;

__device__ __forceinline__ ulonglong2 cand_at(const SelLayout& L, unsigned nL, unsigned t) {
    return t < nL ? make_ulonglong2(L.lk[t], L.li[t]) : make_ulonglong2(L.bk[t - nL], L.bi[t - nL]);
}

// 0xffffffff when (rk, ri) < (mk, mi) lexicographically, else 0: the borrow out of the
// 96-bit subtraction, sign-extended (callers subtract it from a counter)
__device__ __forceinline__ unsigned less96(unsigned long long rk, unsigned ri, unsigned long long mk, unsigned mi) {
    unsigned b;
    asm("{\n\t.reg .u32 t;\n\t"
        "sub.cc.u32 t, %1, %4;\n\t"
        "subc.cc.u32 t, %2, %5;\n\t"
        "subc.cc.u32 t, %3, %6;\n\t"
        "subc.u32 %0, 0, 0;\n\t}"
        : "=r"(b)
        : "r"(ri), "r"(unsigned(rk)), "r"(unsigned(rk >> 32)), "r"(mi), "r"(unsigned(mk)), "r"(unsigned(mk >> 32)));
    return b;
}

__global__ void __launch_bounds__(kRankT) sel_rank_kernel(int64_t k, SelLayout L, int64_t* __restrict__ out) {
    __shared__ ulonglong2 rec[kRankJ];
    __shared__ unsigned part[kRankT / 32][kRankI];
    __shared__ unsigned s_last;
    pdl_wait();
    const unsigned nL = L.w->nL, nC = nL + L.w->nB;
    if (nC > kRankCap) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int kW = kRankT / 32;
    const unsigned ni = (nC + kRankI - 1) / kRankI, nj = (nC + kRankJ - 1) / kRankJ;
    for (unsigned u = blockIdx.x; u < ni * nj; u += gridDim.x) {
        const unsigned ib = u / nj, jb = u % nj;
        const unsigned j0 = jb * kRankJ;
        const unsigned m = nC - j0 < kRankJ ? nC - j0 : kRankJ;
        __syncthreads();  // rec / part reuse
        for (unsigned t = tid; t < m; t += kRankT) rec[t] = cand_at(L, nL, j0 + t);
        unsigned long long mk[kRankR];
        unsigned mi[kRankR], cnt[kRankR];
#pragma unroll
        for (int r = 0; r < kRankR; ++r) {
            const unsigned i = ib * kRankI + r * 32 + lane;
            const ulonglong2 me = i < nC ? cand_at(L, nL, i) : make_ulonglong2(~0ull, ~0ull);
            mk[r] = me.x;
            mi[r] = unsigned(me.y);
            cnt[r] = 0;
        }
        __syncthreads();
        const unsigned per = (m + kW - 1) / kW;
        const unsigned a = warp * per, b = a + per < m ? a + per : m;
#pragma unroll 2
        for (unsigned j = a; j < b; ++j) {
            const ulonglong2 rj = rec[j];
#pragma unroll
            for (int r = 0; r < kRankR; ++r) cnt[r] -= less96(rj.x, unsigned(rj.y), mk[r], mi[r]);
        }
#pragma unroll
        for (int r = 0; r < kRankR; ++r) part[warp][r * 32 + lane] = cnt[r];
        __syncthreads();
        if (tid < int(kRankI)) {
            unsigned c = 0;
#pragma unroll
            for (int w = 0; w < kW; ++w) c += part[w][tid];
            const unsigned i = ib * kRankI + tid;
            if (i < nC && c) atomicAdd(i < nL ? L.lr + i : L.br + (i - nL), c);
        }
    }
    // the last CTA to finish scatters out[rank] = index for rank < k
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&L.w->ticket, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    constexpr int kB = 8;  // independent loads in flight per thread
    for (unsigned i0 = 0; i0 < nC; i0 += kB * kRankT) {
        unsigned rk[kB], id[kB];
#pragma unroll
        for (int r = 0; r < kB; ++r) {
            const unsigned i = i0 + r * kRankT + tid;
            rk[r] = 0xffffffffu;
            id[r] = 0;
            if (i < nC) {
                rk[r] = __ldcg(i < nL ? L.lr + i : L.br + (i - nL));
                id[r] = i < nL ? L.li[i] : L.bi[i - nL];
            }
        }
#pragma unroll
        for (int r = 0; r < kB; ++r)
            if (rk[r] < unsigned(k)) out[rk[r]] = int64_t(id[r]);
    }
    if (tid == 0) L.w->ticket = 0u;
}

// Block (1024 threads) pick of the bin holding 1-based rank `rem` among nb <= 2048
// counters; result in s_pick = {bin, rank inside the bin}.  Ends with a barrier.
__device__ __forceinline__ void block_pick(const unsigned* h, int nb, unsigned rem, unsigned* scanbuf,
                                           unsigned* s_pick) {
    const int tid = threadIdx.x;
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    unsigned mine = 0;
    for (int q = 0; q < per; ++q) {
        const int i = tid * per + q;
        if (i < nb) mine += h[i];
    }
    unsigned x = mine;
    for (int s = 1; s < 32; s <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, s);
        if ((tid & 31) >= s) x += y;
    }
    unsigned btot;
    unsigned run = warp_prefix(__shfl_sync(0xffffffffu, x, 31), scanbuf, &btot) + x - mine;
    for (int q = 0; q < per; ++q) {
        const int i = tid * per + q;
        if (i < nb) {
            const unsigned c = h[i];
            if (run < rem && run + c >= rem) {
                s_pick[0] = unsigned(i);
                s_pick[1] = rem - run;
            }
            run += c;
        }
    }
    __syncthreads();
}

// One CTA: exact (key, index) rank-`rem` element inside bucket d*, then the k pairs
// (all below-bucket pairs + the selected in-bucket ones) sorted by (key, index).
__global__ void __launch_bounds__(kFinT, 1) sel_finish_kernel(int64_t k, SelLayout L, int64_t* __restrict__ out) {
    extern __shared__ unsigned long long fsm[];
    unsigned long long* xk = fsm;                                    // [kSelMaxK]
    unsigned int* xi = reinterpret_cast<unsigned int*>(xk + kSelMaxK);  // [kSelMaxK]
    unsigned long long* ck = reinterpret_cast<unsigned long long*>(xi + kSelMaxK);  // [kSelCacheB]
    unsigned int* ci = reinterpret_cast<unsigned int*>(ck + kSelCacheB);            // [kSelCacheB]
    __shared__ unsigned int h[kBins];
    __shared__ unsigned int red[32];
    __shared__ unsigned int scanbuf[72];
    __shared__ unsigned int s_pick[2];
    __shared__ unsigned int s_cnt;
    __shared__ unsigned long long ra[32], ro[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    pdl_wait();
    const unsigned nL = L.w->nL, nB = L.w->nB;
    const unsigned K = unsigned(k);
    if (nL + nB <= kRankCap) {  // sel_rank_kernel wrote the result: only reset the work area
        for (int i = tid; i < kSelBins; i += blockDim.x) L.w->hist[i] = 0u;
        if (tid == 0) {
            L.w->nL = 0u;
            L.w->nB = 0u;
        }
        return;
    }
    const bool cached = nB <= unsigned(kSelCacheB);
    if (cached)
        for (unsigned j = tid; j < nB; j += blockDim.x) {
            ck[j] = L.bk[j];
            ci[j] = L.bi[j];
        }
    const unsigned long long* BK = cached ? ck : reinterpret_cast<const unsigned long long*>(L.bk);
    const unsigned int* BI = cached ? ci : L.bi;
    const unsigned nBr = (nB + blockDim.x - 1) / blockDim.x * blockDim.x;

    // ---- exact key T of in-bucket rank rem (MSB-first radix select over the varying bits)
    uint64_t a = ~0ull, o = 0ull;
    for (unsigned j = tid; j < nB; j += blockDim.x) {
        a &= BK[j];
        o |= BK[j];
    }
    for (int s = 16; s > 0; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    if (lane == 0) {
        ra[warp] = a;
        ro[warp] = o;
    }
    __syncthreads();
    for (int i = 0; i < nw; ++i) {
        a &= ra[i];
        o |= ro[i];
    }
    uint64_t prefix = a;
    unsigned rem = K - nL;  // >= 1: bucket d* holds rank K
    int bit = (a ^ o) ? 64 - __clzll(static_cast<long long>(a ^ o)) : 0;
    while (bit > 0) {
        const int width = bit >= 11 ? 11 : bit;
        const int sh = bit - width;
        const uint64_t himask = bit >= 64 ? 0ull : (~0ull << bit);
        for (int i = tid; i < kBins; i += blockDim.x) h[i] = 0u;
        __syncthreads();
        for (unsigned j = tid; j < nBr; j += blockDim.x) {
            bool v = false;
            unsigned dg = 0;
            if (j < nB) {
                const uint64_t key = BK[j];
                v = (key & himask) == (prefix & himask);
                dg = unsigned(key >> sh) & ((1u << width) - 1u);
            }
            agg_inc(h, dg, v);
        }
        __syncthreads();
        block_pick(h, 1 << width, rem, scanbuf, s_pick);
        prefix = (prefix & himask) | (uint64_t(s_pick[0]) << sh);
        rem = s_pick[1];
        bit = sh;
        __syncthreads();
    }
    const uint64_t T = prefix;
    const unsigned need = rem;  // keys == T to take, lowest index first
    unsigned eq = 0;
    for (unsigned j = tid; j < nB; j += blockDim.x) eq += BK[j] == T;
    eq = block_sum(eq, red);
    // ---- ties at T: the need-th smallest index among them (indices are unique)
    unsigned istar = 0xffffffffu;
    if (eq > need) {
        unsigned ia = ~0u, io = 0u;
        for (unsigned j = tid; j < nB; j += blockDim.x)
            if (BK[j] == T) {
                ia &= BI[j];
                io |= BI[j];
            }
        for (int s = 16; s > 0; s >>= 1) {
            ia &= __shfl_xor_sync(0xffffffffu, ia, s);
            io |= __shfl_xor_sync(0xffffffffu, io, s);
        }
        __syncthreads();
        if (lane == 0) {
            ra[warp] = ia;
            ro[warp] = io;
        }
        __syncthreads();
        for (int i = 0; i < nw; ++i) {
            ia &= unsigned(ra[i]);
            io |= unsigned(ro[i]);
        }
        unsigned ip = ia, irem = need;
        int ib = (ia ^ io) ? 32 - __clz(int(ia ^ io)) : 0;
        while (ib > 0) {
            const int width = ib >= 11 ? 11 : ib;
            const int sh = ib - width;
            const unsigned himask = ib >= 32 ? 0u : (~0u << ib);
            for (int i = tid; i < kBins; i += blockDim.x) h[i] = 0u;
            __syncthreads();
            for (unsigned j = tid; j < nBr; j += blockDim.x) {
                bool v = false;
                unsigned dg = 0;
                if (j < nB && BK[j] == T) {
                    const unsigned id = BI[j];
                    v = (id & himask) == (ip & himask);
                    dg = (id >> sh) & ((1u << width) - 1u);
                }
                agg_inc(h, dg, v);
            }
            __syncthreads();
            block_pick(h, 1 << width, irem, scanbuf, s_pick);
            ip = (ip & himask) | (s_pick[0] << sh);
            irem = s_pick[1];
            ib = sh;
            __syncthreads();
        }
        istar = ip;
    }
    // ---- gather the k pairs: all below-bucket pairs, then the selected in-bucket ones
    for (unsigned j = tid; j < nL; j += blockDim.x) {
        xk[j] = L.lk[j];
        xi[j] = L.li[j];
    }
    if (tid == 0) s_cnt = nL;
    __syncthreads();
    for (unsigned j = tid; j < nBr; j += blockDim.x) {
        bool take = false;
        uint64_t key = 0;
        unsigned id = 0;
        if (j < nB) {
            key = BK[j];
            id = BI[j];
            take = key < T || (key == T && id <= istar);
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (m) {
            const int leader = __ffs(m) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(&s_cnt, unsigned(__popc(m)));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (take) {
                const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
                xk[pos] = key;
                xi[pos] = id;
            }
        }
    }
    __syncthreads();
    // ---- (key, index) sort of the K pairs
    int P = 1;
    while (P < int(K)) P <<= 1;
    if (P <= int(blockDim.x)) {
        unsigned long long kk = tid < int(K) ? xk[tid] : ~0ull;
        unsigned ii = tid < int(K) ? xi[tid] : 0xffffffffu;
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const bool up = (tid & size) == 0;
                const bool low = (tid & stride) == 0;
                unsigned long long pk;
                unsigned pi;
                if (stride >= 32) {
                    __syncthreads();
                    xk[tid] = kk;
                    xi[tid] = ii;
                    __syncthreads();
                    pk = xk[tid ^ stride];
                    pi = xi[tid ^ stride];
                } else {
                    pk = __shfl_xor_sync(0xffffffffu, kk, stride);
                    pi = __shfl_xor_sync(0xffffffffu, ii, stride);
                }
                if (tid < P) cmpx(kk, ii, pk, pi, up == low);
            }
        }
        if (tid < int(K)) out[tid] = ii;
    } else {
        for (int i = int(K) + tid; i < P; i += blockDim.x) {
            xk[i] = ~0ull;
            xi[i] = 0xffffffffu;
        }
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = tid; i < P; i += blockDim.x) {
                    const int j = i ^ stride;
                    if (j > i) {
                        const bool up = (i & size) == 0;
                        const bool gt = (xk[i] > xk[j]) || (xk[i] == xk[j] && xi[i] > xi[j]);
                        if (gt == up) {
                            const unsigned long long tk = xk[i];
                            xk[i] = xk[j];
                            xk[j] = tk;
                            const unsigned ti = xi[i];
                            xi[i] = xi[j];
                            xi[j] = ti;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int i = tid; i < int(K); i += blockDim.x) out[i] = xi[i];
    }
    // ---- leave the work area clean for the next score_select
    for (int i = tid; i < kSelBins; i += blockDim.x) L.w->hist[i] = 0u;
    if (tid == 0) {
        L.w->nL = 0u;
        L.w->nB = 0u;
    }
}
}  // namespace

size_t sort_pairs_scratch_bytes(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    return al256(8 * size_t(n)) + al256(4 * size_t(n)) + al256(4 * 256 * size_t(ntiles));
}

// Stable LSD radix sort of (u64 key, u32 value) pairs by the low `bits` key bits
// (8-bit digits); result in place.
cudaError_t launch_sort_pairs(const LaunchCtx& c, uint64_t* keys, uint32_t* vals, int64_t n, int bits,
                              void* scratch) {
    if (n <= 1) return cudaSuccess;
    char* p = static_cast<char*>(scratch);
    uint64_t* k2 = reinterpret_cast<uint64_t*>(p);
    p += al256(8 * size_t(n));
    uint32_t* v2 = reinterpret_cast<uint32_t*>(p);
    p += al256(4 * size_t(n));
    uint32_t* hist = reinterpret_cast<uint32_t*>(p);
    const int kt = int((n + kTile - 1) / kTile);
    uint64_t* kk[2] = {keys, k2};
    uint32_t* vv[2] = {vals, v2};
    int cur = 0;
    for (int shift = 0; shift < bits; shift += 8) {
        lsd_hist_kernel<<<kt, kLsdT, 0, c.stream>>>(kk[cur], n, shift, hist, kt, nullptr, nullptr);
        lsd_scan_kernel<<<1, 1024, 0, c.stream>>>(hist, kt, shift, nullptr);
        lsd_scatter_kernel<<<kt, kLsdT, 0, c.stream>>>(kk[cur], vv[cur], n, shift, hist, kt, kk[cur ^ 1], vv[cur ^ 1],
                                                       nullptr, nullptr);
        cur ^= 1;
        note_launches(3);
    }
    if (cur) {
        cudaMemcpyAsync(keys, k2, 8 * size_t(n), cudaMemcpyDeviceToDevice, c.stream);
        cudaMemcpyAsync(vals, v2, 4 * size_t(n), cudaMemcpyDeviceToDevice, c.stream);
    }
    return cudaGetLastError();
}

// Same sort with the item count (<= n_cap) and key bit length in device memory: all eight
// 8-bit passes are launched, those at or beyond *d_bits only copy through.  Result in place.
cudaError_t launch_sort_pairs_dev(const LaunchCtx& c, uint64_t* keys, uint32_t* vals, int64_t n_cap,
                                  const int64_t* d_n, const int32_t* d_bits, void* scratch) {
    if (n_cap <= 0) return cudaSuccess;
    char* p = static_cast<char*>(scratch);
    uint64_t* k2 = reinterpret_cast<uint64_t*>(p);
    p += al256(8 * size_t(n_cap));
    uint32_t* v2 = reinterpret_cast<uint32_t*>(p);
    p += al256(4 * size_t(n_cap));
    uint32_t* hist = reinterpret_cast<uint32_t*>(p);
    const int kt = int((n_cap + kTile - 1) / kTile);
    uint64_t* kk[2] = {keys, k2};
    uint32_t* vv[2] = {vals, v2};
    int cur = 0;
    for (int shift = 0; shift < 64; shift += 8) {  // eight passes: the data ends in keys / vals
        lsd_hist_kernel<<<kt, kLsdT, 0, c.stream>>>(kk[cur], n_cap, shift, hist, kt, d_n, d_bits);
        lsd_scan_kernel<<<1, 1024, 0, c.stream>>>(hist, kt, shift, d_bits);
        lsd_scatter_kernel<<<kt, kLsdT, 0, c.stream>>>(kk[cur], vv[cur], n_cap, shift, hist, kt, kk[cur ^ 1],
                                                       vv[cur ^ 1], d_n, d_bits);
        cur ^= 1;
        note_launches(3);
    }
    return cudaGetLastError();
}

size_t topk_scratch_bytes(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    return al256(sizeof(TopkWork)) + 2 * (al256(8 * size_t(n)) + al256(4 * size_t(n))) +
           al256(4 * 256 * size_t(ntiles));
}

cudaError_t launch_topk(const LaunchCtx& c, const double* d_score, int64_t n, int64_t k, int64_t* d_idx,
                        void* d_scratch) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    char* p = static_cast<char*>(d_scratch);
    TopkWork* w = reinterpret_cast<TopkWork*>(p);
    p += al256(sizeof(TopkWork));
    uint64_t* sk[2];
    uint32_t* sv[2];
    for (int i = 0; i < 2; ++i) {
        sk[i] = reinterpret_cast<uint64_t*>(p);
        p += al256(8 * size_t(n));
        sv[i] = reinterpret_cast<uint32_t*>(p);
        p += al256(4 * size_t(n));
    }
    uint32_t* lsd_hist = reinterpret_cast<uint32_t*>(p);
    // one CTA per SM; cache keys in smem when the per-CTA chunk fits
    int G = c.sm_count;
    const int64_t chunk = (n + G - 1) / G;
    const int cache = chunk <= kSmemKeys ? 1 : 0;
    const int final_sort = k <= kSmallSort ? 1 : 0;
    size_t smem = cache ? size_t(chunk) * 8 : 0;
    if (final_sort) {
        const size_t need = size_t(kSmallSort) * 12;
        if (smem < need) smem = need;
    }
    // one 1024-thread CTA per SM; the smem ceiling is set once to the device maximum and
    // co-residency holds as long as the request fits it
    static std::once_flag once;
    static int optin = 0;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa{};
        attr_err = cudaFuncGetAttributes(&fa, topk_coop_kernel);
        optin -= int(fa.sharedSizeBytes);  // dynamic ceiling = opt-in maximum minus static smem
        if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(topk_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    });
    if (attr_err != cudaSuccess) return attr_err;
    if (smem > size_t(optin)) return cudaErrorCooperativeLaunchTooLarge;
    cudaError_t e = cudaSuccess;
    if (G > 1024) G = 1024;
    void* args[] = {(void*)&d_score, (void*)&n,           (void*)&k,        (void*)&w,          (void*)&sk[0],
                    (void*)&sv[0],   (void*)&d_idx,       (void*)&cache,    (void*)&final_sort};
    e = cudaLaunchCooperativeKernel((const void*)topk_coop_kernel, dim3(G), dim3(kCoopT), args, smem, c.stream);
    if (e != cudaSuccess) return e;
    note_launches(1);
    if (final_sort) return cudaSuccess;
    // stable LSD sort of the k selected pairs (in index order) by key
    const int kt = int((k + kTile - 1) / kTile);
    int cur = 0;
    for (int shift = 0; shift < 64; shift += 8) {
        lsd_hist_kernel<<<kt, kLsdT, 0, c.stream>>>(sk[cur], k, shift, lsd_hist, kt, nullptr, nullptr);
        lsd_scan_kernel<<<1, 1024, 0, c.stream>>>(lsd_hist, kt, shift, nullptr);
        lsd_scatter_kernel<<<kt, kLsdT, 0, c.stream>>>(sk[cur], sv[cur], k, shift, lsd_hist, kt, sk[cur ^ 1],
                                                        sv[cur ^ 1], nullptr, nullptr);
        cur ^= 1;
        note_launches(3);
    }
    const int tg = int((k + 255) / 256 < 1024 ? (k + 255) / 256 : 1024);
    widen_kernel<<<tg, 256, 0, c.stream>>>(sv[cur], k, d_idx);
    note_launches(1);
    return cudaGetLastError();
}

size_t select_scratch_bytes(int64_t n, int64_t k) {
    (void)k;
    return sel_al(sizeof(SelWork)) + sel_al(8 * size_t(kSelMaxK)) + 2 * sel_al(4 * size_t(kSelMaxK)) +
           sel_al(8 * size_t(n)) + 2 * sel_al(4 * size_t(n));
}

uint32_t* select_hist(void* d_sel) { return reinterpret_cast<SelWork*>(d_sel)->hist; }

cudaError_t launch_select(const LaunchCtx& c, const double* d_score, int64_t n, int64_t k, int64_t* d_idx,
                          void* d_sel, const SelHist& sel) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    if (k > kSelMaxK || k > n) return cudaErrorInvalidValue;
    const SelLayout L = sel_layout(d_sel, n);
    int64_t G = 4 * int64_t(c.sm_count);
    const int64_t want = (n + int64_t(kSelT) * kFiltPer - 1) / (int64_t(kSelT) * kFiltPer);
    if (want < G) G = want;
    cudaError_t e = launch_pdl(sel_filter_kernel, dim3(unsigned(G)), dim3(kSelT), 0, c.stream, d_score, n, k, L, sel);
    if (e != cudaSuccess) return e;
    const size_t smem = size_t(kSelMaxK) * 12 + size_t(kSelCacheB) * 12;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [&] {
        attr = cudaFuncSetAttribute(sel_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    });
    if (attr != cudaSuccess) return attr;
    e = launch_pdl(sel_rank_kernel, dim3(2 * c.sm_count), dim3(kRankT), 0, c.stream, k, L, d_idx);
    if (e != cudaSuccess) return e;
    e = launch_pdl(sel_finish_kernel, dim3(1), dim3(kFinT), smem, c.stream, k, L, d_idx);
    note_launches(3);
    return e;
}

}  // namespace etune_b200
