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

__global__ void __launch_bounds__(kLsdT) lsd_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                        uint32_t* __restrict__ hist, int ntiles) {
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
__global__ void __launch_bounds__(1024) lsd_scan_kernel(uint32_t* __restrict__ hist, int ntiles) {
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
                                                           uint64_t* __restrict__ kout, uint32_t* __restrict__ vout) {
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
        lsd_hist_kernel<<<kt, kLsdT, 0, c.stream>>>(kk[cur], n, shift, hist, kt);
        lsd_scan_kernel<<<1, 1024, 0, c.stream>>>(hist, kt);
        lsd_scatter_kernel<<<kt, kLsdT, 0, c.stream>>>(kk[cur], vv[cur], n, shift, hist, kt, kk[cur ^ 1], vv[cur ^ 1]);
        cur ^= 1;
        note_launches(3);
    }
    if (cur) {
        cudaMemcpyAsync(keys, k2, 8 * size_t(n), cudaMemcpyDeviceToDevice, c.stream);
        cudaMemcpyAsync(vals, v2, 4 * size_t(n), cudaMemcpyDeviceToDevice, c.stream);
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
        lsd_hist_kernel<<<kt, kLsdT, 0, c.stream>>>(sk[cur], k, shift, lsd_hist, kt);
        lsd_scan_kernel<<<1, 1024, 0, c.stream>>>(lsd_hist, kt);
        lsd_scatter_kernel<<<kt, kLsdT, 0, c.stream>>>(sk[cur], sv[cur], k, shift, lsd_hist, kt, sk[cur ^ 1],
                                                        sv[cur ^ 1]);
        cur ^= 1;
        note_launches(3);
    }
    const int tg = int((k + 255) / 256 < 1024 ? (k + 255) / 256 : 1024);
    widen_kernel<<<tg, 256, 0, c.stream>>>(sv[cur], k, d_idx);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace etune_b200
