// Selection: the k lowest predictions under the total order (score asc, index asc).
//
// topk (no host synchronisation, everything decided on the device):
//   1. prep      order-preserving 64-bit keys + AND/OR of all keys (which bits vary)
//   2. hist      2048-bin histogram of the top 11 varying bits
//   3. pick      one CTA: bucket d1 that holds the k-th key
//   4. gather    keys of bucket d1 -> small buffer
//   5. refine    one CTA: radix-select the exact k-th key T inside the bucket;
//                need = k - #(key < T)   (ties at T are taken by ascending index)
//   6. count     per tile: #(key < T), #(key == T)
//   7. offsets   one CTA: exclusive scans over tiles
//   8. scatter   stable compaction -> exactly k (key, index) pairs in index order
//   9. order     sort the k pairs by (key, index): one-CTA bitonic for k <= 4096,
//                else the stable LSD radix sort below (k is known on the host)
// Warp-aggregated shared-memory atomics (__match_any_sync) keep heavily tied
// predictions (thousands tie at the k-th value) from serialising.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace etune_b200 {

namespace {

constexpr int kT = 512;            // threads per CTA for streaming kernels
constexpr int kTile = 4096;        // items per tile (count/scatter, LSD sort)
constexpr int kBins = 2048;        // 11-bit digits
constexpr int kSmallSort = 4096;   // one-CTA bitonic bound

__device__ __forceinline__ uint64_t order_key(double x) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct TopkState {
    unsigned long long andor[2];
    unsigned long long T;        // exact k-th key
    unsigned int hist[kBins];
    unsigned int d1;             // bucket of the k-th key
    unsigned int below1;         // #keys in buckets < d1
    unsigned int bucket_n;       // gathered keys
    unsigned int below;          // #(key < T)
    unsigned int need;           // #(key == T) to take, lowest indices first
    int shift;                   // digit = (key >> shift) & 2047
    unsigned int pad[2];
};

// warp-aggregated shared atomic add of 1 to bin[d]
__device__ __forceinline__ void agg_inc(unsigned int* bin, unsigned d, bool valid) {
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const unsigned peers = __match_any_sync(act, d);
    if ((__ffs(peers) - 1) == int(threadIdx.x & 31)) atomicAdd(&bin[d], unsigned(__popc(peers)));
}

__global__ void __launch_bounds__(kT) prep_kernel(const double* __restrict__ score, int64_t n,
                                                  uint64_t* __restrict__ keys, TopkState* st) {
    uint64_t a = ~0ull, o = 0ull;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = order_key(score[i]);
        keys[i] = k;
        a &= k;
        o |= k;
    }
    for (int s = 16; s > 0; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAnd(&st->andor[0], a);
        atomicOr(&st->andor[1], o);
    }
}

__device__ __forceinline__ int top_shift(const TopkState* st) {
    const uint64_t v = st->andor[0] ^ st->andor[1];
    if (v == 0) return 64;  // all keys equal
    const int hb = 63 - __clzll(static_cast<long long>(v));
    return hb >= 10 ? hb - 10 : 0;
}

__global__ void __launch_bounds__(kT) hist_kernel(const uint64_t* __restrict__ keys, int64_t n, TopkState* st) {
    __shared__ unsigned int h[kBins];
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int shift = top_shift(st);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    const int64_t nr = (n + stride - 1) / stride * stride;  // uniform trip count for the warp collectives
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nr; i += stride) {
        const bool v = i < n;
        const unsigned d = (v && shift < 64) ? unsigned(keys[i] >> shift) & (kBins - 1) : 0u;
        agg_inc(h, d, v);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBins; i += blockDim.x)
        if (h[i]) atomicAdd(&st->hist[i], h[i]);
}

// one CTA of 1024: find the bucket holding the k-th smallest key
__global__ void __launch_bounds__(1024) pick_kernel(int64_t k, TopkState* st) {
    __shared__ unsigned int part[1024];
    const int t = threadIdx.x;
    const unsigned a = st->hist[2 * t], b = st->hist[2 * t + 1];
    part[t] = a + b;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const unsigned v = t >= off ? part[t - off] : 0u;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    const unsigned before = part[t] - a - b;  // exclusive
    const unsigned kk = unsigned(k);
    if (before < kk && before + a >= kk) {
        st->d1 = 2 * t;
        st->below1 = before;
    } else if (before + a < kk && before + a + b >= kk) {
        st->d1 = 2 * t + 1;
        st->below1 = before + a;
    }
    if (t == 0) {
        st->shift = top_shift(st);
        st->bucket_n = 0;
    }
}

__global__ void __launch_bounds__(kT) gather_kernel(const uint64_t* __restrict__ keys, int64_t n, TopkState* st,
                                                    uint64_t* __restrict__ bucket) {
    const int shift = st->shift;
    const unsigned d1 = st->d1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t key = keys[i];
        const unsigned d = shift < 64 ? unsigned(key >> shift) & (kBins - 1) : 0u;
        if (d == d1) bucket[atomicAdd(&st->bucket_n, 1u)] = key;
    }
}

// one CTA: exact k-th key inside the bucket by 8-bit MSB radix select on the bits
// below the first digit.
__global__ void __launch_bounds__(1024) refine_kernel(const uint64_t* __restrict__ bucket, int64_t k, TopkState* st) {
    __shared__ unsigned int h[256];
    __shared__ unsigned long long s_prefix;
    __shared__ unsigned int s_rem, s_dig;
    const int t = threadIdx.x;
    const int shift0 = st->shift;
    const unsigned m = st->bucket_n;
    unsigned long long prefix = 0;  // bits below shift0 fixed so far
    unsigned rem = unsigned(k) - st->below1;  // rank (1-based) of the target within the bucket
    int bit = shift0;                         // next digit covers [bit-8, bit)
    if (shift0 >= 64) {  // all keys identical
        if (t == 0) {
            st->T = st->andor[0];
            st->below = 0;
            st->need = unsigned(k);
        }
        return;
    }
    const unsigned long long high = (st->andor[0] >> shift0 << shift0) |  // constant top bits ...
                                    (static_cast<unsigned long long>(st->d1) << shift0);  // ... + bucket digit
    // note: bits above shift0+11 are constant, so (andor[0] >> shift0 << shift0) keeps them
    unsigned long long fixed_mask = ~0ull << shift0;
    while (bit > 0) {
        const int w = bit >= 8 ? 8 : bit;
        const int lo = bit - w;
        for (int i = t; i < 256; i += blockDim.x) h[i] = 0;
        __syncthreads();
        const unsigned mr = (m + 1023u) / 1024u * 1024u;
        for (unsigned i = t; i < mr; i += blockDim.x) {
            bool v = false;
            unsigned d = 0;
            if (i < m) {
                const uint64_t key = bucket[i];
                v = ((key & fixed_mask) & ~(~0ull << shift0)) == prefix;
                d = unsigned(key >> lo) & ((1u << w) - 1u);
            }
            agg_inc(h, d, v);
        }
        __syncthreads();
        if (t == 0) {
            unsigned c = 0, dsel = 0;
            for (unsigned d = 0; d < (1u << w); ++d) {
                if (c + h[d] >= rem) {
                    dsel = d;
                    break;
                }
                c += h[d];
            }
            s_rem = rem - c;
            s_dig = dsel;
        }
        __syncthreads();
        rem = s_rem;
        prefix |= static_cast<unsigned long long>(s_dig) << lo;
        fixed_mask |= ((1ull << w) - 1ull) << lo;
        bit = lo;
        __syncthreads();
    }
    if (t == 0) {
        const unsigned long long T = (high & (~0ull << shift0)) | prefix;
        st->T = T;
        (void)s_prefix;
    }
    __syncthreads();
    // #bucket keys < T -> below = below1 + that
    __shared__ unsigned int s_lt;
    if (t == 0) s_lt = 0;
    __syncthreads();
    const unsigned long long T = st->T;
    unsigned lt = 0;
    for (unsigned i = t; i < m; i += blockDim.x) lt += bucket[i] < T;
    for (int s = 16; s > 0; s >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, s);
    if ((t & 31) == 0) atomicAdd(&s_lt, lt);
    __syncthreads();
    if (t == 0) {
        st->below = st->below1 + s_lt;
        st->need = unsigned(k) - st->below;
    }
}

__global__ void __launch_bounds__(kT) count_kernel(const uint64_t* __restrict__ keys, int64_t n, const TopkState* st,
                                                   unsigned int* __restrict__ lt_cnt, unsigned int* __restrict__ eq_cnt) {
    const unsigned long long T = st->T;
    unsigned lt = 0, eq = 0;
    const int64_t base = int64_t(blockIdx.x) * kTile;
    for (int r = 0; r < kTile / kT; ++r) {
        const int64_t i = base + r * kT + threadIdx.x;
        if (i < n) {
            const uint64_t key = keys[i];
            lt += key < T;
            eq += key == T;
        }
    }
    for (int s = 16; s > 0; s >>= 1) {
        lt += __shfl_xor_sync(0xffffffffu, lt, s);
        eq += __shfl_xor_sync(0xffffffffu, eq, s);
    }
    __shared__ unsigned int sl[kT / 32], se[kT / 32];
    if ((threadIdx.x & 31) == 0) {
        sl[threadIdx.x >> 5] = lt;
        se[threadIdx.x >> 5] = eq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned a = 0, b = 0;
        for (int w = 0; w < kT / 32; ++w) {
            a += sl[w];
            b += se[w];
        }
        lt_cnt[blockIdx.x] = a;
        eq_cnt[blockIdx.x] = b;
    }
}

// exclusive scan of two u32 arrays of length m (one CTA of 1024, m arbitrary)
__global__ void __launch_bounds__(1024) scan2_kernel(unsigned int* __restrict__ a, unsigned int* __restrict__ b, int m) {
    __shared__ unsigned int pa[1024], pb[1024];
    __shared__ unsigned int carry_a, carry_b;
    const int t = threadIdx.x;
    if (t == 0) carry_a = carry_b = 0;
    __syncthreads();
    for (int base = 0; base < m; base += 1024) {
        const int i = base + t;
        const unsigned va = i < m ? a[i] : 0u, vb = i < m ? b[i] : 0u;
        pa[t] = va;
        pb[t] = vb;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const unsigned xa = t >= off ? pa[t - off] : 0u, xb = t >= off ? pb[t - off] : 0u;
            __syncthreads();
            pa[t] += xa;
            pb[t] += xb;
            __syncthreads();
        }
        if (i < m) {
            a[i] = carry_a + pa[t] - va;
            b[i] = carry_b + pb[t] - vb;
        }
        __syncthreads();
        if (t == 1023) {
            carry_a += pa[1023];
            carry_b += pb[1023];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kT) scatter_sel_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                         const TopkState* st, const unsigned int* __restrict__ lt_off,
                                                         const unsigned int* __restrict__ eq_off,
                                                         uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_idx) {
    const unsigned long long T = st->T;
    const unsigned need = st->need;
    __shared__ unsigned int wl[kT / 32], we[kT / 32];
    __shared__ unsigned int run_l, run_e;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        run_l = lt_off[blockIdx.x];
        run_e = eq_off[blockIdx.x];
    }
    const int64_t base = int64_t(blockIdx.x) * kTile;
    const unsigned ltmask = (1u << lane) - 1u;
    for (int r = 0; r < kTile / kT; ++r) {
        const int64_t i = base + r * kT + threadIdx.x;
        uint64_t key = 0;
        bool islt = false, iseq = false;
        if (i < n) {
            key = keys[i];
            islt = key < T;
            iseq = key == T;
        }
        const unsigned bl = __ballot_sync(0xffffffffu, islt), be = __ballot_sync(0xffffffffu, iseq);
        if (lane == 0) {
            wl[warp] = __popc(bl);
            we[warp] = __popc(be);
        }
        __syncthreads();
        unsigned pl = run_l, pe = run_e;
        for (int w = 0; w < warp; ++w) {
            pl += wl[w];
            pe += we[w];
        }
        pl += __popc(bl & ltmask);
        pe += __popc(be & ltmask);
        if (islt || (iseq && pe < need)) {
            const unsigned pos = pl + (pe < need ? pe : need);
            out_key[pos] = key;
            out_idx[pos] = uint32_t(i);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 0; w < kT / 32; ++w) {
                run_l += wl[w];
                run_e += we[w];
            }
        }
        __syncthreads();
    }
}

// one CTA: bitonic sort of m <= kSmallSort (key, idx) pairs, write idx as int64
__global__ void __launch_bounds__(1024) small_sort_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ idx,
                                                         int m, int64_t* __restrict__ out) {
    __shared__ unsigned long long sk[kSmallSort];
    __shared__ unsigned int si[kSmallSort];
    int P = 1;
    while (P < m) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        sk[i] = i < m ? key[i] : ~0ull;
        si[i] = i < m ? idx[i] : 0xffffffffu;
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
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
    for (int i = threadIdx.x; i < m; i += blockDim.x) out[i] = si[i];
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

struct Scratch {
    TopkState* st;
    uint64_t* keys;
    uint64_t* bucket;
    unsigned int* lt;
    unsigned int* eq;
    uint64_t* sel_key[2];
    uint32_t* sel_idx[2];
    uint32_t* lsd_hist;
};

Scratch carve(void* p, int64_t n, int64_t k) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const int64_t ktiles = (k + kTile - 1) / kTile;
    char* c = static_cast<char*>(p);
    Scratch s;
    s.st = reinterpret_cast<TopkState*>(c);
    c += al256(sizeof(TopkState));
    s.keys = reinterpret_cast<uint64_t*>(c);
    c += al256(8 * size_t(n));
    s.bucket = reinterpret_cast<uint64_t*>(c);
    c += al256(8 * size_t(n));
    s.lt = reinterpret_cast<unsigned int*>(c);
    c += al256(4 * size_t(ntiles));
    s.eq = reinterpret_cast<unsigned int*>(c);
    c += al256(4 * size_t(ntiles));
    for (int b = 0; b < 2; ++b) {
        s.sel_key[b] = reinterpret_cast<uint64_t*>(c);
        c += al256(8 * size_t(k));
        s.sel_idx[b] = reinterpret_cast<uint32_t*>(c);
        c += al256(4 * size_t(k));
    }
    s.lsd_hist = reinterpret_cast<uint32_t*>(c);
    (void)ktiles;
    return s;
}

}  // namespace

size_t topk_scratch_bytes(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    return al256(sizeof(TopkState)) + 2 * al256(8 * size_t(n)) + 2 * al256(4 * size_t(ntiles)) +
           2 * (al256(8 * size_t(n)) + al256(4 * size_t(n))) + al256(4 * 256 * size_t(ntiles));
}

cudaError_t launch_topk(const LaunchCtx& c, const double* d_score, int64_t n, int64_t k, int64_t* d_idx,
                        void* d_scratch) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    Scratch s = carve(d_scratch, n, k);
    const int ntiles = int((n + kTile - 1) / kTile);
    cudaError_t e = cudaMemsetAsync(s.st, 0, sizeof(TopkState), c.stream);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(&s.st->andor[0], 0xff, 8, c.stream);
    if (e != cudaSuccess) return e;
    const int grid = int((n + kT - 1) / kT < int64_t(c.sm_count) * 4 ? (n + kT - 1) / kT : int64_t(c.sm_count) * 4);
    prep_kernel<<<grid, kT, 0, c.stream>>>(d_score, n, s.keys, s.st);
    hist_kernel<<<grid, kT, 0, c.stream>>>(s.keys, n, s.st);
    pick_kernel<<<1, 1024, 0, c.stream>>>(k, s.st);
    gather_kernel<<<grid, kT, 0, c.stream>>>(s.keys, n, s.st, s.bucket);
    refine_kernel<<<1, 1024, 0, c.stream>>>(s.bucket, k, s.st);
    count_kernel<<<ntiles, kT, 0, c.stream>>>(s.keys, n, s.st, s.lt, s.eq);
    scan2_kernel<<<1, 1024, 0, c.stream>>>(s.lt, s.eq, ntiles);
    scatter_sel_kernel<<<ntiles, kT, 0, c.stream>>>(s.keys, n, s.st, s.lt, s.eq, s.sel_key[0], s.sel_idx[0]);
    note_launches(8);
    if (k <= kSmallSort) {
        small_sort_kernel<<<1, 1024, 0, c.stream>>>(s.sel_key[0], s.sel_idx[0], int(k), d_idx);
        note_launches(1);
        return cudaGetLastError();
    }
    // stable LSD sort of the k selected pairs (already in index order) by key
    const int kt = int((k + kTile - 1) / kTile);
    int cur = 0;
    for (int shift = 0; shift < 64; shift += 8) {
        lsd_hist_kernel<<<kt, kLsdT, 0, c.stream>>>(s.sel_key[cur], k, shift, s.lsd_hist, kt);
        lsd_scan_kernel<<<1, 1024, 0, c.stream>>>(s.lsd_hist, kt);
        lsd_scatter_kernel<<<kt, kLsdT, 0, c.stream>>>(s.sel_key[cur], s.sel_idx[cur], k, shift, s.lsd_hist, kt,
                                                        s.sel_key[cur ^ 1], s.sel_idx[cur ^ 1]);
        cur ^= 1;
        note_launches(3);
    }
    const int tg = int((k + 255) / 256 < 1024 ? (k + 255) / 256 : 1024);
    widen_kernel<<<tg, 256, 0, c.stream>>>(s.sel_idx[cur], k, d_idx);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace etune_b200
