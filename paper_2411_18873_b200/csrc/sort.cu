// Selection: the k lowest predictions under (score asc, index asc).
//
// Stable LSD radix sort of (order-preserving 64-bit key, u32 index) pairs over
// 8-bit digits, skipping digits that are constant across the batch (predictions of
// one operator share sign/exponent bits, so typically 6-7 of 8 passes run).  Each
// pass: per-tile histogram -> one-CTA exclusive scan in (digit, tile) order ->
// per-tile stable scatter with warp-level __match_any_sync ranking.  Stability of
// every pass plus an index-ordered start gives exactly the (score, index) order.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace etune_b200 {

namespace {

constexpr int kSortThreads = 512;
constexpr int kTile = 4096;
constexpr int kRounds = kTile / kSortThreads;
constexpr int kWarps = kSortThreads / 32;

__device__ __forceinline__ uint64_t order_key(double x) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(kSortThreads) prep_kernel(const double* __restrict__ score, int64_t n,
                                                            uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                            unsigned long long* andor) {
    uint64_t a = ~0ull, o = 0ull;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = order_key(score[i]);
        keys[i] = k;
        vals[i] = uint32_t(i);
        a &= k;
        o |= k;
    }
    for (int s = 16; s > 0; s >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, s);
        o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAnd(andor, a);
        atomicOr(andor + 1, o);
    }
}

__global__ void __launch_bounds__(kSortThreads) hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                            uint32_t* __restrict__ hist, int ntiles) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * kTile;
    for (int r = 0; r < kRounds; ++r) {
        const int64_t i = base + r * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[int64_t(d) * ntiles + blockIdx.x] = h[d];
}

// exclusive scan of hist[0..total) in place (one CTA)
__global__ void __launch_bounds__(1024) scan_kernel(uint32_t* __restrict__ hist, int64_t total) {
    __shared__ uint32_t part[1024];
    const int64_t per = (total + blockDim.x - 1) / blockDim.x;
    const int64_t lo = threadIdx.x * per;
    const int64_t hi = lo + per < total ? lo + per : total;
    uint32_t s = 0;
    for (int64_t i = lo; i < hi; ++i) s += hist[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t v = threadIdx.x >= unsigned(off) ? part[threadIdx.x - off] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = part[threadIdx.x] - s;
    for (int64_t i = lo; i < hi; ++i) {
        const uint32_t c = hist[i];
        hist[i] = run;
        run += c;
    }
}

__global__ void __launch_bounds__(kSortThreads) scatter_kernel(const uint64_t* __restrict__ kin,
                                                               const uint32_t* __restrict__ vin, int64_t n, int shift,
                                                               const uint32_t* __restrict__ offs, int ntiles,
                                                               uint64_t* __restrict__ kout, uint32_t* __restrict__ vout) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t gofs[256];
    __shared__ uint32_t wc[kWarps][257];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int d = tid; d < 256; d += blockDim.x) {
        base[d] = 0;
        gofs[d] = offs[int64_t(d) * ntiles + blockIdx.x];
    }
    const unsigned lt = (1u << lane) - 1u;
    const int64_t tbase = int64_t(blockIdx.x) * kTile;
    for (int r = 0; r < kRounds; ++r) {
        for (int j = tid; j < kWarps * 257; j += blockDim.x) (&wc[0][0])[j] = 0;
        __syncthreads();
        const int64_t i = tbase + r * kSortThreads + tid;
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
            for (int w = 0; w < kWarps; ++w) {
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

__global__ void take_kernel(const uint32_t* __restrict__ vals, int64_t k, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < k; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = vals[i];
}

struct Scratch {
    uint64_t* keys[2];
    uint32_t* vals[2];
    uint32_t* hist;
    unsigned long long* andor;
};

Scratch carve(void* p, int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char* c = static_cast<char*>(p);
    Scratch s;
    s.keys[0] = reinterpret_cast<uint64_t*>(c);
    c += al(8 * size_t(n));
    s.keys[1] = reinterpret_cast<uint64_t*>(c);
    c += al(8 * size_t(n));
    s.vals[0] = reinterpret_cast<uint32_t*>(c);
    c += al(4 * size_t(n));
    s.vals[1] = reinterpret_cast<uint32_t*>(c);
    c += al(4 * size_t(n));
    s.hist = reinterpret_cast<uint32_t*>(c);
    c += al(4 * size_t(256 * ntiles));
    s.andor = reinterpret_cast<unsigned long long*>(c);
    return s;
}

}  // namespace

size_t topk_scratch_bytes(int64_t n) {
    const int64_t ntiles = (n + kTile - 1) / kTile;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    return 2 * al(8 * size_t(n)) + 2 * al(4 * size_t(n)) + al(4 * size_t(256 * ntiles)) + 256;
}

cudaError_t launch_topk(const LaunchCtx& c, const double* d_score, int64_t n, int64_t k, int64_t* d_idx,
                        void* d_scratch) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    Scratch s = carve(d_scratch, n);
    const int ntiles = int((n + kTile - 1) / kTile);
    unsigned long long init[2] = {~0ull, 0ull};
    cudaError_t e = cudaMemcpyAsync(s.andor, init, sizeof(init), cudaMemcpyHostToDevice, c.stream);
    if (e != cudaSuccess) return e;
    int grid = int((n + kSortThreads - 1) / kSortThreads);
    if (grid > c.sm_count * 4) grid = c.sm_count * 4;
    prep_kernel<<<grid, kSortThreads, 0, c.stream>>>(d_score, n, s.keys[0], s.vals[0], s.andor);
    note_launches(1);
    unsigned long long andor[2];
    e = cudaMemcpyAsync(andor, s.andor, sizeof(andor), cudaMemcpyDeviceToHost, c.stream);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(c.stream);
    if (e != cudaSuccess) return e;
    const uint64_t varying = andor[0] ^ andor[1];
    int cur = 0;
    for (int shift = 0; shift < 64; shift += 8) {
        if (((varying >> shift) & 0xffu) == 0) continue;
        hist_kernel<<<ntiles, kSortThreads, 0, c.stream>>>(s.keys[cur], n, shift, s.hist, ntiles);
        scan_kernel<<<1, 1024, 0, c.stream>>>(s.hist, int64_t(256) * ntiles);
        scatter_kernel<<<ntiles, kSortThreads, 0, c.stream>>>(s.keys[cur], s.vals[cur], n, shift, s.hist, ntiles,
                                                               s.keys[cur ^ 1], s.vals[cur ^ 1]);
        cur ^= 1;
        note_launches(3);
    }
    const int tg = int((k + 255) / 256 < 1024 ? (k + 255) / 256 : 1024);
    take_kernel<<<tg, 256, 0, c.stream>>>(s.vals[cur], k, d_idx);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace etune_b200
