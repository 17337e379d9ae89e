// Cost-model scalars on the device: energy_loss (Eq. 1, energy_model.cpp:23-34) per
// sample, and the two sequential sums of snr_db (energy_model.cpp:352-370).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "etune_internal.hpp"
#include "kernels.hpp"

namespace etune_b200 {

namespace {

__global__ void energy_loss_kernel(const double* __restrict__ pred, const double* __restrict__ meas, int64_t n,
                                   double* __restrict__ out, unsigned long long* err) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double m = meas[i];
        if (!(m > 0.0)) {
            atomicMin(err, (static_cast<unsigned long long>(i) << 8) | unsigned(ETUNE_ERR_NON_POSITIVE_ENERGY));
            continue;
        }
        const double d = __dsub_rn(pred[i], m);
        out[3 * i + 0] = __ddiv_rn(__dmul_rn(d, d), m);    // value
        out[3 * i + 1] = __ddiv_rn(__dmul_rn(2.0, d), m);  // gradient
        out[3 * i + 2] = __ddiv_rn(2.0, m);                // hessian
    }
}

// signal = sum m^2, error = sum (p - m)^2, both in index order (one thread: the
// reference's loop is one sequential chain per sum).  Positivity is checked in
// parallel first so the first offending index is reported like the reference's throw.
__global__ void snr_sums_kernel(const double* __restrict__ pred, const double* __restrict__ meas, int64_t n,
                                double* __restrict__ out2, unsigned long long* err) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        if (!(meas[i] > 0.0)) {
            atomicMin(err, (static_cast<unsigned long long>(i) << 8) | unsigned(ETUNE_ERR_NON_POSITIVE_ENERGY));
            bad = 1;
        }
    }
    __syncthreads();
    if (bad || threadIdx.x != 0) return;
    double signal = 0.0, error = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double m = meas[i];
        signal = __dadd_rn(signal, __dmul_rn(m, m));
        const double d = __dsub_rn(pred[i], m);
        error = __dadd_rn(error, __dmul_rn(d, d));
    }
    out2[0] = signal;
    out2[1] = error;
}

__global__ void pack_records_kernel(const double* __restrict__ score, const int64_t* __restrict__ lidx, int64_t kl,
                                    int64_t k, int64_t goff, ShardRec* __restrict__ rec) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < k; j += int64_t(gridDim.x) * blockDim.x) {
        ShardRec r;
        if (j < kl) {
            const int64_t i = lidx[j];
            r.s = score[i];
            r.g = i + goff;
        } else {  // +inf pads sort last
            r.s = __longlong_as_double(0x7ff0000000000000ll);
            r.g = 0x7fffffffffffffffll;
        }
        rec[j] = r;
    }
}

__device__ __forceinline__ uint64_t rec_key(double x) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Merge of W sorted lists (rank-major, k records each) keeping the first k.  The lists come from
// ranks owning ascending, disjoint global index ranges, so the (score, global index) order is the
// (score key, list, position) order: a record at position j of list w has rank
//   j + sum over lists w' < w of #(keys <= its key) + sum over lists w' > w of #(keys < its key),
// each count one binary search.  Every CTA stages the W * k keys in shared memory (16-byte record
// loads, all in flight); a record gets TPR = pow2 >= W threads, thread v of them searches list v,
// and the counts meet by shuffles -- one binary search of latency per record instead of W - 1 in
// sequence.  CTAs split the W * k records (1024 / TPR per CTA); ranks < k are written.
__device__ __forceinline__ uint32_t count_le(const uint64_t* a, uint32_t n, uint64_t x) {  // upper_bound
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint32_t count_lt(const uint64_t* a, uint32_t n, uint64_t x) {  // lower_bound
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(1024) merge_records_kernel(const ShardRec* __restrict__ rec, int W, int k, int tpr,
                                                             int64_t* __restrict__ idx, double* __restrict__ sc) {
    extern __shared__ unsigned long long msm[];
    uint64_t* keys = reinterpret_cast<uint64_t*>(msm);  // [W][k]
    const int tot = W * k;
    const double2* r2 = reinterpret_cast<const double2*>(rec);  // {score, index bits}
    for (int base = 0; base < tot; base += 8 * int(blockDim.x)) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + u * int(blockDim.x) + int(threadIdx.x);
            v[u] = i < tot ? __ldg(r2 + i).x : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + u * int(blockDim.x) + int(threadIdx.x);
            if (i < tot) keys[i] = rec_key(v[u]);
        }
    }
    __syncthreads();
    const int per_cta = int(blockDim.x) / tpr;
    const int sub = int(threadIdx.x) % tpr;                          // the list this thread searches
    const int g = blockIdx.x * per_cta + int(threadIdx.x) / tpr;     // record (list-major)
    const bool valid = g < tot;
    const int w = valid ? g / k : 0, j = valid ? g - w * k : 0;
    const uint64_t x = valid ? keys[g] : 0ull;
    uint32_t cnt = 0;
    for (int v = sub; valid && v < W; v += tpr) {
        if (v == w) continue;
        cnt += v < w ? count_le(keys + v * k, uint32_t(k), x) : count_lt(keys + v * k, uint32_t(k), x);
    }
    for (int o = tpr >> 1; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);  // tpr <= 32 lanes
    const uint32_t r = cnt + uint32_t(j);
    if (valid && sub == 0 && r < uint32_t(k)) {
        const ShardRec q = rec[g];
        idx[r] = q.g;
        if (sc) sc[r] = q.s;
    }
}

__global__ void merge_keys_kernel(const ShardRec* __restrict__ rec, int64_t tot, uint64_t* __restrict__ key,
                                  uint32_t* __restrict__ pos) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < tot; i += int64_t(gridDim.x) * blockDim.x) {
        key[i] = rec_key(rec[i].s);
        pos[i] = uint32_t(i);
    }
}

// the same ranking with the keys in global memory (W * k beyond shared memory): one thread per record
__global__ void merge_rank_kernel(const ShardRec* __restrict__ rec, const uint64_t* __restrict__ keys, int W, int k,
                                  int64_t* __restrict__ idx, double* __restrict__ sc) {
    const int64_t tot = int64_t(W) * k;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < tot; i += int64_t(gridDim.x) * blockDim.x) {
        const int w = int(i / k), j = int(i - int64_t(w) * k);
        const uint64_t x = keys[i];
        uint32_t r = uint32_t(j);
        for (int d = 1; d < W && r < uint32_t(k); ++d) {
            const int v = (w + d) % W;
            r += v < w ? count_le(keys + int64_t(v) * k, uint32_t(k), x) : count_lt(keys + int64_t(v) * k, uint32_t(k), x);
        }
        if (r < uint32_t(k)) {
            idx[r] = rec[i].g;
            if (sc) sc[r] = rec[i].s;
        }
    }
}

__global__ void gather_u64_kernel(const uint64_t* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                                  uint64_t* __restrict__ dst) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        dst[j] = src[idx[j]];
}

__global__ void div_scalar_kernel(const double* __restrict__ x, int64_t n, const double* __restrict__ d,
                                  double* __restrict__ y) {
    const double v = *d;
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        y[j] = __ddiv_rn(x[j], v);
}

}  // namespace

cudaError_t launch_gather_u64(const LaunchCtx& c, const void* d_src, const int64_t* d_idx, int64_t n, void* d_dst) {
    if (n <= 0) return cudaSuccess;
    const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
    gather_u64_kernel<<<grid, 256, 0, c.stream>>>(static_cast<const uint64_t*>(d_src), d_idx, n,
                                                  static_cast<uint64_t*>(d_dst));
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_div_scalar(const LaunchCtx& c, const double* d_x, int64_t n, const double* d_divisor, double* d_y) {
    if (n <= 0) return cudaSuccess;
    const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
    div_scalar_kernel<<<grid, 256, 0, c.stream>>>(d_x, n, d_divisor, d_y);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_pack_records(const LaunchCtx& c, const double* d_score, const int64_t* d_lidx, int64_t kl,
                                int64_t k, int64_t goff, ShardRec* d_rec) {
    const int grid = int(std::min<int64_t>((k + 255) / 256, 1024));
    pack_records_kernel<<<grid, 256, 0, c.stream>>>(d_score, d_lidx, kl, k, goff, d_rec);
    note_launches(1);
    return cudaGetLastError();
}

size_t merge_scratch_bytes(int W, int64_t k) { return size_t(W) * size_t(k) * 24 + 512; }

cudaError_t launch_merge_records(const LaunchCtx& c, const ShardRec* d_rec, int W, int64_t k, int64_t* d_idx,
                                 double* d_sc, void* d_scratch) {
    if (k <= 0 || W <= 0) return cudaSuccess;
    const int64_t tot = int64_t(W) * k;
    const size_t smem = size_t(tot) * 8;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem <= size_t(optin)) {
        static size_t attr = 0;
        if (smem > attr) {
            const cudaError_t e =
                cudaFuncSetAttribute(merge_records_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(optin));
            if (e != cudaSuccess) return e;
            attr = size_t(optin);
        }
        int tpr = 1;
        while (tpr < W && tpr < 32) tpr <<= 1;
        const int per_cta = 1024 / tpr;
        merge_records_kernel<<<int((tot + per_cta - 1) / per_cta), 1024, smem, c.stream>>>(d_rec, W, int(k), tpr,
                                                                                          d_idx, d_sc);
        note_launches(1);
        return cudaGetLastError();
    }
    uint64_t* keys = static_cast<uint64_t*>(d_scratch);
    const int grid = int(std::min<int64_t>((tot + 255) / 256, int64_t(c.sm_count) * 8));
    merge_keys_kernel<<<grid, 256, 0, c.stream>>>(d_rec, tot, keys, reinterpret_cast<uint32_t*>(keys + tot));
    merge_rank_kernel<<<grid, 256, 0, c.stream>>>(d_rec, keys, W, int(k), d_idx, d_sc);
    note_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_energy_loss(const LaunchCtx& c, const double* d_pred, const double* d_meas, int64_t n,
                               double* d_out3) {
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const int grid = int(want < int64_t(c.sm_count) * 8 ? want : int64_t(c.sm_count) * 8);
    energy_loss_kernel<<<grid, 256, 0, c.stream>>>(d_pred, d_meas, n, d_out3, c.d_err);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_snr_sums(const LaunchCtx& c, const double* d_pred, const double* d_meas, int64_t n,
                            double* d_out2) {
    snr_sums_kernel<<<1, 1024, 0, c.stream>>>(d_pred, d_meas, n, d_out2, c.d_err);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace etune_b200
