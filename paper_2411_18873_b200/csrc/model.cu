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

// Merge of W sorted lists (rank-major, k records each) keeping the first k: the lists come from
// ranks owning ascending, disjoint global index ranges, so (score, global index) order equals
// (score key, position in the concatenation) order and the comparison needs no 64-bit index.
// log2(W) rounds of pairwise merge-path merges (co-rank binary search per output) in shared
// memory, ping-pong between two halves; one CTA.
struct MergeView {
    uint64_t* key;
    uint32_t* pos;
};

__device__ __forceinline__ bool mless(const MergeView& v, uint32_t a, uint32_t b) {
    return v.key[a] < v.key[b] || (v.key[a] == v.key[b] && v.pos[a] < v.pos[b]);
}

// element q (< k) of merge(A, B), A = [a0, a0 + k), B = [b0, b0 + k)
__device__ __forceinline__ uint32_t merge_at(const MergeView& v, uint32_t a0, uint32_t b0, uint32_t k, uint32_t q) {
    uint32_t lo = 0, hi = q;  // elements of A among the first q outputs
    while (lo < hi) {
        const uint32_t i = (lo + hi) >> 1, j = q - i;
        if (j > 0 && mless(v, a0 + i, b0 + j - 1)) lo = i + 1;
        else hi = i;
    }
    const uint32_t i = lo, j = q - lo;
    const bool take_a = j >= k || (i < k && mless(v, a0 + i, b0 + j));
    return take_a ? a0 + i : b0 + j;
}

__global__ void __launch_bounds__(1024, 1) merge_records_kernel(const ShardRec* __restrict__ rec, int W, int k,
                                                                int64_t* __restrict__ idx, double* __restrict__ sc) {
    extern __shared__ unsigned long long msm[];
    const int tot = W * k;
    MergeView v[2];
    v[0].key = reinterpret_cast<uint64_t*>(msm);
    v[1].key = v[0].key + tot;
    v[0].pos = reinterpret_cast<uint32_t*>(v[1].key + tot);
    v[1].pos = v[0].pos + tot;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) {
        v[0].key[i] = rec_key(rec[i].s);
        v[0].pos[i] = uint32_t(i);
    }
    __syncthreads();
    int cur = 0, L = W;
    while (L > 1) {
        const int pairs = L >> 1;
        const MergeView& a = v[cur];
        MergeView& b = v[cur ^ 1];
        for (int t = threadIdx.x; t < pairs * k; t += blockDim.x) {
            const int pr = t / k, q = t - pr * k;
            const uint32_t src = merge_at(a, uint32_t(2 * pr * k), uint32_t((2 * pr + 1) * k), uint32_t(k), uint32_t(q));
            b.key[pr * k + q] = a.key[src];
            b.pos[pr * k + q] = a.pos[src];
        }
        if (L & 1)  // the odd list moves down unchanged
            for (int t = threadIdx.x; t < k; t += blockDim.x) {
                b.key[pairs * k + t] = a.key[(L - 1) * k + t];
                b.pos[pairs * k + t] = a.pos[(L - 1) * k + t];
            }
        __syncthreads();
        cur ^= 1;
        L = pairs + (L & 1);
    }
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        const ShardRec r = rec[v[cur].pos[t]];
        idx[t] = r.g;
        if (sc) sc[t] = r.s;
    }
}

// the same merge round by round in global memory (W * k beyond shared memory): one launch per round
__global__ void merge_round_kernel(const uint64_t* __restrict__ ka, const uint32_t* __restrict__ pa, int L, int k,
                                   uint64_t* __restrict__ kb, uint32_t* __restrict__ pb) {
    const MergeView a{const_cast<uint64_t*>(ka), const_cast<uint32_t*>(pa)};
    const int pairs = L >> 1;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < int64_t(pairs + (L & 1)) * k;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int pr = int(t / k), q = int(t - int64_t(pr) * k);
        uint32_t src;
        if (pr < pairs) src = merge_at(a, uint32_t(2 * pr * k), uint32_t((2 * pr + 1) * k), uint32_t(k), uint32_t(q));
        else src = uint32_t((L - 1) * k + q);
        kb[t] = ka[src];
        pb[t] = pa[src];
    }
}

__global__ void merge_keys_kernel(const ShardRec* __restrict__ rec, int64_t tot, uint64_t* __restrict__ key,
                                  uint32_t* __restrict__ pos) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < tot; i += int64_t(gridDim.x) * blockDim.x) {
        key[i] = rec_key(rec[i].s);
        pos[i] = uint32_t(i);
    }
}

__global__ void merge_out_kernel(const ShardRec* __restrict__ rec, const uint32_t* __restrict__ pos, int k,
                                 int64_t* __restrict__ idx, double* __restrict__ sc) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < k; t += gridDim.x * blockDim.x) {
        const ShardRec r = rec[pos[t]];
        idx[t] = r.g;
        if (sc) sc[t] = r.s;
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
    const size_t smem = size_t(tot) * 24;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem <= size_t(optin) && tot < (int64_t(1) << 31)) {
        static size_t attr = 0;
        if (smem > attr) {
            const cudaError_t e =
                cudaFuncSetAttribute(merge_records_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(optin));
            if (e != cudaSuccess) return e;
            attr = size_t(optin);
        }
        merge_records_kernel<<<1, 1024, smem, c.stream>>>(d_rec, W, int(k), d_idx, d_sc);
        note_launches(1);
        return cudaGetLastError();
    }
    uint64_t* k0 = static_cast<uint64_t*>(d_scratch);
    uint64_t* k1 = k0 + tot;
    uint32_t* p0 = reinterpret_cast<uint32_t*>(k1 + tot);
    uint32_t* p1 = p0 + tot;
    const int grid = int(std::min<int64_t>((tot + 255) / 256, int64_t(c.sm_count) * 8));
    merge_keys_kernel<<<grid, 256, 0, c.stream>>>(d_rec, tot, k0, p0);
    int L = W, launches = 2;
    uint64_t* kk[2] = {k0, k1};
    uint32_t* pp[2] = {p0, p1};
    int cur = 0;
    while (L > 1) {
        merge_round_kernel<<<grid, 256, 0, c.stream>>>(kk[cur], pp[cur], L, int(k), kk[cur ^ 1], pp[cur ^ 1]);
        cur ^= 1;
        L = (L >> 1) + (L & 1);
        ++launches;
    }
    merge_out_kernel<<<int((k + 255) / 256), 256, 0, c.stream>>>(d_rec, pp[cur], int(k), d_idx, d_sc);
    note_launches(launches);
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
