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
                                    int64_t k, int64_t goff, double* __restrict__ rs, int64_t* __restrict__ rg) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < k; j += int64_t(gridDim.x) * blockDim.x) {
        if (j < kl) {
            const int64_t i = lidx[j];
            rs[j] = score[i];
            rg[j] = i + goff;
        } else {
            rs[j] = __longlong_as_double(0x7ff0000000000000ll);  // +inf pads sort last
            rg[j] = 0x7fffffffffffffffll;
        }
    }
}

__global__ void gather_records_kernel(const double* __restrict__ gs, const int64_t* __restrict__ gg,
                                      const int64_t* __restrict__ pos, int64_t k, int64_t* __restrict__ idx,
                                      double* __restrict__ sc) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < k; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = pos[j];
        idx[j] = gg[p];
        if (sc) sc[j] = gs[p];
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
                                int64_t k, int64_t goff, double* d_rs, int64_t* d_rg) {
    const int grid = int(std::min<int64_t>((k + 255) / 256, 1024));
    pack_records_kernel<<<grid, 256, 0, c.stream>>>(d_score, d_lidx, kl, k, goff, d_rs, d_rg);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_gather_records(const LaunchCtx& c, const double* d_gs, const int64_t* d_gg, const int64_t* d_pos,
                                  int64_t k, int64_t* d_idx, double* d_sc) {
    const int grid = int(std::min<int64_t>((k + 255) / 256, 1024));
    gather_records_kernel<<<grid, 256, 0, c.stream>>>(d_gs, d_gg, d_pos, k, d_idx, d_sc);
    note_launches(1);
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
