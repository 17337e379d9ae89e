// Three-phase exclusive scan over n items given by a functor (tile sums -> one-CTA
// scan of the tile sums -> per-item apply with the exclusive prefix).  Header-only;
// everything has internal linkage per translation unit.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "pdl.cuh"

namespace etune_b200 {
namespace {

// exclusive scan helpers (three-phase, 1024-wide tiles)
constexpr int kScanT = 1024;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
    __shared__ int64_t ws[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
    for (int s = 1; s < 32; s <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, s);
        if (lane >= s) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    int64_t before = 0, tot = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) {
        if (i < wid) before += ws[i];
        tot += ws[i];
    }
    __syncthreads();
    *total = tot;
    return before + x - v;
}

template <typename F>
__global__ void __launch_bounds__(kScanT) tile_sums_kernel(int64_t n, F f, int64_t* __restrict__ sums) {
    pdl_wait();
    const int64_t i = blockIdx.x * int64_t(kScanT) + threadIdx.x;
    int64_t tot;
    block_excl_scan(i < n ? f(i) : 0, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) scan_sums_kernel(int64_t* __restrict__ sums, int64_t nt,
                                                           int64_t* __restrict__ total) {
    pdl_wait();
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < nt; b += kScanT) {
        const int64_t i = b + threadIdx.x;
        const int64_t v = i < nt ? sums[i] : 0;
        int64_t tot;
        const int64_t ex = block_excl_scan(v, &tot);
        if (i < nt) sums[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// out(i, exclusive prefix) for every i
template <typename F, typename G>
__global__ void __launch_bounds__(kScanT) tile_apply_kernel(int64_t n, F f, const int64_t* __restrict__ sums, G g) {
    pdl_wait();
    const int64_t i = blockIdx.x * int64_t(kScanT) + threadIdx.x;
    int64_t tot;
    const int64_t ex = block_excl_scan(i < n ? f(i) : 0, &tot);
    if (i < n) g(i, sums[blockIdx.x] + ex);
}

template <typename F, typename G>
cudaError_t scan_apply(cudaStream_t st, int64_t n, F f, G g, int64_t* sums, int64_t* total) {
    const int64_t nt = (n + kScanT - 1) / kScanT;
    if (nt == 0) {
        cudaMemsetAsync(total, 0, 8, st);
        return cudaGetLastError();
    }
    // programmatic dependent launches: each kernel waits (pdl_wait) before reading
    cudaError_t e = launch_pdl(tile_sums_kernel<F>, dim3(unsigned(nt)), dim3(kScanT), 0, st, n, f, sums);
    if (e == cudaSuccess) e = launch_pdl(scan_sums_kernel, dim3(1), dim3(kScanT), 0, st, sums, nt, total);
    if (e == cudaSuccess)
        e = launch_pdl(tile_apply_kernel<F, G>, dim3(unsigned(nt)), dim3(kScanT), 0, st, n, f, sums, g);
    note_launches(3);
    return e;
}

}  // namespace
}  // namespace etune_b200
