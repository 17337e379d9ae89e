// Pure-store floor on the B200: 2^20 x 136 B (the feature mode's outputs) written with 16-byte
// streaming stores, 8 buffers cycled; plus a read+write copy of the same size.  us per launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_floor write_floor.cu
#include <cstdint>
#include <cstdio>
__global__ void wr(double2* __restrict__ o, int64_t n2) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x)
        __stcs(o + i, make_double2(double(i), 1.0));
}
__global__ void cp(const double2* __restrict__ a, double2* __restrict__ o, int64_t n2) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x)
        __stcs(o + i, __ldcs(a + i));
}
int main() {
    const int64_t bytes = int64_t(136) << 20, n2 = bytes / 16;
    double2* b[8];
    for (auto& x : b) cudaMalloc(&x, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid : {148 * 4, 148 * 8, 148 * 16, 148 * 64}) {
        for (int i = 0; i < 5; ++i) wr<<<grid, 256>>>(b[i % 8], n2);
        cudaEventRecord(e0);
        for (int i = 0; i < 40; ++i) wr<<<grid, 256>>>(b[i % 8], n2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("write 136 MB grid %5d: %7.1f us  %6.0f GB/s\n", grid, ms * 1e3 / 40, bytes / (ms / 40 * 1e-3) / 1e9);
    }
    for (int grid : {148 * 8, 148 * 64}) {
        for (int i = 0; i < 5; ++i) cp<<<grid, 256>>>(b[i % 8], b[(i + 1) % 8], n2 / 2);
        cudaEventRecord(e0);
        for (int i = 0; i < 40; ++i) cp<<<grid, 256>>>(b[i % 8], b[(i + 1) % 8], n2 / 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("copy 68+68 MB grid %5d: %7.1f us  %6.0f GB/s\n", grid, ms * 1e3 / 40, bytes / (ms / 40 * 1e-3) / 1e9);
    }
    return 0;
}
