// Diagnostic: dependent FP64 add latency on this GPU (cycles per element), operands in
// registers, one chain vs two interleaved chains in one thread vs two warps.
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void chain(const double* __restrict__ g, int n, double* out, long long* cyc) {
    double x[8];
    for (int u = 0; u < 8; ++u) x[u] = g[u + threadIdx.x];
    double r0 = 0.0, r1 = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            r0 = __dadd_rn(r0, x[u]);
            if (CHAINS == 2) r1 = __dadd_rn(r1, x[7 - u]);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = r0 + r1;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double *g, *o; long long* c; cudaMalloc(&g, 4096); cudaMalloc(&o, 4096); cudaMalloc(&c, 16);
    cudaMemset(g, 0, 4096);
    const int n = 1 << 20; long long hc;
    chain<1><<<1, 1>>>(g, n, o, c); cudaDeviceSynchronize();
    chain<1><<<1, 1>>>(g, n, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("one chain, 1 thread: %.2f cycles/add\n", double(hc) / n);
    chain<2><<<1, 1>>>(g, n, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("two chains, 1 thread: %.2f cycles/element (2 adds)\n", double(hc) / n);
    chain<1><<<1, 64>>>(g, n, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("one chain, 2 warps (same SMSP?): %.2f cycles/add\n", double(hc) / n);
    chain<1><<<1, 128>>>(g, n, o, c); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("one chain, 4 warps: %.2f cycles/add\n", double(hc) / n);
}
