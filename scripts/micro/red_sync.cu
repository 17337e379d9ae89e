// Cost of a grid barrier right after every CTA issued reductions (RED) to shared counters:
// 148 CTAs x 1024 threads, back-to-back launches, us per launch.
//   none        barrier only
//   1 addr      one RED per CTA to one word
//   64 padded   64 REDs per CTA, one word per 128-byte line (the super-segment counters)
//   64 dense    64 REDs per CTA to 64 consecutive words
//   4096 dense  4096 REDs per CTA (4 per thread, consecutive words: the segment histogram)
//   4096 strided  the same, thread t owning words 4t..4t+3
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_sync red_sync.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void red_kernel(uint32_t* buf, int mode) {
    const int t = threadIdx.x;
    if (mode == 1 && t == 0) atomicAdd(buf, 1u);
    if (mode == 2 && t < 64) atomicAdd(buf + t * 32, 1u);
    if (mode == 3 && t < 64) atomicAdd(buf + t, 1u);
    if (mode == 4)
        for (int i = t; i < 4096; i += 1024) atomicAdd(buf + i, 1u);
    if (mode == 5)
        for (int i = 0; i < 4; ++i) atomicAdd(buf + 4 * t + i, 1u);
    cg::this_grid().sync();
}

int main() {
    uint32_t* buf;
    cudaMalloc(&buf, 1 << 20);
    cudaMemset(buf, 0, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[6] = {"none", "1 addr", "64 padded", "64 dense", "4096 dense", "4096 strided"};
    for (int mode = 0; mode < 6; ++mode) {
        void* args[] = {&buf, &mode};
        for (int i = 0; i < 10; ++i) cudaLaunchCooperativeKernel((void*)red_kernel, 148, 1024, args, 0, 0);
        cudaEventRecord(a);
        for (int i = 0; i < 200; ++i) cudaLaunchCooperativeKernel((void*)red_kernel, 148, 1024, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-14s %7.2f us/launch (%s)\n", names[mode], ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
