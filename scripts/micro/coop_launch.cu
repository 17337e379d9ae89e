// Back-to-back launch cost on the B200: regular vs cooperative launches of an empty kernel of the
// fused selection's shape (293 CTAs x 512 threads), with and without 100 KB of dynamic shared
// memory, and with 1-3 grid barriers.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 coop_launch.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
template <int S>
__global__ void sync_kernel(int* p) {
    for (int s = 0; s < S; ++s) cg::this_grid().sync();
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
int main() {
    int* d = nullptr;
    cudaMalloc(&d, 4);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int G = 293, T = 512, R = 200;
    auto run = [&](const char* name, auto fn) {
        for (int i = 0; i < 10; ++i) fn();
        cudaEventRecord(a, st);
        for (int i = 0; i < R; ++i) fn();
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %8.2f us/launch  (%s)\n", name, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
    };
    for (size_t smem : {size_t(0), size_t(100 * 1024)}) {
        cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(sync_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(sync_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        printf("dynamic smem %zu\n", smem);
        run("regular empty", [&] { empty_kernel<<<G, T, smem, st>>>(d); });
        void* args[] = {&d};
        run("cooperative empty", [&] {
            cudaLaunchCooperativeKernel((void*)empty_kernel, G, T, args, smem, st);
        });
        run("cooperative 1 grid sync", [&] {
            cudaLaunchCooperativeKernel((void*)sync_kernel<1>, G, T, args, smem, st);
        });
        run("cooperative 3 grid syncs", [&] {
            cudaLaunchCooperativeKernel((void*)sync_kernel<3>, G, T, args, smem, st);
        });
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = G;
        cfg.blockDim = T;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        run("regular empty + PDL attribute", [&] { cudaLaunchKernelEx(&cfg, empty_kernel, d); });
    }
    return 0;
}
