// Floor of the score+select step on the B200: back-to-back cost of
//   - empty kernels (regular / cooperative, 148 x 1024 threads, with the step's dynamic smem),
//   - grid barriers (cooperative_groups vs a one-atomic-per-CTA sense barrier),
//   - a pure stream of the step's HBM traffic (8 B in, 16 B out per candidate, 2^20 candidates),
//   - the same stream plus one dependent 16-byte gather from a 1.35 MB table (L2-resident).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_floor step_floor.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void empty_kernel(int* p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
template <int S>
__global__ void cg_sync_kernel(int* p) {
    for (int s = 0; s < S; ++s) cg::this_grid().sync();
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
// one atomic per CTA, everyone polls one word (generation counter)
__device__ __forceinline__ void my_grid_sync(unsigned* bar, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned gen;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
        __threadfence();
        const unsigned t = atomicAdd(bar, 1u);
        if (t == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
        } else {
            unsigned g2;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g2) : "l"(bar + 1) : "memory");
            } while (g2 == gen);
        }
    }
    __syncthreads();
}
template <int S>
__global__ void my_sync_kernel(unsigned* bar) {
    for (int s = 0; s < S; ++s) my_grid_sync(bar, gridDim.x);
}

// stream: genome in, pred + id out (per = candidates per thread, contiguous per CTA slice)
template <int PER>
__global__ void __launch_bounds__(1024, 1) stream_kernel(const uint64_t* __restrict__ g, double* __restrict__ pred,
                                                         uint64_t* __restrict__ ids, int n) {
    const uint32_t base = blockIdx.x * PER * 1024u;
    uint64_t x[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = base + j * 1024u + threadIdx.x;
        x[j] = i < uint32_t(n) ? __ldcs(g + i) : 0ull;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = base + j * 1024u + threadIdx.x;
        if (i < uint32_t(n)) {
            __stcs(pred + i, double(x[j] & 0xffff));
            __stcs(reinterpret_cast<unsigned long long*>(ids) + i, x[j] * 0x9e3779b97f4a7c15ull);
        }
    }
}
// stream + dependent 16-byte gather
template <int PER>
__global__ void __launch_bounds__(1024, 1) gather_kernel(const uint64_t* __restrict__ g,
                                                         const double2* __restrict__ tab, uint32_t rows,
                                                         double* __restrict__ pred, uint64_t* __restrict__ ids, int n) {
    const uint32_t base = blockIdx.x * PER * 1024u;
    uint64_t x[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = base + j * 1024u + threadIdx.x;
        x[j] = i < uint32_t(n) ? __ldcs(g + i) : 0ull;
    }
    double p[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const double2 r = __ldg(tab + uint32_t(x[j] % rows));
        p[j] = r.x + r.y;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t i = base + j * 1024u + threadIdx.x;
        if (i < uint32_t(n)) {
            __stcs(pred + i, p[j]);
            __stcs(reinterpret_cast<unsigned long long*>(ids) + i, x[j] * 0x9e3779b97f4a7c15ull);
        }
    }
}

int main() {
    const int n = 1 << 20, NB = 16;
    std::vector<uint64_t*> gs(NB);
    std::vector<double*> ps(NB);
    std::vector<uint64_t*> is(NB);
    std::vector<uint64_t> h(n);
    for (int i = 0; i < n; ++i) h[i] = (uint64_t(i) * 2654435761u) ^ (uint64_t(i) << 20);
    for (int b = 0; b < NB; ++b) {
        cudaMalloc(&gs[b], n * 8);
        cudaMalloc(&ps[b], n * 8);
        cudaMalloc(&is[b], n * 8);
        cudaMemcpy(gs[b], h.data(), n * 8, cudaMemcpyHostToDevice);
    }
    const uint32_t rows = 84672;
    double2* tab;
    cudaMalloc(&tab, rows * 16);
    cudaMemset(tab, 0, rows * 16);
    int* d = nullptr;
    cudaMalloc(&d, 4);
    unsigned* bar;
    cudaMalloc(&bar, 8);
    cudaMemset(bar, 0, 8);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int R = 200;
    auto run = [&](const char* name, auto fn) {
        for (int i = 0; i < 10; ++i) fn(i);
        cudaEventRecord(a, st);
        for (int i = 0; i < R; ++i) fn(i);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-52s %8.2f us/launch  (%s)\n", name, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
    };
    const int G = 148, T = 1024;
    for (size_t smem : {size_t(0), size_t(80 * 1024)}) {
        cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(cg_sync_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(cg_sync_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(my_sync_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaFuncSetAttribute(my_sync_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        printf("dynamic smem %zu, %d x %d\n", smem, G, T);
        run("regular empty", [&](int) { empty_kernel<<<G, T, smem, st>>>(d); });
        void* args[] = {&d};
        run("cooperative empty", [&](int) { cudaLaunchCooperativeKernel((void*)empty_kernel, G, T, args, smem, st); });
        run("cooperative cg 1 sync", [&](int) { cudaLaunchCooperativeKernel((void*)cg_sync_kernel<1>, G, T, args, smem, st); });
        run("cooperative cg 4 syncs", [&](int) { cudaLaunchCooperativeKernel((void*)cg_sync_kernel<4>, G, T, args, smem, st); });
        void* bargs[] = {&bar};
        run("cooperative own 1 sync", [&](int) { cudaLaunchCooperativeKernel((void*)my_sync_kernel<1>, G, T, bargs, smem, st); });
        run("cooperative own 4 syncs", [&](int) { cudaLaunchCooperativeKernel((void*)my_sync_kernel<4>, G, T, bargs, smem, st); });
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = G;
        cfg.blockDim = T;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        run("regular empty + PDL", [&](int) { cudaLaunchKernelEx(&cfg, empty_kernel, d); });
        cfg.numAttrs = 2;
        run("cooperative empty + PDL (LaunchKernelEx)", [&](int) { cudaLaunchKernelEx(&cfg, empty_kernel, d); });
        cfg.attrs = at + 1;
        cfg.numAttrs = 1;
        run("cooperative empty (LaunchKernelEx)", [&](int) { cudaLaunchKernelEx(&cfg, empty_kernel, d); });
    }
    // the same launches replayed from a CUDA graph (200 kernels per graph)
    for (int coop = 0; coop < 2; ++coop) {
        const size_t smem = 80 * 1024;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        void* args[] = {&d};
        for (int i = 0; i < R; ++i) {
            if (coop) cudaLaunchCooperativeKernel((void*)cg_sync_kernel<1>, G, T, args, smem, st);
            else empty_kernel<<<G, T, smem, st>>>(d);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-52s %8.2f us/launch  (%s)\n", coop ? "graph: cooperative cg 1 sync, 80 KB smem" : "graph: regular empty, 80 KB smem",
               ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
    }
    // streams of the step's traffic (16 buffers cycled: 384 MB > L2)
    run("stream 8B in 16B out, 2^20, per=7 (147 CTAs)", [&](int i) {
        stream_kernel<7><<<(n + 7 * 1024 - 1) / (7 * 1024), 1024, 0, st>>>(gs[i % NB], ps[i % NB], is[i % NB], n);
    });
    run("stream per=4 (256 CTAs)", [&](int i) {
        stream_kernel<4><<<n / 4096, 1024, 0, st>>>(gs[i % NB], ps[i % NB], is[i % NB], n);
    });
    run("stream per=2 (512 CTAs)", [&](int i) {
        stream_kernel<2><<<n / 2048, 1024, 0, st>>>(gs[i % NB], ps[i % NB], is[i % NB], n);
    });
    run("stream per=1 (1024 CTAs)", [&](int i) {
        stream_kernel<1><<<n / 1024, 1024, 0, st>>>(gs[i % NB], ps[i % NB], is[i % NB], n);
    });
    run("gather per=7 (147 CTAs)", [&](int i) {
        gather_kernel<7><<<(n + 7 * 1024 - 1) / (7 * 1024), 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
    });
    run("gather per=4 (256 CTAs)", [&](int i) {
        gather_kernel<4><<<n / 4096, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
    });
    run("gather per=2 (512 CTAs)", [&](int i) {
        gather_kernel<2><<<n / 2048, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
    });
    run("gather per=1 (1024 CTAs)", [&](int i) {
        gather_kernel<1><<<n / 1024, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
    });
    run("memcpy D2D 8 MB (read 8 + write 8)", [&](int i) {
        cudaMemcpyAsync(ps[i % NB], gs[(i + 1) % NB], n * 8, cudaMemcpyDeviceToDevice, st);
    });
    return 0;
}
