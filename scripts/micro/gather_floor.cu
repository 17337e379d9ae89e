// Phase-A variants of the score step on the B200 (2^20 candidates, 16 population buffers cycled):
// genome (8 B) in -> one dependent gather from an L2-resident row table -> prediction + id (16 B) out.
// What does the dependent gather cost, and which load/store path hides it best?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_floor gather_floor.cu
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int PER, int MODE>  // MODE 0: __ldg 16 B, 1: __ldcg 16 B, 2: __ldg 8 B (f64 table)
__global__ void __launch_bounds__(1024, 1) gather_kernel(const uint64_t* __restrict__ g, const void* __restrict__ tab,
                                                         uint32_t rows, double* __restrict__ pred,
                                                         uint64_t* __restrict__ ids, int n) {
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
        const uint32_t r = __umulhi(uint32_t(x[j]), rows);
        if (MODE == 0) {
            const double2 v = __ldg(static_cast<const double2*>(tab) + r);
            p[j] = v.x + v.y;
        } else if (MODE == 1) {
            const double2 v = __ldcg(static_cast<const double2*>(tab) + r);
            p[j] = v.x + v.y;
        } else {
            p[j] = __ldg(static_cast<const double*>(tab) + r);
        }
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

// TMA: the CTA's genome slice arrives by bulk copies into shared memory (no registers), each thread
// gathers its PER rows, the outputs are staged in shared memory and leave by bulk stores.
template <int PER>
__global__ void __launch_bounds__(1024, 1) tma_kernel(const uint64_t* __restrict__ g, const double2* __restrict__ tab,
                                                      uint32_t rows, double* __restrict__ pred,
                                                      uint64_t* __restrict__ ids, int n) {
    extern __shared__ __align__(128) uint64_t sm[];  // [PER*1024 genomes | PER*1024 preds | PER*1024 ids]
    __shared__ __align__(8) uint64_t bar[PER];
    const uint32_t base = blockIdx.x * PER * 1024u;
    uint64_t* sg = sm;
    double* sp = reinterpret_cast<double*>(sm + PER * 1024);
    uint64_t* si = sm + 2 * PER * 1024;
    if (threadIdx.x == 0) {
        for (int j = 0; j < PER; ++j) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + j)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j < PER; ++j) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + j)), "r"(8192)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sg + j * 1024)),
                "l"(g + base + j * 1024), "r"(8192), "r"(smem_u32(bar + j))
                : "memory");
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar + j))
            : "memory");
        const uint64_t x = sg[j * 1024 + threadIdx.x];
        const double2 v = __ldg(tab + __umulhi(uint32_t(x), rows));
        sp[j * 1024 + threadIdx.x] = v.x + v.y;
        si[j * 1024 + threadIdx.x] = x * 0x9e3779b97f4a7c15ull;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(pred + base),
                     "r"(smem_u32(sp)), "r"(PER * 8192)
                     : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(ids + base),
                     "r"(smem_u32(si)), "r"(PER * 8192)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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
    void* tab;
    cudaMalloc(&tab, 84672 * 16);
    cudaMemset(tab, 0, 84672 * 16);
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
        printf("%-56s %8.2f us/launch  (%s)\n", name, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
    };
    const int G7 = (n + 7167) / 7168;
    for (uint32_t rows : {84672u, 4096u, 256u}) {
        printf("rows %u\n", rows);
        run("ldg 16B per=7", [&](int i) {
            gather_kernel<7, 0><<<G7, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
        });
        run("ldcg 16B per=7", [&](int i) {
            gather_kernel<7, 1><<<G7, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
        });
        run("ldg 8B per=7", [&](int i) {
            gather_kernel<7, 2><<<G7, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
        });
        run("ldg 16B per=8 (128 CTAs)", [&](int i) {
            gather_kernel<8, 0><<<n / 8192, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
        });
        run("ldg 16B per=4", [&](int i) {
            gather_kernel<4, 0><<<n / 4096, 1024, 0, st>>>(gs[i % NB], tab, rows, ps[i % NB], is[i % NB], n);
        });
        const int smem = 3 * 8 * 8192;
        cudaFuncSetAttribute(tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        run("tma per=8 (128 CTAs)", [&](int i) {
            tma_kernel<8><<<n / 8192, 1024, smem, st>>>(gs[i % NB], (const double2*)tab, rows, ps[i % NB], is[i % NB], n);
        });
        cudaFuncSetAttribute(tma_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 7 * 8192);
        run("tma per=7 (147 CTAs; last partial)", [&](int i) {
            tma_kernel<7><<<n / 7168, 1024, 3 * 7 * 8192, st>>>(gs[i % NB], (const double2*)tab, rows, ps[i % NB], is[i % NB], n);
        });
    }
    return 0;
}
