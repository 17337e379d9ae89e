// Measurement harness (north_star (5); the reference's NvmlBackend is a stub that always
// throws, measure.hpp:130-140): run a candidate schedule's kernel on this GPU and
// measure its latency (CUDA events) and energy (NVML's cumulative energy counter,
// nvmlDeviceGetTotalEnergyConsumption, mJ) over a repeat window after a warm-up, the
// protocol of PAPER:164-165 / SPEC:324-332: energy per run = average power x latency.
//
// The candidate kernel is one runtime-parameterised fp32 tiled GEMM that follows the
// Schedule's semantics (schedule.hpp:40-57): grid = blocks_b*blocks_m*blocks_n CTAs of
// threads_b*threads_m*threads_n threads, each thread owning a pt_b x pt_m x pt_n output
// tile; the reduction advances k_tile at a time through shared-memory tiles of
// bt_b*k_tile*(bt_m+bt_n) floats (the counters' glb_ld tile, counters.cpp:32-33), with
// `unroll` reduction steps per inner-loop iteration and `vectorize`-wide loads of the B
// tile.  Conv operators run as implicit GEMM (m = OH*OW, k = Cin*ks^2, opspec.cpp:103-117)
// gathering the input patch on the fly.  Schedules whose per-thread tile exceeds the
// register budget or whose shared tiles exceed shared memory are reported infeasible
// (legality ignores these limits).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "etune_internal.hpp"
#include "kernels.hpp"

namespace etune_b200 {

namespace {

constexpr int kMaxPT = 8;  // per-thread tile bound per dim (m, n): accumulators stay in registers

struct CandGeom {
    int32_t kind;                // 0 mm/mv, 2 conv
    int32_t Bn, M, N, K;         // loop nest
    int32_t blocks[3], threads[3], pt[3];
    int32_t k_tile, unroll, vec;
    // conv
    int32_t H, W, Cin, KS, stride, pad, OH, OW;
};

// A element (batch b, row m, reduction k): plain row-major for matmul, the implicit-GEMM
// patch gather for conv (input NCHW, k = (c, kh, kw))
__device__ __forceinline__ float load_a(const CandGeom& g, const float* __restrict__ A, int b, int m, int k) {
    if (g.kind != 2) return A[(int64_t(b) * g.M + m) * g.K + k];
    const int c = k / (g.KS * g.KS), r = k % (g.KS * g.KS), kh = r / g.KS, kw = r % g.KS;
    const int oh = m / g.OW, ow = m % g.OW;
    const int ih = oh * g.stride - g.pad + kh, iw = ow * g.stride - g.pad + kw;
    if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) return 0.f;
    return A[((int64_t(b) * g.Cin + c) * g.H + ih) * g.W + iw];
}

// B element (batch b, reduction k, column n): row-major K x N for matmul; conv weights
// [Cout][Cin*ks*ks] read transposed
__device__ __forceinline__ const float* b_row(const CandGeom& g, const float* __restrict__ B, int b, int k) {
    return g.kind != 2 ? B + (int64_t(b) * g.K + k) * g.N : nullptr;
}

// MAXPT 4: <= 16 accumulators, fits 1024-thread blocks (64 registers); MAXPT 8: up to 64
template <int MAXPT, int UNROLL, int VEC>
__global__ void __launch_bounds__(MAXPT == 4 ? 1024 : 512) candidate_kernel(CandGeom g, const float* __restrict__ A, const float* __restrict__ B,
                                 float* __restrict__ C) {
    extern __shared__ float tiles[];
    const int btb = g.threads[0] * g.pt[0], btm = g.threads[1] * g.pt[1], btn = g.threads[2] * g.pt[2];
    float* As = tiles;                                    // [btb][btm][k_tile]
    float* Bs = tiles + ((btb * btm * g.k_tile + 3) & ~3);  // [btb][k_tile][btn], 16-byte aligned
    // block / thread coordinates, batch-major like the schedule's spatial order
    int bid = blockIdx.x;
    const int cn = bid % g.blocks[2];
    bid /= g.blocks[2];
    const int cm = bid % g.blocks[1];
    const int cb = bid / g.blocks[1];
    int tid = threadIdx.x;
    const int tn = tid % g.threads[2];
    tid /= g.threads[2];
    const int tm = tid % g.threads[1];
    const int tb = tid / g.threads[1];
    const int nthr = g.threads[0] * g.threads[1] * g.threads[2];
    const int b0 = cb * btb, m0 = cm * btm, n0 = cn * btn;

    for (int pb = 0; pb < g.pt[0]; ++pb) {
        const int lb = tb * g.pt[0] + pb;  // local batch row of this thread
        float acc[MAXPT][MAXPT];
#pragma unroll
        for (int i = 0; i < MAXPT; ++i)
#pragma unroll
            for (int j = 0; j < MAXPT; ++j) acc[i][j] = 0.f;
        for (int k0 = 0; k0 < g.K; k0 += g.k_tile) {
            __syncthreads();
            // cooperative loads of the A and B tiles (every thread of the block)
            const int asz = btb * btm * g.k_tile;
            for (int e = threadIdx.x; e < asz; e += nthr) {
                const int kk = e % g.k_tile, r = e / g.k_tile, mm = r % btm, bb = r / btm;
                As[e] = load_a(g, A, b0 + bb, m0 + mm, k0 + kk);
            }
            const int bsz = btb * g.k_tile * btn;
            if (g.kind != 2) {
                for (int e = threadIdx.x * VEC; e < bsz; e += nthr * VEC) {  // VEC-wide along n
                    const int nn = e % btn, r = e / btn, kk = r % g.k_tile, bb = r / g.k_tile;
                    const float* src = b_row(g, B, b0 + bb, k0 + kk) + n0 + nn;
                    if (VEC == 4) {
                        *reinterpret_cast<float4*>(Bs + e) = *reinterpret_cast<const float4*>(src);
                    } else if (VEC == 2) {
                        *reinterpret_cast<float2*>(Bs + e) = *reinterpret_cast<const float2*>(src);
                    } else {
                        Bs[e] = *src;
                    }
                }
            } else {
                for (int e = threadIdx.x; e < bsz; e += nthr) {
                    const int nn = e % btn, r = e / btn, kk = r % g.k_tile;
                    Bs[e] = B[int64_t(n0 + nn) * g.K + (k0 + kk)];
                }
            }
            __syncthreads();
            const float* Ab = As + (lb * btm + tm * g.pt[1]) * g.k_tile;
            const float* Bb = Bs + lb * g.k_tile * btn + tn * g.pt[2];
            for (int kk = 0; kk < g.k_tile; kk += UNROLL) {
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    float a[MAXPT], bv[MAXPT];
#pragma unroll
                    for (int i = 0; i < MAXPT; ++i) a[i] = i < g.pt[1] ? Ab[i * g.k_tile + kk + u] : 0.f;
#pragma unroll
                    for (int j = 0; j < MAXPT; ++j) bv[j] = j < g.pt[2] ? Bb[(kk + u) * btn + j] : 0.f;
#pragma unroll
                    for (int i = 0; i < MAXPT; ++i)
#pragma unroll
                        for (int j = 0; j < MAXPT; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
                }
            }
        }
        const int b = b0 + lb;
#pragma unroll
        for (int i = 0; i < MAXPT; ++i) {
            if (i >= g.pt[1]) break;
            const int m = m0 + tm * g.pt[1] + i;
#pragma unroll
            for (int j = 0; j < MAXPT; ++j) {
                if (j >= g.pt[2]) break;
                const int n = n0 + tn * g.pt[2] + j;
                if (g.kind != 2) C[(int64_t(b) * g.M + m) * g.N + n] = acc[i][j];
                else C[(int64_t(b) * g.N + n) * g.M + m] = acc[i][j];  // NCHW output: [b][cout][oh*ow]
            }
        }
    }
}

__global__ void fill_kernel(float* __restrict__ x, int64_t n, uint32_t seed) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t h = uint32_t(i) * 2654435761u ^ seed;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        x[i] = float(h & 0xffff) / 65536.f - 0.5f;
    }
}

using KFn = void (*)(CandGeom, const float*, const float*, float*);
template <int P, int U>
KFn pick_vec(int v) {
    return v == 4 ? candidate_kernel<P, U, 4> : v == 2 ? candidate_kernel<P, U, 2> : candidate_kernel<P, U, 1>;
}
template <int P>
KFn pick_unroll(int u, int v) {
    if (u >= 8) return pick_vec<P, 8>(v);
    if (u == 4) return pick_vec<P, 4>(v);
    if (u == 2) return pick_vec<P, 2>(v);
    return pick_vec<P, 1>(v);
}
KFn pick_kernel(const CandGeom& g) {
    return (g.pt[1] <= 4 && g.pt[2] <= 4) ? pick_unroll<4>(g.unroll, g.vec) : pick_unroll<8>(g.unroll, g.vec);
}

// ------------------------------------------------------------------ NVML
struct Nvml {
    void* so = nullptr;
    int (*init)() = nullptr;
    int (*by_pci)(const char*, void**) = nullptr;
    int (*energy)(void*, unsigned long long*) = nullptr;
    int (*power)(void*, unsigned int*) = nullptr;
    bool ok = false;
    std::string why;
};

Nvml& nvml() {
    static Nvml N;
    static std::once_flag once;
    std::call_once(once, [] {
        N.so = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_LOCAL);
        if (!N.so) {
            N.why = "libnvidia-ml.so.1 not found";
            return;
        }
        N.init = reinterpret_cast<int (*)()>(dlsym(N.so, "nvmlInit_v2"));
        N.by_pci = reinterpret_cast<int (*)(const char*, void**)>(dlsym(N.so, "nvmlDeviceGetHandleByPciBusId_v2"));
        N.energy = reinterpret_cast<int (*)(void*, unsigned long long*)>(
            dlsym(N.so, "nvmlDeviceGetTotalEnergyConsumption"));
        N.power = reinterpret_cast<int (*)(void*, unsigned int*)>(dlsym(N.so, "nvmlDeviceGetPowerUsage"));
        if (!N.init || !N.by_pci || !N.energy || !N.power) {
            N.why = "NVML symbols missing";
            return;
        }
        if (N.init() != 0) {
            N.why = "nvmlInit_v2 failed";
            return;
        }
        N.ok = true;
    });
    return N;
}

}  // namespace

bool nvml_available(std::string* why) {
    Nvml& N = nvml();
    if (!N.ok && why) *why = N.why;
    return N.ok;
}

void* nvml_device_handle(int cuda_device, std::string* why) {
    Nvml& N = nvml();
    if (!N.ok) {
        if (why) *why = N.why;
        return nullptr;
    }
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), cuda_device) != cudaSuccess) {
        if (why) *why = "cudaDeviceGetPCIBusId failed";
        return nullptr;
    }
    void* h = nullptr;
    if (N.by_pci(bus, &h) != 0) {
        if (why) *why = std::string("nvmlDeviceGetHandleByPciBusId failed for ") + bus;
        return nullptr;
    }
    return h;
}

bool nvml_energy_mj(void* h, unsigned long long* mj) { return nvml().energy(h, mj) == 0; }
bool nvml_power_mw(void* h, unsigned int* mw) { return nvml().power(h, mw) == 0; }

// Feasibility + launch geometry of one schedule; returns false (infeasible) when the
// per-thread tile or the shared tiles exceed this build's kernel limits.
bool candidate_geometry(const etune_op_spec& op, const int64_t nest[4], const etune_schedule& s, int smem_cap,
                        void* out_geom, size_t* smem, int* grid, int* block) {
    CandGeom g{};
    g.kind = op.kind == 2 ? 2 : 0;
    g.Bn = int32_t(nest[0]);
    g.M = int32_t(nest[1]);
    g.N = int32_t(nest[2]);
    g.K = int32_t(nest[3]);
    for (int d = 0; d < 3; ++d) {
        g.blocks[d] = int32_t(s.spatial[d][0]);
        g.threads[d] = int32_t(s.spatial[d][1]);
        g.pt[d] = int32_t(s.spatial[d][2]);
    }
    g.k_tile = int32_t(s.k_tile);
    g.unroll = int32_t(s.unroll);
    g.vec = int32_t(s.vectorize);
    if (g.kind == 2) {
        g.H = int32_t(op.height);
        g.W = int32_t(op.width);
        g.Cin = int32_t(op.in_channels);
        g.KS = int32_t(op.kernel_size);
        g.stride = int32_t(op.stride);
        g.pad = int32_t(op.padding);
        g.OH = int32_t((op.height + 2 * op.padding - op.kernel_size) / op.stride + 1);
        g.OW = int32_t((op.width + 2 * op.padding - op.kernel_size) / op.stride + 1);
    }
    if (g.pt[1] > kMaxPT || g.pt[2] > kMaxPT || g.unroll > 8) return false;
    const int64_t btb = int64_t(g.threads[0]) * g.pt[0], btm = int64_t(g.threads[1]) * g.pt[1],
                  btn = int64_t(g.threads[2]) * g.pt[2];
    const int64_t floats = ((btb * btm * g.k_tile + 3) & ~int64_t(3)) + btb * g.k_tile * btn;
    if (floats * 4 > smem_cap) return false;
    // vector loads need aligned rows; otherwise this schedule's B tile is loaded scalar
    if (g.kind == 2 || btn % g.vec != 0 || g.N % g.vec != 0) g.vec = 1;
    const int64_t grid64 = int64_t(g.blocks[0]) * g.blocks[1] * g.blocks[2];
    if (grid64 > 0x7fffffff) return false;
    std::memcpy(out_geom, &g, sizeof(g));
    *smem = size_t(floats) * 4;
    *grid = int(grid64);
    *block = g.threads[0] * g.threads[1] * g.threads[2];
    return true;
}

size_t candidate_geom_bytes() { return sizeof(CandGeom); }

// the kernel variant a geometry selects can launch `block` threads (registers x block
// within the register file and the variant's launch bound)
bool candidate_fits(const void* geom, int block) {
    CandGeom g;
    std::memcpy(&g, geom, sizeof(g));
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, pick_kernel(g)) != cudaSuccess) return false;
    return block <= fa.maxThreadsPerBlock && int64_t(block) * fa.numRegs <= 65536;
}

cudaError_t launch_candidate(cudaStream_t st, const void* geom, size_t smem, int grid, int block, const float* A,
                             const float* B, float* C) {
    CandGeom g;
    std::memcpy(&g, geom, sizeof(g));
    KFn k = pick_kernel(g);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
    }
    k<<<grid, block, smem, st>>>(g, A, B, C);
    return cudaGetLastError();
}

cudaError_t launch_fill(cudaStream_t st, float* x, int64_t n, uint32_t seed) {
    fill_kernel<<<1024, 256, 0, st>>>(x, n, seed);
    return cudaGetLastError();
}

}  // namespace etune_b200
