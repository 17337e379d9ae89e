// EnergyModel::train on the device, bit-exact (energy_model.cpp:173-243 with the
// TreeBuilder of 48-169).
//
// Exactness: every floating-point sum the reference forms sequentially
// is formed sequentially here in the same order — the harmonic-mean denominator,
// each node's (grad, hess) totals in sample order, and each (feature, node) running
// prefix in feature-sorted order.  What runs in parallel is everything the reference
// computes independently: the 16 features x frontier nodes chains of one level, the
// split gains at every scan position (evaluated from the stored prefixes, then
// reduced with the reference's rule: strictly larger gain wins, so the earliest
// (feature, position) keeps ties), routing, leaf values and prediction updates.
//
// Layout: 17 index lists of n int32 (16 stable feature orders + the sample order),
// each partitioned into contiguous segments, one per frontier node, in frontier
// order.  A split partitions a segment stably into [left | right] in place, which is
// exactly the order in which the reference's per-node scans and sample-order
// routing visit the children's samples.  Leaves keep their (dead) ranges.
//
// Every kernel reads the data-dependent frontier size from device memory, so one
// tree is a fixed launch sequence: it is captured once as a CUDA graph and replayed
// num_trees times, with no host synchronisation inside a training.
//
// Per level: gather (grad/hess/feature values into list order) -> chains (one warp per
// (list, node): the sequential prefix sums, staged through shared memory) -> gains at
// every position (parallel; per-(node, feature) argmax by two atomic passes) -> decide
// -> left flags -> stable partition (global scan of the left flags + scatter).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "etune_internal.hpp"
#include "kernels.hpp"
#include "pdl.cuh"
#include "scan.cuh"

namespace etune_b200 {

namespace {

constexpr int kF = 16;       // kFeatureDim
constexpr int kLists = kF + 1;
constexpr int kSampleList = kF;
constexpr int kMaxDepth = 10;
constexpr int kMaxSeg = 1 << kMaxDepth;
constexpr int kMaxNodes = (1 << (kMaxDepth + 1)) - 1;
constexpr double kMinSplitGain = 1e-12;  // energy_model.cpp:20

struct TrainCtl {
    int32_t nseg[2];
    int32_t seg_start[2][kMaxSeg], seg_end[2][kMaxSeg], seg_node[2][kMaxSeg];
    int32_t split[kMaxSeg];   // child rank r (children 2r, 2r+1 of the next frontier) or -1
    int32_t nnodes;
    int32_t tree;             // trees finished
    int64_t out_nodes;        // nodes written to the output forest so far
    // current tree
    int32_t feature[kMaxNodes], left[kMaxNodes], right[kMaxNodes];
    double thr[kMaxNodes], value[kMaxNodes], sg[kMaxNodes], sh[kMaxNodes];
    // per (segment, feature) best split: max gain bits (gains are > 0), then min position
    unsigned long long gbits[kMaxSeg][kF];
    int32_t gpos[kMaxSeg][kF];
    double base, reference;
};

__device__ __forceinline__ uint64_t order_key(double x) {
    x = __dadd_rn(x, 0.0);  // -0.0 == +0.0 under operator<, as std::stable_sort sees them
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double obj(double g, double h, double lambda) {  // leaf_objective, cpp 61-63
    return __ddiv_rn(__dmul_rn(g, g), __dadd_rn(h, lambda));
}

// ---------------------------------------------------------------- init
// Sequential sum of x[0..n) in index order by one thread, reading 256-element chunks the
// whole CTA staged into shared memory (the reference's loops are one dependent chain).
__device__ double cta_sequential_sum(const double* __restrict__ x, int64_t n, double* stage) {
    double acc = 0.0;
    for (int64_t base = 0; base < n; base += 1024) {
        const int cnt = int(n - base < 1024 ? n - base : 1024);
        __syncthreads();
        for (int j = threadIdx.x; j < cnt; j += blockDim.x) stage[j] = x[base + j];
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int j = 0; j < cnt; j += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = stage[j + u];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (j + u < cnt) acc = __dadd_rn(acc, v[u]);
            }
        }
    }
    return acc;  // meaningful in thread 0
}

// reference energy (min), NonPositiveEnergy check, targets, harmonic-mean base score
// (one sequential chain, energy_model.cpp:199-202), pred = base; `tmp` is n doubles.
__global__ void __launch_bounds__(1024) init_kernel(const double* __restrict__ energy, int64_t n,
                                                   double* __restrict__ target, double* __restrict__ pred,
                                                   TrainCtl* ctl, unsigned long long* err,
                                                   double* __restrict__ loss0, double* __restrict__ tmp) {
    __shared__ double red[32];
    __shared__ double stage[1024 + 8];
    __shared__ int bad;
    __shared__ double s_base;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    double m = __longlong_as_double(0x7ff0000000000000ll);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double e = energy[i];
        if (!(e > 0.0)) {
            atomicMin(err, (static_cast<unsigned long long>(i) << 8) | unsigned(ETUNE_ERR_NON_POSITIVE_ENERGY));
            bad = 1;
        }
        m = e < m ? e : m;
    }
    for (int s = 16; s > 0; s >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, m, s);
        m = o < m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (bad) return;
    double ref = red[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) ref = red[w] < ref ? red[w] : ref;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double t = __ddiv_rn(energy[i], ref);
        target[i] = t;
        tmp[i] = __ddiv_rn(1.0, t);
    }
    __syncthreads();
    const double inv = cta_sequential_sum(tmp, n, stage);
    if (threadIdx.x == 0) {
        s_base = __ddiv_rn(static_cast<double>(n), inv);
        ctl->base = s_base;
        ctl->reference = ref;
        ctl->out_nodes = 0;
        ctl->tree = 0;
    }
    __syncthreads();
    const double base = s_base;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) pred[i] = base;
    if (loss0) {  // mean_loss() before any tree (cpp 221-227)
        __syncthreads();
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const double d = __dsub_rn(base, target[i]);
            tmp[i] = __ddiv_rn(__dmul_rn(d, d), target[i]);
        }
        __syncthreads();
        const double tot = cta_sequential_sum(tmp, n, stage);
        if (threadIdx.x == 0) loss0[0] = __ddiv_rn(tot, static_cast<double>(n));
    }
}

// ----------------------------------------------------------------- sort
// One CTA per feature: bitonic sort of (order_key(value), index) pairs == std::stable_sort
// by value (energy_model.cpp:204-213); list 16 = identity.  In shared memory when the
// padded column fits (n <= 16384), else in global memory.
__global__ void __launch_bounds__(1024) sort_kernel(const double* __restrict__ feats, int64_t n, int64_t n2,
                                                   int in_smem, uint64_t* __restrict__ kbuf,
                                                   uint32_t* __restrict__ ibuf, int32_t* __restrict__ lists) {
    extern __shared__ uint64_t sortmem[];
    const int f = blockIdx.x;
    int32_t* out = lists + int64_t(f) * n;
    if (f == kSampleList) {
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = int32_t(i);
        return;
    }
    uint64_t* K = in_smem ? sortmem : kbuf + int64_t(f) * n2;
    uint32_t* I = in_smem ? reinterpret_cast<uint32_t*>(sortmem + n2) : ibuf + int64_t(f) * n2;
    for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) {
        K[i] = i < n ? order_key(feats[i * kF + f]) : ~0ull;
        I[i] = i < n ? uint32_t(i) : 0xffffffffu;
    }
    __syncthreads();
    for (int64_t size = 2; size <= n2; size <<= 1) {
        for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) {
                const int64_t j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const uint64_t ki = K[i], kj = K[j];
                    const uint32_t ii = I[i], ij = I[j];
                    const bool gt = ki > kj || (ki == kj && ii > ij);
                    if (gt == up) {
                        K[i] = kj;
                        K[j] = ki;
                        I[i] = ij;
                        I[j] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = int32_t(I[i]);
}

// ----------------------------------------------------- per tree: gradients
__global__ void grad_kernel(const double* __restrict__ pred, const double* __restrict__ target, int64_t n,
                            double* __restrict__ grad, double* __restrict__ hess, TrainCtl* ctl) {
    pdl_wait();
    const int64_t i0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i0 == 0) {  // fresh tree: a single root leaf holding every sample
        ctl->nseg[0] = 1;
        ctl->seg_start[0][0] = 0;
        ctl->seg_end[0][0] = int32_t(n);
        ctl->seg_node[0][0] = 0;
        ctl->nnodes = 1;
        ctl->feature[0] = -1;
        ctl->left[0] = -1;
        ctl->right[0] = -1;
        ctl->thr[0] = 0.0;
        ctl->value[0] = 0.0;
    }
    for (int64_t i = i0; i < n; i += int64_t(gridDim.x) * blockDim.x) {  // energy_loss, cpp 23-34
        const double m = target[i];
        const double d = __dsub_rn(pred[i], m);
        grad[i] = __ddiv_rn(__dmul_rn(2.0, d), m);
        hess[i] = __ddiv_rn(2.0, m);
    }
}

// segment (frontier index) of every position, -1 for dead ranges; identical for all lists
__device__ __forceinline__ int32_t seg_of(int64_t p, int nseg, const int32_t* ss, const int32_t* se) {
    int lo = 0, hi = nseg;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ss[mid] <= p) lo = mid + 1;
        else hi = mid;
    }
    const int k = lo - 1;
    return (k >= 0 && p < se[k]) ? k : -1;
}

// gl/hl[l][p] = grad/hess[list[l][p]], fv[l][p] = feature l of that sample: everything the
// chains and gains read afterwards is contiguous in list order.  With segmap non-null the
// same launch also maps every list position to its frontier segment (-1: a leaf's range).
__global__ void gather_kernel(const int32_t* __restrict__ lists, int64_t n, int nl, const double* __restrict__ grad,
                              const double* __restrict__ hess, const double* __restrict__ feats,
                              double* __restrict__ gl, double* __restrict__ hl, double* __restrict__ fv, int lvl,
                              const TrainCtl* __restrict__ ctl, int32_t* __restrict__ segmap) {
    pdl_wait();
    const int64_t tot = int64_t(nl) * n;
    const int64_t off = int64_t(kLists - nl) * n;  // nl == 1: sample list only
    const int b = lvl & 1;
    const int nseg = ctl->nseg[b];
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = off + q;
        const int32_t idx = lists[g];
        gl[g] = grad[idx];
        hl[g] = hess[idx];
        if (g < int64_t(kF) * n) fv[g] = feats[int64_t(idx) * kF + g / n];
        if (segmap && q < n) segmap[q] = seg_of(q, nseg, ctl->seg_start[b], ctl->seg_end[b]);
    }
}

// Per (list, frontier segment): the sequential running sums, kChunk elements at a time
// staged through shared memory (chain_kernel below).
//   lists 0..15: exclusive prefix at every position (the `run` of cpp 95-121)
//   list 16:     the node's (grad, hess) totals in sample order (cpp 73-76, 150-155)
constexpr int kChunk = 1024;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void bar_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

// Two warps per (list, segment): warp 1 streams chunks in (cp.async, two buffers) and
// the prefixes out, warp 0 only chains (lanes 0/1), so the chain never waits on memory.
// Named barriers 1+b ("buffer b full") and 3+b ("buffer b chained") hand the buffers over.
__global__ void __launch_bounds__(64) chain_kernel(int64_t n, int lvl, int only_totals,
                                                   const double* __restrict__ gl, const double* __restrict__ hl,
                                                   double* __restrict__ pg, double* __restrict__ ph, TrainCtl* ctl) {
    pdl_wait();
    // prefixes overwrite their operands in place (each operand is in registers by then)
    __shared__ __align__(16) double ig[2][kChunk + 8];
    __shared__ __align__(16) double ih[2][kChunk + 8];
    const int b = lvl & 1;
    const int nseg = ctl->nseg[b];
    if (nseg <= 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x;
    const int l = only_totals ? kSampleList : t / nseg;
    const int k = only_totals ? t : t % nseg;
    if (k >= nseg || l >= kLists) return;
    const int s = ctl->seg_start[b][k], e = ctl->seg_end[b][k];
    const int nch = (e - s + kChunk - 1) / kChunk;
    const bool prefixes = l != kSampleList;
    if (warp == 1) {  // ---- io warp
        const double* G = gl + int64_t(l) * n;
        const double* Hh = hl + int64_t(l) * n;
        double* PG = pg + int64_t(l) * n;
        double* PH = ph + int64_t(l) * n;
        auto load = [&](int c) {
            const int base = s + c * kChunk, cnt = min(kChunk, e - base), bb = c & 1;
            for (int j = lane; j < cnt; j += 32) {
                cp_async8(&ig[bb][j], G + base + j);
                cp_async8(&ih[bb][j], Hh + base + j);
            }
            cp_async_commit();
        };
        if (nch == 0) return;
        load(0);
        if (nch > 1) {
            load(1);
            cp_async_wait_prev();
        } else {
            cp_async_wait_all();
        }
        bar_arrive(1);  // chunk 0 in buffer 0
        for (int c = 0; c < nch; ++c) {
            const int bb = c & 1;
            if (c + 1 < nch) {
                cp_async_wait_all();  // chunk c+1 (the only group in flight)
                bar_arrive(1 + (bb ^ 1));
            }
            bar_sync(3 + bb);  // chunk c chained in place
            if (prefixes) {
                const int base = s + c * kChunk, cnt = min(kChunk, e - base);
                for (int j = lane; j < cnt; j += 32) {
                    PG[base + j] = ig[bb][j];
                    PH[base + j] = ih[bb][j];
                }
            }
            __syncwarp();
            if (c + 2 < nch) load(c + 2);
        }
        return;
    }
    // ---- chain warp: lane 0 chains the gradients, lane 1 the hessians (one instruction
    // stream, two independent chains), batches of 8 through double2 shared loads/stores,
    // two register sets alternating; the chain runs near the FP64 add latency (8 cycles,
    // scripts/micro/dadd_latency.cu)
    double racc = 0.0;
    for (int c = 0; c < nch; ++c) {
        const int bb = c & 1;
        const int cnt = min(kChunk, e - (s + c * kChunk));
        bar_sync(1 + bb);
        if (lane < 2) {
            double* cx = lane == 0 ? ig[bb] : ih[bb];
            double2* c2 = reinterpret_cast<double2*>(cx);
            const int nb = cnt >> 3;
            const int full = nb << 3;
            double2 xa[4], xb[4];
            auto ld = [&](double2* x, int bi) {
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = c2[bi * 4 + q];
            };
            auto run = [&](const double2* x, int bi) {
                double2 pv[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    pv[q].x = racc;
                    racc = __dadd_rn(racc, x[q].x);
                    pv[q].y = racc;
                    racc = __dadd_rn(racc, x[q].y);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) c2[bi * 4 + q] = pv[q];
            };
            if (nb > 0) ld(xa, 0);
            int bi = 0;
            for (; bi + 1 < nb; bi += 2) {
                ld(xb, bi + 1);
                run(xa, bi);
                if (bi + 2 < nb) ld(xa, bi + 2);
                run(xb, bi + 1);
            }
            if (bi < nb) run(xa, bi);
            for (int j = full; j < cnt; ++j) {
                const double v = cx[j];
                cx[j] = racc;
                racc = __dadd_rn(racc, v);
            }
        }
        __syncwarp();
        bar_arrive(3 + bb);
    }
    const double rg = __shfl_sync(0xffffffffu, racc, 0), rh = __shfl_sync(0xffffffffu, racc, 1);
    if (lane == 0) {
        if (!prefixes) {
            const int node = ctl->seg_node[b][k];
            ctl->sg[node] = rg;
            ctl->sh[node] = rh;
        } else {
            ctl->gbits[k][l] = 0ull;
            ctl->gpos[k][l] = 0x7fffffff;
        }
    }
}

// split gain at every (feature list, position) (cpp 97-118); per-(node, feature) max
// gain by atomicMax on the (positive) gain's bits
__global__ void gain_kernel(int64_t n, int lvl, const int32_t* __restrict__ segmap, const double* __restrict__ fv,
                            const double* __restrict__ pg, const double* __restrict__ ph, double mlw, double lambda,
                            double* __restrict__ gains, TrainCtl* ctl) {
    pdl_wait();
    const int b = lvl & 1;
    const int64_t tot = int64_t(kF) * n;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = q % n;
        const int l = int(q / n);
        const int k = segmap[p];
        double gain = -1.0;
        if (k >= 0 && p > ctl->seg_start[b][k]) {
            const double v = fv[q], pv = fv[q - 1];
            if (v > pv) {
                const int node = ctl->seg_node[b][k];
                const double tg = ctl->sg[node], th = ctl->sh[node];
                const double rg = pg[q], rh = ph[q];
                const double qg = __dsub_rn(tg, rg), qh = __dsub_rn(th, rh);
                if (rh >= mlw && qh >= mlw) {
                    const double g = __dmul_rn(
                        0.5, __dsub_rn(__dadd_rn(obj(rg, rh, lambda), obj(qg, qh, lambda)), obj(tg, th, lambda)));
                    if (g > kMinSplitGain) {
                        gain = g;
                        atomicMax(&ctl->gbits[k][l], static_cast<unsigned long long>(__double_as_longlong(g)));
                    }
                }
            }
        }
        gains[q] = gain;
    }
}

// earliest position attaining the max (ties: the reference's strict > keeps the first)
__global__ void gainpos_kernel(int64_t n, const int32_t* __restrict__ segmap, const double* __restrict__ gains,
                               TrainCtl* ctl) {
    pdl_wait();
    const int64_t tot = int64_t(kF) * n;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
        const double g = gains[q];
        if (!(g > 0.0)) continue;
        const int64_t p = q % n;
        const int l = int(q / n);
        const int k = segmap[p];
        if (static_cast<unsigned long long>(__double_as_longlong(g)) == ctl->gbits[k][l])
            atomicMin(&ctl->gpos[k][l], int32_t(p));
    }
}

// One CTA: choose each node's split (features in order, strictly larger gain wins,
// cpp 111-117), allocate children in frontier order (cpp 130-143).
__global__ void __launch_bounds__(1024) decide_kernel(int64_t n, int lvl, const double* __restrict__ fv,
                                                      TrainCtl* ctl) {
    pdl_wait();
    const int b = lvl & 1;
    const int nseg = ctl->nseg[b];
    __shared__ int wsum[32];
    __shared__ int s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int k0 = 0; k0 < nseg; k0 += blockDim.x) {
        const int k = k0 + threadIdx.x;
        int bf = -1;
        double bg = 0.0, bt = 0.0;
        if (k < nseg) {
            for (int f = 0; f < kF; ++f) {
                const unsigned long long bits = ctl->gbits[k][f];
                if (bits == 0ull) continue;
                const double g = __longlong_as_double(static_cast<long long>(bits));
                if (g > kMinSplitGain && g > bg) {
                    bg = g;
                    bf = f;
                    const int64_t pos = ctl->gpos[k][f];
                    const double* F = fv + int64_t(f) * n;
                    bt = __dmul_rn(0.5, __dadd_rn(F[pos - 1], F[pos]));  // cpp 115-116
                }
            }
        }
        const int flag = bf >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, flag);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 0) wsum[w] = __popc(bal);
        __syncthreads();
        int before = s_base + __popc(bal & ((1u << lane) - 1u));
        for (int i = 0; i < w; ++i) before += wsum[i];
        int total = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) total += wsum[i];
        if (k < nseg) {
            const int node = ctl->seg_node[b][k];
            if (flag) {
                const int lnode = ctl->nnodes + 2 * before;
                ctl->feature[node] = bf;
                ctl->thr[node] = bt;
                ctl->left[node] = lnode;
                ctl->right[node] = lnode + 1;
                ctl->value[node] = 0.0;
                for (int c = 0; c < 2; ++c) {
                    ctl->feature[lnode + c] = -1;
                    ctl->thr[lnode + c] = 0.0;
                    ctl->left[lnode + c] = -1;
                    ctl->right[lnode + c] = -1;
                    ctl->value[lnode + c] = 0.0;
                    ctl->seg_node[b ^ 1][2 * before + c] = lnode + c;
                }
                ctl->split[k] = before;
            } else {
                ctl->split[k] = -1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctl->nnodes += 2 * s_base;
        ctl->nseg[b ^ 1] = 2 * s_base;
    }
}

// routing decision per sample of a split node: value < threshold goes left (cpp 146-148)
__global__ void leftflag_kernel(const double* __restrict__ feats, const int32_t* __restrict__ lists, int64_t n,
                                int lvl, const int32_t* __restrict__ segmap, const TrainCtl* __restrict__ ctl,
                                uint8_t* __restrict__ lf) {
    pdl_wait();
    const int b = lvl & 1;
    const int32_t* S = lists + int64_t(kSampleList) * n;
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
        const int k = segmap[p];
        if (k < 0 || ctl->split[k] < 0) continue;
        const int node = ctl->seg_node[b][k];
        const int32_t idx = S[p];
        lf[idx] = feats[int64_t(idx) * kF + ctl->feature[node]] < ctl->thr[node] ? 1 : 0;
    }
}

struct LeftFlagFn {  // flag of list position q (0 outside split segments)
    const int32_t* lists;
    const int32_t* segmap;
    const int32_t* split;
    const uint8_t* lf;
    int64_t n;
    __device__ int64_t operator()(int64_t q) const {
        const int k = segmap[q % n];
        return (k >= 0 && split[k] >= 0) ? int64_t(lf[lists[q]]) : 0;
    }
};
struct PrefixWrite {
    int64_t* pfx;
    __device__ void operator()(int64_t q, int64_t ex) const { pfx[q] = ex; }
};

// stable partition of every split segment into [left | right] in every list; list 16
// also writes the children's segment bounds
__global__ void scatter_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                               const int64_t* __restrict__ pfx, const int32_t* __restrict__ segmap, int64_t n,
                               int lvl, TrainCtl* ctl) {
    pdl_wait();
    const int b = lvl & 1;
    const int64_t tot = int64_t(kLists) * n;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t l = q / n, p = q % n;
        const int k = segmap[p];
        int64_t d = p;
        if (k >= 0 && ctl->split[k] >= 0) {
            const int64_t s = ctl->seg_start[b][k], e = ctl->seg_end[b][k];
            const int64_t* P = pfx + l * n;
            const int64_t pl = P[p] - P[s];
            const int64_t L = P[e] - P[s];
            const int64_t left = P[p + 1] - P[p];
            d = left ? s + pl : s + L + (p - s - pl);
            if (l == kSampleList && p == s) {
                const int r = ctl->split[k];
                ctl->seg_start[b ^ 1][2 * r] = int32_t(s);
                ctl->seg_end[b ^ 1][2 * r] = int32_t(s + L);
                ctl->seg_start[b ^ 1][2 * r + 1] = int32_t(s + L);
                ctl->seg_end[b ^ 1][2 * r + 1] = int32_t(e);
            }
        }
        dst[l * n + d] = src[q];
    }
}

// Leaf Newton weights (cpp 161-166) and the tree appended to the output forest.
__global__ void __launch_bounds__(1024) finalize_kernel(double lambda, TrainCtl* ctl,
                                                       int32_t* __restrict__ o_feature, double* __restrict__ o_thr,
                                                       int32_t* __restrict__ o_left, int32_t* __restrict__ o_right,
                                                       double* __restrict__ o_value, int64_t* __restrict__ o_off) {
    pdl_wait();
    const int nn = ctl->nnodes;
    const int64_t base = ctl->out_nodes;
    const int tree = ctl->tree;
    for (int i = threadIdx.x; i < nn; i += blockDim.x) {
        if (ctl->feature[i] < 0) ctl->value[i] = __ddiv_rn(-ctl->sg[i], __dadd_rn(ctl->sh[i], lambda));
        o_feature[base + i] = ctl->feature[i];
        o_thr[base + i] = ctl->thr[i];
        o_left[base + i] = ctl->left[i];
        o_right[base + i] = ctl->right[i];
        o_value[base + i] = ctl->value[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (tree == 0) o_off[0] = 0;
        o_off[tree + 1] = base + nn;
        ctl->out_nodes = base + nn;
        ctl->tree = tree + 1;
    }
}

// pred[i] += lr * tree.eval(feat[i])  (cpp 236-238)
__global__ void update_kernel(const double* __restrict__ feats, int64_t n, double lr, const TrainCtl* __restrict__ ctl,
                              double* __restrict__ pred) {
    pdl_wait();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        int node = 0;
        int f = ctl->feature[0];
        while (f >= 0) {
            node = feats[i * kF + f] < ctl->thr[node] ? ctl->left[node] : ctl->right[node];
            f = ctl->feature[node];
        }
        pred[i] = __dadd_rn(pred[i], __dmul_rn(lr, ctl->value[node]));
    }
}

__global__ void __launch_bounds__(1024) loss_kernel(const double* __restrict__ pred,
                                                   const double* __restrict__ target, int64_t n,
                                                   const TrainCtl* __restrict__ ctl, double* __restrict__ loss,
                                                   double* __restrict__ tmp) {
    pdl_wait();
    __shared__ double stage[1024 + 8];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = __dsub_rn(pred[i], target[i]);
        tmp[i] = __ddiv_rn(__dmul_rn(d, d), target[i]);
    }
    __syncthreads();
    const double tot = cta_sequential_sum(tmp, n, stage);
    if (threadIdx.x == 0) loss[ctl->tree] = __ddiv_rn(tot, static_cast<double>(n));  // after finalize: round t+1
}

int64_t pow2_at_least(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t train_scratch_bytes(int64_t n) {
    const int64_t n2 = pow2_at_least(n);
    const size_t L = size_t(kLists) * size_t(n);
    const size_t F = size_t(kF) * size_t(n);
    return al256(sizeof(TrainCtl)) + 4 * al256(8 * size_t(n))     // target, pred, grad, hess
           + 2 * al256(8 * L)                                     // gl, hl
           + 4 * al256(8 * F)                                     // fv, pg, ph, gains
           + 3 * al256(4 * L)                                     // base lists + 2 work buffers
           + al256(8 * (L + 1))                                   // partition prefix
           + al256(4 * size_t(n)) + al256(size_t(n))              // segmap, left flags
           + al256(8 * ((L + 1023) / 1024 + 2))                   // scan tile sums
           + al256(size_t(kF) * n2 * 12);                         // sort keys + indices
}

int train_max_depth() { return kMaxDepth; }

// tree-graph launches carry the programmatic-dependency attribute: each kernel calls
// pdl_wait() first, and the next node's launch overlaps the previous node's tail
#define PDL(k, g, b, sm, st, ...)                                                     \
    do {                                                                             \
        const cudaError_t pe = launch_pdl(k, dim3(g), dim3(b), sm, st, __VA_ARGS__); \
        if (pe != cudaSuccess && e == cudaSuccess) e = pe;                           \
    } while (0)

cudaError_t launch_train(const LaunchCtx& c, const double* d_feat, const double* d_energy, int64_t n, int num_trees,
                         int max_depth, double lr, double mlw, double lambda, int32_t* o_feature, double* o_thr,
                         int32_t* o_left, int32_t* o_right, double* o_value, int64_t* o_off, double* o_scalars,
                         double* o_loss, void* scratch) {
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += al256(bytes);
        return r;
    };
    const int64_t n2 = pow2_at_least(n);
    const size_t L = size_t(kLists) * size_t(n);
    const size_t F = size_t(kF) * size_t(n);
    TrainCtl* ctl = reinterpret_cast<TrainCtl*>(take(sizeof(TrainCtl)));
    double* target = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* pred = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* grad = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* hess = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* gl = reinterpret_cast<double*>(take(8 * L));
    double* hl = reinterpret_cast<double*>(take(8 * L));
    double* fv = reinterpret_cast<double*>(take(8 * F));
    double* pg = reinterpret_cast<double*>(take(8 * F));
    double* ph = reinterpret_cast<double*>(take(8 * F));
    double* gains = reinterpret_cast<double*>(take(8 * F));
    int32_t* base_lists = reinterpret_cast<int32_t*>(take(4 * L));
    int32_t* work[2] = {reinterpret_cast<int32_t*>(take(4 * L)), reinterpret_cast<int32_t*>(take(4 * L))};
    int64_t* pfx = reinterpret_cast<int64_t*>(take(8 * (L + 1)));
    int32_t* segmap = reinterpret_cast<int32_t*>(take(4 * size_t(n)));
    uint8_t* lf = reinterpret_cast<uint8_t*>(take(size_t(n)));
    int64_t* sums = reinterpret_cast<int64_t*>(take(8 * ((L + 1023) / 1024 + 2)));
    uint64_t* kbuf = reinterpret_cast<uint64_t*>(take(size_t(kF) * n2 * 12));
    uint32_t* ibuf = reinterpret_cast<uint32_t*>(kbuf + size_t(kF) * n2);

    init_kernel<<<1, 1024, 0, c.stream>>>(d_energy, n, target, pred, ctl, c.d_err, o_loss, grad);
    const size_t sort_smem = size_t(n2) * 12;
    const int sort_in_smem = sort_smem <= 200 * 1024 ? 1 : 0;
    if (sort_in_smem) {
        cudaError_t ea = cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sort_smem));
        if (ea != cudaSuccess) return ea;
    }
    sort_kernel<<<kLists, 1024, sort_in_smem ? sort_smem : 0, c.stream>>>(d_feat, n, n2, sort_in_smem, kbuf, ibuf,
                                                                          base_lists);
    note_launches(2);
    if (num_trees == 0) {
        cudaMemsetAsync(o_off, 0, sizeof(int64_t), c.stream);
        cudaMemcpyAsync(o_scalars, &ctl->base, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
        return cudaGetLastError();
    }

    // one tree as a fixed launch sequence, captured once and replayed num_trees times
    cudaStream_t cap = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        cudaStreamDestroy(cap);
        return e;
    }
    auto grid = [&](int64_t items) {
        return int(std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, int64_t(c.sm_count) * 16)));
    };
    int launches = 0;
    PDL(grad_kernel, grid(n), 256, 0, cap, pred, target, n, grad, hess, ctl);
    ++launches;
    const int32_t* cur = base_lists;
    int wb = 0;
    int lvl = 0;
    for (int depth = 0; depth < max_depth; ++depth, ++lvl) {
        const int segs = 1 << depth;  // frontier bound at this depth
        PDL(gather_kernel, grid(int64_t(L)), 256, 0, cap, cur, n, kLists, grad, hess, d_feat, gl, hl, fv, lvl, ctl,
            segmap);
        const int warps = kLists * segs;
        PDL(chain_kernel, warps, 64, 0, cap, n, lvl, 0, gl, hl, pg, ph, ctl);
        PDL(gain_kernel, grid(int64_t(F)), 256, 0, cap, n, lvl, segmap, fv, pg, ph, mlw, lambda, gains, ctl);
        PDL(gainpos_kernel, grid(int64_t(F)), 256, 0, cap, n, segmap, gains, ctl);
        PDL(decide_kernel, 1, 1024, 0, cap, n, lvl, fv, ctl);
        PDL(leftflag_kernel, grid(n), 256, 0, cap, d_feat, cur, n, lvl, segmap, ctl, lf);
        if (e == cudaSuccess)
            e = scan_apply(cap, int64_t(L), LeftFlagFn{cur, segmap, ctl->split, lf, n}, PrefixWrite{pfx}, sums,
                           pfx + L);
        if (e != cudaSuccess) break;
        PDL(scatter_kernel, grid(int64_t(L)), 256, 0, cap, cur, work[wb], pfx, segmap, n, lvl, ctl);
        cur = work[wb];
        wb ^= 1;
        launches += 10;
    }
    // totals of the last frontier (children created at the deepest level)
    PDL(gather_kernel, grid(n), 256, 0, cap, cur, n, 1, grad, hess, d_feat, gl, hl, fv, lvl, ctl,
        static_cast<int32_t*>(nullptr));
    const int segs = 1 << max_depth;
    PDL(chain_kernel, segs, 64, 0, cap, n, lvl, 1, gl, hl, pg, ph, ctl);
    PDL(finalize_kernel, 1, 1024, 0, cap, lambda, ctl, o_feature, o_thr, o_left, o_right, o_value, o_off);
    PDL(update_kernel, grid(n), 256, 0, cap, d_feat, n, lr, ctl, pred);
    launches += 4;
    if (o_loss) {
        PDL(loss_kernel, 1, 1024, 0, cap, pred, target, n, ctl, o_loss, gains);
        launches += 1;
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cap, &graph);
    if (e == cudaSuccess) e = ec;
    cudaGraphExec_t exec = nullptr;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    for (int t = 0; t < num_trees && e == cudaSuccess; ++t) e = cudaGraphLaunch(exec, c.stream);
    note_launches(launches * num_trees);
    // base score + reference energy
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(o_scalars, &ctl->base, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
    if (exec) cudaGraphExecDestroy(exec);  // deferred by the driver until the launches complete
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace etune_b200
