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
// -> stable partition (global scan of the routing flags + scatter).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
    int32_t sfeat[kMaxSeg];   // split feature of frontier segment k or -1, and its threshold:
    double sthr[kMaxSeg];     // the routing flag of a list position without the node lookup
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
__device__ double cta_sequential_sum(const double* x, int64_t n, double* stage) {
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
// The per-tree phases below are device functions shared by the per-kernel graph path
// (thin __global__ wrappers) and the cooperative megakernel (train_mega_kernel): their
// pointers carry no __restrict__, since inside the megakernel every buffer but the
// features and targets is rewritten between phases (no read-only-cache loads).
__device__ __forceinline__ void grad_phase(const double* pred, const double* target, int64_t n, double* grad,
                                           double* hess, TrainCtl* ctl) {
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
__global__ void grad_kernel(const double* __restrict__ pred, const double* __restrict__ target, int64_t n,
                            double* __restrict__ grad, double* __restrict__ hess, TrainCtl* ctl) {
    pdl_wait();
    grad_phase(pred, target, n, grad, hess, ctl);
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
__device__ __forceinline__ void gather_phase(const int32_t* lists, int64_t n, int nl, const double* grad,
                                             const double* hess, const double* feats, double* gl, double* hl,
                                             double* fv, int lvl, const TrainCtl* ctl, int32_t* segmap) {
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
__global__ void gather_kernel(const int32_t* __restrict__ lists, int64_t n, int nl, const double* __restrict__ grad,
                              const double* __restrict__ hess, const double* __restrict__ feats,
                              double* __restrict__ gl, double* __restrict__ hl, double* __restrict__ fv, int lvl,
                              const TrainCtl* __restrict__ ctl, int32_t* __restrict__ segmap) {
    pdl_wait();
    gather_phase(lists, n, nl, grad, hess, feats, gl, hl, fv, lvl, ctl, segmap);
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

// One (list l, frontier segment k) chain by a 64-thread slot: warp 1 streams chunks in
// (cp.async, two buffers) and the prefixes out, warp 0 only chains (lanes 0/1), so the
// chain never waits on memory.  Named barriers bar0+b ("buffer b full") and bar0+2+b
// ("buffer b chained") hand the buffers over; ig/ih are two (kChunk + 8)-double buffers
// each.  Prefixes overwrite their operands in place (each operand is in registers by then).
__device__ __forceinline__ void chain_task(int64_t n, int b, int l, int k, const double* gl, const double* hl,
                                           double* pg, double* ph, TrainCtl* ctl, double* ig, double* ih,
                                           int bar0, int warp, int lane) {
    constexpr int kBuf = kChunk + 8;
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
                cp_async8(&ig[bb * kBuf + j], G + base + j);
                cp_async8(&ih[bb * kBuf + j], Hh + base + j);
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
        bar_arrive(bar0);  // chunk 0 in buffer 0
        for (int c = 0; c < nch; ++c) {
            const int bb = c & 1;
            if (c + 1 < nch) {
                cp_async_wait_all();  // chunk c+1 (the only group in flight)
                bar_arrive(bar0 + (bb ^ 1));
            }
            bar_sync(bar0 + 2 + bb);  // chunk c chained in place
            if (prefixes) {
                const int base = s + c * kChunk, cnt = min(kChunk, e - base);
                for (int j = lane; j < cnt; j += 32) {
                    PG[base + j] = ig[bb * kBuf + j];
                    PH[base + j] = ih[bb * kBuf + j];
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
        bar_sync(bar0 + bb);
        if (lane < 2) {
            double* cx = (lane == 0 ? ig : ih) + bb * kBuf;
            double2* c2 = reinterpret_cast<double2*>(cx);
            const int nb = cnt >> 3;
            const int full = nb << 3;
            double2 xa[4], xb[4];
            auto ld = [&](double2* x, int bi) {
#pragma unroll
                for (int q = 0; q < 4; ++q) x[q] = c2[bi * 4 + q];
            };
            auto run = [&](const double2* x, int bi) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    double2 pv;
                    pv.x = racc;
                    racc = __dadd_rn(racc, x[q].x);
                    pv.y = racc;
                    racc = __dadd_rn(racc, x[q].y);
                    c2[bi * 4 + q] = pv;
                }
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
        bar_arrive(bar0 + 2 + bb);
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

// graph path: one CTA (one slot) per (list, segment)
__global__ void __launch_bounds__(64) chain_kernel(int64_t n, int lvl, int only_totals,
                                                   const double* __restrict__ gl, const double* __restrict__ hl,
                                                   double* __restrict__ pg, double* __restrict__ ph, TrainCtl* ctl) {
    pdl_wait();
    __shared__ __align__(16) double ig[2 * (kChunk + 8)];
    __shared__ __align__(16) double ih[2 * (kChunk + 8)];
    const int b = lvl & 1;
    const int nseg = ctl->nseg[b];
    if (nseg <= 0) return;
    const int t = blockIdx.x;
    const int l = only_totals ? kSampleList : t / nseg;
    const int k = only_totals ? t : t % nseg;
    if (k >= nseg || l >= kLists) return;
    chain_task(n, b, l, k, gl, hl, pg, ph, ctl, ig, ih, 1, threadIdx.x >> 5, threadIdx.x & 31);
}

// split gain at every (feature list, position) (cpp 97-118); per-(node, feature) max
// gain by atomicMax on the (positive) gain's bits
__device__ __forceinline__ void gain_phase(int64_t n, int lvl, const int32_t* segmap, const double* fv,
                                           const double* pg, const double* ph, double mlw, double lambda,
                                           double* gains, TrainCtl* ctl) {
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
__global__ void gain_kernel(int64_t n, int lvl, const int32_t* __restrict__ segmap, const double* __restrict__ fv,
                            const double* __restrict__ pg, const double* __restrict__ ph, double mlw, double lambda,
                            double* __restrict__ gains, TrainCtl* ctl) {
    pdl_wait();
    gain_phase(n, lvl, segmap, fv, pg, ph, mlw, lambda, gains, ctl);
}

// earliest position attaining the max (ties: the reference's strict > keeps the first)
__device__ __forceinline__ void gainpos_phase(int64_t n, const int32_t* segmap, const double* gains, TrainCtl* ctl) {
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
__global__ void gainpos_kernel(int64_t n, const int32_t* __restrict__ segmap, const double* __restrict__ gains,
                               TrainCtl* ctl) {
    pdl_wait();
    gainpos_phase(n, segmap, gains, ctl);
}

// One CTA: choose each node's split (features in order, strictly larger gain wins,
// cpp 111-117), allocate children in frontier order (cpp 130-143).
__device__ __forceinline__ void decide_phase(int64_t n, int lvl, const double* fv, TrainCtl* ctl) {
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
            unsigned long long bits[kF];  // all 16 loads in flight, then the scan in feature order
#pragma unroll
            for (int f = 0; f < kF; ++f) bits[f] = ctl->gbits[k][f];
#pragma unroll
            for (int f = 0; f < kF; ++f) {
                if (bits[f] == 0ull) continue;
                const double g = __longlong_as_double(static_cast<long long>(bits[f]));
                if (g > kMinSplitGain && g > bg) {
                    bg = g;
                    bf = f;
                }
            }
            if (bf >= 0) {
                const int64_t pos = ctl->gpos[k][bf];
                const double* F = fv + int64_t(bf) * n;
                bt = __dmul_rn(0.5, __dadd_rn(F[pos - 1], F[pos]));  // cpp 115-116
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
            ctl->sfeat[k] = bf;
            ctl->sthr[k] = bt;
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
__global__ void __launch_bounds__(1024) decide_kernel(int64_t n, int lvl, const double* __restrict__ fv,
                                                      TrainCtl* ctl) {
    pdl_wait();
    decide_phase(n, lvl, fv, ctl);
}

struct LeftFlagFn {  // routing flag of list position q (0 outside split segments), cpp 146-148
    const int32_t* lists;
    const int32_t* segmap;
    const TrainCtl* ctl;
    const double* feats;
    int64_t n;
    __device__ int64_t operator()(int64_t q) const {
        const int k = segmap[q % n];
        const int f = k >= 0 ? ctl->sfeat[k] : -1;
        if (f < 0) return 0;
        return feats[int64_t(lists[q]) * kF + f] < ctl->sthr[k] ? 1 : 0;
    }
};
struct PrefixWrite {
    int64_t* pfx;
    __device__ void operator()(int64_t q, int64_t ex) const { pfx[q] = ex; }
};

// Stable partition of every split segment into [left | right] in every list (list 16
// also writes the children's segment bounds), fused with the next level's gather: each
// element's (grad, hess, feature value) row and segment (2r / 2r + 1 for the children
// of split rank r, -1 for a leaf's range) are written at its destination.
__device__ __forceinline__ void scatter_phase(const int32_t* src, int32_t* dst, const int64_t* pfx,
                                              const int32_t* segmap, int32_t* nsegmap, int64_t n, int lvl,
                                              TrainCtl* ctl, const double* grad, const double* hess,
                                              const double* feats, double* gl, double* hl, double* fv) {
    const int b = lvl & 1;
    const int64_t tot = int64_t(kLists) * n;
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t l = q / n, p = q % n;
        const int k = segmap[p];
        const int r = k >= 0 ? ctl->split[k] : -1;
        int64_t d = p;
        int nk = -1;
        if (r >= 0) {
            const int64_t s = ctl->seg_start[b][k], e = ctl->seg_end[b][k];
            const int64_t* P = pfx + l * n;
            const int64_t pl = P[p] - P[s];
            const int64_t L = P[e] - P[s];
            const int64_t left = P[p + 1] - P[p];
            d = left ? s + pl : s + L + (p - s - pl);
            nk = left ? 2 * r : 2 * r + 1;
            if (l == kSampleList && p == s) {
                ctl->seg_start[b ^ 1][2 * r] = int32_t(s);
                ctl->seg_end[b ^ 1][2 * r] = int32_t(s + L);
                ctl->seg_start[b ^ 1][2 * r + 1] = int32_t(s + L);
                ctl->seg_end[b ^ 1][2 * r + 1] = int32_t(e);
            }
        }
        const int32_t idx = src[q];
        const int64_t g = l * n + d;
        dst[g] = idx;
        gl[g] = grad[idx];
        hl[g] = hess[idx];
        if (l < kF) fv[g] = feats[int64_t(idx) * kF + l];
        else nsegmap[d] = nk;
    }
}
__global__ void scatter_kernel(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                               const int64_t* __restrict__ pfx, const int32_t* __restrict__ segmap,
                               int32_t* __restrict__ nsegmap, int64_t n, int lvl, TrainCtl* ctl,
                               const double* __restrict__ grad, const double* __restrict__ hess,
                               const double* __restrict__ feats, double* __restrict__ gl, double* __restrict__ hl,
                               double* __restrict__ fv) {
    pdl_wait();
    scatter_phase(src, dst, pfx, segmap, nsegmap, n, lvl, ctl, grad, hess, feats, gl, hl, fv);
}

// Leaf Newton weights (cpp 161-166) and the tree appended to the output forest.
__device__ __forceinline__ void finalize_phase(double lambda, TrainCtl* ctl, int32_t* o_feature, double* o_thr,
                                               int32_t* o_left, int32_t* o_right, double* o_value,
                                               int64_t* o_off) {
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
__global__ void __launch_bounds__(1024) finalize_kernel(double lambda, TrainCtl* ctl,
                                                       int32_t* __restrict__ o_feature, double* __restrict__ o_thr,
                                                       int32_t* __restrict__ o_left, int32_t* __restrict__ o_right,
                                                       double* __restrict__ o_value, int64_t* __restrict__ o_off) {
    pdl_wait();
    finalize_phase(lambda, ctl, o_feature, o_thr, o_left, o_right, o_value, o_off);
}

// pred[i] += lr * tree.eval(feat[i])  (cpp 236-238)
__device__ __forceinline__ void update_phase(const double* feats, int64_t n, double lr, const TrainCtl* ctl,
                                             double* pred) {
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
__global__ void update_kernel(const double* __restrict__ feats, int64_t n, double lr, const TrainCtl* __restrict__ ctl,
                              double* __restrict__ pred) {
    pdl_wait();
    update_phase(feats, n, lr, ctl, pred);
}

__device__ __forceinline__ void loss_phase(const double* pred, const double* target, int64_t n, const TrainCtl* ctl,
                                           double* loss, double* tmp) {
    __shared__ double stage[1024 + 8];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = __dsub_rn(pred[i], target[i]);
        tmp[i] = __ddiv_rn(__dmul_rn(d, d), target[i]);
    }
    __syncthreads();
    const double tot = cta_sequential_sum(tmp, n, stage);
    if (threadIdx.x == 0) loss[ctl->tree] = __ddiv_rn(tot, static_cast<double>(n));  // after finalize: round t+1
}
__global__ void __launch_bounds__(1024) loss_kernel(const double* __restrict__ pred,
                                                   const double* __restrict__ target, int64_t n,
                                                   const TrainCtl* __restrict__ ctl, double* __restrict__ loss,
                                                   double* __restrict__ tmp) {
    pdl_wait();
    loss_phase(pred, target, n, ctl, loss, tmp);
}

// ------------------------------------------------------------ megakernel
// Opt-in alternative (ETUNE_TRAIN_MEGA=1): the whole training (every tree, every
// level) as ONE cooperative launch, the phases above separated by grid-wide barriers
// instead of kernel boundaries.  Every CTA (one per SM) runs kMegaSlots chain slots of
// 64 threads (named barriers 1..12) over dynamic shared memory.  Measured slower than
// the PDL graph ("Training"): with one 512-thread CTA per SM the grid-wide
// phases have 4x fewer loads in flight than the graph's 1-element-per-thread grids,
// and 128 registers per thread leave the chains ~20% slower; kept as a parity-tested
// variant.
constexpr int kMegaSlots = 3;
constexpr int kMegaT = 512;  // warps 0..5: chain slots; all 16 warps run the grid-wide phases
constexpr size_t kMegaSmem = size_t(kMegaSlots) * 4 * (kChunk + 8) * sizeof(double);

struct MegaArgs {
    int64_t n;
    int num_trees, max_depth;
    double lr, mlw, lambda;
    const double* feats;
    const double* target;
    double *pred, *grad, *hess, *gl, *hl, *fv, *pg, *ph, *gains;
    const int32_t* base_lists;
    int32_t* work[2];
    int32_t* segmap[2];
    int64_t* pfx;
    int64_t* sums;
    TrainCtl* ctl;
    int32_t *o_feature, *o_left, *o_right;
    double *o_thr, *o_value, *o_loss;
    int64_t* o_off;
    unsigned long long* trace;  // diagnostic: %globaltimer after every barrier of tree 0 (or null)
};

// routing flag of list position q at frontier parity b (leftflag_kernel + LeftFlagFn)
__device__ __forceinline__ int64_t mega_flag(const MegaArgs& a, const int32_t* cur, const int32_t* segmap, int b,
                                             int64_t q) {
    const int k = segmap[q % a.n];
    const int f = k >= 0 ? a.ctl->sfeat[k] : -1;
    if (f < 0) return 0;
    const int32_t idx = cur[q];
    return a.feats[int64_t(idx) * kF + f] < a.ctl->sthr[k] ? 1 : 0;
}

// the CTA's contiguous share [r0, r1) of the L list positions
__device__ __forceinline__ void mega_range(int64_t L, int64_t* r0, int64_t* r1) {
    const int64_t per = (L + gridDim.x - 1) / gridDim.x;
    *r0 = min(L, int64_t(blockIdx.x) * per);
    *r1 = min(L, *r0 + per);
}

__global__ void __launch_bounds__(kMegaT, 1) train_mega_kernel(const __grid_constant__ MegaArgs a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double mega_smem[];
    const int slot = threadIdx.x >> 6, warp = (threadIdx.x >> 5) & 1, lane = threadIdx.x & 31;
    double* ig = mega_smem + slot * 4 * (kChunk + 8);
    double* ih = ig + 2 * (kChunk + 8);
    const int bar0 = 1 + 4 * slot;
    const int64_t n = a.n, L = int64_t(kLists) * n;
    TrainCtl* ctl = a.ctl;
    const bool chainer = threadIdx.x < 64 * kMegaSlots;
    // task t -> CTA t % grid: one chain per SM before any SM takes a second
    const int slot_id = slot * gridDim.x + blockIdx.x, nslots = gridDim.x * kMegaSlots;
    int tick = 0;
    auto sync = [&]() {
        grid.sync();
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && tick < 256) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[tick] = t;
        }
        ++tick;
    };
    for (int tree = 0; tree < a.num_trees; ++tree) {
        grad_phase(a.pred, a.target, n, a.grad, a.hess, ctl);
        sync();
        gather_phase(a.base_lists, n, kLists, a.grad, a.hess, a.feats, a.gl, a.hl, a.fv, 0, ctl, a.segmap[0]);
        sync();
        const int32_t* cur = a.base_lists;
        for (int depth = 0; depth < a.max_depth; ++depth) {
            const int b = depth & 1;
            const int nseg = ctl->nseg[b];
            for (int t = slot_id; chainer && t < kLists * nseg; t += nslots)
                chain_task(n, b, t / nseg, t % nseg, a.gl, a.hl, a.pg, a.ph, ctl, ig, ih, bar0, warp, lane);
            sync();
            gain_phase(n, b, a.segmap[b], a.fv, a.pg, a.ph, a.mlw, a.lambda, a.gains, ctl);
            sync();
            gainpos_phase(n, a.segmap[b], a.gains, ctl);
            sync();
            if (blockIdx.x == 0) decide_phase(n, b, a.fv, ctl);
            sync();
            // global exclusive scan of the left flags: CTA counts, then CTA prefixes
            int64_t r0, r1, tot;
            mega_range(L, &r0, &r1);
            int64_t cnt = 0;
            for (int64_t q = r0 + threadIdx.x; q < r1; q += blockDim.x) cnt += mega_flag(a, cur, a.segmap[b], b, q);
            block_excl_scan(cnt, &tot);
            if (threadIdx.x == 0) a.sums[blockIdx.x] = tot;
            sync();
            int64_t carry = 0;
            for (int i0 = 0; i0 < int(blockIdx.x); i0 += blockDim.x) {
                const int i = i0 + threadIdx.x;
                block_excl_scan(i < int(blockIdx.x) ? a.sums[i] : 0, &tot);
                carry += tot;
            }
            for (int64_t q0 = r0; q0 < r1; q0 += blockDim.x) {
                const int64_t q = q0 + threadIdx.x;
                const int64_t ex = block_excl_scan(q < r1 ? mega_flag(a, cur, a.segmap[b], b, q) : 0, &tot);
                if (q < r1) a.pfx[q] = carry + ex;
                carry += tot;
            }
            if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) a.pfx[L] = carry;
            sync();
            int32_t* dst = a.work[b];
            scatter_phase(cur, dst, a.pfx, a.segmap[b], a.segmap[b ^ 1], n, b, ctl, a.grad, a.hess, a.feats, a.gl,
                          a.hl, a.fv);
            sync();
            cur = dst;
        }
        // totals of the last frontier, leaf values, the tree appended, predictions
        {
            const int b = a.max_depth & 1;
            const int nseg = ctl->nseg[b];
            for (int t = slot_id; chainer && t < nseg; t += nslots)
                chain_task(n, b, kSampleList, t, a.gl, a.hl, a.pg, a.ph, ctl, ig, ih, bar0, warp, lane);
        }
        sync();
        if (blockIdx.x == 0)
            finalize_phase(a.lambda, ctl, a.o_feature, a.o_thr, a.o_left, a.o_right, a.o_value, a.o_off);
        sync();
        update_phase(a.feats, n, a.lr, ctl, a.pred);
        sync();
        if (a.o_loss && blockIdx.x == 0) loss_phase(a.pred, a.target, n, ctl, a.o_loss, a.gains);
    }
}

int64_t pow2_at_least(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// ETUNE_TRAIN_TRACE=1 (diagnostic): the megakernel records a timestamp after every grid
// barrier into a managed buffer, printed to stderr by the next launch_train
unsigned long long* train_trace_buffer() {
    static unsigned long long* buf = nullptr;
    static bool init = false;
    if (!init) {
        init = true;
        const char* ev = std::getenv("ETUNE_TRAIN_TRACE");
        if (ev && std::atoi(ev) > 0 && cudaMallocManaged(&buf, 256 * sizeof(unsigned long long)) != cudaSuccess)
            buf = nullptr;
    } else if (buf) {
        cudaDeviceSynchronize();
        for (int i = 1; i < 256 && buf[i] > buf[i - 1]; ++i)
            std::fprintf(stderr, "mega %3d %8.2f us\n", i, double(buf[i] - buf[i - 1]) * 1e-3);
    }
    if (buf) std::memset(buf, 0, 256 * sizeof(unsigned long long));
    return buf;
}

// CTAs per SM for the megakernel on the current device (0: use the tree graph)
int train_mega_ctas_per_sm() {
    static int cached[64];
    static bool init[64];
    int device = -1;
    cudaGetDevice(&device);
    if (device < 0 || device >= 64) return 0;
    if (init[device]) return cached[device];
    int want = 0;
    if (const char* ev = std::getenv("ETUNE_TRAIN_MEGA")) want = std::atoi(ev);
    int coop = 0, occ = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (want > 0 && coop &&
        cudaFuncSetAttribute(train_mega_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMegaSmem)) ==
            cudaSuccess &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, train_mega_kernel, kMegaT, kMegaSmem) == cudaSuccess)
        want = std::min(want, occ);
    else
        want = 0;
    cudaGetLastError();
    cached[device] = want;
    init[device] = true;
    return want;
}

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
           + 2 * al256(4 * size_t(n))                             // segment maps
           + al256(8 * ((L + 1023) / 1024 + 4096))                // scan tile / CTA sums
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
    int32_t* segmap2 = reinterpret_cast<int32_t*>(take(4 * size_t(n)));
    int64_t* sums = reinterpret_cast<int64_t*>(take(8 * ((L + 1023) / 1024 + 4096)));
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

    // ETUNE_TRAIN_MEGA=1: the whole training as one cooperative launch (default: the
    // per-kernel tree graph below)
    if (const int per_sm = train_mega_ctas_per_sm(); per_sm > 0) {
        MegaArgs a{};
        a.n = n;
        a.num_trees = num_trees;
        a.max_depth = max_depth;
        a.lr = lr;
        a.mlw = mlw;
        a.lambda = lambda;
        a.feats = d_feat;
        a.target = target;
        a.pred = pred;
        a.grad = grad;
        a.hess = hess;
        a.gl = gl;
        a.hl = hl;
        a.fv = fv;
        a.pg = pg;
        a.ph = ph;
        a.gains = gains;
        a.base_lists = base_lists;
        a.work[0] = work[0];
        a.work[1] = work[1];
        a.segmap[0] = segmap;
        a.segmap[1] = segmap2;
        a.pfx = pfx;
        a.sums = sums;
        a.ctl = ctl;
        a.o_feature = o_feature;
        a.o_left = o_left;
        a.o_right = o_right;
        a.o_thr = o_thr;
        a.o_value = o_value;
        a.o_loss = o_loss;
        a.o_off = o_off;
        a.trace = train_trace_buffer();
        void* args[] = {&a};
        cudaError_t em = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(train_mega_kernel),
                                                     dim3(unsigned(c.sm_count * per_sm)), dim3(kMegaT), args,
                                                     kMegaSmem, c.stream);
        note_launches(1);
        if (em == cudaSuccess)
            em = cudaMemcpyAsync(o_scalars, &ctl->base, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
        return em;
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
    // level 0 rows and segment map; every later level's come from the previous scatter
    PDL(gather_kernel, grid(int64_t(L)), 256, 0, cap, cur, n, kLists, grad, hess, d_feat, gl, hl, fv, 0, ctl, segmap);
    launches += 1;
    int32_t* segmaps[2] = {segmap, segmap2};
    for (int depth = 0; depth < max_depth; ++depth, ++lvl) {
        const int b = lvl & 1;
        const int segs = 1 << depth;  // frontier bound at this depth
        const int warps = kLists * segs;
        PDL(chain_kernel, warps, 64, 0, cap, n, lvl, 0, gl, hl, pg, ph, ctl);
        PDL(gain_kernel, grid(int64_t(F)), 256, 0, cap, n, lvl, segmaps[b], fv, pg, ph, mlw, lambda, gains, ctl);
        PDL(gainpos_kernel, grid(int64_t(F)), 256, 0, cap, n, segmaps[b], gains, ctl);
        PDL(decide_kernel, 1, 1024, 0, cap, n, lvl, fv, ctl);
        if (e == cudaSuccess)
            e = scan_apply(cap, int64_t(L), LeftFlagFn{cur, segmaps[b], ctl, d_feat, n}, PrefixWrite{pfx}, sums,
                           pfx + L);
        if (e != cudaSuccess) break;
        PDL(scatter_kernel, grid(int64_t(L)), 256, 0, cap, cur, work[wb], pfx, segmaps[b], segmaps[b ^ 1], n, lvl,
            ctl, grad, hess, d_feat, gl, hl, fv);
        cur = work[wb];
        wb ^= 1;
        launches += 8;
    }
    // totals of the last frontier (children created at the deepest level)
    const int segs = 1 << max_depth;
    PDL(chain_kernel, segs, 64, 0, cap, n, lvl, 1, gl, hl, pg, ph, ctl);
    PDL(finalize_kernel, 1, 1024, 0, cap, lambda, ctl, o_feature, o_thr, o_left, o_right, o_value, o_off);
    PDL(update_kernel, grid(n), 256, 0, cap, d_feat, n, lr, ctl, pred);
    launches += 3;
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
