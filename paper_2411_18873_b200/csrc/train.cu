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
// Every kernel reads the data-dependent frontier size from device memory, so a whole
// training is one launch sequence with no host synchronisation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "etune_internal.hpp"
#include "kernels.hpp"

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
    int32_t pad;
    int64_t out_nodes;        // nodes written to the output forest so far
    // current tree
    int32_t feature[kMaxNodes], left[kMaxNodes], right[kMaxNodes];
    double thr[kMaxNodes], value[kMaxNodes], sg[kMaxNodes], sh[kMaxNodes];
    // per (segment, feature) best split candidate
    double bgain[kMaxSeg][kF], bthr[kMaxSeg][kF];
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
// reference energy (min), NonPositiveEnergy check, targets, harmonic-mean base score
// (one sequential chain, energy_model.cpp:199-202), pred = base.
__global__ void __launch_bounds__(1024) init_kernel(const double* __restrict__ energy, int64_t n,
                                                   double* __restrict__ target, double* __restrict__ pred,
                                                   TrainCtl* ctl, unsigned long long* err,
                                                   double* __restrict__ loss0) {
    __shared__ double red[32];
    __shared__ int bad;
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
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) target[i] = __ddiv_rn(energy[i], ref);
    __syncthreads();
    __shared__ double s_base;
    if (threadIdx.x == 0) {
        double inv = 0.0;
        for (int64_t i = 0; i < n; ++i) inv = __dadd_rn(inv, __ddiv_rn(1.0, target[i]));
        s_base = __ddiv_rn(static_cast<double>(n), inv);
        ctl->base = s_base;
        ctl->reference = ref;
        ctl->out_nodes = 0;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) pred[i] = s_base;
    if (loss0 && threadIdx.x == 0) {  // mean_loss() before any tree (cpp 221-227)
        double tot = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double d = __dsub_rn(s_base, target[i]);
            tot = __dadd_rn(tot, __ddiv_rn(__dmul_rn(d, d), target[i]));
        }
        loss0[0] = __ddiv_rn(tot, static_cast<double>(n));
    }
}

// ----------------------------------------------------------------- sort
// One CTA per feature: bitonic sort of (order_key(value), index) pairs in global
// memory == std::stable_sort by value (energy_model.cpp:204-213); list 16 = identity.
__global__ void __launch_bounds__(1024) sort_kernel(const double* __restrict__ feats, int64_t n, int64_t n2,
                                                   uint64_t* __restrict__ kbuf, uint32_t* __restrict__ ibuf,
                                                   int32_t* __restrict__ lists) {
    const int f = blockIdx.x;
    int32_t* out = lists + int64_t(f) * n;
    if (f == kSampleList) {
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = int32_t(i);
        return;
    }
    uint64_t* K = kbuf + int64_t(f) * n2;
    uint32_t* I = ibuf + int64_t(f) * n2;
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

// gl/hl[l][pos] = grad/hess[list[l][pos]]: the chains below then stream contiguously
__global__ void gather_kernel(const int32_t* __restrict__ lists, int64_t n, int nl, const double* __restrict__ grad,
                              const double* __restrict__ hess, double* __restrict__ gl, double* __restrict__ hl) {
    const int64_t tot = int64_t(nl) * n;
    const int64_t off = int64_t(kLists - nl) * n;  // nl == 1: sample list only
    for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < tot; q += int64_t(gridDim.x) * blockDim.x) {
        const int32_t idx = lists[off + q];
        gl[off + q] = grad[idx];
        hl[off + q] = hess[idx];
    }
}

// One thread per (list, frontier segment): the sequential running sums.
//   lists 0..15: exclusive prefix at every position (the `run` of cpp 95-121)
//   list 16:     the node's (grad, hess) totals in sample order (cpp 73-76, 150-155)
__global__ void chain_kernel(int64_t n, int lvl, int only_totals, const double* __restrict__ gl,
                             const double* __restrict__ hl, double* __restrict__ pg, double* __restrict__ ph,
                             TrainCtl* ctl) {
    const int b = lvl & 1;
    const int nseg = ctl->nseg[b];
    if (nseg <= 0) return;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = only_totals ? kSampleList : t / nseg;
    const int k = only_totals ? t : t % nseg;
    if (k >= nseg || l >= kLists) return;
    const int s = ctl->seg_start[b][k], e = ctl->seg_end[b][k];
    const double* G = gl + int64_t(l) * n;
    const double* Hh = hl + int64_t(l) * n;
    double rg = 0.0, rh = 0.0;
    if (l == kSampleList) {
        for (int p = s; p < e; ++p) {
            rg = __dadd_rn(rg, G[p]);
            rh = __dadd_rn(rh, Hh[p]);
        }
        const int node = ctl->seg_node[b][k];
        ctl->sg[node] = rg;
        ctl->sh[node] = rh;
        return;
    }
    double* PG = pg + int64_t(l) * n;
    double* PH = ph + int64_t(l) * n;
    for (int p = s; p < e; ++p) {
        PG[p] = rg;
        PH[p] = rh;
        rg = __dadd_rn(rg, G[p]);
        rh = __dadd_rn(rh, Hh[p]);
    }
}

// One CTA per (segment, feature): best split of this node on this feature.
__global__ void __launch_bounds__(256) gain_kernel(const double* __restrict__ feats, const int32_t* __restrict__ lists,
                                                   int64_t n, int lvl, const double* __restrict__ pg,
                                                   const double* __restrict__ ph, double mlw, double lambda,
                                                   TrainCtl* ctl) {
    const int b = lvl & 1;
    const int k = blockIdx.x, f = blockIdx.y;
    if (k >= ctl->nseg[b]) return;
    const int s = ctl->seg_start[b][k], e = ctl->seg_end[b][k];
    const int node = ctl->seg_node[b][k];
    const double tg = ctl->sg[node], th = ctl->sh[node];
    const double tobj = obj(tg, th, lambda);
    const int32_t* L = lists + int64_t(f) * n;
    const double* PG = pg + int64_t(f) * n;
    const double* PH = ph + int64_t(f) * n;
    double best = 0.0, bthr = 0.0;
    int bpos = 0x7fffffff;
    for (int p = s + 1 + int(threadIdx.x); p < e; p += blockDim.x) {
        const double v = feats[int64_t(L[p]) * kF + f];
        const double pv = feats[int64_t(L[p - 1]) * kF + f];
        if (!(v > pv)) continue;
        const double rg = PG[p], rh = PH[p];
        const double qg = __dsub_rn(tg, rg), qh = __dsub_rn(th, rh);
        if (!(rh >= mlw && qh >= mlw)) continue;
        const double gain = __dmul_rn(0.5, __dsub_rn(__dadd_rn(obj(rg, rh, lambda), obj(qg, qh, lambda)), tobj));
        if (gain > kMinSplitGain && (gain > best || (gain == best && p < bpos))) {
            best = gain;
            bpos = p;
            bthr = __dmul_rn(0.5, __dadd_rn(pv, v));
        }
    }
    // block argmax: larger gain, then smaller position
    __shared__ double sgain[256], sthr[256];
    __shared__ int spos[256];
    sgain[threadIdx.x] = best;
    spos[threadIdx.x] = bpos;
    sthr[threadIdx.x] = bthr;
    __syncthreads();
    for (int st = blockDim.x >> 1; st > 0; st >>= 1) {
        if (int(threadIdx.x) < st) {
            const int o = threadIdx.x + st;
            if (sgain[o] > sgain[threadIdx.x] || (sgain[o] == sgain[threadIdx.x] && spos[o] < spos[threadIdx.x])) {
                sgain[threadIdx.x] = sgain[o];
                spos[threadIdx.x] = spos[o];
                sthr[threadIdx.x] = sthr[o];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctl->bgain[k][f] = spos[0] == 0x7fffffff ? 0.0 : sgain[0];
        ctl->bthr[k][f] = sthr[0];
    }
}

// One CTA: choose each node's split (features in order, strictly larger gain wins,
// cpp 111-117), allocate children in frontier order (cpp 130-143).
__global__ void __launch_bounds__(1024) decide_kernel(int lvl, TrainCtl* ctl) {
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
                const double g = ctl->bgain[k][f];
                if (g > kMinSplitGain && g > bg) {
                    bg = g;
                    bf = f;
                    bt = ctl->bthr[k][f];
                }
            }
        }
        const int flag = bf >= 0;
        // exclusive scan of flags over the block
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

// One CTA per list: stable partition of every split segment into [left | right]
// (value < threshold goes left, cpp 146-148).  List 16 also writes the children's
// segment bounds.
__global__ void __launch_bounds__(1024) partition_kernel(const double* __restrict__ feats,
                                                        const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                                                        int32_t* __restrict__ pre, int64_t n, int lvl,
                                                        TrainCtl* ctl) {
    const int b = lvl & 1;
    const int l = blockIdx.x;
    const int nseg = ctl->nseg[b];
    const int32_t* S = src + int64_t(l) * n;
    int32_t* D = dst + int64_t(l) * n;
    int32_t* P = pre + int64_t(l) * (n + 1);
    __shared__ int wsum[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int* ss = ctl->seg_start[b];
    const int* se = ctl->seg_end[b];
    auto seg_of = [&](int64_t p) -> int {  // active segment containing p, or -1
        int lo = 0, hi = nseg;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (ss[mid] <= p) lo = mid + 1;
            else hi = mid;
        }
        const int k = lo - 1;
        return (k >= 0 && p < se[k]) ? k : -1;
    };
    auto goes_left = [&](int64_t p, int k) -> int {
        if (k < 0 || ctl->split[k] < 0) return 0;
        const int node = ctl->seg_node[b][k];
        return feats[int64_t(S[p]) * kF + ctl->feature[node]] < ctl->thr[node] ? 1 : 0;
    };
    // pass 1: exclusive prefix of left flags over the whole list
    const int64_t nr = (n + blockDim.x - 1) / blockDim.x * blockDim.x;
    for (int64_t p0 = 0; p0 < nr; p0 += blockDim.x) {
        const int64_t p = p0 + threadIdx.x;
        const int fl = p < n ? goes_left(p, seg_of(p)) : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, fl);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        if (lane == 0) wsum[w] = __popc(bal);
        __syncthreads();
        int before = carry + __popc(bal & ((1u << lane) - 1u));
        int total = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) {
            if (i < w) before += wsum[i];
            total += wsum[i];
        }
        if (p < n) P[p] = before;
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) P[n] = carry;
    __syncthreads();
    // pass 2: scatter
    for (int64_t p = threadIdx.x; p < n; p += blockDim.x) {
        const int k = seg_of(p);
        int64_t d = p;
        if (k >= 0 && ctl->split[k] >= 0) {
            const int s = ss[k], e = se[k];
            const int pl = P[p] - P[s];
            const int L = P[e] - P[s];
            const int left = P[p + 1] - P[p];
            d = left ? s + pl : s + L + (p - s - pl);
        }
        D[d] = S[p];
    }
    if (l == kSampleList) {
        for (int k = threadIdx.x; k < nseg; k += blockDim.x) {
            const int r = ctl->split[k];
            if (r < 0) continue;
            const int s = ss[k], e = se[k];
            const int L = P[e] - P[s];
            ctl->seg_start[b ^ 1][2 * r] = s;
            ctl->seg_end[b ^ 1][2 * r] = s + L;
            ctl->seg_start[b ^ 1][2 * r + 1] = s + L;
            ctl->seg_end[b ^ 1][2 * r + 1] = e;
        }
    }
}

// Leaf Newton weights (cpp 161-166) and the tree appended to the output forest.
__global__ void __launch_bounds__(1024) finalize_kernel(int tree, double lambda, TrainCtl* ctl,
                                                       int32_t* __restrict__ o_feature, double* __restrict__ o_thr,
                                                       int32_t* __restrict__ o_left, int32_t* __restrict__ o_right,
                                                       double* __restrict__ o_value, int64_t* __restrict__ o_off) {
    const int nn = ctl->nnodes;
    const int64_t base = ctl->out_nodes;
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
    }
}

// pred[i] += lr * tree.eval(feat[i])  (cpp 236-238)
__global__ void update_kernel(const double* __restrict__ feats, int64_t n, double lr, const TrainCtl* __restrict__ ctl,
                              double* __restrict__ pred) {
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

__global__ void loss_kernel(const double* __restrict__ pred, const double* __restrict__ target, int64_t n,
                            double* __restrict__ out) {
    double tot = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = __dsub_rn(pred[i], target[i]);
        tot = __dadd_rn(tot, __ddiv_rn(__dmul_rn(d, d), target[i]));
    }
    *out = __ddiv_rn(tot, static_cast<double>(n));
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
    return al256(sizeof(TrainCtl)) + 3 * al256(8 * size_t(n))         // target, pred, grad
           + al256(8 * size_t(n))                                       // hess
           + 4 * al256(8 * size_t(kLists) * n)                          // gl, hl, pg, ph
           + 3 * al256(4 * size_t(kLists) * n)                          // base lists + 2 work buffers
           + al256(4 * size_t(kLists) * (n + 1))                        // partition prefixes
           + al256(size_t(kF) * n2 * 12);                               // sort keys + indices
}

int train_max_depth() { return kMaxDepth; }

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
    TrainCtl* ctl = reinterpret_cast<TrainCtl*>(take(sizeof(TrainCtl)));
    double* target = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* pred = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* grad = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* hess = reinterpret_cast<double*>(take(8 * size_t(n)));
    double* gl = reinterpret_cast<double*>(take(8 * size_t(kLists) * n));
    double* hl = reinterpret_cast<double*>(take(8 * size_t(kLists) * n));
    double* pg = reinterpret_cast<double*>(take(8 * size_t(kLists) * n));
    double* ph = reinterpret_cast<double*>(take(8 * size_t(kLists) * n));
    int32_t* base_lists = reinterpret_cast<int32_t*>(take(4 * size_t(kLists) * n));
    int32_t* work[2] = {reinterpret_cast<int32_t*>(take(4 * size_t(kLists) * n)),
                        reinterpret_cast<int32_t*>(take(4 * size_t(kLists) * n))};
    int32_t* pre = reinterpret_cast<int32_t*>(take(4 * size_t(kLists) * (n + 1)));
    uint64_t* kbuf = reinterpret_cast<uint64_t*>(take(size_t(kF) * n2 * 12));
    uint32_t* ibuf = reinterpret_cast<uint32_t*>(kbuf + size_t(kF) * n2);

    const int ew = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
    init_kernel<<<1, 1024, 0, c.stream>>>(d_energy, n, target, pred, ctl, c.d_err, o_loss);
    sort_kernel<<<kLists, 1024, 0, c.stream>>>(d_feat, n, n2, kbuf, ibuf, base_lists);
    int launches = 2;
    for (int t = 0; t < num_trees; ++t) {
        grad_kernel<<<ew, 256, 0, c.stream>>>(pred, target, n, grad, hess, ctl);
        const int32_t* cur = base_lists;
        int wb = 0;
        int lvl = 0;
        for (int depth = 0; depth < max_depth; ++depth, ++lvl) {
            const int segs = 1 << depth;  // frontier bound at this depth
            gather_kernel<<<int(std::min<int64_t>((kLists * n + 255) / 256, int64_t(c.sm_count) * 16)), 256, 0,
                            c.stream>>>(cur, n, kLists, grad, hess, gl, hl);
            const int chains = kLists * segs;
            chain_kernel<<<(chains + 63) / 64, 64, 0, c.stream>>>(n, lvl, 0, gl, hl, pg, ph, ctl);
            gain_kernel<<<dim3(segs, kF), 256, 0, c.stream>>>(d_feat, cur, n, lvl, pg, ph, mlw, lambda, ctl);
            decide_kernel<<<1, 1024, 0, c.stream>>>(lvl, ctl);
            partition_kernel<<<kLists, 1024, 0, c.stream>>>(d_feat, cur, work[wb], pre, n, lvl, ctl);
            cur = work[wb];
            wb ^= 1;
            launches += 5;
        }
        // totals of the last frontier (children created at the deepest level)
        gather_kernel<<<int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 16)), 256, 0, c.stream>>>(
            cur, n, 1, grad, hess, gl, hl);
        const int segs = 1 << max_depth;
        chain_kernel<<<(segs + 63) / 64, 64, 0, c.stream>>>(n, lvl, 1, gl, hl, pg, ph, ctl);
        finalize_kernel<<<1, 1024, 0, c.stream>>>(t, lambda, ctl, o_feature, o_thr, o_left, o_right, o_value, o_off);
        update_kernel<<<ew, 256, 0, c.stream>>>(d_feat, n, lr, ctl, pred);
        launches += 4;
        if (o_loss) {
            loss_kernel<<<1, 1, 0, c.stream>>>(pred, target, n, o_loss + t + 1);
            launches += 1;
        }
    }
    if (num_trees == 0) {
        cudaMemsetAsync(o_off, 0, sizeof(int64_t), c.stream);
    }
    // base score + reference energy
    cudaMemcpyAsync(o_scalars, &ctl->base, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
    note_launches(launches);
    return cudaGetLastError();
}

}  // namespace etune_b200
