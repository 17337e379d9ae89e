// reproduce() on the device, bit-exact with the reference's single sequential
// std::mt19937_64 stream (genetic.cpp:137-187).
//
// The obstacle: offspring i consumes a data-dependent number of RNG words
// (1 for a copy, 2-5 for a mutation, >=3 for a crossover, plus rejection and repair
// draws), so offspring i's first word index o_i is a sequential prefix over
// everything before it.  breed_kernel resolves that chain on one CTA per call by
// speculation:
//
//   1. The CTA owns the MT19937-64 state and generates the reference's word stream
//      itself, 312 words per cooperative twist, into a shared-memory ring
//      (the stream never goes to HBM).
//   2. Each round lays out a window of candidate start offsets for the next J
//      offspring (level j centred on j*mean words, +-~4 sd*sqrt(j)), and the 1024
//      threads evaluate breed_one() at every (level, offset) cell in parallel:
//      words consumed, the child genome and the crossover partner.
//   3. One thread walks the chain through the cells (o_{i+1} = o_i + words(i, o_i)),
//      stopping at the first level whose true offset fell outside its window; the
//      resolved children are written out and the next round starts there.
//
// Every resolved child is therefore the exact evaluation at its true offset: the
// speculation only affects speed (how many levels a round resolves), never results.
// The per-offspring work uses the plan's knob tables (tilings in
// enumerate_dim_tilings order, divisors of K), so mutate_knob / pick_different /
// repair_schedule reduce to index arithmetic on the 8-byte genome.
#include <cuda_runtime.h>

#include <cstdint>

#include "etune_internal.hpp"
#include "kernels.hpp"
#include "mt64.cuh"

#include "breed_core.cuh"

namespace etune_b200 {

namespace {

using namespace breedcore;

constexpr int kBreedThreads = 1024;
constexpr int kRing = 4096;           // words of the MT stream kept in shared memory
constexpr int kCells = 2048;          // speculative (offspring, offset) evaluations per round
constexpr int kMaxLevels = 96;        // offspring resolved per round at most (3 per lane of warp 0)
constexpr int kJump = 7;              // pointer-doubling tables: 2^7 >= kMaxLevels

// Sequential reader of the word stream held in the ring; positions at or beyond
// `hi` are not generated yet, which makes the evaluation "unknown".
struct Cursor {
    const uint64_t* ring;
    uint64_t p, hi;
    bool ok;
    __device__ __forceinline__ uint64_t next() {
        if (p >= hi) {
            ok = false;
            return 0;
        }
        return ring[(p++) & (kRing - 1)];
    }
};

__device__ Child breed_one(const BreedConst& K, const PlanHdr& H, int64_t i, const uint64_t* ring, uint64_t start,
                           uint64_t hi) {
    Cursor c{ring, start, hi, true};
    return breed_body(K, H, i, c, start);
}

struct BreedState {
    int64_t resolved;       // offspring written
    uint64_t words;         // RNG words consumed by them
    int32_t status;         // 0 ok, else etune_status
    int32_t pad;
};

__global__ void __launch_bounds__(kBreedThreads, 1)
    breed_kernel(const uint8_t* __restrict__ gplan, uint32_t plan_bytes, int use_smem,
                 const uint64_t* __restrict__ par, const uint64_t* __restrict__ pid, int64_t np, int64_t n,
                 double mut, double mutcro, double total, uint64_t seed, uint64_t* __restrict__ out,
                 int32_t* __restrict__ partner, unsigned long long* err, BreedState* st,
                 const int32_t* __restrict__ skip) {
    if (skip && *skip) return;  // the block-parallel path (breed_par.cu) produced the generation
    // dynamic shared memory: [ring | cell genomes | cell partners | cell words | mt | plan]
    extern __shared__ int4 smem[];
    uint64_t* ring = reinterpret_cast<uint64_t*>(smem);
    uint64_t* cg = ring + kRing;
    int32_t* cp = reinterpret_cast<int32_t*>(cg + kCells);
    uint16_t* cw = reinterpret_cast<uint16_t*>(cp + kCells);
    int16_t* jt = reinterpret_cast<int16_t*>(cw + kCells);     // [kJump][kCells] successor^(2^r)
    uint8_t* clev = reinterpret_cast<uint8_t*>(jt + kJump * kCells);  // level of each cell
    uint64_t* mt = reinterpret_cast<uint64_t*>(clev + kCells);
    __shared__ int32_t lstart[kMaxLevels + 1], llo[kMaxLevels], lhi[kMaxLevels];
    __shared__ int16_t path[kMaxLevels];
    __shared__ int s_levels, s_resolved, s_status, s_other;
    __shared__ uint64_t s_step;
    __shared__ double s_mean, s_var;
    const int tid = threadIdx.x;

    const uint8_t* P = gplan;
    if (use_smem) {
        int4* dst = reinterpret_cast<int4*>(mt + 312);
        const int4* src = reinterpret_cast<const int4*>(gplan);
        for (uint32_t i = tid; i < (plan_bytes >> 4); i += blockDim.x) dst[i] = __ldg(src + i);
        P = reinterpret_cast<const uint8_t*>(dst);
    }
    // has_other: some parent id differs from another (genetic.cpp:172-174)
    if (tid == 0) s_other = 0;
    __syncthreads();
    {
        const uint64_t id0 = __ldg(pid);
        int diff = 0;
        for (int64_t j = tid; j < np; j += blockDim.x) diff |= __ldg(pid + j) != id0;
        if (__syncthreads_or(diff) && tid == 0) s_other = 1;
    }
    if (tid == 0) mt64::seed_state(mt, seed);  // std::mt19937_64(seed)
    __syncthreads();
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    BreedConst K{P, par, pid, np, mut, mutcro, total, s_other};

    uint64_t hi = 0;          // words generated so far (ring holds [hi - kRing, hi) at most)
    uint64_t o0 = 0;          // first word of offspring i0
    int64_t i0 = 0;
    double s1 = 0.0, s2 = 0.0;  // running word-count statistics (warp 0; window placement only)
    if (tid == 0) {
        s_mean = 2.8;
        s_var = 0.6;
    }
    int64_t cnt = 0;
    int status = 0;
    while (i0 < n) {
        // ---- extend the stream: cooperative twists while the ring has room
        while (hi + 312 <= o0 + kRing) {
            mt64::twist_block(mt);
            if (tid < 312) ring[(hi + uint64_t(tid)) & (kRing - 1)] = mt64::temper(mt[tid]);
            hi += 312;
        }
        // ---- level windows (warp 0: widths, then a warp scan of the cell counts)
        if (tid < 32) {
            const float sd = sqrtf(float(s_var > 0.05 ? s_var : 0.05));  // window placement only
            const float mean = float(s_mean);
            int carry = 0, levels = 0;
            for (int q = 0; q < kMaxLevels / 32; ++q) {
                const int j = q * 32 + tid;
                int lo = 0, hi_j = 0;
                if (j > 0) {
                    const float c = mean * float(j);
                    const int h = 2 + int(ceilf(4.0f * sd * sqrtf(float(j))));
                    lo = max(j, int(floorf(c)) - h);
                    hi_j = int(ceilf(c)) + h;
                }
                const int w = hi_j - lo + 1;
                int x = w;  // inclusive scan of widths
                for (int sft = 1; sft < 32; sft <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, sft);
                    if (tid >= sft) x += y;
                }
                const int start = carry + x - w;
                const bool fits = start + w <= kCells && i0 + j < n;
                const unsigned ok = __ballot_sync(0xffffffffu, fits);
                const int take = (~ok) ? __ffs(~ok) - 1 : 32;  // leading levels that fit
                if (tid < take) {
                    lstart[j] = start;
                    llo[j] = lo;
                    lhi[j] = hi_j;
                }
                levels += take;
                carry += __shfl_sync(0xffffffffu, x, 31);
                if (take < 32) {
                    if (tid == take) lstart[j] = start;  // end sentinel
                    break;
                }
                if (q == kMaxLevels / 32 - 1 && tid == 31) lstart[j + 1] = start + w;
            }
            if (tid == 0) s_levels = levels;
        }
        __syncthreads();
        const int J = s_levels, ncell = lstart[J];
        // ---- speculative evaluation of every (level, offset) cell
        for (int cell = tid; cell < ncell; cell += blockDim.x) {
            int lo = 0, hi2 = J;  // level of this cell: last j with lstart[j] <= cell
            while (hi2 - lo > 1) {
                const int mid = (lo + hi2) >> 1;
                if (lstart[mid] <= cell) lo = mid;
                else hi2 = mid;
            }
            const int j = lo;
            const uint64_t off = o0 + uint64_t(llo[j] + (cell - lstart[j]));
            const Child ch = breed_one(K, H, i0 + j, ring, off, hi);
            cg[cell] = ch.g;
            cp[cell] = ch.partner;
            cw[cell] = ch.words;
            clev[cell] = uint8_t(j);
        }
        __syncthreads();
        // ---- the true chain through the cells by pointer doubling:
        // succ(level j, offset x) = (level j+1, x + words) when that offset lies in the window
        for (int cell = tid; cell < ncell; cell += blockDim.x) {
            const int j = clev[cell];
            const uint16_t w = cw[cell];
            int16_t nx = -1;
            if (w != kUnknown && w != kIllegal && j + 1 < J) {
                const int x = llo[j] + (cell - lstart[j]) + int(w);
                if (x >= llo[j + 1] && x <= lhi[j + 1]) nx = int16_t(lstart[j + 1] + (x - llo[j + 1]));
            }
            jt[cell] = nx;
        }
        __syncthreads();
        for (int r = 1; r < kJump; ++r) {
            const int16_t* prev = jt + (r - 1) * kCells;
            int16_t* cur = jt + r * kCells;
            for (int cell = tid; cell < ncell; cell += blockDim.x) {
                const int16_t m = prev[cell];
                cur[cell] = m < 0 ? int16_t(-1) : prev[m];
            }
            __syncthreads();
        }
        if (tid < J) {  // cell of level j on the chain from (level 0, offset 0) = cell 0
            int c = 0;
            for (int r = 0; r < kJump && c >= 0; ++r)
                if ((tid >> r) & 1) c = jt[r * kCells + c];
            path[tid] = int16_t(c);
        }
        if (tid == 0) s_resolved = J;
        __syncthreads();
        if (tid < J) {  // resolved = leading levels whose cell exists and evaluated completely
            const int c = path[tid];
            if (c < 0 || cw[c] == kUnknown || cw[c] == kIllegal) atomicMin(&s_resolved, tid);
        }
        __syncthreads();
        const int R = s_resolved;
        if (tid == 0) {
            int stt = 0;
            if (R < J && path[R] >= 0 && cw[path[R]] == kIllegal) {
                stt = ETUNE_ERR_ILLEGAL_SCHEDULE;
                atomicMin(err, (static_cast<unsigned long long>(i0 + R) << 8) | unsigned(stt));
            } else if (R == 0 && hi + 312 > o0 + kRing) {
                // offspring i0 alone needs more than the ring's words (a crossover whose
                // partner search runs for thousands of draws): beyond this build's window
                stt = ETUNE_ERR_UNSUPPORTED;
                atomicMin(err, (static_cast<unsigned long long>(i0) << 8) | unsigned(stt));
            }
            s_status = stt;
            const int last = R > 0 ? path[R - 1] : -1;
            s_step = R > 0 ? uint64_t(llo[R - 1] + (last - lstart[R - 1]) + int(cw[last])) : 0ull;
        }
        if (tid < R) {
            const int cell = path[tid];
            out[i0 + tid] = cg[cell];
            if (partner) partner[i0 + tid] = cp[cell];
        }
        // running statistics of words per offspring (warp 0; window placement only)
        if (tid < 32 && R > 0) {
            double a1 = 0.0, a2 = 0.0;
            for (int j = tid; j < R; j += 32) {
                const double w = double(cw[path[j]]);
                a1 += w;
                a2 += w * w;
            }
            for (int sft = 16; sft > 0; sft >>= 1) {
                a1 += __shfl_xor_sync(0xffffffffu, a1, sft);
                a2 += __shfl_xor_sync(0xffffffffu, a2, sft);
            }
            s1 += a1;
            s2 += a2;
            cnt += R;
            if (tid == 0) {
                s_mean = s1 / double(cnt);
                s_var = s2 / double(cnt) - s_mean * s_mean;
            }
        }
        __syncthreads();
        o0 += s_step;
        i0 += R;
        status = s_status;
        if (status) break;
    }
    if (tid == 0) {
        st->resolved = i0;
        st->words = o0;
        st->status = status;
    }
}

// Counter mode: one thread per offspring (grid-stride), no chain between them.
__global__ void __launch_bounds__(256) breed_counter_kernel(const uint8_t* __restrict__ gplan, uint32_t plan_bytes,
                                                           int use_smem, const uint64_t* __restrict__ par,
                                                           const uint64_t* __restrict__ pid, int64_t np, int64_t n,
                                                           double mut, double mutcro, double total, uint64_t seed,
                                                           uint64_t* __restrict__ out, int32_t* __restrict__ partner,
                                                           unsigned long long* err) {
    extern __shared__ int4 bsm[];
    __shared__ int s_other;
    const uint8_t* P = gplan;
    if (use_smem) {
        for (uint32_t i = threadIdx.x; i < (plan_bytes >> 4); i += blockDim.x)
            bsm[i] = __ldg(reinterpret_cast<const int4*>(gplan) + i);
        P = reinterpret_cast<const uint8_t*>(bsm);
    }
    if (threadIdx.x == 0) s_other = 0;
    __syncthreads();
    {  // has_other (genetic.cpp:172-174): every CTA derives it from the parent ids
        const uint64_t id0 = __ldg(pid);
        int diff = 0;
        for (int64_t j = threadIdx.x; j < np; j += blockDim.x) diff |= __ldg(pid + j) != id0;
        if (__syncthreads_or(diff) && threadIdx.x == 0) s_other = 1;
    }
    __syncthreads();
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    const BreedConst K{P, par, pid, np, mut, mutcro, total, s_other};
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        CounterCursor c{splitmix64(seed ^ splitmix64(uint64_t(i))), 0, true};
        const Child ch = breed_body(K, H, i, c, 0);
        if (ch.words == kIllegal) {
            atomicMin(err, (static_cast<unsigned long long>(i) << 8) | unsigned(ETUNE_ERR_ILLEGAL_SCHEDULE));
            out[i] = 0;
            if (partner) partner[i] = -1;
            continue;
        }
        out[i] = ch.g;
        if (partner) partner[i] = ch.partner;
    }
}

}  // namespace

cudaError_t launch_breed_counter(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint64_t* d_par,
                                 const uint64_t* d_pid, int64_t np, int64_t n, double mut, double cro, double cpy,
                                 uint64_t seed, uint64_t* d_out, int32_t* d_partner) {
    if (n <= 0) return cudaSuccess;
    const double mutcro = mut + cro;
    const double total = mutcro + cpy;
    const int use_smem = plan_bytes <= 96 * 1024 ? 1 : 0;
    const size_t dyn = use_smem ? plan_bytes : 0;
    if (dyn > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(breed_counter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, breed_counter_kernel, 256, dyn);
    if (e != cudaSuccess) return e;
    const int64_t want = (n + 255) / 256;
    const int64_t cap = int64_t(c.sm_count) * (per_sm > 0 ? per_sm : 1);
    breed_counter_kernel<<<int(want < cap ? want : cap), 256, dyn, c.stream>>>(
        d_plan, plan_bytes, use_smem, d_par, d_pid, np, n, mut, mutcro, total, seed, d_out, d_partner, c.d_err);
    note_launches(1);
    return cudaGetLastError();
}

size_t breed_state_bytes() { return sizeof(BreedState); }

cudaError_t launch_breed(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint64_t* d_par,
                         const uint64_t* d_pid, int64_t np, int64_t n, double mut, double cro, double cpy,
                         uint64_t seed, uint64_t* d_out, int32_t* d_partner, void* d_state, const int32_t* d_skip) {
    if (n <= 0) return cudaSuccess;
    const double mutcro = mut + cro;     // genetic.cpp:169, evaluated like the reference
    const double total = mutcro + cpy;   // genetic.cpp:150: mutation + crossover + copy
    // ~64 KB of working arrays; the plan blob joins them in shared memory when it fits
    constexpr size_t kFixed = size_t(kRing) * 8 + size_t(kCells) * (8 + 4 + 2 + 2 * kJump + 1) + 312 * 8;
    static_assert(kFixed % 16 == 0, "plan section must stay 16-byte aligned");
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int use_smem = (kFixed + plan_bytes + 2048 <= size_t(optin)) ? 1 : 0;
    const size_t dyn = kFixed + (use_smem ? plan_bytes : 0);
    cudaError_t e = cudaFuncSetAttribute(breed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
    if (e != cudaSuccess) return e;
    breed_kernel<<<1, kBreedThreads, dyn, c.stream>>>(d_plan, plan_bytes, use_smem, d_par, d_pid, np, n, mut, mutcro,
                                                      total, seed, d_out, d_partner, c.d_err,
                                                      static_cast<BreedState*>(d_state), d_skip);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace etune_b200
