// sample_random (space.cpp:170-251) on the device, bit-exact with the reference's
// std::mt19937_64(seed) stream.
//
//   large space  (more legal schedules than max(2n, 4096)): attempt j reads words
//                [o_j, o_j + 6) — one Lemire draw per knob — so attempts are evaluated
//                in parallel; illegal ones (block > cap) are skipped and duplicates are
//                removed by first occurrence (stable radix sort of (id, attempt)),
//                then the first n survivors in attempt order are the sample.
//   small space  the legal schedules in ScheduleEnumerator order (parallel filter of
//                the odometer product + ordered compaction), then the partial
//                Fisher-Yates of space.cpp:190-194 resolved in parallel: output i is
//                the content of position j_i before step i, found by following
//                "last earlier step that targeted this position" links.
// Word offsets are the nominal ones (6 per attempt / 1 per swap) unless a draw hits
// libstdc++'s rare Lemire rejection (p ~ r / 2^64, detected from the total of the
// per-item word counts): then one sequential walk recomputes the exact offsets and the
// items are evaluated again, so results stay exact in that case too.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "etune_internal.hpp"
#include "kernels.hpp"
#include "mt64.cuh"
#include "scan.cuh"

namespace etune_b200 {

namespace {

template <typename T>
__device__ __forceinline__ const T* at(const uint8_t* base, uint32_t off) {
    return reinterpret_cast<const T*>(base + off);
}

// the raw word stream of std::mt19937_64(seed): one CTA, 312 words per twist
__global__ void __launch_bounds__(320) mt_words_kernel(uint64_t seed, int64_t nwords, uint64_t* __restrict__ out) {
    __shared__ uint64_t mt[mt64::kN];
    if (threadIdx.x == 0) mt64::seed_state(mt, seed);
    __syncthreads();
    for (int64_t base = 0; base < nwords; base += mt64::kN) {
        mt64::twist_block(mt);
        const int64_t i = base + threadIdx.x;
        if (threadIdx.x < mt64::kN && i < nwords) out[i] = mt64::temper(mt[threadIdx.x]);
    }
}

// Full Lemire draw reading words from `w` at *pos (rejections consume more words).
__device__ __forceinline__ uint64_t lemire_at(const uint64_t* w, int64_t nwords, int64_t* pos, uint64_t r,
                                             bool* overflow) {
    auto next = [&]() -> uint64_t {
        if (*pos >= nwords) {
            *overflow = true;
            return 0;
        }
        return w[(*pos)++];
    };
    uint64_t x = next();
    uint64_t lo = x * r;
    if (lo < r) {
        const uint64_t thr = (0ull - r) % r;
        while (lo < thr && !*overflow) {
            x = next();
            lo = x * r;
        }
    }
    return __umul64hi(x, r);
}

__device__ __forceinline__ int ctz64(int64_t v) { return __ffsll(static_cast<long long>(v)) - 1; }

// One attempt of the large-space loop (space.cpp:216-247) at word offset `off`.
__global__ void attempt_kernel(const uint8_t* __restrict__ P, const uint64_t* __restrict__ w, int64_t nwords,
                               const int64_t* __restrict__ offs, int64_t A, uint64_t* __restrict__ genome,
                               uint64_t* __restrict__ key, uint32_t* __restrict__ val, uint8_t* __restrict__ ok,
                               int32_t* __restrict__ used, int* flags) {
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    const TilingRec* T0 = at<TilingRec>(P, H.off_til[0]);
    const TilingRec* T1 = at<TilingRec>(P, H.off_til[1]);
    const TilingRec* T2 = at<TilingRec>(P, H.off_til[2]);
    const int64_t* divk = at<int64_t>(P, H.off_divk);
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < A; j += int64_t(gridDim.x) * blockDim.x) {
        int64_t pos = offs ? offs[j] : 6 * j;
        const int64_t start = pos;
        bool over = false;
        const uint32_t t0 = uint32_t(lemire_at(w, nwords, &pos, uint64_t(H.nt[0]), &over));
        const uint32_t t1 = uint32_t(lemire_at(w, nwords, &pos, uint64_t(H.nt[1]), &over));
        const uint32_t t2 = uint32_t(lemire_at(w, nwords, &pos, uint64_t(H.nt[2]), &over));
        const uint32_t k = uint32_t(lemire_at(w, nwords, &pos, uint64_t(H.ndk), &over));
        // legal unrolls: u <= max_unroll while k_tile % u == 0 (space.cpp:228-233)
        const int cu = min(H.max_unroll_log2, ctz64(divk[k]));
        const uint32_t u = uint32_t(lemire_at(w, nwords, &pos, uint64_t(cu + 1), &over));
        const TilingRec r0 = T0[t0], r1 = T1[t1], r2 = T2[t2];
        const int cv = min(H.max_vec_log2, ctz64(int64_t(r2.pt)));
        const uint32_t v = uint32_t(lemire_at(w, nwords, &pos, uint64_t(cv + 1), &over));
        if (over) atomicOr(flags, 1);
        used[j] = int32_t(pos - start);
        const uint64_t block = uint64_t(r0.threads) * r1.threads * uint64_t(r2.threads);
        const bool legal = int64_t(block) <= int64_t(H.block_cap);
        ok[j] = legal ? 1 : 0;
        const uint64_t g = genome_pack(t0, t1, t2, k, u, v);
        genome[j] = g;
        val[j] = uint32_t(j);
    }
}

// Rare path (some draw hit a Lemire rejection): exact offsets by one sequential walk.
__global__ void attempt_offsets_serial_kernel(const uint8_t* __restrict__ P, const uint64_t* __restrict__ w,
                                              int64_t nwords, int64_t A, int64_t* __restrict__ offs, int* flags) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
    const TilingRec* T2 = at<TilingRec>(P, H.off_til[2]);
    const int64_t* divk = at<int64_t>(P, H.off_divk);
    int64_t pos = 0;
    bool over = false;
    for (int64_t j = 0; j < A && !over; ++j) {
        offs[j] = pos;
        lemire_at(w, nwords, &pos, uint64_t(H.nt[0]), &over);
        lemire_at(w, nwords, &pos, uint64_t(H.nt[1]), &over);
        const uint32_t t2 = uint32_t(lemire_at(w, nwords, &pos, uint64_t(H.nt[2]), &over));
        const uint32_t k = uint32_t(lemire_at(w, nwords, &pos, uint64_t(H.ndk), &over));
        lemire_at(w, nwords, &pos, uint64_t(min(H.max_unroll_log2, ctz64(divk[k])) + 1), &over);
        lemire_at(w, nwords, &pos, uint64_t(min(H.max_vec_log2, ctz64(int64_t(T2[t2].pt))) + 1), &over);
    }
    if (over) atomicOr(flags, 1);
}

__global__ void fy_offsets_serial_kernel(const uint64_t* __restrict__ w, int64_t nwords, int64_t n, int64_t size,
                                         int64_t* __restrict__ offs, int* flags) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t pos = 0;
    bool over = false;
    for (int64_t i = 0; i < n && !over; ++i) {
        offs[i] = pos;
        lemire_at(w, nwords, &pos, uint64_t(size - i), &over);
    }
    if (over) atomicOr(flags, 1);
}

struct CandIdFn {  // candidate_id of a genome (space.cpp:22-45), operator prefix hoisted
    const uint8_t* P;
    __device__ uint64_t operator()(uint64_t g) const {
        const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
        const Genome x = genome_unpack(g);
        const TilingRec r[3] = {at<TilingRec>(P, H.off_til[0])[x.t0], at<TilingRec>(P, H.off_til[1])[x.t1],
                                at<TilingRec>(P, H.off_til[2])[x.t2]};
        uint64_t h = H.fnv_prefix;
        auto absorb = [&](uint64_t v) {
            for (int b = 0; b < 8; ++b) {
                h ^= (v >> (8 * b)) & 0xffu;
                h *= 1099511628211ull;
            }
        };
        for (int d = 0; d < 3; ++d) {
            absorb(r[d].blocks);
            absorb(r[d].threads);
            absorb(r[d].pt);
        }
        absorb(uint64_t(at<int64_t>(P, H.off_divk)[x.k]));
        absorb(uint64_t(1) << x.u);
        absorb(uint64_t(1) << x.v);
        return h;
    }
};

__global__ void ids_of_kernel(const uint8_t* __restrict__ P, const uint64_t* __restrict__ genome, int64_t n,
                              uint64_t* __restrict__ key) {
    const CandIdFn id{P};
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        key[j] = id(genome[j]);
}

// after the stable sort by id: keep = first LEGAL attempt of each id group
__global__ void first_of_group_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val,
                                      const uint8_t* __restrict__ ok, int64_t A, uint8_t* __restrict__ keep) {
    for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < A; p += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t j = val[p];
        bool first = ok[j] != 0;
        for (int64_t q = p - 1; first && q >= 0 && key[q] == key[p]; --q)
            if (ok[val[q]]) first = false;
        keep[j] = first ? 1 : 0;
    }
}

// ---------------------------------------------------------------- small space
struct EnumDims {
    int64_t n[6];  // tilings0, tilings1, tilings2, k tiles, unrolls, vectors
};

__device__ __forceinline__ uint64_t enum_genome(const EnumDims& d, int64_t q) {
    uint32_t ix[6];
    for (int p = 5; p >= 0; --p) {  // odometer, last position fastest (space.cpp:134-141)
        ix[p] = uint32_t(q % d.n[p]);
        q /= d.n[p];
    }
    return genome_pack(ix[0], ix[1], ix[2], ix[3], ix[4], ix[5]);
}

struct EnumLegal {  // ScheduleEnumerator::current_is_legal (space.cpp:120-130)
    const uint8_t* P;
    EnumDims d;
    __device__ int64_t operator()(int64_t q) const {
        const PlanHdr& H = *reinterpret_cast<const PlanHdr*>(P);
        const Genome x = genome_unpack(enum_genome(d, q));
        const uint64_t block = uint64_t(at<TilingRec>(P, H.off_til[0])[x.t0].threads) *
                               at<TilingRec>(P, H.off_til[1])[x.t1].threads *
                               uint64_t(at<TilingRec>(P, H.off_til[2])[x.t2].threads);
        if (int64_t(block) > int64_t(H.block_cap)) return 0;
        if (at<int64_t>(P, H.off_divk)[x.k] % (int64_t(1) << x.u) != 0) return 0;
        if (int64_t(at<TilingRec>(P, H.off_til[2])[x.t2].pt) % (int64_t(1) << x.v) != 0) return 0;
        return 1;
    }
};

struct EnumWrite {
    EnumDims d;
    EnumLegal legal;
    uint64_t* all;
    __device__ void operator()(int64_t q, int64_t rank) const {
        if (legal(q)) all[rank] = enum_genome(d, q);
    }
};

// j_i = i + uniform(i, size-1) at offset o_i; pairs (j_i << 32 | i) for the link search
__global__ void fy_draw_kernel(const uint64_t* __restrict__ w, int64_t nwords, const int64_t* __restrict__ offs,
                               int64_t n, int64_t size, uint32_t* __restrict__ jv, uint64_t* __restrict__ key,
                               uint32_t* __restrict__ val, int32_t* __restrict__ used, int* flags) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        int64_t pos = offs ? offs[i] : i;
        const int64_t start = pos;
        bool over = false;
        const uint64_t j = uint64_t(i) + lemire_at(w, nwords, &pos, uint64_t(size - i), &over);
        if (over) atomicOr(flags, 1);
        used[i] = int32_t(pos - start);
        jv[i] = uint32_t(j);
        key[i] = (j << 32) | uint64_t(i);
        val[i] = uint32_t(i);
    }
}

// last step s < t that swapped into position `pos`, or -1 (sorted (target << 32 | step) keys)
__device__ __forceinline__ int64_t last_into(const uint64_t* key, int64_t n, uint64_t pos, uint64_t t) {
    const uint64_t probe = (pos << 32) | t;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] < probe) lo = mid + 1;
        else hi = mid;
    }
    if (lo == 0) return -1;
    const uint64_t k = key[lo - 1];
    return (k >> 32) == pos ? int64_t(k & 0xffffffffull) : -1;
}

__global__ void fy_resolve_kernel(const uint64_t* __restrict__ all, const uint32_t* __restrict__ jv,
                                  const uint64_t* __restrict__ key, int64_t n, uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint64_t pos = jv[i], t = uint64_t(i);
        for (;;) {  // content of `pos` just before step t
            const int64_t s = last_into(key, n, pos, t);
            if (s < 0) break;
            pos = uint64_t(s);  // step s moved position s's content (before step s) into pos
            t = uint64_t(s);
        }
        out[i] = all[pos];
    }
}

int grid_of(const LaunchCtx& c, int64_t n) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8)));
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct UsedFn {
    const int32_t* used;
    __device__ int64_t operator()(int64_t i) const { return used[i]; }
};
struct OffsWrite {
    int64_t* offs;
    __device__ void operator()(int64_t i, int64_t ex) const { offs[i] = ex; }
};
struct KeepFn {
    const uint8_t* keep;
    __device__ int64_t operator()(int64_t i) const { return keep[i]; }
};
struct KeepWrite {
    const uint8_t* keep;
    const uint64_t* genome;
    int64_t n;
    uint64_t* out;
    __device__ void operator()(int64_t j, int64_t rank) const {
        if (keep[j] && rank < n) out[rank] = genome[j];
    }
};

}  // namespace

size_t sample_scratch_bytes(int64_t n, int64_t space_or_product, bool small) {
    if (small) {
        const int64_t q = space_or_product;  // odometer product
        return 5 * al256(8 * size_t(n) + 64 * 8) + al256(8 * size_t(q)) + al256(8 * size_t(n)) * 4 +
               sort_pairs_scratch_bytes(n) + al256(8 * ((size_t(q) + 1023) / 1024 + 2)) + 4096;
    }
    const int64_t A = n;  // caller passes the attempt count as n
    return al256(8 * (6 * size_t(A) + 4096)) + 2 * al256(8 * size_t(A)) + al256(4 * size_t(A)) +
           al256(size_t(A)) * 2 + al256(4 * size_t(A)) + al256(8 * size_t(A)) + sort_pairs_scratch_bytes(A) +
           al256(8 * ((size_t(A) + 1023) / 1024 + 2)) + 4096;
}

// Large-space branch.  Returns the number of distinct legal candidates found among the
// A attempts in *d_found (device); the first min(n, found) are written to d_out.
cudaError_t launch_sample_large(const LaunchCtx& c, const uint8_t* d_plan, uint64_t seed, int64_t n, int64_t A,
                                uint64_t* d_out, int64_t* d_found, int* d_flags, void* scratch) {
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t b) {
        char* r = p;
        p += al256(b);
        return r;
    };
    const int64_t nwords = 6 * A + 4096;
    uint64_t* w = reinterpret_cast<uint64_t*>(take(8 * size_t(nwords)));
    uint64_t* genome = reinterpret_cast<uint64_t*>(take(8 * size_t(A)));
    uint64_t* key = reinterpret_cast<uint64_t*>(take(8 * size_t(A)));
    uint32_t* val = reinterpret_cast<uint32_t*>(take(4 * size_t(A)));
    uint8_t* ok = reinterpret_cast<uint8_t*>(take(size_t(A)));
    uint8_t* keep = reinterpret_cast<uint8_t*>(take(size_t(A)));
    int32_t* used = reinterpret_cast<int32_t*>(take(4 * size_t(A)));
    int64_t* offs = reinterpret_cast<int64_t*>(take(8 * size_t(A)));
    void* sort_scr = take(sort_pairs_scratch_bytes(A));
    int64_t* sums = reinterpret_cast<int64_t*>(take(8 * ((size_t(A) + 1023) / 1024 + 2)));
    int64_t* total = reinterpret_cast<int64_t*>(take(64));

    mt_words_kernel<<<1, 320, 0, c.stream>>>(seed, nwords, w);
    note_launches(1);
    const int g = grid_of(c, A);
    cudaMemsetAsync(d_flags, 0, sizeof(int), c.stream);
    attempt_kernel<<<g, 256, 0, c.stream>>>(d_plan, w, nwords, nullptr, A, genome, key, val, ok, used, d_flags);
    note_launches(1);
    // a draw that consumed extra words (Lemire rejection) shifts every later attempt:
    // detect from the total, then take exact offsets from one sequential walk
    {
        cudaError_t e = scan_apply(c.stream, A, UsedFn{used}, OffsWrite{offs}, sums, total);
        if (e != cudaSuccess) return e;
        int64_t h_total = 0;
        cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        if (h_total != 6 * A) {
            attempt_offsets_serial_kernel<<<1, 32, 0, c.stream>>>(d_plan, w, nwords, A, offs, d_flags);
            attempt_kernel<<<g, 256, 0, c.stream>>>(d_plan, w, nwords, offs, A, genome, key, val, ok, used, d_flags);
            note_launches(2);
        }
    }
    ids_of_kernel<<<g, 256, 0, c.stream>>>(d_plan, genome, A, key);
    note_launches(1);
    cudaError_t e = launch_sort_pairs(c, key, val, A, 64, sort_scr);
    if (e != cudaSuccess) return e;
    first_of_group_kernel<<<g, 256, 0, c.stream>>>(key, val, ok, A, keep);
    note_launches(1);
    return scan_apply(c.stream, A, KeepFn{keep}, KeepWrite{keep, genome, n, d_out}, sums, d_found);
}

// Small-space branch: enumerate + parallel partial Fisher-Yates.  *d_found = space size.
cudaError_t launch_sample_small(const LaunchCtx& c, const uint8_t* d_plan, const int64_t dims[6], uint64_t seed,
                                int64_t n, uint64_t* d_out, int64_t* d_found, int* d_flags, void* scratch) {
    EnumDims d;
    int64_t q = 1;
    for (int i = 0; i < 6; ++i) {
        d.n[i] = dims[i];
        q *= dims[i];
    }
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t b) {
        char* r = p;
        p += al256(b);
        return r;
    };
    const int64_t nwords = n + 512;
    uint64_t* w = reinterpret_cast<uint64_t*>(take(8 * size_t(nwords)));
    uint64_t* all = reinterpret_cast<uint64_t*>(take(8 * size_t(q)));
    uint32_t* jv = reinterpret_cast<uint32_t*>(take(4 * size_t(n)));
    uint64_t* key = reinterpret_cast<uint64_t*>(take(8 * size_t(n)));
    uint32_t* val = reinterpret_cast<uint32_t*>(take(4 * size_t(n)));
    int32_t* used = reinterpret_cast<int32_t*>(take(4 * size_t(n)));
    int64_t* offs = reinterpret_cast<int64_t*>(take(8 * size_t(n)));
    void* sort_scr = take(sort_pairs_scratch_bytes(n));
    int64_t* sums = reinterpret_cast<int64_t*>(take(8 * ((size_t(q) + 1023) / 1024 + 2)));
    int64_t* total = reinterpret_cast<int64_t*>(take(64));

    const EnumLegal legal{d_plan, d};
    cudaError_t e = scan_apply(c.stream, q, legal, EnumWrite{d, legal, all}, sums, d_found);
    if (e != cudaSuccess) return e;
    int64_t size = 0;
    cudaMemcpyAsync(&size, d_found, 8, cudaMemcpyDeviceToHost, c.stream);
    mt_words_kernel<<<1, 320, 0, c.stream>>>(seed, nwords, w);
    note_launches(1);
    cudaStreamSynchronize(c.stream);
    if (size < n) return cudaSuccess;  // caller reports SpaceExhausted
    const int g = grid_of(c, n);
    cudaMemsetAsync(d_flags, 0, sizeof(int), c.stream);
    fy_draw_kernel<<<g, 256, 0, c.stream>>>(w, nwords, nullptr, n, size, jv, key, val, used, d_flags);
    note_launches(1);
    {
        e = scan_apply(c.stream, n, UsedFn{used}, OffsWrite{offs}, sums, total);
        if (e != cudaSuccess) return e;
        int64_t h_total = 0;
        cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        if (h_total != n) {
            fy_offsets_serial_kernel<<<1, 32, 0, c.stream>>>(w, nwords, n, size, offs, d_flags);
            fy_draw_kernel<<<g, 256, 0, c.stream>>>(w, nwords, offs, n, size, jv, key, val, used, d_flags);
            note_launches(2);
        }
    }
    e = launch_sort_pairs(c, key, val, n, 64, sort_scr);
    if (e != cudaSuccess) return e;
    fy_resolve_kernel<<<g, 256, 0, c.stream>>>(all, jv, key, n, d_out);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace etune_b200
