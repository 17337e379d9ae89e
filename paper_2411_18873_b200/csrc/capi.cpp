// C ABI (include/etune_cuda.h): handles, argument checking, status mapping and
// launch orchestration.  No compute happens here: every data-parallel step is a
// kernel in kernels.cu / sort.cu.  There is deliberately no CPU fallback — without
// an sm_100 device every entry point returns ETUNE_ERR_NO_DEVICE.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>
#include <thread>

#include <sched.h>
#include <immintrin.h>

#include "forest.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "handles.hpp"

using namespace etune_b200;

namespace etune_b200 {
thread_local std::string g_error;
void ctx_free_now(etune_cu_ctx* c) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaFree(c->d_err);
    cudaFree(c->scratch);
    cudaFree(c->io);
    cudaFree(c->breed);
    cudaFree(c->breedpar);
    cudaFree(c->shard);
    cudaFree(c->sel);
    cudaFree(c->rowsel);
    cudaFree(c->e2e);
    if (c->hpin) cudaFreeHost(c->hpin);
    if (c->hout) cudaFreeHost(c->hout);
    c->pool.reset();
    for (auto& e : c->prof_ev)
        for (cudaEvent_t x : e) cudaEventDestroy(x);
    if (c->h2d) {
        cudaStreamDestroy(c->h2d);
        cudaStreamDestroy(c->d2h);
        for (int b = 0; b < 2; ++b) {
            cudaEventDestroy(c->ev_in[b]);
            cudaEventDestroy(c->ev_done[b]);
            cudaEventDestroy(c->ev_out[b]);
        }
    }
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}


// Handles hold a reference on their ctx: destroying the ctx before its plans, forests
// or searches (any order a garbage collector picks) defers the release until the last
// of them is gone.
void ctx_retain(etune_cu_ctx* c) { c->refs.fetch_add(1); }
void ctx_release(etune_cu_ctx* c) {
    if (c->refs.fetch_sub(1) == 1 && c->closing.load()) ctx_free_now(c);
}
void set_error(const std::string& msg) { g_error = msg; }

// ------------------------------------------------------------ collectives
// NCCL when a communicator is attached (one rank per GPU over NVLink / NVSwitch), else the
// caller's transport callbacks (etune_cu_ctx_attach_transport: e.g. a test running two ranks on
// one GPU over gloo), else a single rank (all-gather = copy, broadcast = no-op).
int ctx_world(const etune_cu_ctx* c) { return c->comm ? c->nranks : c->has_transport ? c->transport.nranks : 1; }
int ctx_rank(const etune_cu_ctx* c) { return c->comm ? c->rank : c->has_transport ? c->transport.rank : 0; }

etune_status coll_allgather(etune_cu_ctx* c, const void* d_send, void* d_recv, size_t bytes) {
    if (c->comm) {
        const ncclResult_t r = ncclAllGather(d_send, d_recv, bytes, ncclUint8, c->comm, c->stream);
        if (r != ncclSuccess) {
            set_error(std::string("ncclAllGather: ") + ncclGetErrorString(r));
            return ETUNE_ERR_CUDA;
        }
        return ETUNE_OK;
    }
    if (c->has_transport) {
        if (c->transport.allgather(c->transport.user, d_send, d_recv, int64_t(bytes), c->stream) != 0) {
            set_error("transport all-gather failed");
            return ETUNE_ERR_BACKEND_UNAVAILABLE;
        }
        return ETUNE_OK;
    }
    if (d_send != d_recv && bytes) {
        const cudaError_t e = cudaMemcpyAsync(d_recv, d_send, bytes, cudaMemcpyDeviceToDevice, c->stream);
        if (e != cudaSuccess) {
            set_error(std::string("all-gather copy: ") + cudaGetErrorString(e));
            return ETUNE_ERR_CUDA;
        }
    }
    return ETUNE_OK;
}

etune_status coll_broadcast(etune_cu_ctx* c, void* d_buf, size_t bytes, int root) {
    if (ctx_world(c) == 1 || bytes == 0) return ETUNE_OK;
    if (c->comm) {
        const ncclResult_t r = ncclBroadcast(d_buf, d_buf, bytes, ncclUint8, root, c->comm, c->stream);
        if (r != ncclSuccess) {
            set_error(std::string("ncclBroadcast: ") + ncclGetErrorString(r));
            return ETUNE_ERR_CUDA;
        }
        return ETUNE_OK;
    }
    if (c->transport.broadcast(c->transport.user, d_buf, int64_t(bytes), root, c->stream) != 0) {
        set_error("transport broadcast failed");
        return ETUNE_ERR_BACKEND_UNAVAILABLE;
    }
    return ETUNE_OK;
}
}  // namespace etune_b200

namespace {

std::mutex g_serial_mu;
uint64_t g_serial = 0;

etune_status fail(etune_status st, const std::string& msg) {
    set_error(msg);
    return st;
}

etune_status cuda_fail(cudaError_t e, const char* where) {
    return fail(ETUNE_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(expr)                                           \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

// Grows by at least 1.5x, so a caller whose size creeps up (the search loop retraining on
// a growing sample set) reallocates O(log) times; stream-ordered, no device-wide sync.
etune_status ensure_scratch(etune_cu_ctx* c, size_t bytes) {
    if (c->scratch_bytes >= bytes) return ETUNE_OK;
    const size_t want = std::max(bytes, c->scratch_bytes + c->scratch_bytes / 2);
    if (c->scratch) {
        CU(cudaFreeAsync(c->scratch, c->stream));
        c->scratch = nullptr;
        c->scratch_bytes = 0;
    }
    CU(cudaMallocAsync(&c->scratch, want, c->stream));
    c->scratch_bytes = want;
    return ETUNE_OK;
}

// Narrow rows [a, b) of the caller's Schedule[] to W-wide fields; false when a field
// does not fit (negative or >= 2^(8 sizeof W)), in which case the chunk is re-packed wider.
template <typename W>
bool narrow_rows(const etune_schedule* src, W* dst, int64_t a, int64_t b) {
    const int64_t* s = reinterpret_cast<const int64_t*>(src);
    uint64_t hi = 0;
    for (int64_t i = 12 * a; i < 12 * b; ++i) {
        const uint64_t v = uint64_t(s[i]);
        hi |= v >> (8 * sizeof(W));
        dst[i] = W(v);
    }
    return hi == 0;
}

// AVX-512 narrowing to u16 with non-temporal stores into the pinned staging (no
// read-for-ownership of the staging lines: the packing is host-DRAM bound).  Element range
// [lo, hi) of the int64 field array; lo must be a multiple of 8, dst 16-byte aligned.
__attribute__((target("avx512f"))) bool narrow_u16_avx512(const int64_t* s, uint16_t* d, int64_t lo, int64_t hi) {
    __m512i acc = _mm512_setzero_si512();
    int64_t i = lo;
    for (; i + 8 <= hi; i += 8) {
        const __m512i v = _mm512_loadu_si512(reinterpret_cast<const void*>(s + i));
        acc = _mm512_or_si512(acc, _mm512_srli_epi64(v, 16));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), _mm512_cvtepi64_epi16(v));
    }
    uint64_t tail = 0;
    for (; i < hi; ++i) {
        tail |= uint64_t(s[i]) >> 16;
        d[i] = uint16_t(s[i]);
    }
    _mm_sfence();  // the DMA engine reads the staging after the pool's hand-off
    return _mm512_test_epi64_mask(acc, acc) == 0 && tail == 0;
}

bool have_avx512() {
    static const bool ok = __builtin_cpu_supports("avx512f");
    return ok;
}

// Host threads for the *_host pipelines: the cores this process may run on, shared with the
// other ranks of the node when several run on it (LOCAL_WORLD_SIZE, set by torchrun), so that
// eight ranks do not oversubscribe the host; ETUNE_HOST_THREADS overrides.
int host_threads() {
    if (const char* e = std::getenv("ETUNE_HOST_THREADS")) return std::max(1, std::atoi(e));
    int n = 0;
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
    if (n < 1) n = int(std::max(1u, std::thread::hardware_concurrency()));
    if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) {
        const int w = std::atoi(lw);
        if (w > 1) n = std::max(1, n / w);
    }
    return n;
}

// Packs m rows into pinned `dst` with the narrowest field width that holds them (2, 4 or 8 bytes),
// split over the host pool.  start() hands the u16 pass to the workers and returns (the caller issues
// CUDA work meanwhile); finish() joins it, runs the wider fallbacks if a field did not fit, and returns
// the field width.  `extra` (optional): more pool tasks in the same dispatch (a previous chunk's
// outputs copied out of staging), run exactly once.  A job must not move while it runs.
struct PackJob {
    etune_cu_ctx* c = nullptr;
    const etune_schedule* src = nullptr;
    int64_t m = 0;
    void* dst = nullptr;
    int tasks = 0, extra_tasks = 0;
    bool simd = false;
    bool active = false;
    std::vector<char> ok;
    std::function<void(int)> extra, fn;

    PackJob() = default;
    PackJob(const PackJob&) = delete;
    PackJob& operator=(const PackJob&) = delete;
    ~PackJob() {  // an early return while the workers still run this job: wait for them
        if (active) c->pool->join();
    }

    void range(int t, int64_t* a, int64_t* b) const {  // even row boundaries: 24 fields = 3 AVX-512 words
        *a = (m * t / tasks) & ~int64_t(1);
        *b = t + 1 == tasks ? m : (m * (t + 1) / tasks) & ~int64_t(1);
    }
    void start(etune_cu_ctx* c_, const etune_schedule* s, int64_t m_, void* d, int xt, std::function<void(int)> xf) {
        c = c_;
        src = s;
        m = m_;
        dst = d;
        tasks = int(std::min<int64_t>(int64_t(c->pool->size()) * 2, std::max<int64_t>(1, m / 2048)));
        extra_tasks = xt;
        extra = std::move(xf);
        ok.assign(size_t(tasks), 1);
        simd = have_avx512() && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
        fn = [this](int t) {
            if (t >= tasks) return extra(t - tasks);
            int64_t a, b;
            range(t, &a, &b);
            ok[size_t(t)] = simd ? narrow_u16_avx512(reinterpret_cast<const int64_t*>(src), static_cast<uint16_t*>(dst),
                                                     12 * a, 12 * b)
                                 : narrow_rows(src, static_cast<uint16_t*>(dst), a, b);
        };
        c->pool->start(tasks + (extra ? extra_tasks : 0), fn);
        active = true;
    }
    int finish() {
        c->pool->join();
        active = false;
        auto all_ok = [&] { return std::all_of(ok.begin(), ok.end(), [](char x) { return x != 0; }); };
        if (all_ok()) return 2;
        c->pool->run(tasks, [&](int t) {
            int64_t a, b;
            range(t, &a, &b);
            ok[size_t(t)] = narrow_rows(src, static_cast<uint32_t*>(dst), a, b);
        });
        if (all_ok()) return 4;
        c->pool->run(tasks, [&](int t) {
            int64_t a, b;
            range(t, &a, &b);
            std::memcpy(static_cast<etune_schedule*>(dst) + a, src + a, size_t(b - a) * sizeof(etune_schedule));
        });
        return 8;
    }
};

etune_status ensure_io(etune_cu_ctx* c, size_t bytes) {
    if (c->io_bytes >= bytes) return ETUNE_OK;
    if (c->io) {
        CU(cudaStreamSynchronize(c->stream));
        CU(cudaFree(c->io));
        c->io = nullptr;
        c->io_bytes = 0;
    }
    CU(cudaMalloc(&c->io, bytes));
    c->io_bytes = bytes;
    return ETUNE_OK;
}

uint64_t order_key_host(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Buckets of the fused selection: the prediction range the forest can produce
// (base + lr * sum of per-tree leaf extremes, floored like EnergyModel::predict,
// energy_model.cpp:245-249), split into kSelBins equal spans of order keys.  Only the
// resolution depends on these bounds: the bucket function clamps, so it stays exact.
void selection_buckets(const ForestHost& F, uint64_t* kmin, uint32_t* shift) {
    double lo = 0.0, hi = 0.0;
    for (int64_t t = 0; t < F.num_trees(); ++t) {
        double tl = 0.0, th = 0.0;
        bool any = false;
        for (int64_t i = F.offsets[t]; i < F.offsets[t + 1]; ++i) {
            if (F.feature[i] >= 0) continue;
            const double v = F.value[i];
            tl = any ? std::min(tl, v) : v;
            th = any ? std::max(th, v) : v;
            any = true;
        }
        lo += tl;
        hi += th;
    }
    double plo = F.base + F.lr * (F.lr >= 0 ? lo : hi);
    double phi = F.base + F.lr * (F.lr >= 0 ? hi : lo);
    plo = std::max(1e-6, plo);
    phi = std::max(1e-6, phi);
    uint64_t a = order_key_host(plo), b = order_key_host(phi);
    if (!(b > a)) b = a + 1;  // degenerate or NaN bounds: any bucketing is still exact
    const uint64_t span = b - a;
    uint32_t s = 0;
    while (s < 63 && (span >> s) >= uint64_t(kSelBins)) ++s;
    *kmin = a;
    *shift = s;
}

constexpr int64_t kLazyWalkMaxN = int64_t(1) << 15;
constexpr int64_t kLazyWalkBudget = int64_t(1) << 18;

// `n` = the population about to be scored (-1: compile regardless)
etune_status get_compiled(etune_cu_forest* f, const etune_cu_plan* p, CompiledScore** out, int64_t n = -1) {
    std::lock_guard<std::mutex> lock(f->mu);
    auto it = f->compiled.find(p->serial);
    if (it != f->compiled.end()) {
        *out = &it->second;
        return ETUNE_OK;
    }
    if (f->lazy_compile && n >= 0 && n <= kLazyWalkMaxN) {
        int64_t& w = f->walked[p->serial];
        const int cap = max_dynamic_smem(f->ctx->device) - score_static_smem();
        if (w + n <= kLazyWalkBudget && p->build.hdr.total <= uint32_t(cap)) {
            static CompiledScore walk_only = [] {
                CompiledScore w0;
                w0.walk = true;
                return w0;
            }();
            w += n;
            *out = &walk_only;
            return ETUNE_OK;
        }
    }
    std::vector<uint8_t> blob;
    std::string err;
    CompiledScore cs;
    const etune_status bst = build_score_blob(f->host, p->build, &blob, &cs.stats, &err);
    if (bst != ETUNE_OK && bst != ETUNE_ERR_UNSUPPORTED) return fail(bst, err);
    const int cap = max_dynamic_smem(f->ctx->device) - score_static_smem();
    if (bst == ETUNE_ERR_UNSUPPORTED || blob.size() > size_t(cap)) {
        // the general path: features + the reference tree walk (any forest)
        if (p->build.hdr.total > uint32_t(cap)) return fail(ETUNE_ERR_UNSUPPORTED, "plan tables exceed shared memory");
        cs.walk = true;
        auto res = f->compiled.emplace(p->serial, cs);
        *out = &res.first->second;
        return ETUNE_OK;
    }
    CU(cudaMalloc(&cs.d_blob, blob.size()));
    CU(cudaMemcpyAsync(cs.d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice, f->ctx->stream));
    CU(cudaStreamSynchronize(f->ctx->stream));
    cs.bytes = uint32_t(blob.size());
    const ScoreHdr* hdr = reinterpret_cast<const ScoreHdr*>(blob.data());
    cs.mask_bits = hdr->mask_bits;
    CU(score_occupancy(cs.mask_bits, cs.bytes, &cs.per_sm));
    cs.params = std::make_shared<ForestParams>();
    std::memset(cs.params.get(), 0, sizeof(ForestParams));
    if (hdr->npairs > 0)
        std::memcpy(cs.params->pair, blob.data() + hdr->off_trees, sizeof(PairRec) * size_t(hdr->npairs));
    else
        std::memcpy(cs.params->rec, blob.data() + hdr->off_trees, sizeof(TreeRec) * size_t(hdr->ntrees));
    selection_buckets(f->host, &cs.sel_kmin, &cs.sel_shift);
    auto res = f->compiled.emplace(p->serial, cs);
    *out = &res.first->second;
    return ETUNE_OK;
}

// The keyed form is compiled on first use by a population of at least kKeyedMinN
// (its table build is a few ms of host work per (forest, plan): small populations,
// e.g. the search loop's per-round scoring, keep the class-table kernel).
constexpr int64_t kKeyedMinN = int64_t(1) << 16;

etune_status ensure_keyed(etune_cu_forest* f, const etune_cu_plan* p, CompiledScore* cs, int64_t n) {
    if (cs->walk || f->keyed_mode == 0 || n < kKeyedMinN) return ETUNE_OK;
    std::lock_guard<std::mutex> lock(f->mu);
    if (cs->keyed_tried) return ETUNE_OK;
    cs->keyed_tried = true;
    std::vector<uint8_t> blob;
    std::string err;
    ScoreStats st;
    KeyedBuild kb;
    if (build_score_blob(f->host, p->build, &blob, &st, &err, &kb, size_t(64) << 20,
                         f->keyed_mode == 2 ? 0 : size_t(64) << 20) != ETUNE_OK ||
        !kb.ok)
        return ETUNE_OK;
    const int cap = max_dynamic_smem(f->ctx->device) - score_static_smem();
    if (kb.blob.size() > size_t(cap)) return ETUNE_OK;
    CU(cudaMalloc(&cs->d_kblob, kb.blob.size()));
    CU(cudaMalloc(&cs->d_ktable, kb.table.size()));
    CU(cudaMalloc(&cs->d_khash, kb.khash.size() * sizeof(uint64_t)));
    CU(cudaMemcpyAsync(cs->d_khash, kb.khash.data(), kb.khash.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                       f->ctx->stream));
    CU(cudaMemcpyAsync(cs->d_kblob, kb.blob.data(), kb.blob.size(), cudaMemcpyHostToDevice, f->ctx->stream));
    CU(cudaMemcpyAsync(cs->d_ktable, kb.table.data(), kb.table.size(), cudaMemcpyHostToDevice, f->ctx->stream));
    CU(cudaStreamSynchronize(f->ctx->stream));
    // the full form's kernel stages (and sizes its shared memory for) the blob prefix it reads
    cs->kbytes = kb.params.kfull ? reinterpret_cast<const KeyedHdr*>(kb.blob.data())->full_bytes
                                 : uint32_t(kb.blob.size());
    cs->ktable_bytes = kb.table.size();
    cs->kparams = std::make_shared<KeyedParams>(kb.params);
    cs->key_bits = kb.key_bits;
    cs->nkeys = int(kb.nkeys);
    cs->nt1 = p->build.hdr.nt[1];
    cs->nt2 = p->build.hdr.nt[2];
    CU(score_keyed_occupancy(cs->kbytes, &cs->keyed_per_sm));
    cs->keyed = true;
    return ETUNE_OK;
}

bool use_keyed(const etune_cu_forest* f, const CompiledScore* cs, int64_t n) {
    return cs->keyed && f->keyed_mode != 0 && n >= kKeyedMinN && n < (int64_t(1) << 32);
}

// ------------------------------------------------------------ scoring forms
// AUTO: the device-compiled row table (rowtab.cu) once the (forest, plan) has scored
// kRowsMinN candidates (or one call brings that many); the tree walk before that (a model
// scored once on a few thousand candidates -- the search loop's per-round model -- is
// cheaper to walk than to tabulate).  Host-compiled forms only on request, or when the
// operator's row table would be too large.
constexpr int64_t kRowsMinN = int64_t(1) << 16;

void free_rowtab(RowTab& rt, cudaStream_t st) {
    cudaFreeAsync(rt.d_meta, st);
    cudaFreeAsync(rt.d_clskuv, st);
    cudaFreeAsync(rt.d_crep, st);
    cudaFreeAsync(rt.d_rowpred, st);
    cudaFreeAsync(rt.d_srows, st);
    cudaFreeAsync(rt.d_rowgid, st);
    cudaFreeAsync(rt.d_rowrec, st);
    rt = RowTab{};
}

void free_compiled(CompiledScore& cs) {
    cudaFree(cs.d_blob);
    cudaFree(cs.d_kblob);
    cudaFree(cs.d_ktable);
    cudaFree(cs.d_khash);
    cs.d_blob = cs.d_kblob = cs.d_ktable = nullptr;
    cs.d_khash = nullptr;
}

// Row table of (forest, plan), compiled on the device on first use: asynchronous on the ctx
// stream, no host arithmetic and no synchronisation.
etune_status ensure_rows(etune_cu_ctx* c, etune_cu_forest* f, const etune_cu_plan* p, RowTab** out) {
    std::lock_guard<std::mutex> lock(f->mu);
    auto it = f->rowtabs.find(p->serial);
    if (it != f->rowtabs.end()) {
        *out = &it->second;
        return ETUNE_OK;
    }
    if (p->rows_cap <= 0)
        return fail(ETUNE_ERR_UNSUPPORTED, "the operator's row table would exceed 2^25 rows (use another form)");
    const int ndk = p->build.hdr.ndk;
    const cudaStream_t st = c->stream;
    RowTab rt;
    void* scratch = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_meta), sizeof(RowTabMeta), st));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_clskuv), size_t(ndk) * 64 * 2, st));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_crep), size_t(p->kuv_domain) * 4, st));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_rowpred), size_t(p->rows_cap) * 8, st));
    CU(cudaMallocAsync(&scratch, rowtab_scratch_bytes(f->nnodes), st));
    const cudaError_t e = launch_rowtab_compile(c->lc(), p->d_blob, p->build.hdr.total, f->d_predict, f->predict_bytes,
                                                f->nnodes, ndk, p->rows_cap, scratch, rt.d_meta, rt.d_clskuv,
                                                rt.d_crep, rt.d_rowpred);
    cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) {
        free_rowtab(rt, st);
        return cuda_fail(e, "launch_rowtab_compile");
    }
    // rows in prediction order and their groups (dense ranks) for the fused selection (device radix sort)
    void* sscratch = nullptr;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_srows), size_t(p->rows_cap) * 4, st));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_rowgid), size_t(p->rows_cap) * 4, st));
    CU(cudaMallocAsync(reinterpret_cast<void**>(&rt.d_rowrec), size_t(p->rows_cap) * sizeof(RowRec), st));
    CU(cudaMallocAsync(&sscratch, rowtab_sort_scratch_bytes(p->rows_cap), st));
    const cudaError_t e2 = launch_rowtab_sort(c->lc(), rt.d_meta, rt.d_rowpred, p->rows_cap, rt.d_srows, rt.d_rowgid,
                                              rt.d_rowrec, sscratch);
    cudaFreeAsync(sscratch, st);
    if (e2 != cudaSuccess) {
        free_rowtab(rt, st);
        return cuda_fail(e2, "launch_rowtab_sort");
    }
    auto res = f->rowtabs.emplace(p->serial, rt);
    *out = &res.first->second;
    return ETUNE_OK;
}

struct Route {
    int kind = 0;  // 0: tree walk, 1: host-compiled form (cs), 2: row table (rt)
    CompiledScore* cs = nullptr;
    RowTab* rt = nullptr;
};

bool walk_fits(const etune_cu_ctx* c, const etune_cu_plan* p) {
    return p->build.hdr.total <= uint32_t(max_dynamic_smem(c->device));
}

// `n` = the population about to be scored; -1 = compile the form a large population would use
etune_status route(etune_cu_ctx* c, etune_cu_forest* f, const etune_cu_plan* p, int64_t n, Route* r) {
    int form = f->form;
    if (form == ETUNE_FORM_AUTO && p->rows_cap > 0) {
        bool have = false;
        int64_t cum = 0;
        {
            std::lock_guard<std::mutex> lock(f->mu);
            have = f->rowtabs.count(p->serial) != 0;
            cum = (f->seen[p->serial] += std::max<int64_t>(n, 0));
        }
        if (have || n < 0 || n >= kRowsMinN || cum >= kRowsMinN || !walk_fits(c, p)) form = ETUNE_FORM_ROWS;
        else form = ETUNE_FORM_WALK;
    }
    if (form == ETUNE_FORM_ROWS) {
        r->kind = 2;
        return ensure_rows(c, f, p, &r->rt);
    }
    if (form == ETUNE_FORM_WALK) {
        if (!walk_fits(c, p)) return fail(ETUNE_ERR_UNSUPPORTED, "plan tables exceed shared memory");
        r->kind = 0;
        return ETUNE_OK;
    }
    // host-compiled forms (AUTO without a row table: the keyed form, as in round 1)
    if (etune_status st = get_compiled(f, p, &r->cs, n)) return st;
    if (etune_status st = ensure_keyed(f, p, r->cs, n < 0 ? kKeyedMinN : n)) return st;
    r->kind = r->cs->walk ? 0 : 1;
    return ETUNE_OK;
}

// Scoring pass of any compiled form; `ev` (nullable) = {start, before the score kernel,
// after it} for etune_cu_profile_score.
etune_status score_dispatch(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f, const Route& r,
                            const uint64_t* d_genome, int64_t n, double* d_pred, uint64_t* d_ids,
                            const SelHist& sel, const cudaEvent_t* ev) {
    if (ev) CU(cudaEventRecord(ev[0], c->stream));
    if (ev) CU(cudaEventRecord(ev[1], c->stream));
    if (r.kind == 0) {
        CU(launch_score_walk(c->lc(), p->d_blob, p->build.hdr.total, f->d_predict, f->predict_bytes, d_genome, n,
                             d_pred, d_ids));
    } else if (r.kind == 2) {
        // one 8-byte gather per candidate from the row table; ids from the per-key FNV state
        CU(launch_score_rows(c->lc(), p->d_blob, p->build.hdr.ndk, r.rt->d_clskuv, r.rt->d_meta, r.rt->d_rowpred,
                             p->d_khk, d_genome, n, d_pred, d_ids, sel));
    } else if (use_keyed(f, r.cs, n)) {
        const CompiledScore* cs = r.cs;
        CU(launch_score_keyed(c->lc(), cs->d_kblob, cs->kbytes, cs->d_ktable, cs->ktable_bytes, cs->d_khash, d_genome,
                              nullptr, n, d_pred, d_ids, cs->keyed_per_sm, *cs->kparams, sel));
    } else {
        const CompiledScore* cs = r.cs;
        CU(launch_score(c->lc(), cs->d_blob, cs->bytes, d_genome, n, d_pred, d_ids, cs->mask_bits, *cs->params,
                        cs->per_sm, sel));
    }
    if (ev) CU(cudaEventRecord(ev[2], c->stream));
    return ETUNE_OK;
}

// Work area of the bucketed selection (sort.cu launch_select), its histogram and list counters
// zeroed unless the previous sequence completed (the finish kernel leaves them zeroed).
etune_status select_work(etune_cu_ctx* c, int64_t n, int64_t k) {
    const size_t need = select_scratch_bytes(n, k);
    if (c->sel_bytes < need) {
        if (c->sel) {
            CU(cudaStreamSynchronize(c->stream));
            CU(cudaFree(c->sel));
            c->sel = nullptr;
            c->sel_bytes = 0;
        }
        CU(cudaMalloc(&c->sel, need));
        c->sel_bytes = need;
        c->sel_dirty = true;
    }
    if (c->sel_dirty) CU(cudaMemsetAsync(c->sel, 0, 8192, c->stream));  // histogram + list counters
    c->sel_dirty = true;
    return ETUNE_OK;
}

// Fused score + keep-the-best on one shard: the score kernel fills the selection
// histogram, sel_filter/sel_finish (sort.cu) resolve the k lowest (score, index).
// Forests on the tree-walk path and k > kSelMaxK use score + the cooperative top-k.
etune_status score_select_local(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f, const Route& r,
                                const uint64_t* d_genome, int64_t n, int64_t k, double* d_pred, uint64_t* d_ids,
                                int64_t* d_idx) {
    if (r.kind == 2 && k > 0 && k <= kSelMaxK) {  // one cooperative kernel: score, row counts, k-th, ties, sort
        if (!c->rowsel) {
            CU(cudaMalloc(&c->rowsel, rowsel_work_bytes()));
            CU(cudaMemsetAsync(c->rowsel, 0, rowsel_work_bytes(), c->stream));
        }
        const bool prof = c->prof_on;
        if (prof && c->prof_used == c->prof_ev.size()) {
            std::array<cudaEvent_t, 4> e{};
            for (cudaEvent_t& x : e) CU(cudaEventCreate(&x));
            c->prof_ev.push_back(e);
        }
        const cudaEvent_t* ev = prof ? c->prof_ev[c->prof_used].data() : nullptr;
        if (ev) {
            CU(cudaEventRecord(ev[0], c->stream));
            CU(cudaEventRecord(ev[1], c->stream));
        }
        const cudaError_t e =
            launch_score_select_rows(c->lc(), p->d_blob, p->build.hdr.ndk, p->nkeys, p->build.hdr.nt,
                                     p->build.hdr.off_divk, r.rt->d_clskuv, r.rt->d_meta,
                                     r.rt->d_rowrec, p->d_khash, d_genome, n, k, d_pred,
                                     d_ids, d_idx, c->rowsel);
        if (e == cudaSuccess) {
            if (ev) {
                CU(cudaEventRecord(ev[2], c->stream));
                CU(cudaEventRecord(ev[3], c->stream));
                ++c->prof_used;
            }
            return ETUNE_OK;
        }
        if (e != cudaErrorNotSupported) return cuda_fail(e, "launch_score_select_rows");
        cudaGetLastError();  // population beyond the grid's registers: the bucketed selection below
    }
    if (r.kind == 0 || k > kSelMaxK || k == 0) {
        if (etune_status st = score_dispatch(c, p, f, r, d_genome, n, d_pred, d_ids, SelHist{}, nullptr)) return st;
        if (k == 0) return ETUNE_OK;
        if (etune_status st = ensure_scratch(c, topk_scratch_bytes(n))) return st;
        CU(launch_topk(c->lc(), d_pred, n, k, d_idx, c->scratch));
        return ETUNE_OK;
    }
    if (etune_status st = select_work(c, n, k)) return st;
    SelHist sh{select_hist(c->sel), 0, 0};
    if (r.kind == 2) sh.dbounds = r.rt->d_meta->bounds;  // exact range of the row predictions
    else {
        sh.kmin = r.cs->sel_kmin;
        sh.shift = r.cs->sel_shift;
    }
    const bool prof = c->prof_on;
    if (prof && c->prof_used == c->prof_ev.size()) {
        std::array<cudaEvent_t, 4> e{};
        for (cudaEvent_t& x : e) CU(cudaEventCreate(&x));
        c->prof_ev.push_back(e);
    }
    const cudaEvent_t* ev = prof ? c->prof_ev[c->prof_used].data() : nullptr;
    if (etune_status st = score_dispatch(c, p, f, r, d_genome, n, d_pred, d_ids, sh, ev)) return st;
    CU(launch_select(c->lc(), d_pred, n, k, d_idx, c->sel, sh));
    if (prof) CU(cudaEventRecord(c->prof_ev[c->prof_used++][3], c->stream));
    c->sel_dirty = false;
    return ETUNE_OK;
}

// records: [k local records | W*k gathered records | k local indices | merge scratch]
struct ShardBufs {
    ShardRec *lrec, *grec;
    int64_t* lidx;
    void* mscratch;
};

etune_status shard_buffers(etune_cu_ctx* c, int64_t k, ShardBufs* b) {
    const int W = ctx_world(c);
    const size_t need = size_t(k) * 16 * (1 + size_t(W)) + size_t(k) * 8 + merge_scratch_bytes(W, k) + 1024;
    if (c->shard_bytes < need) {
        if (c->shard) {
            CU(cudaStreamSynchronize(c->stream));
            CU(cudaFree(c->shard));
            c->shard = nullptr;
            c->shard_bytes = 0;
        }
        CU(cudaMalloc(&c->shard, need));
        c->shard_bytes = need;
    }
    b->lrec = static_cast<ShardRec*>(c->shard);
    b->grec = b->lrec + k;
    b->lidx = reinterpret_cast<int64_t*>(b->grec + size_t(W) * k);
    b->mscratch = b->lidx + k;
    return ETUNE_OK;
}

// Local top-kl indices in b.lidx -> (score, global index) records -> all-gather -> the identical
// merged top-k on every rank (one-CTA W-way merge of the rank-major sorted lists).
etune_status shard_merge(etune_cu_ctx* c, const double* d_score, int64_t kl, int64_t k, int64_t goff,
                         const ShardBufs& b, int64_t* d_idx, double* d_sc) {
    const int W = ctx_world(c);
    CU(launch_pack_records(c->lc(), d_score, b.lidx, kl, k, goff, b.lrec));
    if (etune_status st = coll_allgather(c, b.lrec, b.grec, size_t(k) * sizeof(ShardRec))) return st;
    CU(launch_merge_records(c->lc(), b.grec, W, k, d_idx, d_sc, b.mscratch));
    return ETUNE_OK;
}

}  // namespace

extern "C" {

void etune_default_device_config(etune_device_config* o) {  // device.hpp:17-45
    std::memset(o, 0, sizeof(*o));
    o->num_sms = 108;
    o->constant_power_w = 60.0;
    o->static_power_per_sm_w = 0.55;
    o->dynamic_energy_per_flop_nj = 0.002;
    o->dynamic_energy_per_glb_access_nj = 0.125;
    o->dynamic_energy_per_shared_access_nj = 0.0125;
    o->base_throughput_flops_per_s_per_sm = 1.8e11;
    o->mem_bandwidth_elems_per_s = 3.3e11;
    o->latency_floor_ms = 1e-5;
    o->sampler_hz = 50.0;
    o->warmup_s = 2.0;
    o->noise_sigma_rel = 0.05;
    o->rng_seed = 1234;
}
void etune_default_space_limits(etune_space_limits* o) {  // space.hpp:15-19
    o->max_block_threads = 1024;
    o->max_unroll = 8;
    o->max_vectorize = 4;
}
void etune_default_genetic_rates(etune_genetic_rates* o) {  // genetic.hpp:14-18
    o->mutation = 0.85;
    o->crossover = 0.10;
    o->copy = 0.05;
}
void etune_default_boost_params(etune_boost_params* o) {  // energy_model.hpp:33-41
    o->num_trees = 100;
    o->max_depth = 6;
    o->learning_rate = 0.1;
    o->min_leaf_weight = 1e-3;
    o->reg_lambda = 1.0;
}

const char* etune_cu_last_error(void) { return g_error.c_str(); }
int etune_cu_abi_version(void) { return ETUNE_CUDA_ABI_VERSION; }
uint64_t etune_cu_launch_count(void) { return launch_count(); }

etune_status etune_cu_ctx_create(int device, void* stream, etune_cu_ctx** out) {
    if (!out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "out is null");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
        return fail(ETUNE_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device));
    cudaDeviceProp prop{};
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(ETUNE_ERR_NO_DEVICE, std::string("device is ") + prop.name + " (sm_" + std::to_string(prop.major) +
                                             std::to_string(prop.minor) + "); this library is built for sm_100a");
    CU(cudaSetDevice(device));
    auto c = std::make_unique<etune_cu_ctx>();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->stream = static_cast<cudaStream_t>(stream);  // NULL = the default stream
    CU(cudaMalloc(&c->d_err, sizeof(unsigned long long)));
    CU(cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream));
    // scratch and forest tables are stream-ordered allocations: keep freed blocks in the
    // device pool instead of returning them to the driver at every synchronisation
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = ~uint64_t(0);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    *out = c.release();
    return ETUNE_OK;
}

etune_status etune_cu_ctx_destroy(etune_cu_ctx* c) {
    if (!c) return ETUNE_OK;
    c->closing.store(true);
    ctx_retain(c);
    ctx_release(c);  // frees now unless plans / forests / searches still hold it
    return ETUNE_OK;
}

etune_status etune_cu_ctx_set_stream(etune_cu_ctx* c, void* stream) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "ctx is null");
    CU(cudaStreamSynchronize(c->stream));
    if (c->own_stream) cudaStreamDestroy(c->stream);
    c->own_stream = false;
    c->stream = static_cast<cudaStream_t>(stream);
    return ETUNE_OK;
}

void* etune_cu_ctx_stream(etune_cu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

etune_status etune_cu_synchronize(etune_cu_ctx* c, int64_t* first_bad) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "ctx is null");
    unsigned long long v = kNoError;
    CU(cudaMemcpyAsync(&v, c->d_err, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (first_bad) *first_bad = -1;
    if (v == kNoError) return ETUNE_OK;
    CU(cudaMemsetAsync(c->d_err, 0xff, sizeof(unsigned long long), c->stream));
    const int64_t idx = int64_t(v >> 8);
    const etune_status st = etune_status(v & 0xffu);
    if (first_bad) *first_bad = idx;
    std::string what;
    switch (st) {
    case ETUNE_ERR_ILLEGAL_SCHEDULE:
        what = "schedule " + std::to_string(idx) + " does not fit the operator (validate_schedule)";
        break;
    case ETUNE_ERR_NON_POSITIVE_ENERGY:
        what = "measured energy at element " + std::to_string(idx) + " is not positive";
        break;
    case ETUNE_ERR_UNSUPPORTED:
        what = "element " + std::to_string(idx) + " cannot be represented by this build";
        break;
    default:
        what = "device-side error " + std::to_string(int(st)) + " at element " + std::to_string(idx);
    }
    return fail(st, what);
}

etune_status etune_cu_device_alloc(etune_cu_ctx* c, void** out, int64_t bytes) {
    if (!c || !out || bytes < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    CU(cudaSetDevice(c->device));
    CU(cudaMalloc(out, size_t(bytes > 0 ? bytes : 1)));
    return ETUNE_OK;
}

etune_status etune_cu_device_free(etune_cu_ctx* c, void* p) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    if (!p) return ETUNE_OK;
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaFree(p));
    return ETUNE_OK;
}

etune_status etune_cu_memcpy_h2d(etune_cu_ctx* c, void* d_dst, const void* h_src, int64_t bytes) {
    if (!c || bytes < 0 || (bytes > 0 && (!d_dst || !h_src))) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    if (bytes) CU(cudaMemcpyAsync(d_dst, h_src, size_t(bytes), cudaMemcpyHostToDevice, c->stream));
    return ETUNE_OK;
}

etune_status etune_cu_memcpy_d2h(etune_cu_ctx* c, void* h_dst, const void* d_src, int64_t bytes) {
    if (!c || bytes < 0 || (bytes > 0 && (!h_dst || !d_src))) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    if (bytes) CU(cudaMemcpyAsync(h_dst, d_src, size_t(bytes), cudaMemcpyDeviceToHost, c->stream));
    return ETUNE_OK;
}

etune_status etune_cu_plan_create(etune_cu_ctx* c, const etune_op_spec* op, const etune_device_config* dev,
                                  const etune_space_limits* limits, etune_cu_plan** out) {
    if (!c || !op || !out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    etune_device_config d;
    etune_default_device_config(&d);
    if (dev) d = *dev;
    etune_space_limits l;
    etune_default_space_limits(&l);
    if (limits) l = *limits;
    auto p = std::make_unique<etune_cu_plan>();
    p->ctx = c;
    std::string err;
    if (etune_status st = build_plan(*op, d, l, &p->build, &err)) return fail(st, err);
    CU(cudaSetDevice(c->device));
    CU(cudaMalloc(&p->d_blob, p->build.blob.size()));
    CU(cudaMemcpyAsync(p->d_blob, p->build.blob.data(), p->build.blob.size(), cudaMemcpyHostToDevice, c->stream));
    // row-table form: keys x legal (k_tile, unroll, vec) triples bound the table; per-key FNV state
    {
        const PlanHdr& H = p->build.hdr;
        const int64_t nkeys = int64_t(H.nt[0]) * H.nt[1] * H.nt[2];
        const int64_t dom = rowtab_kuv_domain(p->build.divk.data(), H.ndk);
        p->nkeys = nkeys;
        p->kuv_domain = dom;
        if (H.ndk <= 1024 && nkeys > 0 && nkeys <= (int64_t(1) << 24) && nkeys * dom <= (int64_t(1) << 25)) {
            p->rows_cap = nkeys * dom;
            CU(cudaMalloc(&p->d_khk, size_t(nkeys) * size_t(H.ndk) * 8));
            CU(cudaMalloc(&p->d_khash, size_t(nkeys + 2) * 8));  // + padding: whole 16-byte bulk copies
            CU(launch_key_hash(c->lc(), p->d_blob, nkeys, p->d_khk, p->d_khash));
        }
    }
    CU(cudaStreamSynchronize(c->stream));
    {
        std::lock_guard<std::mutex> lock(g_serial_mu);
        p->serial = ++g_serial;
    }
    ctx_retain(c);
    *out = p.release();
    return ETUNE_OK;
}

etune_status etune_cu_plan_destroy(etune_cu_plan* p) {
    if (!p) return ETUNE_OK;
    etune_cu_ctx* c = p->ctx;
    {  // evict every form compiled for this plan (plan serials are never reused)
        std::lock_guard<std::mutex> lk(c->forests_mu);
        for (etune_cu_forest* f : c->forests) {
            std::lock_guard<std::mutex> lock(f->mu);
            auto it = f->compiled.find(p->serial);
            if (it != f->compiled.end()) {
                free_compiled(it->second);
                f->compiled.erase(it);
            }
            auto rt = f->rowtabs.find(p->serial);
            if (rt != f->rowtabs.end()) {
                free_rowtab(rt->second, c->stream);
                f->rowtabs.erase(rt);
            }
            f->seen.erase(p->serial);
            f->walked.erase(p->serial);
        }
    }
    cudaStreamSynchronize(c->stream);  // kernels still reading the plan's tables
    cudaFree(p->d_khash);
    cudaFree(p->d_khk);
    cudaFree(p->d_blob);
    delete p;
    ctx_release(c);
    return ETUNE_OK;
}

etune_status etune_cu_plan_nest(const etune_cu_plan* p, int64_t out4[4]) {
    if (!p || !out4) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    op_nest(p->build.op, out4);
    return ETUNE_OK;
}

etune_status etune_cu_plan_space_size(const etune_cu_plan* p, int64_t* out) {
    if (!p || !out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    *out = p->build.space_size;
    return ETUNE_OK;
}

#define CHECK_PLAN_ARGS(ptr)                                                   \
    if (!c || !p) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx/plan");    \
    if (n < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "negative n");          \
    if (n > 0 && !(ptr)) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null buffer")

etune_status etune_cu_encode(etune_cu_ctx* c, const etune_cu_plan* p, const etune_schedule* d_sched, int64_t n,
                             uint64_t* d_genome) {
    CHECK_PLAN_ARGS(d_sched && d_genome);
    CU(launch_encode(c->lc(), p->d_blob, p->build.hdr.total, d_sched, n, d_genome));
    return ETUNE_OK;
}

etune_status etune_cu_decode(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_genome, int64_t n,
                             etune_schedule* d_sched) {
    CHECK_PLAN_ARGS(d_sched && d_genome);
    CU(launch_decode(c->lc(), p->d_blob, p->build.hdr.total, d_genome, n, d_sched));
    return ETUNE_OK;
}

etune_status etune_cu_sample_random(etune_cu_ctx* c, const etune_cu_plan* p, int64_t n, uint64_t seed,
                                    uint64_t* d_out, uint64_t* d_ids) {
    if (!c || !p) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx/plan");
    if (n < 1) return fail(ETUNE_ERR_VALIDATION, "sample_random requires n >= 1");
    if (!d_out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null output");
    const PlanBuild& B = p->build;
    const int64_t cap = std::max<int64_t>(2 * n, 4096);  // space.cpp:175
    const int64_t counted = std::min<int64_t>(B.space_size, cap + 1);
    if (counted < n)
        return fail(ETUNE_ERR_SPACE_EXHAUSTED, "requested " + std::to_string(n) + " candidates but only " +
                                                   std::to_string(counted) + " legal schedules exist");
    if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "n >= 2^31");
    int64_t* d_found = nullptr;
    int* d_flags = nullptr;
    if (etune_status st = ensure_scratch(c, 0)) return st;  // no-op; keeps the scratch policy uniform
    CU(cudaMallocAsync(reinterpret_cast<void**>(&d_found), 64, c->stream));
    d_flags = reinterpret_cast<int*>(d_found + 4);
    int64_t found = 0, flags = 0;
    if (counted <= cap) {
        const int64_t dims[6] = {B.hdr.nt[0], B.hdr.nt[1], B.hdr.nt[2], B.hdr.ndk, int64_t(B.unroll_opts.size()),
                                 int64_t(B.vec_opts.size())};
        int64_t q = 1;
        for (int i = 0; i < 6; ++i) q *= dims[i];
        if (etune_status st = ensure_scratch(c, sample_scratch_bytes(n, q, true))) return st;
        CU(launch_sample_small(c->lc(), p->d_blob, dims, seed, n, d_out, d_found, d_flags, c->scratch));
        CU(cudaMemcpyAsync(&found, d_found, 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        if (found != B.space_size) {
            cudaFree(d_found);
            return fail(ETUNE_ERR_CONSISTENCY, "device enumeration disagrees with the plan's space size");
        }
    } else {
        const int64_t max_attempts = 10000 + n * 1000;  // space.cpp:214
        int64_t A = std::min<int64_t>(max_attempts, n + n / 2 + 4096);
        for (;;) {
            if (etune_status st = ensure_scratch(c, sample_scratch_bytes(A, 0, false))) return st;
            CU(launch_sample_large(c->lc(), p->d_blob, seed, n, A, d_out, d_found, d_flags, c->scratch));
            int h_flags = 0;
            CU(cudaMemcpyAsync(&found, d_found, 8, cudaMemcpyDeviceToHost, c->stream));
            CU(cudaMemcpyAsync(&h_flags, d_flags, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            CU(cudaStreamSynchronize(c->stream));
            flags = h_flags;
            if (found >= n) break;
            if (A >= max_attempts || A >= (int64_t(1) << 30)) {
                cudaFree(d_found);
                return fail(ETUNE_ERR_SPACE_EXHAUSTED, "random sampling failed to find enough distinct candidates");
            }
            A = std::min<int64_t>(max_attempts, 2 * A);
        }
    }
    (void)flags;
    CU(cudaFreeAsync(d_found, c->stream));
    if (d_ids) CU(launch_ids(c->lc(), p->d_blob, B.hdr.total, d_out, n, d_ids));
    return ETUNE_OK;
}

etune_status etune_cu_candidate_ids(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_genome, int64_t n,
                                    uint64_t* d_ids) {
    CHECK_PLAN_ARGS(d_ids && d_genome);
    CU(launch_ids(c->lc(), p->d_blob, p->build.hdr.total, d_genome, n, d_ids));
    return ETUNE_OK;
}

etune_status etune_cu_counters(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_genome, int64_t n,
                               etune_counters* d_out) {
    CHECK_PLAN_ARGS(d_out && d_genome);
    CU(launch_counters(c->lc(), p->d_blob, p->build.hdr.total, d_genome, n, d_out));
    return ETUNE_OK;
}

etune_status etune_cu_features(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_genome, int64_t n,
                               double* d_feat, uint64_t* d_ids) {
    CHECK_PLAN_ARGS(d_feat && d_genome);
    CU(launch_features(c->lc(), p->d_blob, p->build.hdr.total, d_genome, n, d_feat, d_ids));
    return ETUNE_OK;
}

etune_status etune_cu_sim_measure(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_genome, int64_t n,
                                  double* d_lat, double* d_pow, double* d_en, int64_t* d_iters) {
    CHECK_PLAN_ARGS(d_genome && d_lat);
    const etune_device_config& D = p->build.dev;
    SimDevice d{D.base_throughput_flops_per_s_per_sm,
                D.mem_bandwidth_elems_per_s,
                D.latency_floor_ms,
                D.dynamic_energy_per_flop_nj,
                D.dynamic_energy_per_glb_access_nj,
                D.dynamic_energy_per_shared_access_nj,
                D.constant_power_w,
                D.static_power_per_sm_w,
                D.sampler_hz,
                D.noise_sigma_rel,
                D.rng_seed};
    CU(launch_sim_measure(c->lc(), p->d_blob, p->build.hdr.total, d_genome, n, d, d_lat, d_pow, d_en, d_iters));
    return ETUNE_OK;
}

void etune_default_nvml_params(etune_nvml_params* o) {
    o->warmup_ms = 50.0;
    o->window_ms = 200.0;
    o->min_iterations = 10;
    o->max_iterations = 1000000;
}

etune_status etune_cu_nvml_available(etune_cu_ctx* c, int* out) {
    if (!c || !out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    std::string why;
    *out = nvml_device_handle(c->device, &why) != nullptr ? 1 : 0;
    return ETUNE_OK;
}

namespace {

struct CandOperands {
    float *a = nullptr, *b = nullptr, *c = nullptr;
    ~CandOperands() {
        cudaFree(a);
        cudaFree(b);
        cudaFree(c);
    }
};

// operand element counts of the op (A, B, C)
void operand_sizes(const etune_op_spec& op, const int64_t nest[4], int64_t* na, int64_t* nb, int64_t* nc) {
    if (op.kind == 2) {
        *na = op.batch * op.in_channels * op.height * op.width;
        *nb = op.out_channels * nest[3];
    } else {
        *na = nest[0] * nest[1] * nest[3];
        *nb = nest[0] * nest[3] * nest[2];
    }
    *nc = nest[0] * nest[1] * nest[2];
}

etune_status prepare_candidate(etune_cu_ctx* c, const etune_cu_plan* p, const etune_schedule& s,
                               std::vector<uint8_t>* geom, size_t* smem, int* grid, int* block, bool* feasible) {
    int64_t nest[4];
    op_nest(p->build.op, nest);
    geom->assign(candidate_geom_bytes(), 0);
    const int cap = max_dynamic_smem(c->device);
    *feasible = candidate_geometry(p->build.op, nest, s, cap, geom->data(), smem, grid, block);
    if (*feasible) *feasible = candidate_fits(geom->data(), *block);
    return ETUNE_OK;
}

}  // namespace

etune_status etune_cu_candidate_run(etune_cu_ctx* c, const etune_cu_plan* p, const etune_schedule* h_sched,
                                    const float* d_a, const float* d_b, float* d_c) {
    if (!c || !p || !h_sched || !d_a || !d_b || !d_c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    std::vector<uint8_t> geom;
    size_t smem = 0;
    int grid = 0, block = 0;
    bool ok = false;
    if (etune_status st = prepare_candidate(c, p, *h_sched, &geom, &smem, &grid, &block, &ok)) return st;
    if (!ok) return fail(ETUNE_ERR_UNSUPPORTED, "schedule infeasible for the candidate kernel");
    CU(launch_candidate(c->stream, geom.data(), smem, grid, block, d_a, d_b, d_c));
    note_launches(1);
    return ETUNE_OK;
}

etune_status etune_cu_candidate_latency(etune_cu_ctx* c, const etune_cu_plan* p, const etune_schedule* h_sched,
                                        int64_t n, int32_t reps, double* h_ms) {
    if (!c || !p || n < 0 || (n > 0 && (!h_sched || !h_ms)) || reps < 1)
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    if (n == 0) return ETUNE_OK;
    int64_t nest[4];
    op_nest(p->build.op, nest);
    int64_t na = 0, nb = 0, nc = 0;
    operand_sizes(p->build.op, nest, &na, &nb, &nc);
    CandOperands ops;
    CU(cudaMalloc(&ops.a, size_t(na) * 4));
    CU(cudaMalloc(&ops.b, size_t(nb) * 4));
    CU(cudaMalloc(&ops.c, size_t(nc) * 4));
    CU(launch_fill(c->stream, ops.a, na, 1u));
    CU(launch_fill(c->stream, ops.b, nb, 2u));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    etune_status result = ETUNE_OK;
    for (int64_t i = 0; i < n; ++i) {
        std::vector<uint8_t> geom;
        size_t smem = 0;
        int grid = 0, block = 0;
        bool ok = false;
        prepare_candidate(c, p, h_sched[i], &geom, &smem, &grid, &block, &ok);
        if (!ok) {
            h_ms[i] = std::numeric_limits<double>::infinity();
            continue;
        }
        cudaError_t e = launch_candidate(c->stream, geom.data(), smem, grid, block, ops.a, ops.b, ops.c);  // warm
        cudaEventRecord(e0, c->stream);
        for (int r = 0; r < reps && e == cudaSuccess; ++r)
            e = launch_candidate(c->stream, geom.data(), smem, grid, block, ops.a, ops.b, ops.c);
        cudaEventRecord(e1, c->stream);
        if (e != cudaSuccess) {
            result = cuda_fail(e, "candidate kernel");
            break;
        }
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        h_ms[i] = double(ms) / reps;
        note_launches(reps + 1);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return result;
}

etune_status etune_cu_nvml_measure(etune_cu_ctx* c, const etune_cu_plan* p, const etune_schedule* h_sched, int64_t n,
                                   const etune_nvml_params* params, etune_measurement* h_out, int64_t* first_bad) {
    if (!c || !p || (n > 0 && (!h_sched || !h_out)) || n < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    if (first_bad) *first_bad = -1;
    if (n == 0) return ETUNE_OK;
    std::string why;
    void* nv = nvml_device_handle(c->device, &why);
    if (!nv) return fail(ETUNE_ERR_BACKEND_UNAVAILABLE, "NVML energy counters unavailable: " + why);
    etune_nvml_params P;
    etune_default_nvml_params(&P);
    if (params) P = *params;
    // legality + ids on the device (validate_schedule, candidate_id)
    etune_schedule* d_s = nullptr;
    uint64_t *d_g = nullptr, *d_id = nullptr;
    CU(cudaMalloc(&d_s, size_t(n) * sizeof(etune_schedule)));
    CU(cudaMalloc(&d_g, size_t(n) * 8));
    CU(cudaMalloc(&d_id, size_t(n) * 8));
    CU(cudaMemcpyAsync(d_s, h_sched, size_t(n) * sizeof(etune_schedule), cudaMemcpyHostToDevice, c->stream));
    CU(launch_encode(c->lc(), p->d_blob, p->build.hdr.total, d_s, n, d_g));
    CU(launch_ids(c->lc(), p->d_blob, p->build.hdr.total, d_g, n, d_id));
    std::vector<uint64_t> ids(static_cast<size_t>(n));
    CU(cudaMemcpyAsync(ids.data(), d_id, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    const etune_status vst = etune_cu_synchronize(c, first_bad);
    cudaFree(d_s);
    cudaFree(d_g);
    cudaFree(d_id);
    if (vst != ETUNE_OK) return vst;
    int64_t nest[4];
    op_nest(p->build.op, nest);
    int64_t na = 0, nb = 0, nc = 0;
    operand_sizes(p->build.op, nest, &na, &nb, &nc);
    CandOperands ops;
    CU(cudaMalloc(&ops.a, size_t(na) * 4));
    CU(cudaMalloc(&ops.b, size_t(nb) * 4));
    CU(cudaMalloc(&ops.c, size_t(nc) * 4));
    CU(launch_fill(c->stream, ops.a, na, 1u));
    CU(launch_fill(c->stream, ops.b, nb, 2u));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    auto now_ms = [] {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    etune_status result = ETUNE_OK;
    for (int64_t i = 0; i < n && result == ETUNE_OK; ++i) {
        etune_measurement& r = h_out[i];
        std::memset(&r, 0, sizeof(r));
        r.candidate_id = ids[size_t(i)];
        std::vector<uint8_t> geom;
        size_t smem = 0;
        int grid = 0, block = 0;
        bool ok = false;
        prepare_candidate(c, p, h_sched[i], &geom, &smem, &grid, &block, &ok);
        if (!ok) {
            r.feasible = 0;
            r.latency_ms = r.energy_mj = std::numeric_limits<double>::infinity();
            continue;
        }
        r.feasible = 1;
        auto run = [&](int64_t reps) -> cudaError_t {
            for (int64_t q = 0; q < reps; ++q) {
                const cudaError_t e = launch_candidate(c->stream, geom.data(), smem, grid, block, ops.a, ops.b, ops.c);
                if (e != cudaSuccess) return e;
            }
            return cudaSuccess;
        };
        // warm-up (pre-heat) and a latency estimate for the window
        int64_t reps = 1;
        double est = 0.0, spent = 0.0;
        while (true) {
            cudaEventRecord(e0, c->stream);
            if (cudaError_t e = run(reps)) {
                result = cuda_fail(e, "candidate kernel");
                break;
            }
            cudaEventRecord(e1, c->stream);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            est = double(ms) / double(reps);
            spent += ms;
            if (spent >= P.warmup_ms) break;
            reps = std::min<int64_t>(reps * 4, std::max<int64_t>(1, int64_t((P.warmup_ms - spent) / std::max(est, 1e-4))));
        }
        if (result != ETUNE_OK) break;
        int64_t iters = int64_t(std::ceil(P.window_ms / std::max(est, 1e-6)));
        iters = std::max<int64_t>(P.min_iterations, std::min<int64_t>(P.max_iterations, iters));
        unsigned long long mj0 = 0, mj1 = 0;
        const double w0 = now_ms();
        nvml_energy_mj(nv, &mj0);
        cudaEventRecord(e0, c->stream);
        if (cudaError_t e = run(iters)) {
            result = cuda_fail(e, "candidate kernel");
            break;
        }
        cudaEventRecord(e1, c->stream);
        // while the repeats run: NVML power samples every ~2 ms (the paper's sampler,
        // PAPER:184-185), used when the energy counter has not ticked over the window
        double psum = 0.0;
        int64_t pn = 0;
        while (cudaEventQuery(e1) == cudaErrorNotReady) {
            unsigned int mw = 0;
            if (nvml_power_mw(nv, &mw)) {
                psum += double(mw);
                ++pn;
            }
            const double t = now_ms();
            while (now_ms() - t < 2.0) {
            }
        }
        cudaEventSynchronize(e1);
        nvml_energy_mj(nv, &mj1);
        const double wall = now_ms() - w0;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        note_launches(int(std::min<int64_t>(iters, 1 << 30)));
        r.iterations = iters;
        r.latency_ms = double(ms) / double(iters);
        if (mj1 > mj0) {
            r.avg_power_w = double(mj1 - mj0) / wall;  // mJ / ms = W
        } else {
            if (pn == 0) {
                unsigned int mw = 0;
                nvml_power_mw(nv, &mw);
                psum = double(mw);
                pn = 1;
            }
            r.avg_power_w = psum / double(pn) / 1000.0;
        }
        r.energy_mj = r.avg_power_w * r.latency_ms;  // SPEC:302 identity (W x ms = mJ)
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return result;
}

etune_status etune_cu_forest_create(etune_cu_ctx* c, const int32_t* feature, const double* threshold,
                                    const int32_t* left, const int32_t* right, const double* value,
                                    const int64_t* tree_offsets, int64_t num_trees, double base_score,
                                    double learning_rate, etune_cu_forest** out) {
    if (!c || !out || !tree_offsets || num_trees < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    auto f = std::make_unique<etune_cu_forest>();
    f->ctx = c;
    const int64_t nn = tree_offsets[num_trees];
    if (nn < 0 || (nn > 0 && (!feature || !threshold || !left || !right || !value)))
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "null node arrays");
    f->host.feature.assign(feature, feature + nn);
    f->host.threshold.assign(threshold, threshold + nn);
    f->host.left.assign(left, left + nn);
    f->host.right.assign(right, right + nn);
    f->host.value.assign(value, value + nn);
    f->host.offsets.assign(tree_offsets, tree_offsets + num_trees + 1);
    f->host.base = base_score;
    f->host.lr = learning_rate;
    std::vector<uint8_t> blob;
    std::string err;
    if (etune_status st = build_predict_blob(f->host, &blob, &err)) return fail(st, err);
    CU(cudaSetDevice(c->device));
    CU(cudaMallocAsync(&f->d_predict, blob.size(), c->stream));
    CU(cudaMemcpyAsync(f->d_predict, blob.data(), blob.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    f->predict_bytes = uint32_t(blob.size());
    f->nnodes = int(nn);
    ctx_retain(c);
    {
        std::lock_guard<std::mutex> lk(c->forests_mu);
        c->forests.insert(f.get());
    }
    *out = f.release();
    return ETUNE_OK;
}

etune_status etune_cu_forest_destroy(etune_cu_forest* f) {
    if (!f) return ETUNE_OK;
    etune_cu_ctx* c = f->ctx;
    {
        std::lock_guard<std::mutex> lk(c->forests_mu);
        c->forests.erase(f);
    }
    cudaFreeAsync(f->d_predict, c->stream);  // stream-ordered: after the forest's last use on the ctx stream
    for (auto& kv : f->compiled) free_compiled(kv.second);
    for (auto& kv : f->rowtabs) free_rowtab(kv.second, c->stream);
    delete f;
    ctx_release(c);
    return ETUNE_OK;
}

etune_status etune_cu_predict(etune_cu_ctx* c, etune_cu_forest* f, const double* d_feat, int64_t n,
                              double* d_pred) {
    if (!c || !f) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx/forest");
    if (n < 0 || (n > 0 && (!d_feat || !d_pred))) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad buffers");
    CU(launch_predict(c->lc(), f->d_predict, f->predict_bytes, d_feat, n, d_pred));
    return ETUNE_OK;
}

etune_status etune_cu_score(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f, const uint64_t* d_genome,
                            int64_t n, double* d_pred, uint64_t* d_ids) {
    CHECK_PLAN_ARGS(d_genome && d_pred);
    if (!f) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null forest");
    Route r;
    if (etune_status st = route(c, f, p, n, &r)) return st;
    return score_dispatch(c, p, f, r, d_genome, n, d_pred, d_ids, SelHist{}, nullptr);
}

etune_status etune_cu_score_select(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f,
                                   const uint64_t* d_genome, int64_t n, int64_t k, double* d_pred, uint64_t* d_ids,
                                   int64_t* d_idx) {
    CHECK_PLAN_ARGS(d_genome && d_pred);
    if (!f) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null forest");
    if (k < 0 || k > n) return fail(ETUNE_ERR_INVALID_ARGUMENT, "need 0 <= k <= n");
    if (k > 0 && !d_idx) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null index buffer");
    if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "n >= 2^31");
    Route r;
    if (etune_status st = route(c, f, p, n, &r)) return st;
    return score_select_local(c, p, f, r, d_genome, n, k, d_pred, d_ids, d_idx);
}

etune_status etune_cu_score_select_sharded(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f,
                                           const uint64_t* d_genome, int64_t n, int64_t goff, int64_t k,
                                           double* d_pred, uint64_t* d_ids, int64_t* d_idx, double* d_sc) {
    CHECK_PLAN_ARGS(d_pred && (n == 0 || d_genome));
    if (!f) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null forest");
    if (k < 0 || goff < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "negative size");
    if (k == 0) return ETUNE_OK;
    if (!d_idx) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null buffer");
    if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "shard >= 2^31");
    Route r;
    if (etune_status st = route(c, f, p, n, &r)) return st;
    ShardBufs sb;
    if (etune_status st = shard_buffers(c, k, &sb)) return st;
    const int64_t kl = std::min(k, n);
    if (etune_status st = score_select_local(c, p, f, r, d_genome, n, kl, d_pred, d_ids, sb.lidx)) return st;
    return shard_merge(c, d_pred, kl, k, goff, sb, d_idx, d_sc);
}

etune_status etune_cu_forest_set_keyed(etune_cu_forest* f, int mode) {
    if (!f || mode < 0 || mode > 2) return fail(ETUNE_ERR_INVALID_ARGUMENT, "mode must be 0, 1 or 2");
    f->keyed_mode = mode;
    f->form = mode == 0 ? ETUNE_FORM_CLASS : mode == 1 ? ETUNE_FORM_KEYED : ETUNE_FORM_KEYED_BYTE;
    return ETUNE_OK;
}

etune_status etune_cu_forest_set_form(etune_cu_forest* f, int form) {
    if (!f || form < ETUNE_FORM_AUTO || form > ETUNE_FORM_KEYED_BYTE)
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "form must be one of ETUNE_FORM_*");
    f->form = form;
    if (form == ETUNE_FORM_CLASS) f->keyed_mode = 0;
    if (form == ETUNE_FORM_KEYED) f->keyed_mode = 1;
    if (form == ETUNE_FORM_KEYED_BYTE) f->keyed_mode = 2;
    return ETUNE_OK;
}

etune_status etune_cu_forest_compile(etune_cu_ctx* c, etune_cu_forest* f, const etune_cu_plan* p) {
    if (!c || !f || !p) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    Route r;
    return route(c, f, p, -1, &r);
}

etune_status etune_cu_forest_rows_info(etune_cu_ctx* c, etune_cu_forest* f, const etune_cu_plan* p, int64_t out[8]) {
    if (!c || !f || !p || !out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    for (int i = 0; i < 8; ++i) out[i] = 0;
    RowTab* rt = nullptr;
    {
        std::lock_guard<std::mutex> lock(f->mu);
        auto it = f->rowtabs.find(p->serial);
        if (it != f->rowtabs.end()) rt = &it->second;
    }
    if (!rt) return ETUNE_OK;
    RowTabMeta m{};
    CU(cudaMemcpyAsync(&m, rt->d_meta, sizeof(m), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    out[0] = p->nkeys;
    out[1] = m.nkc;
    out[2] = p->nkeys * m.nkc;
    out[3] = p->nkeys * m.nkc * 8;
    out[4] = m.nthr[0];
    out[5] = m.nthr[1];
    out[6] = m.nthr[2];
    out[7] = p->kuv_domain;
    return ETUNE_OK;
}

etune_status etune_cu_forest_score_form(etune_cu_forest* f, const etune_cu_plan* p, int* form) {
    if (!f || !p || !form) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    Route r;
    if (etune_status st = route(f->ctx, f, p, -1, &r)) return st;
    if (r.kind == 2) *form = 4;
    else if (r.kind == 0) *form = 3;
    else *form = !use_keyed(f, r.cs, kKeyedMinN) ? 0 : r.cs->kparams->kfull ? 2 : 1;
    return ETUNE_OK;
}

etune_status etune_cu_profile_score(etune_cu_ctx* c, int on, double* prep_ms, double* score_ms, double* select_ms,
                                    int64_t* launches) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    double pre = 0.0, ms = 0.0, sel = 0.0;
    if (c->prof_used) {
        CU(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < c->prof_used; ++i) {
            float a = 0.f, e = 0.f, f = 0.f;
            CU(cudaEventElapsedTime(&a, c->prof_ev[i][0], c->prof_ev[i][1]));
            CU(cudaEventElapsedTime(&e, c->prof_ev[i][1], c->prof_ev[i][2]));
            CU(cudaEventElapsedTime(&f, c->prof_ev[i][2], c->prof_ev[i][3]));
            pre += a;
            ms += e;
            sel += f;
        }
    }
    if (prep_ms) *prep_ms = pre;
    if (score_ms) *score_ms = ms;
    if (select_ms) *select_ms = sel;
    if (launches) *launches = int64_t(c->prof_used);
    c->prof_used = 0;
    c->prof_on = on != 0;
    return ETUNE_OK;
}

}  // extern "C"

namespace {

// Host-buffer pipeline of etune_cu_score_host / etune_cu_score_select_host.  k > 0: the chunks'
// predictions stay on the device (d_all) and every score kernel also fills the selection
// histogram; after the last chunk the k best by (prediction, index) are resolved on the device
// and only the k indices come back besides the predictions.
etune_status host_pipeline(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f, const etune_schedule* h_sched,
                           int64_t n, double* h_pred, uint64_t* h_ids, int64_t k, int64_t* h_idx,
                           int64_t* first_bad) {
    if (first_bad) *first_bad = -1;
    if (n == 0) return ETUNE_OK;
    Route r;
    if (etune_status st = route(c, f, p, n, &r)) return st;
    double* d_all = nullptr;
    int64_t* d_idx = nullptr;
    SelHist sh{};
    if (k > 0) {
        const size_t need = size_t(n) * 8 + size_t(k) * 8 + 256;
        if (c->e2e_bytes < need) {
            if (c->e2e) {
                CU(cudaStreamSynchronize(c->stream));
                CU(cudaFree(c->e2e));
                c->e2e = nullptr;
                c->e2e_bytes = 0;
            }
            CU(cudaMalloc(&c->e2e, need));
            c->e2e_bytes = need;
        }
        d_all = static_cast<double*>(c->e2e);
        d_idx = reinterpret_cast<int64_t*>(static_cast<char*>(c->e2e) + ((size_t(n) * 8 + 255) & ~size_t(255)));
        if (r.kind != 0 && k <= kSelMaxK) {
            if (etune_status st = select_work(c, n, k)) return st;
            sh.hist = select_hist(c->sel);
            if (r.kind == 2) sh.dbounds = r.rt->d_meta->bounds;
            else {
                sh.kmin = r.cs->sel_kmin;
                sh.shift = r.cs->sel_shift;
            }
        }
    }
    // Chunked pipeline over two staging buffers.  The host pool narrows chunk i's rows
    // into pinned staging (24 B/row when every field fits 16 bits) while the GPU works
    // on chunk i-1; then H2D of chunk i (copy-in stream) overlaps encode+score of chunk
    // i-1 (ctx stream) and D2H of chunk i-2 (copy-out stream).  One synchronisation at
    // the end.
    static const int chunk_log2 = [] {  // ETUNE_E2E_CHUNK_LOG2 (diagnostic), default 2^17 rows
        const char* ev = std::getenv("ETUNE_E2E_CHUNK_LOG2");
        const int v = ev ? std::atoi(ev) : 17;
        return v < 12 ? 12 : v > 22 ? 22 : v;
    }();
    const int64_t chunk = int64_t(1) << chunk_log2;
    const size_t per = sizeof(etune_schedule) + 8 + 8 + 8;  // rows (widest), genome, pred, id
    const int64_t cap = n < chunk ? n : chunk;
    if (etune_status st = ensure_io(c, 2 * size_t(cap) * per)) return st;
    const size_t pin_need = 2 * size_t(cap) * sizeof(etune_schedule);
    if (c->hpin_bytes < pin_need) {
        if (c->hpin) {
            CU(cudaStreamSynchronize(c->stream));
            CU(cudaFreeHost(c->hpin));
            c->hpin = nullptr;
            c->hpin_bytes = 0;
        }
        CU(cudaHostAlloc(&c->hpin, pin_need, cudaHostAllocDefault));
        c->hpin_bytes = pin_need;
    }
    if (!c->pool) c->pool.reset(new HostPool(host_threads() - 1));
    if (!c->h2d) {
        CU(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            CU(cudaEventCreateWithFlags(&c->ev_in[b], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c->ev_done[b], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c->ev_out[b], cudaEventDisableTiming));
        }
    }
    // When the caller's rows are pinned, every raw_every-th chunk skips the host narrowing:
    // the copy engine moves its 96-byte rows as they are (the device encodes 8-byte
    // fields) while the host pool narrows the next chunks, so copy engine and host
    // memory bandwidth both work (ETUNE_E2E_RAW_EVERY, default 4; 0 disables).
    static const int raw_every = [] {
        const char* ev = std::getenv("ETUNE_E2E_RAW_EVERY");
        return ev ? std::atoi(ev) : 4;
    }();
    auto is_pinned = [](const void* ptr) {
        cudaPointerAttributes pa{};
        const bool r = ptr && cudaPointerGetAttributes(&pa, ptr) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        return r;
    };
    const bool pinned = is_pinned(h_sched);
    // Outputs into pageable memory (a std::vector<double>, a numpy array) would make every D2H
    // synchronous: they land in pinned staging instead and the host pool copies them out while the
    // next chunks run.
    const bool stage_out = (h_pred && !is_pinned(h_pred)) || (h_ids && !is_pinned(h_ids));
    if (stage_out && c->hout_bytes < 2 * size_t(cap) * 16) {
        if (c->hout) {
            CU(cudaStreamSynchronize(c->d2h));
            CU(cudaFreeHost(c->hout));
            c->hout = nullptr;
            c->hout_bytes = 0;
        }
        CU(cudaHostAlloc(&c->hout, 2 * size_t(cap) * 16, cudaHostAllocDefault));
        c->hout_bytes = 2 * size_t(cap) * 16;
    }
    int64_t pend_lo[2] = {-1, -1}, pend_m[2] = {0, 0};  // staged chunk waiting in hout buffer b
    auto out_tasks = [&](int64_t m2) {
        return int(std::min<int64_t>(int64_t(c->pool->size()) * 2, std::max<int64_t>(1, m2 / 4096)));
    };
    // part t of staging buffer b's outputs (rows [lo2, lo2 + m2) of the call) to the caller's arrays
    auto out_copy = [=](int b, int64_t lo2, int64_t m2, int t, int tasks) {
        const double* sp = reinterpret_cast<const double*>(static_cast<char*>(c->hout) + size_t(b) * size_t(cap) * 16);
        const uint64_t* si = reinterpret_cast<const uint64_t*>(sp + cap);
        const int64_t a = m2 * t / tasks, e = m2 * (t + 1) / tasks;
        if (h_pred) std::memcpy(h_pred + lo2 + a, sp + a, size_t(e - a) * 8);
        if (h_ids) std::memcpy(h_ids + lo2 + a, si + a, size_t(e - a) * 8);
    };
    auto drain = [&](int b) -> etune_status {  // (the pool must be idle)
        if (pend_lo[b] < 0) return ETUNE_OK;
        CU(cudaEventSynchronize(c->ev_out[b]));
        const int64_t lo2 = pend_lo[b], m2 = pend_m[b];
        const int tasks = out_tasks(m2);
        c->pool->run(tasks, [&](int t) { out_copy(b, lo2, m2, t, tasks); });
        pend_lo[b] = -1;
        return ETUNE_OK;
    };
    // chunk sizes: full chunks, then the last full chunk split so that the final one is a quarter chunk
    // (the tail after the last narrowing -- its copy in, scoring, copy out -- shrinks with it)
    std::vector<std::pair<int64_t, int64_t>> chunks;  // (first row, rows)
    for (int64_t lo = 0, m = 0; lo < n; lo += m) {
        const int64_t rem = n - lo, q = chunk / 4;
        m = rem <= q ? rem : rem <= chunk + q ? rem - q : chunk;
        chunks.emplace_back(lo, m);
    }
    const int nch = int(chunks.size());
    auto is_raw = [&](int i) { return pinned && raw_every > 0 && i % raw_every == 0 && chunks[size_t(i)].second == chunk; };
    // the caller's earlier work on the ctx stream happens-before this call's copies
    CU(cudaEventRecord(c->ev_done[0], c->stream));
    CU(cudaStreamWaitEvent(c->h2d, c->ev_done[0], 0));
    CU(cudaStreamWaitEvent(c->d2h, c->ev_done[0], 0));
    // ETUNE_E2E_TRACE=1 (diagnostic): host time spent joining the narrowing and waiting for staging, per call
    static const bool e2e_trace = std::getenv("ETUNE_E2E_TRACE") != nullptr;
    double e2e_pack_us = 0.0, e2e_wait_us = 0.0;
    const auto e2e_t0 = std::chrono::steady_clock::now();
    char* io = static_cast<char*>(c->io);
    char* pin = static_cast<char*>(c->hpin);
    PackJob jobs[2];
    // Chunk i's narrowing starts on the pool workers before chunk i-1's CUDA work is issued by this
    // thread (which then joins it), so the launches and copies of one chunk overlap the next one's
    // narrowing.  Its staging buffer i & 1 was read by chunk i-2's H2D; chunk i-2's outputs, still in
    // output staging buffer i & 1, leave it in the same dispatch when their D2H has landed.
    auto begin = [&](int i) -> etune_status {
        if (is_raw(i)) return ETUNE_OK;
        const int b = i & 1;
        const auto tw0 = std::chrono::steady_clock::now();
        if (i >= 2) CU(cudaEventSynchronize(c->ev_in[b]));
        if (e2e_trace) e2e_wait_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tw0).count();
        int xt = 0;
        std::function<void(int)> xf;
        if (stage_out && pend_lo[b] >= 0 && cudaEventQuery(c->ev_out[b]) == cudaSuccess) {
            const int64_t lo2 = pend_lo[b], m2 = pend_m[b];
            xt = out_tasks(m2);
            xf = [out_copy, b, lo2, m2, xt](int t) { out_copy(b, lo2, m2, t, xt); };
            pend_lo[b] = -1;
        }
        jobs[b].start(c, h_sched + chunks[size_t(i)].first, chunks[size_t(i)].second,
                      pin + size_t(b) * size_t(cap) * sizeof(etune_schedule), xt, std::move(xf));
        return ETUNE_OK;
    };
    if (etune_status st = begin(0)) return st;
    for (int i = 0; i < nch; ++i) {
        const int64_t lo = chunks[size_t(i)].first, m = chunks[size_t(i)].second;
        const int b = i & 1;
        char* base = io + size_t(b) * size_t(cap) * per;
        void* d_rows = base;
        auto* d_gen = reinterpret_cast<uint64_t*>(base + size_t(cap) * sizeof(etune_schedule));
        auto* d_pred = d_all ? d_all + lo : reinterpret_cast<double*>(base + size_t(cap) * (sizeof(etune_schedule) + 8));
        auto* d_ids = reinterpret_cast<uint64_t*>(base + size_t(cap) * (sizeof(etune_schedule) + 16));
        void* h_rows = pin + size_t(b) * size_t(cap) * sizeof(etune_schedule);
        const bool raw = is_raw(i);
        int fb = 8;
        if (!raw) {
            const auto tw1 = std::chrono::steady_clock::now();
            fb = jobs[b].finish();
            if (e2e_trace)
                e2e_pack_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tw1).count();
        }
        // chunk i-2's outputs still in output staging buffer b (not copied out with a narrowing): now,
        // while the pool is idle
        if (stage_out)
            if (etune_status st = drain(b)) return st;
        if (i + 1 < nch)
            if (etune_status st = begin(i + 1)) return st;
        if (i >= 2) CU(cudaStreamWaitEvent(c->h2d, c->ev_out[b], 0));  // buffer b drained by chunk i-2's D2H
        CU(cudaMemcpyAsync(d_rows, raw ? static_cast<const void*>(h_sched + lo) : h_rows,
                           size_t(m) * 12 * size_t(fb), cudaMemcpyHostToDevice, c->h2d));
        CU(cudaEventRecord(c->ev_in[b], c->h2d));
        CU(cudaStreamWaitEvent(c->stream, c->ev_in[b], 0));
        CU(launch_encode_packed(c->lc(), p->d_blob, p->build.hdr.total, d_rows, fb, m, d_gen, lo));
        if (etune_status st = score_dispatch(c, p, f, r, d_gen, m, d_pred, h_ids ? d_ids : nullptr, sh, nullptr))
            return st;
        CU(cudaEventRecord(c->ev_done[b], c->stream));
        CU(cudaStreamWaitEvent(c->d2h, c->ev_done[b], 0));
        if (stage_out) {
            double* sp = reinterpret_cast<double*>(static_cast<char*>(c->hout) + size_t(b) * size_t(cap) * 16);
            if (h_pred) CU(cudaMemcpyAsync(sp, d_pred, size_t(m) * 8, cudaMemcpyDeviceToHost, c->d2h));
            if (h_ids) CU(cudaMemcpyAsync(sp + cap, d_ids, size_t(m) * 8, cudaMemcpyDeviceToHost, c->d2h));
            pend_lo[b] = lo;
            pend_m[b] = m;
        } else {
            if (h_pred) CU(cudaMemcpyAsync(h_pred + lo, d_pred, size_t(m) * 8, cudaMemcpyDeviceToHost, c->d2h));
            if (h_ids) CU(cudaMemcpyAsync(h_ids + lo, d_ids, size_t(m) * 8, cudaMemcpyDeviceToHost, c->d2h));
        }
        CU(cudaEventRecord(c->ev_out[b], c->d2h));
    }
    if (k > 0) {  // keep the best over the whole population (its predictions are on the device)
        if (sh.hist) {
            CU(launch_select(c->lc(), d_all, n, k, d_idx, c->sel, sh));
            c->sel_dirty = false;
        } else {
            if (etune_status st = ensure_scratch(c, topk_scratch_bytes(n))) return st;
            CU(launch_topk(c->lc(), d_all, n, k, d_idx, c->scratch));
        }
        CU(cudaMemcpyAsync(h_idx, d_idx, size_t(k) * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    if (stage_out)
        for (int b = 0; b < 2; ++b)
            if (etune_status st = drain(b)) return st;
    CU(cudaEventRecord(c->ev_out[0], c->d2h));
    CU(cudaStreamWaitEvent(c->stream, c->ev_out[0], 0));
    const etune_status fin = etune_cu_synchronize(c, first_bad);
    if (e2e_trace)
        std::fprintf(stderr, "e2e n=%lld: total %.0f us, narrowing joins %.0f us, staging waits %.0f us, pool %d threads\n",
                     (long long)n,
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - e2e_t0).count(),
                     e2e_pack_us, e2e_wait_us, c->pool->size());
    return fin;
}

}  // namespace

extern "C" {

etune_status etune_cu_score_host(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f,
                                 const etune_schedule* h_sched, int64_t n, double* h_pred, uint64_t* h_ids,
                                 int64_t* first_bad) {
    CHECK_PLAN_ARGS(h_sched && h_pred);
    if (!f) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null forest");
    return host_pipeline(c, p, f, h_sched, n, h_pred, h_ids, 0, nullptr, first_bad);
}

etune_status etune_cu_score_select_host(etune_cu_ctx* c, const etune_cu_plan* p, etune_cu_forest* f,
                                        const etune_schedule* h_sched, int64_t n, int64_t k, double* h_pred,
                                        int64_t* h_idx, int64_t* first_bad) {
    CHECK_PLAN_ARGS(h_sched);
    if (!f) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null forest");
    if (k < 0 || k > n) return fail(ETUNE_ERR_INVALID_ARGUMENT, "need 0 <= k <= n");
    if (k > 0 && !h_idx) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null index buffer");
    if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "n >= 2^31");
    return host_pipeline(c, p, f, h_sched, n, h_pred, nullptr, k, h_idx, first_bad);
}

etune_status etune_cu_train(etune_cu_ctx* c, const double* d_feat, const double* d_energy, int64_t n,
                            const etune_boost_params* params, int32_t* d_feature, double* d_threshold,
                            int32_t* d_left, int32_t* d_right, double* d_value, int64_t* d_off, double* d_scalars,
                            double* d_loss) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    if (n < 2) return fail(ETUNE_ERR_INSUFFICIENT_DATA, "training needs at least 2 samples, got " + std::to_string(n));
    if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "more than 2^31 samples");
    etune_boost_params bp;
    etune_default_boost_params(&bp);
    if (params) bp = *params;
    if (bp.num_trees < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "num_trees < 0");
    if (bp.max_depth < 0 || bp.max_depth > train_max_depth())
        return fail(ETUNE_ERR_UNSUPPORTED, "max_depth outside [0, " + std::to_string(train_max_depth()) + "]");
    if (!d_feat || !d_energy || !d_feature || !d_threshold || !d_left || !d_right || !d_value || !d_off ||
        !d_scalars)
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "null buffer");
    if (etune_status st = ensure_scratch(c, train_scratch_bytes(n))) return st;
    CU(launch_train(c->lc(), d_feat, d_energy, n, bp.num_trees, bp.max_depth, bp.learning_rate, bp.min_leaf_weight,
                    bp.reg_lambda, d_feature, d_threshold, d_left, d_right, d_value, d_off, d_scalars, d_loss,
                    c->scratch));
    return ETUNE_OK;
}

etune_status etune_cu_energy_loss(etune_cu_ctx* c, const double* d_pred, const double* d_meas, int64_t n,
                                  double* d_out) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    if (n < 0 || (n > 0 && (!d_pred || !d_meas || !d_out))) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad buffers");
    CU(launch_energy_loss(c->lc(), d_pred, d_meas, n, d_out));
    return ETUNE_OK;
}

etune_status etune_cu_snr_db(etune_cu_ctx* c, const double* d_pred, const double* d_meas, int64_t n, double* h_out,
                             int64_t* first_bad) {
    if (!c || !h_out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    if (first_bad) *first_bad = -1;
    if (n == 0) return fail(ETUNE_ERR_EMPTY_INPUT, "snr_db requires non-empty input");
    if (n < 0 || !d_pred || !d_meas) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad buffers");
    if (etune_status st = ensure_scratch(c, 256)) return st;
    double* d2 = static_cast<double*>(c->scratch);
    CU(launch_snr_sums(c->lc(), d_pred, d_meas, n, d2));
    double sums[2] = {0, 0};
    CU(cudaMemcpyAsync(sums, d2, sizeof(sums), cudaMemcpyDeviceToHost, c->stream));
    if (etune_status st = etune_cu_synchronize(c, first_bad)) return st;
    // energy_model.cpp:368-369
    *h_out = sums[1] <= 0.0 ? 100.0 : std::min(100.0, 10.0 * std::log10(sums[0] / sums[1]));
    return ETUNE_OK;
}

etune_status etune_cu_forest_from_device(etune_cu_ctx* c, const int32_t* d_feature, const double* d_threshold,
                                         const int32_t* d_left, const int32_t* d_right, const double* d_value,
                                         const int64_t* d_off, int64_t num_trees, const double* d_scalars,
                                         double learning_rate, etune_cu_forest** out) {
    if (!c || !out || !d_off || !d_scalars || num_trees < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    if (etune_status st = etune_cu_synchronize(c, nullptr)) return st;
    std::vector<int64_t> off(size_t(num_trees) + 1, 0);
    double sc[2] = {0, 0};
    CU(cudaMemcpy(off.data(), d_off, off.size() * 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(sc, d_scalars, sizeof(sc), cudaMemcpyDeviceToHost));
    const int64_t nn = off[size_t(num_trees)];
    if (nn < 0) return fail(ETUNE_ERR_CONSISTENCY, "negative node count");
    const size_t m = static_cast<size_t>(nn);
    std::vector<int32_t> fe(m), le(m), ri(m);
    std::vector<double> th(m), va(m);
    if (nn > 0) {
        CU(cudaMemcpy(fe.data(), d_feature, size_t(nn) * 4, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(le.data(), d_left, size_t(nn) * 4, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(ri.data(), d_right, size_t(nn) * 4, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(th.data(), d_threshold, size_t(nn) * 8, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(va.data(), d_value, size_t(nn) * 8, cudaMemcpyDeviceToHost));
    }
    return etune_cu_forest_create(c, fe.data(), th.data(), le.data(), ri.data(), va.data(), off.data(), num_trees,
                                  sc[0], learning_rate, out);
}

namespace {
// generations of at least this many offspring take the block-parallel exact path.  Diagnostic
// knobs (read per call; tests use them to force every fallback): ETUNE_BREED_PAR_MIN (a huge
// value keeps every call on the single-CTA chain), ETUNE_BREED_PAR_SD (window half-width in
// standard deviations; small values force window misses), ETUNE_BREED_PAR_WORDS (stream
// capacity; small values force the single-CTA fallback).
int64_t breed_par_min() {
    if (const char* e = std::getenv("ETUNE_BREED_PAR_MIN")) return int64_t(std::atoll(e));
    return int64_t(4096);
}
double breed_par_sd() {  // P(|Z| > 4) = 6.3e-5 per block: a 2^20 generation walks ~0.03 blocks exactly
    if (const char* e = std::getenv("ETUNE_BREED_PAR_SD")) return std::atof(e);
    return 4.0;
}
size_t breed_par_words() {
    if (const char* e = std::getenv("ETUNE_BREED_PAR_WORDS")) return size_t(std::atoll(e));
    return 0;
}

etune_status reproduce_impl(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_par, int64_t np, int64_t n,
                            const etune_genetic_rates* rates, uint64_t seed, uint64_t* d_out, int32_t* d_partner,
                            uint64_t* d_ids, bool counter) {
    if (!c || !p) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx/plan");
    if (n < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "negative n");
    if (np < 1 || !d_par) return fail(ETUNE_ERR_VALIDATION, "reproduce requires at least one parent");
    etune_genetic_rates r;
    etune_default_genetic_rates(&r);
    if (rates) r = *rates;
    if (!(r.mutation + r.crossover + r.copy > 0.0))
        return fail(ETUNE_ERR_VALIDATION, "genetic rates must not all be zero");
    if (n == 0) return ETUNE_OK;
    if (!d_out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null offspring buffer");
    if (np >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "more than 2^31 parents");
    const size_t need = 256 + size_t(np) * 8;
    if (c->breed_bytes < need) {
        if (c->breed) {
            CU(cudaStreamSynchronize(c->stream));
            CU(cudaFree(c->breed));
            c->breed = nullptr;
            c->breed_bytes = 0;
        }
        CU(cudaMalloc(&c->breed, need));
        c->breed_bytes = need;
    }
    uint64_t* d_pid = reinterpret_cast<uint64_t*>(static_cast<char*>(c->breed) + 256);
    CU(launch_ids(c->lc(), p->d_blob, p->build.hdr.total, d_par, np, d_pid));
    if (counter)
        CU(launch_breed_counter(c->lc(), p->d_blob, p->build.hdr.total, d_par, d_pid, np, n, r.mutation, r.crossover,
                                r.copy, seed, d_out, d_partner));
    else {
        // exact mode: the block-parallel path for large generations (the single-CTA chain
        // kernel after it exits at once unless the parallel path could not hold the generation)
        const int32_t* d_done = nullptr;
        if (n >= breed_par_min()) {
            const int S = breed_par_block(n);
            size_t words = 0, pool = 0;
            const size_t pneed = breed_par_bytes(n, S, &words, &pool);
            if (c->breedpar_bytes < pneed) {
                if (c->breedpar) {
                    CU(cudaStreamSynchronize(c->stream));
                    CU(cudaFree(c->breedpar));
                    c->breedpar = nullptr;
                    c->breedpar_bytes = 0;
                }
                CU(cudaMalloc(&c->breedpar, pneed));
                c->breedpar_bytes = pneed;
            }
            int32_t* done = nullptr;
            CU(launch_breed_par(c->lc(), p->d_blob, p->build.hdr.total, d_par, d_pid, np, n, r.mutation, r.crossover,
                                r.copy, seed, d_out, d_partner, c->breedpar, S, breed_par_sd(), breed_par_words(),
                                (std::getenv("ETUNE_BREED_PAR_SPLITGEN") ? 1 : 0) | (std::getenv("ETUNE_BREED_PAR_PROF") ? 2 : 0) |
                                    (std::getenv("ETUNE_BREED_PAR_CHECK") ? 4 : 0), p->build.hdr.off_gridkey, &done));
            d_done = done;
        }
        CU(launch_breed(c->lc(), p->d_blob, p->build.hdr.total, d_par, d_pid, np, n, r.mutation, r.crossover, r.copy,
                        seed, d_out, d_partner, c->breed, d_done));
    }
    if (d_ids) CU(launch_ids(c->lc(), p->d_blob, p->build.hdr.total, d_out, n, d_ids));
    return ETUNE_OK;
}

}  // namespace

etune_status etune_cu_reproduce(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_par, int64_t np,
                                int64_t n, const etune_genetic_rates* rates, uint64_t seed, uint64_t* d_out,
                                int32_t* d_partner, uint64_t* d_ids) {
    return reproduce_impl(c, p, d_par, np, n, rates, seed, d_out, d_partner, d_ids, false);
}

etune_status etune_cu_reproduce_counter(etune_cu_ctx* c, const etune_cu_plan* p, const uint64_t* d_par, int64_t np,
                                        int64_t n, const etune_genetic_rates* rates, uint64_t seed, uint64_t* d_out,
                                        int32_t* d_partner, uint64_t* d_ids) {
    return reproduce_impl(c, p, d_par, np, n, rates, seed, d_out, d_partner, d_ids, true);
}

etune_status etune_cu_topk(etune_cu_ctx* c, const double* d_score, int64_t n, int64_t k, int64_t* d_idx) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    if (n < 0 || k < 0 || k > n) return fail(ETUNE_ERR_INVALID_ARGUMENT, "need 0 <= k <= n");
    if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "n >= 2^31");
    if (k == 0) return ETUNE_OK;
    if (!d_score || !d_idx) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null buffer");
    if (etune_status st = ensure_scratch(c, topk_scratch_bytes(n))) return st;
    CU(launch_topk(c->lc(), d_score, n, k, d_idx, c->scratch));
    return ETUNE_OK;
}

etune_status etune_cu_nccl_unique_id(void* out_id) {
    if (!out_id) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null id");
    static_assert(sizeof(ncclUniqueId) == ETUNE_NCCL_UNIQUE_ID_BYTES, "NCCL id size");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(ETUNE_ERR_CUDA, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out_id, &id, sizeof(id));
    return ETUNE_OK;
}

etune_status etune_cu_ctx_attach_nccl(etune_cu_ctx* c, const void* unique_id, int nranks, int rank) {
    if (!c || !unique_id || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad communicator arguments");
    CU(cudaSetDevice(c->device));
    if (c->comm) {
        ncclCommDestroy(c->comm);
        c->comm = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    const ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        return fail(ETUNE_ERR_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    c->nranks = nranks;
    c->rank = rank;
    return ETUNE_OK;
}

etune_status etune_cu_topk_sharded(etune_cu_ctx* c, const double* d_score, int64_t n, int64_t goff, int64_t k,
                                   int64_t* d_idx, double* d_sc) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    if (n < 0 || k < 0 || goff < 0) return fail(ETUNE_ERR_INVALID_ARGUMENT, "negative size");
    if (k == 0) return ETUNE_OK;
    if (!d_idx || (n > 0 && !d_score)) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null buffer");
    ShardBufs sb;
    if (etune_status st = shard_buffers(c, k, &sb)) return st;
    const int64_t kl = std::min(k, n);
    if (kl > 0) {
        if (n >= (int64_t(1) << 31)) return fail(ETUNE_ERR_UNSUPPORTED, "shard >= 2^31");
        if (etune_status st = ensure_scratch(c, topk_scratch_bytes(n))) return st;
        CU(launch_topk(c->lc(), d_score, n, kl, sb.lidx, c->scratch));
    }
    return shard_merge(c, d_score, kl, k, goff, sb, d_idx, d_sc);
}

etune_status etune_cu_broadcast(etune_cu_ctx* c, void* d_buf, int64_t bytes, int root) {
    if (!c || bytes < 0 || (bytes > 0 && !d_buf)) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad arguments");
    if (root < 0 || root >= ctx_world(c)) return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad root");
    return coll_broadcast(c, d_buf, size_t(bytes), root);
}

etune_status etune_cu_ctx_attach_transport(etune_cu_ctx* c, const etune_transport* t) {
    if (!c) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null ctx");
    if (!t) {
        c->has_transport = false;
        return ETUNE_OK;
    }
    if (t->nranks < 1 || t->rank < 0 || t->rank >= t->nranks || !t->allgather || !t->broadcast)
        return fail(ETUNE_ERR_INVALID_ARGUMENT, "bad transport");
    if (c->comm) return fail(ETUNE_ERR_INVALID_ARGUMENT, "an NCCL communicator is already attached");
    c->transport = *t;
    c->has_transport = true;
    return ETUNE_OK;
}

}  // extern "C"

extern "C" etune_status etune_cu_forest_compile_stats(etune_cu_forest* f, const etune_cu_plan* p, int64_t out[8]) {
    if (!f || !p || !out) return fail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    CompiledScore* cs = nullptr;
    if (etune_status st = get_compiled(f, p, &cs)) return st;
    out[0] = cs->stats.internal_nodes_in;
    out[1] = cs->stats.tests_folded;
    out[2] = cs->stats.lut_entries;
    out[3] = cs->stats.max_leaves;
    out[4] = cs->stats.total_leaves;
    out[5] = cs->bytes;
    out[6] = cs->stats.channels_used;
    out[7] = f->host.num_trees();
    return ETUNE_OK;
}
