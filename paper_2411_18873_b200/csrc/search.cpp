// Algorithm 1: the energy-aware genetic search loop.
// The reference has no code for it, so this is the repo's restatement; the CPU oracle
// (oracle/etune_oracle.cpp, orc_run_search) runs the same loop step for step and the
// GPU tests compare their round reports bit for bit.
//
// Host C++ orchestrates; every population-sized step is a kernel of this library,
// called through its own C ABI:
//   round r:  reproduce -> SimBackend latency -> top-M -> score with the model ->
//             top-ceil(k M) -> SimBackend energy -> SNR -> append samples -> retrain ->
//             parents = top-ceil(M/2) by prediction.
// Only the per-round scalars (k, SNR, the measured records for the best-so-far) cross
// to the host.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>
#include <vector>

#include "handles.hpp"

using namespace etune_b200;

struct etune_cu_search {
    etune_cu_ctx* ctx = nullptr;
    const etune_cu_plan* plan = nullptr;
    etune_search_config cfg{};
    int k5 = 5;
    int64_t round = -1;  // -1: initial round not run yet
    int64_t cumulative = 0;
    int stall = 0;
    // best measured (energy, latency, id)
    bool have_best = false;
    uint64_t best_id = 0, best_genome = 0;
    double best_lat = 0, best_en = 0, best_pow = 0;
    // device buffers
    uint64_t *pop = nullptr, *mgen = nullptr, *selgen = nullptr, *par = nullptr, *ids = nullptr;
    double *lat = nullptr, *mpred = nullptr, *psel = nullptr, *mlat = nullptr, *mpow = nullptr, *men = nullptr,
           *mnorm = nullptr, *psel_scratch = nullptr;
    int64_t *idx = nullptr, *sel = nullptr;
    int64_t np = 0;
    // training samples (grow by doubling)
    double *feat = nullptr, *energy = nullptr;
    int64_t nsamples = 0, cap = 0;
    // model arrays
    int32_t *m_feature = nullptr, *m_left = nullptr, *m_right = nullptr;
    double *m_thr = nullptr, *m_value = nullptr, *m_sc = nullptr;
    int64_t* m_off = nullptr;
    etune_cu_forest* model = nullptr;
    std::vector<void*> allocs;
    // the next round's reproduce, launched on a side stream as soon as its parents exist
    // so that it runs beside this round's retrain (one CTA: the rest of the GPU trains)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_par = nullptr, ev_pop = nullptr;
    int64_t pop_round = -1;  // round whose generation is in flight / in `pop`
    // ReplayBackend (backend 2): the log's records by candidate id, most recent winning
    std::unordered_map<uint64_t, etune_measurement> replay;
    bool replay_set = false;
    uint64_t* gids = nullptr;  // generation-sized id buffer for replay lookups
};

namespace {

etune_status sfail(etune_status st, const std::string& msg) {
    set_error(msg);
    return st;
}

#define SCU(expr)                                                                                   \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess) return sfail(ETUNE_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)
#define SOK(expr)                            \
    do {                                     \
        etune_status _s = (expr);            \
        if (_s != ETUNE_OK) return _s;       \
    } while (0)

template <typename T>
etune_status dalloc(etune_cu_search* s, T** p, int64_t n) {
    void* v = nullptr;
    SCU(cudaMalloc(&v, size_t(std::max<int64_t>(n, 1)) * sizeof(T)));
    s->allocs.push_back(v);
    *p = static_cast<T*>(v);
    return ETUNE_OK;
}

// reproduce(parents, G, seed + r) for round r on the side stream, ordered after the
// parents on the ctx stream; round r waits for ev_pop before it reads `pop`
etune_status prelaunch_reproduce(etune_cu_search* s, int64_t r) {
    etune_cu_ctx* c = s->ctx;
    if (!s->side) {
        int least = 0, greatest = 0;  // the single breed CTA is dispatched ahead of the training grids
        SCU(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        SCU(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, greatest));
        SCU(cudaEventCreateWithFlags(&s->ev_par, cudaEventDisableTiming));
        SCU(cudaEventCreateWithFlags(&s->ev_pop, cudaEventDisableTiming));
    }
    SCU(cudaEventRecord(s->ev_par, c->stream));
    SCU(cudaStreamWaitEvent(s->side, s->ev_par, 0));
    const cudaStream_t main_stream = c->stream;
    c->stream = s->side;  // the ctx's launches go to the side stream for this call only
    const etune_status st =
        (s->cfg.counter_rng ? etune_cu_reproduce_counter : etune_cu_reproduce)(
            c, s->plan, s->par, s->np, s->cfg.generation_size, &s->cfg.rates, s->cfg.rng_seed + uint64_t(r), s->pop,
            nullptr, nullptr);
    c->stream = main_stream;
    SOK(st);
    SCU(cudaEventRecord(s->ev_pop, s->side));
    s->pop_round = r;
    return ETUNE_OK;
}

int64_t ceil_fifths(int k5, int64_t M) {  // ceil(k * M) with k = k5 / 5, minimum 1
    const int64_t v = (int64_t(k5) * M + 4) / 5;
    return v < 1 ? 1 : v;
}

// append n measured candidates (features of `gen`, energies) to the training set
etune_status append_samples(etune_cu_search* s, const uint64_t* gen, const double* en, int64_t n) {
    etune_cu_ctx* c = s->ctx;
    if (s->nsamples + n > s->cap) {
        int64_t nc = std::max<int64_t>(s->cap * 2, s->nsamples + n);
        double *f2 = nullptr, *e2 = nullptr;
        // stream-ordered: no device-wide synchronisation (the next round's reproduce may
        // be running on the side stream)
        SCU(cudaMallocAsync(&f2, size_t(nc) * 16 * 8, c->stream));
        SCU(cudaMallocAsync(&e2, size_t(nc) * 8, c->stream));
        if (s->nsamples) {
            SCU(cudaMemcpyAsync(f2, s->feat, size_t(s->nsamples) * 16 * 8, cudaMemcpyDeviceToDevice, c->stream));
            SCU(cudaMemcpyAsync(e2, s->energy, size_t(s->nsamples) * 8, cudaMemcpyDeviceToDevice, c->stream));
        }
        if (s->feat) SCU(cudaFreeAsync(s->feat, c->stream));
        if (s->energy) SCU(cudaFreeAsync(s->energy, c->stream));
        s->feat = f2;
        s->energy = e2;
        s->cap = nc;
    }
    SOK(etune_cu_features(c, s->plan, gen, n, s->feat + s->nsamples * 16, nullptr));
    SCU(cudaMemcpyAsync(s->energy + s->nsamples, en, size_t(n) * 8, cudaMemcpyDeviceToDevice, c->stream));
    s->nsamples += n;
    return ETUNE_OK;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

etune_status retrain(etune_cu_search* s) {
    etune_cu_ctx* c = s->ctx;
    static const bool trace = std::getenv("ETUNE_SEARCH_TRACE") != nullptr;
    const double t0 = trace ? now_ms() : 0.0;
    // population-sharded search: rank 0 trains, the model arrays are broadcast (north_star: NCCL
    // carries only the per-shard top-k records and the model); a single rank just trains
    const int W = ctx_world(c);
    if (W == 1 || ctx_rank(c) == 0)
        SOK(etune_cu_train(c, s->feat, s->energy, s->nsamples, &s->cfg.boost, s->m_feature, s->m_thr, s->m_left,
                           s->m_right, s->m_value, s->m_off, s->m_sc, nullptr));
    if (W > 1) {
        const size_t nodes = size_t(s->cfg.boost.num_trees) * ((size_t(1) << (s->cfg.boost.max_depth + 1)) - 1);
        SOK(coll_broadcast(c, s->m_feature, nodes * 4, 0));
        SOK(coll_broadcast(c, s->m_left, nodes * 4, 0));
        SOK(coll_broadcast(c, s->m_right, nodes * 4, 0));
        SOK(coll_broadcast(c, s->m_thr, nodes * 8, 0));
        SOK(coll_broadcast(c, s->m_value, nodes * 8, 0));
        SOK(coll_broadcast(c, s->m_off, size_t(s->cfg.boost.num_trees + 1) * 8, 0));
        SOK(coll_broadcast(c, s->m_sc, 16, 0));
    }
    if (trace) {
        const double t1 = now_ms();
        cudaStreamSynchronize(c->stream);
        std::fprintf(stderr, "  train: issue %.3f ms, device %.3f ms\n", t1 - t0, now_ms() - t1);
    }
    etune_cu_forest* f = nullptr;
    SOK(etune_cu_forest_from_device(c, s->m_feature, s->m_thr, s->m_left, s->m_right, s->m_value, s->m_off,
                                    s->cfg.boost.num_trees, s->m_sc, s->cfg.boost.learning_rate, &f));
    f->lazy_compile = true;  // scored once per round (M candidates): walk instead of compiling
    if (s->model) etune_cu_forest_destroy(s->model);
    s->model = f;
    return ETUNE_OK;
}

etune_status measure_energy(etune_cu_search* s, const uint64_t* gen, int64_t n);

// run_latency_only: best-so-far = lowest latency (then id) among the rounds' fastest
// candidates; the fastest of this round (gen[0], the latency-sorted M) has its energy
// measured for the report.  improved = best latency dropped by more than improve_rel.
etune_status update_best_latency(etune_cu_search* s, const uint64_t* gen, bool* improved) {
    etune_cu_ctx* c = s->ctx;
    SOK(measure_energy(s, gen, 1));
    SOK(etune_cu_candidate_ids(c, s->plan, gen, 1, s->ids));
    uint64_t id = 0, g = 0;
    double l = 0, p = 0, e = 0;
    SCU(cudaMemcpyAsync(&id, s->ids, 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(&g, gen, 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(&l, s->mlat, 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(&p, s->mpow, 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(&e, s->men, 8, cudaMemcpyDeviceToHost, c->stream));
    SOK(etune_cu_synchronize(c, nullptr));
    const double before = s->have_best ? s->best_lat : std::numeric_limits<double>::infinity();
    if (!s->have_best || l < s->best_lat || (l == s->best_lat && id < s->best_id)) {
        s->have_best = true;
        s->best_lat = l;
        s->best_en = e;
        s->best_pow = p;
        s->best_id = id;
        s->best_genome = g;
    }
    *improved = s->best_lat < before * (1.0 - s->cfg.improve_rel);
    return ETUNE_OK;
}

// best-so-far over the n measured records of this round
etune_status update_best(etune_cu_search* s, const uint64_t* gen, int64_t n, bool* improved) {
    etune_cu_ctx* c = s->ctx;
    SOK(etune_cu_candidate_ids(c, s->plan, gen, n, s->ids));
    const size_t m = static_cast<size_t>(n);
    std::vector<uint64_t> ids(m), g(m);
    std::vector<double> lat(m), en(m), pw(m);
    SCU(cudaMemcpyAsync(ids.data(), s->ids, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(g.data(), gen, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(lat.data(), s->mlat, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(en.data(), s->men, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    SCU(cudaMemcpyAsync(pw.data(), s->mpow, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    SOK(etune_cu_synchronize(c, nullptr));
    const double before = s->have_best ? s->best_en : std::numeric_limits<double>::infinity();
    for (int64_t i = 0; i < n; ++i) {
        const bool better = !s->have_best || en[i] < s->best_en ||
                            (en[i] == s->best_en && (lat[i] < s->best_lat ||
                                                     (lat[i] == s->best_lat && ids[i] < s->best_id)));
        if (better) {
            s->have_best = true;
            s->best_en = en[i];
            s->best_lat = lat[i];
            s->best_id = ids[i];
            s->best_pow = pw[i];
            s->best_genome = g[i];
        }
    }
    // "improvement > 0.1 %" of the best measured energy
    *improved = s->best_en < before * (1.0 - s->cfg.improve_rel);
    return ETUNE_OK;
}

void fill_report(const etune_cu_search* s, int kb, double snr, int64_t measured, double ms, etune_round_report* r) {
    if (!r) return;
    r->round = s->round;
    r->k_before_fifths = kb;
    r->k_after_fifths = s->k5;
    r->snr_db = snr;
    r->measured = measured;
    r->cumulative_measured = s->cumulative;
    r->best_id = s->best_id;
    r->best_latency_ms = s->best_lat;
    r->best_energy_mj = s->best_en;
    r->best_power_w = s->best_pow;
    r->wall_ms = ms;
}

// host copies of device genomes as the reference's Schedule records
etune_status host_schedules(etune_cu_search* s, const uint64_t* gen, int64_t n, std::vector<etune_schedule>* out) {
    etune_cu_ctx* c = s->ctx;
    etune_schedule* d = nullptr;
    SCU(cudaMalloc(&d, size_t(std::max<int64_t>(n, 1)) * sizeof(etune_schedule)));
    etune_status st = etune_cu_decode(c, s->plan, gen, n, d);
    out->resize(static_cast<size_t>(n));
    if (st == ETUNE_OK && n > 0) {
        const cudaError_t e =
            cudaMemcpyAsync(out->data(), d, size_t(n) * sizeof(etune_schedule), cudaMemcpyDeviceToHost, c->stream);
        if (e != cudaSuccess) st = sfail(ETUNE_ERR_CUDA, cudaGetErrorString(e));
    }
    if (st == ETUNE_OK) st = etune_cu_synchronize(c, nullptr);
    cudaFree(d);
    return st;
}

// LatencyEvaAndPick's measurement: the backend's latency of n device genomes into d_lat
// ReplayBackend (measure.hpp:116-128): the logged records of n device genomes, by id;
// TraceMiss names the first id the log lacks
etune_status replay_lookup(etune_cu_search* s, const uint64_t* gen, int64_t n, std::vector<etune_measurement>* rec) {
    if (!s->gids) SOK(dalloc(s, &s->gids, s->cfg.generation_size));
    SOK(etune_cu_candidate_ids(s->ctx, s->plan, gen, n, s->gids));
    std::vector<uint64_t> ids(static_cast<size_t>(n));
    SCU(cudaMemcpyAsync(ids.data(), s->gids, size_t(n) * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
    SOK(etune_cu_synchronize(s->ctx, nullptr));
    rec->resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const auto it = s->replay.find(ids[size_t(i)]);
        if (it == s->replay.end())
            return sfail(ETUNE_ERR_TRACE_MISS, "candidate id " + std::to_string(ids[size_t(i)]) +
                                                   " is not in the replay log");
        (*rec)[size_t(i)] = it->second;
        (*rec)[size_t(i)].feasible = 1;  // a logged record is a completed measurement
    }
    return ETUNE_OK;
}

etune_status measure_latency(etune_cu_search* s, const uint64_t* gen, int64_t n, double* d_lat);

// LatencyEvaAndPick(gen, M) -> the M fastest by (latency, index) into s->idx.  Sharded: every rank
// holds the whole generation (reproduce is replicated: one RNG stream), measures the latencies of
// its contiguous slice only, keeps its slice's M fastest and the all-gathered per-rank lists are
// merged into the identical global M on every rank (etune_cu_topk_sharded).
etune_status latency_pick(etune_cu_search* s, const uint64_t* gen, int64_t n, int64_t M) {
    etune_cu_ctx* c = s->ctx;
    const int W = ctx_world(c), R = ctx_rank(c);
    if (W == 1) {
        SOK(measure_latency(s, gen, n, s->lat));
        return etune_cu_topk(c, s->lat, n, M, s->idx);
    }
    const int64_t lo = n * R / W, hi = n * (R + 1) / W;
    SOK(measure_latency(s, gen + lo, hi - lo, s->lat + lo));
    return etune_cu_topk_sharded(c, s->lat + lo, hi - lo, lo, M, s->idx, s->psel_scratch);
}

etune_status measure_latency(etune_cu_search* s, const uint64_t* gen, int64_t n, double* d_lat) {
    if (s->cfg.backend == 0) return etune_cu_sim_measure(s->ctx, s->plan, gen, n, d_lat, nullptr, nullptr, nullptr);
    if (s->cfg.backend == 2) {
        std::vector<etune_measurement> rec;
        SOK(replay_lookup(s, gen, n, &rec));
        std::vector<double> lat(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) lat[size_t(i)] = rec[size_t(i)].latency_ms;
        SCU(cudaMemcpyAsync(d_lat, lat.data(), size_t(n) * 8, cudaMemcpyHostToDevice, s->ctx->stream));
        return etune_cu_synchronize(s->ctx, nullptr);
    }
    std::vector<etune_schedule> h;
    SOK(host_schedules(s, gen, n, &h));
    std::vector<double> lat(static_cast<size_t>(n));
    SOK(etune_cu_candidate_latency(s->ctx, s->plan, h.data(), n, s->cfg.latency_reps, lat.data()));
    SCU(cudaMemcpyAsync(d_lat, lat.data(), size_t(n) * 8, cudaMemcpyHostToDevice, s->ctx->stream));
    return etune_cu_synchronize(s->ctx, nullptr);
}

// NVMLMeasurement: latency, power and energy of n device genomes into mlat/mpow/men.
// A selected schedule the candidate kernel cannot run gets a finite penalty energy
// (1e30 mJ) so that training stays finite; it is never the best.
etune_status measure_energy_local(etune_cu_search* s, const uint64_t* gen, int64_t n, double* lat, double* pw,
                                  double* en);

// Sharded: rank r measures the slice [n r / W, n (r+1) / W) (on the GPU backend, every GPU runs
// its own candidates at once), the three arrays are all-gathered in slices padded to ceil(n / W).
etune_status measure_energy(etune_cu_search* s, const uint64_t* gen, int64_t n) {
    etune_cu_ctx* c = s->ctx;
    const int W = ctx_world(c), R = ctx_rank(c);
    if (W == 1) return measure_energy_local(s, gen, n, s->mlat, s->mpow, s->men);
    const int64_t per = (n + W - 1) / W;
    const int64_t lo = n * R / W, hi = n * (R + 1) / W;
    double* st = nullptr;  // [3][per] local, then [W][3][per] gathered
    SCU(cudaMallocAsync(reinterpret_cast<void**>(&st), size_t(per) * 3 * 8 * size_t(1 + W), c->stream));
    double* g = st + 3 * per;
    etune_status rs = measure_energy_local(s, gen + lo, hi - lo, st, st + per, st + 2 * per);
    if (rs == ETUNE_OK) rs = coll_allgather(c, st, g, size_t(per) * 3 * 8);
    for (int w = 0; w < W && rs == ETUNE_OK; ++w) {
        const int64_t a = n * w / W, m = n * (w + 1) / W - a;
        double* dst[3] = {s->mlat, s->mpow, s->men};
        for (int q = 0; q < 3 && m > 0; ++q) {
            const cudaError_t e = cudaMemcpyAsync(dst[q] + a, g + (int64_t(w) * 3 + q) * per, size_t(m) * 8,
                                                  cudaMemcpyDeviceToDevice, c->stream);
            if (e != cudaSuccess) rs = sfail(ETUNE_ERR_CUDA, cudaGetErrorString(e));
        }
    }
    cudaFreeAsync(st, c->stream);
    return rs;
}

etune_status measure_energy_local(etune_cu_search* s, const uint64_t* gen, int64_t n, double* mlat, double* mpow,
                                  double* men) {
    if (n <= 0) return ETUNE_OK;
    if (s->cfg.backend == 0)
        return etune_cu_sim_measure(s->ctx, s->plan, gen, n, mlat, mpow, men, nullptr);
    std::vector<etune_measurement> rec(static_cast<size_t>(n));
    if (s->cfg.backend == 2) {
        SOK(replay_lookup(s, gen, n, &rec));
    } else {
        std::vector<etune_schedule> h;
        SOK(host_schedules(s, gen, n, &h));
        SOK(etune_cu_nvml_measure(s->ctx, s->plan, h.data(), n, &s->cfg.nvml, rec.data(), nullptr));
    }
    std::vector<double> lat(static_cast<size_t>(n)), pw(static_cast<size_t>(n)), en(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const etune_measurement& r = rec[size_t(i)];
        lat[size_t(i)] = r.feasible ? r.latency_ms : 1e30;
        pw[size_t(i)] = r.feasible ? r.avg_power_w : 0.0;
        en[size_t(i)] = r.feasible ? r.energy_mj : 1e30;
    }
    cudaStream_t st = s->ctx->stream;
    SCU(cudaMemcpyAsync(mlat, lat.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
    SCU(cudaMemcpyAsync(mpow, pw.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
    SCU(cudaMemcpyAsync(men, en.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
    return etune_cu_synchronize(s->ctx, nullptr);
}


}  // namespace

extern "C" {

void etune_default_search_config(etune_search_config* o) {
    std::memset(o, 0, sizeof(*o));
    o->M = 512;
    o->generation_size = 2048;
    o->k_init_fifths = 5;
    o->max_rounds = 10;
    o->patience = 5;
    o->inverted_semantics = 0;
    o->mu_db = 20.0;
    o->improve_rel = 0.001;
    o->rng_seed = 42;
    etune_default_genetic_rates(&o->rates);
    etune_default_boost_params(&o->boost);
    o->backend = 0;
    o->latency_reps = 3;
    etune_default_nvml_params(&o->nvml);
}

etune_status etune_cu_search_create(etune_cu_ctx* c, const etune_cu_plan* p, const etune_search_config* cfg,
                                    etune_cu_search** out) {
    if (!c || !p || !out) return sfail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    etune_search_config C;
    etune_default_search_config(&C);
    if (cfg) C = *cfg;
    if (!(C.M > 0 && C.M <= C.generation_size))
        return sfail(ETUNE_ERR_VALIDATION, "SearchConfig needs 0 < M <= generation_size");
    if (C.k_init_fifths < 0 || C.k_init_fifths > 5) return sfail(ETUNE_ERR_VALIDATION, "k must lie in [0, 1]");
    if (!std::isfinite(C.mu_db)) return sfail(ETUNE_ERR_VALIDATION, "mu_db must be finite");
    if (C.backend < 0 || C.backend > 2)
        return sfail(ETUNE_ERR_VALIDATION, "backend must be 0 (sim), 1 (gpu) or 2 (replay)");
    if (C.backend == 1) {
        std::string why;
        if (!nvml_device_handle(c->device, &why))
            return sfail(ETUNE_ERR_BACKEND_UNAVAILABLE, "NVML energy counters unavailable: " + why);
    }
    if (C.boost.max_depth < 0 || C.boost.max_depth > train_max_depth() || C.boost.num_trees < 0)
        return sfail(ETUNE_ERR_UNSUPPORTED, "boost parameters outside this build's range");
    auto s = std::make_unique<etune_cu_search>();
    s->ctx = c;
    s->plan = p;
    s->cfg = C;
    s->k5 = C.k_init_fifths;
    const int64_t G = C.generation_size, M = C.M;
    SOK(dalloc(s.get(), &s->pop, G));
    SOK(dalloc(s.get(), &s->lat, G));
    SOK(dalloc(s.get(), &s->idx, M));
    SOK(dalloc(s.get(), &s->mgen, M));
    SOK(dalloc(s.get(), &s->mpred, M));
    SOK(dalloc(s.get(), &s->sel, M));
    SOK(dalloc(s.get(), &s->selgen, M));
    SOK(dalloc(s.get(), &s->psel, M));
    SOK(dalloc(s.get(), &s->psel_scratch, M));  // scores of the merged sharded latency pick
    SOK(dalloc(s.get(), &s->mlat, M));
    SOK(dalloc(s.get(), &s->mpow, M));
    SOK(dalloc(s.get(), &s->men, M));
    SOK(dalloc(s.get(), &s->mnorm, M));
    SOK(dalloc(s.get(), &s->par, M));
    SOK(dalloc(s.get(), &s->ids, M));
    const int64_t nodes = int64_t(C.boost.num_trees) * ((int64_t(1) << (C.boost.max_depth + 1)) - 1);
    SOK(dalloc(s.get(), &s->m_feature, nodes));
    SOK(dalloc(s.get(), &s->m_left, nodes));
    SOK(dalloc(s.get(), &s->m_right, nodes));
    SOK(dalloc(s.get(), &s->m_thr, nodes));
    SOK(dalloc(s.get(), &s->m_value, nodes));
    SOK(dalloc(s.get(), &s->m_off, C.boost.num_trees + 1));
    SOK(dalloc(s.get(), &s->m_sc, 2));
    ctx_retain(c);
    *out = s.release();
    return ETUNE_OK;
}

etune_status etune_cu_search_destroy(etune_cu_search* s) {
    if (!s) return ETUNE_OK;
    cudaStreamSynchronize(s->ctx->stream);
    if (s->side) {
        cudaStreamSynchronize(s->side);
        cudaStreamDestroy(s->side);
        cudaEventDestroy(s->ev_par);
        cudaEventDestroy(s->ev_pop);
    }
    if (s->model) etune_cu_forest_destroy(s->model);
    for (void* p : s->allocs) cudaFree(p);
    cudaFree(s->feat);
    cudaFree(s->energy);
    etune_cu_ctx* c = s->ctx;
    delete s;
    ctx_release(c);
    return ETUNE_OK;
}

etune_status etune_cu_search_set_replay(etune_cu_search* s, const etune_measurement* records, int64_t n) {
    if (!s || n < 0 || (n > 0 && !records)) return sfail(ETUNE_ERR_INVALID_ARGUMENT, "bad replay records");
    s->replay.clear();
    s->replay.reserve(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) s->replay[records[i].candidate_id] = records[i];  // later lines win
    s->replay_set = true;
    return ETUNE_OK;
}

// initial_round: sample, latency-filter to M, measure all M, first model.
etune_status etune_cu_search_initial(etune_cu_search* s, etune_round_report* rep) {
    if (!s) return sfail(ETUNE_ERR_INVALID_ARGUMENT, "null search");
    if (s->cfg.backend == 2 && !s->replay_set)
        return sfail(ETUNE_ERR_BACKEND_UNAVAILABLE, "replay backend without a log (etune_cu_search_set_replay)");
    etune_cu_ctx* c = s->ctx;
    const double t0 = now_ms();
    const int64_t G = s->cfg.generation_size, M = s->cfg.M;
    SOK(etune_cu_sample_random(c, s->plan, G, s->cfg.rng_seed, s->pop, nullptr));
    SOK(latency_pick(s, s->pop, G, M));  // LatencyEvaAndPick(Kernel_generation, M)
    SCU(launch_gather_u64(c->lc(), s->pop, s->idx, M, s->mgen));
    if (s->cfg.latency_only) {  // run_latency_only: no energy model at all
        SCU(cudaMemcpyAsync(s->par, s->mgen, size_t(M) * 8, cudaMemcpyDeviceToDevice, c->stream));
        s->np = M;
        s->round = 0;
        s->cumulative = 1;
        bool improved = false;
        SOK(update_best_latency(s, s->mgen, &improved));
        fill_report(s, s->k5, std::numeric_limits<double>::quiet_NaN(), 1, now_ms() - t0, rep);
        return ETUNE_OK;
    }
    SOK(measure_energy(s, s->mgen, M));
    SCU(cudaMemcpyAsync(s->par, s->mgen, size_t(M) * 8, cudaMemcpyDeviceToDevice, c->stream));
    s->np = M;
    if (s->cfg.max_rounds >= 1) SOK(prelaunch_reproduce(s, 1));
    SOK(append_samples(s, s->mgen, s->men, M));
    SOK(retrain(s));
    s->round = 0;
    s->cumulative = M;
    bool improved = false;
    SOK(update_best(s, s->mgen, M, &improved));
    fill_report(s, s->k5, std::numeric_limits<double>::quiet_NaN(), M, now_ms() - t0, rep);
    return ETUNE_OK;
}

// round
etune_status etune_cu_search_round(etune_cu_search* s, etune_round_report* rep) {
    if (!s) return sfail(ETUNE_ERR_INVALID_ARGUMENT, "null search");
    if (s->round < 0) return sfail(ETUNE_ERR_VALIDATION, "initial round has not run");
    etune_cu_ctx* c = s->ctx;
    const double t0 = now_ms();
    const int64_t G = s->cfg.generation_size, M = s->cfg.M;
    const int64_t r = s->round + 1;
    // ETUNE_SEARCH_TRACE=1 (diagnostic): synchronise after every stage and print its time
    static const bool trace = std::getenv("ETUNE_SEARCH_TRACE") != nullptr;
    double tl = t0;
    auto stage = [&](const char* name) {
        if (!trace) return;
        cudaStreamSynchronize(c->stream);
        const double t = now_ms();
        std::fprintf(stderr, "round %lld %-10s %9.3f ms (samples %lld)\n", static_cast<long long>(r), name, t - tl,
                     static_cast<long long>(s->nsamples));
        tl = t;
    };
    // 1. GeneticReproduction(Kernel_parents): usually already running beside the previous
    // retrain (prelaunch_reproduce)
    if (s->pop_round == r) {
        SCU(cudaStreamWaitEvent(c->stream, s->ev_pop, 0));
    } else {
        SOK((s->cfg.counter_rng ? etune_cu_reproduce_counter : etune_cu_reproduce)(
            c, s->plan, s->par, s->np, G, &s->cfg.rates, s->cfg.rng_seed + uint64_t(r), s->pop, nullptr, nullptr));
    }
    stage("reproduce");
    // 2. LatencyEvaAndPick(Kernel_generation, M)
    SOK(latency_pick(s, s->pop, G, M));
    SCU(launch_gather_u64(c->lc(), s->pop, s->idx, M, s->mgen));
    stage("latency");
    if (s->cfg.latency_only) {  // steps 3-8 replaced by parent selection on latency
        const int64_t np = (M + 1) / 2;  // the ceil(M/2) fastest (mgen is latency-sorted)
        SCU(cudaMemcpyAsync(s->par, s->mgen, size_t(np) * 8, cudaMemcpyDeviceToDevice, c->stream));
        s->np = np;
        s->round = r;
        s->cumulative += 1;
        bool improved = false;
        SOK(update_best_latency(s, s->mgen, &improved));
        s->stall = improved ? 0 : s->stall + 1;
        fill_report(s, s->k5, std::numeric_limits<double>::quiet_NaN(), 1, now_ms() - t0, rep);
        return ETUNE_OK;
    }
    // 3. EnergyModelEvaAndPick(Kernel_M, EnergyModel, k*M)
    SOK(etune_cu_score(c, s->plan, s->model, s->mgen, M, s->mpred, nullptr));
    const int64_t km = ceil_fifths(s->k5, M);
    SOK(etune_cu_topk(c, s->mpred, M, km, s->sel));
    SCU(launch_gather_u64(c->lc(), s->mgen, s->sel, km, s->selgen));
    SCU(launch_gather_u64(c->lc(), s->mpred, s->sel, km, s->psel));
    stage("score");
    // 4. NVMLMeasurement(Kernel_kM)
    SOK(measure_energy(s, s->selgen, km));
    stage("energy");
    // 6. SNR of step-3 predictions vs the measurements in the model's normalised units
    SCU(launch_div_scalar(c->lc(), s->men, km, s->m_sc + 1, s->mnorm));
    double snr = 0.0;
    SOK(etune_cu_snr_db(c, s->psel, s->mnorm, km, &snr, nullptr));
    // 8. parents <- ceil(0.5 M) lowest model-scored of the M
    const int64_t np = (M + 1) / 2;
    SOK(etune_cu_topk(c, s->mpred, M, np, s->idx));
    SCU(launch_gather_u64(c->lc(), s->mgen, s->idx, np, s->par));
    s->np = np;
    if (r + 1 <= s->cfg.max_rounds) SOK(prelaunch_reproduce(s, r + 1));
    stage("snr+parents");
    // 5. ModelUpdate on all accumulated samples
    SOK(append_samples(s, s->selgen, s->men, km));
    stage("append");
    SOK(retrain(s));
    stage("retrain");
    // 7. k controller, k in integer fifths
    const int kb = s->k5;
    const bool poor = s->cfg.inverted_semantics ? !(snr < s->cfg.mu_db) : (snr < s->cfg.mu_db);
    s->k5 = poor ? std::min(5, s->k5 + 1) : std::max(0, s->k5 - 1);
    s->round = r;
    s->cumulative += km;
    bool improved = false;
    SOK(update_best(s, s->selgen, km, &improved));
    s->stall = improved ? 0 : s->stall + 1;
    fill_report(s, kb, snr, km, now_ms() - t0, rep);
    return ETUNE_OK;
}

etune_status etune_cu_search_run(etune_cu_search* s, etune_round_report* reports, int64_t cap, int64_t* n_reports) {
    if (!s) return sfail(ETUNE_ERR_INVALID_ARGUMENT, "null search");
    int64_t n = 0;
    etune_round_report r{};
    if (s->round < 0) {
        SOK(etune_cu_search_initial(s, &r));
        if (reports && n < cap) reports[n] = r;
        ++n;
    }
    while (s->round < s->cfg.max_rounds && s->stall < s->cfg.patience) {
        SOK(etune_cu_search_round(s, &r));
        if (reports && n < cap) reports[n] = r;
        ++n;
    }
    if (n_reports) *n_reports = n;
    return ETUNE_OK;
}

etune_status etune_cu_search_best(etune_cu_search* s, etune_schedule* h_sched, uint64_t* h_id, double* h_lat,
                                  double* h_en) {
    if (!s || !s->have_best) return sfail(ETUNE_ERR_VALIDATION, "no measured candidate yet");
    if (h_id) *h_id = s->best_id;
    if (h_lat) *h_lat = s->best_lat;
    if (h_en) *h_en = s->best_en;
    if (h_sched) {
        etune_cu_ctx* c = s->ctx;
        SCU(cudaMemcpyAsync(s->ids, &s->best_genome, 8, cudaMemcpyHostToDevice, c->stream));
        etune_schedule* d = nullptr;
        SCU(cudaMalloc(&d, sizeof(etune_schedule)));
        SOK(etune_cu_decode(c, s->plan, s->ids, 1, d));
        SCU(cudaMemcpyAsync(h_sched, d, sizeof(etune_schedule), cudaMemcpyDeviceToHost, c->stream));
        SCU(cudaStreamSynchronize(c->stream));
        cudaFree(d);
    }
    return ETUNE_OK;
}

etune_status etune_cu_search_parents(etune_cu_search* s, uint64_t* d_out, int64_t cap, int64_t* n) {
    if (!s || !n) return sfail(ETUNE_ERR_INVALID_ARGUMENT, "null argument");
    *n = s->np;
    const int64_t m = std::min(cap, s->np);
    if (m > 0 && d_out)
        SCU(cudaMemcpyAsync(d_out, s->par, size_t(m) * 8, cudaMemcpyDeviceToDevice, s->ctx->stream));
    return ETUNE_OK;
}

}  // extern "C"
