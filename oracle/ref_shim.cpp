// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libetune_ref.so).  Python tests / the golden-fixture generator /
// bench.py's `--impl reference` arm call these through ctypes.  Every entry
// point calls only public `etune::` APIs; nothing here re-implements reference
// behaviour.
//
// Encodings (shared with oracle/etune_oracle.h and include/etune_cuda.h):
//   op      : int64[12] = kind,batch,m,n,k,height,width,in_ch,out_ch,ks,stride,pad
//             (field order of candidate_id, space.cpp:24-35)
//   sched   : int64[12] = b0,t0,p0,b1,t1,p1,b2,t2,p2,k_tile,unroll,vectorize
//             (field order of candidate_id, space.cpp:36-43)
//   limits  : int64[3]  = max_block_threads,max_unroll,max_vectorize (space.hpp:15-19)
//   status  : 0 ok, else the etune_status code of the thrown exception class.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "etune/counters.hpp"
#include "etune/device.hpp"
#include "etune/energy_model.hpp"
#include "etune/errors.hpp"
#include "etune/features.hpp"
#include "etune/genetic.hpp"
#include "etune/metrics.hpp"
#include "etune/opspec.hpp"
#include "etune/schedule.hpp"
#include "etune/space.hpp"

using namespace etune;

namespace {

thread_local std::string g_last_error;

int status_of(const std::exception& e) {
    // 1:1 with include/etune_cuda.h etune_status (errors.hpp:15-100)
    if (dynamic_cast<const ParseError*>(&e)) return 1;
    if (dynamic_cast<const ValidationError*>(&e)) return 2;
    if (dynamic_cast<const SpaceExhausted*>(&e)) return 3;
    if (dynamic_cast<const IllegalSchedule*>(&e)) return 4;
    if (dynamic_cast<const TooLarge*>(&e)) return 5;
    if (dynamic_cast<const NonPositiveEnergy*>(&e)) return 6;
    if (dynamic_cast<const InsufficientData*>(&e)) return 7;
    if (dynamic_cast<const SchemaMismatch*>(&e)) return 8;
    if (dynamic_cast<const VersionMismatch*>(&e)) return 9;
    if (dynamic_cast<const LengthMismatch*>(&e)) return 10;
    if (dynamic_cast<const EmptyInput*>(&e)) return 11;
    if (dynamic_cast<const IoError*>(&e)) return 12;
    if (dynamic_cast<const ConsistencyError*>(&e)) return 13;
    if (dynamic_cast<const BackendUnavailable*>(&e)) return 14;
    if (dynamic_cast<const TraceMiss*>(&e)) return 15;
    return 99;
}

#define GUARD_BEGIN try {
#define GUARD_END                                  \
    }                                              \
    catch (const std::exception& e) {              \
        g_last_error = e.what();                   \
        return status_of(e);                       \
    }                                              \
    return 0;

OperatorSpec op_from(const int64_t* w) {
    OperatorSpec op;
    op.kind = static_cast<OpKind>(w[0]);
    op.batch = w[1];
    op.m = w[2];
    op.n = w[3];
    op.k = w[4];
    op.height = w[5];
    op.width = w[6];
    op.in_channels = w[7];
    op.out_channels = w[8];
    op.kernel_size = w[9];
    op.stride = w[10];
    op.padding = w[11];
    return op;
}

Schedule sched_from(const int64_t* w) {
    Schedule s;
    for (int d = 0; d < 3; ++d) {
        s.spatial[d].blocks = w[3 * d + 0];
        s.spatial[d].threads = w[3 * d + 1];
        s.spatial[d].per_thread = w[3 * d + 2];
    }
    s.k_tile = w[9];
    s.unroll = w[10];
    s.vectorize = w[11];
    return s;
}

void sched_to(const Schedule& s, int64_t* w) {
    for (int d = 0; d < 3; ++d) {
        w[3 * d + 0] = s.spatial[d].blocks;
        w[3 * d + 1] = s.spatial[d].threads;
        w[3 * d + 2] = s.spatial[d].per_thread;
    }
    w[9] = s.k_tile;
    w[10] = s.unroll;
    w[11] = s.vectorize;
}

SpaceLimits limits_from(const int64_t* w) {
    SpaceLimits l;
    if (w) {
        l.max_block_threads = w[0];
        l.max_unroll = w[1];
        l.max_vectorize = w[2];
    }
    return l;
}

DeviceConfig dev_with_sms(int num_sms) {
    DeviceConfig d = DeviceConfig::a100_like();
    if (num_sms > 0) d.num_sms = num_sms;
    return d;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

int ref_op_validate(const int64_t* op) {
    GUARD_BEGIN
    op_from(op).validate();
    GUARD_END
}

int ref_op_nest(const int64_t* op, int64_t* out4) {
    GUARD_BEGIN
    const LoopNest n = op_from(op).nest();
    out4[0] = n.batch;
    out4[1] = n.m;
    out4[2] = n.n;
    out4[3] = n.k;
    GUARD_END
}

int ref_parse_operator(const char* text, int64_t* out_op) {
    GUARD_BEGIN
    const OperatorSpec op = parse_operator(text);
    out_op[0] = static_cast<int64_t>(op.kind);
    out_op[1] = op.batch;
    out_op[2] = op.m;
    out_op[3] = op.n;
    out_op[4] = op.k;
    out_op[5] = op.height;
    out_op[6] = op.width;
    out_op[7] = op.in_channels;
    out_op[8] = op.out_channels;
    out_op[9] = op.kernel_size;
    out_op[10] = op.stride;
    out_op[11] = op.padding;
    GUARD_END
}

int ref_count_schedules(const int64_t* op, const int64_t* limits, int64_t cap,
                        int64_t* out) {
    GUARD_BEGIN
    *out = count_schedules(op_from(op), limits_from(limits), cap);
    GUARD_END
}

// Writes at most `cap` schedules in enumeration order; *out_n = total written.
int ref_enumerate(const int64_t* op, const int64_t* limits, int64_t cap,
                  int64_t* out_sched, int64_t* out_n) {
    GUARD_BEGIN
    ScheduleEnumerator en(op_from(op), limits_from(limits));
    int64_t n = 0;
    while (n < cap) {
        auto s = en.next();
        if (!s) break;
        sched_to(*s, out_sched + 12 * n);
        ++n;
    }
    *out_n = n;
    GUARD_END
}

int ref_candidate_ids(const int64_t* op, const int64_t* sched, int64_t n,
                      uint64_t* out) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    for (int64_t i = 0; i < n; ++i) out[i] = candidate_id(o, sched_from(sched + 12 * i));
    GUARD_END
}

// Per-candidate legality (1 legal / 0 illegal); never throws for illegal.
int ref_is_legal(const int64_t* op, const int64_t* sched, int64_t n, uint8_t* out) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    for (int64_t i = 0; i < n; ++i) out[i] = schedule_is_legal(o, sched_from(sched + 12 * i));
    GUARD_END
}

// counters: int64[10] per candidate: grid,block,flops,int_ops,glb_ld,glb_st,
// shared_ld,shared_st,sm_efficiency(bits of double),active_sms
int ref_counters(const int64_t* op, const int64_t* sched, int64_t n, int num_sms,
                 int64_t* out) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    const DeviceConfig dev = dev_with_sms(num_sms);
    for (int64_t i = 0; i < n; ++i) {
        const CounterSet c = derive_counters(o, sched_from(sched + 12 * i), dev);
        int64_t* w = out + 10 * i;
        w[0] = c.grid;
        w[1] = c.block;
        w[2] = c.flops;
        w[3] = c.int_ops;
        w[4] = c.glb_ld;
        w[5] = c.glb_st;
        w[6] = c.shared_ld;
        w[7] = c.shared_st;
        std::memcpy(&w[8], &c.sm_efficiency, 8);
        w[9] = c.active_sms;
    }
    GUARD_END
}

int ref_interpret_counters(const int64_t* op, const int64_t* sched, int num_sms,
                           int64_t* out) {
    GUARD_BEGIN
    const CounterSet c =
        interpret_counters(op_from(op), sched_from(sched), dev_with_sms(num_sms));
    out[0] = c.grid;
    out[1] = c.block;
    out[2] = c.flops;
    out[3] = c.int_ops;
    out[4] = c.glb_ld;
    out[5] = c.glb_st;
    out[6] = c.shared_ld;
    out[7] = c.shared_st;
    std::memcpy(&out[8], &c.sm_efficiency, 8);
    out[9] = c.active_sms;
    GUARD_END
}

int ref_features(const int64_t* op, const int64_t* sched, int64_t n, int num_sms,
                 double* out) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    const DeviceConfig dev = dev_with_sms(num_sms);
    for (int64_t i = 0; i < n; ++i) {
        const FeatureVector f = extract_features(o, sched_from(sched + 12 * i), dev);
        std::memcpy(out + 16 * i, f.data(), 16 * sizeof(double));
    }
    GUARD_END
}

double ref_log1p(double x) { return std::log1p(x); }

int ref_sample_random(const int64_t* op, int64_t n, uint64_t seed,
                      const int64_t* limits, int64_t* out_sched, uint64_t* out_ids) {
    GUARD_BEGIN
    const auto cands = sample_random(op_from(op), n, seed, limits_from(limits));
    for (size_t i = 0; i < cands.size(); ++i) {
        sched_to(cands[i].schedule, out_sched + 12 * i);
        out_ids[i] = cands[i].id;
    }
    GUARD_END
}

// lineage: uint64[2*n]; lineage_len: int8[n] (1 or 2)
int ref_reproduce(const int64_t* op, const int64_t* parent_sched, int64_t num_parents,
                  int64_t n, const double* rates, uint64_t seed, const int64_t* limits,
                  int64_t* out_sched, uint64_t* out_ids, uint64_t* out_lineage,
                  int8_t* out_lineage_len) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    std::vector<Candidate> parents;
    parents.reserve(static_cast<size_t>(num_parents));
    for (int64_t p = 0; p < num_parents; ++p) {
        parents.push_back(make_candidate(o, sched_from(parent_sched + 12 * p)));
    }
    GeneticRates r;
    if (rates) {
        r.mutation = rates[0];
        r.crossover = rates[1];
        r.copy = rates[2];
    }
    const auto kids = reproduce(parents, n, r, seed, limits_from(limits));
    for (size_t i = 0; i < kids.size(); ++i) {
        sched_to(kids[i].schedule, out_sched + 12 * i);
        out_ids[i] = kids[i].id;
        out_lineage[2 * i] = kids[i].lineage.size() > 0 ? kids[i].lineage[0] : 0;
        out_lineage[2 * i + 1] = kids[i].lineage.size() > 1 ? kids[i].lineage[1] : 0;
        out_lineage_len[i] = static_cast<int8_t>(kids[i].lineage.size());
    }
    GUARD_END
}

// ---------------------------------------------------------------- cost model

struct RefModel {
    EnergyModel model;
};

// Trains on (features[n*16], energy[n]) with params {num_trees,max_depth,lr,
// min_leaf_weight,reg_lambda}; returns an owned handle.
int ref_train(const double* feats, const double* energy, int64_t n, int num_trees,
              int max_depth, double lr, double min_leaf_weight, double reg_lambda,
              void** out_handle) {
    GUARD_BEGIN
    std::vector<EnergySample> samples(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        std::memcpy(samples[i].features.data(), feats + 16 * i, 16 * sizeof(double));
        samples[i].measured_energy_mj = energy[i];
    }
    BoostParams p;
    p.num_trees = num_trees;
    p.max_depth = max_depth;
    p.learning_rate = lr;
    p.min_leaf_weight = min_leaf_weight;
    p.reg_lambda = reg_lambda;
    auto* h = new RefModel{EnergyModel::train(samples, p)};
    *out_handle = h;
    GUARD_END
}

int ref_model_from_json(const char* text, void** out_handle) {
    GUARD_BEGIN
    auto* h = new RefModel{EnergyModel::from_json(text)};
    *out_handle = h;
    GUARD_END
}

void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

// Returns required length incl. NUL; copies when cap suffices.
int64_t ref_model_to_json(void* h, char* out, int64_t cap) {
    const std::string s = static_cast<RefModel*>(h)->model.to_json();
    const int64_t need = static_cast<int64_t>(s.size()) + 1;
    if (out && cap >= need) std::memcpy(out, s.c_str(), static_cast<size_t>(need));
    return need;
}

int ref_model_info(void* h, double* base_score, double* lr, double* ref_energy,
                   int64_t* num_trees, int64_t* total_nodes) {
    const EnergyModel& m = static_cast<RefModel*>(h)->model;
    *base_score = m.base_score();
    *lr = m.params().learning_rate;
    *ref_energy = m.reference_energy_mj();
    *num_trees = static_cast<int64_t>(m.trees().size());
    int64_t total = 0;
    for (const auto& t : m.trees()) total += static_cast<int64_t>(t.nodes.size());
    *total_nodes = total;
    return 0;
}

// Flat node arrays in tree order; tree_offsets[num_trees+1].
int ref_model_nodes(void* h, int32_t* feature, double* threshold, int32_t* left,
                    int32_t* right, double* value, int64_t* tree_offsets) {
    const EnergyModel& m = static_cast<RefModel*>(h)->model;
    int64_t k = 0;
    int64_t t = 0;
    for (const auto& tree : m.trees()) {
        tree_offsets[t++] = k;
        for (const auto& nd : tree.nodes) {
            feature[k] = nd.feature;
            threshold[k] = nd.threshold;
            left[k] = nd.left;
            right[k] = nd.right;
            value[k] = nd.value;
            ++k;
        }
    }
    tree_offsets[t] = k;
    return 0;
}

int ref_training_loss(void* h, double* out, int64_t cap, int64_t* out_n) {
    const auto& l = static_cast<RefModel*>(h)->model.training_loss_per_round();
    *out_n = static_cast<int64_t>(l.size());
    for (int64_t i = 0; i < cap && i < *out_n; ++i) out[i] = l[static_cast<size_t>(i)];
    return 0;
}

int ref_predict(void* h, const double* feats, int64_t n, double* out) {
    GUARD_BEGIN
    const EnergyModel& m = static_cast<RefModel*>(h)->model;
    FeatureVector f;
    for (int64_t i = 0; i < n; ++i) {
        std::memcpy(f.data(), feats + 16 * i, 16 * sizeof(double));
        out[i] = m.predict(f);
    }
    GUARD_END
}

int ref_snr_db(const double* pred, const double* meas, int64_t n, double* out) {
    GUARD_BEGIN
    std::vector<double> p(pred, pred + n), m(meas, meas + n);
    *out = snr_db(p, m);
    GUARD_END
}

int ref_energy_loss(double pred, double meas, double* out3) {
    GUARD_BEGIN
    const LossTerms t = energy_loss(pred, meas);
    out3[0] = t.value;
    out3[1] = t.gradient;
    out3[2] = t.hessian;
    GUARD_END
}

int ref_spearman(const double* a, const double* b, int64_t n, double* out) {
    GUARD_BEGIN
    std::vector<double> x(a, a + n), y(b, b + n);
    *out = spearman(x, y);
    GUARD_END
}

// The reference's own scoring path (extract_features + EnergyModel::predict,
// features.cpp:48-51, energy_model.cpp:245-249), partitioned over `threads`
// std::threads (the reference itself is single-threaded; partitioning is the
// harness, not a change to the path).  Used by bench.py --impl reference.
int ref_score_threads(const int64_t* op, const int64_t* sched, int64_t n, int num_sms,
                      void* h, int threads, double* out_pred) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    const DeviceConfig dev = dev_with_sms(num_sms);
    const EnergyModel& m = static_cast<RefModel*>(h)->model;
    if (threads < 1) threads = 1;
    std::atomic<int> failed{0};
    auto work = [&](int64_t lo, int64_t hi) {
        try {
            for (int64_t i = lo; i < hi; ++i) {
                out_pred[i] = m.predict(extract_features(o, sched_from(sched + 12 * i), dev));
            }
        } catch (...) {
            failed = 1;
        }
    };
    std::vector<std::thread> pool;
    const int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = t * chunk;
        const int64_t hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
    if (failed) throw IllegalSchedule("scoring failed in a worker thread");
    GUARD_END
}

// The reference's scoring path followed by "keep the best" (the k lowest
// predictions, ties by index -- SURVEY H3), both over `threads` std::threads: each thread
// scores its contiguous chunk and keeps its chunk's k best by (prediction, index) with
// std::partial_sort; the chunk winners (threads x k) are merged by one more partial_sort.
// out_idx[0..k) sorted.  bench.py --impl reference times exactly this (like for like with
// etune_cu_score_select).
int ref_score_select_threads(const int64_t* op, const int64_t* sched, int64_t n, int num_sms, void* h,
                             int threads, int64_t k, double* out_pred, int64_t* out_idx) {
    GUARD_BEGIN
    const OperatorSpec o = op_from(op);
    const DeviceConfig dev = dev_with_sms(num_sms);
    const EnergyModel& m = static_cast<RefModel*>(h)->model;
    if (threads < 1) threads = 1;
    if (k < 0 || k > n) throw ValidationError("need 0 <= k <= n");
    using Rec = std::pair<double, int64_t>;
    std::vector<std::vector<Rec>> best{size_t(threads)};
    std::atomic<int> failed{0};
    auto work = [&](int t, int64_t lo, int64_t hi) {
        try {
            std::vector<Rec> recs;
            recs.reserve(size_t(hi - lo));
            for (int64_t i = lo; i < hi; ++i) {
                const double p = m.predict(extract_features(o, sched_from(sched + 12 * i), dev));
                out_pred[i] = p;
                recs.emplace_back(p, i);
            }
            const int64_t kk = std::min<int64_t>(k, hi - lo);
            std::partial_sort(recs.begin(), recs.begin() + kk, recs.end());
            recs.resize(size_t(kk));
            best[size_t(t)] = std::move(recs);
        } catch (...) {
            failed = 1;
        }
    };
    std::vector<std::thread> pool;
    const int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const int64_t lo = t * chunk;
        const int64_t hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back(work, t, lo, hi);
    }
    for (auto& th : pool) th.join();
    if (failed) throw IllegalSchedule("scoring failed in a worker thread");
    std::vector<Rec> all;
    for (auto& b : best) all.insert(all.end(), b.begin(), b.end());
    std::partial_sort(all.begin(), all.begin() + k, all.end());
    for (int64_t j = 0; j < k; ++j) out_idx[j] = all[size_t(j)].second;
    GUARD_END
}

// ---- persistence formats (device.cpp:44-101, energy_model.cpp:372-420)
// dev: double[11] in etune_device_config field order (constant_power_w ..
// noise_sigma_rel), plus num_sms, rng_seed and name.
int64_t ref_device_profile_to_json(int num_sms, const double* dev, uint64_t seed, const char* name, char* out,
                                   int64_t cap) {
    DeviceConfig d;
    d.name = name;
    d.num_sms = num_sms;
    d.constant_power_w = dev[0];
    d.static_power_per_sm_w = dev[1];
    d.dynamic_energy_per_flop_nj = dev[2];
    d.dynamic_energy_per_glb_access_nj = dev[3];
    d.dynamic_energy_per_shared_access_nj = dev[4];
    d.base_throughput_flops_per_s_per_sm = dev[5];
    d.mem_bandwidth_elems_per_s = dev[6];
    d.latency_floor_ms = dev[7];
    d.sampler_hz = dev[8];
    d.warmup_s = dev[9];
    d.noise_sigma_rel = dev[10];
    d.rng_seed = seed;
    const std::string s = device_profile_to_json(d);
    const int64_t need = static_cast<int64_t>(s.size()) + 1;
    if (out && cap >= need) std::memcpy(out, s.c_str(), static_cast<size_t>(need));
    return need;
}

int ref_device_profile_from_json(const char* text, int* num_sms, double* dev, uint64_t* seed, char* name,
                                 int64_t cap) {
    GUARD_BEGIN
    const DeviceConfig d = device_profile_from_json(text);
    *num_sms = d.num_sms;
    const double v[11] = {d.constant_power_w, d.static_power_per_sm_w, d.dynamic_energy_per_flop_nj,
                          d.dynamic_energy_per_glb_access_nj, d.dynamic_energy_per_shared_access_nj,
                          d.base_throughput_flops_per_s_per_sm, d.mem_bandwidth_elems_per_s, d.latency_floor_ms,
                          d.sampler_hz, d.warmup_s, d.noise_sigma_rel};
    std::memcpy(dev, v, sizeof(v));
    *seed = d.rng_seed;
    if (cap > 0) {
        std::strncpy(name, d.name.c_str(), static_cast<size_t>(cap - 1));
        name[cap - 1] = '\0';
    }
    GUARD_END
}

int ref_samples_save(const double* feats, const double* meas, const double* norm, int64_t n, const char* path) {
    GUARD_BEGIN
    std::vector<EnergySample> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        std::memcpy(v[static_cast<size_t>(i)].features.data(), feats + 16 * i, 16 * sizeof(double));
        v[static_cast<size_t>(i)].measured_energy_mj = meas[i];
        v[static_cast<size_t>(i)].normalized_energy = norm[i];
    }
    save_energy_samples(v, path);
    GUARD_END
}

int ref_samples_load(const char* path, double* feats, double* meas, double* norm, int64_t cap, int64_t* n) {
    GUARD_BEGIN
    const std::vector<EnergySample> v = load_energy_samples(path);
    *n = static_cast<int64_t>(v.size());
    for (int64_t i = 0; i < cap && i < *n; ++i) {
        std::memcpy(feats + 16 * i, v[static_cast<size_t>(i)].features.data(), 16 * sizeof(double));
        meas[i] = v[static_cast<size_t>(i)].measured_energy_mj;
        norm[i] = v[static_cast<size_t>(i)].normalized_energy;
    }
    GUARD_END
}

} // extern "C"
