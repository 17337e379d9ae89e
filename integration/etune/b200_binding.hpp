// etune/b200_binding.hpp -- the reference-side binding of libetune_cuda.so.
//
// This is the file a maintainer of the reference (/root/reference/proj, namespace etune) adds to
// its include/etune/ directory to route the hot path -- scoring a population with the energy
// model and keeping the best, reproduction, sampling -- to a B200.  It uses only the reference's
// public types and the C ABI in include/etune_cuda.h; it is compiled against the reference's own
// headers by tests/cpp/Makefile (binding_test) and checked on the GPU against the reference's
// EnergyModel::predict(extract_features(...)) (tests/test_gpu_binding.py).
//
// Reference interfaces replaced (file:line in /root/reference/proj/include/etune/):
//   extract_features + EnergyModel::predict/predict_many   features.hpp:35-41, energy_model.hpp:72-73
//   keep-the-best by (prediction, index)                   SPEC:403-404 (no reference code)
//   reproduce                                              genetic.hpp:48-51
//   sample_random                                          space.hpp:80-82
//   etune::Error subclasses                                errors.hpp:9-100 (rethrow maps every status)
#pragma once

#include <etune_cuda.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "etune/device.hpp"
#include "etune/energy_model.hpp"
#include "etune/errors.hpp"
#include "etune/genetic.hpp"
#include "etune/opspec.hpp"
#include "etune/schedule.hpp"
#include "etune/space.hpp"

namespace etune::b200 {

static_assert(sizeof(Schedule) == sizeof(etune_schedule), "schedule.hpp:40-44: 12 x int64 in candidate_id order");

// Every etune_status maps onto the exception class the reference throws for it (errors.hpp:15-100,
// 1:1 with the enum in etune_cuda.h).  The statuses without a reference analogue -- a bad argument
// to the C ABI, a CUDA failure, no B200 present, a shape beyond this build's tables -- surface as
// BackendUnavailable (the reference's "this backend cannot do it" error, measure.hpp:130-140) and
// ValidationError (bad argument).
[[noreturn]] inline void rethrow(etune_status st, int64_t index = -1) {
    const std::string w = std::string(etune_cu_last_error()) +
                          (index >= 0 ? " (element " + std::to_string(index) + ")" : std::string());
    switch (st) {
    case ETUNE_ERR_PARSE: throw ParseError(w);
    case ETUNE_ERR_VALIDATION: throw ValidationError(w);
    case ETUNE_ERR_SPACE_EXHAUSTED: throw SpaceExhausted(w);
    case ETUNE_ERR_ILLEGAL_SCHEDULE: throw IllegalSchedule(w);
    case ETUNE_ERR_TOO_LARGE: throw TooLarge(w);
    case ETUNE_ERR_NON_POSITIVE_ENERGY: throw NonPositiveEnergy(w);
    case ETUNE_ERR_INSUFFICIENT_DATA: throw InsufficientData(w);
    case ETUNE_ERR_SCHEMA_MISMATCH: throw SchemaMismatch(w);
    case ETUNE_ERR_VERSION_MISMATCH: throw VersionMismatch(w);
    case ETUNE_ERR_LENGTH_MISMATCH: throw LengthMismatch(w);
    case ETUNE_ERR_EMPTY_INPUT: throw EmptyInput(w);
    case ETUNE_ERR_IO: throw IoError(w);
    case ETUNE_ERR_CONSISTENCY: throw ConsistencyError(w);
    case ETUNE_ERR_BACKEND_UNAVAILABLE: throw BackendUnavailable(w);
    case ETUNE_ERR_TRACE_MISS: throw TraceMiss(w);
    case ETUNE_ERR_INVALID_ARGUMENT: throw ValidationError(w);
    default: throw BackendUnavailable(w);  // CUDA, NO_DEVICE, UNSUPPORTED
    }
}

inline void check(etune_status st, int64_t index = -1) {
    if (st != ETUNE_OK) rethrow(st, index);
}

inline etune_op_spec to_c(const OperatorSpec& o) {  // opspec.hpp:30-47, candidate_id word order
    return {int64_t(o.kind), o.batch, o.m, o.n, o.k, o.height, o.width, o.in_channels, o.out_channels,
            o.kernel_size, o.stride, o.padding};
}

inline etune_device_config to_c(const DeviceConfig& d) {  // device.hpp:17-45, every numeric field
    etune_device_config c{};
    c.num_sms = d.num_sms;
    c.constant_power_w = d.constant_power_w;
    c.static_power_per_sm_w = d.static_power_per_sm_w;
    c.dynamic_energy_per_flop_nj = d.dynamic_energy_per_flop_nj;
    c.dynamic_energy_per_glb_access_nj = d.dynamic_energy_per_glb_access_nj;
    c.dynamic_energy_per_shared_access_nj = d.dynamic_energy_per_shared_access_nj;
    c.base_throughput_flops_per_s_per_sm = d.base_throughput_flops_per_s_per_sm;
    c.mem_bandwidth_elems_per_s = d.mem_bandwidth_elems_per_s;
    c.latency_floor_ms = d.latency_floor_ms;
    c.sampler_hz = d.sampler_hz;
    c.warmup_s = d.warmup_s;
    c.noise_sigma_rel = d.noise_sigma_rel;
    c.rng_seed = d.rng_seed;
    return c;
}

inline etune_space_limits to_c(const SpaceLimits& l) { return {l.max_block_threads, l.max_unroll, l.max_vectorize}; }

class Engine;

// An EnergyModel resident on the device (its flat TreeNode arrays, energy_model.hpp:45-57).  The
// first large population scored for an operator compiles the model's row table on the device
// (no host work); the model is immutable afterwards, like EnergyModel.
class Model {
public:
    Model(Engine& e, const EnergyModel& m);
    ~Model() { etune_cu_forest_destroy(f_); }
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;
    etune_cu_forest* handle() const { return f_; }

private:
    etune_cu_forest* f_ = nullptr;
};

// One per thread and GPU (the reference's pure functions are thread-safe; a ctx is
// thread-compatible).  Plans -- an operator's knob and feature tables -- are created once per
// (operator, DeviceConfig, SpaceLimits) and cached, so a model's compiled forms are reused across
// calls; destroying the Engine destroys its plans, which evicts every form compiled for them.
class Engine {
public:
    explicit Engine(int device = 0, void* stream = nullptr) { check(etune_cu_ctx_create(device, stream, &ctx_)); }
    ~Engine() {
        for (auto& kv : plans_) etune_cu_plan_destroy(kv.second);
        etune_cu_ctx_destroy(ctx_);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    etune_cu_ctx* ctx() const { return ctx_; }

    etune_cu_plan* plan(const OperatorSpec& op, const DeviceConfig& dev, const SpaceLimits& lim = {}) {
        const etune_op_spec o = to_c(op);
        const etune_device_config d = to_c(dev);
        const etune_space_limits l = to_c(lim);
        std::string key(reinterpret_cast<const char*>(&o), sizeof(o));
        key.append(reinterpret_cast<const char*>(&d), sizeof(d));
        key.append(reinterpret_cast<const char*>(&l), sizeof(l));
        std::lock_guard<std::mutex> lock(mu_);
        auto it = plans_.find(key);
        if (it != plans_.end()) return it->second;
        etune_cu_plan* p = nullptr;
        check(etune_cu_plan_create(ctx_, &o, &d, &l, &p));
        plans_.emplace(key, p);
        return p;
    }

    // for (c : pop) out[i] = model.predict(extract_features(op, c.schedule, dev))
    // (features.hpp:35-41 + energy_model.cpp:245-257), bit-identical; IllegalSchedule names the
    // first candidate the reference's loop would have thrown on.
    std::vector<double> predict_many(const Model& m, const OperatorSpec& op, const DeviceConfig& dev,
                                     const std::vector<Candidate>& pop) {
        const std::vector<Schedule> s = schedules(pop);
        std::vector<double> pred(pop.size());
        int64_t bad = -1;
        const etune_status st = etune_cu_score_host(ctx_, plan(op, dev), m.handle(), as_c(s), int64_t(s.size()),
                                                    pred.data(), nullptr, &bad);
        check(st, bad);
        return pred;
    }

    // The k candidates with the lowest predicted energy, ties by position, sorted;
    // `pred` (optional) receives every prediction.
    std::vector<std::size_t> keep_best(const Model& m, const OperatorSpec& op, const DeviceConfig& dev,
                                       const std::vector<Candidate>& pop, std::size_t k,
                                       std::vector<double>* pred = nullptr) {
        const std::vector<Schedule> s = schedules(pop);
        if (pred) pred->resize(pop.size());
        std::vector<int64_t> idx(k);
        int64_t bad = -1;
        const etune_status st =
            etune_cu_score_select_host(ctx_, plan(op, dev), m.handle(), as_c(s), int64_t(s.size()), int64_t(k),
                                       pred ? pred->data() : nullptr, idx.data(), &bad);
        check(st, bad);
        return std::vector<std::size_t>(idx.begin(), idx.end());
    }

    // etune::reproduce (genetic.hpp:48-51): the same offspring, ids and lineage from the same
    // std::mt19937_64(seed) stream, computed on the device.
    std::vector<Candidate> reproduce(const std::vector<Candidate>& parents, std::int64_t n,
                                     const GeneticRates& rates = {}, std::uint64_t seed = 0,
                                     const SpaceLimits& lim = {}) {
        if (parents.empty()) throw ValidationError("reproduce requires at least one parent");
        const OperatorSpec& op = parents.front().op;
        etune_cu_plan* p = plan(op, DeviceConfig::a100_like(), lim);
        const std::vector<Schedule> s = schedules(parents);
        const int64_t np = int64_t(parents.size());
        Dev<etune_schedule> d_s(ctx_, np > n ? np : n);
        Dev<uint64_t> d_par(ctx_, np), d_out(ctx_, n), d_ids(ctx_, n);
        Dev<int32_t> d_partner(ctx_, n);
        check(etune_cu_memcpy_h2d(ctx_, d_s.p, s.data(), np * int64_t(sizeof(etune_schedule))));
        check(etune_cu_encode(ctx_, p, d_s.p, np, d_par.p));
        const etune_genetic_rates r{rates.mutation, rates.crossover, rates.copy};
        check(etune_cu_reproduce(ctx_, p, d_par.p, np, n, &r, seed, d_out.p, d_partner.p, d_ids.p));
        check(etune_cu_decode(ctx_, p, d_out.p, n, d_s.p));
        std::vector<Schedule> kids(static_cast<size_t>(n));
        std::vector<uint64_t> ids(static_cast<size_t>(n));
        std::vector<int32_t> partner(static_cast<size_t>(n));
        check(etune_cu_memcpy_d2h(ctx_, kids.data(), d_s.p, n * int64_t(sizeof(etune_schedule))));
        check(etune_cu_memcpy_d2h(ctx_, ids.data(), d_ids.p, n * 8));
        check(etune_cu_memcpy_d2h(ctx_, partner.data(), d_partner.p, n * 4));
        int64_t bad = -1;
        check(etune_cu_synchronize(ctx_, &bad), bad);
        std::vector<Candidate> out(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            Candidate& c = out[size_t(i)];
            c.id = ids[size_t(i)];
            c.op = op;
            c.schedule = kids[size_t(i)];
            const Candidate& base = parents[size_t(i % np)];
            c.lineage = partner[size_t(i)] < 0 ? std::vector<std::uint64_t>{base.id}
                                               : std::vector<std::uint64_t>{base.id, parents[size_t(partner[size_t(i)])].id};
        }
        return out;
    }

    // etune::sample_random (space.hpp:80-82) on the device: the same candidates in the same order.
    std::vector<Candidate> sample_random(const OperatorSpec& op, std::int64_t n, std::uint64_t seed,
                                         const SpaceLimits& lim = {}) {
        etune_cu_plan* p = plan(op, DeviceConfig::a100_like(), lim);
        Dev<uint64_t> d_g(ctx_, n), d_ids(ctx_, n);
        Dev<etune_schedule> d_s(ctx_, n);
        check(etune_cu_sample_random(ctx_, p, n, seed, d_g.p, d_ids.p));
        check(etune_cu_decode(ctx_, p, d_g.p, n, d_s.p));
        std::vector<Schedule> s(static_cast<size_t>(n));
        std::vector<uint64_t> ids(static_cast<size_t>(n));
        check(etune_cu_memcpy_d2h(ctx_, s.data(), d_s.p, n * int64_t(sizeof(etune_schedule))));
        check(etune_cu_memcpy_d2h(ctx_, ids.data(), d_ids.p, n * 8));
        check(etune_cu_synchronize(ctx_, nullptr));
        std::vector<Candidate> out(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            out[size_t(i)].id = ids[size_t(i)];
            out[size_t(i)].op = op;
            out[size_t(i)].schedule = s[size_t(i)];
        }
        return out;
    }

private:
    template <typename T>
    struct Dev {  // device buffer owned by one binding call
        etune_cu_ctx* c;
        T* p = nullptr;
        Dev(etune_cu_ctx* ctx, int64_t n) : c(ctx) {
            check(etune_cu_device_alloc(c, reinterpret_cast<void**>(&p), int64_t(n > 0 ? n : 1) * int64_t(sizeof(T))));
        }
        ~Dev() { etune_cu_device_free(c, p); }
    };

    static std::vector<Schedule> schedules(const std::vector<Candidate>& pop) {
        std::vector<Schedule> s(pop.size());
        for (size_t i = 0; i < pop.size(); ++i) s[i] = pop[i].schedule;
        return s;
    }
    static const etune_schedule* as_c(const std::vector<Schedule>& s) {
        return reinterpret_cast<const etune_schedule*>(s.data());
    }

    etune_cu_ctx* ctx_ = nullptr;
    std::mutex mu_;
    std::map<std::string, etune_cu_plan*> plans_;
};

inline Model::Model(Engine& e, const EnergyModel& m) {
    std::vector<int32_t> f, l, r;
    std::vector<double> t, v;
    std::vector<int64_t> off{0};
    for (const RegressionTree& tree : m.trees()) {
        for (const TreeNode& nd : tree.nodes) {
            f.push_back(nd.feature);
            t.push_back(nd.threshold);
            l.push_back(nd.left);
            r.push_back(nd.right);
            v.push_back(nd.value);
        }
        off.push_back(int64_t(f.size()));
    }
    check(etune_cu_forest_create(e.ctx(), f.data(), t.data(), l.data(), r.data(), v.data(), off.data(),
                                 int64_t(m.trees().size()), m.base_score(), m.params().learning_rate, &f_));
}

}  // namespace etune::b200
