// etune_b200.hpp — the C++ host-side mirror of the reference's API (namespace etune,
// /root/reference/proj/include/etune/*.hpp) over the C ABI of libetune_cuda.so.
//
// Same names, argument meaning and error behaviour as the reference, with the work done
// on an sm_100a device:
//   extract_features        features.hpp:35-41         -> etune_cu_encode + etune_cu_features
//   EnergyModel::train      energy_model.hpp:69-70     -> etune_cu_train
//   EnergyModel::predict(_many) energy_model.hpp:72-73 -> etune_cu_predict
//   snr_db                  energy_model.hpp:108-109   -> etune_cu_snr_db
//   candidate_id            space.hpp:32               -> etune_cu_candidate_ids
//   sample_random           space.hpp:80-82            -> etune_cu_sample_random
//   reproduce               genetic.hpp:48-51          -> etune_cu_reproduce
//   derive_counters         counters.hpp:35            -> etune_cu_counters
// plus the batch / device-resident calls the reference does not have (score a whole
// population in one call, top-k, the Algorithm-1 search loop).  Errors throw
// etune_b200::Error subclasses named like etune::Error's (errors.hpp:9-100); a batch
// call reports the lowest offending index, the element the reference's loop would
// have thrown on.  Header-only: link libetune_cuda.so and the CUDA runtime.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "etune_cuda.h"

namespace etune_b200 {

// ------------------------------------------------------------------ errors
class Error : public std::runtime_error {
public:
    Error(etune_status code, const std::string& what, int64_t index)
        : std::runtime_error(what), code_(code), index_(index) {}
    etune_status code() const { return code_; }
    int64_t index() const { return index_; }  // offending element of a batch, or -1

private:
    etune_status code_;
    int64_t index_;
};
#define ETUNE_B200_ERROR(Name)                                                               \
    struct Name : Error {                                                                    \
        Name(etune_status c, const std::string& w, int64_t i) : Error(c, w, i) {}            \
    };
ETUNE_B200_ERROR(ParseError)
ETUNE_B200_ERROR(ValidationError)
ETUNE_B200_ERROR(SpaceExhausted)
ETUNE_B200_ERROR(IllegalSchedule)
ETUNE_B200_ERROR(TooLarge)
ETUNE_B200_ERROR(NonPositiveEnergy)
ETUNE_B200_ERROR(InsufficientData)
ETUNE_B200_ERROR(SchemaMismatch)
ETUNE_B200_ERROR(VersionMismatch)
ETUNE_B200_ERROR(LengthMismatch)
ETUNE_B200_ERROR(EmptyInput)
ETUNE_B200_ERROR(IoError)
ETUNE_B200_ERROR(ConsistencyError)
ETUNE_B200_ERROR(BackendUnavailable)
ETUNE_B200_ERROR(TraceMiss)
ETUNE_B200_ERROR(DeviceError)  // invalid argument / CUDA / no device / unsupported: no reference analogue
#undef ETUNE_B200_ERROR

[[noreturn]] inline void throw_status(etune_status st, int64_t index = -1) {
    const std::string w = etune_cu_last_error();
    switch (st) {
    case ETUNE_ERR_PARSE: throw ParseError(st, w, index);
    case ETUNE_ERR_VALIDATION: throw ValidationError(st, w, index);
    case ETUNE_ERR_SPACE_EXHAUSTED: throw SpaceExhausted(st, w, index);
    case ETUNE_ERR_ILLEGAL_SCHEDULE: throw IllegalSchedule(st, w, index);
    case ETUNE_ERR_TOO_LARGE: throw TooLarge(st, w, index);
    case ETUNE_ERR_NON_POSITIVE_ENERGY: throw NonPositiveEnergy(st, w, index);
    case ETUNE_ERR_INSUFFICIENT_DATA: throw InsufficientData(st, w, index);
    case ETUNE_ERR_SCHEMA_MISMATCH: throw SchemaMismatch(st, w, index);
    case ETUNE_ERR_VERSION_MISMATCH: throw VersionMismatch(st, w, index);
    case ETUNE_ERR_LENGTH_MISMATCH: throw LengthMismatch(st, w, index);
    case ETUNE_ERR_EMPTY_INPUT: throw EmptyInput(st, w, index);
    case ETUNE_ERR_IO: throw IoError(st, w, index);
    case ETUNE_ERR_CONSISTENCY: throw ConsistencyError(st, w, index);
    case ETUNE_ERR_BACKEND_UNAVAILABLE: throw BackendUnavailable(st, w, index);
    case ETUNE_ERR_TRACE_MISS: throw TraceMiss(st, w, index);
    default: throw DeviceError(st, w, index);
    }
}

inline void check(etune_status st) {
    if (st != ETUNE_OK) throw_status(st);
}

// ------------------------------------------------------------ value types
using OperatorSpec = etune_op_spec;   // opspec.hpp:30-47, words in candidate_id order
using Schedule = etune_schedule;      // schedule.hpp:40-44
using CounterSet = etune_counters;    // counters.hpp:13-24
using DeviceConfig = etune_device_config;
using SpaceLimits = etune_space_limits;
using GeneticRates = etune_genetic_rates;
using BoostParams = etune_boost_params;
using FeatureVector = std::array<double, 16>;  // features.hpp:29

inline OperatorSpec make_mm(int64_t batch, int64_t m, int64_t n, int64_t k) {  // opspec.hpp:49-52
    return OperatorSpec{0, batch, m, n, k, 0, 0, 0, 0, 0, 1, 0};
}
inline OperatorSpec make_mv(int64_t batch, int64_t n, int64_t k) {
    return OperatorSpec{1, batch, 1, n, k, 0, 0, 0, 0, 0, 1, 0};
}
inline OperatorSpec make_conv(int64_t batch, int64_t h, int64_t w, int64_t cin, int64_t cout, int64_t ks,
                              int64_t stride, int64_t pad) {
    return OperatorSpec{2, batch, 1, 1, 1, h, w, cin, cout, ks, stride, pad};
}
inline DeviceConfig a100_like() {  // DeviceConfig::a100_like(), device.hpp:44
    DeviceConfig d;
    etune_default_device_config(&d);
    return d;
}
inline SpaceLimits default_limits() {
    SpaceLimits l;
    etune_default_space_limits(&l);
    return l;
}
inline BoostParams default_boost() {
    BoostParams b;
    etune_default_boost_params(&b);
    return b;
}
inline GeneticRates default_rates() {
    GeneticRates r;
    etune_default_genetic_rates(&r);
    return r;
}

struct Candidate {  // space.hpp:22-30
    uint64_t id = 0;
    Schedule schedule{};
    std::vector<uint64_t> lineage;
};

struct EnergySample {  // energy_model.hpp:27-31
    FeatureVector features{};
    double measured_energy_mj = 0.0;
    double normalized_energy = 0.0;
};

// ------------------------------------------------------- device plumbing
template <typename T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t n) { resize(n); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer() { cudaFree(p_); }
    void resize(size_t n) {
        if (n <= cap_) {
            n_ = n;
            return;
        }
        cudaFree(p_);
        p_ = nullptr;
        if (cudaMalloc(&p_, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) throw_status(ETUNE_ERR_CUDA);
        cap_ = n_ = n;
    }
    void upload(const T* h, size_t n) {
        resize(n);
        if (n && cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
            throw_status(ETUNE_ERR_CUDA);
    }
    std::vector<T> download(size_t n) const {
        std::vector<T> h(n);
        if (n && cudaMemcpy(h.data(), p_, n * sizeof(T), cudaMemcpyDeviceToHost) != cudaSuccess)
            throw_status(ETUNE_ERR_CUDA);
        return h;
    }
    T* get() const { return static_cast<T*>(p_); }
    size_t size() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0, cap_ = 0;
};

// One GPU + stream (etune_cu_ctx).  Not copyable; one per thread of use.
class Device {
public:
    explicit Device(int device = 0, cudaStream_t stream = nullptr) { check(etune_cu_ctx_create(device, stream, &h_)); }
    ~Device() { etune_cu_ctx_destroy(h_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    etune_cu_ctx* get() const { return h_; }
    // waits for the device; rethrows a data error found on the device with its index
    void synchronize() const {
        int64_t bad = -1;
        const etune_status st = etune_cu_synchronize(h_, &bad);
        if (st != ETUNE_OK) throw_status(st, bad);
    }

private:
    etune_cu_ctx* h_ = nullptr;
};

// An operator's knob and feature tables on the device (per OperatorSpec + DeviceConfig).
class Plan {
public:
    Plan(Device& dev, const OperatorSpec& op, const DeviceConfig& cfg = a100_like(),
         const SpaceLimits& limits = default_limits())
        : dev_(&dev), op_(op) {
        check(etune_cu_plan_create(dev.get(), &op, &cfg, &limits, &h_));
    }
    ~Plan() { etune_cu_plan_destroy(h_); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    etune_cu_plan* get() const { return h_; }
    Device& device() const { return *dev_; }
    const OperatorSpec& op() const { return op_; }
    std::array<int64_t, 4> nest() const {  // OperatorSpec::nest, opspec.cpp:103-117
        std::array<int64_t, 4> v{};
        check(etune_cu_plan_nest(h_, v.data()));
        return v;
    }
    int64_t count_schedules() const {  // space.cpp:152-160 (uncapped)
        int64_t v = 0;
        check(etune_cu_plan_space_size(h_, &v));
        return v;
    }
    // Schedules -> device genomes (validates like validate_schedule, schedule.cpp:26-61)
    void encode(const std::vector<Schedule>& s, DeviceBuffer<uint64_t>& genome) const {
        DeviceBuffer<Schedule> ds;
        ds.upload(s.data(), s.size());
        genome.resize(s.size());
        check(etune_cu_encode(dev_->get(), h_, ds.get(), int64_t(s.size()), genome.get()));
        dev_->synchronize();
    }
    std::vector<Schedule> decode(const DeviceBuffer<uint64_t>& genome, size_t n) const {
        DeviceBuffer<Schedule> ds(n);
        check(etune_cu_decode(dev_->get(), h_, genome.get(), int64_t(n), ds.get()));
        dev_->synchronize();
        return ds.download(n);
    }

private:
    Device* dev_;
    OperatorSpec op_;
    etune_cu_plan* h_ = nullptr;
};

// ------------------------------------------------------------- analysis
inline std::vector<uint64_t> candidate_ids(const Plan& plan, const std::vector<Schedule>& s) {
    DeviceBuffer<uint64_t> g, ids(s.size());
    plan.encode(s, g);
    check(etune_cu_candidate_ids(plan.device().get(), plan.get(), g.get(), int64_t(s.size()), ids.get()));
    plan.device().synchronize();
    return ids.download(s.size());
}
inline uint64_t candidate_id(const Plan& plan, const Schedule& s) { return candidate_ids(plan, std::vector<Schedule>{s})[0]; }

inline std::vector<CounterSet> derive_counters(const Plan& plan, const std::vector<Schedule>& s) {
    DeviceBuffer<uint64_t> g;
    plan.encode(s, g);
    DeviceBuffer<CounterSet> out(s.size());
    check(etune_cu_counters(plan.device().get(), plan.get(), g.get(), int64_t(s.size()), out.get()));
    plan.device().synchronize();
    return out.download(s.size());
}

// extract_features (features.hpp:35-41) — batch form; the per-candidate form routes to n = 1
inline std::vector<FeatureVector> extract_features(const Plan& plan, const std::vector<Schedule>& s) {
    DeviceBuffer<uint64_t> g;
    plan.encode(s, g);
    DeviceBuffer<FeatureVector> out(s.size());
    check(etune_cu_features(plan.device().get(), plan.get(), g.get(), int64_t(s.size()),
                            reinterpret_cast<double*>(out.get()), nullptr));
    plan.device().synchronize();
    return out.download(s.size());
}
inline FeatureVector extract_features(const Plan& plan, const Schedule& s) { return extract_features(plan, std::vector<Schedule>{s})[0]; }

// ------------------------------------------------------------ cost model
class EnergyModel {  // energy_model.hpp:59-97
public:
    // EnergyModel::train (energy_model.cpp:173-243) on the device, bit-exact.
    static EnergyModel train(Device& dev, const std::vector<EnergySample>& samples,
                             const BoostParams& params = default_boost()) {
        const int64_t n = int64_t(samples.size());
        std::vector<double> f(size_t(n) * 16), e(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            for (int j = 0; j < 16; ++j) f[size_t(i) * 16 + j] = samples[size_t(i)].features[size_t(j)];
            e[size_t(i)] = samples[size_t(i)].measured_energy_mj;
        }
        DeviceBuffer<double> df, de;
        df.upload(f.data(), f.size());
        de.upload(e.data(), e.size());
        const size_t cap = size_t(std::max(params.num_trees, 0)) * ((size_t(1) << (params.max_depth + 1)) - 1);
        DeviceBuffer<int32_t> fe(cap), le(cap), ri(cap);
        DeviceBuffer<double> th(cap), va(cap), sc(2), loss(size_t(params.num_trees) + 1);
        DeviceBuffer<int64_t> off(size_t(params.num_trees) + 1);
        check(etune_cu_train(dev.get(), df.get(), de.get(), n, &params, fe.get(), th.get(), le.get(), ri.get(),
                             va.get(), off.get(), sc.get(), loss.get()));
        dev.synchronize();
        EnergyModel m(dev);
        m.params_ = params;
        m.offsets_ = off.download(size_t(params.num_trees) + 1);
        const size_t nn = size_t(m.offsets_.back());
        m.feature_ = fe.download(nn);
        m.left_ = le.download(nn);
        m.right_ = ri.download(nn);
        m.threshold_ = th.download(nn);
        m.value_ = va.download(nn);
        const auto s2 = sc.download(2);
        m.base_score_ = s2[0];
        m.reference_energy_mj_ = s2[1];
        m.training_loss_ = loss.download(size_t(params.num_trees) + 1);
        m.upload();
        return m;
    }
    // A model from the reference's flat TreeNode arrays (e.g. loaded by etune::EnergyModel::load).
    static EnergyModel from_nodes(Device& dev, std::vector<int32_t> feature, std::vector<double> threshold,
                                  std::vector<int32_t> left, std::vector<int32_t> right, std::vector<double> value,
                                  std::vector<int64_t> offsets, double base_score, double learning_rate,
                                  double reference_energy_mj = 1.0) {
        EnergyModel m(dev);
        m.feature_ = std::move(feature);
        m.threshold_ = std::move(threshold);
        m.left_ = std::move(left);
        m.right_ = std::move(right);
        m.value_ = std::move(value);
        m.offsets_ = std::move(offsets);
        m.base_score_ = base_score;
        m.params_ = default_boost();
        m.params_.learning_rate = learning_rate;
        m.params_.num_trees = int32_t(m.offsets_.size()) - 1;
        m.reference_energy_mj_ = reference_energy_mj;
        m.upload();
        return m;
    }

    // EnergyModel::predict / predict_many (energy_model.cpp:245-257)
    std::vector<double> predict_many(const std::vector<FeatureVector>& f) const {
        DeviceBuffer<double> df, out(f.size());
        df.upload(reinterpret_cast<const double*>(f.data()), f.size() * 16);
        check(etune_cu_predict(dev_->get(), forest_.get(), df.get(), int64_t(f.size()), out.get()));
        dev_->synchronize();
        return out.download(f.size());
    }
    double predict(const FeatureVector& f) const { return predict_many(std::vector<FeatureVector>{f})[0]; }

    // The north-star pass: schedules -> predicted normalised energy (features never leave the device).
    std::vector<double> score(const Plan& plan, const std::vector<Schedule>& s) const {
        std::vector<double> out(s.size());
        int64_t bad = -1;
        const etune_status st = etune_cu_score_host(dev_->get(), plan.get(), forest_.get(), s.data(),
                                                    int64_t(s.size()), out.data(), nullptr, &bad);
        if (st != ETUNE_OK) throw_status(st, bad);
        return out;
    }

    // EnergyModel::to_json / from_json / save / load (energy_model.cpp:259-350): the
    // reference's "etune-model-v1" text, byte-identical to its own writer.
    std::string to_json() const {
        int64_t len = 0;
        check(etune_model_to_json(feature_.data(), threshold_.data(), left_.data(), right_.data(), value_.data(),
                                  offsets_.data(), int64_t(offsets_.size()) - 1, &params_, base_score_,
                                  reference_energy_mj_, nullptr, 0, &len));
        std::string s(size_t(len) + 1, '\0');
        check(etune_model_to_json(feature_.data(), threshold_.data(), left_.data(), right_.data(), value_.data(),
                                  offsets_.data(), int64_t(offsets_.size()) - 1, &params_, base_score_,
                                  reference_energy_mj_, &s[0], len + 1, &len));
        s.resize(size_t(len));
        return s;
    }
    static EnergyModel from_json(Device& dev, const std::string& text) {
        etune_model_host h;
        check(etune_model_from_json(text.data(), int64_t(text.size()), &h));
        const size_t nn = size_t(h.num_nodes);
        EnergyModel m(dev);
        m.feature_.assign(h.feature, h.feature + nn);
        m.threshold_.assign(h.threshold, h.threshold + nn);
        m.left_.assign(h.left, h.left + nn);
        m.right_.assign(h.right, h.right + nn);
        m.value_.assign(h.value, h.value + nn);
        m.offsets_.assign(h.tree_offsets, h.tree_offsets + h.num_trees + 1);
        m.params_ = h.params;
        m.base_score_ = h.base_score;
        m.reference_energy_mj_ = h.reference_energy_mj;
        etune_model_host_free(&h);
        m.upload();
        return m;
    }
    void save(const std::string& path) const {
        std::ofstream out(path);
        if (!out) throw IoError(ETUNE_ERR_IO, "cannot write model file '" + path + "'", -1);
        out << to_json() << '\n';
        if (!out) throw IoError(ETUNE_ERR_IO, "failed writing model file '" + path + "'", -1);
    }
    static EnergyModel load(Device& dev, const std::string& path) {
        std::ifstream in(path);
        if (!in) throw IoError(ETUNE_ERR_IO, "cannot open model file '" + path + "'", -1);
        std::ostringstream buf;
        buf << in.rdbuf();
        return from_json(dev, buf.str());
    }

    double base_score() const { return base_score_; }
    double reference_energy_mj() const { return reference_energy_mj_; }
    const BoostParams& params() const { return params_; }
    const std::vector<double>& training_loss_per_round() const { return training_loss_; }
    const std::vector<int64_t>& tree_offsets() const { return offsets_; }
    const std::vector<int32_t>& node_feature() const { return feature_; }
    const std::vector<double>& node_threshold() const { return threshold_; }
    const std::vector<int32_t>& node_left() const { return left_; }
    const std::vector<int32_t>& node_right() const { return right_; }
    const std::vector<double>& node_value() const { return value_; }
    etune_cu_forest* forest() const { return forest_.get(); }

private:
    explicit EnergyModel(Device& dev) : dev_(&dev) {}
    void upload() {
        etune_cu_forest* f = nullptr;
        check(etune_cu_forest_create(dev_->get(), feature_.data(), threshold_.data(), left_.data(), right_.data(),
                                     value_.data(), offsets_.data(), int64_t(offsets_.size()) - 1, base_score_,
                                     params_.learning_rate, &f));
        forest_ = std::shared_ptr<etune_cu_forest>(f, [](etune_cu_forest* p) { etune_cu_forest_destroy(p); });
    }
    Device* dev_;
    BoostParams params_{};
    double base_score_ = 0.0, reference_energy_mj_ = 1.0;
    std::vector<int32_t> feature_, left_, right_;
    std::vector<double> threshold_, value_, training_loss_;
    std::vector<int64_t> offsets_;
    std::shared_ptr<etune_cu_forest> forest_;
};

// snr_db (energy_model.cpp:352-370)
inline double snr_db(Device& dev, const std::vector<double>& predicted, const std::vector<double>& measured) {
    if (predicted.size() != measured.size())
        throw LengthMismatch(ETUNE_ERR_LENGTH_MISMATCH, "snr_db requires equal-length vectors", -1);
    DeviceBuffer<double> p, m;
    p.upload(predicted.data(), predicted.size());
    m.upload(measured.data(), measured.size());
    double out = 0.0;
    int64_t bad = -1;
    const etune_status st = etune_cu_snr_db(dev.get(), p.get(), m.get(), int64_t(predicted.size()), &out, &bad);
    if (st != ETUNE_OK) throw_status(st, bad);
    return out;
}

// ------------------------------------------------------------- population
// save_energy_samples / load_energy_samples (energy_model.cpp:372-420)
inline void save_energy_samples(const std::vector<EnergySample>& samples, const std::string& path) {
    std::vector<double> f, m, z;
    for (const EnergySample& s : samples) {
        f.insert(f.end(), s.features.begin(), s.features.end());
        m.push_back(s.measured_energy_mj);
        z.push_back(s.normalized_energy);
    }
    int64_t len = 0;
    const int64_t n = int64_t(samples.size());
    check(etune_samples_to_jsonl(f.data(), m.data(), z.data(), n, nullptr, 0, &len));
    std::string text(size_t(len) + 1, '\0');
    check(etune_samples_to_jsonl(f.data(), m.data(), z.data(), n, &text[0], len + 1, &len));
    std::ofstream out(path);
    if (!out) throw IoError(ETUNE_ERR_IO, "cannot write samples file '" + path + "'", -1);
    out.write(text.data(), len);
    if (!out) throw IoError(ETUNE_ERR_IO, "failed writing samples file '" + path + "'", -1);
}
inline std::vector<EnergySample> load_energy_samples(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError(ETUNE_ERR_IO, "cannot open samples file '" + path + "'", -1);
    std::ostringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();
    etune_samples_host h;
    check(etune_samples_from_jsonl(text.data(), int64_t(text.size()), &h));
    std::vector<EnergySample> out(static_cast<size_t>(h.n));
    for (int64_t i = 0; i < h.n; ++i) {
        std::copy(h.features + 16 * i, h.features + 16 * (i + 1), out[size_t(i)].features.begin());
        out[size_t(i)].measured_energy_mj = h.measured_energy_mj[i];
        out[size_t(i)].normalized_energy = h.normalized_energy[i];
    }
    etune_samples_host_free(&h);
    return out;
}
// device_profile_to_json / device_profile_from_json (device.cpp:44-101)
inline std::string device_profile_to_json(const DeviceConfig& dev, const std::string& name = "a100-like") {
    int64_t len = 0;
    check(etune_device_profile_to_json(&dev, name.c_str(), nullptr, 0, &len));
    std::string s(size_t(len) + 1, '\0');
    check(etune_device_profile_to_json(&dev, name.c_str(), &s[0], len + 1, &len));
    s.resize(size_t(len));
    return s;
}
inline DeviceConfig device_profile_from_json(const std::string& text, std::string* name = nullptr) {
    DeviceConfig d{};
    std::vector<char> nm(text.size() + 1);
    check(etune_device_profile_from_json(text.data(), int64_t(text.size()), &d, nm.data(), int64_t(nm.size())));
    if (name) *name = nm.data();
    return d;
}

// MeasurementRecord / MeasurementLog / log_append / log_load (measure.hpp:17-83)
struct MeasurementRecord {
    uint64_t candidate_id = 0;
    double latency_ms = 0.0, avg_power_w = 0.0, energy_mj = 0.0;
    int64_t iterations = 0;
    std::string backend, timestamp;
};
class MeasurementLog {
public:
    void add(const MeasurementRecord& r) {
        by_id_[r.candidate_id] = records_.size();
        records_.push_back(r);
    }
    const std::vector<MeasurementRecord>& records() const { return records_; }
    bool contains(uint64_t id) const { return by_id_.count(id) != 0; }
    const MeasurementRecord& lookup(uint64_t id) const {  // most recent record; TraceMiss when absent
        const auto it = by_id_.find(id);
        if (it == by_id_.end())
            throw TraceMiss(ETUNE_ERR_TRACE_MISS, "candidate id " + std::to_string(id) + " is not in the log", -1);
        return records_[it->second];
    }

private:
    std::vector<MeasurementRecord> records_;
    std::map<uint64_t, size_t> by_id_;
};
inline etune_log_record to_log_record(const MeasurementRecord& r) {
    etune_log_record x{};
    x.m.candidate_id = r.candidate_id;
    x.m.latency_ms = r.latency_ms;
    x.m.avg_power_w = r.avg_power_w;
    x.m.energy_mj = r.energy_mj;
    x.m.iterations = r.iterations;
    x.m.feasible = 1;
    std::strncpy(x.backend, r.backend.c_str(), sizeof(x.backend) - 1);
    std::strncpy(x.timestamp, r.timestamp.c_str(), sizeof(x.timestamp) - 1);
    return x;
}
inline void log_append(const std::string& path, const MeasurementRecord& r) {
    const etune_log_record x = to_log_record(r);
    int64_t len = 0;
    check(etune_measurement_log_to_jsonl(&x, 1, nullptr, 0, &len));
    std::string text(size_t(len) + 1, '\0');
    check(etune_measurement_log_to_jsonl(&x, 1, &text[0], len + 1, &len));
    std::ofstream out(path, std::ios::app);
    if (!out) throw IoError(ETUNE_ERR_IO, "cannot append to measurement log '" + path + "'", -1);
    out.write(text.data(), len);
    if (!out) throw IoError(ETUNE_ERR_IO, "failed writing measurement log '" + path + "'", -1);
}
inline MeasurementLog log_load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError(ETUNE_ERR_IO, "cannot open measurement log '" + path + "'", -1);
    std::ostringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();
    etune_log_record* recs = nullptr;
    int64_t n = 0;
    check(etune_measurement_log_from_jsonl(text.data(), int64_t(text.size()), &recs, &n));
    MeasurementLog log;
    for (int64_t i = 0; i < n; ++i) {
        const etune_log_record& x = recs[i];
        log.add(MeasurementRecord{x.m.candidate_id, x.m.latency_ms, x.m.avg_power_w, x.m.energy_mj, x.m.iterations,
                                  std::string(x.backend, strnlen(x.backend, sizeof(x.backend))),
                                  std::string(x.timestamp, strnlen(x.timestamp, sizeof(x.timestamp)))});
    }
    etune_measurement_log_free(recs);
    return log;
}

inline std::vector<Candidate> to_candidates(const Plan& plan, const DeviceBuffer<uint64_t>& g, size_t n) {
    DeviceBuffer<uint64_t> ids(n);
    check(etune_cu_candidate_ids(plan.device().get(), plan.get(), g.get(), int64_t(n), ids.get()));
    const std::vector<Schedule> s = plan.decode(g, n);
    const std::vector<uint64_t> id = ids.download(n);
    std::vector<Candidate> out(n);
    for (size_t i = 0; i < n; ++i) {
        out[i].id = id[i];
        out[i].schedule = s[i];
    }
    return out;
}

// sample_random (space.cpp:170-251)
inline std::vector<Candidate> sample_random(const Plan& plan, int64_t n, uint64_t seed) {
    DeviceBuffer<uint64_t> g(size_t(std::max<int64_t>(n, 1)));
    check(etune_cu_sample_random(plan.device().get(), plan.get(), n, seed, g.get(), nullptr));
    return to_candidates(plan, g, size_t(n));
}

// reproduce (genetic.cpp:137-187), lineage = {base id} or {base id, partner id}
inline std::vector<Candidate> reproduce(const Plan& plan, const std::vector<Candidate>& parents, int64_t n,
                                        const GeneticRates& rates, uint64_t seed) {
    std::vector<Schedule> ps(parents.size());
    for (size_t i = 0; i < parents.size(); ++i) ps[i] = parents[i].schedule;
    DeviceBuffer<uint64_t> pg, out(size_t(std::max<int64_t>(n, 1)));
    plan.encode(ps, pg);
    DeviceBuffer<int32_t> partner(size_t(std::max<int64_t>(n, 1)));
    const etune_status st = etune_cu_reproduce(plan.device().get(), plan.get(), pg.get(), int64_t(parents.size()),
                                               n, &rates, seed, out.get(), partner.get(), nullptr);
    if (st != ETUNE_OK) throw_status(st);
    plan.device().synchronize();
    std::vector<Candidate> kids = to_candidates(plan, out, size_t(n));
    const std::vector<int32_t> pt = partner.download(size_t(n));
    for (int64_t i = 0; i < n; ++i) {
        const Candidate& base = parents[size_t(i) % parents.size()];
        kids[size_t(i)].lineage = {base.id};
        if (pt[size_t(i)] >= 0) kids[size_t(i)].lineage.push_back(parents[size_t(pt[size_t(i)])].id);
    }
    return kids;
}

// k lowest scores under (score asc, index asc) — the selection of SPEC:403-409
inline std::vector<int64_t> select_lowest(Device& dev, const std::vector<double>& score, int64_t k) {
    DeviceBuffer<double> d;
    d.upload(score.data(), score.size());
    DeviceBuffer<int64_t> idx(size_t(std::max<int64_t>(k, 1)));
    check(etune_cu_topk(dev.get(), d.get(), int64_t(score.size()), k, idx.get()));
    dev.synchronize();
    return idx.download(size_t(k));
}

// ------------------------------------------------------------------ search
class Search {  // Algorithm 1: SimBackend, the GPU itself, or a ReplayBackend log
public:
    Search(Plan& plan, const etune_search_config& cfg) : plan_(&plan) {
        check(etune_cu_search_create(plan.device().get(), plan.get(), &cfg, &h_));
    }
    // ReplayBackend (measure.hpp:116-128) for cfg.backend == 2
    void set_replay(const MeasurementLog& log) {
        std::vector<etune_measurement> m;
        m.reserve(log.records().size());
        for (const MeasurementRecord& r : log.records()) m.push_back(to_log_record(r).m);
        check(etune_cu_search_set_replay(h_, m.data(), int64_t(m.size())));
    }
    ~Search() { etune_cu_search_destroy(h_); }
    Search(const Search&) = delete;
    Search& operator=(const Search&) = delete;
    etune_round_report initial_round() {
        etune_round_report r{};
        check(etune_cu_search_initial(h_, &r));
        return r;
    }
    etune_round_report round() {
        etune_round_report r{};
        check(etune_cu_search_round(h_, &r));
        return r;
    }
    std::vector<etune_round_report> run() {
        std::vector<etune_round_report> r(1024);
        int64_t n = 0;
        check(etune_cu_search_run(h_, r.data(), int64_t(r.size()), &n));
        r.resize(size_t(std::min<int64_t>(n, int64_t(r.size()))));
        return r;
    }
    Candidate best(double* latency_ms = nullptr, double* energy_mj = nullptr) const {
        Candidate c;
        check(etune_cu_search_best(h_, &c.schedule, &c.id, latency_ms, energy_mj));
        return c;
    }

private:
    Plan* plan_;
    etune_cu_search* h_ = nullptr;
};

}  // namespace etune_b200
