// The C++ host mirror (include/etune_b200.hpp) exercised like the reference's own API:
// etune::-named calls on host vectors, checked against the CPU oracle (oracle/lib,
// test infrastructure).  Run on a B200 by tests/test_gpu_mirror.py; prints MIRROR OK.
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/etune_b200.hpp"
#include "../../oracle/etune_oracle.h"

using namespace etune_b200;

static int failures = 0;
#define EXPECT(cond)                                                         \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);      \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

static std::vector<int64_t> words(const OperatorSpec& op) {
    const int64_t* p = &op.kind;
    return std::vector<int64_t>(p, p + 12);
}
static std::vector<int64_t> rows(const std::vector<Schedule>& s) {
    std::vector<int64_t> out(s.size() * 12);
    std::memcpy(out.data(), s.data(), out.size() * 8);
    return out;
}
static bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

int main() {
    Device dev(0);
    const OperatorSpec op = make_conv(1, 56, 56, 64, 64, 3, 1, 1);  // BASELINE configs[1]
    Plan plan(dev, op);
    const auto opw = words(op);
    const int64_t lim[3] = {1024, 8, 4};

    // sample_random == reference order (space.cpp:170-251)
    const int64_t n = 4096;
    std::vector<Candidate> pop = sample_random(plan, n, 1234);
    std::vector<int64_t> osched(size_t(n) * 12);
    std::vector<uint64_t> oids(static_cast<size_t>(n));
    EXPECT(orc_sample_random(opw.data(), n, 1234, lim, osched.data(), oids.data()) == 0);
    std::vector<Schedule> sched(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        sched[size_t(i)] = pop[size_t(i)].schedule;
        EXPECT(pop[size_t(i)].id == oids[size_t(i)]);
    }
    EXPECT(std::memcmp(osched.data(), sched.data(), osched.size() * 8) == 0);

    // extract_features (features.cpp:48-51)
    const std::vector<FeatureVector> feats = extract_features(plan, sched);
    std::vector<double> of(size_t(n) * 16);
    EXPECT(orc_features(opw.data(), rows(sched).data(), n, 108, of.data()) == 0);
    EXPECT(std::memcmp(of.data(), feats.data(), of.size() * 8) == 0);
    EXPECT(candidate_id(plan, sched[7]) == oids[7]);

    // EnergyModel::train on device == oracle (energies: a smooth positive function)
    std::vector<EnergySample> samples(static_cast<size_t>(n));
    std::vector<double> energy(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        samples[size_t(i)].features = feats[size_t(i)];
        energy[size_t(i)] = 1.0 + 0.3 * feats[size_t(i)][2] + 0.1 * feats[size_t(i)][13] + 0.01 * double(i % 7);
        samples[size_t(i)].measured_energy_mj = energy[size_t(i)];
    }
    BoostParams bp = default_boost();
    bp.num_trees = 40;
    const EnergyModel model = EnergyModel::train(dev, samples, bp);
    const size_t cap = size_t(bp.num_trees) * 127;
    std::vector<int32_t> fe(cap), le(cap), ri(cap);
    std::vector<double> th(cap), va(cap), loss(size_t(bp.num_trees) + 1);
    std::vector<int64_t> off(size_t(bp.num_trees) + 1);
    double base = 0, ref = 0;
    EXPECT(orc_train(of.data(), energy.data(), n, bp.num_trees, bp.max_depth, bp.learning_rate, bp.min_leaf_weight,
                     bp.reg_lambda, fe.data(), th.data(), le.data(), ri.data(), va.data(), off.data(), &base, &ref,
                     loss.data()) == 0);
    EXPECT(model.tree_offsets() == off);
    const size_t nn = size_t(off.back());
    for (size_t i = 0; i < nn; ++i) {
        EXPECT(model.node_feature()[i] == fe[i]);
        EXPECT(same_bits(model.node_threshold()[i], th[i]));
        EXPECT(same_bits(model.node_value()[i], va[i]));
    }
    EXPECT(same_bits(model.base_score(), base));
    EXPECT(same_bits(model.reference_energy_mj(), ref));
    for (size_t t = 0; t < loss.size(); ++t) EXPECT(same_bits(model.training_loss_per_round()[t], loss[t]));

    // predict_many / score (energy_model.cpp:245-257) == oracle predict
    std::vector<double> want(static_cast<size_t>(n));
    EXPECT(orc_predict(fe.data(), th.data(), le.data(), ri.data(), va.data(), off.data(), bp.num_trees, base,
                       bp.learning_rate, of.data(), n, want.data()) == 0);
    const std::vector<double> p1 = model.predict_many(feats);
    const std::vector<double> p2 = model.score(plan, sched);
    for (int64_t i = 0; i < n; ++i) {
        EXPECT(same_bits(p1[size_t(i)], want[size_t(i)]));
        EXPECT(same_bits(p2[size_t(i)], want[size_t(i)]));
    }
    EXPECT(same_bits(model.predict(feats[3]), want[3]));

    // persistence (energy_model.cpp:259-420, device.cpp:44-101): save -> load round trips
    {
        const std::string mp = "/tmp/etune_mirror_model.json", sp = "/tmp/etune_mirror_samples.jsonl";
        model.save(mp);
        const EnergyModel back = EnergyModel::load(dev, mp);
        EXPECT(back.to_json() == model.to_json());
        const std::vector<double> p3 = back.predict_many(feats);
        for (int64_t i = 0; i < n; ++i) EXPECT(same_bits(p3[size_t(i)], want[size_t(i)]));
        save_energy_samples(samples, sp);
        const std::vector<EnergySample> sb = load_energy_samples(sp);
        EXPECT(sb.size() == samples.size());
        for (size_t i = 0; i < sb.size(); ++i) {
            EXPECT(std::memcmp(sb[i].features.data(), samples[i].features.data(), 128) == 0);
            EXPECT(same_bits(sb[i].measured_energy_mj, samples[i].measured_energy_mj));
        }
        std::string nm;
        const DeviceConfig d2 = device_profile_from_json(device_profile_to_json(a100_like(), "dev"), &nm);
        EXPECT(nm == "dev" && d2.num_sms == 108 && same_bits(d2.constant_power_w, 60.0));
        bool threw = false;
        try {
            EnergyModel::from_json(dev, "{\"model_version\":\"v0\"}");
        } catch (const VersionMismatch&) {
            threw = true;
        }
        EXPECT(threw);
        std::remove(mp.c_str());
        std::remove(sp.c_str());
        // MeasurementLog (measure.hpp:63-83): append -> load keeps every record; lookup returns
        // the most recent record of an id; an unknown id throws TraceMiss
        const std::string lp = "/tmp/etune_mirror_measurements.jsonl";
        std::remove(lp.c_str());
        MeasurementRecord r1{12345678901234567890ull, 0.0347, 239.0, 239.0 * 0.0347, 1000, "sim", "2026-10-17T00:00:00Z"};
        MeasurementRecord r2 = r1;
        r2.latency_ms = 0.05;
        r2.energy_mj = r2.avg_power_w * r2.latency_ms;
        log_append(lp, r1);
        log_append(lp, r2);
        const MeasurementLog lg = log_load(lp);
        EXPECT(lg.records().size() == 2 && lg.contains(r1.candidate_id));
        EXPECT(same_bits(lg.lookup(r1.candidate_id).latency_ms, 0.05) && lg.records()[0].backend == "sim");
        threw = false;
        try {
            lg.lookup(7);
        } catch (const TraceMiss&) {
            threw = true;
        }
        EXPECT(threw);
        std::remove(lp.c_str());
    }

    // snr_db
    std::vector<double> meas(energy.begin(), energy.begin() + 100), pr(want.begin(), want.begin() + 100);
    double osnr = 0;
    EXPECT(orc_snr_db(pr.data(), meas.data(), 100, &osnr) == 0);
    EXPECT(same_bits(snr_db(dev, pr, meas), osnr));

    // reproduce (genetic.cpp:137-187) incl. lineage
    std::vector<Candidate> parents(pop.begin(), pop.begin() + 256);
    const std::vector<Candidate> kids = reproduce(plan, parents, 5000, default_rates(), 7);
    std::vector<int64_t> ks(5000 * 12);
    std::vector<uint64_t> kid(5000), lin(10000);
    std::vector<int8_t> ll(5000);
    const double rates[3] = {0.85, 0.10, 0.05};
    std::vector<int64_t> prow = rows(std::vector<Schedule>(sched.begin(), sched.begin() + 256));
    EXPECT(orc_reproduce(opw.data(), prow.data(), 256, 5000, rates, 7, lim, ks.data(), kid.data(), lin.data(),
                         ll.data()) == 0);
    for (int i = 0; i < 5000; ++i) {
        EXPECT(kids[size_t(i)].id == kid[size_t(i)]);
        EXPECT(int(kids[size_t(i)].lineage.size()) == ll[size_t(i)]);
        for (size_t j = 0; j < kids[size_t(i)].lineage.size(); ++j)
            EXPECT(kids[size_t(i)].lineage[j] == lin[size_t(i) * 2 + j]);
    }

    // selection order and errors behave like the reference's exceptions
    const std::vector<int64_t> top = select_lowest(dev, want, 10);
    std::vector<int64_t> otop(10);
    EXPECT(orc_topk(want.data(), n, 10, otop.data()) == 0);
    EXPECT(top == otop);
    std::vector<Schedule> bad(sched.begin(), sched.begin() + 50);
    bad[17].unroll = 3;
    bool threw = false;
    try {
        extract_features(plan, bad);
    } catch (const IllegalSchedule& e) {
        threw = e.index() == 17;
    }
    EXPECT(threw);
    threw = false;
    try {
        EnergyModel::train(dev, std::vector<EnergySample>{samples[0]}, bp);
    } catch (const InsufficientData&) {
        threw = true;
    }
    EXPECT(threw);

    // Algorithm 1 through the mirror
    etune_search_config cfg;
    etune_default_search_config(&cfg);
    cfg.M = 64;
    cfg.generation_size = 256;
    cfg.max_rounds = 3;
    Search search(plan, cfg);
    const auto reports = search.run();
    EXPECT(reports.size() == 4);
    double lat = 0, en = 0;
    const Candidate best = search.best(&lat, &en);
    EXPECT(best.id == reports.back().best_id && en == reports.back().best_energy_mj);

    std::printf(failures ? "MIRROR FAILED (%d)\n" : "MIRROR OK\n", failures);
    return failures ? 1 : 0;
}
