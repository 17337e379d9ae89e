// TEST INFRASTRUCTURE: the reference-side binding (integration/etune/b200_binding.hpp) compiled
// against the reference's own headers and linked with the unmodified reference library
// (oracle/_ref/libetune_ref.so) and libetune_cuda.so.  Run on a B200 by tests/test_gpu_binding.py:
//
//   binding_test <model.json> <op text> <n>
//
// The reference computes every result on the CPU through its public API; the binding computes the
// same on the GPU; every value must be identical.  Prints "binding ok ..." and exits 0.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "etune/b200_binding.hpp"
#include "etune/features.hpp"

using namespace etune;

#define EXPECT(cond, ...)                                     \
    do {                                                      \
        if (!(cond)) {                                        \
            std::fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            std::fprintf(stderr, __VA_ARGS__);                \
            std::fprintf(stderr, "\n");                       \
            return 1;                                         \
        }                                                     \
    } while (0)

static bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: binding_test <model.json> <op> <n>\n");
        return 2;
    }
    std::ifstream in(argv[1]);
    std::stringstream ss;
    ss << in.rdbuf();
    const EnergyModel model = EnergyModel::from_json(ss.str());
    const OperatorSpec op = parse_operator(argv[2]);
    const std::int64_t n = std::atoll(argv[3]);
    const DeviceConfig dev = DeviceConfig::a100_like();

    // the reference's population: reproduce(sample_random(op, 1024, 42), n, {}, 7)
    const std::vector<Candidate> parents = sample_random(op, 1024, 42);
    const std::vector<Candidate> pop = reproduce(parents, n, GeneticRates{}, 7);

    b200::Engine eng(0);
    b200::Model m(eng, model);

    // 1. predict_many == the reference's predict(extract_features) for every candidate
    const std::vector<double> got = eng.predict_many(m, op, dev, pop);
    std::vector<double> ref(pop.size());
    for (size_t i = 0; i < pop.size(); ++i) ref[i] = model.predict(extract_features(op, pop[i].schedule, dev));
    for (size_t i = 0; i < pop.size(); ++i)
        EXPECT(same_bits(got[i], ref[i]), "prediction %zu: %.17g vs %.17g", i, got[i], ref[i]);

    // 2. keep_best == partial_sort by (prediction, index)
    const size_t k = 1024;
    std::vector<double> pred2;
    const std::vector<size_t> best = eng.keep_best(m, op, dev, pop, k, &pred2);
    std::vector<size_t> order(pop.size());
    std::iota(order.begin(), order.end(), size_t(0));
    std::partial_sort(order.begin(), order.begin() + k, order.end(),
                      [&](size_t a, size_t b) { return ref[a] < ref[b] || (ref[a] == ref[b] && a < b); });
    for (size_t j = 0; j < k; ++j) EXPECT(best[j] == order[j], "top-%zu position %zu: %zu vs %zu", k, j, best[j], order[j]);
    for (size_t i = 0; i < pop.size(); ++i) EXPECT(same_bits(pred2[i], ref[i]), "keep_best prediction %zu", i);

    // 3. the same model again (cached plan, compiled row table): still identical
    const std::vector<double> again = eng.predict_many(m, op, dev, pop);
    for (size_t i = 0; i < pop.size(); ++i) EXPECT(same_bits(again[i], ref[i]), "second call, prediction %zu", i);

    // 4. reproduce on the device == etune::reproduce: schedules, ids, lineage
    const std::vector<Candidate> kids_ref = reproduce(parents, 20000, GeneticRates{}, 9);
    const std::vector<Candidate> kids = eng.reproduce(parents, 20000, GeneticRates{}, 9);
    for (size_t i = 0; i < kids.size(); ++i) {
        EXPECT(kids[i].id == kids_ref[i].id, "offspring %zu id", i);
        EXPECT(std::memcmp(&kids[i].schedule, &kids_ref[i].schedule, sizeof(Schedule)) == 0, "offspring %zu", i);
        EXPECT(kids[i].lineage == kids_ref[i].lineage, "offspring %zu lineage", i);
    }

    // 5. sample_random on the device == etune::sample_random
    const std::vector<Candidate> smp_ref = sample_random(op, 4096, 5);
    const std::vector<Candidate> smp = eng.sample_random(op, 4096, 5);
    for (size_t i = 0; i < smp.size(); ++i) {
        EXPECT(smp[i].id == smp_ref[i].id, "sample %zu id", i);
        EXPECT(std::memcmp(&smp[i].schedule, &smp_ref[i].schedule, sizeof(Schedule)) == 0, "sample %zu", i);
    }

    // 6. an illegal schedule throws the reference's IllegalSchedule naming the element
    std::vector<Candidate> bad = pop;
    bad[123].schedule.k_tile = 7;
    bool threw = false;
    try {
        eng.predict_many(m, op, dev, bad);
    } catch (const IllegalSchedule& e) {
        threw = std::string(e.what()).find("(element 123)") != std::string::npos;
    }
    EXPECT(threw, "IllegalSchedule with the element index");

    // 7. every status maps to its reference exception class
    struct Case {
        etune_status st;
        const char* cls;
    } cases[] = {{ETUNE_ERR_PARSE, "ParseError"},          {ETUNE_ERR_VALIDATION, "ValidationError"},
                 {ETUNE_ERR_SPACE_EXHAUSTED, "SpaceExhausted"}, {ETUNE_ERR_ILLEGAL_SCHEDULE, "IllegalSchedule"},
                 {ETUNE_ERR_TOO_LARGE, "TooLarge"},          {ETUNE_ERR_NON_POSITIVE_ENERGY, "NonPositiveEnergy"},
                 {ETUNE_ERR_INSUFFICIENT_DATA, "InsufficientData"}, {ETUNE_ERR_SCHEMA_MISMATCH, "SchemaMismatch"},
                 {ETUNE_ERR_VERSION_MISMATCH, "VersionMismatch"}, {ETUNE_ERR_LENGTH_MISMATCH, "LengthMismatch"},
                 {ETUNE_ERR_EMPTY_INPUT, "EmptyInput"},      {ETUNE_ERR_IO, "IoError"},
                 {ETUNE_ERR_CONSISTENCY, "ConsistencyError"}, {ETUNE_ERR_BACKEND_UNAVAILABLE, "BackendUnavailable"},
                 {ETUNE_ERR_TRACE_MISS, "TraceMiss"}};
    for (const Case& c : cases) {
        std::string caught;
        try {
            b200::rethrow(c.st);
        } catch (const ParseError&) { caught = "ParseError"; }
        catch (const ValidationError&) { caught = "ValidationError"; }
        catch (const SpaceExhausted&) { caught = "SpaceExhausted"; }
        catch (const IllegalSchedule&) { caught = "IllegalSchedule"; }
        catch (const TooLarge&) { caught = "TooLarge"; }
        catch (const NonPositiveEnergy&) { caught = "NonPositiveEnergy"; }
        catch (const InsufficientData&) { caught = "InsufficientData"; }
        catch (const SchemaMismatch&) { caught = "SchemaMismatch"; }
        catch (const VersionMismatch&) { caught = "VersionMismatch"; }
        catch (const LengthMismatch&) { caught = "LengthMismatch"; }
        catch (const EmptyInput&) { caught = "EmptyInput"; }
        catch (const IoError&) { caught = "IoError"; }
        catch (const ConsistencyError&) { caught = "ConsistencyError"; }
        catch (const BackendUnavailable&) { caught = "BackendUnavailable"; }
        catch (const TraceMiss&) { caught = "TraceMiss"; }
        EXPECT(caught == c.cls, "status %d -> %s, expected %s", int(c.st), caught.c_str(), c.cls);
    }
    std::printf("binding ok: %lld candidates of %s, top-%zu, 20000 offspring, 4096 samples identical to the reference\n",
                static_cast<long long>(n), argv[2], k);
    return 0;
}
