// Forest compiler: reference TreeNode arrays -> (a) generic predict blob,
// (b) per-plan score blob (rank bins + partially evaluated perfect trees).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "etune_internal.hpp"
#include "plan.hpp"

namespace etune_b200 {

struct ForestHost {
    std::vector<int32_t> feature, left, right;
    std::vector<double> threshold, value;
    std::vector<int64_t> offsets;  // num_trees + 1
    double base = 0.0, lr = 0.0;
    int64_t num_trees() const { return int64_t(offsets.size()) - 1; }
};

etune_status forest_validate(const ForestHost& F, std::string* err);
etune_status build_predict_blob(const ForestHost& F, std::vector<uint8_t>* blob, std::string* err);

struct ScoreStats {
    int64_t internal_nodes_in = 0;   // reference interior nodes
    int64_t tests_folded = 0;        // tests resolved at compile time for this op
    int64_t lut_entries = 0;         // class->mask entries referenced by trees
    int max_leaves = 0;
    int total_leaves = 0;
    int channels_used = 0;           // bitmask of channels still tested after folding
};
// Keyed form (KeyedHdr): built alongside the score blob when every tree has <= 32 leaves
// and the key table fits `max_table_bytes`; `ok` false otherwise.
struct KeyedBuild {
    bool ok = false;
    std::vector<uint8_t> blob;
    std::vector<uint8_t> table;   // [nkeys][row_bytes]
    std::vector<uint64_t> khash;  // [nkeys]: FNV-1a state after the operator words and the key's tilings
    KeyedParams params{};
    int64_t nkeys = 0;
    int key_bits = 0;
};
etune_status build_score_blob(const ForestHost& F, const PlanBuild& P, std::vector<uint8_t>* blob,
                              ScoreStats* stats, std::string* err, KeyedBuild* keyed = nullptr,
                              size_t max_table_bytes = size_t(64) << 20, size_t max_full_bytes = size_t(64) << 20);

}  // namespace etune_b200
