// Host planner: per-operator knob tables and feature tables (see etune_internal.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "etune_internal.hpp"

namespace etune_b200 {

struct PlanBuild {
    etune_op_spec op{};
    etune_space_limits limits{};
    int num_sms = 108;
    etune_device_config dev{};        // the simulated device (SimBackend)
    PlanHdr hdr{};
    std::vector<uint8_t> blob;  // hdr + tables, 16-byte aligned sections

    // host mirrors (the forest compiler and the exact-mode breeder read these)
    std::vector<int64_t> div[3];      // divisors of B, M, N (space.cpp:57-67)
    std::vector<int64_t> divk;        // divisors of K
    std::vector<TilingRec> til[3];    // enumerate_dim_tilings order (space.cpp:69-78)
    std::vector<int64_t> grid_values; // sorted distinct grid sizes
    std::vector<uint16_t> gridkey;    // [nd0][nd1][nd2]
    std::vector<GridRec> grid;
    std::vector<double> int2;         // [nd1][nd2]
    std::vector<GlbRec> glb2;         // [nd1][nd2]
    std::vector<BlockRec> block;      // [1025]
    std::vector<double> ptn;          // [nd2]
    std::vector<double> steps;        // [ndk]
    double lvl[4] = {0, 0, 0, 0};
    int64_t space_size = 0;           // count_schedules(op, limits)
    std::vector<int64_t> unroll_opts; // powers_of_two_up_to(max(1,max_unroll)) (space.cpp:100)
    std::vector<int64_t> vec_opts;    // powers_of_two_up_to(min(4,max(1,max_vec))) (101-102)
};

// Validates like OperatorSpec::validate (opspec.cpp:65-93) and builds every table.
// Returns ETUNE_OK, ETUNE_ERR_VALIDATION or ETUNE_ERR_UNSUPPORTED (+ message).
etune_status build_plan(const etune_op_spec& op, const etune_device_config& dev,
                        const etune_space_limits& limits, PlanBuild* out, std::string* err);

// LoopNest (opspec.cpp:103-117)
void op_nest(const etune_op_spec& op, int64_t out[4]);
etune_status op_validate(const etune_op_spec& op, std::string* err);

std::vector<int64_t> divisors_of(int64_t e);

}  // namespace etune_b200
