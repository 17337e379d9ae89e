// Handle definitions shared by the C ABI (capi.cpp) and the host search driver
// (search.cpp).  Not part of the public interface.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <utility>
#include <vector>

#include "forest.hpp"
#include "host_pool.hpp"
#include "kernels.hpp"
#include "plan.hpp"

struct etune_cu_ctx {
    std::atomic<int> refs{0};        // live plans / forests / searches
    std::atomic<bool> closing{false};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 0;
    unsigned long long* d_err = nullptr;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    // staging for the *_host path
    void* io = nullptr;
    size_t io_bytes = 0;
    void* breed = nullptr;  // BreedState + parent ids
    size_t breed_bytes = 0;
    void* breedpar = nullptr;  // block-parallel exact reproduce work area (breed_par.cu)
    size_t breedpar_bytes = 0;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    etune_transport transport{};  // caller's collectives when no NCCL communicator is attached
    bool has_transport = false;
    void* shard = nullptr;  // sharded-selection records
    size_t shard_bytes = 0;
    void* e2e = nullptr;    // score_select_host: the population's predictions + the k indices on the device
    size_t e2e_bytes = 0;
    void* rowsel = nullptr; // row-table score_select work area (RowSelWork, rowtab.cu), zeroed once
    void* sel = nullptr;    // fused score_select work area (histogram, bucket lists)
    size_t sel_bytes = 0;
    bool sel_dirty = false; // a score_select sequence did not complete: re-zero first
    // optional device timing of the score kernel inside score_select (bench / profiling)
    bool prof_on = false;
    std::vector<std::array<cudaEvent_t, 4>> prof_ev;  // start, before score, after score, after select
    size_t prof_used = 0;
    // *_host pipelines: pinned staging of narrowed Schedule rows, packed by a host pool
    void* hpin = nullptr;
    size_t hpin_bytes = 0;
    void* hout = nullptr;  // pinned staging of outputs bound for pageable caller memory
    size_t hout_bytes = 0;
    std::unique_ptr<etune_b200::HostPool> pool;
    // *_host pipelines: copy-in / copy-out streams and per-buffer events
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    // forests alive on this ctx: a destroyed plan evicts its compiled forms from each of them
    std::mutex forests_mu;
    std::set<etune_cu_forest*> forests;
    etune_b200::LaunchCtx lc() const { return etune_b200::LaunchCtx{stream, sm_count, d_err}; }
};

namespace etune_b200 {
void ctx_retain(etune_cu_ctx* c);
void ctx_release(etune_cu_ctx* c);
// collectives over the ctx's ranks (capi.cpp): NCCL, else the attached transport, else one rank
int ctx_world(const etune_cu_ctx* c);
int ctx_rank(const etune_cu_ctx* c);
etune_status coll_allgather(etune_cu_ctx* c, const void* d_send, void* d_recv, size_t bytes);
etune_status coll_broadcast(etune_cu_ctx* c, void* d_buf, size_t bytes, int root);
}  // namespace etune_b200

struct etune_cu_plan {
    etune_cu_ctx* ctx = nullptr;
    etune_b200::PlanBuild build;
    uint8_t* d_blob = nullptr;
    uint64_t serial = 0;
    // row-table form (rowtab.cu): per tiling-triple key the FNV-1a state of candidate_id after
    // the operator and the three tilings; rows_cap = keys x legal (k_tile, unroll, vec) triples
    // (0: the operator's row table would be too large, the form is not offered)
    uint64_t* d_khash = nullptr;  // per key: after the three tilings
    uint64_t* d_khk = nullptr;    // per (key, k_tile index): after k_tile as well
    int64_t nkeys = 0, kuv_domain = 0, rows_cap = 0;
};

// Row-table form of one (forest, plan): Kuv class table, class representatives, row
// predictions and the selection bounds, all written on the device (rowtab.cu).
struct RowTab {
    etune_b200::RowTabMeta* d_meta = nullptr;
    uint16_t* d_clskuv = nullptr;
    uint32_t* d_crep = nullptr;
    double* d_rowpred = nullptr;
    uint32_t* d_srows = nullptr;   // rows in prediction order (ties by row)
    uint32_t* d_rowgid = nullptr;  // a row's group: the dense rank of its prediction
    etune_b200::RowRec* d_rowrec = nullptr;  // {prediction, group} per row: the fused selection's gather
};

struct CompiledScore {
    bool walk = false;        // compiled form unsupported / too large: general tree-walk kernel
    uint8_t* d_blob = nullptr;
    uint32_t bytes = 0;
    int mask_bits = 32;
    int per_sm = 1;           // resident CTAs per SM (queried once at compile time)
    std::shared_ptr<etune_b200::ForestParams> params;  // tree records, passed by value to the kernel
    uint64_t sel_kmin = 0;    // fused selection buckets: order key of the lowest possible
    uint32_t sel_shift = 0;   // prediction, and the key bits one bucket spans
    // keyed form (forest.hpp KeyedBuild): blob, key table, sort key width, occupancy
    bool keyed = false, keyed_tried = false;
    uint8_t* d_kblob = nullptr;
    uint32_t kbytes = 0;
    uint8_t* d_ktable = nullptr;
    uint64_t* d_khash = nullptr;  // per key: FNV-1a state after the operator and the three tilings
    size_t ktable_bytes = 0;
    std::shared_ptr<etune_b200::KeyedParams> kparams;
    int key_bits = 0, nkeys = 0, nt1 = 0, nt2 = 0, keyed_per_sm = 1;
    etune_b200::ScoreStats stats;
};

struct etune_cu_forest {
    etune_cu_ctx* ctx = nullptr;
    etune_b200::ForestHost host;
    uint8_t* d_predict = nullptr;
    uint32_t predict_bytes = 0;
    int nnodes = 0;
    std::mutex mu;
    std::map<uint64_t, CompiledScore> compiled;  // by plan serial (host-compiled class / keyed forms)
    std::map<uint64_t, RowTab> rowtabs;          // by plan serial (device-compiled row tables)
    std::map<uint64_t, int64_t> seen;            // by plan serial: candidates scored so far (AUTO form)
    int form = ETUNE_FORM_AUTO;
    int keyed_mode = 1;  // 1: keyed path (full form when it fits), 2: keyed byte form only, 0: class tables only
    // Lazy compile (set on the search loop's per-round models, each scored once): small
    // populations take the tree-walk kernel until kLazyWalkBudget candidates per plan
    // have been walked, instead of paying the ms-scale host compile per model.
    bool lazy_compile = false;
    std::map<uint64_t, int64_t> walked;  // by plan serial
};

