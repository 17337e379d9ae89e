// Host-side launchers for the sm_100a kernels (kernels.cu, sort.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "etune_internal.hpp"

namespace etune_b200 {

struct LaunchCtx {
    cudaStream_t stream;
    int sm_count;                 // physical SMs of the GPU (148 on B200)
    unsigned long long* d_err;    // packed (index << 8 | status), min wins
};

// d_err sentinel: no error
constexpr unsigned long long kNoError = ~0ull;

cudaError_t launch_encode(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                          const etune_schedule* d_sched, int64_t n, uint64_t* d_genome,
                          int64_t index_base = 0);
// encode from host-narrowed rows: 12 fields of field_bytes (2, 4; 8 = the reference layout)
cudaError_t launch_encode_packed(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const void* d_rows,
                                 int field_bytes, int64_t n, uint64_t* d_genome, int64_t index_base);
cudaError_t launch_decode(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                          const uint64_t* d_genome, int64_t n, etune_schedule* d_sched);
cudaError_t launch_ids(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                       const uint64_t* d_genome, int64_t n, uint64_t* d_ids);
cudaError_t launch_counters(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                            const uint64_t* d_genome, int64_t n, etune_counters* d_out);
// SimBackend (measure.hpp:29-60, 102-114): latency only when pow/en/iters are null.
struct SimDevice {
    double tput, bw, floor_ms, e_flop, e_glb, e_shared, constant, static_sm, hz, sigma;
    uint64_t seed;
};
cudaError_t launch_sim_measure(const LaunchCtx& c, const uint8_t* d_plan, uint32_t bytes, const uint64_t* d_genome,
                               int64_t n, const SimDevice& d, double* d_lat, double* d_pow, double* d_en,
                               int64_t* d_iters);
cudaError_t launch_features(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                            const uint64_t* d_genome, int64_t n, double* d_feat, uint64_t* d_ids);
// Fused selection (score_select): the score kernel also counts every prediction into
// kSelBins buckets of its order-preserving key.  The bucket function is monotone
// (keys below kmin -> 0, above the range -> last bucket), so it is exact for any
// bounds; the forest's leaf-value bounds only decide how finely the buckets resolve.
constexpr int kSelBins = 1024;
constexpr int kSelMaxK = 4096;  // one-CTA final sort bound
struct SelHist {
    uint32_t* hist;  // kSelBins global counters (null: no histogram)
    uint64_t kmin;
    uint32_t shift;
};
// resident CTAs per SM of the compiled score kernel for a blob size (sets the smem ceiling)
cudaError_t score_occupancy(int mask_bits, uint32_t bytes, int* per_sm);
// static shared memory the score kernel holds besides the compiled blob
int score_static_smem();
cudaError_t launch_score(const LaunchCtx& c, const uint8_t* d_score, uint32_t score_bytes,
                         const uint64_t* d_genome, int64_t n, double* d_pred, uint64_t* d_ids,
                         int mask_bits, const ForestParams& fp, int per_sm, const SelHist& sel = SelHist{});
// Keyed score path (KeyedHdr / KeyedParams): one byte per (tiling-triple key, tree)
// from the key table; results at the original index (d_order nullable).  d_khash: per key,
// the FNV-1a state after the operator words and the key's three tiling records.
cudaError_t score_keyed_occupancy(uint32_t bytes, int* per_sm);
cudaError_t launch_score_keyed(const LaunchCtx& c, const uint8_t* d_kblob, uint32_t bytes, const uint8_t* d_table,
                               size_t table_bytes, const uint64_t* d_khash, const uint64_t* d_genome,
                               const uint32_t* d_order, int64_t n,
                               double* d_pred, uint64_t* d_ids, int per_sm, const KeyedParams& kp,
                               const SelHist& sel = SelHist{});
// Selection from the histogram the score kernel filled: filter (keys below the k-th
// key's bucket + the bucket itself) -> one-CTA radix select inside the bucket and
// (key, index) sort of the k.  Leaves the histogram zeroed for the next call.
// Scratch from select_scratch_bytes(n, k); zero it once (cudaMemset) after allocation.
size_t select_scratch_bytes(int64_t n, int64_t k);
uint32_t* select_hist(void* d_sel);
cudaError_t launch_select(const LaunchCtx& c, const double* d_score, int64_t n, int64_t k, int64_t* d_idx,
                          void* d_sel, const SelHist& sel);
// General path: features + reference tree walk (any forest the reference can train).
cudaError_t launch_score_walk(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint8_t* d_pred,
                              uint32_t pred_bytes, const uint64_t* d_genome, int64_t n, double* d_out,
                              uint64_t* d_ids);
cudaError_t launch_predict(const LaunchCtx& c, const uint8_t* d_pred_blob, uint32_t bytes,
                           const double* d_feat, int64_t n, double* d_pred);

// (score asc, index asc) top-k; scratch sized by topk_scratch_bytes(n).
size_t topk_scratch_bytes(int64_t n);
cudaError_t launch_topk(const LaunchCtx& c, const double* d_score, int64_t n, int64_t k,
                        int64_t* d_idx, void* d_scratch);

// reproduce (genetic.cpp:137-187): one CTA resolves the RNG-offset chain by speculation
// and writes offspring genomes (+ crossover partner index, -1 otherwise).
size_t breed_state_bytes();
cudaError_t launch_breed(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint64_t* d_par,
                         const uint64_t* d_pid, int64_t np, int64_t n, double mut, double cro, double cpy,
                         uint64_t seed, uint64_t* d_out, int32_t* d_partner, void* d_state);

// EnergyModel::train (energy_model.cpp:173-243), bit-exact; scratch from train_scratch_bytes(n).
size_t train_scratch_bytes(int64_t n);
int train_max_depth();
cudaError_t launch_train(const LaunchCtx& c, const double* d_feat, const double* d_energy, int64_t n, int num_trees,
                         int max_depth, double lr, double mlw, double lambda, int32_t* o_feature, double* o_thr,
                         int32_t* o_left, int32_t* o_right, double* o_value, int64_t* o_off, double* o_scalars,
                         double* o_loss, void* scratch);

// energy_loss (Eq. 1) per sample -> out[3*i..] = {value, gradient, hessian}
cudaError_t launch_energy_loss(const LaunchCtx& c, const double* d_pred, const double* d_meas, int64_t n,
                               double* d_out3);
// snr_db's sequential sums {signal, error}
cudaError_t launch_snr_sums(const LaunchCtx& c, const double* d_pred, const double* d_meas, int64_t n,
                            double* d_out2);

// sharded selection helpers (model.cu): records of the local top-k (padded to k with
// +inf / INT64_MAX), and the final gather of (gidx, score) by merged positions
cudaError_t launch_pack_records(const LaunchCtx& c, const double* d_score, const int64_t* d_lidx, int64_t kl,
                                int64_t k, int64_t goff, double* d_rs, int64_t* d_rg);
cudaError_t launch_gather_records(const LaunchCtx& c, const double* d_gs, const int64_t* d_gg, const int64_t* d_pos,
                                  int64_t k, int64_t* d_idx, double* d_sc);

// stable LSD radix sort of (u64 key, u32 value) pairs by the low `bits` bits, in place
size_t sort_pairs_scratch_bytes(int64_t n);
cudaError_t launch_sort_pairs(const LaunchCtx& c, uint64_t* keys, uint32_t* vals, int64_t n, int bits,
                              void* scratch);

// sample_random (space.cpp:170-251): large-space attempts / small-space enumerate + Fisher-Yates.
// Scratch: sample_scratch_bytes(attempts, 0, false) / (n, odometer product, true).
size_t sample_scratch_bytes(int64_t n, int64_t space_or_product, bool small);
cudaError_t launch_sample_large(const LaunchCtx& c, const uint8_t* d_plan, uint64_t seed, int64_t n, int64_t A,
                                uint64_t* d_out, int64_t* d_found, int* d_flags, void* scratch);
cudaError_t launch_sample_small(const LaunchCtx& c, const uint8_t* d_plan, const int64_t dims[6], uint64_t seed,
                                int64_t n, uint64_t* d_out, int64_t* d_found, int* d_flags, void* scratch);

// dst[j] = src[idx[j]] for 8-byte elements (genomes, doubles); y = x / *divisor
cudaError_t launch_gather_u64(const LaunchCtx& c, const void* d_src, const int64_t* d_idx, int64_t n, void* d_dst);
cudaError_t launch_div_scalar(const LaunchCtx& c, const double* d_x, int64_t n, const double* d_divisor, double* d_y);

// measurement harness (harness.cu): candidate GEMM/conv kernel per Schedule + NVML energy
bool nvml_available(std::string* why);
void* nvml_device_handle(int cuda_device, std::string* why);
bool nvml_energy_mj(void* handle, unsigned long long* mj);
bool nvml_power_mw(void* handle, unsigned int* mw);
size_t candidate_geom_bytes();
bool candidate_geometry(const etune_op_spec& op, const int64_t nest[4], const etune_schedule& s, int smem_cap,
                        void* out_geom, size_t* smem, int* grid, int* block);
bool candidate_fits(const void* geom, int block);
cudaError_t launch_candidate(cudaStream_t st, const void* geom, size_t smem, int grid, int block, const float* A,
                             const float* B, float* C);
cudaError_t launch_fill(cudaStream_t st, float* x, int64_t n, uint32_t seed);

// process-wide count of kernel launches (incremented by every launcher)
void note_launches(int k);
uint64_t launch_count();

// Largest dynamic smem the score kernel may use on this device.
int max_dynamic_smem(int device);

}  // namespace etune_b200
