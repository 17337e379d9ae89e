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
constexpr int kSelBins = 1024;  // selbin.cuh derives the bucket shift from this being 2^10
constexpr int kSelMaxK = 4096;  // one-CTA final sort bound
struct SelHist {
    uint32_t* hist;  // kSelBins global counters (null: no histogram)
    uint64_t kmin;
    uint32_t shift;
    // non-null: the bounds are device-resident {lowest, highest order key} written by an
    // earlier kernel (the row-table build); kmin / shift are derived from them on the
    // device (sel_resolve, plan_core.cuh) after the kernel's dependency wait
    const uint64_t* dbounds = nullptr;
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
// Row-table form (rowtab.cu): the prediction as a function of (tiling-triple key, Kuv class),
// compiled on the device from the plan and the forest's predict blob.
struct RowTabMeta {
    uint64_t bounds[2];  // lowest / highest order key of the row predictions (SelHist::dbounds)
    int32_t nkc;         // Kuv classes = rows per key
    int32_t nthr[3];     // thresholds the forest tests on f10, f7, f6
    int64_t rows;        // keys x nkc
    int64_t groups;      // distinct row predictions (dense ranks 0 .. groups-1)
};
// the fused selection's per-row record: prediction and group (dense rank of the prediction)
struct RowRec {
    double pred;
    uint32_t gid, pad;
};
static_assert(sizeof(RowRec) == 16, "one 16-byte gather per candidate");
// rows per key before class compression: the legal (k_tile, unroll, vectorize) triples
int64_t rowtab_kuv_domain(const int64_t* divk, int ndk);
size_t rowtab_scratch_bytes(int nnodes);
// candidate_id's FNV state per (tiling-triple key, k_tile index) after k_tile (d_khk, nkeys * ndk)
// and per key after the three tilings (d_khash, nkeys)
cudaError_t launch_key_hash(const LaunchCtx& c, const uint8_t* d_plan, int64_t nkeys, uint64_t* d_khk,
                            uint64_t* d_khash);
// d_clskuv: ndk * 64 u16; d_crep: one u32 per class (<= rowtab_kuv_domain); d_rowpred: rows_cap doubles
cudaError_t launch_rowtab_compile(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes,
                                  const uint8_t* d_pred, uint32_t pred_bytes, int nnodes, int ndk, int64_t rows_cap,
                                  void* d_scratch, RowTabMeta* d_meta, uint16_t* d_clskuv, uint32_t* d_crep,
                                  double* d_rowpred);
// Rows in prediction order and each row's group (dense rank of its prediction) for the fused
// selection: d_srows[p] = the row at position p, d_rowgid[row] = its group, both rows_cap u32;
// scratch rowtab_sort_scratch_bytes(rows_cap).
size_t rowtab_sort_scratch_bytes(int64_t rows_cap);
cudaError_t launch_rowtab_sort(const LaunchCtx& c, RowTabMeta* d_meta, const double* d_rowpred, int64_t rows_cap,
                               uint32_t* d_srows, uint32_t* d_rowgid, RowRec* d_rowrec, void* d_scratch);
// Fused score + keep-the-best on the row table in ONE cooperative kernel (rowtab.cu): every
// candidate's prediction and id, group counts, the k-th group, ties by index, the k sorted by
// (prediction, index).  0 < k <= kSelMaxK; returns cudaErrorNotSupported when n exceeds what the
// grid holds in registers (the caller falls back to the bucketed selection).
size_t rowsel_work_bytes();
cudaError_t launch_score_select_rows(const LaunchCtx& c, const uint8_t* d_plan, int ndk, int64_t nkeys,
                                     const int32_t* nt, uint32_t off_divk, const uint16_t* d_clskuv, const RowTabMeta* d_meta, const RowRec* d_rowrec,
                                     const uint64_t* d_khash, const uint64_t* d_genome, int64_t n, int64_t k,
                                     double* d_pred, uint64_t* d_ids, int64_t* d_idx, void* d_work);
cudaError_t launch_score_rows(const LaunchCtx& c, const uint8_t* d_plan, int ndk, const uint16_t* d_clskuv,
                              const RowTabMeta* d_meta, const double* d_rowpred, const uint64_t* d_khash,
                              const uint64_t* d_genome, int64_t n, double* d_pred, uint64_t* d_ids,
                              const SelHist& sel = SelHist{});
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
                         uint64_t seed, uint64_t* d_out, int32_t* d_partner, void* d_state,
                         const int32_t* d_skip = nullptr);

// reproduce, exact and block-parallel (breed_par.cu): the same children as launch_breed on the
// whole GPU.  Work area from breed_par_bytes(n, S, ...), S = breed_par_block(n).  *d_done is set
// to 1 on the device when the parallel path produced the generation; launch_breed(..., d_done)
// after it produces the generation otherwise (a stream or snapshot capacity did not fit).
int breed_par_block(int64_t n);
size_t breed_par_bytes(int64_t n, int S, size_t* stream_words, size_t* pool_cap);
cudaError_t launch_breed_par(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint64_t* d_par,
                             const uint64_t* d_pid, int64_t np, int64_t n, double mut, double cro, double cpy,
                             uint64_t seed, uint64_t* d_out, int32_t* d_partner, void* d_work, int S,
                             double sd_mult, size_t words_cap, int split_gen, uint32_t plan_pre,
                             int32_t** d_done);

// reproduce in the opt-in counter mode: offspring i draws from its own counter-based stream
// (breed.cu CounterCursor), one thread per offspring; same decision logic as the exact mode.
cudaError_t launch_breed_counter(const LaunchCtx& c, const uint8_t* d_plan, uint32_t plan_bytes, const uint64_t* d_par,
                                 const uint64_t* d_pid, int64_t np, int64_t n, double mut, double cro, double cpy,
                                 uint64_t seed, uint64_t* d_out, int32_t* d_partner);

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

// sharded selection (model.cu): a rank's local top-k as (score, global index) records, padded to
// k with (+inf, INT64_MAX); the merge of W such sorted lists (rank-major) into the global top-k:
// one CTA merging in shared memory when W * k * 24 bytes fit, else round by round in global
// memory (scratch merge_scratch_bytes(W, k))
struct ShardRec {
    double s;
    int64_t g;
};
cudaError_t launch_pack_records(const LaunchCtx& c, const double* d_score, const int64_t* d_lidx, int64_t kl,
                                int64_t k, int64_t goff, ShardRec* d_rec);
size_t merge_scratch_bytes(int W, int64_t k);
cudaError_t launch_merge_records(const LaunchCtx& c, const ShardRec* d_rec, int W, int64_t k, int64_t* d_idx,
                                 double* d_sc, void* d_scratch);

// stable LSD radix sort of (u64 key, u32 value) pairs by the low `bits` bits, in place
size_t sort_pairs_scratch_bytes(int64_t n);
cudaError_t launch_sort_pairs(const LaunchCtx& c, uint64_t* keys, uint32_t* vals, int64_t n, int bits,
                              void* scratch);
// the same with the count (<= n_cap) and key bit length in device memory (scratch: sort_pairs_scratch_bytes(n_cap))
cudaError_t launch_sort_pairs_dev(const LaunchCtx& c, uint64_t* keys, uint32_t* vals, int64_t n_cap,
                                  const int64_t* d_n, const int32_t* d_bits, void* scratch);

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
