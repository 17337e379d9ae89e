/*
 * etune_cuda.h — C ABI of libetune_cuda.so, the B200 (sm_100a) implementation of the
 * candidate-schedule scoring hot path of arXiv 2411.18873's energy-aware search.
 *
 * Drop-in boundary.  Each entry point replaces one reference interface
 * (/root/reference/proj/include/etune/, one header per module); the citation is on each declaration.
 * INTEGRATION.md shows the binding a reference maintainer adds (the reference's own
 * functions forwarding to these), and the repo's C++ host mirror
 * (paper_2411_18873_b200/host/etune_b200.hpp) keeps the reference's names.
 *
 * Conventions
 *  - Plain C: POD structs, raw pointers, int64 sizes.  No torch / C++ types.
 *  - Pointers named d_* are DEVICE pointers (caller-owned, on the ctx's device);
 *    h_* are HOST pointers (pinned memory recommended for the *_host calls).
 *  - Device work is enqueued on the ctx stream and is asynchronous unless the name
 *    ends in _host or _sync.  Data-dependent errors raised on the device (an illegal
 *    schedule in a batch) are reported by etune_cu_synchronize(), which returns the
 *    status and the lowest offending index — the element the reference, walking the
 *    batch in order, would have thrown on.
 *  - Status codes map 1:1 onto the reference exception classes (errors.hpp:15-100).
 *  - Bit-exactness: ids, counters, feature vectors, genomes, selected indices and
 *    offspring are bit-identical to the reference; predictions are bit-identical too
 *    (FP64, the reference's summation order, no FMA contraction).
 */
#ifndef ETUNE_CUDA_H
#define ETUNE_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ETUNE_CUDA_ABI_VERSION 2

typedef enum etune_status {
    ETUNE_OK = 0,
    ETUNE_ERR_PARSE = 1,                 /* etune::ParseError          errors.hpp:15 */
    ETUNE_ERR_VALIDATION = 2,            /* etune::ValidationError     errors.hpp:21 */
    ETUNE_ERR_SPACE_EXHAUSTED = 3,       /* etune::SpaceExhausted      errors.hpp:27 */
    ETUNE_ERR_ILLEGAL_SCHEDULE = 4,      /* etune::IllegalSchedule     errors.hpp:33 */
    ETUNE_ERR_TOO_LARGE = 5,             /* etune::TooLarge            errors.hpp:39 */
    ETUNE_ERR_NON_POSITIVE_ENERGY = 6,   /* etune::NonPositiveEnergy   errors.hpp:45 */
    ETUNE_ERR_INSUFFICIENT_DATA = 7,     /* etune::InsufficientData    errors.hpp:51 */
    ETUNE_ERR_SCHEMA_MISMATCH = 8,       /* etune::SchemaMismatch      errors.hpp:57 */
    ETUNE_ERR_VERSION_MISMATCH = 9,      /* etune::VersionMismatch     errors.hpp:63 */
    ETUNE_ERR_LENGTH_MISMATCH = 10,      /* etune::LengthMismatch      errors.hpp:68 */
    ETUNE_ERR_EMPTY_INPUT = 11,          /* etune::EmptyInput          errors.hpp:73 */
    ETUNE_ERR_IO = 12,                   /* etune::IoError             errors.hpp:79 */
    ETUNE_ERR_CONSISTENCY = 13,          /* etune::ConsistencyError    errors.hpp:85 */
    ETUNE_ERR_BACKEND_UNAVAILABLE = 14,  /* etune::BackendUnavailable  errors.hpp:91 */
    ETUNE_ERR_TRACE_MISS = 15,           /* etune::TraceMiss           errors.hpp:97 */
    ETUNE_ERR_INVALID_ARGUMENT = 64,     /* null pointer / bad size (no reference analogue) */
    ETUNE_ERR_CUDA = 65,                 /* CUDA runtime failure */
    ETUNE_ERR_NO_DEVICE = 66,            /* no sm_100 device: the library never falls back to CPU */
    ETUNE_ERR_UNSUPPORTED = 67           /* shape outside this build's table limits */
} etune_status;

/* OperatorSpec (opspec.hpp:30-47), words in candidate_id order (space.cpp:24-35).
 * kind: 0 MM, 1 MV, 2 CONV.  Unused fields keep the reference defaults
 * (m=n=k=1 for conv, stride=1, padding=0 and conv fields 0 for mm/mv). */
typedef struct etune_op_spec {
    int64_t kind, batch, m, n, k, height, width, in_channels, out_channels, kernel_size,
        stride, padding;
} etune_op_spec;

/* Schedule (schedule.hpp:40-44): spatial[d] = {blocks, threads, per_thread} for
 * d = batch, m, n; then k_tile, unroll, vectorize.  96 bytes, int64 like the reference. */
typedef struct etune_schedule {
    int64_t spatial[3][3];
    int64_t k_tile, unroll, vectorize;
} etune_schedule;

/* SpaceLimits (space.hpp:15-19). */
typedef struct etune_space_limits {
    int64_t max_block_threads, max_unroll, max_vectorize;
} etune_space_limits;

/* CounterSet (counters.hpp:13-24), same field order, 80 bytes. */
typedef struct etune_counters {
    int64_t grid, block, flops, int_ops, glb_ld, glb_st, shared_ld, shared_st;
    double sm_efficiency;
    int64_t active_sms;
} etune_counters;

/* DeviceConfig (device.hpp:17-45) numeric fields. */
typedef struct etune_device_config {
    int32_t num_sms;
    int32_t reserved;
    double constant_power_w, static_power_per_sm_w, dynamic_energy_per_flop_nj,
        dynamic_energy_per_glb_access_nj, dynamic_energy_per_shared_access_nj,
        base_throughput_flops_per_s_per_sm, mem_bandwidth_elems_per_s, latency_floor_ms,
        sampler_hz, warmup_s, noise_sigma_rel;
    uint64_t rng_seed;
} etune_device_config;

/* GeneticRates (genetic.hpp:14-18). */
typedef struct etune_genetic_rates {
    double mutation, crossover, copy;
} etune_genetic_rates;

/* BoostParams (energy_model.hpp:33-41). */
typedef struct etune_boost_params {
    int32_t num_trees, max_depth;
    double learning_rate, min_leaf_weight, reg_lambda;
} etune_boost_params;

/* Defaults identical to the reference's: DeviceConfig::a100_like() (device.cpp:40),
 * SpaceLimits{} , GeneticRates{}, BoostParams{}. */
void etune_default_device_config(etune_device_config* out);
void etune_default_space_limits(etune_space_limits* out);
void etune_default_genetic_rates(etune_genetic_rates* out);
void etune_default_boost_params(etune_boost_params* out);

const char* etune_cu_last_error(void); /* thread-local message of the last failure */
int etune_cu_abi_version(void);
/* Number of kernels this library has launched in the process (diagnostics / bench). */
uint64_t etune_cu_launch_count(void);

/* ------------------------------------------------------------------ context */
typedef struct etune_cu_ctx etune_cu_ctx;

/* stream: the cudaStream_t every call of this ctx is ordered on (NULL = default stream). */
etune_status etune_cu_ctx_create(int device, void* stream, etune_cu_ctx** out);
etune_status etune_cu_ctx_destroy(etune_cu_ctx* ctx);
etune_status etune_cu_ctx_set_stream(etune_cu_ctx* ctx, void* stream);
void* etune_cu_ctx_stream(etune_cu_ctx* ctx);
/* Device memory and copies on the ctx's device / stream, so a C or C++ caller (e.g. the reference-side
 * binding) needs no CUDA runtime of its own.  The copies are asynchronous on the ctx
 * stream (host memory pinned or pageable); etune_cu_synchronize waits for them. */
etune_status etune_cu_device_alloc(etune_cu_ctx* ctx, void** out, int64_t bytes);
etune_status etune_cu_device_free(etune_cu_ctx* ctx, void* p);
etune_status etune_cu_memcpy_h2d(etune_cu_ctx* ctx, void* d_dst, const void* h_src, int64_t bytes);
etune_status etune_cu_memcpy_d2h(etune_cu_ctx* ctx, void* h_dst, const void* d_src, int64_t bytes);
/* Waits for the ctx stream; reports a device-detected data error (first bad index). */
etune_status etune_cu_synchronize(etune_cu_ctx* ctx, int64_t* first_bad_index);

/* ------------------------------------------------------------------- plans */
/* A plan holds an operator's knob tables on the device: the ordered tilings of each
 * spatial extent (space.cpp:69-78), divisors of K (57-67), and the per-operator
 * feature tables (features.cpp:15-46 factored by the knobs each feature depends on;
 * log1p evaluated once per distinct counter on the host with the platform libm, the
 * function the reference calls).  Replaces the per-candidate setup inside
 * extract_features (features.hpp:35) / ScheduleEnumerator (space.hpp:45).
 * Throws-equivalents: VALIDATION (op invalid, opspec.cpp:65-93), UNSUPPORTED. */
typedef struct etune_cu_plan etune_cu_plan;
etune_status etune_cu_plan_create(etune_cu_ctx* ctx, const etune_op_spec* op,
                                  const etune_device_config* dev /*NULL=a100_like*/,
                                  const etune_space_limits* limits /*NULL=defaults*/,
                                  etune_cu_plan** out);
etune_status etune_cu_plan_destroy(etune_cu_plan* plan);
/* LoopNest of the op (opspec.cpp:103-117) and legal-space size (space.cpp:152-160). */
etune_status etune_cu_plan_nest(const etune_cu_plan* plan, int64_t out4[4]);
etune_status etune_cu_plan_space_size(const etune_cu_plan* plan, int64_t* out);

/* ---------------------------------------------------------- population codec */
/* Device-resident populations are 8-byte genomes (uint64 per candidate): indices of
 * the candidate's knobs in the plan's tables.  encode validates exactly like
 * validate_schedule (schedule.cpp:26-61); an illegal row is reported by
 * etune_cu_synchronize as ETUNE_ERR_ILLEGAL_SCHEDULE with its index. */
etune_status etune_cu_encode(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                             const etune_schedule* d_sched, int64_t n, uint64_t* d_genome);
etune_status etune_cu_decode(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                             const uint64_t* d_genome, int64_t n, etune_schedule* d_sched);

/* sample_random (space.hpp:80-82, space.cpp:170-251) on the device, bit-exact with
 * the reference's std::mt19937_64(seed) stream: n distinct legal genomes in the
 * reference's order (d_ids nullable).  Synchronous (the attempt count is data
 * dependent).  Errors: VALIDATION (n < 1), SPACE_EXHAUSTED (fewer than n legal
 * schedules, or the reference's attempt budget 10000 + 1000 n exceeded). */
etune_status etune_cu_sample_random(etune_cu_ctx* ctx, const etune_cu_plan* plan, int64_t n,
                                    uint64_t seed, uint64_t* d_genome, uint64_t* d_ids /*nullable*/);

/* candidate_id (space.hpp:32, space.cpp:22-45) */
etune_status etune_cu_candidate_ids(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                    const uint64_t* d_genome, int64_t n, uint64_t* d_ids);
/* derive_counters (counters.hpp:35, counters.cpp:9-49) */
etune_status etune_cu_counters(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                               const uint64_t* d_genome, int64_t n, etune_counters* d_out);
/* extract_features (features.hpp:35, features.cpp:48-51): d_feat is n x 16 doubles
 * (FeatureVector layout); d_ids optional (NULL). */
etune_status etune_cu_features(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                               const uint64_t* d_genome, int64_t n, double* d_feat,
                               uint64_t* d_ids);

/* ------------------------------------------------------------ measurement */
/* SimBackend (measure.hpp:102-114) on device genomes, with the plan's DeviceConfig:
 * sim_true_power_and_latency (measure.hpp:29-41) and nvml_sim_measure's
 * sampler average (measure.hpp:43-60).  d_latency_ms is required
 * (measure_latency_ms); d_power_w / d_energy_mj / d_iterations are nullable — all
 * three NULL is the cheap latency-only evaluation used by the latency filter.
 * The reference ships no implementation of these; parity is against the repo's CPU
 * restatement (oracle/), whose operation order and noise generator (SPEC:327's
 * multiplicative Gaussian: a polar-method normal over splitmix64 words with a log built
 * from IEEE +, *, / -- no libm) this kernel follows bit for bit. */
etune_status etune_cu_sim_measure(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                  const uint64_t* d_genome, int64_t n, double* d_latency_ms,
                                  double* d_power_w, double* d_energy_mj, int64_t* d_iterations);

/* NVML measurement harness (north_star (5); the reference's NvmlBackend, measure.hpp:
 * 130-140, is a stub that always throws BackendUnavailable).  Each schedule runs as a
 * runtime-tiled fp32 GEMM / implicit-GEMM conv kernel honouring its tiling, k_tile,
 * unroll and vectorize; after warmup_ms of repeats, iterations = clamp(window_ms /
 * latency, min_iterations, max_iterations) runs are timed with CUDA events and the
 * NVML cumulative energy counter (nvmlDeviceGetTotalEnergyConsumption) is read around
 * them: avg_power_w = energy delta / wall time, energy_mj = avg_power_w x latency_ms
 * (PAPER:164-165).  Schedules the kernel cannot run (per-thread tile
 * above 8x8 in (m, n), shared tiles beyond the device limit, too many registers for the
 * block) get feasible = 0 and infinite latency/energy. */
typedef struct etune_nvml_params {
    double warmup_ms, window_ms;
    int64_t min_iterations, max_iterations;
} etune_nvml_params;
typedef struct etune_measurement {   /* MeasurementRecord (measure.hpp:17-25) */
    uint64_t candidate_id;
    double latency_ms, avg_power_w, energy_mj;
    int64_t iterations;
    int32_t feasible, reserved;
} etune_measurement;
void etune_default_nvml_params(etune_nvml_params* out);  /* 50 ms, 200 ms, 10, 1e6 */
/* *out = 1 when NVML energy counters are readable for the ctx's GPU */
etune_status etune_cu_nvml_available(etune_cu_ctx* ctx, int* out);
/* one run of a schedule's candidate kernel on caller buffers (mm: A[B][M][K], B[B][K][N],
 * C[B][M][N]; conv: input NCHW, weights [Cout][Cin*ks*ks], output [B][Cout][OH*OW]);
 * UNSUPPORTED when the schedule is infeasible for the kernel */
etune_status etune_cu_candidate_run(etune_cu_ctx* ctx, const etune_cu_plan* plan, const etune_schedule* h_sched,
                                    const float* d_a, const float* d_b, float* d_c);
/* measured latency only (the LatencyEvaAndPick step on hardware): one warm run, then
 * `reps` timed runs per schedule; infinity for infeasible schedules */
etune_status etune_cu_candidate_latency(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                        const etune_schedule* h_sched, int64_t n, int32_t reps,
                                        double* h_latency_ms);
/* measure n host schedules (synchronous); ILLEGAL_SCHEDULE with *first_bad like the
 * reference; BACKEND_UNAVAILABLE without NVML */
etune_status etune_cu_nvml_measure(etune_cu_ctx* ctx, const etune_cu_plan* plan, const etune_schedule* h_sched,
                                   int64_t n, const etune_nvml_params* params, etune_measurement* h_out,
                                   int64_t* first_bad /*nullable*/);

/* ------------------------------------------------------------- cost model */
/* EnergyModel trees in the reference's flat TreeNode form (energy_model.hpp:45-57):
 * node arrays concatenated in tree order, tree_offsets[num_trees+1]. */
typedef struct etune_cu_forest etune_cu_forest;
etune_status etune_cu_forest_create(etune_cu_ctx* ctx, const int32_t* feature,
                                    const double* threshold, const int32_t* left,
                                    const int32_t* right, const double* value,
                                    const int64_t* tree_offsets, int64_t num_trees,
                                    double base_score, double learning_rate,
                                    etune_cu_forest** out);
etune_status etune_cu_forest_destroy(etune_cu_forest* forest);

/* EnergyModel::predict_many (energy_model.hpp:73, energy_model.cpp:245-257) on
 * feature vectors already in device memory (n x 16 doubles). */
etune_status etune_cu_predict(etune_cu_ctx* ctx, etune_cu_forest* forest,
                              const double* d_feat, int64_t n, double* d_pred);

/* Fused extract_features + predict (the north-star scoring pass): genome in,
 * prediction (and optionally candidate id) out.  The forest is compiled per plan
 * (exact partial evaluation + per-feature rank bins) on first use and cached. */
etune_status etune_cu_score(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                            etune_cu_forest* forest, const uint64_t* d_genome, int64_t n,
                            double* d_pred, uint64_t* d_ids /*nullable*/);

/* One step of the hot path: fused score of a device population, then its k best by
 * (prediction asc, index asc) into d_idx (sorted).  d_ids nullable.  Same result as
 * etune_cu_score + etune_cu_topk; for k <= 4096 the score kernel also buckets every
 * prediction, so the selection reads the predictions once and resolves one bucket.
 * Replaces the reference's predict_many (energy_model.hpp:72) + partial sort. */
etune_status etune_cu_score_select(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                   etune_cu_forest* forest, const uint64_t* d_genome, int64_t n,
                                   int64_t k, double* d_pred, uint64_t* d_ids /*nullable*/,
                                   int64_t* d_idx);

/* Device time, summed over the etune_cu_score_select calls since the last call, of
 * (a) work before the score kernel (0 on the current paths), (b) the score kernel,
 * (c) the selection kernels (CUDA events on the ctx stream; synchronises when any were
 * recorded); then switches that timing on (on != 0) or off.  For benchmarks and
 * profiling (the events serialise the launches they separate). */
etune_status etune_cu_profile_score(etune_cu_ctx* ctx, int on, double* pre_ms /*nullable*/,
                                    double* score_ms /*nullable*/, double* select_ms /*nullable*/,
                                    int64_t* calls /*nullable*/);

/* Scoring forms (all bit-identical; the choice only affects speed):
 *  ROWS   the default for populations of >= 2^16 candidates per (forest, plan): the forest is
 *         compiled ON THE DEVICE (three launches, no host work) into one prediction per
 *         (tiling-triple key, Kuv class) row -- a candidate's prediction depends only on which
 *         side of each threshold its features fall, and only f6/f7/f10 vary with (k_tile,
 *         unroll, vectorize) -- so scoring is one 8-byte gather per candidate (rowtab.cu);
 *  WALK   features + the reference tree walk per candidate (any forest; no compile);
 *  CLASS / KEYED / KEYED_BYTE  the host-compiled QuickScorer forms of round 1 (forest.cpp).
 * AUTO (default) = ROWS once the (forest, plan) has scored >= 2^16 candidates in total (or
 * one call has), WALK before; CLASS tables when the operator's row table would exceed
 * 2^25 rows. */
#define ETUNE_FORM_AUTO 0
#define ETUNE_FORM_ROWS 1
#define ETUNE_FORM_WALK 2
#define ETUNE_FORM_CLASS 3
#define ETUNE_FORM_KEYED 4
#define ETUNE_FORM_KEYED_BYTE 5
etune_status etune_cu_forest_set_form(etune_cu_forest* forest, int form);
/* Compiles the forest for the plan in the form the next large scoring call would use (ROWS:
 * enqueued on the ctx stream, asynchronous; host forms: synchronous).  Lets a caller time
 * or overlap the compile of a freshly trained model. */
etune_status etune_cu_forest_compile(etune_cu_ctx* ctx, etune_cu_forest* forest, const etune_cu_plan* plan);
/* Row-table diagnostics (synchronises the ctx stream): {tiling-triple keys, Kuv classes,
 * rows, row-table bytes, thresholds on f10, f7, f6, legal (k, u, v) triples}; all zero when
 * the table has not been compiled. */
etune_status etune_cu_forest_rows_info(etune_cu_ctx* ctx, etune_cu_forest* forest, const etune_cu_plan* plan,
                                       int64_t out[8]);
/* Legacy selector (round 1), kept for the tests of the host-compiled forms: 1 = KEYED, 2 = KEYED_BYTE, 0 = CLASS.
 * Scoring form for populations of >= 2^16 candidates: 1 (default) = keyed path where the
 * forest compiles to it (<= 128 trees of <= 32 leaves, <= 256 distinct non-Kuv masks per
 * Kuv tree): the full form (5-bit exit slots per (tiling triple, Kuv class), table
 * <= 64 MB) or else the byte form (per tiling triple); 2 = byte form only; 0 = class-table
 * kernel only.  All are bit-identical.  Set it before the first large scoring call. */
etune_status etune_cu_forest_set_keyed(etune_cu_forest* forest, int mode);

/* Which form scores populations of >= 2^16 candidates of this plan (compiling it now if
 * needed): 0 = class-table kernel, 1 = keyed byte form, 2 = keyed full form, 3 = the
 * general tree-walk kernel, 4 = the row table.  Diagnostic. */
etune_status etune_cu_forest_score_form(etune_cu_forest* forest, const etune_cu_plan* plan, int* form);

/* Reference-facing end-to-end call with HOST buffers: schedules in the reference's
 * Schedule layout -> predictions (+ ids).  Host->device copy, encode (legality check),
 * fused score and device->host copy, synchronised.  Equivalent to
 *   for c in population: pred[i] = model.predict(extract_features(op, c.schedule, dev))
 * and returns ETUNE_ERR_ILLEGAL_SCHEDULE (with *first_bad) where that loop would throw. */
etune_status etune_cu_score_host(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                 etune_cu_forest* forest, const etune_schedule* h_sched,
                                 int64_t n, double* h_pred, uint64_t* h_ids /*nullable*/,
                                 int64_t* first_bad /*nullable*/);

/* The reference-facing "score the population and keep the best" with HOST buffers (the
 * reference's predict_many + partial sort by (prediction, index)): schedules in
 * the reference's 96-byte layout (pinned or pageable), all predictions back into h_pred
 * (nullable) and the k best indices, sorted, into h_idx.  Same pipeline as etune_cu_score_host;
 * the predictions stay on the device and the selection runs there, so only k indices come back
 * besides the predictions.  ILLEGAL_SCHEDULE (with *first_bad) like etune_cu_score_host. */
etune_status etune_cu_score_select_host(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                        etune_cu_forest* forest, const etune_schedule* h_sched,
                                        int64_t n, int64_t k, double* h_pred /*nullable*/,
                                        int64_t* h_idx, int64_t* first_bad /*nullable*/);
/* Diagnostics of the per-plan forest compilation: {reference interior nodes, tests
 * folded for this operator, class->mask table entries, max leaves per tree, total
 * leaves, blob bytes, bitmask of feature channels still tested, trees}. */
etune_status etune_cu_forest_compile_stats(etune_cu_forest* forest, const etune_cu_plan* plan,
                                           int64_t out[8]);

/* ------------------------------------------------------ cost-model update */
/* EnergyModel::train (energy_model.hpp:69-70, energy_model.cpp:173-243) on device
 * samples: d_feat n x 16 doubles, d_energy n measured energies (mJ).  Bit-exact with
 * the reference: every node (feature, threshold, left, right, value), the base score,
 * the reference energy and the per-round training loss.  params NULL = BoostParams{};
 * max_depth <= 10 in this build.
 * Outputs (device, caller-owned): node arrays with capacity
 * num_trees * (2^(max_depth+1) - 1), tree_offsets[num_trees + 1] (node ranges, tree
 * order, node indices local to their tree like RegressionTree::nodes),
 * d_scalars[2] = {base_score, reference_energy_mj}, d_training_loss[num_trees + 1]
 * (nullable: training_loss_per_round, energy_model.hpp:81-85).
 * Errors: INSUFFICIENT_DATA (n < 2, host-side); NON_POSITIVE_ENERGY reported by
 * etune_cu_synchronize with the first offending index; UNSUPPORTED (max_depth > 10). */
etune_status etune_cu_train(etune_cu_ctx* ctx, const double* d_feat, const double* d_energy, int64_t n,
                            const etune_boost_params* params, int32_t* d_feature, double* d_threshold,
                            int32_t* d_left, int32_t* d_right, double* d_value, int64_t* d_tree_offsets,
                            double* d_scalars, double* d_training_loss /*nullable*/);

/* energy_loss (Eq. 1; energy_model.hpp:19-24, energy_model.cpp:23-34) for n samples:
 * d_out[3i..3i+2] = {value, gradient, hessian}.  NON_POSITIVE_ENERGY (first index) at
 * etune_cu_synchronize. */
etune_status etune_cu_energy_loss(etune_cu_ctx* ctx, const double* d_pred, const double* d_meas, int64_t n,
                                  double* d_out);

/* snr_db (energy_model.hpp:108-109, energy_model.cpp:352-370): the two sums are formed
 * on the device in the reference's order; the final scalar 10*log10(signal/error),
 * capped at 100 dB, is taken with the platform libm like the reference.  Synchronous.
 * Errors: EMPTY_INPUT (n == 0), NON_POSITIVE_ENERGY (with *first_bad). */
etune_status etune_cu_snr_db(etune_cu_ctx* ctx, const double* d_pred, const double* d_meas, int64_t n,
                             double* h_out, int64_t* first_bad /*nullable*/);

/* A forest built from device-resident trained arrays (as written by etune_cu_train);
 * synchronises the ctx stream, then behaves like etune_cu_forest_create. */
etune_status etune_cu_forest_from_device(etune_cu_ctx* ctx, const int32_t* d_feature,
                                         const double* d_threshold, const int32_t* d_left,
                                         const int32_t* d_right, const double* d_value,
                                         const int64_t* d_tree_offsets, int64_t num_trees,
                                         const double* d_scalars, double learning_rate,
                                         etune_cu_forest** out);

/* ---------------------------------------------------------- reproduction */
/* reproduce (genetic.hpp:48-51, genetic.cpp:137-187) on device genomes, bit-exact with
 * the reference's ONE sequential std::mt19937_64(seed) stream: offspring i starts from
 * parents[i % num_parents] and is a mutation / crossover / copy drawn exactly as the
 * reference draws it (the stream is generated on the device; the data-dependent word
 * offsets are resolved there by speculation).  rates NULL = GeneticRates{}.
 * d_partner[i] (nullable) = crossover partner's parent index, -1 for mutation/copy, so
 * lineage = {id(parents[i % P])} or {id(base), id(parents[d_partner[i]])}.
 * d_ids (nullable) = candidate_id of every offspring.
 * Errors: VALIDATION (num_parents < 1, rates summing to <= 0 — genetic.cpp:140-152);
 * ILLEGAL_SCHEDULE at the first offspring whose repair fails (reported by
 * etune_cu_synchronize with its index, like the reference's throw from repair). */
etune_status etune_cu_reproduce(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                const uint64_t* d_parents, int64_t num_parents, int64_t n,
                                const etune_genetic_rates* rates, uint64_t seed,
                                uint64_t* d_offspring, int32_t* d_partner /*nullable*/,
                                uint64_t* d_ids /*nullable*/);

/* reproduce with the opt-in counter-based RNG (NOT the reference's stream): the same decisions,
 * transforms and word order per offspring (coin, knob, Lemire draws, partner redraws, mask, repair),
 * but offspring i draws from its own stream word_j = splitmix64(key_i + j), key_i =
 * splitmix64(seed ^ splitmix64(i)), so the generation has no sequential chain: one thread per
 * offspring (2^20 offspring in about a millisecond, where the exact mode resolves the reference's
 * one mt19937_64 stream on a single CTA).  Its oracle is orc_reproduce_counter (oracle/), bit for
 * bit.  Same arguments and errors as etune_cu_reproduce. */
etune_status etune_cu_reproduce_counter(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                        const uint64_t* d_parents, int64_t num_parents, int64_t n,
                                        const etune_genetic_rates* rates, uint64_t seed,
                                        uint64_t* d_offspring, int32_t* d_partner /*nullable*/,
                                        uint64_t* d_ids /*nullable*/);
/* ------------------------------------------------------------- selection */
/* The k smallest of d_score[0..n) under the total order (score asc, index asc)
 * ("lowest predicted energy"; SURVEY H3 tie rule), written sorted to
 * d_idx (int64).  Scratch is taken from the ctx. */
etune_status etune_cu_topk(etune_cu_ctx* ctx, const double* d_score, int64_t n, int64_t k,
                           int64_t* d_idx);

/* ------------------------------------------------------ search (Algorithm 1) */
/* The energy-aware genetic search of PAPER:223-254 / SPEC:372-457 (the reference ships
 * it only as a spec; there is no reference code).  Every data-parallel step runs on the
 * device through this library; the host keeps the per-round scalars (k, SNR, best).
 * Choices where the spec is silent: initial parents = the M
 * fastest of the initial sample; round r reproduces with seed rng_seed + r; k is kept
 * in integer fifths; SNR compares step-3 predictions with the measured energies
 * normalised by the model's reference energy; selections break ties by index. */
typedef struct etune_search_config {
    int64_t M;                 /* kept per round after the latency filter */
    int64_t generation_size;   /* > M */
    int32_t k_init_fifths;     /* 5 == k 1.0 */
    int32_t max_rounds;
    int32_t patience;          /* rounds without > improve_rel best-energy gain (5) */
    int32_t inverted_semantics;/* 1: the paper's literal prose reading of the k rule */
    double mu_db;              /* SNR threshold (20 dB) */
    double improve_rel;        /* 0.001 */
    uint64_t rng_seed;
    etune_genetic_rates rates;
    etune_boost_params boost;
    int32_t backend;           /* 0: SimBackend (device formula), 1: the GPU itself (candidate kernels:
                                  CUDA-event latency filter, NVML energy of the selected), 2: ReplayBackend
                                  (measure.hpp:116-128: records of a log, etune_cu_search_set_replay) */
    int32_t latency_reps;      /* backend 1: timed runs per candidate in the latency filter */
    etune_nvml_params nvml;    /* backend 1: energy measurement protocol */
    int32_t latency_only;      /* 1: run_latency_only: no cost model; parents = the
                                  ceil(M/2) fastest of the M; best = lowest latency (then id), whose
                                  energy is measured for the report (one measurement per round) */
    int32_t counter_rng;       /* 1: reproduce with etune_cu_reproduce_counter (not the reference's stream) */
} etune_search_config;

typedef struct etune_round_report {   /* RoundReport */
    int64_t round;                    /* 0 = initial_round */
    int32_t k_before_fifths, k_after_fifths;
    double snr_db;                    /* NaN for round 0 */
    int64_t measured;                 /* energy measurements this round */
    int64_t cumulative_measured;
    uint64_t best_id;
    double best_latency_ms, best_energy_mj, best_power_w;
    double wall_ms;                   /* host wall time of the round, device synchronised */
} etune_round_report;

typedef struct etune_cu_search etune_cu_search;
void etune_default_search_config(etune_search_config* out);
/* Backend 0: the plan's SimBackend (etune_cu_sim_measure); backend 1: measurements on
 * this GPU (etune_cu_candidate_latency + etune_cu_nvml_measure). */
etune_status etune_cu_search_create(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                    const etune_search_config* cfg, etune_cu_search** out);
etune_status etune_cu_search_destroy(etune_cu_search* s);
/* ReplayBackend's log (backend 2): latency filter and energy measurements are looked up by
 * candidate id, the most recent record of an id winning (MeasurementLog::lookup); an id
 * the log lacks fails the round with ETUNE_ERR_TRACE_MISS.  Copies the records. */
etune_status etune_cu_search_set_replay(etune_cu_search* s, const etune_measurement* records, int64_t n);
etune_status etune_cu_search_initial(etune_cu_search* s, etune_round_report* out);  /* initial_round */
etune_status etune_cu_search_round(etune_cu_search* s, etune_round_report* out);    /* round */
/* run_search: initial round (if not yet run) then rounds until max_rounds or patience;
 * writes up to cap reports, *n_reports = rounds run. */
etune_status etune_cu_search_run(etune_cu_search* s, etune_round_report* reports, int64_t cap,
                                 int64_t* n_reports);
/* best measured candidate: energy, then latency, then id */
etune_status etune_cu_search_best(etune_cu_search* s, etune_schedule* h_sched, uint64_t* h_id,
                                  double* h_latency_ms, double* h_energy_mj);
/* current parents (device genomes; *n = count, at most cap written) */
etune_status etune_cu_search_parents(etune_cu_search* s, uint64_t* d_out, int64_t cap, int64_t* n);

/* ------------------------------------------------------- multi-GPU (NCCL) */
/* One rank per GPU over NVLink/NVSwitch.  The population shards by index: rank r owns
 * the contiguous global range [global_offset, global_offset + n) with offsets
 * increasing with rank.  NCCL carries only the per-shard top-k records and the
 * broadcast of trained model arrays (north_star); everything else is shard-local. */
#define ETUNE_NCCL_UNIQUE_ID_BYTES 128
etune_status etune_cu_nccl_unique_id(void* out_id /* ETUNE_NCCL_UNIQUE_ID_BYTES */);
/* Caller-provided collectives, used when no NCCL communicator is attached (e.g. ranks that
 * share one GPU, or a host-side transport in tests).  Device pointers on the ctx's device;
 * `stream` is the ctx stream (cudaStream_t): the callback must order its work after the
 * stream's pending work and before the stream's subsequent work (synchronising it is enough).
 * allgather: every rank contributes `bytes` at d_send; d_recv receives nranks * bytes in rank
 * order.  broadcast: root's d_buf to every rank.  Return 0 on success.  NULL detaches. */
typedef struct etune_transport {
    void* user;
    int32_t nranks, rank;
    int32_t (*allgather)(void* user, const void* d_send, void* d_recv, int64_t bytes, void* stream);
    int32_t (*broadcast)(void* user, void* d_buf, int64_t bytes, int32_t root, void* stream);
} etune_transport;
etune_status etune_cu_ctx_attach_transport(etune_cu_ctx* ctx, const etune_transport* t);
/* Collective over all ranks: binds an NCCL communicator to the ctx (its device/stream). */
etune_status etune_cu_ctx_attach_nccl(etune_cu_ctx* ctx, const void* unique_id, int nranks, int rank);

/* Population-sharded selection: every rank passes its shard's scores; on return every
 * rank holds the SAME k global indices (and scores, nullable), sorted by
 * (score asc, global index asc) — identical to etune_cu_topk over the concatenated
 * population.  Local top-k -> ncclAllGather of (score, index) records -> on-device
 * merge.  Without an attached communicator it is the single-rank case. */
etune_status etune_cu_topk_sharded(etune_cu_ctx* ctx, const double* d_score, int64_t n,
                                   int64_t global_offset, int64_t k, int64_t* d_idx_global,
                                   double* d_score_out /*nullable*/);

/* etune_cu_score_select on a shard: fused score of the rank's n candidates (global
 * indices [global_offset, global_offset + n)), its local k best, then the same
 * all-gather + merge as etune_cu_topk_sharded: every rank returns the same k global
 * indices (and scores, nullable). */
etune_status etune_cu_score_select_sharded(etune_cu_ctx* ctx, const etune_cu_plan* plan,
                                           etune_cu_forest* forest, const uint64_t* d_genome,
                                           int64_t n, int64_t global_offset, int64_t k,
                                           double* d_pred, uint64_t* d_ids /*nullable*/,
                                           int64_t* d_idx_global, double* d_score_out /*nullable*/);

/* ---------------------------------------------------------------- persistence
 * The reference's on-disk formats, host-only, no device needed:
 * a forest trained on the device round-trips through the reference's own loader.
 * Writers follow nlohmann::json's output (sorted keys, shortest round-trip doubles,
 * nlohmann's number layout); readers parse numbers with strtod, so every double is
 * preserved bit for bit.  Writers: out == NULL queries the length (*out_len, excluding
 * the terminating NUL); otherwise cap must be >= *out_len + 1. */
typedef struct etune_model_host {   /* library-allocated; release with etune_model_host_free */
    int64_t num_trees, num_nodes;
    int32_t* feature;
    double* threshold;
    int32_t* left;
    int32_t* right;
    double* value;
    int64_t* tree_offsets;          /* num_trees + 1 */
    etune_boost_params params;
    double base_score, reference_energy_mj;
} etune_model_host;

/* EnergyModel::to_json (energy_model.cpp:259-284), "etune-model-v1". */
etune_status etune_model_to_json(const int32_t* feature, const double* threshold, const int32_t* left,
                                 const int32_t* right, const double* value, const int64_t* tree_offsets,
                                 int64_t num_trees, const etune_boost_params* params, double base_score,
                                 double reference_energy_mj, char* out /*nullable*/, int64_t cap,
                                 int64_t* out_len);
/* EnergyModel::from_json (energy_model.cpp:286-336): ETUNE_ERR_IO on unreadable text, missing
 * keys or an empty tree; ETUNE_ERR_VERSION_MISMATCH on model_version / feature_schema. */
etune_status etune_model_from_json(const char* text, int64_t len, etune_model_host* out);
void etune_model_host_free(etune_model_host* m);

typedef struct etune_samples_host { /* library-allocated; release with etune_samples_host_free */
    int64_t n;
    double* features;               /* n x 16 */
    double* measured_energy_mj;
    double* normalized_energy;
} etune_samples_host;

/* save_energy_samples (energy_model.cpp:372-383): one JSON object per line. */
etune_status etune_samples_to_jsonl(const double* features, const double* measured_energy_mj,
                                    const double* normalized_energy, int64_t n, char* out /*nullable*/,
                                    int64_t cap, int64_t* out_len);
/* load_energy_samples (energy_model.cpp:385-420): ETUNE_ERR_IO (bad line),
 * ETUNE_ERR_SCHEMA_MISMATCH (width != 16), ETUNE_ERR_NON_POSITIVE_ENERGY. */
etune_status etune_samples_from_jsonl(const char* text, int64_t len, etune_samples_host* out);
void etune_samples_host_free(etune_samples_host* s);

/* MeasurementLog (measure.hpp:63-83): append-only JSONL, one
 * MeasurementRecord per line.  The reference declares the log but ships no writer, so the
 * line layout follows its other JSONL files (nlohmann dump(), keys in sorted order). */
typedef struct etune_log_record {
    etune_measurement m;          /* candidate_id, latency_ms, avg_power_w, energy_mj, iterations */
    char backend[16];             /* NUL-terminated backend tag ("sim", "nvml", ...) */
    char timestamp[32];           /* NUL-terminated UTC timestamp */
} etune_log_record;
/* log_append: the JSONL text of n records (append it to the log file). */
etune_status etune_measurement_log_to_jsonl(const etune_log_record* records, int64_t n, char* out /*nullable*/,
                                            int64_t cap, int64_t* out_len);
/* log_load: empty text = empty log; ETUNE_ERR_IO (unparsable line), ETUNE_ERR_CONSISTENCY
 * (energy_mj != avg_power_w * latency_ms beyond 1e-9 relative, line number in the message). */
etune_status etune_measurement_log_from_jsonl(const char* text, int64_t len, etune_log_record** out, int64_t* n);
void etune_measurement_log_free(etune_log_record* records);

/* device_profile_to_json (device.cpp:44-62), "etune-profile-v1", dump(2) + newline. */
etune_status etune_device_profile_to_json(const etune_device_config* dev, const char* name /*nullable*/,
                                          char* out /*nullable*/, int64_t cap, int64_t* out_len);
/* device_profile_from_json (device.cpp:64-101) incl. DeviceConfig::validate:
 * ETUNE_ERR_PARSE, ETUNE_ERR_VERSION_MISMATCH, ETUNE_ERR_VALIDATION. */
etune_status etune_device_profile_from_json(const char* text, int64_t len, etune_device_config* out,
                                            char* name_out /*nullable*/, int64_t name_cap);

/* ncclBroadcast of `bytes` device bytes from `root` (trained forest arrays). */
etune_status etune_cu_broadcast(etune_cu_ctx* ctx, void* d_buf, int64_t bytes, int root);

#ifdef __cplusplus
}
#endif
#endif
