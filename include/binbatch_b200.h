/*
 * binbatch_b200.h -- the C ABI of the B200-native Multi-Bin Batching engine.
 *
 * This is the drop-in boundary for the reference simulator's hot path
 * (/root/reference/proj/include/binbatch/, "binbatch", header-only C++20).
 * The reference has no FFI; its operator API is the C++ header API, so every
 * entry point below is the flattened (POD, plain pointers and sizes, status
 * codes instead of exceptions) form of one reference function, cited
 * file:line.  The C++ drop-in header include/binbatch_b200/binbatch.hpp
 * restores the reference's types, names and exception behaviour on top of
 * this ABI.
 *
 * All hot work runs in hand-written sm_100a kernels
 * (paper_2412_04504_b200/csrc/*.cu).  There is no CPU fallback: without a
 * CUDA device every compute entry point returns BB_ECUDA.
 *
 * Threading: entry points are re-entrant; calls on the same device serialise
 * on a per-device lock.  Host-buffer entry points block until results are on
 * the host.  The *_device entry points take device pointers and a
 * cudaStream_t (as void*) and are stream-ordered (no host sync) unless
 * documented otherwise.
 */
#ifndef BINBATCH_B200_H
#define BINBATCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BB_ABI_VERSION 2
#define BB_MAX_BINS 64        /* generated mode (fused kernel) */
#define BB_TRACE_MAX_BINS 32  /* trace mode (one warp lane per bin) */
#define BB_NO_BATCH 0xFFFFFFFFu

/* Status codes: the reference's exception categories.
 * BB_EINVAL  <-> std::invalid_argument   (simulator.hpp:153-167, binning.hpp:31-44, ...)
 * BB_EDOMAIN <-> std::domain_error       (simulator.hpp:189-190, binning.hpp:135-140)
 * BB_ERUNTIME<-> std::runtime_error      (experiment.hpp:356-358)               */
typedef enum {
  BB_OK = 0,
  BB_EINVAL = 1,
  BB_EDOMAIN = 2,
  BB_ERUNTIME = 3,
  BB_ECUDA = 4,
  BB_EUNSUPPORTED = 5
} bb_status;

/* ServiceDist (service_dist.hpp:27-40) + the trace modes of replay_trace
 * (simulator.hpp:57-60, :349-352) + the samplers BASELINE configs 3 and 5 need
 * (tokens_to_time, workload.hpp:167-170; log-normal). */
typedef enum {
  BB_SVC_UNIFORM = 0,        /* lo + (hi-lo)*u                        */
  BB_SVC_EXPONENTIAL = 1,    /* -log1p(-u)/rate                       */
  BB_SVC_EMPIRICAL = 2,      /* sorted table, sampled with replacement */
  BB_SVC_TRACE_CYCLIC = 3,   /* table[id % n_table]                   */
  BB_SVC_TRACE_RESAMPLE = 4, /* table sampled with replacement        */
  BB_SVC_LINEAR = 6,         /* lin_b*len + lin_a, len ~ U[lo,hi]      */
  BB_SVC_LOGNORMAL = 7       /* exp(mu + sigma*Z)                      */
} bb_service_kind;

/* ErrorModel (binning.hpp:148-162) */
typedef enum { BB_ERR_PERFECT = 0, BB_ERR_SYMMETRIC = 1, BB_ERR_CONFUSION = 2 } bb_error_kind;

/* Where the random streams come from.
 *   BB_RNG_PHILOX:    counter-based Philox4x32-10 on the device (generated mode;
 *                     agrees with the reference in distribution, 3-sigma).
 *   BB_RNG_REFERENCE: the reference's own streams (mt19937_64 seeded through
 *                     splitmix64, rng.hpp:16-53) are produced on the host and
 *                     the engine runs on them -> bit-exact with the reference. */
typedef enum { BB_RNG_PHILOX = 0, BB_RNG_REFERENCE = 1 } bb_rng_kind;

/* SimConfig, simulator.hpp:62-74 (+ the BinConfig edges, binning.hpp:23-29). */
typedef struct bb_sim_config {
  double arrival_rate;     /* requests per unit time; +INFINITY == kOverload */
  uint64_t n_requests;
  uint64_t batch_size;
  uint64_t n_servers;      /* S >= 1 (Philox generated mode: S > 1 needs a finite rate) */
  uint64_t seed;
  int32_t flush_partial;   /* default 1 */
  int32_t has_max_batch_wait; /* timers, simulator.hpp:70 */
  double max_batch_wait;
  const double* edges;     /* k+1 strictly increasing, top may be +inf */
  uint64_t n_edges;
  int32_t error_kind;      /* bb_error_kind */
  int32_t service_kind;    /* bb_service_kind */
  double p_error;          /* Symmetric */
  const double* confusion; /* Confusion: row-major rows[true-1][pred-1], confusion_k^2 */
  double lo, hi;           /* Uniform [lo,hi]; Linear len range */
  double rate;             /* Exponential */
  double lin_a, lin_b;     /* Linear: t = lin_b*len + lin_a */
  double mu, sigma;        /* LogNormal */
  const double* table;     /* Empirical samples / trace lengths */
  uint64_t n_table;
  int32_t rng;             /* bb_rng_kind */
  int32_t device;          /* CUDA ordinal; -1 = current */
  uint64_t confusion_k;    /* rows (== columns) of `confusion`; must equal k
                              ("sim config: confusion matrix size does not match
                              bin count", simulator.hpp:163-165) */
} bb_sim_config;

/* SimMetrics, simulator.hpp:76-87 */
typedef struct bb_sim_metrics {
  double throughput;
  double makespan;
  double latency_mean;
  double latency_p50;
  double latency_p99;
  double server_busy_fraction;
  uint64_t n_completed;
  uint64_t n_batches;
  uint64_t k;
  uint64_t per_bin_batch_counts[BB_MAX_BINS];
  double busy_time;    /* sum of batch service times (diagnostic) */
  double latency_sum;  /* sum of completed latencies (diagnostic) */
} bb_sim_metrics;

/* SimResult requests / batches (simulator.hpp:37-54, :89-93), caller-owned.
 * Any pointer may be NULL.  Request arrays hold n_requests entries; batch
 * arrays hold batch_capacity entries (n_requests always suffices); members
 * holds n_requests ids.  Batches are in dispatch order == the reference's
 * `batches` vector order. */
typedef struct bb_sim_detail {
  double* req_arrival;
  double* req_service;
  uint8_t* req_true_bin;
  uint8_t* req_pred_bin;
  uint32_t* req_batch;       /* BB_NO_BATCH == kNoBatch */
  double* req_completion;    /* NaN when unserved */
  uint64_t batch_capacity;
  uint8_t* bat_bin;
  uint32_t* bat_size;
  uint32_t* bat_first;       /* offset of the batch's members in members[] */
  double* bat_formed;
  double* bat_start;
  double* bat_finish;
  double* bat_service;
  uint32_t* members;         /* ascending request ids per batch */
} bb_sim_detail;

/* Trace-mode inputs: the engine consumes the request streams instead of
 * drawing them (the reference's detail::Engine, simulator.hpp:118-326, driven
 * by given arrivals/services/error uniforms). */
typedef struct bb_trace_in {
  const double* arrivals;  /* n, non-decreasing (required) */
  const double* services;  /* n (required) */
  const double* u_err;     /* n or NULL: error-stream uniforms (binning.hpp:240,251) */
  const uint8_t* pred_bin; /* n or NULL: predicted bins 1..k, overrides the error model */
} bb_trace_in;

/* PointResult, experiment.hpp:166-184 */
typedef struct bb_point_result {
  double arrival_rate;
  uint64_t k, batch_size, n_servers;
  int32_t error_kind;
  double p_error;
  uint64_t n_requests, replications;
  double throughput_mean, throughput_std;
  double latency_mean, latency_std;
  double latency_p50, latency_p99;
  double makespan_mean, busy_fraction_mean;
  double analytic_throughput, analytic_latency, analytic_max_throughput;
} bb_point_result;

/* Per-replication metrics as run_point collects them (experiment.hpp:256-265),
 * structure-of-arrays on the device: [6][n_points * replications]. */
enum { BB_REP_THROUGHPUT = 0, BB_REP_LATENCY = 1, BB_REP_P50 = 2, BB_REP_P99 = 3,
       BB_REP_MAKESPAN = 4, BB_REP_BUSY = 5, BB_REP_FIELDS = 6 };

/* RunTemplate / ServiceSpec / BinRule / ErrorSpec, experiment.hpp:34-73 */
typedef enum { BB_KIND_UNIFORM = 0, BB_KIND_EXPONENTIAL = 1, BB_KIND_TRACE = 2,
               BB_KIND_LINEAR = 3, BB_KIND_LOGNORMAL = 4 } bb_template_service;
typedef struct bb_run_template {
  double arrival_rate;
  uint64_t n_requests, batch_size, n_servers;
  int32_t flush_partial;
  int32_t has_max_batch_wait;
  double max_batch_wait;
  int32_t service;            /* bb_template_service */
  int32_t trace_cyclic;       /* trace: 1 = cyclic, 0 = resample (ServiceSpec default) */
  double min_time, max_time;  /* uniform; linear len range */
  double rate;                /* exponential */
  double lin_a, lin_b;        /* linear */
  double mu, sigma;           /* lognormal */
  const double* trace_times;  /* trace: resolved service times */
  uint64_t n_trace;
  uint64_t k;                 /* BinRule.k */
  const double* edges;        /* BinRule.edges (NULL -> derived) */
  uint64_t n_edges;
  int32_t error_kind;
  double p_error;
  const double* confusion;    /* the resolved matrix (ResolvedWorkload::confusion), row-major */
  uint64_t confusion_k;       /* its rows (== columns); checked against the point's k */
} bb_run_template;

/* SweepAxis / ExperimentSpec, experiment.hpp:75-87 */
typedef enum { BB_AXIS_LAMBDA = 0, BB_AXIS_K = 1, BB_AXIS_B = 2, BB_AXIS_P_E = 3,
               BB_AXIS_N_SERVERS = 4 } bb_axis_param;
typedef struct bb_sweep_axis {
  int32_t param;          /* bb_axis_param */
  const double* values;
  uint64_t n_values;
} bb_sweep_axis;
typedef struct bb_experiment_spec {
  bb_run_template base;
  bb_sweep_axis axes[2];
  uint64_t n_axes;        /* <= 2 */
  uint64_t replications;
  uint64_t seed;
  int32_t rng;            /* bb_rng_kind: PHILOX (fused kernel) or REFERENCE
                             (the reference's streams, bit-exact, slower) */
  const char* name;       /* ExperimentSpec::name (NULL: "experiment"); per-point
                             failures come back as BB_ERUNTIME "experiment '<name>':
                             sweep point <i> failed: ..." (experiment.hpp:352-358) */
} bb_experiment_spec;

/* ---------------------------------------------------------------- errors */
const char* bb_last_error(void);          /* thread-local message of the last failure */
int bb_abi_version(void);
bb_status bb_device_info(int32_t device, char* name, size_t name_len, int32_t* sm_count,
                         int32_t* cc_major, int32_t* cc_minor);

/* ------------------------------------------------ simulator.hpp entry points */
/* run_simulation, simulator.hpp:338 */
bb_status bb_run_simulation(const bb_sim_config* cfg, bb_sim_metrics* out);
/* run_simulation_detailed, simulator.hpp:331 */
bb_status bb_run_simulation_detailed(const bb_sim_config* cfg, bb_sim_metrics* out,
                                     bb_sim_detail* detail);
/* replay_trace, simulator.hpp:356 (lengths borrowed for the call) */
bb_status bb_replay_trace(const bb_sim_config* cfg, const double* lengths, uint64_t n_lengths,
                          bb_sim_metrics* out);
/* replay_trace_detailed, simulator.hpp:344 */
bb_status bb_replay_trace_detailed(const bb_sim_config* cfg, const double* lengths,
                                   uint64_t n_lengths, bb_sim_metrics* out,
                                   bb_sim_detail* detail);
/* detail::Engine::run on given streams (trace mode), simulator.hpp:128-150.
 * Host pointers in `in` and `detail`. */
bb_status bb_run_trace(const bb_sim_config* cfg, const bb_trace_in* in, bb_sim_metrics* out,
                       bb_sim_detail* detail);
/* Same, device pointers, stream-ordered except that the metrics (and any
 * error) are read back on `stream` before return. */
bb_status bb_run_trace_device(const bb_sim_config* cfg, const bb_trace_in* in_dev,
                              bb_sim_metrics* out, bb_sim_detail* detail_dev, void* stream);

/* ------------------------------------------------ experiment.hpp entry points */
/* replication_seed, experiment.hpp:90-92 */
uint64_t bb_replication_seed(uint64_t master, uint64_t rep);
/* run_point, experiment.hpp:254-307 (generated mode, all replications in one launch) */
bb_status bb_run_point(const bb_run_template* t, uint64_t master_seed, uint64_t replications,
                       bb_point_result* out);
/* run_experiment, experiment.hpp:312-370; `jobs` is accepted and ignored
 * (results never depend on it).  *n_points receives the point count; `out`
 * must hold that many (call with out == NULL to query). */
bb_status bb_run_experiment(const bb_experiment_spec* spec, unsigned jobs, bb_point_result* out,
                            uint64_t capacity, uint64_t* n_points);

/* Sharded sweep for multi-GPU callers (one process per GPU):
 * simulate replications [rep_begin, rep_end) of every point of `spec` on the
 * current device into the device array `rep_metrics_dev`
 * ([BB_REP_FIELDS][n_points*replications] doubles, replica-major within a
 * point; entries outside the shard are left untouched).  Stream-ordered (no
 * host synchronisation): a device-side error (a service outside the bin
 * support) is reported by the next *_reduce_device call on the device. */
bb_status bb_sweep_shard_device(const bb_experiment_spec* spec, uint64_t rep_begin,
                                uint64_t rep_end, double* rep_metrics_dev, void* stream);
/* The same for an explicit list of sweep points (points whose parameters do
 * not form a cartesian grid, e.g. lambda as a fraction of each point's
 * capacity).  Replication r of every point uses replication_seed(seed, r). */
bb_status bb_points_shard_device(const bb_run_template* points, uint64_t n_points,
                                 uint64_t replications, uint64_t seed, uint64_t rep_begin,
                                 uint64_t rep_end, double* rep_metrics_dev, void* stream);
/* run_point over a list of templates in one launch; host results. */
bb_status bb_run_points(const bb_run_template* points, uint64_t n_points, uint64_t replications,
                        uint64_t seed, int32_t rng, bb_point_result* out);
bb_status bb_points_reduce_device(const bb_run_template* points, uint64_t n_points,
                                  uint64_t replications, const double* rep_metrics_dev,
                                  bb_point_result* out, void* stream);
/* One process per GPU, gather instead of all-reduce: shard
 * [rep_begin, rep_end) written as its own block [BB_REP_FIELDS][n_points]
 * [rep_end - rep_begin] (no zero padding); the blocks of shards
 * [R c / C, R (c+1) / C), c = 0..C-1, concatenated in shard order (an
 * all-gather) are reduced by bb_points_reduce_gathered_device in replication
 * order, bit-identical to a single-device run.  Stream-ordered: a device-side
 * error is reported by the next reduce on the same device. */
bb_status bb_points_shard_local_device(const bb_run_template* points, uint64_t n_points,
                                       uint64_t replications, uint64_t seed, uint64_t rep_begin,
                                       uint64_t rep_end, double* shard_dev, void* stream);
bb_status bb_points_reduce_gathered_device(const bb_run_template* points, uint64_t n_points,
                                           uint64_t replications, uint32_t n_shards,
                                           const double* gathered_dev, bb_point_result* out,
                                           void* stream);
/* Devices the host-side sweeps (bb_run_experiment / bb_run_points /
 * bb_run_point, Philox streams) spread their replications over in this
 * process: one host thread per entry, results gathered on devices[0] by peer
 * stores and reduced there (the reference's std::thread pool over points,
 * experiment.hpp:342-368, as a pool over GPUs).  Entries may repeat (shards
 * on one device run on separate streams); n = 0 restores the default, the
 * calling thread's current device.  Results never depend on the list. */
bb_status bb_set_devices(const int32_t* devices, uint32_t n);
/* Per-point aggregation of a complete rep_metrics array (mean_std,
 * experiment.hpp:188-200 + run_point :266-306); blocks until `out` is filled. */
bb_status bb_sweep_reduce_device(const bb_experiment_spec* spec, const double* rep_metrics_dev,
                                 bb_point_result* out, void* stream);
/* Number of sweep points spec expands to (experiment.hpp:316-340). */
bb_status bb_experiment_points(const bb_experiment_spec* spec, uint64_t* n_points);

/* ------------------------------------------------ helpers (host formulas) */
/* uniform_boundaries / exponential_boundaries / empirical_boundaries,
 * binning.hpp:47-128; out holds k+1 doubles */
bb_status bb_uniform_boundaries(uint64_t k, double min_time, double max_time, double* out);
bb_status bb_exponential_boundaries(uint64_t k, double rate, uint64_t batch_size, double* out);
bb_status bb_empirical_boundaries(uint64_t k, const double* samples, uint64_t n, double* out);
/* analytics.hpp:55-108 closed forms */
double bb_analytic_throughput(uint64_t batch_size, uint64_t k, double lo, double hi);
double bb_analytic_latency(uint64_t batch_size, uint64_t k, double lo, double hi, double lambda);

/* analytics.hpp:55-126 with the reference's argument checks (BB_EINVAL on
 * B == 0, k == 0, !(0 <= lo < hi), a non-positive or infinite rate, ...). */
bb_status bb_expected_service_time(uint64_t batch_size, uint64_t bins, double min_time,
                                   double max_time, double* out);           /* :55-62 */
bb_status bb_throughput(uint64_t batch_size, uint64_t bins, double min_time, double max_time,
                        double* out);                                        /* :64-69 */
bb_status bb_max_throughput(uint64_t batch_size, double min_time, double max_time,
                            double* out);                                    /* :71-77 */
bb_status bb_min_bins_for_throughput(uint64_t batch_size, double min_time, double max_time,
                                     double epsilon, uint64_t* out);         /* :79-98 */
bb_status bb_expected_latency(uint64_t batch_size, uint64_t bins, double min_time,
                              double max_time, double arrival_rate, double* out); /* :100-108 */
bb_status bb_exponential_service_bound(uint64_t batch_size, uint64_t bins, double rate,
                                       double* out);                         /* :110-126 */
/* harmonic_number, service_dist.hpp:82-87 */
bb_status bb_harmonic_number(uint64_t n, double* out);
/* assign_bin, binning.hpp:133-144 (host; BB_EDOMAIN outside [e_0, e_k]) */
bb_status bb_assign_bin(const double* edges, uint64_t n_edges, double length, uint64_t* bin);
/* brute_force_boundaries, binning.hpp:268-351: family 0 = Uniform(p0, p1),
 * 1 = Exponential(rate p0); out holds k+1 edges */
bb_status bb_brute_force_boundaries(uint64_t k, int32_t family, double p0, double p1,
                                    uint64_t batch_size, uint64_t grid_points, double* out);

/* Philox4x32-10 on the host (the same function the kernels inline), for
 * known-answer tests: out[4] = philox(ctr[4], key[2]). */
void bb_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* The engine's exponential variates E = -log1p(-x 2^-53) (rng.hpp:43) of
 * 53-bit keys, on the device: table = 1 the inter-arrival gap function,
 * 0 the service-key function (accuracy tests). */
bb_status bb_exponential_variates(const uint64_t* keys, uint64_t n, int32_t table, double* out);

/* The bin edges a run template materialises to (materialize,
 * experiment.hpp:128-146; log-normal: exp(mu + sigma*Phi^-1(j/k)) with an open
 * top bin).  *n_edges receives k+1; out (may be NULL) must hold that many. */
bb_status bb_template_edges(const bb_run_template* t, double* out, uint64_t capacity,
                            uint64_t* n_edges);
/* The service time the generated-mode kernels assign to each 53-bit service
 * key (key = the Philox draw; cyclic traces: the table rank), on the device
 * -- lets a test rebuild a replication's services exactly. */
bb_status bb_service_of_keys(const bb_run_template* t, const uint64_t* keys, uint64_t n,
                             double* out);

/* Generated mode computes every replication's exact latency p50/p99 like the
 * reference's finish() (simulator.hpp:289-301), on by default.  Turning it off
 * (A/B measurements only) leaves p50/p99 NaN.  Returns the previous setting. */
int bb_set_generated_quantiles(int on);

/* Kernel launches issued by this thread since the last reset (evidence for
 * bench.py's gpu_launches). */
uint64_t bb_launch_count(int reset);
/* Host<->device bytes this library copied (cumulative; reset clears), for
 * bench.py's e2e h2d/d2h accounting. */
void bb_transfer_bytes(uint64_t* h2d_bytes, uint64_t* d2h_bytes, int reset);
/* Device time (ms, CUDA events on the launch stream) of the last dominant
 * kernel launched by this thread and the launch count it covered. */
double bb_last_kernel_ms(const char** name);
/* Trace-mode CUDA graph accounting (cumulative; reset clears): runs captured
 * into a graph and runs replayed from one.  The sync-free trace pipeline
 * (no max_batch_wait, no detail batch copies) is captured on the second
 * identical call and replayed from the third. */
void bb_trace_graph_stats(uint64_t* captures, uint64_t* replays, int reset);

#ifdef __cplusplus
}
#endif
#endif /* BINBATCH_B200_H */
