/*
 * bb_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11) of the reference "binbatch" simulation path,
 * used as the parity checker for the B200 engine.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline leg may load it;
 * the product library (paper_2412_04504_b200/libbinbatch_b200.so) never links
 * or calls anything under oracle/.
 *
 * Parity pinning: this restatement is checked bit-for-bit against the
 * reference itself (oracle/_ref/libbbref.so, compiled from
 * /root/reference/proj/include by oracle/Makefile) and against the reference
 * tests' known-answer values (tests/golden/, tests/test_oracle_*.py).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/binbatch/).
 */
#ifndef BB_ORACLE_H
#define BB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes == the reference's exception types */
enum {
  BBO_OK = 0,
  BBO_EINVAL = 1,   /* std::invalid_argument */
  BBO_EDOMAIN = 2,  /* std::domain_error */
  BBO_ERUNTIME = 3, /* std::runtime_error */
  BBO_EUNSUPPORTED = 4
};

/* service kinds (service_dist.hpp:27-40 + simulator.hpp:344-354 trace modes,
 * plus the two injected samplers BASELINE configs 3 and 5 need) */
enum {
  BBO_SVC_UNIFORM = 0,     /* Uniform{lo,hi}: lo + (hi-lo)*u        rng.hpp:40 */
  BBO_SVC_EXPONENTIAL = 1, /* -log1p(-u)/rate                         rng.hpp:43 */
  BBO_SVC_EMPIRICAL = 2,   /* table[e() % n] (sorted table)           service_dist.hpp:98 */
  BBO_SVC_TRACE_CYCLIC = 3,   /* table[id % n]                        simulator.hpp:350 */
  BBO_SVC_TRACE_RESAMPLE = 4, /* table[e() % n]                       simulator.hpp:351 */
  BBO_SVC_ARRAYS = 5,      /* services[] given by the caller (trace mode) */
  BBO_SVC_LINEAR = 6,      /* t = a + b*len, len = lo + (hi-lo)*u      workload.hpp:167-170 */
  BBO_SVC_LOGNORMAL = 7    /* exp(mu + sigma*Z), Z Box-Muller from two service draws */
};

enum { BBO_ERR_PERFECT = 0, BBO_ERR_SYMMETRIC = 1, BBO_ERR_CONFUSION = 2 };

typedef struct {
  double arrival_rate;   /* +INFINITY == kOverload (simulator.hpp:33) */
  uint64_t n_requests;
  uint64_t batch_size;
  uint64_t n_servers;
  uint64_t seed;
  int32_t flush_partial;
  int32_t has_max_batch_wait;
  double max_batch_wait;
  const double* edges;   /* k+1 strictly increasing, top may be +inf */
  uint64_t n_edges;
  int32_t error_kind;
  int32_t service_kind;
  double p_error;
  const double* confusion; /* k*k row-major, rows[true-1][pred-1] */
  double lo, hi, rate;     /* uniform / exponential / linear-len range */
  double lin_a, lin_b;     /* linear: t = lin_a + lin_b*len */
  double mu, sigma;        /* lognormal */
  const double* table;     /* empirical samples (sorted) or trace lengths */
  uint64_t n_table;
} bbo_config;

typedef struct {
  /* optional caller-provided streams ("trace mode"); NULL -> generated from
   * the reference's RandomStream recipe with cfg->seed */
  const double* arrivals;  /* n, non-decreasing */
  const double* services;  /* n, required iff service_kind == ARRAYS */
  const double* u_err;     /* n, the error stream's uniforms, consumed only
                              when the error model draws (binning.hpp:239-251) */
  const uint8_t* pred_bin; /* n, predicted bins 1..k; overrides the error model */
} bbo_inputs;

typedef struct {
  double throughput, makespan, latency_mean, latency_p50, latency_p99;
  double server_busy_fraction;
  uint64_t n_completed;
  uint64_t n_batches;
  double busy_time;
  double latency_sum;
} bbo_metrics;

typedef struct {
  /* all optional (NULL = skip); request arrays have n entries, batch arrays
   * have room for n entries, members has room for n ids */
  double* req_arrival;
  double* req_service;
  uint32_t* req_true_bin;
  uint32_t* req_pred_bin;
  uint64_t* req_batch;      /* UINT64_MAX == kNoBatch */
  double* req_completion;   /* NaN when unserved */
  uint32_t* bat_bin;
  uint64_t* bat_size;
  uint64_t* bat_first;      /* offset of the batch's members in members[] */
  double* bat_formed;
  double* bat_start;
  double* bat_finish;
  double* bat_service;
  uint64_t* members;
  uint64_t* per_bin_batch_counts; /* k */
} bbo_detail;

/* rng.hpp:16-21 */
uint64_t bbo_splitmix64(uint64_t x);
/* experiment.hpp:90-92 */
uint64_t bbo_replication_seed(uint64_t master, uint64_t rep);
/* rng.hpp:33-35 + :38 -- n uniform01 draws of stream `stream_id` of `seed` */
void bbo_stream_uniform01(uint64_t seed, uint64_t stream_id, uint64_t n, double* out);
/* RandomStream(seed).uniform01() x n, rng.hpp:30,38 */
void bbo_plain_uniform01(uint64_t seed, uint64_t n, double* out);
/* schedule_arrivals, simulator.hpp:174-185 */
void bbo_generate_arrivals(uint64_t seed, double rate, uint64_t n, double* out);

/* binning.hpp:133-144; returns 0 and sets *bin, or BBO_EDOMAIN */
int bbo_assign_bin(const double* edges, uint64_t n_edges, double length, uint32_t* bin);

/* The engine: simulator.hpp:118-326 (+ run_simulation_detailed :331 and
 * replay_trace_detailed :344 for the sampler choice). */
int bbo_run(const bbo_config* cfg, const bbo_inputs* in, bbo_metrics* m, bbo_detail* d);

/* interpolated_quantile, binning.hpp:98-104 (sorted ascending input) */
double bbo_interpolated_quantile(const double* sorted, uint64_t n, double q);

/* mean_std, experiment.hpp:188-200 */
void bbo_mean_std(const double* xs, uint64_t n, double* mean, double* sd);

const char* bbo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
