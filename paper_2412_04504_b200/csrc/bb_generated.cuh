// bb_generated.cuh -- generated-mode (Philox) engine interface.
#pragma once
#include "bb_common.cuh"

namespace bb {

// One sweep point, flattened for the device (materialize(),
// experiment.hpp:110-155, resolved to key space).
struct GenPoint {
  SvcParams svc;
  double inv_lambda;        // 0 => overload (kOverload, simulator.hpp:33)
  uint32_t n, B, k;
  uint32_t flush;           // flush_partial
  uint32_t err_kind;        // 0 perfect, 1 symmetric, 2 confusion
  uint32_t check_domain;    // keys outside [vlo, vhi] raise domain_error
  uint32_t gidx;            // global point index (output row)
  uint32_t n_servers;       // S (simulator.hpp:68)
  double max_batch_wait;    // W > 0, or 0 (no timers; simulator.hpp:70)
  uint64_t vlo, vhi;
  uint64_t e_t1, e_t2;      // symmetric: u < p <=> x < t1 ; u >= 1-p <=> x >= t2
  const double* edges;      // k+1 (device), input of the threshold setup
  const uint64_t* conf_thr; // confusion: k*k cumulative thresholds (device)
  const uint32_t* cyc_rank; // cyclic: sorted rank of lengths[j] (device)
  uint64_t thr[BB_MAX_BINS + 1];  // thr[j], j=1..k-1: bin > j <=> x >= thr[j]
  // bin lookup over 256 key buckets (x >> bkt_shift): bkt[b] = (next << 8) | c
  // with c = #{j : thr[j] <= bucket start} and next = thr[c+1] (or 2^55 when
  // c+1 == k); bin = c + 1 + (x >= next).  Exact when no bucket holds two
  // thresholds (bkt_ok); otherwise the binary search over thr.
  uint64_t bkt[256];
  uint32_t bkt_shift;
  uint32_t bkt_ok;
};

struct GenLaunch {
  const GenPoint* pts_dev;  // n_points (thresholds already resolved)
  uint32_t n_points;        // points in this launch
  uint32_t points_total;    // rows of the output array
  uint32_t k_max;
  uint64_t master;          // run_point master seed; replica seed = replication_seed(master, r)
  int32_t single_seed;      // 1: replica 0 uses `master` itself as the seed (run_simulation)
  uint32_t reps_total;      // replications per point (array stride)
  uint32_t rep_begin, rep_end;
  int32_t err_kind;
  int32_t cyclic;
  int32_t svc_kind;          // SvcKind of every point in this launch
  int32_t overload;
  int32_t track;             // finite rate without flush: track open arrival sums
  double* out;              // [BB_REP_FIELDS][points_total][out_reps]
  uint32_t out_reps;        // replications per point row of `out` (0: reps_total)
  uint32_t out_rep0;        // replication stored in column 0 (a shard's own slice)
  AtanhCoef coef;           // exponential-variate polynomial (param space)
  uint32_t s_max;           // largest n_servers in the launch
  double* srv;              // server free times scratch (set by gen_run)
  uint32_t nb_max;          // overload, S > 1: most batches of any point (n/B + k)
  double* ovS;              // overload, S > 1: per-thread batch services (set by gen_run)
  uint16_t* ovM;            //   ... and member counts
  DevError* err;
  // quantile mode (bb_quantile.cuh): exact per-replication p50/p99
  int32_t timers;           // some point has max_batch_wait (the timer kernels)
  int32_t quant;
  uint32_t n_max;           // most requests of any point in the launch
  uint32_t nf_max;          // most batches of any point (n/B + k + 1)
  double* qA;               // request log: arrivals (set by gen_run; layout in bb_quantile.cuh)
  uint32_t* qI;             //   batch ids
  uint16_t* qK;             //   level-0 histogram bucket per request (selection scratch)
  double* qF;               //   completion per batch id [slot][q_nf]
  uint64_t q_n, q_nf;
};

// Grow-only per-device HBM scratch of the fused kernel, reused in stream
// order (acquire waits for the previous user's work; release records it).
cudaError_t gen_scratch_acquire(size_t bytes, cudaStream_t s, void** out);
void gen_scratch_release(cudaStream_t s);
// Bytes the scratch may grow to (free HBM + what it already holds, less a
// reserve).  want: what the caller needs; when the scratch already holds that
// much, its size is returned without querying the device (cudaMemGetInfo
// stalled the timed launches by 0.1-40 ms at random on the B200).
uint64_t gen_scratch_budget(uint64_t want = 0);

// Resolves key-space thresholds (bisection on the device sampler).
cudaError_t gen_setup_thresholds(GenPoint* pts_dev, uint32_t n_points, cudaStream_t s);
// The fused per-replica kernel of one service family (bb_gen_<family>.cu).
template <int SVC>
cudaError_t gen_run_svc(const GenLaunch& L, cudaStream_t s);
// The fused per-replica kernel.  Returns the launch error.
cudaError_t gen_run(const GenLaunch& L, cudaStream_t s);
// svc_of_key_t of every key (test support: bb_service_of_keys).
cudaError_t service_of_keys(const SvcParams& p, const uint64_t* x, uint64_t n, double* out,
                            cudaStream_t s);
// mean_std per point over replica order (experiment.hpp:188-200, :275-281).
// stats_out: [n_points][8] = thr mean, thr std, lat mean, lat std, p50, p99, makespan, busy
// chunks > 1: the array is the concatenation of `chunks` shard arrays, shard
// c holding replications [reps c / chunks, reps (c+1) / chunks) in its own
// [field][point][replication] layout (a gather of shard slices)
cudaError_t gen_point_reduce(const double* rep, uint32_t n_points, uint32_t reps,
                             double* stats_out, cudaStream_t s, uint32_t chunks = 1);

}  // namespace bb
