// bb_trace.cuh -- trace-mode (bit-exact) pipeline interface.
#pragma once
#include "bb_common.cuh"

namespace bb {

// Everything on the device; outputs optional (nullptr).
struct TraceArgs {
  uint32_t n, B, k;
  uint32_t n_servers;        // 0/1: Lindley scan; > 1: Kiefer-Wolfowitz dispatch
  int32_t flush;
  int32_t err_kind;          // 0 perfect, 1 symmetric, 2 confusion (needs u_err)
  double p_error;
  const double* edges;       // k+1 (device)
  const double* conf;        // k*k row-major (device) -- confusion rows
  const double* a;           // arrivals, non-decreasing
  const double* s;           // services
  const double* u_err;       // nullable
  const uint8_t* pred;       // nullable, overrides the error model
  double max_batch_wait;     // > 0: timers (simulator.hpp:200-201,223-235); 0: none
  // detail outputs (device, nullable)
  uint8_t* req_true_bin;
  uint8_t* req_pred_bin;   // copy of the partition's predicted bins
  uint32_t* req_batch;
  double* req_completion;
  uint8_t* bat_bin;
  uint32_t* bat_size;
  uint32_t* bat_first;
  double* bat_formed;
  double* bat_start;
  double* bat_finish;
  double* bat_service;
  uint32_t* members;
};

struct TraceResult {
  int status;               // bb_status
  char message[256];
  uint64_t n_batches, n_completed, k;
  uint64_t per_bin[BB_TRACE_MAX_BINS];
  double makespan, throughput, busy, busy_fraction, latency_sum, latency_mean, p50, p99;
  int32_t path;             // 0 fast (no tie group > B), 1 single tie group (overload)
  // timings (ms) of the stages, CUDA events on the launch stream
  float ms_partition, ms_total;
};

// Runs the pipeline on `stream`; synchronises on it (metrics are read back).
void trace_run(const TraceArgs& A, TraceResult* R, cudaStream_t stream);
// runs captured into / replayed from the pipeline's CUDA graph
void trace_graph_stats(uint64_t* captures, uint64_t* replays, bool reset);

}  // namespace bb
