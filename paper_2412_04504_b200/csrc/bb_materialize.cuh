// bb_materialize.cuh -- Philox stream materialization for single runs.
#pragma once
#include "bb_common.cuh"

namespace bb {

struct MatArgs {
  uint32_t n;
  uint32_t c2, c3;        // whitened seed words (Philox counter c2:c3)
  int32_t overload;
  double inv_lambda;
  SvcParams svc;
  const uint32_t* cyc_rank;
  double* gap;            // scratch n
  double* s;              // out n
  double* u_err;          // out n or nullptr
  unsigned int* count;    // unused (nullptr)
};

// Draws gaps/services/error uniforms and scans gaps into `arrivals`.
cudaError_t materialize_streams(const MatArgs& M, double* arrivals, cudaStream_t s);
// E = -log1p(-x 2^-53) for 53-bit keys: table = 1 the gap variate of the
// generated engine (exp1_tab), 0 the service-key variate (exp1_from_bits53).
cudaError_t exp1_variates(const uint64_t* x, uint64_t n, int table, double* out, cudaStream_t s);

}  // namespace bb
