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

}  // namespace bb
