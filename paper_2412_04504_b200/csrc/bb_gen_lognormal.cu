// Fused generated-mode kernels for kSvcLogNormal services (bb_gen_kernel.cuh).
#include "bb_gen_kernel.cuh"

namespace bb {
template cudaError_t gen_run_svc<kSvcLogNormal>(const GenLaunch&, cudaStream_t);
}  // namespace bb
