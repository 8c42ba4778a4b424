// bb_generated.cu -- generated-mode host entry points: key-space threshold
// setup, the per-family kernel dispatch (bb_gen_kernel.cuh) and the
// per-point replica reduction.
#include <mutex>

#include "bb_generated.cuh"

namespace bb {
namespace {

__global__ void thresholds_kernel(GenPoint* pts, uint32_t n_points) {
  const uint32_t p = blockIdx.x;
  if (p >= n_points) return;
  GenPoint& P = pts[p];
  const uint32_t k = P.k;
  const uint64_t D = P.svc.key_domain;
  __shared__ uint64_t s_pos, s_above;
  for (uint32_t j = threadIdx.x; j <= k + 2; j += blockDim.x) {
    // smallest key whose service satisfies the predicate (monotone in the key)
    uint64_t lo = 0, hi = D;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      const double s = svc_of_key(P.svc, mid);
      bool ok;
      if (j <= k) ok = s >= P.edges[j];       // e_j <= s   (assign_bin upper_bound)
      else if (j == k + 1) ok = s > 0.0;      // positive   (simulator.hpp:189)
      else ok = s > P.edges[k];               // above the top edge (binning.hpp:135)
      if (ok) hi = mid;
      else lo = mid + 1;
    }
    if (j <= k) P.thr[j] = lo;
    else if (j == k + 1) s_pos = lo;
    else s_above = lo;
  }
  __syncthreads();
  // bucket table over the top 8 bits of the key domain
  {
    __shared__ int s_multi;
    uint32_t shift = 0;
    while (shift < 56 && ((D - 1) >> shift) >= 256) ++shift;
    if (threadIdx.x == 0) s_multi = 0;
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) {
      const uint64_t lo = (uint64_t)b << shift, hi = lo + (1ull << shift);
      uint32_t c = 0, inside = 0;
      for (uint32_t j = 1; j < k; ++j) {
        c += P.thr[j] <= lo;
        inside += P.thr[j] > lo && P.thr[j] < hi;
      }
      const uint64_t next = c + 1 < k ? P.thr[c + 1] : (1ull << 55);
      P.bkt[b] = (next << 8) | c;
      if (inside > 1) atomicOr(&s_multi, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      P.bkt_shift = shift;
      P.bkt_ok = !s_multi;
    }
  }
  if (threadIdx.x == 0) {
    const uint64_t vlo = P.thr[0] > s_pos ? P.thr[0] : s_pos;
    if (s_above == 0) {  // every key is above the support
      P.vlo = 1;
      P.vhi = 0;
      P.check_domain = 1;
    } else {
      P.vlo = vlo;
      P.vhi = s_above - 1;
      P.check_domain = !(vlo == 0 && s_above == D);
    }
  }
}

// mean_std (experiment.hpp:188-200) in replica order, bit-for-bit the
// reference's sequential sums: every operation is an explicitly rounded
// intrinsic, so no FMA contraction can fuse `ss += d * d` (the reference is
// built without -march, i.e. without contraction).  One block per
// point, one thread per field.
__global__ void point_reduce_kernel(const double* __restrict__ rep, uint32_t n_points,
                                    uint32_t reps, uint32_t chunks, double* __restrict__ out) {
  const uint32_t p = blockIdx.x, f = threadIdx.x;
  if (p >= n_points || f >= BB_REP_FIELDS) return;
  // replication i lives in chunk c = the shard [R c / C, R (c+1) / C) that
  // wrote it, laid out [field][point][its replications] at 6 P (R c / C)
  // (chunks = 1: the plain [field][point][replication] array)
  auto walk = [&](auto&& fn) {
    for (uint32_t c = 0; c < chunks; ++c) {
      const uint64_t lo = (uint64_t)reps * c / chunks, hi = (uint64_t)reps * (c + 1) / chunks;
      const uint64_t len = hi - lo;
      const double* x = rep + (uint64_t)BB_REP_FIELDS * n_points * lo + (uint64_t)f * n_points * len +
                        (uint64_t)p * len;
      for (uint64_t i = 0; i < len; ++i) fn(x[i]);
    }
  };
  const double nn = (double)reps;
  double sum = 0;
  walk([&](double x) { sum = __dadd_rn(sum, x); });
  const double mean = __ddiv_rn(sum, nn);
  double sd = 0;
  if (reps >= 2 && (f == BB_REP_THROUGHPUT || f == BB_REP_LATENCY)) {
    double ss = 0;
    walk([&](double x) {
      const double d = __dsub_rn(x, mean);
      ss = __dadd_rn(ss, __dmul_rn(d, d));
    });
    sd = __dsqrt_rn(__ddiv_rn(ss, __dsub_rn(nn, 1.0)));
  }
  double* o = out + (uint64_t)p * 8;
  switch (f) {
    case BB_REP_THROUGHPUT: o[0] = mean; o[1] = sd; break;
    case BB_REP_LATENCY: o[2] = mean; o[3] = sd; break;
    case BB_REP_P50: o[4] = mean; break;
    case BB_REP_P99: o[5] = mean; break;
    case BB_REP_MAKESPAN: o[6] = mean; break;
    case BB_REP_BUSY: o[7] = mean; break;
  }
}

// The service time the fused kernel assigns to each key (svc_of_key_t, the
// same inlined function and compilation flags as bb_gen_<family>.cu): lets a
// test rebuild a replication's services on the host (bb_service_of_keys).
template <int KIND>
__global__ void svc_keys_kernel(const SvcParams p, const uint64_t* __restrict__ x, uint64_t n,
                                double* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = svc_of_key_t<KIND>(p, x[i]);
}

}  // namespace

cudaError_t service_of_keys(const SvcParams& p, const uint64_t* x, uint64_t n, double* out,
                            cudaStream_t s) {
  if (!n) return cudaSuccess;
  const uint64_t b = (n + 255) / 256;
  const unsigned grid = (unsigned)(b < 4096 ? b : 4096);
  switch (p.kind) {
    case kSvcUniform: svc_keys_kernel<kSvcUniform><<<grid, 256, 0, s>>>(p, x, n, out); break;
    case kSvcLinear: svc_keys_kernel<kSvcLinear><<<grid, 256, 0, s>>>(p, x, n, out); break;
    case kSvcExponential: svc_keys_kernel<kSvcExponential><<<grid, 256, 0, s>>>(p, x, n, out); break;
    case kSvcLogNormal: svc_keys_kernel<kSvcLogNormal><<<grid, 256, 0, s>>>(p, x, n, out); break;
    case kSvcTable: svc_keys_kernel<kSvcTable><<<grid, 256, 0, s>>>(p, x, n, out); break;
    default: svc_keys_kernel<kSvcCyclic><<<grid, 256, 0, s>>>(p, x, n, out); break;
  }
  note_launch();
  return cudaGetLastError();
}

namespace {
struct Scratch {
  std::mutex mu;
  void* p = nullptr;
  size_t bytes = 0;
  cudaEvent_t ev = nullptr;
};
Scratch g_scratch[64];
int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return d & 63;
}
}  // namespace

cudaError_t gen_scratch_acquire(size_t bytes, cudaStream_t s, void** out) {
  Scratch& S = g_scratch[cur_dev()];
  S.mu.lock();
  cudaError_t e = cudaSuccess;
  if (!S.ev) e = cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming);
  else e = cudaStreamWaitEvent(s, S.ev, 0);
  if (e == cudaSuccess && bytes > S.bytes) {
    if (S.p) cudaFree(S.p);  // synchronises: earlier users are done
    S.p = nullptr;
    S.bytes = 0;
    e = cudaMalloc(&S.p, bytes);
    if (e == cudaSuccess) S.bytes = bytes;
    else S.p = nullptr;
  }
  if (e != cudaSuccess) {
    S.mu.unlock();
    return e;
  }
  *out = S.p;
  return cudaSuccess;
}

void gen_scratch_release(cudaStream_t s) {
  Scratch& S = g_scratch[cur_dev()];
  cudaEventRecord(S.ev, s);
  S.mu.unlock();
}

uint64_t gen_scratch_budget(uint64_t want) {
  const uint64_t held = g_scratch[cur_dev()].bytes;
  if (want && want <= held) return held;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return 0;
  const uint64_t have = free_b + g_scratch[cur_dev()].bytes;
  const uint64_t reserve = (uint64_t)6 << 30;  // leave room for the caller's own tensors
  return have > reserve ? (uint64_t)((have - reserve) * 0.92) : 0;
}

cudaError_t gen_setup_thresholds(GenPoint* pts_dev, uint32_t n_points, cudaStream_t s) {
  if (!n_points) return cudaSuccess;
  thresholds_kernel<<<n_points, 64, 0, s>>>(pts_dev, n_points);
  note_launch();
  return cudaGetLastError();
}

cudaError_t gen_run(const GenLaunch& L0, cudaStream_t s) {
  GenLaunch L = L0;
  L.coef = make_atanh_coef();
  switch (L.svc_kind) {
    case kSvcUniform: return gen_run_svc<kSvcUniform>(L, s);
    case kSvcLinear: return gen_run_svc<kSvcLinear>(L, s);
    case kSvcExponential: return gen_run_svc<kSvcExponential>(L, s);
    case kSvcLogNormal: return gen_run_svc<kSvcLogNormal>(L, s);
    case kSvcTable: return gen_run_svc<kSvcTable>(L, s);
    case kSvcCyclic: return gen_run_svc<kSvcCyclic>(L, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t gen_point_reduce(const double* rep, uint32_t n_points, uint32_t reps, double* stats,
                             cudaStream_t s, uint32_t chunks) {
  if (!n_points) return cudaSuccess;
  point_reduce_kernel<<<n_points, 32, 0, s>>>(rep, n_points, reps, chunks ? chunks : 1, stats);
  note_launch();
  return cudaGetLastError();
}

}  // namespace bb
