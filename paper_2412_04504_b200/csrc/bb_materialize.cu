// bb_materialize.cu -- Philox request streams for single runs
// (run_simulation / replay_trace in BB_RNG_PHILOX mode).
//
// One thread per request draws exactly the values the fused generated-mode
// kernel draws for that request (same counters), writes the inter-arrival
// gap, the service time s(key) and the error uniform, and a decoupled
// look-back scan turns the gaps into arrival times.  The trace pipeline then
// runs on these arrays, which yields per-request results (detailed mode) and
// exact latency quantiles for a single long replica.
#include "bb_common.cuh"
#include "bb_materialize.cuh"

namespace bb {
namespace {

constexpr int MT = 256, MI = 8, MTILE = MT * MI;

__global__ void draw_kernel(MatArgs M) {
  __shared__ double2 s_logtab[kLogTab];
  init_log_table(s_logtab);
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.n) return;
  const uint4 r = philox(i, kStreamArrivalService, M.c2, M.c3);
  const uint64_t xg = bits53(r.x, r.y);
  // the fused kernel's gap variate (bb_gen_kernel.cuh), so a materialized
  // replica equals the fused one
  M.gap[i] = M.overload ? 0.0 : exp1_tab(xg, s_logtab) * M.inv_lambda;
  uint64_t xs;
  if (M.svc.kind == kSvcCyclic) xs = M.cyc_rank[i % M.svc.n_table];
  else xs = bits53(r.z, r.w);
  M.s[i] = svc_of_key(M.svc, xs);
  if (M.u_err) {
    const uint4 e = philox(i >> 1, kStreamError, M.c2, M.c3);
    const uint64_t xe = (i & 1u) ? bits53(e.z, e.w) : bits53(e.x, e.y);
    M.u_err[i] = (double)xe * 0x1.0p-53;
  }
  if (M.count) atomicAdd(M.count, 1u);
}

// inclusive prefix sum of gaps -> arrivals (decoupled look-back, fp64)
__global__ void __launch_bounds__(MT) scan_kernel(const double* __restrict__ g, double* __restrict__ out,
                                                  uint32_t n, double* aggv, double* incv,
                                                  uint32_t* flag, uint32_t* counter) {
  __shared__ double s_w[MT / 32];
  __shared__ double s_pre;
  __shared__ uint32_t s_blk;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_blk = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const uint64_t d0 = (uint64_t)blk * MTILE + tid * MI;
  double v[MI];
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    v[i] = d0 + i < n ? g[d0 + i] : 0.0;
    acc += v[i];
    v[i] = acc;
  }
  double x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    double agg = 0.0;
    for (int q = 0; q < MT / 32; ++q) agg += s_w[q];
    if (lane == 0) {
      if (blk == 0) incv[0] = agg;
      else aggv[blk] = agg;
      __threadfence();
      atomicExch(&flag[blk], blk == 0 ? 2u : 1u);
    }
    double pre = 0.0;
    if (blk > 0) {  // warp-cooperative look-back: 32 predecessors per round trip
      int64_t base = (int64_t)blk - 1;
      while (true) {
        const int64_t p = base - (int64_t)lane;
        uint32_t f = 2;
        double v = 0.0;
        if (p >= 0) {
          do {
            f = *(volatile uint32_t*)&flag[p];
          } while (f == 0);
          __threadfence();
          v = f == 2 ? *(volatile double*)&incv[p] : *(volatile double*)&aggv[p];
        }
        const uint32_t incm = __ballot_sync(0xffffffffu, f == 2);
        const uint32_t last = incm ? (uint32_t)(__ffs(incm) - 1) : 31u;
        if (lane > last) v = 0.0;
        // sum in tile order (earliest first), as a sequential look-back would
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double other = __shfl_down_sync(0xffffffffu, v, o);
          if (lane + o <= last) v = other + v;
        }
        pre = __shfl_sync(0xffffffffu, v, 0) + pre;
        if (incm) break;
        base -= 32;
      }
      if (lane == 0) {
        incv[blk] = pre + agg;
        __threadfence();
        atomicExch(&flag[blk], 2u);
      }
    }
    if (lane == 0) s_pre = pre;
  }
  __syncthreads();
  double pre = s_pre;
  for (uint32_t q = 0; q < w; ++q) pre += s_w[q];
  const double xl = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane > 0) pre += xl;
#pragma unroll
  for (int i = 0; i < MI; ++i)
    if (d0 + i < n) out[d0 + i] = pre + v[i];
}

}  // namespace

cudaError_t materialize_streams(const MatArgs& M, double* arrivals, cudaStream_t s) {
  const uint32_t n = M.n;
  draw_kernel<<<(n + 255) / 256, 256, 0, s>>>(M);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  if (M.overload) return cudaMemsetAsync(arrivals, 0, (size_t)n * 8, s);
  const uint32_t nb = (n + MTILE - 1) / MTILE;
  double *aggv, *incv;
  uint32_t *flag, *counter;
  if ((e = cudaMallocAsync((void**)&aggv, (size_t)nb * 8, s))) return e;
  if ((e = cudaMallocAsync((void**)&incv, (size_t)nb * 8, s))) return e;
  if ((e = cudaMallocAsync((void**)&flag, (size_t)nb * 4 + 4, s))) return e;
  counter = flag + nb;
  if ((e = cudaMemsetAsync(flag, 0, (size_t)nb * 4 + 4, s))) return e;
  scan_kernel<<<nb, MT, 0, s>>>(M.gap, arrivals, n, aggv, incv, flag, counter);
  note_launch();
  e = cudaGetLastError();
  cudaFreeAsync(aggv, s);
  cudaFreeAsync(incv, s);
  cudaFreeAsync(flag, s);
  return e;
}

__global__ void exp1_kernel(const uint64_t* __restrict__ x, uint64_t n, int table,
                            double* __restrict__ out) {
  __shared__ double2 s_logtab[kLogTab];
  init_log_table(s_logtab);
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = table ? exp1_tab(x[i], s_logtab) : exp1_from_bits53(x[i]);
}

cudaError_t exp1_variates(const uint64_t* x, uint64_t n, int table, double* out, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const uint64_t blocks = (n + 255) / 256;
  exp1_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(x, n, table, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace bb
