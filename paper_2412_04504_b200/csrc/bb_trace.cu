// bb_trace.cu -- trace-mode pipeline: the reference engine's results,
// bit-for-bit, from given request streams.
//
//   K2 partition_kernel   one pass over the requests (decoupled look-back):
//        service check + assign_bin + predict_bin            binning.hpp:133-144, :231-261
//        stable per-bin rank (warp ballots, k-vector look-back) simulator.hpp:196-197
//        batch service = max over the B members (fragment maxima in smem,
//          open-batch max carried across tiles by a 2nd look-back) :237-254
//        closing records in closing-request order (R = closing arrival)   :198-199
//   finalize / order      drain partials, dispatch order (App. A.2)      :203-221
//   K5 Lindley            D = fl(max(D,R) + S): max-plus scan -> certified
//                         busy-period splits -> exact serial segments   :256-277
//   K6 request pass       completion, latency, sum, quantile keys        :279-301
//   select                exact order statistics for p50/p99 (radix refine)
//
// HBM layout: inputs a[], s[] (fp64, 8 B/request) and pred[] (u8) or u_err[]
// (fp64); per-request scratch pb8 (u8) + rank (u32); per-batch SoA records.
#include <algorithm>
#include <atomic>
#include <cstdio>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstring>
#include <vector>

#include "bb_trace.cuh"

namespace bb {
namespace {

constexpr unsigned long long KEY_UNSERVED = ~0ull;
constexpr uint32_t FL_NONMONO = 1, FL_TIE_GT_B = 2, FL_NOT_ALL_EQUAL = 4;
constexpr int LB = 256, LI = 8, LTILE = LB * LI;  // Lindley scan tile
constexpr int HBITS = 12, HBINS = 1 << HBITS;

__device__ __forceinline__ void st_release32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per-run facts computed on the device by finalize_kernel and read back.
struct Info {
  uint32_t nclose, nb, npartial, Z, path, flags;
  unsigned long long nc;
  uint32_t F[BB_TRACE_MAX_BINS], rem[BB_TRACE_MAX_BINS], nbat[BB_TRACE_MAX_BINS];
  uint32_t bin_base[BB_TRACE_MAX_BINS];   // first map slot of bin b
  uint32_t dbase[BB_TRACE_MAX_BINS];      // overload+flush: drain position base of bin b
  unsigned long long dreq[BB_TRACE_MAX_BINS];  // overload+flush: requests before bin b's drain
  uint32_t pfirst[BB_TRACE_MAX_BINS];     // fast path: members offset of bin b's partial
  uint32_t cfirst[BB_TRACE_MAX_BINS];     // overload: closing index of batch (b,0)
  uint32_t tpos[BB_TRACE_MAX_BINS];       // overload + timers: timer batch position after the closings
  uint32_t treq[BB_TRACE_MAX_BINS];       //   ... and requests in timer batches before it
  uint32_t sbase[BB_TRACE_MAX_BINS];      // first batch-maximum slot (WS::smax) of bin b
};

struct WS {
  uint32_t* counters;            // [1] lindley tiles, [2] binade tiles
  uint32_t* tcount;              // [k][ntiles] per-tile bin counts -> exclusive tile prefixes
  unsigned long long* smax;      // batch services (IEEE bits) at sbase[bin] + j
  uint8_t* pb8;
  uint32_t* rank;
  double* recR;
  uint8_t* recBin;
  uint32_t *recJ, *recC;
  unsigned long long* fin_cnt;   // [k] requests per bin
  uint32_t* flags;
  DevError* err;
  Info* info;
};

struct PartArgs {
  const double* a;
  const double* s;
  const double* u_err;
  const uint8_t* pred;
  const double* edges;
  const double* conf;
  uint8_t* tb_out;
  uint32_t n, B, k, ntiles;
  uint32_t vec_ok;  // every array 16-byte aligned (8 for the predictions): vector and bulk loads
  int32_t err_kind;
  double p, one_minus_p;
  FastDiv divB;
  WS ws;
};

// assign_bin, binning.hpp:133-144 (0 = out of support)
__device__ __forceinline__ uint32_t assign_bin(const double* e, uint32_t k, double len) {
  if (!(len >= e[0]) || !(len <= e[k])) return 0;
  if (len == e[k]) return k;
  uint32_t lo = 1, hi = k;  // first index in [1,k] with e[idx] > len
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (e[mid] > len) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// ----------------------------------------------------------- K2 partition
// Three streaming passes over the requests -- no look-back chain, so no tile
// waits for another:
//   count_kernel  per tile of PTILE requests: the predicted bin of every
//                 request (written to pb8 when it is drawn from u_err; a given
//                 pred[] is used in place), per-bin counts by warp ballots
//   tscan_kernel  per bin: exclusive prefix of the tile counts (in place),
//                 totals, and the slot base of each bin's batch maxima
//   place_kernel  per tile: service checks, stable rank of every request in
//                 its bin (tile prefix + in-warp match_any ranks), batch
//                 service = max over the members (fragment maxima in shared
//                 memory, then one global atomicMax per (bin, batch) fragment
//                 on the IEEE bits of the positive services), closing records
//                 in closing-request order (closings before the tile are
//                 sum_b floor(prefix_b / B))
constexpr int PT = 256, PIPT = 8, PTILE = PT * PIPT, PNW = PT / 32;


// the predicted bin of request idx (0: invalid, error raised); tb: true bin
__device__ __forceinline__ uint32_t part_bin(const PartArgs& P, const double* edges, uint64_t idx,
                                             double sv, uint32_t& tb) {
  const uint32_t k = P.k;
  tb = 0;
  if (!(sv > 0) || !isfinite(sv)) {
    raise_error(P.ws.err, idx, BB_EDOMAIN, sv, 1);  // simulator.hpp:189-190
    return 0;
  }
  if ((tb = assign_bin(edges, k, sv)) == 0) {
    raise_error(P.ws.err, idx, BB_EDOMAIN, sv, 2);  // binning.hpp:135-140
    return 0;
  }
  if (P.err_kind == 1) {  // Symmetric, binning.hpp:238-246
    const double u = P.u_err[idx];
    if (tb == 1) return u < P.p ? 2 : 1;
    if (tb == k) return u < P.p ? k - 1 : k;
    if (u < P.p) return tb - 1;
    if (u >= P.one_minus_p) return tb + 1;
    return tb;
  }
  if (P.err_kind == 2) {  // Confusion, binning.hpp:247-257
    const double u = P.u_err[idx];
    const double* row = P.conf + (uint64_t)(tb - 1) * k;
    double cum = 0.0;
    for (uint32_t q = 0; q < k; ++q) {
      cum = __dadd_rn(cum, row[q]);
      if (u < cum) return q + 1;
    }
    return k;
  }
  return tb;
}

// Counting needs no order: thread t takes the PIPT consecutive requests at
// tile + t * PIPT, loaded as one 8-byte vector of predictions (or 16-byte
// vectors of services and error uniforms) when aligned.  Blocks stride over
// the tiles (a few per block, the next tile's predictions loaded while the
// current one is counted): per-tile work is small, so block launches and
// load latency, not bytes, would bound a block per tile.
__device__ __forceinline__ uint2 count_load_pred(const PartArgs& P, uint32_t tile, uint32_t tid) {
  const uint64_t i0 = (uint64_t)tile * PTILE + (uint64_t)tid * PIPT;
  if (i0 + PIPT <= P.n && P.vec_ok) return *reinterpret_cast<const uint2*>(P.pred + i0);
  uint2 v = make_uint2(0, 0);
#pragma unroll
  for (int j = 0; j < PIPT; ++j)
    if (i0 + j < P.n) (j < 4 ? v.x : v.y) |= (uint32_t)P.pred[i0 + j] << (8 * (j & 3));
  return v;
}

template <int NG>  // 4-bit count groups of 8 bins: ceil(k / 8)
__global__ void __launch_bounds__(PT) count_kernel(PartArgs P) {
  __shared__ double s_edges[BB_TRACE_MAX_BINS + 1];
  __shared__ uint32_t s_cnt[PNW][32];
  static_assert(PIPT == 8, "one 8-byte vector of predictions per thread");
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t k = P.k, n = P.n;
  uint2 nxt = make_uint2(0, 0);
  if (P.pred && blockIdx.x < P.ntiles) nxt = count_load_pred(P, blockIdx.x, tid);
  for (uint32_t i = tid; i <= k; i += PT) s_edges[i] = P.edges[i];
  __syncthreads();
  for (uint32_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    const uint64_t i0 = (uint64_t)tile * PTILE + (uint64_t)tid * PIPT;
    const bool full = i0 + PIPT <= n && P.vec_ok;
    uint32_t b[PIPT];
    if (P.pred) {
      const uint2 v = nxt;
      if (tile + gridDim.x < P.ntiles) nxt = count_load_pred(P, tile + gridDim.x, tid);
#pragma unroll
      for (int j = 0; j < PIPT; ++j) b[j] = ((j < 4 ? v.x : v.y) >> (8 * (j & 3))) & 0xFF;
      // every byte in [1, k]? (four at a time; the per-request check only on a miss or the tail)
      const uint32_t kk = k * 0x01010101u;
      const bool ok = i0 + PIPT <= n && !(__vcmpeq4(v.x, 0u) | __vcmpeq4(v.y, 0u) |
                                          __vcmpgtu4(v.x, kk) | __vcmpgtu4(v.y, kk));
      if (!ok) {
#pragma unroll
        for (int j = 0; j < PIPT; ++j)
          if (i0 + j < n && (b[j] < 1 || b[j] > k)) {
            raise_error(P.ws.err, i0 + j, BB_EINVAL, (double)b[j], 3);
            b[j] = 0;
          }
      }
    } else {
      double sv[PIPT];
      if (full) {
#pragma unroll
        for (int j = 0; j < PIPT; j += 2) {
          const double2 x = *reinterpret_cast<const double2*>(P.s + i0 + j);
          sv[j] = x.x;
          sv[j + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < PIPT; ++j) sv[j] = i0 + j < n ? P.s[i0 + j] : 0.0;
      }
      uint32_t tbs[PIPT];
#pragma unroll
      for (int j = 0; j < PIPT; ++j) {
        b[j] = tbs[j] = 0;
        if (i0 + j < n) b[j] = part_bin(P, s_edges, i0 + j, sv[j], tbs[j]);
      }
      if (full) {  // predicted (and true) bins, one vector store each
        uint2 pv = make_uint2(0, 0), tv = make_uint2(0, 0);
#pragma unroll
        for (int j = 0; j < PIPT; ++j) {
          (j < 4 ? pv.x : pv.y) |= b[j] << (8 * (j & 3));
          (j < 4 ? tv.x : tv.y) |= tbs[j] << (8 * (j & 3));
        }
        *reinterpret_cast<uint2*>(P.ws.pb8 + i0) = pv;
        if (P.tb_out) *reinterpret_cast<uint2*>(P.tb_out + i0) = tv;
      } else {
#pragma unroll
        for (int j = 0; j < PIPT; ++j)
          if (i0 + j < n) {
            P.ws.pb8[i0 + j] = (uint8_t)b[j];
            if (P.tb_out) P.tb_out[i0 + j] = (uint8_t)tbs[j];
          }
      }
    }
    // per-thread counts in 4-bit fields (bin q+1 at nib[q / 8], bits 4 (q % 8);
    // at most PIPT = 8 per thread), then spread to 16-bit fields and summed over
    // the warp with one integer reduction per four bins (<= 256 per field)
    uint32_t nib[NG] = {};
#pragma unroll
    for (int j = 0; j < PIPT; ++j) {
      if (NG == 1) {  // b in [0, 8] (0: invalid, not counted)
        nib[0] += b[j] ? 1u << (4 * b[j] - 4) : 0u;
      } else {
        const uint32_t q = b[j] - 1, inc = b[j] ? 1u << (4 * (q & 7)) : 0u;
#pragma unroll
        for (int g = 0; g < NG; ++g) nib[g] += (q >> 3) == (uint32_t)g ? inc : 0u;
      }
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const uint32_t ev = nib[g] & 0x0F0F0F0Fu, od = (nib[g] >> 4) & 0x0F0F0F0Fu;
      const uint32_t r0 = __reduce_add_sync(0xffffffffu, ev & 0x00FF00FFu);         // bins 8g+1, +5
      const uint32_t r1 = __reduce_add_sync(0xffffffffu, (ev >> 8) & 0x00FF00FFu);  // bins 8g+3, +7
      const uint32_t r2 = __reduce_add_sync(0xffffffffu, od & 0x00FF00FFu);         // bins 8g+2, +6
      const uint32_t r3 = __reduce_add_sync(0xffffffffu, (od >> 8) & 0x00FF00FFu);  // bins 8g+4, +8
      if (lane == 0) {
        const uint32_t c[8] = {r0 & 0xFFFF, r2 & 0xFFFF, r1 & 0xFFFF, r3 & 0xFFFF,
                               r0 >> 16, r2 >> 16, r1 >> 16, r3 >> 16};
#pragma unroll
        for (int q = 0; q < 8; ++q) s_cnt[w][8 * g + q] = c[q];
      }
    }
    __syncthreads();
    if (w == 0 && lane < k) {
      uint32_t c = 0;
      for (int w2 = 0; w2 < PNW; ++w2) c += s_cnt[w2][lane];
      P.ws.tcount[(uint64_t)lane * P.ntiles + tile] = c;  // bin-major: a bin's tiles contiguous
    }
    __syncthreads();  // s_cnt is rewritten by the next tile
  }
}

// one block per bin: exclusive scan of its row of tile counts (each thread a
// contiguous run of tiles, all loads in flight, one block-wide scan)
constexpr int TS_T = 1024, TS_R = 8;  // threads, tiles per thread per round
__global__ void __launch_bounds__(TS_T) tscan_kernel(WS ws, uint32_t ntiles, uint32_t k, uint32_t B) {
  __shared__ uint32_t s_w[TS_T / 32];
  __shared__ uint32_t s_carry;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5, b = blockIdx.x;
  uint32_t* row = ws.tcount + (uint64_t)b * ntiles;
  if (tid == 0) s_carry = 0;
  for (uint32_t t0 = 0; t0 < ntiles; t0 += TS_T * TS_R) {
    uint32_t v[TS_R], sum = 0;
#pragma unroll
    for (int r = 0; r < TS_R; ++r) {
      const uint32_t t = t0 + tid * TS_R + r;
      v[r] = t < ntiles ? row[t] : 0u;
      sum += v[r];
    }
    uint32_t x = sum;  // inclusive scan of the thread sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    __syncthreads();  // s_carry of the previous round is final
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t y = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= (uint32_t)o) y += z;
      }
      s_w[lane] = y - s_w[lane];  // exclusive warp offsets
    }
    __syncthreads();
    uint32_t run = s_carry + s_w[w] + x - sum;
#pragma unroll
    for (int r = 0; r < TS_R; ++r) {
      const uint32_t t = t0 + tid * TS_R + r;
      if (t < ntiles) row[t] = run;
      run += v[r];
    }
    __syncthreads();
    if (tid == TS_T - 1) s_carry = run;
  }
  __syncthreads();
  if (tid == 0) ws.fin_cnt[b] = s_carry;
}


// Three barriers per tile: warp 0 lays out the tile's per-bin bases while
// every warp ranks its own requests (no barrier before that); each warp then
// adds the earlier warps' counts itself.
template <bool TBOUT>  // true bins requested with given predictions (detail output)
__global__ void __launch_bounds__(PT, 3) place_kernel(PartArgs P) {
  __shared__ uint32_t s_run[PNW][32];   // per warp: its requests per bin
  __shared__ uint32_t s_base[PNW][32];  // per warp: its rank base per bin
  __shared__ uint32_t s_excl[32];       // tile prefix per bin
  __shared__ uint32_t s_fr0[32];        // fragment index of the bin's batch 0 (fbase - jlo)
  __shared__ uint32_t s_soff[32];       // smax slot of fragment f of the bin: f + soff
  __shared__ uint32_t s_shi[PTILE + 32], s_slo[PTILE + 32];  // fragment maxima: high, low words
  __shared__ uint8_t s_fbin[PTILE + 32];                     // the bin of each fragment
  __shared__ uint32_t s_wclose[PNW], s_wflags[PNW];
  __shared__ uint32_t s_closebase, s_nfrag_total;

  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t k = P.k, n = P.n, B = P.B, t = blockIdx.x;
  // the tile's requests first: their loads are in flight across the prologue
  const uint64_t wbase = (uint64_t)t * PTILE + w * (32 * PIPT);
  const double a0 = P.a[0];
  const uint8_t* pbsrc = P.pred ? P.pred : P.ws.pb8;
  double av[PIPT], sv[PIPT];
  uint32_t pr[PIPT];  // predicted bin | rank within the warp's requests of that bin << 8
#pragma unroll
  for (int j = 0; j < PIPT; ++j) {
    const uint64_t idx = wbase + j * 32 + lane;
    const bool v = idx < n;
    av[j] = v ? P.a[idx] : 0.0;
    sv[j] = v ? P.s[idx] : 0.0;
    pr[j] = v ? pbsrc[idx] : 0u;
  }
  s_run[w][lane] = 0;
  if (w == 0) {  // the tile's per-bin bases (read after the first barrier)
    uint32_t jlo = 0, nfrag = 0, excl = 0;
    if (lane < k) {
      excl = P.ws.tcount[(uint64_t)lane * P.ntiles + t];
      const uint32_t nxt = t + 1 < P.ntiles ? P.ws.tcount[(uint64_t)lane * P.ntiles + t + 1]
                                            : (uint32_t)P.ws.fin_cnt[lane];
      jlo = P.divB.div(excl);
      nfrag = nxt > excl ? P.divB.div(nxt - 1) - jlo + 1 : 0;  // batches this tile touches
    }
    // batch-maximum slots: floor(total / B) full + 1 open batch per bin
    const uint32_t nslot = lane < k ? P.divB.div((uint32_t)P.ws.fin_cnt[lane]) + 1 : 0u;
    uint32_t incl = nfrag, sincl = nslot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      const uint32_t sv2 = __shfl_up_sync(0xffffffffu, sincl, o);
      if (lane >= (uint32_t)o) incl += v, sincl += sv2;
    }
    const uint32_t fbase = incl - nfrag, sbase = sincl - nslot;
    if (lane < k) {
      s_excl[lane] = excl;
      s_fr0[lane] = fbase - jlo;
      s_soff[lane] = sbase + jlo - fbase;
      if (t == 0) P.ws.info->sbase[lane] = sbase;  // for the kernels after this one
      for (uint32_t x = 0; x < nfrag; ++x) s_fbin[fbase + x] = (uint8_t)lane;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t i = lane; i < total; i += 32) s_shi[i] = s_slo[i] = 0u;
    uint32_t cb = lane < k ? jlo : 0;  // closings before this tile = sum_b floor(excl_b / B)
#pragma unroll
    for (int o = 16; o; o >>= 1) cb += __shfl_xor_sync(0xffffffffu, cb, o);
    if (lane == 0) {
      s_closebase = cb;
      s_nfrag_total = total;
    }
  }
#pragma unroll
  for (int j = 0; j < PIPT; ++j)
    if (pr[j] > k) pr[j] = 0;  // an invalid given prediction (count_kernel reported it)
  __syncwarp();

  uint32_t flags = 0, ties = 0;
  const uint32_t lt = lanemask_lt();
  // service support test on the IEEE bits: positive finite doubles order
  // like their bit patterns, so lo <= x <= hi is one subtraction and one
  // unsigned compare (negative, NaN and infinite services fall outside)
  const double e_lo = P.edges[0], e_hi = P.edges[k];
  const double lo_v = e_lo > 0 ? e_lo : 4.9406564584124654e-324;
  const bool none = !(e_hi >= lo_v) || isnan(e_lo);
  const unsigned long long lo_b = (unsigned long long)__double_as_longlong(lo_v);
  const unsigned long long span =
      none ? 0ull : (unsigned long long)__double_as_longlong(fmin(e_hi, 1.7976931348623157e308)) - lo_b;
  uint32_t pbk[PIPT / 4] = {};  // the bins, packed (the records need them after pr holds ranks)
#pragma unroll
  for (int j = 0; j < PIPT; ++j) {
    const uint64_t idx = wbase + j * 32 + lane;
    const bool valid = idx < n;
    const uint32_t pb = pr[j];
    pbk[j / 4] |= pb << (8 * (j & 3));
    // predecessor arrival for the monotonicity / tie checks
    double prev = __shfl_up_sync(0xffffffffu, av[j], 1);
    const double prevj = __shfl_sync(0xffffffffu, av[j > 0 ? j - 1 : 0], 31);
    if (lane == 0) prev = j > 0 ? prevj : (idx > 0 && valid ? P.a[idx - 1] : av[j]);
    if (valid) {
      if (idx > 0) {
        if (!(av[j] >= prev)) flags |= FL_NONMONO;
        else if (av[j] == prev) ties |= 1u << j;  // checked against a[idx - B] below (rare)
      }
      if (av[j] != a0) flags |= FL_NOT_ALL_EQUAL;
      if (P.pred) {  // given predictions: the services are still checked (and binned)
        const double sj = sv[j];
        if (TBOUT) {
          uint32_t tb = 0;
          if (!(sj > 0) || !isfinite(sj)) raise_error(P.ws.err, idx, BB_EDOMAIN, sj, 1);
          else if ((tb = assign_bin(P.edges, k, sj)) == 0) raise_error(P.ws.err, idx, BB_EDOMAIN, sj, 2);
          P.tb_out[idx] = (uint8_t)tb;
        } else if (none || (unsigned long long)__double_as_longlong(sj) - lo_b > span) {
          raise_error(P.ws.err, idx, BB_EDOMAIN, sj, !(sj > 0) || !isfinite(sj) ? 1 : 2);
        }
      }
    }
    // stable rank within the warp's requests of the same bin (match_any)
    const uint32_t peers = __match_any_sync(0xffffffffu, pb);
    const uint32_t mine = pb ? peers : 0u;
    const uint32_t run = pb ? s_run[w][pb - 1] : 0u;
    pr[j] = pb | ((run + __popc(mine & lt)) << 8);
    __syncwarp();
    if (pb && !(mine & lt)) s_run[w][pb - 1] = run + __popc(mine);
    __syncwarp();
  }
  if (ties) {  // a run of equal arrivals: longer than B?
#pragma unroll
    for (int j = 0; j < PIPT; ++j) {
      const uint64_t idx = wbase + j * 32 + lane;
      if (((ties >> j) & 1u) && idx >= B && P.a[idx - B] == av[j]) flags |= FL_TIE_GT_B;
    }
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0) s_wflags[w] = flags;
  __syncthreads();  // (1) per-warp counts, the tile's bases
  if (lane < k) {  // this warp's rank base per bin: tile prefix + earlier warps
    uint32_t acc = s_excl[lane];
    for (uint32_t w2 = 0; w2 < w; ++w2) acc += s_run[w2][lane];
    s_base[w][lane] = acc;
  }
  if (tid == 0) {
    uint32_t f = 0;
#pragma unroll
    for (int w2 = 0; w2 < PNW; ++w2) f |= s_wflags[w2];
    if (f) atomicOr(P.ws.flags, f);
  }
  __syncwarp();

  // global rank, batch, fragment maximum (the IEEE bits of the positive
  // services order like their values: a max of the high words, then of the
  // low words among the members holding that high word -- native 32-bit
  // shared atomics); closings counted per warp
  uint32_t wclose = 0, cmask = 0;
  uint32_t fr[PIPT];
#pragma unroll
  for (int j = 0; j < PIPT; ++j) {
    const uint32_t pb = pr[j] & 0xFF;
    bool closing = false;
    fr[j] = ~0u;
    if (pb) {
      const uint32_t b = pb - 1;
      const uint32_t rk = s_base[w][b] + (pr[j] >> 8);
      const uint32_t jb = P.divB.div(rk);
      fr[j] = s_fr0[b] + jb;
      atomicMax(&s_shi[fr[j]], (uint32_t)__double2hiint(sv[j]));
      closing = rk - jb * B == B - 1;
      pr[j] = jb;  // from here on: the batch (the bin stays in pbk)
      const uint64_t idx = wbase + j * 32 + lane;
      P.ws.rank[idx] = rk;
    }
    cmask |= (uint32_t)closing << j;
    wclose += __popc(__ballot_sync(0xffffffffu, closing));
  }
  if (lane == 0) s_wclose[w] = wclose;
  __syncthreads();  // (2) high words final
#pragma unroll
  for (int j = 0; j < PIPT; ++j)
    if (fr[j] != ~0u && s_shi[fr[j]] == (uint32_t)__double2hiint(sv[j]))
      atomicMax(&s_slo[fr[j]], (uint32_t)__double2loint(sv[j]));
  // closing records, in closing-request order (dispatch order on the fast path)
  uint32_t run = s_closebase;
  for (uint32_t w2 = 0; w2 < w; ++w2) run += s_wclose[w2];
#pragma unroll
  for (int j = 0; j < PIPT; ++j) {
    const bool closing = (cmask >> j) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, closing);
    if (closing) {
      const uint64_t idx = wbase + j * 32 + lane;
      const uint32_t q = run + __popc(bal & lt);
      P.ws.recR[q] = av[j];
      P.ws.recBin[q] = (uint8_t)(pbk[j / 4] >> (8 * (j & 3)));
      P.ws.recJ[q] = pr[j];
      P.ws.recC[q] = (uint32_t)idx;
    }
    run += __popc(bal);
  }
  __syncthreads();  // (3) low words final
  // fragment maxima into the (bin, batch) slots: one global max per fragment
  for (uint32_t f = tid; f < s_nfrag_total; f += PT)
    atomicMax(P.ws.smax + f + s_soff[s_fbin[f]], ((unsigned long long)s_shi[f] << 32) | s_slo[f]);
}

// the service of batch (bin b+1, j): max over its members (place_kernel)
__device__ __forceinline__ double batch_service(const WS& ws, uint32_t b, uint32_t j) {
  return __longlong_as_double((long long)ws.smax[ws.info->sbase[b] + j]);
}

// Drain partials, batch counts, dispatch-order bases (one warp).
__global__ void finalize_kernel(WS ws, const double* a, uint32_t n, uint32_t k, uint32_t B,
                                int32_t flush, double mbw) {
  const uint32_t lane = threadIdx.x;
  Info* I = ws.info;
  const uint32_t fl = *ws.flags;
  // overload without flush but with max_batch_wait: the partial batches form
  // when their timers fire at W (simulator.hpp:223-235)
  const bool tmo = !(fl & FL_NOT_ALL_EQUAL) && !(fl & FL_NONMONO) && !flush && mbw > 0;
  uint32_t F = 0, rem = 0, part = 0;
  if (lane < k) {
    const uint32_t cnt = (uint32_t)ws.fin_cnt[lane];
    F = cnt / B;
    rem = cnt - F * B;
    part = (flush || tmo) && rem > 0;
  }
  auto scan = [&](uint32_t v) {
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    return x;  // inclusive
  };
  const uint32_t nbat = F + part;
  const uint32_t ib = scan(nbat), iF = scan(F), ip = scan(part), iz = scan(F >= 1 ? 1u : 0u);
  const uint32_t dcount = (F ? F - 1 : 0) + part;
  const uint32_t id = scan(dcount);
  const uint32_t prem = part ? rem : 0;
  const uint32_t ipr = scan(prem);
  const uint32_t nclose = __shfl_sync(0xffffffffu, iF, 31);
  const uint32_t npart = __shfl_sync(0xffffffffu, ip, 31);
  const uint32_t Z = __shfl_sync(0xffffffffu, iz, 31);
  // requests before bin b's drain batches (overload + flush)
  unsigned long long dr = (unsigned long long)B * (F ? F - 1 : 0) + prem, idr = dr;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, idr, o);
    if (lane >= o) idr += y;
  }
  if (lane < k) {
    I->F[lane] = F;
    I->rem[lane] = rem;
    I->nbat[lane] = nbat;
    I->bin_base[lane] = ib - nbat;
    I->dbase[lane] = id - dcount;
    I->dreq[lane] = (unsigned long long)B * Z + (idr - dr);
    I->pfirst[lane] = nclose * B + (ipr - prem);
    I->cfirst[lane] = 0xFFFFFFFFu;
    if (part) {  // on_drain partial: formed at the last arrival (simulator.hpp:203-205,220)
      const uint32_t q = nclose + (ip - part);
      ws.recR[q] = tmo ? mbw : a[n - 1];  // (or by its timer at W)
      ws.recBin[q] = (uint8_t)(lane + 1);
      ws.recJ[q] = F;
      ws.recC[q] = 0xFFFFFFFFu;
    }
  }
  unsigned long long ncl = lane < k ? (unsigned long long)F * B + ((flush || tmo) ? rem : 0) : 0;
  for (int o = 16; o; o >>= 1) ncl += __shfl_xor_sync(0xffffffffu, ncl, o);
  if (lane == 0) {
    I->nclose = nclose;
    I->npartial = npart;
    I->nb = nclose + npart;
    I->Z = Z;
    I->nc = ncl;
    I->flags = fl;
    I->path = (fl & FL_NONMONO) ? 3 : !(fl & FL_NOT_ALL_EQUAL) ? 1 : (fl & FL_TIE_GT_B) ? 2 : 0;
  }
}

// overload + timers: every bin's first arrival (rank 0 in its bin)
__global__ void first_arrival_kernel(const uint8_t* __restrict__ pb8, const uint32_t* __restrict__ rank,
                                     uint32_t n, uint32_t* first) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && rank[i] == 0 && pb8[i]) first[pb8[i] - 1] = i;
}

// Overload: closing index of each bin's first batch (round-0 order key).
__global__ void ovl_first_kernel(WS ws) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (ws.info->path != 1) return;  // (launched before the host knows the path)
  if (q < ws.info->nclose && ws.recJ[q] == 0) ws.info->cfirst[ws.recBin[q] - 1] = ws.recC[q];
}

// Dispatch position of every record + map (bin, j) -> position + member offset.
// path 0: closing order, partials after (App. A.2 strictly increasing arrivals)
// path 1: one tie group (overload): rounds in first-closing order, drains.
__global__ void order_kernel(WS ws, uint32_t* map, uint32_t* order, uint32_t* dfirst,
                             uint32_t k, uint32_t B, int32_t flush, int32_t path, int32_t tmo) {
  const Info* I = ws.info;
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= I->nb) return;
  if (path < 0) {  // the device's own path (path 2 starts from closing order)
    path = I->path == 2 ? 0 : (int32_t)I->path;
    if (path == 3) return;
  }
  const uint32_t b = ws.recBin[q] - 1, j = ws.recJ[q];
  const bool partial = q >= I->nclose;
  uint32_t pos;
  unsigned long long before;
  if (path == 0) {
    pos = q;
    before = partial ? I->pfirst[b] : (unsigned long long)q * B;
  } else {
    const uint32_t Fb = I->F[b];
    if (partial && tmo) {  // timer batches at W, after every t = 0 formation
      pos = I->nclose + I->tpos[b];
      before = (unsigned long long)B * I->nclose + I->treq[b];
    } else if (partial) {
      pos = I->Z + I->dbase[b] + (Fb ? Fb - 1 : 0);
      before = I->dreq[b] + (unsigned long long)B * (Fb ? Fb - 1 : 0);
    } else if (flush && j >= 1) {
      pos = I->Z + I->dbase[b] + (j - 1);
      before = I->dreq[b] + (unsigned long long)B * (j - 1);
    } else {
      const uint32_t cb = I->cfirst[b];
      uint32_t p = 0;
      for (uint32_t q2 = 0; q2 < k; ++q2) {
        const uint32_t F = I->F[q2];
        if (!flush) p += F < j ? F : j;
        p += (I->cfirst[q2] < cb) && (F > j);
      }
      pos = p;
      before = (unsigned long long)B * p;
    }
  }
  order[pos] = q;
  map[I->bin_base[b] + j] = pos;
  dfirst[pos] = (uint32_t)before;
}

// ------------------------------------------------ general tie groups (path 2)
// A maximal group G = [s, e) of equal arrival times t.
// Every bin enters G with fewer than B queued, all of G's arrivals (rank 1)
// are processed before any formation at t (rank 2), and a bin schedules one
// formation, at its closing request c_b (queue.size() == B,
// simulator.hpp:196-199).  on_formation re-schedules itself at the back while
// the bin still holds >= B (:208-216), so the batches formed at t go out in
// rounds: round j holds every bin with more than j batches in G, in c_b
// order.  In the final group with flush the drains (scheduled after round 0's
// formations, :202-205) take, bin by bin, the remaining full batches and then
// the partial (:218-221); the re-scheduled formations then find < B.
// A group of at most B arrivals forms at most one batch per bin, in closing
// order: the fast path's identity.  So only groups of more than B arrivals
// are re-ordered here, each inside its own range of closing records.

// groups of more than B equal arrivals: (start, end) pairs, any order
__global__ void tie_groups_kernel(const double* __restrict__ a, uint32_t n, uint32_t B, uint2* groups,
                                  uint32_t* ngroups, const Info* I) {
  if (I->path != 2) return;  // (launched before the host knows the path)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = a[i];
    if (i > 0 && a[i - 1] == v) continue;
    if ((uint64_t)i + B >= n || a[i + B] != v) continue;
    uint32_t lo = i + B + 1, hi = n;  // first index past the group (a is non-decreasing)
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (a[mid] == v) lo = mid + 1;
      else hi = mid;
    }
    groups[atomicAdd(ngroups, 1u)] = make_uint2(i, lo);
  }
}

struct TieArgs {
  const uint2* groups;
  const uint32_t* ngroups;
  uint32_t ntiles;                  // partition tiles (WS::tcount: exclusive tile prefixes)
  WS ws;
  uint32_t *map, *order, *dfirst;
  uint32_t n, k, B;
  int32_t flush;
};

// One block per group: per-bin counts at its ends (tile prefix + the tile's
// head), the round-robin / drain position of each of its records.
__global__ void __launch_bounds__(256) tie_order_kernel(TieArgs T) {
  __shared__ uint32_t s_c[2][32], s_F[32], s_j0[32], s_cf[32], s_rem[32];
  __shared__ uint32_t s_fb[32], s_pc[32], s_pr[32];
  __shared__ uint32_t s_qlo, s_qhi, s_Z;
  const Info* I = T.ws.info;
  const uint32_t tid = threadIdx.x, k = T.k, B = T.B;
  for (uint32_t g = blockIdx.x; g < *T.ngroups; g += gridDim.x) {
    const uint2 G = T.groups[g];
    __syncthreads();
    if (tid < 32) s_c[0][tid] = s_c[1][tid] = 0;
    __syncthreads();
    // count_b[0, x) = the tile's exclusive prefix + this tile's head
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const uint32_t x = side ? G.y : G.x;
      const uint32_t t = x / PTILE;
      if (tid < k)
        atomicAdd(&s_c[side][tid], t < T.ntiles ? T.ws.tcount[(uint64_t)tid * T.ntiles + t] : (uint32_t)T.ws.fin_cnt[tid]);
      for (uint32_t i = t * PTILE + tid; i < x; i += blockDim.x) {
        const uint32_t b = T.ws.pb8[i];
        if (b - 1u < k) atomicAdd(&s_c[side][b - 1], 1u);
      }
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t cs = tid < k ? s_c[0][tid] : 0, ce = tid < k ? s_c[1][tid] : 0;
      const uint32_t js = cs / B, je = ce / B, F = je - js;
      s_F[tid] = F;
      s_j0[tid] = js;
      s_cf[tid] = 0xFFFFFFFFu;
      const uint32_t rem = (T.flush && G.y == T.n) ? ce - je * B : 0;  // the final partials
      s_rem[tid] = rem;
      uint32_t qlo = js, qhi = je, Z = F >= 1;
      // drain bookkeeping: exclusive sums over lower bins
      uint32_t fb = F ? F - 1 : 0, pc = rem != 0, pr = rem;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a1 = __shfl_up_sync(0xffffffffu, fb, o), a2 = __shfl_up_sync(0xffffffffu, pc, o),
                       a3 = __shfl_up_sync(0xffffffffu, pr, o);
        if (tid >= o) fb += a1, pc += a2, pr += a3;
      }
      s_fb[tid] = fb - (F ? F - 1 : 0);
      s_pc[tid] = pc - (rem != 0);
      s_pr[tid] = pr - rem;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        qlo += __shfl_xor_sync(0xffffffffu, qlo, o);
        qhi += __shfl_xor_sync(0xffffffffu, qhi, o);
        Z += __shfl_xor_sync(0xffffffffu, Z, o);
      }
      if (tid == 0) s_qlo = qlo, s_qhi = qhi, s_Z = Z;
    }
    __syncthreads();
    const uint32_t qlo = s_qlo, qhi = s_qhi;
    // c_b: the closing request of bin b's first batch in G (its round-0 key)
    for (uint32_t q = qlo + tid; q < qhi; q += blockDim.x) {
      const uint32_t b = T.ws.recBin[q] - 1;
      if (T.ws.recJ[q] == s_j0[b]) s_cf[b] = T.ws.recC[q];
    }
    __syncthreads();
    const bool final_drain = T.flush && G.y == T.n;
    const uint32_t qend = final_drain ? I->nb : qhi;
    for (uint32_t x = qlo + tid; x < qend; x += blockDim.x) {
      const uint32_t q = x < qhi ? x : I->nclose + (x - qhi);  // then the partial records
      if (q >= I->nb) break;
      const uint32_t b = T.ws.recBin[q] - 1, jg = T.ws.recJ[q], Fb = s_F[b];
      uint32_t pos;
      unsigned long long before;
      if (x >= qhi) {  // on_drain's partial, after the bin's remaining full batches
        const uint32_t f = s_fb[b] + (Fb ? Fb - 1 : 0);
        pos = qlo + s_Z + f + s_pc[b];
        before = (unsigned long long)B * (qlo + s_Z + f) + s_pr[b];
      } else {
        const uint32_t jr = jg - s_j0[b];
        if (final_drain && jr >= 1) {  // on_drain: full batches in bin order
          const uint32_t f = s_fb[b] + (jr - 1);
          pos = qlo + s_Z + f + s_pc[b];
          before = (unsigned long long)B * (qlo + s_Z + f) + s_pr[b];
        } else {  // round jr, first-closing order
          uint32_t p = 0;
          const uint32_t cb = s_cf[b];
          for (uint32_t b2 = 0; b2 < k; ++b2) {
            const uint32_t F2 = s_F[b2];
            if (!final_drain) p += F2 < jr ? F2 : jr;
            p += (s_cf[b2] < cb) && (F2 > jr);
          }
          pos = qlo + p;
          before = (unsigned long long)B * pos;
        }
      }
      T.order[pos] = q;
      T.map[I->bin_base[b] + jg] = pos;
      T.dfirst[pos] = (uint32_t)before;
    }
  }
}

__global__ void gather_kernel(WS ws, const uint32_t* order, int32_t path, uint32_t B, double* dR,
                              double* dS, uint8_t* dBin, uint32_t* dSize) {
  const Info* I = ws.info;
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= I->nb) return;
  if (path < 0) path = (int32_t)I->path;
  const uint32_t q = path == 0 ? d : order[d];
  dR[d] = ws.recR[q];
  dS[d] = batch_service(ws, ws.recBin[q] - 1, ws.recJ[q]);
  const uint8_t b = ws.recBin[q];
  if (dBin) dBin[d] = b;
  if (dSize) dSize[d] = q < I->nclose ? B : I->rem[b - 1];
}

// ---------------------------------------------------------------- Lindley
struct LArgs {
  const double* R;
  const double* S;
  const uint32_t* nbp;  // batch count (device: known after the partition)
  uint8_t* split;   // 1 = certified idle start, 2 = ambiguous, 0 = certified busy
  double* Dt;       // approximate D after each batch (binade prediction)
  double* busy_part;
  double *aggA, *aggC, *incA, *incC;
  uint32_t* flag;
  uint32_t* counter;
  double tol_rel;
};

enum : uint8_t { kBusy = 0, kSplit = 1, kAmbiguous = 2 };

struct MP {  // f(x) = max(x + A, C)
  double A, C;
};
__device__ __forceinline__ MP compose(const MP& f, const MP& g) {  // g after f
  return MP{f.A + g.A, fmax(f.C + g.A, g.C)};
}

// Warp-cooperative decoupled look-back (all 32 lanes of one warp): lane i
// inspects predecessor tile base-i, so one round trip covers 32
// predecessors.  `op(earlier, later)` is the scan's associative operator
// (not necessarily commutative); each window is reduced in tile order with
// shuffles.  load(p, inclusive) reads tile p's published value after its flag.
__device__ __forceinline__ double shfl_dn(double v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ double shfl_ix(double v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ MP shfl_dn(const MP& v, int o) {
  return MP{__shfl_down_sync(0xffffffffu, v.A, o), __shfl_down_sync(0xffffffffu, v.C, o)};
}
__device__ __forceinline__ MP shfl_ix(const MP& v, int l) {
  return MP{__shfl_sync(0xffffffffu, v.A, l), __shfl_sync(0xffffffffu, v.C, l)};
}

template <class T, class Load, class Op>
__device__ __forceinline__ T warp_lookback(const uint32_t* flag, int64_t t, T identity, Load load,
                                           Op op) {
  const uint32_t lane = threadIdx.x & 31;
  T acc = identity;  // composition of the windows already visited (the later part)
  int64_t base = t - 1;
  while (true) {
    const int64_t p = base - (int64_t)lane;
    uint32_t f = 2;
    T v = identity;
    if (p >= 0) {
      do {
        f = ld_acquire32(&flag[p]);
      } while (f == 0);
      v = load(p, f == 2);
    }
    const uint32_t incm = __ballot_sync(0xffffffffu, f == 2);
    const uint32_t last = incm ? (uint32_t)(__ffs(incm) - 1) : 31u;
    if (lane > last) v = identity;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T other = shfl_dn(v, o);
      if (lane + o <= last) v = op(other, v);
    }
    acc = op(shfl_ix(v, 0), acc);  // lane 0: v[last] then ... then v[0]
    if (incm) return acc;
    base -= 32;
  }
}

__global__ void __launch_bounds__(LB) lindley_scan_kernel(LArgs L) {
  __shared__ MP s_w[LB / 32];
  __shared__ MP s_prefix;
  __shared__ double s_busy[LB / 32];
  __shared__ uint32_t s_blk;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_blk = atomicAdd(L.counter, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const uint32_t nb = *L.nbp;
  if ((uint64_t)blk * LTILE >= nb) return;  // grid sized for the upper bound
  const uint64_t d0 = (uint64_t)blk * LTILE + tid * LI;
  double R[LI], S[LI];
  MP f{0.0, -CUDART_INF};
  double bs = 0.0;
#pragma unroll
  for (int i = 0; i < LI; ++i) {
    const bool v = d0 + i < nb;
    R[i] = v ? L.R[d0 + i] : -CUDART_INF;
    S[i] = v ? L.S[d0 + i] : 0.0;
    f = compose(f, MP{S[i], R[i] + S[i]});
    bs += S[i];
  }
  // inclusive scan over the block's threads
  MP x = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    MP y;
    y.A = __shfl_up_sync(0xffffffffu, x.A, o);
    y.C = __shfl_up_sync(0xffffffffu, x.C, o);
    if (lane >= o) x = compose(y, x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) bs += __shfl_xor_sync(0xffffffffu, bs, o);
  if (lane == 31) s_w[w] = x;
  if (lane == 0) s_busy[w] = bs;
  __syncthreads();
  if (w == 0) {
    MP agg{0.0, -CUDART_INF};
    for (int w2 = 0; w2 < LB / 32; ++w2) agg = compose(agg, s_w[w2]);
    if (lane == 0) {
      double b2 = 0.0;
      for (int w2 = 0; w2 < LB / 32; ++w2) b2 += s_busy[w2];
      L.busy_part[blk] = b2;
      if (blk == 0) {
        L.incA[0] = agg.A;
        L.incC[0] = agg.C;
      } else {
        L.aggA[blk] = agg.A;
        L.aggC[blk] = agg.C;
      }
      __threadfence();
      st_release32(&L.flag[blk], blk == 0 ? 2u : 1u);
    }
    MP pre{0.0, -CUDART_INF};
    if (blk > 0) {
      pre = warp_lookback(
          L.flag, blk, MP{0.0, -CUDART_INF},
          [&](int64_t p, bool inc) {
            return inc ? MP{*(volatile double*)&L.incA[p], *(volatile double*)&L.incC[p]}
                       : MP{*(volatile double*)&L.aggA[p], *(volatile double*)&L.aggC[p]};
          },
          [](const MP& a, const MP& b) { return compose(a, b); });
      if (lane == 0) {
        const MP inc = compose(pre, agg);
        L.incA[blk] = inc.A;
        L.incC[blk] = inc.C;
        __threadfence();
        st_release32(&L.flag[blk], 2);
      }
    }
    if (lane == 0) s_prefix = pre;
  }
  __syncthreads();
  // exclusive prefix of this thread = block prefix, earlier warps, earlier lanes
  MP pre = s_prefix;
  for (uint32_t w2 = 0; w2 < w; ++w2) pre = compose(pre, s_w[w2]);
  MP xl;
  xl.A = __shfl_up_sync(0xffffffffu, x.A, 1);
  xl.C = __shfl_up_sync(0xffffffffu, x.C, 1);
  if (lane > 0) pre = compose(pre, xl);
  double Dp = pre.C;  // applied to D_{-1} = -inf (server idle before the first batch)
#pragma unroll
  for (int i = 0; i < LI; ++i) {
    if (d0 + i < nb) {
      uint8_t code;
      if (Dp == -CUDART_INF) {
        code = kSplit;
      } else {
        const double tol = L.tol_rel * fmax(fabs(Dp), fabs(R[i]));
        code = R[i] > Dp + tol ? kSplit : (R[i] >= Dp - tol ? kAmbiguous : kBusy);
      }
      L.split[d0 + i] = code;
      Dp = fmax(Dp, R[i]) + S[i];
      L.Dt[d0 + i] = Dp;
    }
  }
}

// Exact serial recurrence inside every certified busy period.
__global__ void lindley_segments_kernel(const double* __restrict__ R, const double* __restrict__ S,
                                        const uint8_t* __restrict__ split, const uint32_t* nbp,
                                        double* __restrict__ start, double* __restrict__ finish,
                                        const int* __restrict__ bad) {
  if (!*bad) return;  // fallback only: the binade scan produced exact values
  const uint32_t nb = *nbp;
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nb || split[d] != kSplit) return;
  double D = __dadd_rn(R[d], S[d]);  // idle server: start = formation time
  start[d] = R[d];
  finish[d] = D;
  constexpr int CH = 16;
  for (uint32_t e0 = d + 1; e0 < nb; e0 += CH) {
    double r[CH], s[CH];
    uint8_t sp[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const bool v = e0 + i < nb;
      sp[i] = v ? split[e0 + i] == kSplit : 1;
      r[i] = v ? R[e0 + i] : 0.0;
      s[i] = v ? S[e0 + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (sp[i]) return;
      const double st = fmax(D, r[i]);
      D = __dadd_rn(st, s[i]);
      start[e0 + i] = st;
      finish[e0 + i] = D;
    }
  }
}

// ----------------------------------------------------- exact parallel Lindley
// Inside a busy period D_d = fl(D_{d-1} + S_d).  While D stays in one binade
// [2^E, 2^(E+1)) every value is a multiple of u = 2^(E-52): D = a*u with the
// integer a in [2^52, 2^53), and round-to-nearest-even of a*u + S is
//     a + q + [f > 1/2] + [f == 1/2 and (a + q) odd],   S/u = q + f,
// an increment that depends on a only through its parity.  Such maps
// (inc for even a, inc for odd a) compose associatively, so a segmented scan
// evaluates the sequential fp64 chain exactly.  Runs of one binade are cut at
// certified idle starts, ambiguous reset points and predicted binade
// crossings ("heads"); one thread per busy period then walks its few heads
// (exact fp64 steps), and every other batch reads its value from its run's
// head and its prefix map.  Any violated assumption (a prediction off by a
// binade) raises a flag and the host falls back to the serial kernel.
struct PMap {
  long long i0, i1;  // increment for even / odd starting integer
};
__device__ __forceinline__ PMap pcompose(const PMap& x, const PMap& y) {  // y after x
  return PMap{x.i0 + ((x.i0 & 1) ? y.i1 : y.i0), x.i1 + ((x.i1 & 1) ? y.i0 : y.i1)};
}
// x * 2^n as ldexp rounds it, by one multiplication when 2^n is a normal
// double (the library ldexp is a long branchy call)
__device__ __forceinline__ double ldexp2(double x, int n) {
  if (n >= -1022 && n <= 1023) return __dmul_rn(x, __longlong_as_double((long long)(n + 1023) << 52));
  return ldexp(x, n);
}
__device__ __forceinline__ int binade(double v) { return (int)((__double_as_longlong(v) >> 52) & 0x7FF) - 1023; }

// Is batch d a run head?  (needs d's code and the approximate D before/after)
__device__ __forceinline__ bool run_head(uint8_t code, double dprev, double dcur, double tol_rel) {
  if (code != kBusy) return true;
  if (!(dprev > 0.0) || !(dcur > 0.0)) return true;
  const int e = binade(dcur);
  if (binade(dprev) != e) return true;
  const double lo = ldexp2(1.0, e), hi = ldexp2(1.0, e + 1);
  return dprev < lo * (1.0 + 4 * tol_rel) || dcur > hi * (1.0 - 4 * tol_rel);
}

// map of one batch in binade e (q = floor(S/u), f = S/u - q exact)
__device__ __forceinline__ PMap batch_map(double S, int e) {
  const double x = ldexp2(S, 52 - e);
  const double qd = floor(x);
  const double f = x - qd;
  const long long q = (long long)qd;
  const long long up = f > 0.5;
  const long long half = f == 0.5;
  // a + q + 0.5 with (a+q) odd rounds up; even a: parity of q decides
  return PMap{q + up + (half & (q & 1)), q + up + (half & ((q + 1) & 1))};
}

// What the chain walk needs of a run, written once at its last batch: one
// dependent load per run head instead of three.
struct RunInfo {
  long long p0, p1;   // prefix map of the run's last batch
  double Rn, Sn;      // formation time and service of the batch after the run
  uint32_t last;      // the run's last batch
  int32_t e;          // the binade predicted for the run's last value
  uint32_t next_code; // split code of the batch after the run (kSplit: the busy period ends)
  uint32_t pad;
};

struct BArgs {
  const double* R;
  const double* S;
  const double* Dt;
  const uint8_t* code;
  const uint32_t* nbp;  // batch count (device)
  double tol_rel;
  long long* p0;       // prefix map per batch (within its run)
  long long* p1;
  uint32_t* head_of;   // run head of each batch
  uint32_t* run_last;  // last batch of each run, indexed by head
  RunInfo* run_info;   // ... and what the chain walk needs of it, indexed by head
  // look-back
  long long *ag0, *ag1, *in0, *in1;
  uint32_t *agh, *inh, *agf, *inf;  // head position (+1, 0 = none) and head flag
  uint32_t* flag;
  uint32_t* counter;
};

struct SegV {
  PMap m;
  uint32_t hp;   // 1 + index of the latest head (0 = none)
  uint32_t hf;   // contains a head
};
__device__ __forceinline__ SegV shfl_dn(const SegV& v, int o) {
  SegV r;
  r.m.i0 = __shfl_down_sync(0xffffffffu, v.m.i0, o);
  r.m.i1 = __shfl_down_sync(0xffffffffu, v.m.i1, o);
  r.hp = __shfl_down_sync(0xffffffffu, v.hp, o);
  r.hf = __shfl_down_sync(0xffffffffu, v.hf, o);
  return r;
}
__device__ __forceinline__ SegV shfl_ix(const SegV& v, int l) {
  SegV r;
  r.m.i0 = __shfl_sync(0xffffffffu, v.m.i0, l);
  r.m.i1 = __shfl_sync(0xffffffffu, v.m.i1, l);
  r.hp = __shfl_sync(0xffffffffu, v.hp, l);
  r.hf = __shfl_sync(0xffffffffu, v.hf, l);
  return r;
}
__device__ __forceinline__ SegV scomb(const SegV& x, const SegV& y) {  // y after x
  SegV r;
  r.m = y.hf ? y.m : pcompose(x.m, y.m);
  r.hp = y.hp > x.hp ? y.hp : x.hp;
  r.hf = x.hf | y.hf;
  return r;
}

__global__ void __launch_bounds__(LB) binade_scan_kernel(BArgs A) {
  __shared__ SegV s_w[LB / 32];
  __shared__ SegV s_pre;
  __shared__ uint32_t s_blk;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_blk = atomicAdd(A.counter, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const uint32_t nb = *A.nbp;
  if ((uint64_t)blk * LTILE >= nb) return;  // grid sized for the upper bound
  const uint64_t d0 = (uint64_t)blk * LTILE + tid * LI;
  SegV v[LI];
  SegV acc{{0, 0}, 0, 0};
#pragma unroll
  for (int i = 0; i < LI; ++i) {
    const uint64_t d = d0 + i;
    SegV e{{0, 0}, 0, 0};
    if (d < nb) {
      const double dcur = A.Dt[d];
      const double dprev = d ? A.Dt[d - 1] : -1.0;
      if (run_head(A.code[d], dprev, dcur, A.tol_rel)) {
        e.hf = 1;
        e.hp = (uint32_t)d + 1;
      } else {
        e.m = batch_map(A.S[d], binade(dcur));
      }
    }
    acc = scomb(acc, e);
    v[i] = acc;
  }
  SegV x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    SegV y;
    y.m.i0 = __shfl_up_sync(0xffffffffu, x.m.i0, o);
    y.m.i1 = __shfl_up_sync(0xffffffffu, x.m.i1, o);
    y.hp = __shfl_up_sync(0xffffffffu, x.hp, o);
    y.hf = __shfl_up_sync(0xffffffffu, x.hf, o);
    if (lane >= o) x = scomb(y, x);
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    SegV agg{{0, 0}, 0, 0};
    for (int q = 0; q < LB / 32; ++q) agg = scomb(agg, s_w[q]);
    if (lane == 0) {
      if (blk == 0) {
        A.in0[0] = agg.m.i0; A.in1[0] = agg.m.i1; A.inh[0] = agg.hp; A.inf[0] = agg.hf;
      } else {
        A.ag0[blk] = agg.m.i0; A.ag1[blk] = agg.m.i1; A.agh[blk] = agg.hp; A.agf[blk] = agg.hf;
      }
      __threadfence();
      st_release32(&A.flag[blk], blk == 0 ? 2u : 1u);
    }
    SegV pre{{0, 0}, 0, 0};
    if (blk > 0) {
      pre = warp_lookback(
          A.flag, blk, SegV{{0, 0}, 0, 0},
          [&](int64_t p, bool inc) {
            SegV t;
            if (inc) {
              t.m.i0 = *(volatile long long*)&A.in0[p]; t.m.i1 = *(volatile long long*)&A.in1[p];
              t.hp = *(volatile uint32_t*)&A.inh[p]; t.hf = *(volatile uint32_t*)&A.inf[p];
            } else {
              t.m.i0 = *(volatile long long*)&A.ag0[p]; t.m.i1 = *(volatile long long*)&A.ag1[p];
              t.hp = *(volatile uint32_t*)&A.agh[p]; t.hf = *(volatile uint32_t*)&A.agf[p];
            }
            return t;
          },
          [](const SegV& a, const SegV& b) { return scomb(a, b); });
      if (lane == 0) {
        const SegV inc = scomb(pre, agg);
        A.in0[blk] = inc.m.i0; A.in1[blk] = inc.m.i1; A.inh[blk] = inc.hp; A.inf[blk] = inc.hf;
        __threadfence();
        st_release32(&A.flag[blk], 2);
      }
    }
    if (lane == 0) s_pre = pre;
  }
  __syncthreads();
  SegV pre = s_pre;
  for (uint32_t q = 0; q < w; ++q) pre = scomb(pre, s_w[q]);
  SegV xl;
  xl.m.i0 = __shfl_up_sync(0xffffffffu, x.m.i0, 1);
  xl.m.i1 = __shfl_up_sync(0xffffffffu, x.m.i1, 1);
  xl.hp = __shfl_up_sync(0xffffffffu, x.hp, 1);
  xl.hf = __shfl_up_sync(0xffffffffu, x.hf, 1);
  if (lane > 0) pre = scomb(pre, xl);
#pragma unroll
  for (int i = 0; i < LI; ++i) {
    const uint64_t d = d0 + i;
    if (d >= nb) break;
    const SegV r = scomb(pre, v[i]);
    A.p0[d] = r.m.i0;
    A.p1[d] = r.m.i1;
    const uint32_t h = r.hp - 1;  // batch 0 is always a head
    A.head_of[d] = h;
    bool last = d + 1 == nb;
    if (!last) last = run_head(A.code[d + 1], A.Dt[d], A.Dt[d + 1], A.tol_rel);
    if (last) {
      A.run_last[h] = (uint32_t)d;
      RunInfo ri;
      ri.p0 = r.m.i0;
      ri.p1 = r.m.i1;
      ri.last = (uint32_t)d;
      ri.e = binade(A.Dt[d]);
      const bool more = d + 1 < nb;
      ri.next_code = more ? A.code[d + 1] : (uint32_t)kSplit;
      ri.Rn = more ? A.R[d + 1] : 0.0;
      ri.Sn = more ? A.S[d + 1] : 0.0;
      ri.pad = 0;
      A.run_info[h] = ri;
    }
  }
}


// one thread per busy period: walk its run heads (exact fp64 steps)
__global__ void binade_chain_kernel(const double* __restrict__ R, const double* __restrict__ S,
                                    const double* __restrict__ Dt, const uint8_t* __restrict__ code,
                                    const long long* __restrict__ p0, const long long* __restrict__ p1,
                                    const RunInfo* __restrict__ run_info, const uint32_t* nbp,
                                    double* __restrict__ start, double* __restrict__ finish,
                                    int* bad) {
  const uint32_t nb = *nbp;
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nb || code[d] != kSplit) return;
  uint32_t h = d;
  double D = __dadd_rn(R[h], S[h]);  // idle server: start = formation time
  start[h] = R[h];
  finish[h] = D;
  while (true) {
    const RunInfo ri = run_info[h];  // the walk's only dependent load per run
    if (ri.last != h) {  // run_end: the head's value through the run's prefix map
      if (binade(D) != ri.e) {
        *bad = 1;
        return;
      }
      const long long a = (long long)ldexp2(D, 52 - ri.e);
      const long long al = a + ((a & 1) ? ri.p1 : ri.p0);
      if (al > (1ll << 53)) *bad = 1;
      D = ldexp2((double)al, ri.e - 52);
    }
    const uint32_t nx = ri.last + 1;
    if (nx >= nb || ri.next_code == kSplit) return;
    h = nx;
    const double st = fmax(D, ri.Rn);  // ambiguous reset or binade crossing: exact step
    D = __dadd_rn(st, ri.Sn);
    start[h] = st;
    finish[h] = D;
  }
}

// every non-head batch: value from its run head and prefix map
__global__ void binade_fill_kernel(const double* __restrict__ S, const double* __restrict__ Dt,
                                   const uint8_t* __restrict__ code, const long long* __restrict__ p0,
                                   const long long* __restrict__ p1, const uint32_t* __restrict__ head_of,
                                   const uint32_t* nbp, double tol_rel, double* __restrict__ start,
                                   double* __restrict__ finish, int* bad) {
  const uint32_t nb = *nbp;
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nb) return;
  const double dprev = d ? Dt[d - 1] : -1.0;
  if (run_head(code[d], dprev, Dt[d], tol_rel)) return;
  const uint32_t h = head_of[d];
  const double Dh = finish[h];
  const int e = binade(Dt[d]);
  if (binade(Dh) != e) {
    *bad = 1;
    return;
  }
  const long long a = (long long)ldexp2(Dh, 52 - e);
  const long long ap = (d - 1 == h) ? a : a + ((a & 1) ? p1[d - 1] : p0[d - 1]);
  const long long ad = a + ((a & 1) ? p1[d] : p0[d]);
  const long long q = (long long)floor(ldexp2(S[d], 52 - e));
  if (ap + q >= (1ll << 53) || ad > (1ll << 53) || ap < (1ll << 52)) *bad = 1;
  start[d] = ldexp2((double)ap, e - 52);
  finish[d] = ldexp2((double)ad, e - 52);
}

// the last value of a device-counted array (0 when empty)
__global__ void last_of_kernel(const double* v, const uint32_t* nbp, double* out) {
  const uint32_t nb = *nbp;
  *out = nb ? v[nb - 1] : 0.0;
}

// --------------------------------- multi-server dispatch, chunk-parallel
// S > 1 servers (simulator.hpp:256-277): the central queue is FIFO, so batch
// i starts on the earliest-free server, start_i = max(R_i, min_j V_j), and
// that server's free time becomes finish_i = fl(start_i + S_i) (the
// Kiefer-Wolfowitz recursion; a server freed at R_i is idle for a batch
// formed at R_i because batch_done events rank first, :108-114).
// Kiefer-Wolfowitz in parallel: the batches split into chunks of KWP_CH;
// each chunk is first dispatched from an all-idle server state
// (kw_spec_kernel, one thread per chunk, its heap of S free times in global
// scratch).  That speculation is exact whenever every server is free at the
// chunk's first formation time: free times <= R_first stay <= every later R
// (R is non-decreasing in dispatch order), so they act exactly like -inf in
// start = max(R, min free).  kw_fix_kernel walks the chunks in order with
// the true incoming state and re-dispatches (serially, from that state) only
// the chunks whose check fails -- light load runs in parallel, heavy load
// degrades to the serial recursion.  The busy time (a sequential fp64 sum
// in dispatch order, simulator.hpp:263) comes from the exact Lindley
// pipeline run on (R = 0, S) (D_n = S_1 + ... + S_n in order).
constexpr uint32_t KWP_CH = 1024;

__device__ __forceinline__ void kw_run(const double* R, const double* S, uint32_t lo, uint32_t hi, double* heap,
                                       uint32_t nsrv, double* start, double* finish, double& last) {
  for (uint32_t j = lo; j < hi; ++j) {
    const double r = R[j], sv = S[j];  // (read before the in-place writes)
    const double st = fmax(heap[0], r);
    const double f = __dadd_rn(st, sv);
    start[j] = st;
    finish[j] = f;
    last = fmax(last, f);
    uint32_t h = 0;  // replace the minimum by f (f >= old minimum) and sift down
    for (;;) {
      uint32_t c = 2 * h + 1;
      if (c >= nsrv) break;
      if (c + 1 < nsrv && heap[c + 1] < heap[c]) ++c;
      if (!(heap[c] < f)) break;
      heap[h] = heap[c];
      h = c;
    }
    heap[h] = f;
  }
}

__global__ void kw_spec_kernel(const double* __restrict__ R, const double* __restrict__ S, const uint32_t* nbp,
                               uint32_t nsrv, double* heaps, double* __restrict__ start,
                               double* __restrict__ finish, double* chunk_last) {
  const uint32_t nb = *nbp, g = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lo = g * KWP_CH;
  if (lo >= nb) return;
  double* heap = heaps + (size_t)g * nsrv;
  for (uint32_t q = 0; q < nsrv; ++q) heap[q] = -CUDART_INF;  // all idle
  double last = 0.0;
  kw_run(R, S, lo, min(nb, lo + KWP_CH), heap, nsrv, start, finish, last);
  chunk_last[g] = last;
}

// The chunks in order (one block): a chunk whose check fails is staged in
// shared memory and re-dispatched by one thread from the true incoming
// state (its heap in shared memory up to KWP_HEAP servers).
constexpr uint32_t KWP_HEAP = 2048;
__global__ void __launch_bounds__(256) kw_fix_kernel(const double* __restrict__ R, const double* __restrict__ S,
                                                     const uint32_t* nbp, uint32_t nsrv, double* heaps,
                                                     double* __restrict__ start, double* __restrict__ finish,
                                                     double* chunk_last, double* last_out, uint32_t* refixed) {
  __shared__ double sR[KWP_CH], sS[KWP_CH];  // (R, S) in, (start, finish) out in place
  __shared__ double sheap[KWP_HEAP];
  __shared__ int s_fix;
  const uint32_t nb = *nbp, G = (nb + KWP_CH - 1) / KWP_CH;
  double last = G ? chunk_last[0] : 0.0, in_max = last;  // (the state's largest free time)
  uint32_t fixed = 0;
  for (uint32_t g = 1; g < G; ++g) {
    const uint32_t lo = g * KWP_CH, m = min(KWP_CH, nb - lo);
    if (threadIdx.x == 0) s_fix = !(in_max <= R[lo]);  // a server busy at the first formation
    __syncthreads();
    if (s_fix) {
      double* heap = nsrv <= KWP_HEAP ? sheap : heaps + (size_t)g * nsrv;
      const double* prev = heaps + (size_t)(g - 1) * nsrv;
      for (uint32_t q = threadIdx.x; q < nsrv; q += blockDim.x) heap[q] = prev[q];  // the true state
      for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
        sR[j] = R[lo + j];
        sS[j] = S[lo + j];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double cl = 0.0;
        kw_run(sR, sS, 0, m, heap, nsrv, sR, sS, cl);
        chunk_last[g] = cl;
        ++fixed;
      }
      __syncthreads();
      for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) {
        start[lo + j] = sR[j];
        finish[lo + j] = sS[j];
      }
      if (nsrv <= KWP_HEAP)  // the chunk's outgoing state, for the next chunk
        for (uint32_t q = threadIdx.x; q < nsrv; q += blockDim.x) heaps[(size_t)g * nsrv + q] = sheap[q];
      __syncthreads();
    }
    in_max = fmax(in_max, chunk_last[g]);
    last = fmax(last, chunk_last[g]);
  }
  if (threadIdx.x == 0) {
    *last_out = last;
    *refixed = fixed;
  }
}

// ------------------------------------------------------------- requests
struct QArgs {
  const double* a;
  const uint8_t* pb8;
  const uint32_t* rank;
  const uint32_t* map;
  const double* finish;
  const uint32_t* dfirst;
  const Info* info;
  FastDiv divB;
  uint32_t n, B, k;
  unsigned long long* key;
  double* lat_part;
  unsigned long long* kminmax;
  double* completion;
  uint32_t* batch;
  uint32_t* members;
};


#ifndef BB_RQ_E
#define BB_RQ_E 4
#endif
constexpr int RQ_T = 256, RQ_E = BB_RQ_E;  // request pass: threads, requests per thread
__global__ void __launch_bounds__(RQ_T) request_kernel(QArgs Q) {
  __shared__ double s_sum[RQ_T / 32];
  __shared__ unsigned long long s_min[RQ_T / 32], s_max[RQ_T / 32];
  __shared__ uint32_t s_nbat[BB_TRACE_MAX_BINS], s_base[BB_TRACE_MAX_BINS];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < BB_TRACE_MAX_BINS) {
    s_nbat[threadIdx.x] = Q.info->nbat[threadIdx.x];
    s_base[threadIdx.x] = Q.info->bin_base[threadIdx.x];
  }
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * (RQ_T * RQ_E) + threadIdx.x;
  uint32_t bin[RQ_E], rk[RQ_E], d[RQ_E];
  double a[RQ_E], comp[RQ_E];
  // every load of a stage in flight before the next stage uses it
#pragma unroll
  for (int e = 0; e < RQ_E; ++e) {
    const uint64_t i = base + e * RQ_T;
    const bool v = i < Q.n;
    bin[e] = v ? Q.pb8[i] : 0u;
    if (bin[e] > Q.k) bin[e] = 0;  // an invalid given prediction: the run reports the error
    rk[e] = v ? Q.rank[i] : 0u;
    a[e] = v ? Q.a[i] : 0.0;
  }
#pragma unroll
  for (int e = 0; e < RQ_E; ++e) {
    d[e] = BB_NO_BATCH;
    if (bin[e]) {
      const uint32_t j = Q.divB.div(rk[e]);
      if (j < s_nbat[bin[e] - 1]) d[e] = Q.map[s_base[bin[e] - 1] + j];
    }
  }
#pragma unroll
  for (int e = 0; e < RQ_E; ++e) comp[e] = d[e] != BB_NO_BATCH ? Q.finish[d[e]] : BB_QNAN;
  double lat = 0.0;
  unsigned long long kmin = KEY_UNSERVED, kmax = 0;
#pragma unroll
  for (int e = 0; e < RQ_E; ++e) {
    const uint64_t i = base + e * RQ_T;
    if (i >= Q.n) continue;
    unsigned long long key = KEY_UNSERVED;
    if (d[e] != BB_NO_BATCH) {
      const double x = __dsub_rn(comp[e], a[e]);  // simulator.hpp:294
      lat += x;
      key = (unsigned long long)__double_as_longlong(x);
      kmin = key < kmin ? key : kmin;
      kmax = key > kmax ? key : kmax;
      if (Q.members) Q.members[Q.dfirst[d[e]] + (rk[e] - Q.divB.div(rk[e]) * Q.B)] = (uint32_t)i;
    }
    Q.key[i] = key;
    if (Q.completion) Q.completion[i] = comp[e];
    if (Q.batch) Q.batch[i] = d[e];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lat += __shfl_xor_sync(0xffffffffu, lat, o);
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, kmin, o);
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmin = x < kmin ? x : kmin;
    kmax = y > kmax ? y : kmax;
  }
  if (lane == 0) {
    s_sum[w] = lat;
    s_min[w] = kmin;
    s_max[w] = kmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int q = 0; q < RQ_T / 32; ++q) {
      sum += s_sum[q];
      kmin = s_min[q] < kmin ? s_min[q] : kmin;
      kmax = s_max[q] > kmax ? s_max[q] : kmax;
    }
    Q.lat_part[blockIdx.x] = sum;
    if (kmin != KEY_UNSERVED) {
      atomicMin(&Q.kminmax[0], kmin);
      atomicMax(&Q.kminmax[1], kmax);
    }
  }
}

// deterministic sum of block partials (one block)
// nbp: m = the Lindley tiles of *nbp batches (device count)
__global__ void sum_kernel(const double* part, uint32_t m, double* out, const uint32_t* nbp = nullptr) {
  __shared__ double s[256];
  if (nbp) m = (*nbp + LTILE - 1) / LTILE;
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < m; i += 256) acc += part[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// the run's last completion (simulator.hpp:275; one server: the last batch's
// finish) and first arrival, for makespan = last - a[0] (:284-285)
__global__ void scalars_kernel(const Info* I, const double* finish, const double* last_ms,
                               const double* a, double* out) {
  const uint32_t nb = I->nb;
  out[0] = last_ms ? *last_ms : (nb ? finish[nb - 1] : 0.0);
  out[1] = a[0];
}

// --------------------------------------------------------------- selection
// Visit every key, four per thread per step (two 16-byte loads in flight).
template <class F>
__device__ __forceinline__ void for_keys(const unsigned long long* __restrict__ key, uint32_t m, F&& f) {
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < m; i += step) {
    if (i + 4 <= m) {
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(key + i);
      const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(key + i + 2);
      f(x.x);
      f(x.y);
      f(y.x);
      f(y.y);
    } else {
      for (uint64_t q = i; q < m; ++q) f(key[q]);
    }
  }
}

__global__ void hist_kernel(const unsigned long long* __restrict__ key, uint32_t m,
                            unsigned long long lo, unsigned long long hi, uint32_t shift,
                            uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[HBINS];
  for (int i = threadIdx.x; i < HBINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for_keys(key, m, [&](unsigned long long v) {
    if (v >= lo && v <= hi) atomicAdd(&h[(uint32_t)((v - lo) >> shift)], 1u);
  });
  __syncthreads();
  for (int i = threadIdx.x; i < HBINS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void collect_kernel(const unsigned long long* __restrict__ key, uint32_t m,
                               unsigned long long lo, unsigned long long hi,
                               unsigned long long* __restrict__ out, uint32_t* __restrict__ count) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const unsigned long long v = key[i];
    if (v >= lo && v <= hi) out[atomicAdd(count, 1u)] = v;
  }
}


// ------------------------------------------- device-side exact selection
// One shared level-1 histogram over [kmin, kmax] (read from device memory),
// bucket search for every target rank, one collect pass over the union of
// the target buckets, then a single block refines every target in shared
// memory -- no host round trip until the results are read back.
constexpr int kSelMax = 4;
struct SelState {
  unsigned long long rank[kSelMax];
  unsigned long long lo[kSelMax], hi[kSelMax];
  unsigned long long result[kSelMax];
  unsigned long long base, top;
  uint32_t shift, nt, need_collect, overflow, ncand;
  uint32_t bucket[kSelMax];
  // direct: the level-1 target buckets' keys fit the candidate buffer, so the
  // level-2 pass also lists them (ncand1 of them) and the collect pass reads
  // that list instead of every key
  uint32_t direct, ncand1;
};

// interpolated_quantile's ranks (binning.hpp:98-104) from the completed count
// (pos = q (n-1) rounded as on the host, no contraction), then the range
__global__ void sel_init_kernel(SelState* S, const unsigned long long* kminmax, const Info* I) {
  const unsigned long long nc = I->nc;
  uint32_t nt = 0;
  if (nc > 0) {
    const double qs[2] = {0.50, 0.99};
    for (int q = 0; q < 2; ++q) {
      const double pos = __dmul_rn(qs[q], (double)(nc - 1));
      const unsigned long long idx = (unsigned long long)pos;
      S->rank[nt++] = idx;
      if (idx + 1 < nc) S->rank[nt++] = idx + 1;
    }
  }
  S->nt = nt;
  const unsigned long long lo = kminmax[0], hi = kminmax[1];
  S->base = lo;
  S->top = hi;
  const unsigned long long span = hi - lo;
  const int bits = span ? 64 - __clzll(span) : 0;
  S->shift = bits > HBITS ? (uint32_t)(bits - HBITS) : 0u;
  S->ncand = 0;
  S->overflow = 0;
  S->direct = 0;
  S->ncand1 = 0;
}

__global__ void sel_hist_kernel(const unsigned long long* __restrict__ key, uint32_t m,
                                const SelState* S, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[HBINS];
  for (int i = threadIdx.x; i < HBINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned long long lo = S->base, hi = S->top;
  const uint32_t shift = S->shift;
  for_keys(key, m, [&](unsigned long long v) {
    if (v >= lo && v <= hi) atomicAdd(&h[(uint32_t)((v - lo) >> shift)], 1u);
  });
  __syncthreads();
  for (int i = threadIdx.x; i < HBINS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Block-wide bucket search (blockDim == 1024): the bucket b of h[0..nb) with
// prefix(b) <= r < prefix(b) + h[b]; writes *bucket and *before.
__device__ __forceinline__ void block_find(const uint32_t* h, int nb, unsigned long long r,
                                           uint32_t* bucket, unsigned long long* before) {
  __shared__ unsigned long long s_ws[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int per = nb / 1024;
  unsigned long long loc = 0;
  for (int i = 0; i < per; ++i) loc += h[t * per + i];
  unsigned long long x = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_ws[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long v = s_ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    s_ws[lane] = v;  // inclusive per warp
  }
  __syncthreads();
  const unsigned long long excl = x - loc + (w ? s_ws[w - 1] : 0ull);
  if (r >= excl && r < excl + loc) {
    unsigned long long acc = excl;
    for (int i = 0; i < per; ++i) {
      const uint32_t c = h[t * per + i];
      if (r < acc + c) {
        *bucket = (uint32_t)(t * per + i);
        *before = acc;
        break;
      }
      acc += c;
    }
  }
  __syncthreads();
}

// per target: bucket, residual rank, range (1024 threads; a block-wide
// search per target over the level-1 histogram)
__global__ void __launch_bounds__(1024) sel_find_kernel(SelState* S, const uint32_t* hist,
                                                        uint32_t cap) {
  __shared__ uint32_t h[HBINS];
  __shared__ uint32_t s_b;
  __shared__ unsigned long long s_before;
  const int t = threadIdx.x;
  for (int i = t; i < HBINS; i += blockDim.x) h[i] = hist[i];
  __syncthreads();
  unsigned long long need = 0;
  if (t == 0) S->need_collect = 0;
  const uint32_t nt = S->nt;
  for (uint32_t q = 0; q < nt; ++q) {
    block_find(h, HBINS, S->rank[q], &s_b, &s_before);
    if (t == 0) {
      const uint32_t b = s_b;
      S->rank[q] -= s_before;
      S->bucket[q] = b;
      const unsigned long long blo = S->base + ((unsigned long long)b << S->shift);
      unsigned long long bhi = blo + ((1ull << S->shift) - 1);
      if (bhi > S->top || bhi < blo) bhi = S->top;
      S->lo[q] = blo;
      S->hi[q] = bhi;
      if (blo == bhi) {
        S->result[q] = blo;
      } else {
        bool dup = false;
        for (uint32_t z = 0; z < q; ++z) dup |= S->lo[z] == blo && S->hi[z] != S->lo[z];
        if (!dup) need += h[b];
        S->need_collect = 1;
      }
    }
    __syncthreads();
  }
  if (t == 0) S->direct = need <= cap;
}

// level 2 over the full key array: every unresolved target's bucket split
// into 2048 sub-buckets at once (per-target shared histograms)
constexpr int kSub = 2048;
__global__ void sel_hist2_kernel(const unsigned long long* __restrict__ key, uint32_t m,
                                 SelState* S, uint32_t* __restrict__ hist2,
                                 unsigned long long* __restrict__ out, uint32_t cap) {
  __shared__ uint32_t h[kSelMax][kSub];
  __shared__ unsigned long long s_lo[kSelMax], s_hi[kSelMax];
  __shared__ uint32_t s_sh[kSelMax];
  for (int i = threadIdx.x; i < kSelMax * kSub; i += blockDim.x) (&h[0][0])[i] = 0;
  if (threadIdx.x < kSelMax) {
    const uint32_t q = threadIdx.x;
    const bool live = q < S->nt && S->lo[q] != S->hi[q];
    s_lo[q] = live ? S->lo[q] : 1;
    s_hi[q] = live ? S->hi[q] : 0;
    const unsigned long long span = live ? S->hi[q] - S->lo[q] : 0;
    const int bits = span ? 64 - __clzll(span) : 0;
    s_sh[q] = bits > 11 ? (uint32_t)(bits - 11) : 0u;
  }
  __syncthreads();
  if (!S->need_collect) return;
  const bool direct = S->direct != 0;
  for_keys(key, m, [&](unsigned long long v) {
    bool in = false;
#pragma unroll
    for (int q = 0; q < kSelMax; ++q)
      if (v >= s_lo[q] && v <= s_hi[q]) {
        atomicAdd(&h[q][(uint32_t)((v - s_lo[q]) >> s_sh[q])], 1u);
        in = true;
      }
    if (direct && in) {  // the level-1 candidates (the union of the target buckets)
      const uint32_t slot = atomicAdd(&S->ncand1, 1u);
      if (slot < cap) out[slot] = v;
    }
  });
  __syncthreads();
  for (int i = threadIdx.x; i < kSelMax * kSub; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(&hist2[i], (&h[0][0])[i]);
}

// narrow every unresolved target to its level-2 sub-bucket (1024 threads)
__global__ void __launch_bounds__(1024) sel_find2_kernel(SelState* S, const uint32_t* hist2,
                                                         uint32_t cap) {
  __shared__ uint32_t s_b;
  __shared__ unsigned long long s_before;
  if (!S->need_collect) return;
  for (uint32_t q = 0; q < S->nt; ++q) {
    if (S->lo[q] == S->hi[q]) continue;  // uniform across the block
    block_find(hist2 + q * kSub, kSub, S->rank[q], &s_b, &s_before);
    if (threadIdx.x == 0) {
      const unsigned long long span = S->hi[q] - S->lo[q];
      const int bits = 64 - __clzll(span);
      const uint32_t sh = bits > 11 ? (uint32_t)(bits - 11) : 0u;
      S->rank[q] -= s_before;
      const unsigned long long nlo = S->lo[q] + ((unsigned long long)s_b << sh);
      unsigned long long nhi = nlo + ((1ull << sh) - 1);
      if (nhi > S->hi[q] || nhi < nlo) nhi = S->hi[q];
      S->lo[q] = nlo;
      S->hi[q] = nhi;
      if (nlo == nhi) S->result[q] = nlo;
      S->bucket[q] = hist2[q * kSub + s_b];  // candidate count of the sub-bucket
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    unsigned long long need = 0;
    uint32_t live = 0;
    for (uint32_t q = 0; q < S->nt; ++q) {
      if (S->lo[q] == S->hi[q]) continue;
      bool dup = false;
      for (uint32_t z = 0; z < q; ++z) dup |= S->lo[z] == S->lo[q] && S->hi[z] == S->hi[q];
      if (!dup) need += S->bucket[q];
      ++live;
    }
    S->need_collect = live != 0;
    S->overflow = need > cap;
  }
}

__global__ void sel_collect_kernel(const unsigned long long* __restrict__ key, uint32_t m,
                                   const unsigned long long* __restrict__ l1, SelState* S,
                                   unsigned long long* __restrict__ out, uint32_t cap) {
  if (!S->need_collect || S->overflow) return;
  if (S->direct) {  // the level-1 candidates listed by the level-2 pass
    key = l1;
    m = S->ncand1;
  }
  unsigned long long lo[kSelMax], hi[kSelMax];
  const uint32_t nt = S->nt;
  for (uint32_t q = 0; q < kSelMax; ++q) {
    lo[q] = q < nt ? S->lo[q] : 1;
    hi[q] = q < nt && S->lo[q] != S->hi[q] ? S->hi[q] : 0;
  }
  for_keys(key, m, [&](unsigned long long v) {
    bool in = false;
#pragma unroll
    for (int q = 0; q < kSelMax; ++q) in |= v >= lo[q] && v <= hi[q];
    if (in) {
      const uint32_t slot = atomicAdd(&S->ncand, 1u);
      if (slot < cap) out[slot] = v;
    }
  });
}

// refine every unresolved target on the candidates, all levels in smem
constexpr uint32_t kRefineDirect = 512;
__global__ void __launch_bounds__(1024) sel_refine_kernel(SelState* S,
                                                          const unsigned long long* __restrict__ cand) {
  __shared__ uint32_t h[HBINS];
  __shared__ unsigned long long s_lo, s_hi, s_rank;
  __shared__ unsigned long long s_c[kRefineDirect];
  if (!S->need_collect || S->overflow) return;
  const uint32_t m = S->ncand;
  if (m <= kRefineDirect) {  // few candidates: rank each one directly (m^2 compares)
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) s_c[i] = cand[i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const unsigned long long v = s_c[i];
      for (uint32_t q = 0; q < S->nt; ++q) {
        const unsigned long long lo = S->lo[q], hi = S->hi[q];
        if (lo == hi || v < lo || v > hi) continue;
        uint32_t lt = 0, eq = 0;
        for (uint32_t j = 0; j < m; ++j) {
          const unsigned long long c = s_c[j];
          const bool in = c >= lo && c <= hi;
          lt += in && c < v;
          eq += c == v;
        }
        const unsigned long long r = S->rank[q];
        if (lt <= r && r < (unsigned long long)lt + eq) S->result[q] = v;  // (ties write the same value)
      }
    }
    return;
  }
  for (uint32_t q = 0; q < S->nt; ++q) {
    if (threadIdx.x == 0) {
      s_lo = S->lo[q];
      s_hi = S->hi[q];
      s_rank = S->rank[q];
    }
    __syncthreads();
    while (s_lo < s_hi) {
      const unsigned long long lo = s_lo, hi = s_hi;
      const unsigned long long span = hi - lo;
      const int bits = 64 - __clzll(span);
      const uint32_t shift = bits > HBITS ? (uint32_t)(bits - HBITS) : 0u;
      for (int i = threadIdx.x; i < HBINS; i += blockDim.x) h[i] = 0;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const unsigned long long v = cand[i];
        if (v >= lo && v <= hi) atomicAdd(&h[(uint32_t)((v - lo) >> shift)], 1u);
      }
      __syncthreads();
      __shared__ uint32_t s_b;
      __shared__ unsigned long long s_before;
      block_find(h, HBINS, s_rank, &s_b, &s_before);
      if (threadIdx.x == 0) {
        s_rank -= s_before;
        const unsigned long long nlo = lo + ((unsigned long long)s_b << shift);
        unsigned long long nhi = nlo + ((1ull << shift) - 1);
        if (nhi > hi || nhi < nlo) nhi = hi;
        s_lo = nlo;
        s_hi = nhi;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) S->result[q] = s_lo;
    __syncthreads();
  }
}

// -------------------------------------------------------- max_batch_wait
// Timers (simulator.hpp:200-201,223-235) with strictly increasing arrivals:
// a bin's batch starting at its front f closes at the B-th member's arrival
// if that comes no later than a_f + W (an arrival at exactly the due time is
// processed first: rank 1 < 2), otherwise at a_f + W with the members that
// arrived by then; the bin is then empty, so the next batch starts at the
// next arrival.  The segmentation depends only on the bin's own arrivals.
// The last open batch of a bin forms at its due time, or -- with flush, if
// the due time is after the last arrival -- at the last arrival (on_drain).
// Dispatch order = formation order; at equal times the reference's event
// sequence puts the timer (armed earlier) before a formation scheduled by an
// arrival, and both before the drains, which run in bin order.
enum : uint32_t { TM_TIMER = 0, TM_FULL = 1, TM_DRAIN = 2 };

__global__ void tie_kernel(const double* __restrict__ a, uint32_t n, uint32_t* flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (i < n && a[i] == a[i - 1]) *flag = 1;
}

// list[binoff[b] + rank[i]] = i: every bin's requests in arrival order
__global__ void bin_list_kernel(const uint8_t* __restrict__ pb8, const uint32_t* __restrict__ rank,
                                const uint32_t* __restrict__ binoff, uint32_t n, uint32_t* list) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) list[binoff[pb8[i] - 1] + rank[i]] = i;
}

// One warp per bin walks its list in 32-request chunks; records are written
// bin-major (slot binoff[b] + j for the bin's j-th batch), and segj maps each
// list position to j.
struct TmArgs {
  const double* a;
  const double* s;
  const uint32_t* list;
  const uint32_t* binoff;
  const uint32_t* bincnt;
  uint32_t B;
  double W, a_last;
  int32_t flush;
  double* recF;      // formation time
  double* recS;      // service = max member service
  uint32_t* recP;    // first list position (bin-relative)
  uint32_t* recN;    // members
  uint8_t* recB;     // bin (0-based)
  unsigned long long* key1;  // formation time bits (~0: unused slot)
  unsigned long long* key2;  // event class << 32 | (timer: its front's request index
                             //   = the arming order, the event seq; else the bin)
  uint32_t* segj;    // per list position
  uint32_t* nrec;    // per bin
};

__global__ void __launch_bounds__(32) tm_segment_kernel(TmArgs T) {
  const uint32_t b = blockIdx.x, lane = threadIdx.x;
  const uint32_t off = T.binoff[b], cnt = T.bincnt[b];
  uint32_t nseg = 0, f = 0;
  bool open = false;
  double due = 0.0, smax = 0.0;
  auto emit = [&](double formed, uint32_t cls, uint32_t size) {
    if (lane == 0) {
      const uint32_t q = off + nseg;
      T.recF[q] = formed;
      T.recS[q] = smax;
      T.recP[q] = f;
      T.recN[q] = size;
      T.recB[q] = (uint8_t)b;
      T.key1[q] = (unsigned long long)__double_as_longlong(formed);
      T.key2[q] = ((unsigned long long)cls << 32) | (cls == TM_TIMER ? T.list[off + f] : b);
    }
    ++nseg;
    open = false;
  };
  for (uint32_t base = 0; base < cnt; base += 32) {
    const uint32_t p = base + lane;
    const bool valid = p < cnt;
    const uint32_t idx = valid ? T.list[off + p] : 0;
    const double av = valid ? T.a[idx] : CUDART_INF;
    const double sv = valid ? T.s[idx] : 0.0;
    const uint32_t cend = min(base + 32, cnt);
    uint32_t q = base;  // next position to place (warp-uniform)
    while (q < cend) {
      if (!open) {
        f = q;
        due = __dadd_rn(__shfl_sync(0xffffffffu, av, q - base), T.W);  // armed at the front's arrival
        smax = 0.0;
        open = true;
      }
      const uint32_t over = __ballot_sync(0xffffffffu, valid && p >= q && av > due);
      uint32_t lim = min(cend, f + T.B);
      if (over) lim = min(lim, base + (uint32_t)(__ffs(over) - 1));
      // members [q, lim): segment id and the running service max
      double m = (p >= q && p < lim) ? sv : 0.0;
      if (p >= q && p < lim) T.segj[off + p] = nseg;
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      smax = fmax(smax, m);
      q = lim;
      if (q == f + T.B) {  // the B-th member arrived first: formation at its arrival
        emit(__shfl_sync(0xffffffffu, av, q - 1 - base), TM_FULL, T.B);
      } else if (over && q < cend) {  // the timer fired first
        emit(due, TM_TIMER, q - f);
      }
    }
  }
  if (open) {  // the bin's last batch: its timer, or the drain at the last arrival
    if (T.flush && due > T.a_last) emit(T.a_last, TM_DRAIN, cnt - f);
    else emit(due, TM_TIMER, cnt - f);
  }
  if (lane == 0) T.nrec[b] = nseg;
  for (uint32_t j = nseg + lane; j < cnt; j += 32) T.key1[off + j] = ~0ull;  // unused slots sort last
}

__global__ void tm_gather_keys(const unsigned long long* __restrict__ src, const uint32_t* __restrict__ idx,
                               uint32_t m, unsigned long long* dst) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m) dst[j] = src[idx[j]];
}

// dispatch-ordered records: (R, S, bin, size), map[record] = position
__global__ void tm_gather_kernel(const uint32_t* __restrict__ order, const uint8_t* __restrict__ recB,
                                 const double* __restrict__ recF, const double* __restrict__ recS,
                                 const uint32_t* __restrict__ recN, uint32_t nb, double* dR, double* dS,
                                 uint8_t* dBin, uint32_t* dSize, uint32_t* map) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nb) return;
  const uint32_t q = order[d];
  dR[d] = recF[q];
  dS[d] = recS[q];
  if (dBin) dBin[d] = (uint8_t)(recB[q] + 1);
  dSize[d] = recN[q];
  map[q] = d;
}

// per request: completion, batch, members, latency key (as request_kernel)
__global__ void __launch_bounds__(256) tm_request_kernel(
    const double* __restrict__ a, const uint8_t* __restrict__ pb8, const uint32_t* __restrict__ rank,
    const uint32_t* __restrict__ binoff, const uint32_t* __restrict__ segj,
    const uint32_t* __restrict__ recP, const uint32_t* __restrict__ map,
    const double* __restrict__ finish, const uint32_t* __restrict__ dfirst, uint32_t n,
    unsigned long long* key_out, double* lat_part, unsigned long long* kminmax, double* completion,
    uint32_t* batch, uint32_t* members) {
  __shared__ double s_sum[8];
  __shared__ unsigned long long s_min[8], s_max[8];
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double lat = 0.0;
  unsigned long long kmin = KEY_UNSERVED, kmax = 0;
  if (i < n) {
    const uint32_t off = binoff[pb8[i] - 1], r = rank[i];
    const uint32_t q = off + segj[off + r];
    const uint32_t d = map[q];
    const double comp = finish[d];
    lat = __dsub_rn(comp, a[i]);  // simulator.hpp:294
    const unsigned long long key = (unsigned long long)__double_as_longlong(lat);
    kmin = kmax = key;
    if (members) members[dfirst[d] + (r - recP[q])] = i;
    key_out[i] = key;
    if (completion) completion[i] = comp;
    if (batch) batch[i] = d;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    lat += __shfl_xor_sync(0xffffffffu, lat, o);
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, kmin, o);
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmin = x < kmin ? x : kmin;
    kmax = y > kmax ? y : kmax;
  }
  if (lane == 0) {
    s_sum[w] = lat;
    s_min[w] = kmin;
    s_max[w] = kmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sm = 0.0;
    for (int q = 0; q < 8; ++q) {
      sm += s_sum[q];
      kmin = s_min[q] < kmin ? s_min[q] : kmin;
      kmax = s_max[q] > kmax ? s_max[q] : kmax;
    }
    lat_part[blockIdx.x] = sm;
    if (kmin != KEY_UNSERVED) {
      atomicMin(&kminmax[0], kmin);
      atomicMax(&kminmax[1], kmax);
    }
  }
}

// ------------------------------------------------------------------ host
#define BB_CK(x)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      R->status = BB_ECUDA;                                                             \
      snprintf(R->message, sizeof R->message, "CUDA error %s at %s:%d",                 \
               cudaGetErrorString(e_), __FILE__, __LINE__);                             \
      goto cleanup;                                                                     \
    }                                                                                   \
  } while (0)

// Scratch of one trace run: a bump allocator over a per-device arena of
// cached chunks (no allocation API call per buffer; the pipeline asks for
// ~50 buffers).  Callers hold the device's mutex, so one run uses the arena
// at a time; a run's stream waits for the previous run's end event before
// reusing the memory (runs may come on different streams).
struct Arena {
  std::vector<std::pair<char*, size_t>> chunks;
  cudaEvent_t done = nullptr;
};
Arena g_arena[64];

struct Pool {
  cudaStream_t s = nullptr;
  Arena* ar = nullptr;
  size_t chunk = 0, off = 0;
  // first use in this run: the stream waits for the previous run's end
  cudaError_t attach() {
    if (ar) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    ar = &g_arena[dev & 63];
    return ar->done ? cudaStreamWaitEvent(s, ar->done, 0) : cudaSuccess;
  }
  cudaError_t alloc(void** p, size_t bytes) {
    if (!ar) {
      cudaError_t e = attach();
      if (e != cudaSuccess) return e;
    }
    bytes = ((bytes ? bytes : 8) + 255) & ~(size_t)255;
    while (chunk < ar->chunks.size() && off + bytes > ar->chunks[chunk].second) {
      ++chunk;
      off = 0;
    }
    if (chunk == ar->chunks.size()) {
      const size_t cb = bytes > ((size_t)256 << 20) ? bytes : ((size_t)256 << 20);
      char* c = nullptr;
      cudaError_t e = cudaMalloc(&c, cb);
      if (e != cudaSuccess) return e;
      ar->chunks.push_back({c, cb});
      off = 0;
    }
    *p = ar->chunks[chunk].first + off;
    off += bytes;
    return cudaSuccess;
  }
  ~Pool() {
    if (!ar) return;
    if (!ar->done) cudaEventCreateWithFlags(&ar->done, cudaEventDisableTiming);
    cudaEventRecord(ar->done, s);
  }
};

unsigned grid_for(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// Select the exact order statistics of `rank`s among keys (all keys of
// completed requests lie in [kmin, kmax]; unserved keys are above).
static cudaError_t select_ranks(const unsigned long long* keys, uint32_t n,
                                unsigned long long kmin, unsigned long long kmax,
                                const std::vector<unsigned long long>& ranks,
                                std::vector<unsigned long long>& vals, Pool& pool,
                                cudaStream_t s) {
  vals.assign(ranks.size(), kmin);
  if (kmin == kmax) return cudaSuccess;
  uint32_t* d_hist = nullptr;
  uint32_t* d_cnt = nullptr;
  unsigned long long *bufA = nullptr, *bufB = nullptr;
  cudaError_t e;
  if ((e = pool.alloc((void**)&d_hist, HBINS * sizeof(uint32_t)))) return e;
  if ((e = pool.alloc((void**)&d_cnt, sizeof(uint32_t)))) return e;
  std::vector<uint32_t> h(HBINS);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 4;
  for (size_t t = 0; t < ranks.size(); ++t) {
    unsigned long long lo = kmin, hi = kmax, rank = ranks[t];
    const unsigned long long* buf = keys;
    uint32_t m = n;
    while (lo < hi) {
      const unsigned long long span = hi - lo;
      const int bits = 64 - __builtin_clzll(span);
      const uint32_t shift = bits > HBITS ? (uint32_t)(bits - HBITS) : 0u;
      if ((e = cudaMemsetAsync(d_hist, 0, HBINS * sizeof(uint32_t), s))) return e;
      hist_kernel<<<grid, 256, 0, s>>>(buf, m, lo, hi, shift, d_hist);
      note_launch();
      if ((e = cudaMemcpyAsync(h.data(), d_hist, HBINS * sizeof(uint32_t), cudaMemcpyDeviceToHost, s))) return e;
      if ((e = cudaStreamSynchronize(s))) return e;
      unsigned long long acc = 0;
      uint32_t bk = 0;
      for (; bk < HBINS; ++bk) {
        if (acc + h[bk] > rank) break;
        acc += h[bk];
      }
      if (bk == HBINS) return cudaErrorUnknown;  // rank beyond the population
      rank -= acc;
      const unsigned long long nlo = lo + ((unsigned long long)bk << shift);
      unsigned long long nhi = nlo + ((1ull << shift) - 1);
      if (nhi > hi || nhi < nlo) nhi = hi;
      lo = nlo;
      hi = nhi;
      if (lo == hi) break;
      // compact the bucket's members for the next level (sizes only shrink)
      unsigned long long* dst;
      if (buf == keys) {
        if ((e = pool.alloc((void**)&bufA, (size_t)h[bk] * 8))) return e;
        if ((e = pool.alloc((void**)&bufB, (size_t)h[bk] * 8))) return e;
        dst = bufA;
      } else {
        dst = buf == bufA ? bufB : bufA;
      }
      if ((e = cudaMemsetAsync(d_cnt, 0, sizeof(uint32_t), s))) return e;
      collect_kernel<<<grid, 256, 0, s>>>(buf, m, lo, hi, dst, d_cnt);
      note_launch();
      buf = dst;
      m = h[bk];
    }
    vals[t] = lo;
  }
  return cudaSuccess;
}

// Everything the host reads back at the end of a run (one round trip).
struct Readback {
  Info info;
  DevError herr;
  double sc[2];  // last completion, first arrival
  double busy, lsum;
  unsigned long long mm[2];  // completed keys' min / max
  SelState hs;
};

// Everything the host reads back, gathered on the device by one small
// kernel: one copy (or, into the graph's pinned struct, none) instead of
// seven.
struct ReadbackSrc {
  const Info* info;
  const DevError* err;
  const double *scal, *busy, *lsum;
  const unsigned long long* mm;
  const SelState* hs;
};
__global__ void readback_kernel(ReadbackSrc S, Readback* out) {
  auto cp = [](void* d, const void* s, size_t bytes) {
    for (size_t i = threadIdx.x; i < bytes / 4; i += blockDim.x)
      static_cast<uint32_t*>(d)[i] = static_cast<const uint32_t*>(s)[i];
  };
  static_assert(sizeof(Info) % 4 == 0 && sizeof(DevError) % 4 == 0 && sizeof(SelState) % 4 == 0, "word copies");
  cp(&out->info, S.info, sizeof(Info));
  cp(&out->herr, S.err, sizeof(DevError));
  cp(&out->hs, S.hs, sizeof(SelState));
  if (threadIdx.x == 0) {
    out->sc[0] = S.scal[0];
    out->sc[1] = S.scal[1];
    out->busy = *S.busy;
    out->lsum = *S.lsum;
    out->mm[0] = S.mm[0];
    out->mm[1] = S.mm[1];
  }
}

// the partition's verdict: a request error, or non-monotone arrivals
static bool trace_input_error(const DevError& herr, const Info& info, TraceResult* R) {
  if (herr.packed != ~0ull) {
    const unsigned long long idx = herr.packed >> 8;
    const int code = (int)(herr.packed & 0xFF);
    R->status = code;
    if (code == BB_EDOMAIN && herr.aux == 1)
      snprintf(R->message, sizeof R->message, "simulation: drew a non-positive service time");
    else if (code == BB_EDOMAIN)
      snprintf(R->message, sizeof R->message, "assign_bin: length %.17g outside bin support", herr.value);
    else
      snprintf(R->message, sizeof R->message, "request %llu: predicted bin %g out of range", idx, herr.value);
    return true;
  }
  if (info.path == 3) {
    R->status = BB_EINVAL;
    snprintf(R->message, sizeof R->message, "trace arrays: arrivals must be non-decreasing");
    return true;
  }
  return false;
}

// finish(), simulator.hpp:283-301, from the read-back scalars.  p50/p99 are
// interpolated_quantile (binning.hpp:98-104) over the ranks sel_init
// selected.  Returns false when the one-launch selection overflowed and no
// key array is at hand (a graph replay): the caller reruns the direct path.
static bool trace_report(const TraceArgs& A, TraceResult* R, const Readback& rb, unsigned long long nc,
                         const unsigned long long* keys, Pool* pool, cudaStream_t s) {
  if (nc == 0) return true;
  const SelState& hs = rb.hs;
  if (hs.overflow && !keys) return false;
  const double last = rb.sc[0], a0 = rb.sc[1];
  R->makespan = last - a0;
  R->throughput = (double)nc / R->makespan;
  R->busy = rb.busy;
  R->busy_fraction = rb.busy / ((double)(A.n_servers > 1 ? A.n_servers : 1) * R->makespan);
  R->latency_sum = rb.lsum;
  R->latency_mean = rb.lsum / (double)nc;
  const double qs[2] = {0.50, 0.99};
  std::vector<unsigned long long> ranks(hs.rank, hs.rank + hs.nt);
  unsigned long long idxs[2];
  double fracs[2];
  for (int q = 0; q < 2; ++q) {
    const volatile double pos = qs[q] * (double)(nc - 1);
    idxs[q] = (unsigned long long)pos;
    fracs[q] = pos - (double)idxs[q];
  }
  std::vector<unsigned long long> vals;
  if (hs.overflow) {  // multi-launch refine as the fallback
    const cudaError_t e = select_ranks(keys, A.n, rb.mm[0], rb.mm[1], ranks, vals, *pool, s);
    if (e != cudaSuccess) {
      R->status = BB_ECUDA;
      snprintf(R->message, sizeof R->message, "CUDA error %s (quantile selection)", cudaGetErrorString(e));
      return true;
    }
  } else {
    for (size_t q = 0; q < ranks.size(); ++q) vals.push_back(hs.result[q]);
  }
  size_t vi = 0;
  double outq[2];
  for (int q = 0; q < 2; ++q) {
    double lo, hi;
    std::memcpy(&lo, &vals[vi++], 8);
    if (idxs[q] + 1 >= nc) {
      outq[q] = lo;
      continue;
    }
    std::memcpy(&hi, &vals[vi++], 8);
    const volatile double diff = hi - lo;
    const volatile double prod = fracs[q] * diff;
    outq[q] = lo + prod;
  }
  R->p50 = outq[0];
  R->p99 = outq[1];
  return true;
}

// A captured run of the sync-free pipeline (no max_batch_wait, no detail
// batch copies), replayed when the same arguments come again: one graph
// launch instead of ~30 kernel and memset launches.  The arena chunks it
// points into are never freed; the bin edges and confusion rows are copied
// into graph-owned buffers before each launch, so callers that re-upload
// them per call still hit.  Callers hold the device's mutex.
struct TraceGraph {
  bool have = false, pend = false;
  TraceArgs key{}, pend_key{};
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev[3] = {};
  Readback* rb = nullptr;  // pinned
  double *edges = nullptr, *conf = nullptr;
  unsigned long long launches = 0;
};
TraceGraph g_tgraph[64];
std::atomic<unsigned long long> g_tg_captures{0}, g_tg_replays{0};

static_assert(sizeof(TraceArgs) == 184, "TraceArgs has padding: the graph key compares it bytewise");

static TraceArgs graph_key(const TraceArgs& A) {
  TraceArgs k = A;
  k.edges = nullptr;
  k.conf = A.conf ? reinterpret_cast<const double*>(1) : nullptr;
  return k;
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("BB_TRACE_GRAPH");
    return !(e && e[0] == '0');
  }();
  return on;
}

static void trace_run_impl(const TraceArgs& A, TraceResult* R, cudaStream_t s, TraceGraph* cap) {

  std::memset(R, 0, sizeof *R);
  R->status = BB_OK;
  R->k = A.k;
  Pool pool;
  pool.s = s;
  const uint32_t n = A.n, k = A.k, B = A.B;
  const uint32_t ntiles = (n + PTILE - 1) / PTILE;
  const uint64_t rec_cap = (uint64_t)n / B + k + 1;
  WS ws{};
  Info info{};
  DevError herr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  double *dR = nullptr, *dS = nullptr, *start = nullptr, *finish = nullptr;
  uint32_t *map = nullptr, *order = nullptr, *dfirst = nullptr, *dsize = nullptr;
  uint8_t *dbin = nullptr, *split = nullptr;
  bool tm = false;   // max_batch_wait timer path
  bool tmo = false;  // overload without flush, with timers: partials at W
  unsigned long long nc_run = 0, tm_nc = 0;
  uint32_t tm_counts[1] = {0};
  bool capturing = false;
  unsigned long long launches0 = 0;
  // timing events: recorded as graph nodes under capture
  auto record = [&](cudaEvent_t e) {
    return cap ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s);
  };
  auto input_error = [&]() -> bool { return trace_input_error(herr, info, R); };
  // Without max_batch_wait the pipeline runs to the end with no host round
  // trip: buffers are sized for the batch-count bound n/B + k + 1 and the
  // kernels read the batch count, path and completed count from the device.
  // Timers order their batches on the host (below): one sync here.
  const bool host_sync = A.max_batch_wait > 0;

  uint32_t *tm_list = nullptr, *tm_off = nullptr, *tm_segj = nullptr, *tm_recP = nullptr;
  if (cap) {
    ev0 = cap->ev[0];
    ev1 = cap->ev[1];
    ev2 = cap->ev[2];
  } else {
    BB_CK(cudaEventCreate(&ev0));
    BB_CK(cudaEventCreate(&ev1));
    BB_CK(cudaEventCreate(&ev2));
  }
  if (cap) {  // capture from here to the read-back (the arena wait stays outside)
    BB_CK(pool.attach());
    BB_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    capturing = true;
    launches0 = launches_noted_here();
  }
  BB_CK(pool.alloc((void**)&ws.counters, 16));
  BB_CK(pool.alloc((void**)&ws.tcount, (size_t)ntiles * k * 4));
  BB_CK(pool.alloc((void**)&ws.smax, (rec_cap + 32) * 8));
  if (A.pred) ws.pb8 = const_cast<uint8_t*>(A.pred);  // given predictions are read in place
  else BB_CK(pool.alloc((void**)&ws.pb8, n));
  BB_CK(pool.alloc((void**)&ws.rank, (size_t)n * 4));
  BB_CK(pool.alloc((void**)&ws.recR, rec_cap * 8));
  BB_CK(pool.alloc((void**)&ws.recBin, rec_cap));
  BB_CK(pool.alloc((void**)&ws.recJ, rec_cap * 4));
  BB_CK(pool.alloc((void**)&ws.recC, rec_cap * 4));
  BB_CK(pool.alloc((void**)&ws.fin_cnt, 32 * 8));
  BB_CK(pool.alloc((void**)&ws.flags, 4));
  BB_CK(pool.alloc((void**)&ws.err, sizeof(DevError)));
  BB_CK(pool.alloc((void**)&ws.info, sizeof(Info)));
  BB_CK(cudaMemsetAsync(ws.counters, 0, 16, s));
  BB_CK(cudaMemsetAsync(ws.fin_cnt, 0, 32 * 8, s));
  BB_CK(cudaMemsetAsync(ws.smax, 0, (rec_cap + 32) * 8, s));
  BB_CK(cudaMemsetAsync(ws.flags, 0, 4, s));
  BB_CK(cudaMemsetAsync(ws.err, 0xFF, 8, s));
  BB_CK(record(ev0));
  {
    PartArgs P{};
    P.a = A.a;
    P.s = A.s;
    P.u_err = A.u_err;
    P.pred = A.pred;
    P.edges = A.edges;
    P.conf = A.conf;
    P.tb_out = A.req_true_bin;
    P.n = n;
    P.B = B;
    P.k = k;
    P.ntiles = ntiles;
    P.err_kind = A.err_kind;
    P.p = A.p_error;
    P.one_minus_p = 1.0 - A.p_error;
    P.divB = FastDiv(B);
    P.ws = ws;
    {
      auto al = [](const void* q, uintptr_t m) { return ((uintptr_t)q & (m - 1)) == 0; };
      P.vec_ok = al(A.a, 16) && al(A.s, 16) && (!A.u_err || al(A.u_err, 16)) && (!A.pred || al(A.pred, 16)) &&
                 al(ws.pb8, 16) && (!A.req_true_bin || al(A.req_true_bin, 16));
    }
    {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const uint32_t cg = std::min<uint32_t>(ntiles, (uint32_t)sms * 8);
      if (k <= 8) count_kernel<1><<<cg, PT, 0, s>>>(P);
      else if (k <= 16) count_kernel<2><<<cg, PT, 0, s>>>(P);
      else count_kernel<4><<<cg, PT, 0, s>>>(P);
    }
    tscan_kernel<<<k, TS_T, 0, s>>>(ws, ntiles, k, B);
    if (P.pred && P.tb_out) place_kernel<true><<<ntiles, PT, 0, s>>>(P);
    else place_kernel<false><<<ntiles, PT, 0, s>>>(P);
    note_launch(3);
    BB_CK(cudaGetLastError());
  }
  BB_CK(record(ev1));
  if (A.req_pred_bin && A.req_pred_bin != ws.pb8)
    BB_CK(cudaMemcpyAsync(A.req_pred_bin, ws.pb8, n, cudaMemcpyDeviceToDevice, s));
  finalize_kernel<<<1, 32, 0, s>>>(ws, A.a, n, k, B, A.flush, A.max_batch_wait);
  note_launch();
  BB_CK(cudaGetLastError());
  if (host_sync) {
    BB_CK(cudaMemcpyAsync(&info, ws.info, sizeof(Info), cudaMemcpyDeviceToHost, s));
    BB_CK(cudaMemcpyAsync(&herr, ws.err, sizeof(DevError), cudaMemcpyDeviceToHost, s));
    BB_CK(cudaStreamSynchronize(s));
    if (input_error()) goto cleanup;
    R->path = (int32_t)info.path;
  }
  // max_batch_wait: overload with flush drains every bin at t = 0, so the
  // timers go stale and the plain pipeline applies; otherwise the timer path
  tm = A.max_batch_wait > 0 && info.path != 1;
  tmo = A.max_batch_wait > 0 && info.path == 1 && !A.flush;
  if (tmo) {
    // fire order at W: timers armed at the bins' first arrivals (bins that
    // never filled a batch), then those re-armed by each bin's last
    // round-robin formation (its position among the t = 0 batches)
    uint32_t* dfa;
    std::vector<uint32_t> fa(k, 0);
    BB_CK(pool.alloc((void**)&dfa, (size_t)k * 4));
    BB_CK(cudaMemsetAsync(dfa, 0, (size_t)k * 4, s));
    if (info.nclose) ovl_first_kernel<<<grid_for(info.nclose, 256), 256, 0, s>>>(ws);
    first_arrival_kernel<<<grid_for(n, 256), 256, 0, s>>>(ws.pb8, ws.rank, n, dfa);
    note_launch(2);
    BB_CK(cudaGetLastError());
    BB_CK(cudaMemcpyAsync(fa.data(), dfa, (size_t)k * 4, cudaMemcpyDeviceToHost, s));
    BB_CK(cudaMemcpyAsync(info.cfirst, ws.info->cfirst, sizeof info.cfirst, cudaMemcpyDeviceToHost, s));
    BB_CK(cudaStreamSynchronize(s));
    std::vector<std::pair<unsigned long long, uint32_t>> keyb;
    for (uint32_t b = 0; b < k; ++b) {
      if (!info.rem[b]) continue;
      const uint32_t Fb = info.F[b];
      unsigned long long key = fa[b];
      if (Fb) {  // position of batch (b, Fb-1) in the round-robin order (order_kernel, no flush)
        const uint32_t j = Fb - 1;
        unsigned long long p = 0;
        for (uint32_t q = 0; q < k; ++q) {
          p += info.F[q] < j ? info.F[q] : j;
          p += (info.cfirst[q] < info.cfirst[b]) && (info.F[q] > j);
        }
        key = (unsigned long long)n + p;
      }
      keyb.push_back({key, b});
    }
    std::sort(keyb.begin(), keyb.end());
    uint32_t req = 0;
    for (uint32_t x = 0; x < keyb.size(); ++x) {
      info.tpos[keyb[x].second] = x;
      info.treq[keyb[x].second] = req;
      req += info.rem[keyb[x].second];
    }
    BB_CK(cudaMemcpyAsync(ws.info->tpos, info.tpos, sizeof info.tpos, cudaMemcpyHostToDevice, s));
    BB_CK(cudaMemcpyAsync(ws.info->treq, info.treq, sizeof info.treq, cudaMemcpyHostToDevice, s));
  }
  if (tm) {
    uint32_t* tflag;
    uint32_t htie = 0;
    BB_CK(pool.alloc((void**)&tflag, 4));
    BB_CK(cudaMemsetAsync(tflag, 0, 4, s));
    if (n > 1) tie_kernel<<<grid_for(n - 1, 256), 256, 0, s>>>(A.a, n, tflag);
    note_launch();
    BB_CK(cudaGetLastError());
    BB_CK(cudaMemcpyAsync(&htie, tflag, 4, cudaMemcpyDeviceToHost, s));
    BB_CK(cudaStreamSynchronize(s));
    if (htie) {
      R->status = BB_EUNSUPPORTED;
      snprintf(R->message, sizeof R->message,
               "max_batch_wait with equal arrival times is not supported yet");
      goto cleanup;
    }
  }
  {
    uint32_t nb = host_sync ? info.nb : (uint32_t)rec_cap;  // (without sync: the bound; grids and buffers)
    if (tm) {  // ---- timer path: per-bin segmentation, sort by formation
      std::vector<uint32_t> hoff(k), hcnt(k), hn(k);
      uint32_t acc = 0;
      for (uint32_t b = 0; b < k; ++b) {
        hcnt[b] = info.F[b] * B + info.rem[b];
        hoff[b] = acc;
        acc += hcnt[b];
      }
      uint32_t *d_off, *d_cnt, *list, *segj, *nrec, *recP, *recN, *val, *valb;
      unsigned long long *key2, *key2b;
      uint8_t* recB;
      unsigned long long *key1, *key1b;
      double *recF, *recS, a_last = 0;
      BB_CK(pool.alloc((void**)&d_off, (size_t)k * 4));
      BB_CK(pool.alloc((void**)&d_cnt, (size_t)k * 4));
      BB_CK(pool.alloc((void**)&nrec, (size_t)k * 4));
      BB_CK(pool.alloc((void**)&list, (size_t)n * 4));
      BB_CK(pool.alloc((void**)&segj, (size_t)n * 4));
      BB_CK(pool.alloc((void**)&recP, (size_t)n * 4));
      BB_CK(pool.alloc((void**)&recN, (size_t)n * 4));
      BB_CK(pool.alloc((void**)&recB, (size_t)n));
      BB_CK(pool.alloc((void**)&recF, (size_t)n * 8));
      BB_CK(pool.alloc((void**)&recS, (size_t)n * 8));
      BB_CK(pool.alloc((void**)&key1, (size_t)n * 8));
      BB_CK(pool.alloc((void**)&key1b, (size_t)n * 8));
      BB_CK(pool.alloc((void**)&key2, (size_t)n * 8));
      BB_CK(pool.alloc((void**)&key2b, (size_t)n * 8));
      BB_CK(pool.alloc((void**)&val, (size_t)n * 4));
      BB_CK(pool.alloc((void**)&valb, (size_t)n * 4));
      BB_CK(cudaMemcpyAsync(d_off, hoff.data(), (size_t)k * 4, cudaMemcpyHostToDevice, s));
      BB_CK(cudaMemcpyAsync(d_cnt, hcnt.data(), (size_t)k * 4, cudaMemcpyHostToDevice, s));
      BB_CK(cudaMemcpyAsync(&a_last, A.a + n - 1, 8, cudaMemcpyDeviceToHost, s));
      BB_CK(cudaStreamSynchronize(s));
      bin_list_kernel<<<grid_for(n, 256), 256, 0, s>>>(ws.pb8, ws.rank, d_off, n, list);
      note_launch();
      BB_CK(cudaGetLastError());
      {
        TmArgs T{A.a, A.s, list, d_off, d_cnt, B, A.max_batch_wait, a_last, A.flush,
                 recF, recS, recP, recN, recB, key1, key2, segj, nrec};
        tm_segment_kernel<<<k, 32, 0, s>>>(T);
        note_launch();
        BB_CK(cudaGetLastError());
      }
      BB_CK(cudaMemcpyAsync(hn.data(), nrec, (size_t)k * 4, cudaMemcpyDeviceToHost, s));
      BB_CK(cudaStreamSynchronize(s));
      nb = 0;
      for (uint32_t b = 0; b < k; ++b) {
        nb += hn[b];
        R->per_bin[b] = hn[b];
      }
      // dispatch order: stable radix sorts, (event class, arming order | bin) first, then time
      {
        std::vector<uint32_t> iota(n);
        for (uint32_t i = 0; i < n; ++i) iota[i] = i;
        BB_CK(cudaMemcpyAsync(val, iota.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
        cub::DoubleBuffer<unsigned long long> k2(key2, key2b);
        cub::DoubleBuffer<uint32_t> v2(val, valb);
        size_t tb1 = 0, tb2 = 0;
        void* tmp = nullptr;
        BB_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb1, k2, v2, (int)n, 0, 34, s));
        cub::DoubleBuffer<unsigned long long> k1(key1, key1b);
        BB_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, k1, v2, (int)n, 0, 64, s));
        BB_CK(pool.alloc(&tmp, std::max(tb1, tb2)));
        // the time keys must follow the first sort's permutation: sort
        // (class|bin, (time, index)) then (time, index) -- gather time by index
        BB_CK(cub::DeviceRadixSort::SortPairs(tmp, tb1, k2, v2, (int)n, 0, 34, s));
        note_launch();
        uint32_t* perm = v2.Current();
        // key1 in the class|bin order
        unsigned long long* k1p = k1.Alternate();
        tm_gather_keys<<<grid_for(n, 256), 256, 0, s>>>(key1, perm, n, k1p);
        note_launch();
        BB_CK(cudaGetLastError());
        k1.selector ^= 1;
        BB_CK(cub::DeviceRadixSort::SortPairs(tmp, tb2, k1, v2, (int)n, 0, 64, s));
        note_launch();
        order = v2.Current();
      }
      BB_CK(pool.alloc((void**)&map, (size_t)n * 4 + 4));
      BB_CK(pool.alloc((void**)&dfirst, (size_t)nb * 4 + 4));
      BB_CK(pool.alloc((void**)&dR, (size_t)nb * 8 + 8));
      BB_CK(pool.alloc((void**)&dS, (size_t)nb * 8 + 8));
      BB_CK(pool.alloc((void**)&dsize, (size_t)nb * 4 + 4));
      BB_CK(pool.alloc((void**)&split, nb + 1));
      if (nb) tm_gather_kernel<<<grid_for(nb, 256), 256, 0, s>>>(order, recB, recF, recS, recN, nb, dR, dS,
                                                                 A.bat_bin, dsize, map);
      note_launch();
      BB_CK(cudaGetLastError());
      if (A.bat_size && nb)
        BB_CK(cudaMemcpyAsync(A.bat_size, dsize, (size_t)nb * 4, cudaMemcpyDeviceToDevice, s));
      {
        size_t tb = 0;
        void* tmp = nullptr;
        BB_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, dsize, dfirst, (int)nb, s));
        BB_CK(pool.alloc(&tmp, tb));
        if (nb) BB_CK(cub::DeviceScan::ExclusiveSum(tmp, tb, dsize, dfirst, (int)nb, s));
        note_launch();
      }
      tm_list = list;
      tm_off = d_off;
      tm_segj = segj;
      tm_recP = recP;
      nc_run = n;  // every request completes: drained, or formed by its timer
      // the kernels below read the batch and completed counts on the device
      tm_counts[0] = nb;
      tm_nc = nc_run;
      BB_CK(cudaMemcpyAsync(&ws.info->nb, &tm_counts[0], 4, cudaMemcpyHostToDevice, s));
      BB_CK(cudaMemcpyAsync(&ws.info->nc, &tm_nc, 8, cudaMemcpyHostToDevice, s));
    } else {
      BB_CK(pool.alloc((void**)&map, (size_t)nb * 4 + 4));
      BB_CK(pool.alloc((void**)&order, (size_t)nb * 4 + 4));
      BB_CK(pool.alloc((void**)&dfirst, (size_t)nb * 4 + 4));
      BB_CK(pool.alloc((void**)&dR, (size_t)nb * 8 + 8));
      BB_CK(pool.alloc((void**)&dS, (size_t)nb * 8 + 8));
      BB_CK(pool.alloc((void**)&split, nb + 1));
    }
    const uint32_t* nbp = &ws.info->nb;
    // nb == 0 (nothing served, finish() :283) still runs the request pass so
    // every request reports kNoBatch / NaN completion
    start = A.bat_start;
    finish = A.bat_finish;
    if (!start) BB_CK(pool.alloc((void**)&start, (size_t)nb * 8 + 8));
    if (!finish) BB_CK(pool.alloc((void**)&finish, (size_t)nb * 8 + 8));
    if (!tm && !tmo && nb) {  // overload: first closings (a no-op on the other paths)
      ovl_first_kernel<<<grid_for(nb, 256), 256, 0, s>>>(ws);
      note_launch();
      BB_CK(cudaGetLastError());
    }
    if (!tm) {
      // path 2 (tie groups of more than B at finite times): closing order
      // first, then each such group re-orders its own range of records
      // (the device's path unless the host synchronised)
      const int32_t opath = !host_sync ? -1 : info.path == 2 ? 0 : (int32_t)info.path;
      if (nb) order_kernel<<<grid_for(nb, 256), 256, 0, s>>>(ws, map, order, dfirst, k, B, A.flush,
                                                     opath, (int32_t)tmo);
      note_launch();
      BB_CK(cudaGetLastError());
      if ((!host_sync || info.path == 2) && nb) {
        const uint32_t gcap = n / (B + 1) + 1;
        uint2* groups;
        uint32_t* ngroups;
        BB_CK(pool.alloc((void**)&groups, (size_t)gcap * 8));
        BB_CK(pool.alloc((void**)&ngroups, 4));
        BB_CK(cudaMemsetAsync(ngroups, 0, 4, s));
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        tie_groups_kernel<<<std::min<uint32_t>(grid_for(n, 256), sms * 8), 256, 0, s>>>(A.a, n, B, groups,
                                                                                      ngroups, ws.info);
        TieArgs T{groups, ngroups, ntiles, ws, map, order, dfirst, n, k, B, A.flush};
        tie_order_kernel<<<std::min<uint32_t>(gcap, sms * 4), 256, 0, s>>>(T);
        note_launch(2);
        BB_CK(cudaGetLastError());
      }
      if (nb) gather_kernel<<<grid_for(nb, 256), 256, 0, s>>>(ws, order, host_sync ? (int32_t)info.path : -1,
                                                      B, dR, dS, A.bat_bin, A.bat_size);
      note_launch();
      BB_CK(cudaGetLastError());
    }
    double *busy_sum, *last_dev;
    BB_CK(pool.alloc((void**)&busy_sum, 8));
    BB_CK(pool.alloc((void**)&last_dev, 8));
    BB_CK(cudaMemsetAsync(last_dev, 0, 8, s));
    // the exact Lindley recursion D = fl(max(D, R) + S) over (R, S) in
    // dispatch order into (st, fn): max-plus scan, certified busy-period
    // splits, binade parity scan, serial segments only as a fallback
    auto exact_lindley = [&](const double* dRl, const double* dSl, double* st, double* fn,
                             double** busy_part_out) -> cudaError_t {
      const double* dR = dRl;
      const double* dS = dSl;
      double* start = st;
      double* finish = fn;
      cudaError_t e_ = cudaSuccess;
#define BB_LCK(x)                             \
  do {                                        \
    if ((e_ = (x)) != cudaSuccess) return e_; \
  } while (0)
      BB_LCK(cudaMemsetAsync(ws.counters + 1, 0, 8, s));  // the scans' tile tickets
      // Lindley: certified busy-period splits, then exact serial segments
      const uint32_t lt = nb ? (nb + LTILE - 1) / LTILE : 1;
      double *aggA, *aggC, *incA, *incC, *busy_part;
      (void)dR;
      uint32_t* lflag;
      BB_LCK(pool.alloc((void**)&aggA, (size_t)lt * 8));
      BB_LCK(pool.alloc((void**)&aggC, (size_t)lt * 8));
      BB_LCK(pool.alloc((void**)&incA, (size_t)lt * 8));
      BB_LCK(pool.alloc((void**)&incC, (size_t)lt * 8));
      BB_LCK(pool.alloc((void**)&busy_part, (size_t)lt * 8));
      BB_LCK(pool.alloc((void**)&lflag, (size_t)lt * 4));
      BB_LCK(cudaMemsetAsync(lflag, 0, (size_t)lt * 4, s));
      const double tol_rel = (double)(nb + 4096) * 0x1.0p-50;
      double* Dt;
      BB_LCK(pool.alloc((void**)&Dt, (size_t)nb * 8 + 8));
      {
        LArgs L{dR, dS, nbp, split, Dt, busy_part, aggA, aggC, incA, incC, lflag, ws.counters + 1,
                tol_rel};
        if (nb) lindley_scan_kernel<<<lt, LB, 0, s>>>(L);
        note_launch();
        BB_LCK(cudaGetLastError());
      }
      // exact values: binade parity scan (parallel), serial segments only as a fallback
      int* bad;
      BB_LCK(pool.alloc((void**)&bad, 4));
      BB_LCK(cudaMemsetAsync(bad, 0, 4, s));
      if (nb) {
        BArgs Bq{};
        Bq.R = dR;
        Bq.S = dS;
        Bq.Dt = Dt;
        Bq.code = split;
        Bq.nbp = nbp;
        Bq.tol_rel = tol_rel;
        BB_LCK(pool.alloc((void**)&Bq.p0, (size_t)nb * 8));
        BB_LCK(pool.alloc((void**)&Bq.p1, (size_t)nb * 8));
        BB_LCK(pool.alloc((void**)&Bq.head_of, (size_t)nb * 4));
        BB_LCK(pool.alloc((void**)&Bq.run_last, (size_t)nb * 4));
        BB_LCK(pool.alloc((void**)&Bq.run_info, (size_t)nb * sizeof(RunInfo)));
        BB_LCK(pool.alloc((void**)&Bq.ag0, (size_t)lt * 8));
        BB_LCK(pool.alloc((void**)&Bq.ag1, (size_t)lt * 8));
        BB_LCK(pool.alloc((void**)&Bq.in0, (size_t)lt * 8));
        BB_LCK(pool.alloc((void**)&Bq.in1, (size_t)lt * 8));
        BB_LCK(pool.alloc((void**)&Bq.agh, (size_t)lt * 4));
        BB_LCK(pool.alloc((void**)&Bq.inh, (size_t)lt * 4));
        BB_LCK(pool.alloc((void**)&Bq.agf, (size_t)lt * 4));
        BB_LCK(pool.alloc((void**)&Bq.inf, (size_t)lt * 4));
        BB_LCK(pool.alloc((void**)&Bq.flag, (size_t)lt * 4));
        BB_LCK(cudaMemsetAsync(Bq.flag, 0, (size_t)lt * 4, s));
        Bq.counter = ws.counters + 2;
        binade_scan_kernel<<<lt, LB, 0, s>>>(Bq);
        note_launch();
        BB_LCK(cudaGetLastError());
        binade_chain_kernel<<<grid_for(nb, 128), 128, 0, s>>>(dR, dS, Dt, split, Bq.p0, Bq.p1,
                                                              Bq.run_info, nbp, start, finish, bad);
        note_launch();
        BB_LCK(cudaGetLastError());
        binade_fill_kernel<<<grid_for(nb, 256), 256, 0, s>>>(dS, Dt, split, Bq.p0, Bq.p1, Bq.head_of,
                                                             nbp, tol_rel, start, finish, bad);
        note_launch();
        BB_LCK(cudaGetLastError());
        lindley_segments_kernel<<<grid_for(nb, 128), 128, 0, s>>>(dR, dS, split, nbp, start, finish, bad);
        note_launch();
        BB_LCK(cudaGetLastError());
      }
      *busy_part_out = busy_part;
#undef BB_LCK
      return cudaSuccess;
    };
    if (A.n_servers > 1) {  // S servers: Kiefer-Wolfowitz in dispatch order, chunk-parallel
      const uint32_t G = nb / KWP_CH + 1;
      double *heaps, *chunk_last, *zeros, *bst, *bfn;
      uint32_t* refixed;
      BB_CK(pool.alloc((void**)&heaps, (size_t)G * A.n_servers * 8));
      BB_CK(pool.alloc((void**)&chunk_last, (size_t)G * 8));
      BB_CK(pool.alloc((void**)&refixed, 4));
      kw_spec_kernel<<<grid_for(G, 128), 128, 0, s>>>(dR, dS, nbp, A.n_servers, heaps, start, finish,
                                                      chunk_last);
      kw_fix_kernel<<<1, 256, 0, s>>>(dR, dS, nbp, A.n_servers, heaps, start, finish, chunk_last, last_dev,
                                      refixed);
      note_launch(2);
      BB_CK(cudaGetLastError());
      // busy time: the sequential sum of the services in dispatch order, exactly
      BB_CK(pool.alloc((void**)&zeros, (size_t)nb * 8 + 8));
      BB_CK(pool.alloc((void**)&bst, (size_t)nb * 8 + 8));
      BB_CK(pool.alloc((void**)&bfn, (size_t)nb * 8 + 8));
      BB_CK(cudaMemsetAsync(zeros, 0, (size_t)nb * 8 + 8, s));
      double* bp = nullptr;
      if (nb) {
        cudaError_t el = exact_lindley(zeros, dS, bst, bfn, &bp);
        if (el != cudaSuccess) BB_CK(el);
      }
      last_of_kernel<<<1, 1, 0, s>>>(bfn, nbp, busy_sum);
      note_launch();
      BB_CK(cudaGetLastError());
    } else {
      double* busy_part = nullptr;
      if (nb) {
        cudaError_t el = exact_lindley(dR, dS, start, finish, &busy_part);
        if (el != cudaSuccess) BB_CK(el);
      }
      if (busy_part) sum_kernel<<<1, 256, 0, s>>>(busy_part, 0, busy_sum, nbp);
      else BB_CK(cudaMemsetAsync(busy_sum, 0, 8, s));
      note_launch();
      BB_CK(cudaGetLastError());
    }
    // per-request pass
    unsigned long long *keys, *kminmax;
    double *lat_part, *lat_sum;
    const uint32_t qb = grid_for(n, RQ_T * RQ_E);
    const uint32_t qb_tm = grid_for(n, 256);
    BB_CK(pool.alloc((void**)&keys, (size_t)n * 8));
    BB_CK(pool.alloc((void**)&kminmax, 16));
    BB_CK(pool.alloc((void**)&lat_part, (size_t)std::max(qb, qb_tm) * 8));
    BB_CK(pool.alloc((void**)&lat_sum, 8));
    {
      static_assert(KEY_UNSERVED == ~0ull, "kminmax[0] starts all ones");
      BB_CK(cudaMemsetAsync(kminmax, 0xFF, 8, s));
      BB_CK(cudaMemsetAsync(kminmax + 1, 0, 8, s));
      QArgs Q{};
      Q.a = A.a;
      Q.pb8 = ws.pb8;
      Q.rank = ws.rank;
      Q.map = map;
      Q.finish = finish;
      Q.dfirst = dfirst;
      Q.info = ws.info;
      Q.divB = FastDiv(B);
      Q.n = n;
      Q.B = B;
      Q.k = k;
      Q.key = keys;
      Q.lat_part = lat_part;
      Q.kminmax = kminmax;
      Q.completion = A.req_completion;
      Q.batch = A.req_batch;
      Q.members = A.members;
      if (tm)
        tm_request_kernel<<<qb_tm, 256, 0, s>>>(A.a, ws.pb8, ws.rank, tm_off, tm_segj, tm_recP, map, finish,
                                             dfirst, n, keys, lat_part, kminmax, A.req_completion,
                                             A.req_batch, A.members);
      else
        request_kernel<<<qb, RQ_T, 0, s>>>(Q);
      note_launch();
      BB_CK(cudaGetLastError());
      sum_kernel<<<1, 256, 0, s>>>(lat_part, tm ? qb_tm : qb, lat_sum);
      note_launch();
      BB_CK(cudaGetLastError());
    }
    // exact p50/p99: device-side selection of interpolated_quantile's ranks
    // (binning.hpp:98-104), computed on the device from the completed count
    SelState* ds;
    {
      uint32_t* dh;
      unsigned long long* dc;
      const uint32_t cap = n < (1u << 22) ? n : (1u << 22);
      BB_CK(pool.alloc((void**)&ds, sizeof(SelState)));
      BB_CK(pool.alloc((void**)&dh, HBINS * 4));
      BB_CK(pool.alloc((void**)&dc, (size_t)cap * 8));
      BB_CK(cudaMemsetAsync(ds, 0, sizeof(SelState), s));
      BB_CK(cudaMemsetAsync(dh, 0, HBINS * 4, s));
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      sel_init_kernel<<<1, 1, 0, s>>>(ds, kminmax, ws.info);
      sel_hist_kernel<<<sms * 4, 256, 0, s>>>(keys, n, ds, dh);
      sel_find_kernel<<<1, 1024, 0, s>>>(ds, dh, cap);
      uint32_t* dh2;
      BB_CK(pool.alloc((void**)&dh2, (size_t)kSelMax * kSub * 4));
      BB_CK(cudaMemsetAsync(dh2, 0, (size_t)kSelMax * kSub * 4, s));
      unsigned long long* dl1;
      BB_CK(pool.alloc((void**)&dl1, (size_t)cap * 8));
      sel_hist2_kernel<<<sms * 2, 512, 0, s>>>(keys, n, ds, dh2, dl1, cap);
      sel_find2_kernel<<<1, 1024, 0, s>>>(ds, dh2, cap);
      sel_collect_kernel<<<sms * 4, 256, 0, s>>>(keys, n, dl1, ds, dc, cap);
      sel_refine_kernel<<<1, 1024, 0, s>>>(ds, dc);
      note_launch(7);
      BB_CK(cudaGetLastError());
    }
    double* scal;  // last completion, first arrival
    BB_CK(pool.alloc((void**)&scal, 16));
    scalars_kernel<<<1, 1, 0, s>>>(ws.info, finish, A.n_servers > 1 ? last_dev : nullptr, A.a, scal);
    note_launch();
    BB_CK(record(ev2));
    // one host round trip for everything the host reports
    Readback local{};
    Readback* rb = cap ? cap->rb : &local;
    {
      Readback* rdev = nullptr;  // the graph's pinned struct directly; else a device copy
      if (cap) BB_CK(cudaHostGetDevicePointer((void**)&rdev, cap->rb, 0));
      else BB_CK(pool.alloc((void**)&rdev, sizeof(Readback)));
      readback_kernel<<<1, 128, 0, s>>>(ReadbackSrc{ws.info, ws.err, scal, busy_sum, lat_sum, kminmax, ds}, rdev);
      note_launch();
      BB_CK(cudaGetLastError());
      if (!cap) BB_CK(cudaMemcpyAsync(rb, rdev, sizeof(Readback), cudaMemcpyDeviceToHost, s));
    }
    if (capturing) {
      cudaGraph_t g = nullptr;
      capturing = false;
      BB_CK(cudaStreamEndCapture(s, &g));
      const cudaError_t ei = cudaGraphInstantiate(&cap->exec, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) cap->exec = nullptr;
      BB_CK(ei);
      cap->launches = launches_noted_here() - launches0;
      BB_CK(cudaGraphLaunch(cap->exec, s));
    }
    BB_CK(cudaStreamSynchronize(s));
    if (!host_sync) {
      info = rb->info;
      herr = rb->herr;
      if (input_error()) goto cleanup;
      R->path = (int32_t)info.path;
    }
    if (!tm) {  // (the timer path counted its own batches)
      nb = info.nb;
      nc_run = info.nc;
      for (uint32_t b = 0; b < k; ++b) R->per_bin[b] = info.nbat[b];
    }
    R->n_batches = nb;
    R->n_completed = nc_run;
    // detail copies of the dispatch-ordered batch records
    if (A.bat_formed || A.bat_service || A.bat_first) {
      if (A.bat_formed) BB_CK(cudaMemcpyAsync(A.bat_formed, dR, (size_t)nb * 8, cudaMemcpyDeviceToDevice, s));
      if (A.bat_service) BB_CK(cudaMemcpyAsync(A.bat_service, dS, (size_t)nb * 8, cudaMemcpyDeviceToDevice, s));
      if (A.bat_first) BB_CK(cudaMemcpyAsync(A.bat_first, dfirst, (size_t)nb * 4, cudaMemcpyDeviceToDevice, s));
      BB_CK(cudaStreamSynchronize(s));
    }
    trace_report(A, R, *rb, nc_run, keys, &pool, s);
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    R->ms_partition = ms;
    cudaEventElapsedTime(&ms, ev0, ev2);
    R->ms_total = ms;
  }
cleanup:
  if (capturing) {  // a failed capture: end it and drop the graph
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    (void)cudaGetLastError();
  }
  if (!cap) {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
  }
  (void)dsize;
  (void)dbin;
}

// A replay of the captured pipeline; false when its selection overflowed
// (the caller reruns the direct path, which has the keys at hand).
static bool trace_replay(TraceGraph& G, const TraceArgs& A, TraceResult* R, cudaStream_t s) {
  std::memset(R, 0, sizeof *R);
  R->status = BB_OK;
  R->k = A.k;
  Pool pool;
  pool.s = s;
  cudaError_t e = pool.attach();
  if (e == cudaSuccess) e = cudaMemcpyAsync(G.edges, A.edges, (size_t)(A.k + 1) * 8, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && A.conf)
    e = cudaMemcpyAsync(G.conf, A.conf, (size_t)A.k * A.k * 8, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaGraphLaunch(G.exec, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    R->status = BB_ECUDA;
    snprintf(R->message, sizeof R->message, "CUDA error %s (trace graph)", cudaGetErrorString(e));
    return true;
  }
  note_launch((unsigned)G.launches);
  g_tg_replays.fetch_add(1);
  const Readback& rb = *G.rb;
  if (trace_input_error(rb.herr, rb.info, R)) return true;
  R->path = (int32_t)rb.info.path;
  for (uint32_t b = 0; b < A.k; ++b) R->per_bin[b] = rb.info.nbat[b];
  R->n_batches = rb.info.nb;
  R->n_completed = rb.info.nc;
  if (!trace_report(A, R, rb, rb.info.nc, nullptr, nullptr, s)) return false;
  float ms = 0;
  cudaEventElapsedTime(&ms, G.ev[0], G.ev[1]);
  R->ms_partition = ms;
  cudaEventElapsedTime(&ms, G.ev[0], G.ev[2]);
  R->ms_total = ms;
  return true;
}

static void trace_run_graph(const TraceArgs& A, TraceResult* R, cudaStream_t s);
void trace_run(const TraceArgs& A, TraceResult* R, cudaStream_t s) {
  trace_run_graph(A, R, s);
  static const bool dbg = getenv("BB_TRACE_MS") != nullptr;
  if (dbg) fprintf(stderr, "trace ms partition %.4f total %.4f\n", R->ms_partition, R->ms_total);
}
static void trace_run_graph(const TraceArgs& A, TraceResult* R, cudaStream_t s) {
  const bool graphable = s != nullptr && graphs_enabled() && !(A.max_batch_wait > 0) && !A.bat_formed &&
                         !A.bat_service && !A.bat_first && A.k >= 1 && A.k <= BB_TRACE_MAX_BINS;
  if (!graphable) return trace_run_impl(A, R, s, nullptr);
  int dev = 0;
  cudaGetDevice(&dev);
  TraceGraph& G = g_tgraph[dev & 63];
  const TraceArgs key = graph_key(A);
  if (G.have && std::memcmp(&key, &G.key, sizeof key) == 0) {
    if (trace_replay(G, A, R, s)) return;
    return trace_run_impl(A, R, s, nullptr);
  }
  if (!G.pend || std::memcmp(&key, &G.pend_key, sizeof key) != 0) {  // first sight: run directly
    G.pend = true;
    G.pend_key = key;
    return trace_run_impl(A, R, s, nullptr);
  }
  // the second identical call: capture it
  G.pend = false;
  G.have = false;
  if (G.exec) cudaGraphExecDestroy(G.exec);
  G.exec = nullptr;
  bool ok = true;
  for (int i = 0; i < 3 && ok; ++i)
    if (!G.ev[i]) ok = cudaEventCreate(&G.ev[i]) == cudaSuccess;
  if (ok && !G.rb) ok = cudaHostAlloc((void**)&G.rb, sizeof(Readback), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess;
  if (ok && !G.edges) ok = cudaMalloc((void**)&G.edges, (BB_TRACE_MAX_BINS + 1) * 8) == cudaSuccess;
  if (ok && !G.conf) ok = cudaMalloc((void**)&G.conf, BB_TRACE_MAX_BINS * BB_TRACE_MAX_BINS * 8) == cudaSuccess;
  if (ok) ok = cudaMemcpyAsync(G.edges, A.edges, (size_t)(A.k + 1) * 8, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
  if (ok && A.conf)
    ok = cudaMemcpyAsync(G.conf, A.conf, (size_t)A.k * A.k * 8, cudaMemcpyDeviceToDevice, s) == cudaSuccess;
  if (!ok) {
    (void)cudaGetLastError();
    return trace_run_impl(A, R, s, nullptr);
  }
  TraceArgs A2 = A;
  A2.edges = G.edges;
  A2.conf = A.conf ? G.conf : nullptr;
  trace_run_impl(A2, R, s, &G);
  G.have = G.exec != nullptr && R->status != BB_ECUDA;
  if (G.have) {
    G.key = key;
    g_tg_captures.fetch_add(1);
  }
}

void trace_graph_stats(uint64_t* captures, uint64_t* replays, bool reset) {
  const uint64_t c = reset ? g_tg_captures.exchange(0) : g_tg_captures.load();
  const uint64_t r = reset ? g_tg_replays.exchange(0) : g_tg_replays.load();
  if (captures) *captures = c;
  if (replays) *replays = r;
}

}  // namespace bb
