// bb_quantile.cuh -- exact per-replication latency quantiles for the fused
// generated-mode kernel.
//
// The reference computes p50/p99 of every replication (finish(),
// simulator.hpp:289-301: sort the completed requests' latencies, then
// interpolated_quantile, binning.hpp:97-104), and run_point averages them
// (experiment.hpp:262-263,278-279).  The fused kernel keeps one replication
// per lane in registers, so the latencies are not materialised during the
// simulation.  Instead the forward pass logs, per request, its arrival time
// and a byte (predicted bin | closing flag), and per closed batch its
// completion time; afterwards the warp selects the order statistics of one
// replication at a time:
//
//   source (finite rate): the request log read backwards in 32-request
//     tiles.  A request belongs to the batch closed by the next closing
//     request of its bin (or to its bin's drained partial), so
//     __match_any_sync over the bins + a ballot of the closing flags give
//     each lane the completion of its batch; a per-bin carry crosses tiles.
//     latency = completion - arrival, exactly the reference's subtraction.
//   source (overload): the batches' completions weighted by member counts.
//
//   select: radix histograms over the IEEE bit patterns of the (positive)
//     latencies -- 2048 buckets per pass, the first pass spanning
//     [min, max] from the forward pass, each further pass one bucket of the
//     previous -- until the buckets holding the wanted ranks fit in shared
//     memory; one more pass collects them and the ranks are resolved by
//     counting.  Typically two passes over the log (9 B/request each).
//
// Every value is an exact order statistic of the same multiset the reference
// sorts, and the interpolation uses the reference's operation order without
// contraction, so p50/p99 of a replication are bit-identical to the
// reference's finish() on the same completion and arrival times.
#pragma once
#include "bb_common.cuh"

namespace bb {

constexpr uint32_t kQBuckets = 2048;       // histogram buckets (8 KB of u32)
constexpr uint32_t kQRegionMin = 8192;     // per-warp shared region (histogram | candidates)
constexpr uint32_t kQFull = 0xFFFFFFFFu;
constexpr uint32_t kQBinInvalid = 0x7F;    // bin byte of lanes past the end

__device__ __forceinline__ uint64_t qkey(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ bool qin(uint64_t key, uint64_t lo, uint32_t sh) {
  return key >= lo && (sh >= 64 || ((key - lo) >> sh) == 0);
}
__device__ __forceinline__ uint64_t qwidth(uint32_t sh) { return sh >= 64 ? ~0ull : (1ull << sh); }

// Sources hand every (value, weight) of one replication to a functor, 32
// lanes at a time; kQGroup tiles are loaded before any is used so a warp has
// that many independent HBM loads in flight (the pass is latency bound
// otherwise).
constexpr int kQGroup = 8;
constexpr int kQChunk = 16;  // latency source: tiles per pipelined step

// Request-log layout (finite rate).  A warp's 32 replications share rows
// interleaved in blocks of 32 requests: request i of lane l lives at
// [(i/32)*1024 + l*32 + i%32] (arrivals, then latencies, fp64; the bytes
// alike).  The lanes walk their requests in lockstep, so a warp's stores and
// loads of one block stay inside 8 KB (full sectors once L2 merges them),
// and one replication's 32-request run is a contiguous 256 B that a warp
// reads in one coalesced access.  Completions of full batches: [c*32 + l].
// Rows are padded to a multiple of 32 requests.

// Finite arrival rate: one replication's latencies (NaN: never completed, or
// padding), converted in place from the request log by q_log_to_latency.
// L points at the replication's first run (stride 1024 doubles per run).
struct QSrcLat {
  const double* L;
  uint32_t n, lane;

  template <class Fn>
  __device__ void for_each(Fn&& f) const {
    // kQChunk tiles per step; the next step's loads are issued before this
    // step's values are used
    const uint32_t nt = (n + 31) / 32;
    double nx[kQChunk];
    auto load = [&](uint32_t t0) {
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) {
        const uint32_t t = t0 + u;
        nx[u] = (t < nt && t * 32 + lane < n) ? L[(size_t)t * 1024 + lane] : BB_QNAN;
      }
    };
    load(0);
    for (uint32_t t0 = 0; t0 < nt; t0 += kQChunk) {
      double x[kQChunk];
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) x[u] = nx[u];
      if (t0 + kQChunk < nt) load(t0 + kQChunk);
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) f(x[u], isnan(x[u]) ? 0u : 1u);
    }
  }
};

// Finite arrival rate, first pass: one replication's request log read
// newest tile first.  A request belongs to the batch closed by the next
// closing request of its bin (or to its bin's drained partial), so
// __match_any_sync over the bins and a ballot of the closing flags give each
// lane the completion of its batch; a per-bin carry crosses tiles.  latency =
// completion - arrival (the reference's subtraction, simulator.hpp:293) is
// written over the arrival, so later passes read QSrcLat, and summed per lane
// (latency_mean).  kQGroup tiles are loaded, then their completions gathered,
// before any carry is resolved.
struct QSrcLogRev {
  double* A;            // the replication's first run (stride 1024 per run)
  const uint8_t* Bf;    //   its bytes, same layout
  const double* F;      // completions: F[c*32] for closing c
  const double* P;      // per bin: P[b*32] completion of the drained partial (NaN: none)
  double* carry;        // shared, per bin
  uint32_t n, nclose, k, lane;
  double sum;           // this lane's share of the latency sum

  template <class Fn>
  __device__ void for_each(Fn&& f) {
    for (uint32_t b = lane; b < k; b += 32) carry[b] = P[b * 32];
    __syncwarp();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t cend = nclose;
    for (int32_t thi = (int32_t)((n + 31) / 32); thi > 0; thi -= kQGroup) {
      double a[kQGroup], fin[kQGroup];
      uint32_t byte[kQGroup], peers[kQGroup], cm[kQGroup];
      int32_t fi[kQGroup];
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) {  // tile thi-1-u, all loads issued together
        const int32_t t = thi - 1 - u;
        const bool valid = t >= 0 && (uint32_t)t * 32u + lane < n;
        a[u] = valid ? A[(size_t)t * 1024 + lane] : 0.0;
        byte[u] = valid ? (uint32_t)Bf[(size_t)t * 1024 + lane] : kQBinInvalid;
      }
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) {
        const uint32_t b = byte[u] & 0x7F, c = byte[u] >> 7;
        peers[u] = __match_any_sync(kQFull, b);
        cm[u] = __ballot_sync(kQFull, c);
        const uint32_t cbase = cend - __popc(cm[u]);
        const uint32_t cand = peers[u] & cm[u] & ~lt;  // closings of my bin at or after me
        fi[u] = cand ? (int32_t)(cbase + __popc(cm[u] & ((1u << (__ffs(cand) - 1)) - 1u))) : -1;
        cend = cbase;
      }
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) fin[u] = fi[u] >= 0 ? F[(size_t)fi[u] * 32] : BB_QNAN;
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) {  // per-bin carry, newest tile first
        const uint32_t b = byte[u] & 0x7F, c = byte[u] >> 7;
        if (fi[u] < 0 && b != kQBinInvalid) fin[u] = carry[b];
        __syncwarp();
        if (c && !(peers[u] & cm[u] & lt)) carry[b] = fin[u];  // earliest closing of its bin
        __syncwarp();
      }
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) {
        const int32_t t = thi - 1 - u;
        const bool valid = byte[u] != kQBinInvalid;
        const double x = valid ? __dsub_rn(fin[u], a[u]) : BB_QNAN;
        if (t >= 0) A[(size_t)t * 1024 + lane] = x;  // padding lanes become NaN
        const bool ok = !isnan(x);
        if (ok) sum += x;
        f(x, ok ? 1u : 0u);
      }
    }
  }
};

// Overload (and any batch list): completion per batch, weighted by members.
struct QSrcBatches {
  const double* V;
  const uint16_t* M;
  size_t stride;
  uint32_t nb, lane;

  template <class Fn>
  __device__ void for_each(Fn&& f) const {
    for (uint32_t t0 = 0; t0 * 32 < nb; t0 += kQGroup) {
      double x[kQGroup];
      uint32_t w[kQGroup];
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) {
        const uint32_t i = (t0 + u) * 32 + lane;
        x[u] = i < nb ? V[(size_t)i * stride] : 0.0;
        w[u] = i < nb ? M[(size_t)i * stride] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kQGroup; ++u) f(x[u], w[u]);
    }
  }
};

// Exact p50 and p99 (interpolated_quantile, binning.hpp:97-104) of the
// multiset produced by `src` (m = total weight, every value in [lmin, lmax],
// all positive).  Warp-collective; results are warp-uniform.
// region: >= kQRegionMin bytes of shared memory (histogram, then candidates);
// ans: 4 doubles of shared memory.
template <class Src1, class Src>
__device__ void q_select(Src1& first, const Src& src, uint64_t m, double lmin, double lmax, unsigned char* region,
                         uint32_t region_bytes, double* ans, uint32_t lane, double& p50,
                         double& p99) {
  uint32_t* hist = reinterpret_cast<uint32_t*>(region);
  const uint32_t cap = ((region_bytes - 1024u) / 10u) & ~7u;  // + a 256-bucket histogram
  double* cx = reinterpret_cast<double*>(region);
  uint16_t* cw = reinterpret_cast<uint16_t*>(region + (size_t)cap * 8u);

  // wanted ranks: idx and idx+1 of both quantiles
  const double pos50 = __dmul_rn(0.5, (double)(m - 1));
  const double pos99 = __dmul_rn(0.99, (double)(m - 1));
  const uint64_t i50 = (uint64_t)pos50, i99 = (uint64_t)pos99;
  uint64_t rk[4] = {i50, i50 + 1 < m ? i50 + 1 : i50, i99, i99 + 1 < m ? i99 + 1 : i99};
  uint64_t klo[4], below[4], cnt[4];
  uint32_t sh[4];
  double val[4];
  bool done[4];
  const uint64_t kbase = qkey(lmin), kspan = qkey(lmax) - kbase;
  uint32_t sh0 = 0;
  while (sh0 < 63 && (kspan >> sh0) >= kQBuckets) ++sh0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    klo[t] = kbase;
    sh[t] = 64;
    below[t] = 0;
    cnt[t] = m;
    done[t] = false;
    val[t] = 0.0;
  }

  // one histogram pass over the range (glo, gsh); every target in that range
  // moves to the sub-bucket holding its rank
  auto refine = [&](auto& source, uint64_t glo, uint32_t gsh) {
    const uint32_t s2 = gsh >= 64 ? sh0 : (gsh > 11 ? gsh - 11 : 0);
    for (uint32_t j = lane; j < kQBuckets; j += 32) hist[j] = 0;
    __syncwarp();
    const uint64_t gw = qwidth(gsh);
    source.for_each([&](double x, uint32_t w) {
      const uint64_t d = qkey(x) - glo;
      if (w && d < gw) {
        const uint64_t bk = d >> s2;
        atomicAdd(&hist[bk < kQBuckets ? bk : kQBuckets - 1], w);
      }
    });
    __syncwarp();
    uint32_t loc = 0;
    for (uint32_t j = 0; j < kQBuckets / 32; ++j) loc += hist[lane * (kQBuckets / 32) + j];
    uint32_t pre = loc;  // inclusive scan over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kQFull, pre, o);
      if (lane >= (uint32_t)o) pre += v;
    }
    pre -= loc;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (done[t] || klo[t] != glo || sh[t] != gsh) continue;
      const uint64_t r = rk[t] - below[t];
      const bool mine = r >= pre && r < (uint64_t)pre + loc;
      const uint32_t who = __ffs(__ballot_sync(kQFull, mine)) - 1;
      uint32_t b = 0, c = 0, h = 0;
      if (mine) {
        c = pre;
        for (uint32_t j = 0; j < kQBuckets / 32; ++j) {
          h = hist[lane * (kQBuckets / 32) + j];
          if (r < (uint64_t)c + h) {
            b = lane * (kQBuckets / 32) + j;
            break;
          }
          c += h;
        }
      }
      b = __shfl_sync(kQFull, b, who);
      c = __shfl_sync(kQFull, c, who);
      h = __shfl_sync(kQFull, h, who);
      klo[t] = glo + ((uint64_t)b << s2);
      sh[t] = s2;
      below[t] += c;
      cnt[t] = h;
    }
    __syncwarp();
  };

  refine(first, kbase, 64);
  for (int iter = 0; iter < 64; ++iter) {
    // a range of one bit pattern holds equal values: resolved without a pass
    uint64_t total = 0;
    int big = -1;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (done[t]) continue;
      if (sh[t] == 0) {
        done[t] = true;
        val[t] = __longlong_as_double((long long)klo[t]);
        continue;
      }
      bool first = true;  // count each distinct range once
#pragma unroll
      for (int u = 0; u < t; ++u)
        if (!done[u] && klo[u] == klo[t] && sh[u] == sh[t]) first = false;
      if (first) {
        total += cnt[t];
        if (big < 0 || cnt[t] > cnt[big]) big = t;
      }
    }
    if (big < 0 || total <= cap) break;
    uint64_t glo = 0;
    uint32_t gsh = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t == big) glo = klo[t], gsh = sh[t];
    refine(src, glo, gsh);
  }

  bool open = false;
#pragma unroll
  for (int t = 0; t < 4; ++t) open |= !done[t];
  if (open) {
    // collect the candidates of every open range
    uint32_t nc = 0;
    uint64_t wlo[4], ww[4];  // open ranges (width 0: closed)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      wlo[t] = klo[t];
      ww[t] = done[t] ? 0ull : qwidth(sh[t]);
    }
    src.for_each([&](double x, uint32_t w) {
      const uint64_t key = qkey(x);
      bool hit = false;
#pragma unroll
      for (int t = 0; t < 4; ++t) hit |= (key - wlo[t]) < ww[t];
      hit &= w != 0;
      const uint32_t hm = __ballot_sync(kQFull, hit);
      if (hit) {
        const uint32_t at = nc + __popc(hm & ((1u << lane) - 1u));
        if (at < cap) {
          cx[at] = x;
          cw[at] = (uint16_t)w;
        }
      }
      nc += __popc(hm);
    });
    if (nc > cap) nc = cap;  // cannot happen: the ranges were refined to fit
    __syncwarp();
    // resolve each open rank among the candidates: 256-bucket histograms of
    // the candidates in shared memory until at most 32 remain, then count
    uint32_t* h2 = reinterpret_cast<uint32_t*>(region + (size_t)cap * 10u);
#pragma unroll 1
    for (int t = 0; t < 4; ++t) {
      if (done[t]) continue;
      uint64_t lo = klo[t], r = rk[t] - below[t], cn = cnt[t];
      uint32_t s = sh[t];
      while (cn > 32 && s > 0) {
        const uint32_t s2 = s > 8 ? s - 8 : 0;
        for (uint32_t j = lane; j < 256; j += 32) h2[j] = 0;
        __syncwarp();
        for (uint32_t c = lane; c < nc; c += 32) {
          const uint64_t key = qkey(cx[c]);
          if (qin(key, lo, s)) atomicAdd(&h2[(key - lo) >> s2], (uint32_t)cw[c]);
        }
        __syncwarp();
        uint32_t loc = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) loc += h2[lane * 8 + j];
        uint32_t pre = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(kQFull, pre, o);
          if (lane >= (uint32_t)o) pre += v;
        }
        pre -= loc;
        const bool mine = r >= pre && r < (uint64_t)pre + loc;
        const uint32_t who = __ffs(__ballot_sync(kQFull, mine)) - 1;
        uint32_t bsel = 0, cb = 0, hb = 0;
        if (mine) {
          cb = pre;
          for (uint32_t j = 0; j < 8; ++j) {
            hb = h2[lane * 8 + j];
            if (r < (uint64_t)cb + hb) {
              bsel = lane * 8 + j;
              break;
            }
            cb += hb;
          }
        }
        bsel = __shfl_sync(kQFull, bsel, who);
        cb = __shfl_sync(kQFull, cb, who);
        hb = __shfl_sync(kQFull, hb, who);
        lo += (uint64_t)bsel << s2;
        s = s2;
        r -= cb;
        cn = hb;
        __syncwarp();
      }
      if (s == 0) {  // one bit pattern: all equal
        val[t] = __longlong_as_double((long long)lo);
        continue;
      }
      // <= 32 candidates (weights >= 1) left: one per lane, then count
      double* fy = reinterpret_cast<double*>(h2);
      uint32_t* fw = h2 + 64;
      uint32_t got = 0;
      for (uint32_t c0 = 0; c0 < nc; c0 += 32) {
        const uint32_t c = c0 + lane;
        const bool in = c < nc && qin(qkey(cx[c]), lo, s);
        const uint32_t m = __ballot_sync(kQFull, in);
        if (in) {
          const uint32_t at = got + __popc(m & ((1u << lane) - 1u));
          fy[at] = cx[c];
          fw[at] = cw[c];
        }
        got += __popc(m);
      }
      __syncwarp();
      const double y = lane < got ? fy[lane] : 0.0;
      const uint32_t wy = lane < got ? fw[lane] : 0u;
      __syncwarp();
      uint64_t lt = 0, le = 0;
      for (uint32_t j = 0; j < got; ++j) {
        const double z = __shfl_sync(kQFull, y, j);
        const uint32_t wz = __shfl_sync(kQFull, wy, j);
        lt += z < y ? wz : 0u;
        le += z <= y ? wz : 0u;
      }
      const bool ans_here = lane < got && lt <= r && r < le;
      const uint32_t wl = __ffs(__ballot_sync(kQFull, ans_here)) - 1;
      val[t] = __shfl_sync(kQFull, y, wl);
    }
  }
  // interpolated_quantile (binning.hpp:97-104), no contraction
  const double f50 = __dsub_rn(pos50, (double)i50), f99 = __dsub_rn(pos99, (double)i99);
  p50 = i50 + 1 >= m ? val[0] : __dadd_rn(val[0], __dmul_rn(f50, __dsub_rn(val[1], val[0])));
  p99 = i99 + 1 >= m ? val[2] : __dadd_rn(val[2], __dmul_rn(f99, __dsub_rn(val[3], val[2])));
  __syncwarp();
}

}  // namespace bb
