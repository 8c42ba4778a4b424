// bb_quantile.cuh -- exact per-replication latency quantiles for the fused
// generated-mode kernel.
//
// The reference computes p50/p99 of every replication (finish(),
// simulator.hpp:289-301: sort the completed requests' latencies, then
// interpolated_quantile, binning.hpp:97-104), and run_point averages them
// (experiment.hpp:262-263,278-279).  The fused kernel keeps one replication
// per lane in registers, so the latencies are not materialised during the
// simulation.  Instead the forward pass logs, per request, its arrival time
// and its batch's id (batches get ids when their first member arrives), and
// per batch id its completion time; afterwards the warp selects the order
// statistics of one replication at a time:
//
//   source (finite rate): latency_i = F[id_i] - a_i, the reference's
//     subtraction, for every request independently (QFast::level0 streams
//     the log with a three-stage software pipeline; QSrcLog for later passes).
//   source (overload): the batches' completions weighted by member counts.
//
//   select: level 0 is a 2048-bucket histogram of a monotone 32-bit function
//     of the latencies' IEEE bits over [min, max] from the forward pass,
//     leaving each request's bucket id; when the wanted ranks' buckets fit
//     in shared memory one more pass collects them by bucket id (2 B per
//     request) and the ranks are resolved by 256-bucket refinements and
//     counting; otherwise further histogram passes narrow the buckets first.
//
// Every value is an exact order statistic of the same multiset the reference
// sorts, and the interpolation uses the reference's operation order without
// contraction, so p50/p99 of a replication are bit-identical to the
// reference's finish() on the same completion and arrival times.
#pragma once
#include "bb_common.cuh"

namespace bb {

#ifndef BB_QL0AGG
#define BB_QL0AGG 0  // A/B: warp-aggregated level-0 increments (match_any): 284 vs 232 ms, off
#endif
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
#ifndef BB_QCHUNK
#define BB_QCHUNK 8
#endif
constexpr int kQChunk = BB_QCHUNK;  // request-log sources: runs per pipelined step

// Request-log layout (finite rate).  Every batch gets an id when its first
// member arrives (its bin's open batch; ids count openings per replication),
// and every request logs (arrival, batch id); a batch's completion is written
// once, at its id, when it is dispatched (drained partials at the end; NaN if
// it never completes).  So latency_i = F[id_i] - a_i -- the reference's
// subtraction (simulator.hpp:293) -- for every request independently.
//
// A warp's 32 replications share rows interleaved in runs of kQRun
// requests: request i of lane l lives at [(i/R)*32R + l*R + i%R] (arrival
// fp64, id u32).  The lanes walk their requests in lockstep, so one store
// instruction of the forward pass covers 32 runs side by side (few cache
// lines), and the selection's warp-wide reads of one replication cover
// 32/R runs.  Completions: a contiguous row per lane.  Rows are padded to a
// multiple of 32 requests.
#ifndef BB_QRUN
#define BB_QRUN 32
#endif
constexpr uint32_t kQRun = BB_QRUN;
// completions by batch id: a row per lane (stride 1) or the warp's 32 rows
// interleaved (stride 32: lanes closing batches together store nearby)
#ifndef BB_QFSTRIDE
#define BB_QFSTRIDE 1
#endif
constexpr uint32_t kQFStride = BB_QFSTRIDE;
__host__ __device__ __forceinline__ size_t qlog_index(uint32_t i) {
  return (size_t)(i / kQRun) * (32 * kQRun) + (i % kQRun);
}
// the same with the distance between a replication's consecutive runs given:
// 32 kQRun in the interleaved warp rows, kQRun in a replication's own
// contiguous log (the warp-per-replication kernel, bb_genw_kernel.cuh)
__host__ __device__ __forceinline__ size_t qlog_index(uint32_t i, uint32_t run_stride) {
  return (size_t)(i / kQRun) * run_stride + (i % kQRun);
}

template <bool WRITE>
struct QSrcLog {
  double* A;            // the replication's first run (+ qlog_index(i, rs))
  const uint32_t* Id;   //   its batch ids, same layout
  const double* F;      // its completions by batch id
  uint32_t n, lane;
  uint32_t rs = 32 * kQRun;  // run stride

  template <class Fn>
  __device__ void for_each(Fn&& f) const {
    // kQChunk runs per step; the next step's loads are issued before this
    // step's values are used
    const uint32_t nt = (n + 31) / 32;
    double na[kQChunk];
    uint32_t nid[kQChunk];
    auto load = [&](uint32_t t0) {
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) {
        const uint32_t t = t0 + u;
        const bool v = t < nt && t * 32 + lane < n;
        const size_t o = qlog_index(t * 32 + lane, rs);
        na[u] = v ? A[o] : 0.0;
        nid[u] = v ? Id[o] : 0xFFFFFFFFu;
      }
    };
    load(0);
    for (uint32_t t0 = 0; t0 < nt; t0 += kQChunk) {
      double a[kQChunk], fin[kQChunk];
      uint32_t id[kQChunk];
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) {
        a[u] = na[u];
        id[u] = nid[u];
      }
      if (t0 + kQChunk < nt) load(t0 + kQChunk);
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) fin[u] = id[u] != 0xFFFFFFFFu ? F[(size_t)id[u] * kQFStride] : BB_QNAN;
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) {
        const double x = __dsub_rn(fin[u], a[u]);
        const uint32_t t = t0 + u;
        if (WRITE && t < nt) A[qlog_index(t * 32 + lane, rs)] = x;  // later passes read QSrcLat
        f(x, isnan(x) ? 0u : 1u, t * 32 + lane);
      }
    }
  }
};

// Later passes: the latencies the first pass wrote over the arrivals.
struct QSrcLat {
  const double* L;
  uint32_t n, lane;

  template <class Fn>
  __device__ void for_each(Fn&& f) const {
    const uint32_t nt = (n + 31) / 32;
    double nx[kQChunk];
    auto load = [&](uint32_t t0) {
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) {
        const uint32_t t = t0 + u;
        nx[u] = (t < nt && t * 32 + lane < n) ? L[qlog_index(t * 32 + lane)] : BB_QNAN;
      }
    };
    load(0);
    for (uint32_t t0 = 0; t0 < nt; t0 += kQChunk) {
      double x[kQChunk];
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) x[u] = nx[u];
      if (t0 + kQChunk < nt) load(t0 + kQChunk);
#pragma unroll
      for (int u = 0; u < kQChunk; ++u) f(x[u], isnan(x[u]) ? 0u : 1u, (t0 + u) * 32 + lane);
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
      for (int u = 0; u < kQGroup; ++u) f(x[u], w[u], (t0 + u) * 32 + lane);
    }
  }
};

// Fast collection for the request log: the first pass leaves every request's
// level-0 histogram bucket (u16, 0xFFFF: not completed) in the log layout, so
// the collect pass scans 2 B per request -- eight requests per lane and load
// -- and keeps only the indices of requests in the wanted buckets; their
// latencies are then gathered with independent loads.
struct QFast {
  uint16_t* Bk;         // the replication's buckets (+ qlog_index(i, rs))
  const double* A;      // its arrivals
  const uint32_t* Id;   // its batch ids
  const double* F;      // its completions by batch id
  uint32_t n, lane;
  uint32_t rs = 32 * kQRun;  // run stride

  // Level 0 of the selection in one lean pass over the log: every request's
  // latency F[id] - a (the reference's subtraction), their sum, a histogram
  // of b = min((hi32(key) - hbase) >> s, 2047) -- a monotone function of the
  // key, so every bucket is a contiguous key range [(hbase + b 2^s) 2^32,
  // + 2^(s+32)) -- and b itself per request (0xFFFF: never completed) for
  // the collect pass.  A lane reads request t*32 + lane of the replication,
  // so each run of 32 is one 256 B (arrivals) + 128 B (ids) access; 32-bit
  // offsets, no predication outside the ragged last run.
  __device__ double level0(uint32_t* hist, uint32_t hbase, uint32_t s) const {
    const uint32_t full = n / 32, nt = (n + 31) / 32;
    const double* a_p = A + lane;
    const uint32_t* i_p = Id + lane;
    uint16_t* k_p = Bk + lane;
    double acc = 0.0;
    auto one = [&](double a, double f, bool valid, uint32_t off) {
      const double x = __dsub_rn(f, a);
      const bool done = valid && x == x;  // NaN: the batch never completed
      uint32_t b = 0xFFFFu;
      if (done) {
        b = min((uint32_t)(__double2hiint(x) - (int)hbase) >> s, kQBuckets - 1);
#if BB_QL0AGG
        // neighbouring requests share buckets: one shared atomic per bucket
        const uint32_t peers = __match_any_sync(__activemask(), b);
        if ((peers & ((1u << lane) - 1u)) == 0) atomicAdd(&hist[b], (uint32_t)__popc(peers));
#else
        atomicAdd(&hist[b], 1u);
#endif
        acc += x;
      }
      if (valid) k_p[off] = (uint16_t)b;
    };
    // three-stage software pipeline over chunks of C runs: while chunk t is
    // used, chunk t+1's completions (gathered by its batch ids) and chunk
    // t+2's arrivals and ids are in flight -- the id -> completion gather
    // is a second dependent round trip, so it is issued one chunk early
#ifndef BB_QL0C
#define BB_QL0C 6
#endif
    constexpr int C = BB_QL0C;
    const uint32_t R = rs;
    uint32_t t = 0;
    double a1[C], f1[C], a2[C];
    uint32_t i2[C];
    if (2 * C <= full) {
#pragma unroll
      for (int u = 0; u < C; ++u) {
        a1[u] = a_p[u * R];
        a2[u] = a_p[(C + u) * R];
        i2[u] = i_p[(C + u) * R];
      }
#pragma unroll
      for (int u = 0; u < C; ++u) f1[u] = F[i_p[u * R]];
      for (; t + 2 * C <= full; t += C) {
        double a[C], f[C];
#pragma unroll
        for (int u = 0; u < C; ++u) {
          a[u] = a1[u];
          f[u] = f1[u];
          a1[u] = a2[u];
          f1[u] = F[i2[u]];  // chunk t+1
        }
        if (t + 3 * C <= full) {
#pragma unroll
          for (int u = 0; u < C; ++u) {  // chunk t+2
            a2[u] = a_p[(t + 2 * C + u) * R];
            i2[u] = i_p[(t + 2 * C + u) * R];
          }
        }
#pragma unroll
        for (int u = 0; u < C; ++u) one(a[u], f[u], true, (t + u) * R);
      }
      // chunk t (its a1/f1 are loaded) is the last full one of the pipeline
#pragma unroll
      for (int u = 0; u < C; ++u) one(a1[u], f1[u], true, (t + u) * R);
      t += C;
    }
    for (; t < nt; ++t) {
      const bool v = t * 32 + lane < n;
      one(v ? a_p[t * R] : 0.0, v ? F[i_p[t * R]] : 0.0, v, t * R);
    }
    return acc;
  }

  // indices of the requests whose level-0 bucket lies in [w0, w0 + d0] or
  // [w2, w2 + d2] into slots[] (raw 64-bit words); returns how many.  The
  // ranges are exact (the buckets of ranks i and i+1 are equal or every
  // bucket between them is empty), and hits are sparse: a lane tests its
  // eight buckets with two range compares each and the warp only places
  // hits when some lane has one.
  __device__ uint32_t collect(uint32_t w0, uint32_t d0, uint32_t w2, uint32_t d2,
                              unsigned long long* slots) const {
    static_assert(kQRun % 8 == 0, "eight buckets per lane load");
    constexpr int G = 4;  // loads in flight per lane
    const uint32_t ng = (n + 7) / 8;  // groups of 8 requests
    uint32_t nc = 0;
    for (uint32_t g0 = 0; g0 < ng; g0 += 32 * G) {
      uint4 v[G];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const uint32_t g = g0 + u * 32 + lane;
        v[u] = g < ng ? *reinterpret_cast<const uint4*>(Bk + qlog_index(g * 8, rs))
                      : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        const uint32_t base = (g0 + u * 32 + lane) * 8;
        uint32_t hm = 0;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const uint32_t bk = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
          hm |= (uint32_t)((bk - w0 <= d0) | (bk - w2 <= d2)) << h;
        }
        if (base + 8 > n) hm &= base < n ? (1u << (n - base)) - 1u : 0u;  // (padding is never written)
        if (!__any_sync(kQFull, hm != 0)) continue;
        const uint32_t c = __popc(hm);
        uint32_t pre = c;  // inclusive scan of the hit counts over the lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kQFull, pre, o);
          if (lane >= (uint32_t)o) pre += y;
        }
        uint32_t at = nc + pre - c;
        while (hm) {
          const uint32_t h = __ffs(hm) - 1;
          hm &= hm - 1;
          slots[at++] = (unsigned long long)(base + h);
        }
        nc += __shfl_sync(kQFull, pre, 31);
      }
    }
    return nc;
  }
  __device__ double latency(uint32_t i) const {
    const size_t o = qlog_index(i, rs);
    return __dsub_rn(F[(size_t)Id[o] * kQFStride], A[o]);
  }
};

// Later passes of the request log, reading only the requests whose level-0
// bucket is one of want[0..3] (every open target lies inside its level-0
// bucket): a scan of the 2-byte bucket ids, the latency recomputed for the
// few hits.  f is called by all lanes in lockstep (weight 0 for no element),
// once per row of eight buckets in which some lane has a hit.
struct QBkSrc {
  const QFast* qf;
  uint32_t want[4];

  template <class Fn>
  __device__ void for_each(Fn&& f) const {
    const uint32_t n = qf->n, lane = qf->lane;
    const uint32_t ng = (n + 7) / 8;
    for (uint32_t g0 = 0; g0 < ng; g0 += 32) {
      const uint32_t g = g0 + lane;
      const uint4 v = g < ng ? *reinterpret_cast<const uint4*>(qf->Bk + qlog_index(g * 8, qf->rs))
                             : make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t hm = 0;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const uint32_t bk = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
        hm |= (uint32_t)(bk == want[0] || bk == want[1] || bk == want[2] || bk == want[3]) << h;
      }
      const uint32_t base = g * 8;
      if (base + 8 > n) hm &= base < n ? (1u << (n - base)) - 1u : 0u;
      uint32_t rows = __reduce_or_sync(kQFull, hm);
      while (rows) {
        const int h = __ffs(rows) - 1;
        rows &= rows - 1;
        const bool hit = (hm >> h) & 1u;
        const double x = hit ? qf->latency(base + h) : 0.0;
        f(x, hit ? 1u : 0u, base + h);
      }
    }
  }
};

// Exact p50 and p99 (interpolated_quantile, binning.hpp:97-104) of the
// multiset produced by `src` (m = total weight, every value in [lmin, lmax],
// all positive).  Warp-collective; results are warp-uniform.
// region: >= kQRegionMin bytes of shared memory (histogram, then candidates);
// ans: 4 doubles of shared memory.
// BK: the slow path (targets' level-0 buckets too full for shared memory)
// re-reads only the requests of those buckets through their bucket ids
// (QBkSrc) instead of the whole log -- the long replications of the warp
// kernel reach it often; the lane kernel rarely does and keeps its registers
template <class Src1, class Src, bool BK = false>
__device__ void q_select(Src1& first, const Src& src, uint64_t m, double lmin, double lmax, unsigned char* region,
                         uint32_t region_bytes, double* ans, uint32_t lane, double& p50,
                         double& p99, double* wsum, const QFast* qf = nullptr) {
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
  uint32_t fast_nc = 0;
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
  // (the first pass also sums the values for the caller, when asked)
  auto refine = [&](auto& source, uint64_t glo, uint32_t gsh, bool sum) {
    const uint32_t s2 = gsh >= 64 ? sh0 : (gsh > 11 ? gsh - 11 : 0);
    for (uint32_t j = lane; j < kQBuckets; j += 32) hist[j] = 0;
    __syncwarp();
    const uint64_t gw = qwidth(gsh);
    double acc = 0.0;
    source.for_each([&](double x, uint32_t w, uint32_t i) {
      if (sum && w) acc += x * (double)w;
      const uint64_t d = qkey(x) - glo;
      uint32_t b16 = 0xFFFFu;
      if (w && d < gw) {
        const uint64_t bk = d >> s2;
        b16 = (uint32_t)(bk < kQBuckets ? bk : kQBuckets - 1);
        atomicAdd(&hist[b16], w);
      }
    });
    if (sum) {
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kQFull, acc, o);
      *wsum = acc;
    }
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

  uint32_t hb = 0, hs = 0;  // request log: level-0 buckets over the keys' high words
  QBkSrc bksrc{qf, {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}};
  if (qf) {
    hb = (uint32_t)(kbase >> 32);
    const uint32_t hspan = (uint32_t)(qkey(lmax) >> 32) - hb;
    while ((hspan >> hs) >= kQBuckets) ++hs;
    for (uint32_t j = lane; j < kQBuckets; j += 32) hist[j] = 0;
    __syncwarp();
    double acc = qf->level0(hist, hb, hs);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kQFull, acc, o);
    if (wsum) *wsum = acc;
    __syncwarp();
    // bucket b holds the keys [(hb + b 2^hs) 2^32, + 2^(hs+32))
    uint32_t loc = 0;
    for (uint32_t j = 0; j < kQBuckets / 32; ++j) loc += hist[lane * (kQBuckets / 32) + j];
    uint32_t pre = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kQFull, pre, o);
      if (lane >= (uint32_t)o) pre += v;
    }
    pre -= loc;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint64_t r = rk[t];
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
      if constexpr (BK) bksrc.want[t] = b;
      klo[t] = (uint64_t)(hb + (b << hs)) << 32;
      sh[t] = hs + 32;
      below[t] = __shfl_sync(kQFull, c, who);
      cnt[t] = __shfl_sync(kQFull, h, who);
    }
    __syncwarp();
  } else {
    refine(first, kbase, 64, wsum != nullptr);
  }
  // fast path: the level-0 buckets of the wanted ranks hold few enough values
  bool fast = false;
  if (qf) {
    uint64_t total = cnt[0] + cnt[2];
    if (klo[1] != klo[0]) total += cnt[1];
    if (klo[3] != klo[2]) total += cnt[3];
    if (klo[2] == klo[0] || klo[2] == klo[1]) total -= cnt[2];
    if (klo[3] != klo[2] && (klo[3] == klo[0] || klo[3] == klo[1])) total -= cnt[3];
    if (total <= cap) {
      fast = true;
      __syncwarp();  // the histogram is done with; the region holds candidates
      unsigned long long* slots = reinterpret_cast<unsigned long long*>(cx);
      // buckets of ranks i and i+1: equal, or every bucket between them empty
      const uint32_t b0 = (uint32_t)((klo[0] >> 32) - hb) >> hs, b1 = (uint32_t)((klo[1] >> 32) - hb) >> hs;
      const uint32_t b2 = (uint32_t)((klo[2] >> 32) - hb) >> hs, b3 = (uint32_t)((klo[3] >> 32) - hb) >> hs;
      const uint32_t ncol = qf->collect(b0, b1 - b0, b2, b3 - b2, slots);
      __syncwarp();
      for (uint32_t c = lane; c < ncol; c += 32) {
        const double x = qf->latency((uint32_t)slots[c]);
        cx[c] = x;
        cw[c] = 1;
      }
      __syncwarp();
      fast_nc = ncol;
    }
  }
  for (int iter = 0; !fast && iter < 64; ++iter) {
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
    if constexpr (BK) {
      if (qf) refine(bksrc, glo, gsh, false);  // (only the targets' level-0 buckets)
      else refine(src, glo, gsh, false);
    } else {
      refine(src, glo, gsh, false);
    }
  }

  bool open = false;
#pragma unroll
  for (int t = 0; t < 4; ++t) open |= !done[t];
  if (open) {
    // collect the candidates of every open range
    uint32_t nc = fast ? fast_nc : 0;
    uint64_t wlo[4], ww[4];  // open ranges (width 0: closed)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      wlo[t] = klo[t];
      ww[t] = done[t] ? 0ull : qwidth(sh[t]);
    }
    auto keep = [&](double x, uint32_t w, uint32_t) {
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
    };
    if (!fast) {
      if constexpr (BK) {
        if (qf) bksrc.for_each(keep);  // (only the targets' level-0 buckets)
        else src.for_each(keep);
      } else {
        src.for_each(keep);
      }
    }
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
