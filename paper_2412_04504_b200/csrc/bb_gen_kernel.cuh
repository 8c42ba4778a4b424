// bb_generated.cu -- generated-mode Monte Carlo engine (K1 + K7 + K6 of SURVEY §2.3).
//
// One thread simulates one replication end to end, a warp owns 32
// replications of one sweep point, and a persistent grid walks the
// (point, 32-replication chunk) work list.  Per request the thread draws one
// Philox4x32-10 block (53-bit inter-arrival uniform + 53-bit service key),
// assigns the bin in key space, folds the request into its bin's packed
// (max key, count) word in shared memory and, when the bin reaches B, closes
// the batch with the single-server Lindley step
//     D = max(D, R) + S,  R = arrival of the closing request
// (simulator.hpp:256-267 with one server).  Nothing per request
// touches HBM: the kernel is SM-issue bound.
//
// Dispatch semantics reproduced:
//   finite lambda -- batches dispatch in closing-request order, then the
//     final partials in bin order 1..k (drain events, simulator.hpp:203-205);
//   overload -- one tie group: round 0 in first-closing order, then either
//     round-robin rounds (no flush) or per-bin drains (flush).  Positions are
//     closed-form from a first counting pass; the second pass replays the
//     same counter-based draws.
#pragma once
#include <type_traits>

#include "bb_generated.cuh"
#include "bb_quantile.cuh"

namespace bb {
namespace {

#ifndef BB_GEN_THREADS
#define BB_GEN_THREADS 256
#endif
constexpr int kGenThreads = BB_GEN_THREADS;
constexpr int kGenWarps = kGenThreads / 32;
constexpr uint64_t kCntBits = 11;
constexpr uint64_t kCntMask = (1ull << kCntBits) - 1;  // B <= 2047 in the packed state


// 1 + #{j in 1..k-1 : thr[j] <= x}  (== assign_bin for monotone s(x))
// bucket path: one 8-byte table read and one compare, (x<<8 | 0xFF) >= bkt[b]
// <=> x >= next (the low byte holds c <= 255)
__device__ __forceinline__ uint32_t bin_bkt(const uint64_t* bkt, uint32_t shift, uint64_t x) {
  const uint64_t e = bkt[x >> shift];
  return (uint32_t)(e & 0xFF) + 1 + (((x << 8) | 0xFF) >= e);
}
__device__ __forceinline__ uint32_t bin_of(const uint64_t* thr, const uint64_t* bkt, bool bkt_ok,
                                           uint32_t shift, uint32_t k, uint32_t top, uint64_t x) {
  if (bkt_ok) return bin_bkt(bkt, shift, x);
  uint32_t pos = 0;
  for (uint32_t step = top; step; step >>= 1)
    if (pos + step < k && thr[pos + step] <= x) pos += step;
  return pos + 1;
}

// predict_bin, binning.hpp:231-261, in key space of the error uniform
template <int ERR>
__device__ __forceinline__ uint32_t predict(const GenPoint& P, uint32_t tb, uint32_t k,
                                            uint64_t xe) {
  if (ERR == 1) {
    if (tb == 1) return xe < P.e_t1 ? 2u : 1u;
    if (tb == k) return xe < P.e_t1 ? k - 1 : k;
    if (xe < P.e_t1) return tb - 1;
    if (xe >= P.e_t2) return tb + 1;
    return tb;
  } else if (ERR == 2) {
    const uint64_t* row = P.conf_thr + (uint64_t)(tb - 1) * k;
    uint32_t pb = 1;
    for (uint32_t j = 0; j + 1 < k; ++j) pb += xe >= row[j];
    return pb;
  }
  return tb;
}

struct Draw {
  uint64_t xg;  // inter-arrival uniform (53-bit)
  uint64_t xs;  // service key
};

template <int SVC>
__device__ __forceinline__ Draw draw(const uint32_t* __restrict__ cyc_rank, uint32_t n_table,
                                     uint32_t i, uint32_t c2, uint32_t c3, uint32_t& cyc) {
  Draw d;
  const uint4 r = philox(i, kStreamArrivalService, c2, c3);
  d.xg = bits53(r.x, r.y);
  if (SVC == kSvcCyclic) {
    d.xs = cyc_rank[cyc];
    if (++cyc == n_table) cyc = 0;
  } else {
    d.xs = bits53(r.z, r.w);
  }
  return d;
}

// Per-replication state of the finite-rate simulation (registers).
struct Rep {
  double t, D, busy, latw, asum;
  uint64_t ncomp;
};

// S servers' free times (multi-server runs only), strided per thread.
struct Servers {
  uint32_t S;
  double* V;
  uint32_t stride;
};

// dispatch, simulator.hpp:256-267: a batch formed at R.t starts when a server
// is free (FIFO: the Kiefer-Wolfowitz recursion; with one server the Lindley
// step D = max(D, R) + S, and D is also the last completion).
// MS selects the S-server code at compile time so that the one-server kernel
// keeps its register budget (128 regs, 16 warps/SM).
template <bool MS, bool LAT = true>
__device__ __forceinline__ double dispatch(Rep& R, const Servers& sv, double S, uint32_t members) {
  double fin;
  if (!MS) {
    fin = R.D = __dadd_rn(fmax(R.D, R.t), S);
  } else {
    double vmin = sv.V[0];
    uint32_t im = 0;
    for (uint32_t q = 1; q < sv.S; ++q) {
      const double v = sv.V[(size_t)q * sv.stride];
      if (v < vmin) {
        vmin = v;
        im = q;
      }
    }
    fin = __dadd_rn(fmax(vmin, R.t), S);
    sv.V[(size_t)im * sv.stride] = fin;
    R.D = fmax(R.D, fin);  // last completion (simulator.hpp:275)
  }
  R.busy += S;
  if (LAT) R.latw += (double)members * fin;  // (quantile mode sums the latencies themselves)
  R.ncomp += members;
  return fin;
}

// Quantile mode (bb_quantile.cuh): the forward pass's request log, this
// lane's view of its warp's interleaved rows (layout in bb_quantile.cuh).
struct QLog {
  double* A;       // arrival of request i at A[qlog_index(i)]
  uint32_t* Id;    // its batch id, same layout
  double* F;       // completion of batch id q at F[q] (this lane's row)
  uint32_t nb;     // batch ids issued
  double* lm;      // shared: [0] a lower bound of the latencies, [32] an upper bound
};

// One request folded into its bin; closes the batch at B members
// (on_arrival + form_batch, simulator.hpp:187-254).  Returns the bin's new
// member count (0: it closed).
// Quantile mode: osum holds the bin's previous closing time, bid its open
// batch's id; *id receives the request's batch id.
template <int SVC, bool track, bool MS, bool Q>
__device__ __forceinline__ uint32_t fold(Rep& R, uint64_t* __restrict__ slot, double* __restrict__ osum,
                                         uint32_t* __restrict__ bid, uint64_t xs, uint32_t B,
                                         const SvcParams& svc, const Servers& sv, QLog& q,
                                         uint32_t& id) {
  const uint64_t s0 = *slot;
  const uint64_t km = max(s0 & ~kCntMask, xs << kCntBits);
  const uint32_t cnt = (uint32_t)(s0 & kCntMask) + 1;
  if (Q) {
    id = cnt == 1 ? q.nb++ : *bid;  // the first member opens a batch
    if (cnt == 1 && cnt != B) *bid = id;
  }
  if (cnt == B) {
    *slot = 0;
    const double fin = dispatch<MS, !Q>(R, sv, svc_of_key_t<SVC>(svc, km >> kCntBits), B);
    if (track) *osum = 0.0;
    if (Q) {
      q.F[(size_t)id * kQFStride] = fin;
      const double lo = __dsub_rn(fin, R.t), hi = __dsub_rn(fin, *osum);
      if (lo < q.lm[0]) q.lm[0] = lo;    // closing member: the batch's smallest latency
      if (hi > q.lm[32]) q.lm[32] = hi;  // bounds the first member's (it arrived later)
      *osum = R.t;
    }
    return 0u;
  }
  *slot = km | cnt;
  if (track) *osum += R.t;
  return cnt;
}

#ifndef BB_QV256
#define BB_QV256 1  // request-log stores as 256-bit vectors (sm_100 STG.E.256)
#endif
#ifndef BB_QWRITE
#define BB_QWRITE 1  // 1: the first selection pass writes the latencies for the later ones
#endif
#ifndef BB_QSTAGE
#define BB_QSTAGE 3  // A/B only: 1 = request log, 2 = + latencies, 3 = + selection
#endif
#ifndef BB_GEN_MINB
#define BB_GEN_MINB 1
#endif
#ifndef BB_GEN_PIPE
#define BB_GEN_PIPE 0  // software-pipeline the next group's draws (A/B: slower, 134 regs)
#endif
#ifndef BB_GEN_UNROLL
#define BB_GEN_UNROLL 4  // requests in flight per thread (even)
#endif
// shared bytes of one warp's state rows, and of its whole region
// (quantile mode, finite rate: the second row set holds each bin's previous
// closing time instead of the open arrival sums, a third (u32) its open
// batch's id)
// (max_batch_wait: finite rate, a row with each bin's front arrival; overload,
// two u32 rows with each bin's first arrival and last round-robin formation)
__host__ __device__ __forceinline__ uint32_t gen_core_bytes(uint32_t kmax, bool ovl, bool track, bool q) {
  if (ovl) return kmax * 768u;
  return q ? kmax * 640u + 512u : kmax * 256u * (track ? 2u : 1u);
}
__host__ __device__ __forceinline__ uint32_t gen_state_bytes(uint32_t kmax, bool ovl, bool track, bool q,
                                                            bool tm = false) {
  return gen_core_bytes(kmax, ovl, track, q) + (tm ? kmax * 256u : 0u);
}
__host__ __device__ __forceinline__ uint32_t gen_warp_bytes(uint32_t kmax, bool ovl, bool track, bool q,
                                                           bool tm = false) {
  const uint32_t st = gen_state_bytes(kmax, ovl, track, q, tm);
  return q ? (st > kQRegionMin ? st : kQRegionMin) + 32u : st;
}

template <int SVC, int ERR, bool OVL, bool TRACK, bool MS, bool Q, bool TM>
__global__ void __launch_bounds__(kGenThreads, Q ? 2 : BB_GEN_MINB) gen_kernel(const __grid_constant__ GenLaunch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t s_thr[kGenWarps][BB_MAX_BINS + 1];
  __shared__ __align__(16) uint64_t s_bkt[kGenWarps][256];
  __shared__ double2 s_logtab[kLogTab];
  init_log_table(s_logtab);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5, tid = threadIdx.x;
  const uint32_t kmax = L.k_max;
  // per-warp shared region: state rows of 32 lanes ([kmax] packed (key<<11 | cnt),
  // then open arrival sums (finite, no flush) or four u32 tables (overload));
  // in quantile mode the same region then holds the selection histogram
  const uint32_t wbytes = gen_warp_bytes(kmax, OVL, TRACK, Q, TM);
  unsigned char* wreg = smem_raw + (size_t)wib * wbytes;
  uint64_t* st = reinterpret_cast<uint64_t*>(wreg);
  double* s_osum = reinterpret_cast<double*>(st + (size_t)kmax * 32);  // finite, no flush
  uint32_t* s_F = reinterpret_cast<uint32_t*>(st + (size_t)kmax * 32);  // overload
  uint32_t* s_rem = s_F + (size_t)kmax * 32;
  uint32_t* s_cf = s_rem + (size_t)kmax * 32;
  uint32_t* s_jd = s_cf + (size_t)kmax * 32;
  uint32_t* s_bid = reinterpret_cast<uint32_t*>(st + (size_t)kmax * 64);  // quantile mode
  // max_batch_wait: finite rate, each bin's front arrival; overload, each
  // bin's first arrival and last round-robin formation
  double* s_front = reinterpret_cast<double*>(wreg + gen_core_bytes(kmax, OVL, TRACK, Q));
  uint32_t* s_fa = reinterpret_cast<uint32_t*>(s_front);
  uint32_t* s_li = s_fa + (size_t)kmax * 32;
  const uint32_t qregion = gen_state_bytes(kmax, OVL, TRACK, Q, TM) > kQRegionMin
                               ? gen_state_bytes(kmax, OVL, TRACK, Q, TM) : kQRegionMin;
  double* q_ans = reinterpret_cast<double*>(wreg + qregion);  // [4]

  const uint32_t nrep = L.rep_end - L.rep_begin;
  const uint32_t chunks = (nrep + 31) / 32;
  const uint64_t n_items = (uint64_t)chunks * L.n_points;
  const uint32_t out_reps = L.out_reps ? L.out_reps : L.reps_total;
  const uint64_t stride = (uint64_t)L.points_total * out_reps;
  const uint64_t gwarp = (uint64_t)blockIdx.x * kGenWarps + wib;
  const uint64_t nwarps = (uint64_t)gridDim.x * kGenWarps;

  for (uint64_t w = gwarp; w < n_items; w += nwarps) {
    const uint32_t p = (uint32_t)(w / chunks), c = (uint32_t)(w % chunks);
    const GenPoint& P = L.pts_dev[p];
    const uint32_t k = P.k, B = P.B, n = P.n;
    for (uint32_t j = lane; j <= k; j += 32) s_thr[wib][j] = P.thr[j];
#pragma unroll
    for (int q = 0; q < 8; ++q) s_bkt[wib][lane + 32 * q] = P.bkt[lane + 32 * q];
    __syncwarp();
    const uint32_t r = L.rep_begin + c * 32 + lane;
    // quantile mode: this lane's request log and what the warp's selection needs
    const size_t qslot = (size_t)blockIdx.x * kGenThreads + tid;
    const size_t qwarp = (size_t)blockIdx.x * kGenWarps + wib;
    QLog q{nullptr, nullptr, nullptr, 0u, nullptr};
    double q_lmin = CUDART_INF, q_lmax = 0.0;  // (overload: bounds of the batch completions)
    bool q_ok = false;
    uint64_t q_m = 0;
    uint32_t q_nb = 0;
    double q_p50 = BB_QNAN, q_p99 = BB_QNAN;
    double thr_out = 0.0, lat_out = 0.0, mk_out = 0.0, busy_out = 0.0;
    const size_t gstride = (size_t)gridDim.x * blockDim.x;
    if (r < L.rep_end) {
      const uint64_t seed = L.single_seed ? L.master : replication_seed(L.master, r);
      const uint64_t sw = splitmix64(seed);  // RandomStream(seed) whitening, rng.hpp:30
      const uint32_t c2 = (uint32_t)sw, c3 = (uint32_t)(sw >> 32);
      // point parameters in registers (the closures read them, not global memory)
      const SvcParams svc = P.svc;
      const uint32_t* __restrict__ cyc_rank = P.cyc_rank;
      const uint64_t* __restrict__ conf_thr = P.conf_thr;
      const uint64_t* thr = s_thr[wib];
      const uint64_t* bkt = s_bkt[wib];
      const bool bkt_ok = P.bkt_ok != 0;
      const uint32_t bshift = P.bkt_shift;
      const uint32_t top = k > 1 ? (1u << (31 - __clz(k - 1))) : 0u;
      const bool check = P.check_domain != 0;
      const uint64_t vlo = P.vlo, vhi = P.vhi, et1 = P.e_t1, et2 = P.e_t2;
      const bool flush = P.flush != 0;
      const uint32_t nt = svc.n_table;
      for (uint32_t b = 0; b < k; ++b) st[b * 32 + lane] = 0;
      uint32_t cyc = 0;
      bool failed = false;

      // bin of a key, then the error model (predict_bin, binning.hpp:231-261)
      // the error model on a true bin (predict_bin, binning.hpp:231-261)
      auto pred_of = [&](uint32_t tb, uint64_t xe) -> uint32_t {
        if (ERR == 1) {
          if (tb == 1) return xe < et1 ? 2u : 1u;
          if (tb == k) return xe < et1 ? k - 1 : k;
          if (xe < et1) return tb - 1;
          if (xe >= et2) return tb + 1;
          return tb;
        } else if (ERR == 2) {
          const uint64_t* row = conf_thr + (uint64_t)(tb - 1) * k;
          uint32_t pb = 1;
          for (uint32_t j = 0; j + 1 < k; ++j) pb += xe >= row[j];
          return pb;
        }
        return tb;
      };
      auto bin_pred = [&](uint64_t xs, uint64_t xe) -> uint32_t {
        return pred_of(bin_of(thr, bkt, bkt_ok, bshift, k, top, xs), xe);
      };
      // the error stream's two uniforms for requests (2m, 2m+1)
      auto err_pair = [&](uint32_t i, uint64_t& e0, uint64_t& e1) {
        if (ERR != 0) {
          const uint4 e = philox(i >> 1, kStreamError, c2, c3);
          e0 = bits53(e.x, e.y);
          e1 = bits53(e.z, e.w);
        }
      };
      auto out_of_support = [&](uint64_t xs) { return check && (xs < vlo || xs > vhi); };

      if (!OVL) {
        // ------------------------------------------------ finite arrival rate
        const double inv_lambda = P.inv_lambda;
        constexpr bool track = TRACK;  // no flush at a finite rate: leftover sums needed
        static_assert(!(TRACK && Q), "quantile mode sums the latencies themselves");
        if (track || Q)  // (Q: previous closing time per bin)
          for (uint32_t b = 0; b < k; ++b) s_osum[b * 32 + lane] = 0.0;
        Rep R{0.0, 0.0, 0.0, 0.0, 0.0, 0};
        if (Q) {
          q.A = L.qA + qwarp * L.q_n * 32 + lane * kQRun;
          q.Id = L.qI + qwarp * L.q_n * 32 + lane * kQRun;
          q.F = kQFStride == 1 ? L.qF + qslot * L.q_nf : L.qF + qwarp * L.q_nf * 32 + lane;
          q.lm = reinterpret_cast<double*>(s_bid + (size_t)kmax * 32) + lane;
          q.lm[0] = CUDART_INF;
          q.lm[32] = 0.0;

        }
        Servers srv{MS && P.n_servers ? P.n_servers : 1u, nullptr, 0};
        if (MS && srv.S > 1) {  // all servers idle at t = 0
          srv.stride = gridDim.x * blockDim.x;
          srv.V = L.srv + (size_t)blockIdx.x * blockDim.x + tid;
          for (uint32_t q = 0; q < srv.S; ++q) srv.V[(size_t)q * srv.stride] = 0.0;
        }
        uint32_t cyc0 = 0;
        const double a0 = __dmul_rn(exp1_tab(draw<SVC>(cyc_rank, nt, 0, c2, c3, cyc0).xg, s_logtab), inv_lambda);
        // max_batch_wait (simulator.hpp:200-201,223-235): a bin's batch also
        // forms when its front request has waited W.  With no arrival ties a
        // bin never holds more than B, so the bin empties at every formation
        // and its timer is the one armed by its front's arrival.  next_due is
        // a lower bound on the earliest pending due time (stale dues of bins
        // that filled up are skipped by the rescan).
        const double W = TM ? P.max_batch_wait : 0.0;
        double next_due = CUDART_INF;
        auto fire_until = [&](double t) {  // on_flush_timer for every due < t, in due order
          while (next_due < t) {
            double best = CUDART_INF;
            uint32_t bb = 0;
            for (uint32_t b = 0; b < k; ++b)
              if (st[b * 32 + lane] & kCntMask) {
                const double due = __dadd_rn(s_front[b * 32 + lane], W);
                if (due < best) {
                  best = due;
                  bb = b;
                }
              }
            next_due = best;
            if (!(best < t)) break;
            const uint64_t s0 = st[bb * 32 + lane];
            const double tn = R.t;
            R.t = best;  // the batch forms (and joins the FIFO) at the timer's time
            const double fin = dispatch<MS, !Q>(R, srv, svc_of_key_t<SVC>(svc, s0 >> kCntBits),
                                                (uint32_t)(s0 & kCntMask));
            R.t = tn;
            st[bb * 32 + lane] = 0;
            if (track) s_osum[bb * 32 + lane] = 0.0;
            if (Q) {
              q.F[(size_t)s_bid[bb * 32 + lane] * kQFStride] = fin;
              const double lo = __dsub_rn(fin, best), hi = __dsub_rn(fin, s_osum[bb * 32 + lane]);
              if (lo < q.lm[0]) q.lm[0] = lo;
              if (hi > q.lm[32]) q.lm[32] = hi;
              s_osum[bb * 32 + lane] = best;
            }
          }
        };
        // U requests per iteration: their draws, exponentials and bins are
        // independent, so the latencies overlap; the folds stay in order
        constexpr int U = BB_GEN_UNROLL;
        static_assert(!Q || (U % 4 == 0 && kQRun % 4 == 0), "the request log packs 4 requests per lane");
        // software pipeline: the next group's Philox blocks (integer pipes)
        // are issued in the same basic block as this group's exponentials
        // (fp64 pipe) so the scheduler interleaves them (cyclic traces keep a
        // running table index and are not pipelined)
        constexpr bool PIPE = BB_GEN_PIPE && SVC != kSvcCyclic;
        uint32_t i = 0;
        Draw d[U];
        uint64_t e[U];
        if (PIPE && U <= n) {
#pragma unroll
          for (int u = 0; u < U; ++u) d[u] = draw<SVC>(cyc_rank, nt, u, c2, c3, cyc);
#pragma unroll
          for (int u = 0; u < U; u += 2) {
            e[u] = e[u + 1] = 0;
            err_pair(u, e[u], e[u + 1]);
          }
        }
        uint4 idh = make_uint4(0u, 0u, 0u, 0u);  // quantile mode: ids held for the next store
        // the bucket lookup is warp-uniform: one copy of the loop per path
        auto main_loop = [&](auto bk) {
          constexpr bool BK = decltype(bk)::value;
          for (; i + U <= n; i += U) {
            double g[U];
            uint32_t pb[U];
            Draw dn[U];
            uint64_t en[U];
            if (!PIPE) {
#pragma unroll
              for (int u = 0; u < U; ++u) d[u] = draw<SVC>(cyc_rank, nt, i + u, c2, c3, cyc);
#pragma unroll
              for (int u = 0; u < U; u += 2) {
                e[u] = e[u + 1] = 0;
                err_pair(i + u, e[u], e[u + 1]);
              }
            } else {
#pragma unroll
              for (int u = 0; u < U; ++u) dn[u] = draw<SVC>(cyc_rank, nt, i + U + u, c2, c3, cyc);
#pragma unroll
              for (int u = 0; u < U; u += 2) {
                en[u] = en[u + 1] = 0;
                err_pair(i + U + u, en[u], en[u + 1]);
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = __dmul_rn(exp1_tab(d[u].xg, s_logtab), inv_lambda);
            bool oos = false;
#pragma unroll
            for (int u = 0; u < U; ++u) oos |= out_of_support(d[u].xs);
            if (oos) {  // first offending request (no dynamic indexing: keeps d[] in registers)
              uint32_t bad = 0;
              uint64_t bx = 0;
#pragma unroll
              for (int u = U - 1; u >= 0; --u)
                if (out_of_support(d[u].xs)) bad = (uint32_t)u, bx = d[u].xs;
              raise_error(L.err, ((uint64_t)P.gidx << 32) | (i + bad), BB_EDOMAIN, svc_of_key_t<SVC>(svc, bx), r);
              failed = true;
              break;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
              pb[u] = pred_of(BK ? bin_bkt(bkt, bshift, d[u].xs)
                                 : bin_of(thr, bkt, false, bshift, k, top, d[u].xs), e[u]);
            uint32_t qid[U];
            double at[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              R.t = __dadd_rn(R.t, g[u]);  // exponential inter-arrival, simulator.hpp:181 (no contraction)
              if (TM) fire_until(R.t);
              if (!Q) R.asum += R.t;
              at[u] = R.t;
              const uint32_t c1 = fold<SVC, TRACK, MS, Q>(
                  R, st + (pb[u] - 1) * 32 + lane, s_osum + (pb[u] - 1) * 32 + lane,
                  s_bid + (pb[u] - 1) * 32 + lane, d[u].xs, B, svc, srv, q, qid[u]);
              if (TM && c1 == 1) {  // the bin's front: arm its timer
                s_front[(pb[u] - 1) * 32 + lane] = R.t;
                const double due = __dadd_rn(R.t, W);
                next_due = due < next_due ? due : next_due;
              }
            }
            if (Q) {  // request log: arrivals and batch ids (full 32 B sectors)
              const size_t o = qlog_index(i);  // (i % 4 == 0: 4 requests stay in one run)
#if BB_QV256
#pragma unroll
              for (int u = 0; u < U; u += 4)  // one 256-bit store (STG.E.256) per four arrivals
                asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(q.A + o + u), "d"(at[u]),
                             "d"(at[u + 1]), "d"(at[u + 2]), "d"(at[u + 3])
                             : "memory");
#else
#pragma unroll
              for (int u = 0; u < U; u += 2)
                *reinterpret_cast<double2*>(q.A + o + u) = make_double2(at[u], at[u + 1]);
#endif
              // ids: a lane's eight consecutive ids are one 32 B sector; store
              // them together (half-sector stores cost several times more)
              static_assert(U == 4 || U % 8 == 0, "ids go out a full 32 B sector at a time");
              if constexpr (U == 4) {  // held for one iteration
                if ((i & 4u) == 0) {
                  idh = make_uint4(qid[0], qid[1], qid[2], qid[3]);
                } else {
#if BB_QV256
                  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(q.Id + o - 4),
                               "r"(idh.x), "r"(idh.y), "r"(idh.z), "r"(idh.w), "r"(qid[0]), "r"(qid[1]),
                               "r"(qid[2]), "r"(qid[3])
                               : "memory");
#else
                  *reinterpret_cast<uint4*>(q.Id + o - 4) = idh;
                  *reinterpret_cast<uint4*>(q.Id + o) = make_uint4(qid[0], qid[1], qid[2], qid[3]);
#endif
                }
              } else {
#pragma unroll
                for (int u = 0; u < U; u += 4)
                  *reinterpret_cast<uint4*>(q.Id + o + u) = make_uint4(qid[u], qid[u + 1], qid[u + 2], qid[u + 3]);
              }
            }
            if (PIPE) {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                d[u] = dn[u];
                e[u] = en[u];
              }
            }
          }
        };
        if (bkt_ok) main_loop(std::true_type{});
        else main_loop(std::false_type{});
        if (Q && U == 4 && (i & 4u)) *reinterpret_cast<uint4*>(q.Id + qlog_index(i - 4)) = idh;
        // tail: fewer than U requests left, one at a time
        for (; !failed && i < n; ++i) {
          const Draw d0 = draw<SVC>(cyc_rank, nt, i, c2, c3, cyc);
          uint64_t e0 = 0, e1 = 0;
          err_pair(i & ~1u, e0, e1);
          if (i & 1u) e0 = e1;
          if (out_of_support(d0.xs)) {
            raise_error(L.err, ((uint64_t)P.gidx << 32) | i, BB_EDOMAIN, svc_of_key_t<SVC>(svc, d0.xs), r);
            failed = true;
          } else {
            const uint32_t p0 = bin_pred(d0.xs, e0);
            R.t = __dadd_rn(R.t, __dmul_rn(exp1_tab(d0.xg, s_logtab), inv_lambda));
            if (TM) fire_until(R.t);
            if (!Q) R.asum += R.t;
            uint32_t id0 = 0;
            const uint32_t c1 = fold<SVC, TRACK, MS, Q>(R, st + (p0 - 1) * 32 + lane, s_osum + (p0 - 1) * 32 + lane,
                                    s_bid + (p0 - 1) * 32 + lane, d0.xs, B, svc, srv, q, id0);
            if (TM && c1 == 1) {
              s_front[(p0 - 1) * 32 + lane] = R.t;
              const double due = __dadd_rn(R.t, W);
              next_due = due < next_due ? due : next_due;
            }
            if (Q) {
              q.A[qlog_index(i)] = R.t;
              q.Id[qlog_index(i)] = id0;
            }
          }
        }
        double leftover = 0.0;
        // without flush the open batches still form when their timers fire
        if (TM && !failed && !flush) fire_until(CUDART_INF);
        // with flush, a timer due exactly at the last arrival was armed before
        // the drains were scheduled (lower seq): it fires first (:203-205)
        if (TM && !failed && flush) fire_until(__longlong_as_double(__double_as_longlong(R.t) + 1));
        if (!failed) {
          for (uint32_t b = 0; b < k; ++b) {
            const uint64_t s0 = st[b * 32 + lane];
            const uint32_t cnt = (uint32_t)(s0 & kCntMask);
            if (!cnt) continue;
            if (flush) {  // on_drain partials at the last arrival, bin order
              const double fin = dispatch<MS, !Q>(R, srv, svc_of_key_t<SVC>(svc, s0 >> kCntBits), cnt);
              if (Q) {
                q.F[(size_t)s_bid[b * 32 + lane] * kQFStride] = fin;
                const double lo = __dsub_rn(fin, R.t), hi = __dsub_rn(fin, s_osum[b * 32 + lane]);
                if (lo < q.lm[0]) q.lm[0] = lo;
                if (hi > q.lm[32]) q.lm[32] = hi;
              }
            } else {
              leftover += s_osum[b * 32 + lane];
              if (Q) q.F[(size_t)s_bid[b * 32 + lane] * kQFStride] = BB_QNAN;  // never completes
            }
          }
        }
        if (!failed && R.ncomp > 0) {  // finish(), simulator.hpp:279-301
          mk_out = R.D - a0;
          thr_out = (double)R.ncomp / mk_out;
          busy_out = R.busy / ((double)srv.S * mk_out);  // simulator.hpp:287-288
          lat_out = (R.latw - (R.asum - leftover)) / (double)R.ncomp;
          q_ok = Q;
          q_m = R.ncomp;
          if (Q) {
            q_lmin = q.lm[0];
            q_lmax = q.lm[32];
          }
        } else {
          mk_out = thr_out = busy_out = lat_out = failed ? BB_QNAN : 0.0;
        }
      } else {
        // ------------------------------------------------------- overload
        for (uint32_t b = 0; b < k; ++b) {
          s_F[b * 32 + lane] = 0;
          s_cf[b * 32 + lane] = 0xFFFFFFFFu;
        }
        uint64_t e0 = 0, e1 = 0;
        for (uint32_t i = 0; i < n; ++i) {  // pass 1: per-bin totals, first closings
          const Draw d = draw<SVC>(cyc_rank, nt, i, c2, c3, cyc);
          if ((i & 1u) == 0) err_pair(i, e0, e1);
          if (out_of_support(d.xs)) {
            raise_error(L.err, ((uint64_t)P.gidx << 32) | i, BB_EDOMAIN, svc_of_key_t<SVC>(svc, d.xs), r);
            failed = true;
            break;
          }
          const uint32_t pb = bin_pred(d.xs, (i & 1u) ? e1 : e0);
          const uint32_t cnt = ++s_F[(pb - 1) * 32 + lane];
          if (cnt == B) s_cf[(pb - 1) * 32 + lane] = i;
          if (TM && cnt == 1) s_fa[(pb - 1) * 32 + lane] = i;  // arms the bin's first timer
        }
        if (!failed) {
          uint32_t Z = 0;
          uint64_t nc = 0;
          for (uint32_t b = 0; b < k; ++b) {
            const uint32_t cnt = s_F[b * 32 + lane];
            const uint32_t F = cnt / B, rem = cnt - F * B;
            s_F[b * 32 + lane] = F;
            s_rem[b * 32 + lane] = rem;
            s_jd[b * 32 + lane] = 0;
            Z += F >= 1;
            nc += (uint64_t)F * B + (flush ? rem : 0);
          }
          // max_batch_wait without flush: the partial batches form when their
          // timers fire at W, after every t = 0 formation (below)
          const bool timers = TM && !flush && P.max_batch_wait > 0.0;
          cyc = 0;
          double busy = 0.0, latw = 0.0;
          // S > 1 servers: pass 2 files each batch (service, members) under its
          // dispatch index, then the Kiefer-Wolfowitz recursion runs in order
          double* ovS = (MS || Q) ? L.ovS + qslot : nullptr;
          uint16_t* ovM = (MS || Q) ? L.ovM + qslot : nullptr;
          const uint64_t nc0 = nc;  // requests in batches formed at t = 0
          for (uint32_t i = 0; i < n; ++i) {  // pass 2: same draws, batch positions
            const Draw d = draw<SVC>(cyc_rank, nt, i, c2, c3, cyc);
            if ((i & 1u) == 0) err_pair(i, e0, e1);
            const uint32_t pb = bin_pred(d.xs, (i & 1u) ? e1 : e0);
            uint64_t* slot = st + (pb - 1) * 32 + lane;
            const uint64_t s0 = *slot;
            const uint64_t km = max(s0 & ~kCntMask, d.xs << kCntBits);
            const uint32_t cnt = (uint32_t)(s0 & kCntMask) + 1;
            if (cnt == B) {
              *slot = 0;
              const uint32_t b = pb - 1;
              const uint32_t j = s_jd[b * 32 + lane]++;
              const uint32_t cfb = s_cf[b * 32 + lane];
              uint64_t before;  // requests dispatched before this batch
              uint32_t idx;     // batches dispatched before this batch
              if (flush && j > 0) {  // drain phase, bins in order (on_drain, :218-221)
                before = (uint64_t)B * Z + (uint64_t)B * (j - 1);
                idx = Z + (j - 1);
                for (uint32_t q = 0; q < b; ++q) {
                  const uint32_t F = s_F[q * 32 + lane];
                  const uint32_t rq = s_rem[q * 32 + lane];
                  before += (uint64_t)B * (F ? F - 1 : 0) + rq;
                  idx += (F ? F - 1 : 0) + (rq != 0);
                }
              } else {  // round j, first-closing order (on_formation, :208-216)
                uint64_t pos = 0;
                for (uint32_t q = 0; q < k; ++q) {
                  const uint32_t F = s_F[q * 32 + lane];
                  const uint32_t cq = s_cf[q * 32 + lane];
                  if (!flush) pos += F < j ? F : j;
                  pos += (cq < cfb) && (F > j);
                }
                before = (uint64_t)B * pos;
                idx = (uint32_t)pos;
              }
              const double S = svc_of_key_t<SVC>(svc, km >> kCntBits);
              if (TM && j + 1 == s_F[b * 32 + lane]) s_li[b * 32 + lane] = idx;  // rearm_timer's seq
              if (MS || Q) {
                ovS[idx * gstride] = S;
                ovM[idx * gstride] = (uint16_t)B;
              }
              if (!MS) {
                busy += S;
                latw += S * (double)(nc0 - before);
              }
            } else {
              *slot = km | cnt;
            }
          }
          uint32_t nbt = 0;  // batches in total
          for (uint32_t b = 0; b < k; ++b) nbt += s_F[b * 32 + lane];
          if (flush) {
            uint64_t base = (uint64_t)B * Z;
            nbt = Z;
            for (uint32_t b = 0; b < k; ++b) {
              const uint32_t F = s_F[b * 32 + lane];
              const uint32_t rem = s_rem[b * 32 + lane];
              base += (uint64_t)B * (F ? F - 1 : 0);
              nbt += F ? F - 1 : 0;
              if (rem) {
                const double S = svc_of_key_t<SVC>(svc, st[b * 32 + lane] >> kCntBits);
                if (MS || Q) {
                  ovS[(size_t)nbt * gstride] = S;
                  ovM[(size_t)nbt * gstride] = (uint16_t)rem;
                }
                if (!MS) {
                  busy += S;
                  latw += S * (double)(nc - base);
                }
                ++nbt;
              }
              base += rem;
            }
          }
          double mk = busy;  // one server: all requests arrive at t=0, the server never idles
          const uint32_t nb0 = nbt;  // batches formed at t = 0
          if (timers) {
            // fire order at W (simulator.hpp:223-235): the timers armed at the
            // bins' first arrivals (bins that never filled a batch), then the
            // ones re-armed by each bin's last round-robin formation
            const double Wt = P.max_batch_wait;
            const uint32_t done_bit = 0x80000000u;
            for (;;) {
              uint32_t bb = 0xFFFFFFFFu;
              uint64_t best = ~0ull;
              for (uint32_t b = 0; b < k; ++b) {
                const uint32_t rem = s_rem[b * 32 + lane];
                if (!rem || (rem & done_bit)) continue;
                const uint32_t F = s_F[b * 32 + lane];
                const uint64_t key = F ? (uint64_t)n + s_li[b * 32 + lane] : s_fa[b * 32 + lane];
                if (key < best) {
                  best = key;
                  bb = b;
                }
              }
              if (bb == 0xFFFFFFFFu) break;
              const uint32_t rem = s_rem[bb * 32 + lane];
              s_rem[bb * 32 + lane] = rem | done_bit;
              const double S = svc_of_key_t<SVC>(svc, st[bb * 32 + lane] >> kCntBits);
              nc += rem;
              if (MS || Q) {
                ovS[(size_t)nbt * gstride] = S;
                ovM[(size_t)nbt * gstride] = (uint16_t)rem;
              }
              if (!MS) {  // one server: D = max(D, W) + S
                mk = __dadd_rn(fmax(mk, Wt), S);
                busy += S;
                latw += (double)rem * mk;
              }
              ++nbt;
            }
            for (uint32_t b = 0; b < k; ++b) s_rem[b * 32 + lane] &= ~done_bit;
          }
          if (MS) {  // S servers: FIFO dispatch over the batches in order (R = 0, or W for timers)
            Rep R{0.0, 0.0, 0.0, 0.0, 0.0, 0};
            Servers srv{P.n_servers ? P.n_servers : 1u, L.srv + (size_t)blockIdx.x * blockDim.x + tid,
                        (uint32_t)gstride};
            for (uint32_t q = 0; q < srv.S; ++q) srv.V[(size_t)q * srv.stride] = 0.0;
            for (uint32_t x = 0; x < nbt; ++x) {
              R.t = x < nb0 ? 0.0 : P.max_batch_wait;
              const double fin = dispatch<true>(R, srv, ovS[(size_t)x * gstride], ovM[(size_t)x * gstride]);
              if (Q) {  // the batch list now holds completions
                ovS[(size_t)x * gstride] = fin;
                q_lmin = fmin(q_lmin, fin);
                q_lmax = fmax(q_lmax, fin);
              }
            }
            busy = R.busy;
            latw = R.latw;
            mk = R.D;
          } else if (Q) {  // one server: completions are the running sum in dispatch order
            // (the makespan and busy sum are the reference's dispatch-order
            // sums, simulator.hpp:261-263, not the closing-order ones above)
            double D = 0.0, bsum = 0.0;
            for (uint32_t x = 0; x < nbt; ++x) {
              const double S = ovS[(size_t)x * gstride];
              D = __dadd_rn(x < nb0 ? D : fmax(D, P.max_batch_wait), S);
              bsum = __dadd_rn(bsum, S);
              ovS[(size_t)x * gstride] = D;
              q_lmin = fmin(q_lmin, D);
              q_lmax = fmax(q_lmax, D);
            }
            mk = D;
            busy = bsum;
          }
          if (nc > 0) {
            mk_out = mk;
            thr_out = (double)nc / mk_out;
            busy_out = busy / ((double)(MS && P.n_servers ? P.n_servers : 1u) * mk_out);
            lat_out = latw / (double)nc;
            q_ok = Q;
            q_m = nc;
            q_nb = nbt;
          } else {
            mk_out = thr_out = busy_out = lat_out = 0.0;
          }
        } else {
          mk_out = thr_out = busy_out = lat_out = BB_QNAN;
        }
      }
      // no completed request: finish() leaves the defaults (0); failed: NaN
      if (!failed && !q_ok) q_p50 = q_p99 = 0.0;
    }
    if (Q && BB_QSTAGE >= 3) {  // the warp selects each of its replications' p50/p99 in turn
      uint32_t pend = __ballot_sync(kQFull, q_ok);
      while (pend) {
        const uint32_t l = __ffs(pend) - 1;
        pend &= pend - 1;
        const uint64_t m = __shfl_sync(kQFull, q_m, l);
        const double lmin = __shfl_sync(kQFull, q_lmin, l), lmax = __shfl_sync(kQFull, q_lmax, l);
        const size_t ls = (size_t)blockIdx.x * kGenThreads + wib * 32 + l;
        double v50, v99;
        if (!OVL) {
          double* A_l = L.qA + qwarp * L.q_n * 32 + l * kQRun;
          const uint32_t* I_l = L.qI + qwarp * L.q_n * 32 + l * kQRun;
          const double* F_l = kQFStride == 1 ? L.qF + ls * L.q_nf : L.qF + qwarp * L.q_nf * 32 + l;
          double sum = 0.0;  // latency_mean from the latencies themselves
          const QSrcLog<false> src{A_l, I_l, F_l, n, lane};
          const QFast qf{L.qK + qwarp * L.q_n * 32 + l * kQRun, A_l, I_l, F_l, n, lane};
          q_select(src, src, m, lmin, lmax, wreg, qregion, q_ans, lane, v50, v99, &sum, &qf);
          if (lane == l) lat_out = sum / (double)m;
        } else {
          const uint32_t nb = __shfl_sync(kQFull, q_nb, l);
          QSrcBatches src{L.ovS + ls, L.ovM + ls, gstride, nb, lane};
          q_select(src, src, m, lmin, lmax, wreg, qregion, q_ans, lane, v50, v99, nullptr);
        }
        if (lane == l) {
          q_p50 = v50;
          q_p99 = v99;
        }
      }
    }
    if (r < L.rep_end) {
      const uint64_t o = (uint64_t)P.gidx * out_reps + (r - L.out_rep0);
      L.out[BB_REP_THROUGHPUT * stride + o] = thr_out;
      L.out[BB_REP_LATENCY * stride + o] = lat_out;
      // without quantile mode p50/p99 are not tracked (NaN)
      L.out[BB_REP_P50 * stride + o] = Q ? q_p50 : BB_QNAN;
      L.out[BB_REP_P99 * stride + o] = Q ? q_p99 : BB_QNAN;
      L.out[BB_REP_MAKESPAN * stride + o] = mk_out;
      L.out[BB_REP_BUSY * stride + o] = busy_out;
    }
    __syncwarp();
  }
}



template <int SVC, int ERR, bool OVL, bool TRACK, bool MS, bool Q, bool TM = false>
cudaError_t launch_gen(const GenLaunch& L, cudaStream_t s) {
  const size_t smem = (size_t)gen_warp_bytes(L.k_max, OVL, TRACK, Q, TM) * kGenWarps;
  auto kern = gen_kernel<SVC, ERR, OVL, TRACK, MS, Q, TM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenThreads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const uint32_t nrep = L.rep_end - L.rep_begin;
  const uint64_t items = (uint64_t)((nrep + 31) / 32) * L.n_points;
  const uint64_t want = (items + kGenWarps - 1) / kGenWarps;
  const uint64_t cap = (uint64_t)sms * occ;
  unsigned grid = (unsigned)(want < cap ? want : cap);
  if (grid == 0) return cudaSuccess;
  GenLaunch L2 = L;
  double* srv = nullptr;
  // per-resident-thread HBM scratch: overload batch lists (S > 1 servers or
  // quantile mode), the finite-rate request log (quantile mode)
  const bool blist = OVL && (MS || Q), rlog = Q && !OVL;
  const uint64_t q_n = rlog ? ((uint64_t)L.n_max + 31) & ~31ull : 0, q_nf = rlog ? L.nf_max : 0;
  const uint64_t per_thread = (blist ? (uint64_t)L.nb_max * (sizeof(double) + sizeof(uint16_t)) : 0) +
                              (rlog ? q_n * 14 + q_nf * sizeof(double) : 0);
  bool held = false;
  if (per_thread) {
    // quantile mode may use most of HBM (a 10^5-request log is 0.9 MB per
    // thread); the S > 1 batch lists alone stay within 4 GiB as before
    const uint64_t budget =
        Q ? gen_scratch_budget((uint64_t)grid * kGenThreads * per_thread + 2048) : ((uint64_t)4 << 30);
    const uint64_t max_grid = budget / (per_thread * kGenThreads);  // (the budget keeps its own reserve)
    if (max_grid == 0) return cudaErrorMemoryAllocation;
    grid = (unsigned)(grid < max_grid ? grid : max_grid);
    const uint64_t slots = (uint64_t)grid * kGenThreads;
    const uint64_t nbl = blist ? slots * L.nb_max : 0;
    const uint64_t bytes = nbl * (sizeof(double) + sizeof(uint16_t)) + slots * (q_n * 14 + q_nf * 8) + 2048;
    unsigned char* base = nullptr;
    e = gen_scratch_acquire(bytes, s, reinterpret_cast<void**>(&base));
    if (e != cudaSuccess) return e;
    held = true;
    // doubles first, then u16, then bytes (alignment)
    size_t off = 0;
    auto carve = [&](size_t b) {
      unsigned char* p = base + off;
      off += (b + 255) & ~(size_t)255;
      return p;
    };
    if (blist) L2.ovS = reinterpret_cast<double*>(carve(nbl * sizeof(double)));
    if (rlog) {
      L2.qA = reinterpret_cast<double*>(carve(slots * q_n * sizeof(double)));
      L2.qF = reinterpret_cast<double*>(carve(slots * q_nf * sizeof(double)));
      L2.qI = reinterpret_cast<uint32_t*>(carve(slots * q_n * sizeof(uint32_t)));
      L2.qK = reinterpret_cast<uint16_t*>(carve(slots * q_n * sizeof(uint16_t)));
    }
    if (blist) L2.ovM = reinterpret_cast<uint16_t*>(carve(nbl * sizeof(uint16_t)));
    L2.q_n = q_n;
    L2.q_nf = q_nf;
  }
  if (L.s_max > 1) {  // free times of S servers per resident thread
    e = cudaMallocAsync((void**)&srv, (size_t)grid * kGenThreads * L.s_max * sizeof(double), s);
    if (e != cudaSuccess) {
      if (held) gen_scratch_release(s);
      return e;
    }
    L2.srv = srv;
  }
  kern<<<grid, kGenThreads, smem, s>>>(L2);
  note_launch();
  e = cudaGetLastError();
  if (srv) cudaFreeAsync(srv, s);
  if (held) gen_scratch_release(s);
  return e;
}

template <int SVC, int ERR, bool Q, bool TM>
cudaError_t launch_mode_qt(const GenLaunch& L, cudaStream_t s) {
  if (L.overload)
    return L.s_max > 1 ? launch_gen<SVC, ERR, true, false, true, Q, TM>(L, s)
                       : launch_gen<SVC, ERR, true, false, false, Q, TM>(L, s);
  // S > 1 servers: leftover sums kept; quantile mode sums the latencies
  // themselves (no open arrival sums)
  if (L.s_max > 1) return launch_gen<SVC, ERR, false, !Q, true, Q, TM>(L, s);
  if constexpr (!Q) {
    if (L.track) return launch_gen<SVC, ERR, false, true, false, Q, TM>(L, s);
  }
  return launch_gen<SVC, ERR, false, false, false, Q, TM>(L, s);
}

template <int SVC, int ERR, bool Q>
cudaError_t launch_mode_q(const GenLaunch& L, cudaStream_t s) {
  return L.timers ? launch_mode_qt<SVC, ERR, Q, true>(L, s) : launch_mode_qt<SVC, ERR, Q, false>(L, s);
}

#include "bb_genw_kernel.cuh"

// Quantile mode with long replications: when the lane kernel's request logs
// (14 B per request per lane) would not fit a full grid in HBM, one warp per
// replication (bb_genw_kernel.cuh) keeps the grid full.  BB_WARP_MODE=0/1
// forces the choice (tests; the results are identical either way).
inline bool use_warp_mode(const GenLaunch& L) {
  if (!L.quant || L.overload || L.s_max > 1 || L.timers || L.k_max > 32) return false;
  static const int env = [] {
    const char* v = getenv("BB_WARP_MODE");
    return v ? (v[0] == '1' ? 1 : 0) : -1;
  }();
  if (env >= 0) return env == 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t per_lane = (((uint64_t)L.n_max + 31) & ~31ull) * 14 + (uint64_t)L.nf_max * 8;
  const uint64_t lanes = (uint64_t)sms * 2 * kGenThreads;  // the lane kernel's full grid
  return per_lane * lanes > gen_scratch_budget(per_lane * lanes);
}

template <int SVC, int ERR>
cudaError_t launch_mode(const GenLaunch& L, cudaStream_t s) {
  if (use_warp_mode(L)) return launch_genw<SVC, ERR>(L, s);
  return L.quant ? launch_mode_q<SVC, ERR, true>(L, s) : launch_mode_q<SVC, ERR, false>(L, s);
}

template <int SVC>
cudaError_t launch_svc(const GenLaunch& L, cudaStream_t s) {
  switch (L.err_kind) {
    case 0: return launch_mode<SVC, 0>(L, s);
    case 1: return launch_mode<SVC, 1>(L, s);
    case 2: return launch_mode<SVC, 2>(L, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// One service family's kernels; explicitly instantiated per family in
// bb_gen_<family>.cu so the instantiations compile in parallel.
template <int SVC>
cudaError_t gen_run_svc(const GenLaunch& L, cudaStream_t s) {
  return launch_svc<SVC>(L, s);
}

}  // namespace bb
