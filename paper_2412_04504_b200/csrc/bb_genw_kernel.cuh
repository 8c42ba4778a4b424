// bb_genw_kernel.cuh -- generated mode with exact quantiles for LONG
// replications: one warp per replication (included by bb_gen_kernel.cuh).
//
// The lane-per-replication kernel keeps a request log of ~14 B per request
// for each of its 32 lanes until the warp selects their quantiles, so with
// 10^6-request replications (BASELINE config 5) HBM capacity, not the SMs,
// bounds how many replications run at once.  Here a warp simulates ONE
// replication, 32 consecutive requests per step (lane = request), so a warp
// logs one replication and the whole grid fits:
//   * draws, gaps, bins and predictions per lane (the same counter-based
//     draws and functions as the lane kernel);
//   * the arrival clock t += gap stays the reference's sequential fp64 sum
//     (simulator.hpp:181): every lane adds the 32 broadcast gaps in request
//     order, so all lanes hold the clock and each keeps its own arrival;
//   * each request's place in its bin (match_any + the bin's carried count),
//     its batch and the batch's id (ids in opening order, as the lane kernel);
//   * batch service = max over the members' keys (a warp max per (bin,
//     batch) group, combined with the carried open maximum);
//   * closings in request order: the one-server Lindley step
//     D = fl(max(D, R) + S) (simulator.hpp:256-267), busy time, completions;
//   * at the end, on_drain's partials in bin order (or never-completing
//     leftovers without flush), then the selection of bb_quantile.cuh over
//     the replication's own contiguous log.
// Every per-replication output equals the lane kernel's bit for bit (same
// values, same operation order; tests/test_gpu_quantiles.py).
// Envelope: finite rate, one server, no max_batch_wait, k <= 32, quantiles on.
// (A fragment of bb_gen_kernel.cuh, included inside its namespace.)

constexpr uint32_t kWRegion = 9216;  // per-warp shared memory: histogram, then candidates
// 2^e as a double from its exponent bits (normal range), without ldexp
__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

// The 32 arrivals of one step, t_i = fl(t_{i-1} + g_i) in request order
// (simulator.hpp:181), exactly, without a 32-long dependent chain.  While
// the clock stays in one binade [2^E, 2^(E+1)) every value is a multiple of
// u = 2^(E-52): t = a u with an integer a, and rounding a u + g to nearest
// even adds q + [f > 1/2] + [f == 1/2 and (a + q) odd] for g / u = q + f --
// an increment that depends on a only through its parity.  Those (even,
// odd) increment pairs compose associatively (the trace path's binade scan,
// bb_trace.cu), so a warp scan gives every lane its exact arrival.  A step
// that may leave the binade (or starts at t = 0) takes the serial chain.
// g >= 0 per lane (0 past the last request); t is warp-uniform and advanced.
__device__ __forceinline__ double warp_clock(double& t, double g, uint32_t lane) {
  const int E = (int)((__double_as_longlong(t) >> 52) & 0x7FF) - 1023;
  if (t > 0.0 && E > -960 && E < 960) {
    const double x = g * pow2i(52 - E);  // exact scaling
    const double qd = floor(x);
    const double f = x - qd;
    const long long q = (long long)qd;
    const bool up = f > 0.5, half = f == 0.5;
    const long long a = (long long)(t * pow2i(52 - E));  // t = a u, a in [2^52, 2^53)
    long long i0 = q + up;
    if (!__any_sync(0xffffffffu, half)) {
      // no exact tie: the increments do not depend on parity -- a plain sum
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long j = __shfl_up_sync(0xffffffffu, i0, o);
        if (lane >= (uint32_t)o) i0 += j;
      }
      const long long end = a + __shfl_sync(0xffffffffu, i0, 31);
      if (end < (1ll << 53)) {  // (monotone: every partial sum stays in the binade)
        const double ti = (double)(a + i0) * pow2i(E - 52);
        t = (double)end * pow2i(E - 52);
        return ti;
      }
    } else {
      long long i1 = i0 + (half & ((q + 1) & 1));
      i0 += half & (q & 1);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // inclusive scan: (earlier) then (mine)
        const long long j0 = __shfl_up_sync(0xffffffffu, i0, o), j1 = __shfl_up_sync(0xffffffffu, i1, o);
        if (lane >= (uint32_t)o) {
          const long long n0 = j0 + ((j0 & 1) ? i1 : i0), n1 = j1 + ((j1 & 1) ? i0 : i1);
          i0 = n0;
          i1 = n1;
        }
      }
      const long long mine = a + ((a & 1) ? i1 : i0);
      const long long end = __shfl_sync(0xffffffffu, mine, 31);
      if (__all_sync(0xffffffffu, x < 0x1.0p52) && end < (1ll << 53)) {
        t = (double)end * pow2i(E - 52);
        return (double)mine * pow2i(E - 52);
      }
    }
  }
  double ti = 0.0;  // the first step (t = 0), a binade crossing: the serial chain
#pragma unroll 8
  for (int l = 0; l < 32; ++l) {
    t = __dadd_rn(t, __shfl_sync(0xffffffffu, g, l));
    if (lane == (uint32_t)l) ti = t;
  }
  return ti;
}

__host__ __device__ __forceinline__ uint32_t genw_warp_bytes() {
  return kWRegion + 64 + 3 * 32 * 4 + 32 * 8 + 2 * 64 * 4 + 32 * 8;
}

template <int SVC, int ERR>
__global__ void __launch_bounds__(kGenThreads, 2) genw_kernel(const __grid_constant__ GenLaunch L) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t s_thr[kGenWarps][BB_MAX_BINS + 1];
  __shared__ __align__(16) uint64_t s_bkt[kGenWarps][256];
  __shared__ double2 s_logtab[kLogTab];
  init_log_table(s_logtab);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  unsigned char* wreg = smem_raw + (size_t)wib * genw_warp_bytes();
  double* q_ans = reinterpret_cast<double*>(wreg + kWRegion);
  uint32_t* s_ncnt = reinterpret_cast<uint32_t*>(wreg + kWRegion + 64);  // per bin: new open count
  uint32_t* s_nid = s_ncnt + 32;                                         //   ... open batch id
  uint32_t* s_seen = s_nid + 32;                                         //   ... seen this step
  uint64_t* s_nkey = reinterpret_cast<uint64_t*>(wreg + kWRegion + 64 + 3 * 32 * 4);  // ... its max key
  uint32_t* s_shi = reinterpret_cast<uint32_t*>(s_nkey + 32);  // [64] batch maxima of a step: high words
  uint32_t* s_slo = s_shi + 64;                                 //   ... low words
  double* s_nprev = reinterpret_cast<double*>(s_slo + 64);      // per bin: its last closing time

  const uint32_t nrep = L.rep_end - L.rep_begin;
  const uint64_t n_items = (uint64_t)nrep * L.n_points;
  const uint32_t out_reps = L.out_reps ? L.out_reps : L.reps_total;
  const uint64_t stride = (uint64_t)L.points_total * out_reps;
  const uint64_t gwarp = (uint64_t)blockIdx.x * kGenWarps + wib;
  const uint64_t nwarps = (uint64_t)gridDim.x * kGenWarps;
  // this warp's log: one replication, contiguous runs of 32 requests
  double* logA = L.qA + gwarp * L.q_n;
  uint32_t* logI = L.qI + gwarp * L.q_n;
  uint16_t* logK = L.qK + gwarp * L.q_n;
  double* logF = L.qF + gwarp * L.q_nf;

  for (uint64_t w = gwarp; w < n_items; w += nwarps) {
    const uint32_t p = (uint32_t)(w / nrep), r = L.rep_begin + (uint32_t)(w % nrep);
    const GenPoint& P = L.pts_dev[p];
    const uint32_t k = P.k, B = P.B, n = P.n;
    __syncwarp();
    for (uint32_t j = lane; j <= k; j += 32) s_thr[wib][j] = P.thr[j];
#pragma unroll
    for (int q = 0; q < 8; ++q) s_bkt[wib][lane + 32 * q] = P.bkt[lane + 32 * q];
    __syncwarp();
    const uint64_t seed = L.single_seed ? L.master : replication_seed(L.master, r);
    const uint64_t sw = splitmix64(seed);
    const uint32_t c2 = (uint32_t)sw, c3 = (uint32_t)(sw >> 32);
    const SvcParams svc = P.svc;
    const uint64_t* thr = s_thr[wib];
    const uint64_t* bkt = s_bkt[wib];
    const bool bkt_ok = P.bkt_ok != 0;
    const uint32_t bshift = P.bkt_shift;
    const uint32_t top = k > 1 ? (1u << (31 - __clz(k - 1))) : 0u;
    const bool check = P.check_domain != 0;
    const uint64_t vlo = P.vlo, vhi = P.vhi, et1 = P.e_t1, et2 = P.e_t2;
    const double inv_lambda = P.inv_lambda;
    const FastDiv divB(B);

    // lane b: bin b+1's open batch (count, max key, id) and previous closing time
    uint32_t cnt = 0, oid = 0;
    uint64_t okey = 0;
    double oprev = 0.0;
    double t = 0.0, D = 0.0, busy = 0.0, a0 = 0.0, lmin = CUDART_INF, lmax = 0.0;
    uint64_t ncomp = 0;
    uint32_t nb = 0;  // batch ids issued
    bool failed = false;
    // Closings wait in a per-warp buffer (the selection's region, free until
    // the end) and are served 32 at a time: every lane computes one batch's
    // service (the log-normal's inverse CDF and exp no longer run with one
    // lane active per step), then the Lindley chain walks them in request
    // order -- the same fp64 steps in the same order.  Nothing in the
    // arrival process depends on the server, so deferring is exact.
    double* c_R = reinterpret_cast<double*>(wreg);   // closing time (= formation)
    double* c_P = c_R + 64;                           // the bin's previous closing time
    uint64_t* c_K = reinterpret_cast<uint64_t*>(c_P + 64);  // the batch's max key
    uint32_t* c_I = reinterpret_cast<uint32_t*>(c_K + 64);  // its id
    uint32_t c_n = 0;
    auto serve_closings = [&]() {
      __syncwarp();
      for (uint32_t b0 = 0; b0 < c_n; b0 += 32) {
        const uint32_t j = b0 + lane, m = c_n - b0 < 32 ? c_n - b0 : 32;
        const bool v = j < c_n;
        const double Rj = v ? c_R[j] : 0.0;
        const double S = v ? svc_of_key_t<SVC>(svc, c_K[j]) : 0.0;
        double fin = 0.0;
        for (uint32_t c = 0; c < m; ++c) {
          const double Sc = __shfl_sync(kQFull, S, c);
          D = __dadd_rn(fmax(D, __shfl_sync(kQFull, Rj, c)), Sc);
          busy += Sc;
          if (lane == c) fin = D;
        }
        if (v) {
          logF[c_I[j]] = fin;
          const double lo = __dsub_rn(fin, Rj), hi = __dsub_rn(fin, c_P[j]);
          lmin = lo < lmin ? lo : lmin;  // the closing member: the batch's smallest latency
          lmax = hi > lmax ? hi : lmax;  // bounds the first member's (it arrived later)
        }
      }
      c_n = 0;
      __syncwarp();
    };
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t i = base + lane;
      const bool valid = i < n;
      uint64_t xg = 0, xs = 0, xe = 0;
      if (valid) {
        const uint4 rr = philox(i, kStreamArrivalService, c2, c3);
        xg = bits53(rr.x, rr.y);
        xs = SVC == kSvcCyclic ? (uint64_t)P.cyc_rank[i % svc.n_table] : bits53(rr.z, rr.w);
        if (ERR != 0) {
          const uint4 e = philox(i >> 1, kStreamError, c2, c3);
          xe = (i & 1u) ? bits53(e.z, e.w) : bits53(e.x, e.y);
        }
      }
      const bool oos = valid && check && (xs < vlo || xs > vhi);
      const uint32_t bad = __ballot_sync(kQFull, oos);
      if (bad) {  // the first offending request (simulator.hpp:189-190, binning.hpp:135-140)
        if (lane == (uint32_t)(__ffs(bad) - 1))
          raise_error(L.err, ((uint64_t)P.gidx << 32) | i, BB_EDOMAIN, svc_of_key_t<SVC>(svc, xs), r);
        failed = true;
        break;
      }
      const double g = valid ? __dmul_rn(exp1_tab(xg, s_logtab), inv_lambda) : 0.0;
      uint32_t pb = 0;
      if (valid) {
        const uint32_t tb = bin_of(thr, bkt, bkt_ok, bshift, k, top, xs);
        pb = predict<ERR>(P, tb, k, xe);
      }
      // the arrival clock: the reference's sequential fp64 sum, exactly
      const double ti = warp_clock(t, g, lane);
      if (base == 0) a0 = __shfl_sync(kQFull, ti, 0);
      // place in the bin: position after the bin's open members
      const uint32_t peers = __match_any_sync(kQFull, pb);
      const uint32_t before = __shfl_sync(kQFull, cnt, pb ? pb - 1 : 0);
      const uint32_t pos = before + __popc(peers & lt);
      const uint32_t jb = divB.div(pos), within = pos - jb * B;
      const bool opening = pb && within == 0, closing = pb && within == B - 1;
      // batch ids in opening (request) order; my batch's opener is the bin's
      // last opener at or before me (none: the batch was open before this step)
      const uint32_t omask = __ballot_sync(kQFull, opening);
      const uint32_t mine = pb ? omask & peers & ((2u << lane) - 1u) : 0u;
      const uint32_t opener = mine ? 31 - __clz(mine) : 32u + (pb ? pb - 1 : 0);
      const uint32_t coid = __shfl_sync(kQFull, oid, pb ? pb - 1 : 0);
      const uint32_t myid = mine ? nb + __popc(omask & ((1u << (opener & 31)) - 1u)) : coid;
      nb += __popc(omask);
      // batch maximum of the members so far: a shared slot per batch of this
      // step (its opener's lane; 32 + bin for the carried open batch), the
      // high words first, then the low words of the members holding the max
      // (the positive IEEE keys order like their values)
      s_shi[lane] = 0u;
      s_slo[lane] = 0u;
      s_shi[32 + lane] = lane < k ? (uint32_t)(okey >> 32) : 0u;
      s_slo[32 + lane] = 0u;
      __syncwarp();
      if (pb) atomicMax(&s_shi[opener], (uint32_t)(xs >> 32));
      __syncwarp();
      if (pb && s_shi[opener] == (uint32_t)(xs >> 32)) atomicMax(&s_slo[opener], (uint32_t)xs);
      if (lane < k && okey && s_shi[32 + lane] == (uint32_t)(okey >> 32))
        atomicMax(&s_slo[32 + lane], (uint32_t)okey);
      __syncwarp();
      const uint64_t bkey = pb ? ((uint64_t)s_shi[opener] << 32) | s_slo[opener] : 0ull;
      if (valid) {
        logA[i] = ti;
        logI[i] = myid;
      }
      // closings: queued in request order (served 32 at a time, above)
      const uint32_t cm = __ballot_sync(kQFull, closing);
      ncomp += (uint64_t)B * __popc(cm);
      // the bin's previous closing: an earlier closing lane of the bin, else carried
      const uint32_t ecl = cm & peers & lt;
      const double prev_e = __shfl_sync(kQFull, ti, ecl ? 31 - __clz(ecl) : lane);
      const double prev_c = __shfl_sync(kQFull, oprev, pb ? pb - 1 : 0);
      if (closing) {
        const uint32_t slot = c_n + __popc(cm & lt);
        c_R[slot] = ti;
        c_P[slot] = ecl ? prev_e : prev_c;
        c_K[slot] = bkey;
        c_I[slot] = myid;
      }
      c_n += __popc(cm);
      if (c_n >= 32) serve_closings();
      // carry each bin's open batch (its last member) and last closing time to the next step
      s_seen[lane] = 0;
      __syncwarp();
      if (pb && (peers >> lane) == 1u) {  // the bin's highest lane this step
        s_ncnt[pb - 1] = closing ? 0u : within + 1;
        s_nid[pb - 1] = myid;
        s_nkey[pb - 1] = closing ? 0ull : bkey;
        atomicOr(&s_seen[pb - 1], 1u);
      }
      if (closing && !(cm & peers & ~lt & ~(1u << lane))) {  // the bin's last closing this step
        s_nprev[pb - 1] = ti;
        atomicOr(&s_seen[pb - 1], 2u);
      }
      __syncwarp();
      if (lane < k && (s_seen[lane] & 2)) oprev = s_nprev[lane];
      if (lane < k && (s_seen[lane] & 1)) {
        cnt = s_ncnt[lane];
        oid = s_nid[lane];
        okey = s_nkey[lane];
      }
      __syncwarp();
    }
    if (!failed) serve_closings();
    double mk_out = 0.0, thr_out = 0.0, busy_out = 0.0, lat_out = 0.0;
    double q_p50 = BB_QNAN, q_p99 = BB_QNAN;
#pragma unroll
    for (int o = 16; o; o >>= 1) {  // the closing lanes' latency bounds
      lmin = fmin(lmin, __shfl_xor_sync(kQFull, lmin, o));
      lmax = fmax(lmax, __shfl_xor_sync(kQFull, lmax, o));
    }
    if (!failed) {
      // after the last arrival: on_drain partials in bin order (simulator.hpp:203-205,218-221),
      // or leftovers that never complete (no flush)
      for (uint32_t b = 0; b < k; ++b) {
        const uint32_t cb = __shfl_sync(kQFull, cnt, b);
        if (!cb) continue;
        const uint32_t idb = __shfl_sync(kQFull, oid, b);
        if (P.flush) {
          const double S = svc_of_key_t<SVC>(svc, __shfl_sync(kQFull, okey, b));
          const double fin = D = __dadd_rn(fmax(D, t), S);  // formed at the last arrival
          busy += S;
          ncomp += cb;
          const double lo = __dsub_rn(fin, t), hi = __dsub_rn(fin, __shfl_sync(kQFull, oprev, b));
          lmin = lo < lmin ? lo : lmin;
          lmax = hi > lmax ? hi : lmax;
          if (lane == 0) logF[idb] = fin;
        } else if (lane == 0) {
          logF[idb] = BB_QNAN;  // never completes
        }
      }
      __syncwarp();
      if (ncomp > 0) {  // finish(), simulator.hpp:279-301
        mk_out = D - a0;
        thr_out = (double)ncomp / mk_out;
        busy_out = busy / mk_out;  // one server (simulator.hpp:287-288)
        double v50, v99, sum = 0.0;
        QSrcLog<false> src{logA, logI, logF, n, lane};
        src.rs = kQRun;
        QFast qf{logK, logA, logI, logF, n, lane};
        qf.rs = kQRun;
        q_select<QSrcLog<false>, QSrcLog<false>, true>(src, src, ncomp, lmin, lmax, wreg, kWRegion, q_ans, lane,
                                                       v50, v99, &sum, &qf);
        lat_out = sum / (double)ncomp;
        q_p50 = v50;
        q_p99 = v99;
      } else {
        q_p50 = q_p99 = 0.0;  // nothing completed: finish() leaves the defaults
      }
    } else {
      mk_out = thr_out = busy_out = lat_out = BB_QNAN;
    }
    if (lane == 0) {
      const uint64_t o = (uint64_t)P.gidx * out_reps + (r - L.out_rep0);
      L.out[BB_REP_THROUGHPUT * stride + o] = thr_out;
      L.out[BB_REP_LATENCY * stride + o] = lat_out;
      L.out[BB_REP_P50 * stride + o] = q_p50;
      L.out[BB_REP_P99 * stride + o] = q_p99;
      L.out[BB_REP_MAKESPAN * stride + o] = mk_out;
      L.out[BB_REP_BUSY * stride + o] = busy_out;
    }
    __syncwarp();
  }
}

// The warp kernel's launch: a persistent grid, one warp-sized log per warp.
template <int SVC, int ERR>
cudaError_t launch_genw(const GenLaunch& L, cudaStream_t s) {
  const size_t smem = (size_t)genw_warp_bytes() * kGenWarps;
  auto kern = genw_kernel<SVC, ERR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGenThreads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const uint64_t items = (uint64_t)(L.rep_end - L.rep_begin) * L.n_points;
  const uint64_t want = (items + kGenWarps - 1) / kGenWarps;
  unsigned grid = (unsigned)std::min<uint64_t>(want, (uint64_t)sms * occ);
  if (grid == 0) return cudaSuccess;
  const uint64_t q_n = ((uint64_t)L.n_max + 31) & ~31ull, q_nf = L.nf_max;
  const uint64_t per_warp = q_n * 14 + q_nf * 8 + 1024;
  const uint64_t max_grid = gen_scratch_budget((uint64_t)grid * per_warp * kGenWarps + 4096) / (per_warp * kGenWarps);
  if (max_grid == 0) return cudaErrorMemoryAllocation;
  grid = (unsigned)std::min<uint64_t>(grid, max_grid);
  const uint64_t warps = (uint64_t)grid * kGenWarps;
  unsigned char* base = nullptr;
  e = gen_scratch_acquire(warps * per_warp + 4096, s, reinterpret_cast<void**>(&base));
  if (e != cudaSuccess) return e;
  size_t off = 0;
  auto carve = [&](size_t b) {
    unsigned char* q = base + off;
    off += (b + 255) & ~(size_t)255;
    return q;
  };
  GenLaunch L2 = L;
  L2.qA = reinterpret_cast<double*>(carve(warps * q_n * sizeof(double)));
  L2.qF = reinterpret_cast<double*>(carve(warps * q_nf * sizeof(double)));
  L2.qI = reinterpret_cast<uint32_t*>(carve(warps * q_n * sizeof(uint32_t)));
  L2.qK = reinterpret_cast<uint16_t*>(carve(warps * q_n * sizeof(uint16_t)));
  L2.q_n = q_n;
  L2.q_nf = q_nf;
  kern<<<grid, kGenThreads, smem, s>>>(L2);
  note_launch();
  e = cudaGetLastError();
  gen_scratch_release(s);
  return e;
}


