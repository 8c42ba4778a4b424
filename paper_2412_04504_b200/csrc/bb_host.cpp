// bb_host.cpp -- the C ABI (include/binbatch_b200.h): validation with the
// reference's exception categories, materialisation of run templates and
// sweeps, request-stream production, and orchestration of the sm_100a
// kernels.  There is no CPU compute path: every simulation result comes from
// the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "binbatch_b200.h"
#include "bb_generated.cuh"
#include "bb_materialize.cuh"
#include "bb_trace.cuh"

namespace bb {
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<unsigned long long> g_h2d{0}, g_d2h{0};
// generated mode: exact per-replication p50/p99 (the reference always computes
// them, simulator.hpp:289-301); off only for A/B measurements
static std::atomic<int> g_gen_quantiles{1};
static thread_local unsigned long long t_launches = 0;
void note_launch(unsigned n) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  t_launches += n;
}
unsigned long long launches_noted_here() { return t_launches; }
}  // namespace bb

namespace {

thread_local std::string g_err;
thread_local cudaEvent_t g_ev[2] = {nullptr, nullptr};
thread_local const char* g_ev_name = "";
thread_local bool g_ev_valid = false;
thread_local double g_trace_ms = -1.0;  // partition kernel of the last trace run

bb_status fail(bb_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

struct CudaFail {
  cudaError_t e;
};
#define CK(x)                                    \
  do {                                           \
    cudaError_t e_ = (x);                        \
    if (e_ != cudaSuccess) throw CudaFail{e_};   \
  } while (0)

struct BBError {
  bb_status st;
  std::string msg;
};
[[noreturn]] void raise(bb_status st, const std::string& m) { throw BBError{st, m}; }

struct DevCtx {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  // stream-ordered shards (bb_*_shard_device) leave their device error flag
  // here; the next reduce on the device reads it (one sync per sweep)
  bb::DevError* pending = nullptr;
  std::vector<std::pair<double, double>> pending_support;  // per point: edges front/back
};
DevCtx g_ctx[64];

// Keep freed blocks cached in the device's stream-ordered pool: the per-call
// buffers (bin edges, uploads) must not be unmapped and mapped again at
// every synchronisation, whichever stream the caller passes.
void keep_pool(int dev) {
  static std::atomic<bool> pool_set[64];
  if (pool_set[dev & 63].exchange(true)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

int current_device(int32_t want) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    raise(BB_ECUDA, "no CUDA device available (the engine has no CPU path)");
  int dev = want;
  if (dev < 0) CK(cudaGetDevice(&dev));
  if (dev >= n) raise(BB_EINVAL, "device ordinal out of range");
  CK(cudaSetDevice(dev));
  keep_pool(dev);
  return dev;
}

cudaStream_t ctx_stream(int dev) {
  DevCtx& c = g_ctx[dev];
  if (!c.stream) {
    CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    keep_pool(dev);
  }
  return c.stream;
}

template <class F>
bb_status guarded(F&& f) {
  try {
    f();
    return BB_OK;
  } catch (const BBError& e) {
    return fail(e.st, e.msg);
  } catch (const CudaFail& e) {
    return fail(BB_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e.e));
  } catch (const std::bad_alloc&) {
    return fail(BB_ERUNTIME, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(BB_ERUNTIME, e.what());
  }
}

// ------------------------------------------------------------ device buffers
struct DBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t bytes, cudaStream_t st) : s(st) { CK(cudaMallocAsync(&p, bytes ? bytes : 8, st)); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      if (p) cudaFreeAsync(p, s);
      p = o.p;
      s = o.s;
      o.p = nullptr;
    }
    return *this;
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <class T>
DBuf upload(const T* h, size_t n, cudaStream_t s) {
  DBuf b(n * sizeof(T), s);
  if (n) CK(cudaMemcpyAsync(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  bb::g_h2d += n * sizeof(T);
  return b;
}
void h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
  bb::g_h2d += bytes;
}
void d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
  bb::g_d2h += bytes;
}

// --------------------------------------------------------- host formulas
// (host-side materialisation: the reference computes edges on the host too)
uint64_t smix(uint64_t x) { return bb::splitmix64(x); }

void check_edges(const double* e, uint64_t n) {  // make_bin_config, binning.hpp:31-44
  if (!e || n < 2) raise(BB_EINVAL, "bin config: need at least two edges");
  for (uint64_t i = 0; i < n; ++i) {
    const bool last = i + 1 == n;
    if (std::isnan(e[i]) || (!last && !std::isfinite(e[i])) ||
        (last && e[i] == -std::numeric_limits<double>::infinity()))
      raise(BB_EINVAL, "bin config: only the top edge may be infinite");
  }
  for (uint64_t i = 1; i < n; ++i)
    if (!(e[i - 1] < e[i])) raise(BB_EINVAL, "bin config: edges must be strictly increasing");
}

std::vector<double> uniform_edges(uint64_t k, double lo, double hi) {  // binning.hpp:47-57
  if (k == 0) raise(BB_EINVAL, "uniform_boundaries: k must be >= 1");
  if (!(lo >= 0) || !(lo < hi)) raise(BB_EINVAL, "uniform_boundaries: need 0 <= min_time < max_time");
  std::vector<double> e(k + 1);
  for (uint64_t i = 0; i <= k; ++i) {
    const volatile double frac = (double)i / (double)k;
    const volatile double span = frac * (hi - lo);
    e[i] = lo + span;
  }
  e[0] = lo;
  e[k] = hi;
  check_edges(e.data(), e.size());
  return e;
}

double harmonic(uint64_t n) {  // service_dist.hpp:141-146
  double sum = 0.0;
  for (uint64_t j = n; j >= 1; --j) sum += 1.0 / (double)j;
  return sum;
}

std::vector<double> exponential_edges(uint64_t k, double rate, uint64_t B) {  // binning.hpp:61-93
  if (k == 0) raise(BB_EINVAL, "exponential_boundaries: k must be >= 1");
  if (!(rate > 0)) raise(BB_EINVAL, "exponential_boundaries: rate must be positive");
  if (B == 0) raise(BB_EINVAL, "l_sequence: batch size must be >= 1");
  std::vector<double> seq;
  if (k > 1) {
    seq.push_back(harmonic(B));
    for (uint64_t m = 2; m < k; ++m) {
      if (!(seq.back() > 0)) raise(BB_EDOMAIN, "l_sequence: non-positive term, log undefined");
      seq.push_back(1.0 + std::log(seq.back()));
    }
  }
  std::vector<double> e{0.0};
  double ls = 0.0;
  for (uint64_t i = 1; i < k; ++i) {
    ls += std::log(seq[k - i - 1]);
    e.push_back(ls / rate);
  }
  e.push_back(std::numeric_limits<double>::infinity());
  check_edges(e.data(), e.size());
  return e;
}

double interp_quantile(const std::vector<double>& sorted, double q) {  // binning.hpp:98-104
  const volatile double pos = q * (double)(sorted.size() - 1);
  const size_t idx = (size_t)pos;
  if (idx + 1 >= sorted.size()) return sorted.back();
  const volatile double frac = pos - (double)idx;
  const volatile double prod = frac * (sorted[idx + 1] - sorted[idx]);
  return sorted[idx] + prod;
}

std::vector<double> empirical_edges(uint64_t k, const double* s, uint64_t n) {  // binning.hpp:110-128
  if (k == 0) raise(BB_EINVAL, "empirical_boundaries: k must be >= 1");
  if (n == 0) raise(BB_EINVAL, "empirical_boundaries: sample set is empty");
  std::vector<double> sorted(s, s + n);
  std::sort(sorted.begin(), sorted.end());
  std::vector<double> distinct(sorted);
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  if (distinct.size() < k)
    raise(BB_EINVAL, "empirical_boundaries: k exceeds the number of distinct sample values");
  std::vector<double> e(k + 1);
  e[0] = sorted.front();
  e[k] = sorted.back();
  for (uint64_t j = 1; j < k; ++j) e[j] = interp_quantile(sorted, (double)j / (double)k);
  for (uint64_t i = 1; i <= k; ++i)
    if (!(e[i - 1] < e[i])) raise(BB_EINVAL, "empirical_boundaries: bins collapse (duplicate quantiles)");
  check_edges(e.data(), e.size());
  return e;
}

// inverse standard normal CDF (Acklam's rational approximation + one Halley
// step on erfc) for the log-normal quantile edges of BASELINE config 5
double norm_ppf(double p) {
  if (p <= 0) return -std::numeric_limits<double>::infinity();
  if (p >= 1) return std::numeric_limits<double>::infinity();
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  double x;
  if (p < 0.02425) {
    const double q = std::sqrt(-2 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else if (p > 1 - 0.02425) {
    const double q = std::sqrt(-2 * std::log(1 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else {
    const double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
  }
  const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
  const double u = e * std::sqrt(2 * M_PI) * std::exp(x * x / 2);
  return x - u / (1 + x * u / 2);
}

std::vector<double> lognormal_edges(uint64_t k, double mu, double sigma) {
  if (k == 0) raise(BB_EINVAL, "lognormal boundaries: k must be >= 1");
  std::vector<double> e(k + 1);
  e[0] = 0.0;
  for (uint64_t j = 1; j < k; ++j) e[j] = std::exp(mu + sigma * norm_ppf((double)j / (double)k));
  e[k] = std::numeric_limits<double>::infinity();
  check_edges(e.data(), e.size());
  return e;
}

// analytics.hpp:55-108
double an_service(uint64_t B, uint64_t k, double lo, double hi) {
  const double mid = (lo + hi) / 2.0;
  const double bb = (double)B;
  const double gap = (bb * hi + lo) / (bb + 1.0) - mid;
  return mid + gap / (double)k;
}
double an_throughput(uint64_t B, uint64_t k, double lo, double hi) {
  return (double)B / an_service(B, k, lo, hi);
}
double an_latency(uint64_t B, uint64_t k, double lo, double hi, double lam) {
  const double wait = (double)(B - 1) * (double)k / (2.0 * lam);
  return an_service(B, k, lo, hi) + wait;
}

// --------------------------------------------------------------- configs
struct SimSpec {  // a validated, materialised SimConfig
  double lambda;
  uint64_t n, B, S, seed;
  bool flush;
  std::vector<double> edges;
  int err_kind;  // effective: symmetric with k==1 || p==0 draws nothing -> still 1 for the stream
  double p;
  std::vector<double> conf;
  int svc;       // bb_service_kind
  double lo, hi, rate, lin_a, lin_b, mu, sigma;
  std::vector<double> table;
  int rng;
  double mbw = 0.0;  // max_batch_wait (0: none)
  uint64_t k() const { return edges.size() - 1; }
  bool error_draws() const {
    return (err_kind == BB_ERR_SYMMETRIC && k() > 1 && p != 0) || err_kind == BB_ERR_CONFUSION;
  }
};

void check_service(int kind, double lo, double hi, double rate, const double* table,
                   uint64_t n_table) {
  switch (kind) {
    case BB_SVC_UNIFORM:  // make_uniform, service_dist.hpp:42-46
      if (!(lo >= 0) || !(lo < hi) || !std::isfinite(hi))
        raise(BB_EINVAL, "uniform service: need 0 <= min_time < max_time");
      break;
    case BB_SVC_EXPONENTIAL:
      if (!(rate > 0) || !std::isfinite(rate))
        raise(BB_EINVAL, "exponential service: rate must be positive");
      break;
    case BB_SVC_EMPIRICAL:
      if (!table || !n_table) raise(BB_EINVAL, "empirical service: sample set is empty");
      for (uint64_t i = 0; i < n_table; ++i)
        if (!(table[i] > 0) || !std::isfinite(table[i]))
          raise(BB_EINVAL, "empirical service: all samples must be positive");
      break;
    case BB_SVC_TRACE_CYCLIC:
    case BB_SVC_TRACE_RESAMPLE:  // replay_trace, simulator.hpp:345-348
      if (!table || !n_table) raise(BB_EINVAL, "replay_trace: empty trace");
      for (uint64_t i = 0; i < n_table; ++i)
        if (!(table[i] > 0) || !std::isfinite(table[i]))
          raise(BB_EINVAL, "replay_trace: trace lengths must be positive");
      break;
    case BB_SVC_LINEAR:
      if (!(lo >= 0) || !(lo < hi) || !std::isfinite(hi))
        raise(BB_EINVAL, "linear service: need 0 <= min_len < max_len");
      break;
    case BB_SVC_LOGNORMAL:
      break;
    default:
      raise(BB_EINVAL, "unknown service kind");
  }
}

SimSpec make_spec(const bb_sim_config* c, bool single = true) {
  if (!c) raise(BB_EINVAL, "null config");
  SimSpec s;
  // simulator.hpp:153-167 (validate) -- bins first, as the reference does
  if (c->n_edges < 2 || !c->edges) raise(BB_EINVAL, "sim config: bins not configured");
  check_edges(c->edges, c->n_edges);
  s.edges.assign(c->edges, c->edges + c->n_edges);
  if (c->n_requests < c->batch_size) raise(BB_EINVAL, "sim config: n_requests must be >= batch_size");
  if (c->batch_size == 0) raise(BB_EINVAL, "sim config: batch size must be >= 1");
  if (c->n_servers == 0) raise(BB_EINVAL, "sim config: need at least one server");
  if (!(c->arrival_rate > 0)) raise(BB_EINVAL, "sim config: arrival rate must be positive (or overload)");
  if (c->has_max_batch_wait && !(c->max_batch_wait > 0))
    raise(BB_EINVAL, "sim config: max_batch_wait must be positive");
  s.mbw = c->has_max_batch_wait ? c->max_batch_wait : 0.0;
  const uint64_t k = c->n_edges - 1;
  s.err_kind = c->error_kind;
  s.p = c->p_error;
  if (c->error_kind == BB_ERR_SYMMETRIC) {  // make_symmetric, binning.hpp:164-168
    if (!(c->p_error >= 0) || !(c->p_error <= 0.5))
      raise(BB_EINVAL, "symmetric error model: need 0 <= p_error <= 0.5");
  } else if (c->error_kind == BB_ERR_CONFUSION) {
    // make_confusion (binning.hpp:170-188) on the matrix as given, then
    // validate()'s size check (simulator.hpp:163-165)
    const uint64_t ck = c->confusion_k;
    if (!c->confusion || ck == 0) raise(BB_EINVAL, "confusion matrix: empty");
    s.conf.assign(c->confusion, c->confusion + ck * ck);
    for (uint64_t i = 0; i < ck; ++i) {
      double sum = 0.0;
      for (uint64_t j = 0; j < ck; ++j) {
        if (!(s.conf[i * ck + j] >= 0)) raise(BB_EINVAL, "confusion matrix: negative entry");
        sum += s.conf[i * ck + j];
      }
      if (std::abs(sum - 1.0) > 1e-9) {
        char buf[128];
        snprintf(buf, sizeof buf, "confusion matrix: row %llu sums to %g, expected 1",
                 (unsigned long long)(i + 1), sum);
        raise(BB_EINVAL, buf);
      }
    }
    if (ck != k) raise(BB_EINVAL, "sim config: confusion matrix size does not match bin count");
  } else if (c->error_kind != BB_ERR_PERFECT) {
    raise(BB_EINVAL, "unknown error model");
  }
  check_service(c->service_kind, c->lo, c->hi, c->rate, c->table, c->n_table);
  s.lambda = c->arrival_rate;
  s.n = c->n_requests;
  s.B = c->batch_size;
  s.S = c->n_servers;
  s.seed = c->seed;
  s.flush = c->flush_partial != 0;
  s.svc = c->service_kind;
  s.lo = c->lo;
  s.hi = c->hi;
  s.rate = c->rate;
  s.lin_a = c->lin_a;
  s.lin_b = c->lin_b;
  s.mu = c->mu;
  s.sigma = c->sigma;
  if (c->table) s.table.assign(c->table, c->table + c->n_table);
  s.rng = c->rng;
  if (!single) return s;
  // the GPU envelope (SURVEY §8f lists these as the next rows)
  if (c->n_servers >= (1ull << 32)) raise(BB_EUNSUPPORTED, "n_servers must be < 2^32");
  if (k > BB_TRACE_MAX_BINS) raise(BB_EUNSUPPORTED, "more than 32 bins is not supported for single runs");
  if (c->n_requests >= (1ull << 32) - 1) raise(BB_EUNSUPPORTED, "n_requests must be < 2^32");
  return s;
}

// ------------------------------------------- request streams (reference RNG)
// RandomStream::derive + draws, rng.hpp:16-53, exactly as the reference
// engine consumes them (simulator.hpp:174-206).
std::mt19937_64 derive(uint64_t master, uint64_t id) {
  return std::mt19937_64(smix(smix(master ^ (0x632BE59BD9B4E019ULL * (id + 1)))));
}
inline double u01(std::mt19937_64& e) { return (double)(e() >> 11) * 0x1.0p-53; }

struct HostStreams {
  std::vector<double> a, s, u;
};

void reference_streams(const SimSpec& c, HostStreams& H) {
  const uint64_t n = c.n;
  H.a.resize(n);
  H.s.resize(n);
  std::thread ta([&] {
    std::mt19937_64 g = derive(c.seed, 0);
    double t = 0.0;
    const bool ovl = std::isinf(c.lambda);
    for (uint64_t i = 0; i < n; ++i) {
      if (ovl) t = 0.0;
      else {
        const volatile double gap = -std::log1p(-u01(g)) / c.lambda;
        t += gap;
      }
      H.a[i] = t;
    }
  });
  std::thread te;
  if (c.error_draws()) {
    H.u.resize(n);
    te = std::thread([&] {
      std::mt19937_64 g = derive(c.seed, 2);
      for (uint64_t i = 0; i < n; ++i) H.u[i] = u01(g);
    });
  }
  {
    std::mt19937_64 g = derive(c.seed, 1);
    std::vector<double> sorted;
    if (c.svc == BB_SVC_EMPIRICAL) {
      sorted = c.table;
      std::sort(sorted.begin(), sorted.end());  // make_empirical sorts
    }
    const uint64_t nt = c.table.size();
    for (uint64_t i = 0; i < n; ++i) {
      double v;
      switch (c.svc) {
        case BB_SVC_UNIFORM: {
          const volatile double span = (c.hi - c.lo) * u01(g);
          v = c.lo + span;
          break;
        }
        case BB_SVC_EXPONENTIAL: v = -std::log1p(-u01(g)) / c.rate; break;
        case BB_SVC_EMPIRICAL: v = sorted[g() % nt]; break;
        case BB_SVC_TRACE_CYCLIC: v = c.table[i % nt]; break;
        case BB_SVC_TRACE_RESAMPLE: v = c.table[g() % nt]; break;
        case BB_SVC_LINEAR: {
          const volatile double span = (c.hi - c.lo) * u01(g);
          const double len = c.lo + span;
          const volatile double prod = c.lin_b * len;
          v = prod + c.lin_a;
          break;
        }
        default: {  // log-normal, Box-Muller on two service draws
          const double u1 = u01(g), u2 = u01(g);
          const double z = std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(6.283185307179586 * u2);
          const volatile double sz = c.sigma * z;
          v = std::exp(c.mu + sz);
        }
      }
      H.s[i] = v;
    }
  }
  ta.join();
  if (te.joinable()) te.join();
}

// -------------------------------------------------- svc params (key space)
struct SvcDev {
  bb::SvcParams p{};
  DBuf table, rank;
};

void svc_params(const SimSpec& c, bb::SvcParams& p) {
  p = bb::SvcParams{};
  p.lo = c.lo;
  p.hi = c.hi;
  p.rate = c.rate;
  p.mu = c.mu;
  p.sigma = c.sigma;
  p.lin_a = c.lin_a;
  p.lin_b = c.lin_b;
  p.key_domain = bb::kKeyDomain53;
  p.n_table = (uint32_t)c.table.size();
  switch (c.svc) {
    case BB_SVC_UNIFORM: p.kind = bb::kSvcUniform; break;
    case BB_SVC_EXPONENTIAL: p.kind = bb::kSvcExponential; break;
    case BB_SVC_LINEAR: p.kind = bb::kSvcLinear; break;
    case BB_SVC_LOGNORMAL: p.kind = bb::kSvcLogNormal; break;
    case BB_SVC_EMPIRICAL:
    case BB_SVC_TRACE_RESAMPLE: p.kind = bb::kSvcTable; break;
    case BB_SVC_TRACE_CYCLIC:
      p.kind = bb::kSvcCyclic;
      p.key_domain = c.table.size();
      break;
  }
}

void make_svc(const SimSpec& c, SvcDev& D, cudaStream_t st) {
  bb::SvcParams& p = D.p;
  p.lo = c.lo;
  p.hi = c.hi;
  p.rate = c.rate;
  p.mu = c.mu;
  p.sigma = c.sigma;
  p.lin_a = c.lin_a;
  p.lin_b = c.lin_b;
  p.key_domain = bb::kKeyDomain53;
  switch (c.svc) {
    case BB_SVC_UNIFORM: p.kind = bb::kSvcUniform; break;
    case BB_SVC_EXPONENTIAL: p.kind = bb::kSvcExponential; break;
    case BB_SVC_LINEAR: p.kind = bb::kSvcLinear; break;
    case BB_SVC_LOGNORMAL: p.kind = bb::kSvcLogNormal; break;
    case BB_SVC_EMPIRICAL:
    case BB_SVC_TRACE_RESAMPLE: {
      std::vector<double> sorted = c.table;
      std::sort(sorted.begin(), sorted.end());
      D.table = upload(sorted.data(), sorted.size(), st);
      p.kind = bb::kSvcTable;
      p.table = D.table.as<double>();
      p.n_table = (uint32_t)sorted.size();
      break;
    }
    case BB_SVC_TRACE_CYCLIC: {
      const size_t nt = c.table.size();
      std::vector<uint32_t> idx(nt);
      for (size_t i = 0; i < nt; ++i) idx[i] = (uint32_t)i;
      std::stable_sort(idx.begin(), idx.end(), [&](uint32_t x, uint32_t y) { return c.table[x] < c.table[y]; });
      std::vector<double> sorted(nt);
      std::vector<uint32_t> rank(nt);
      for (size_t r = 0; r < nt; ++r) {
        sorted[r] = c.table[idx[r]];
        rank[idx[r]] = (uint32_t)r;
      }
      D.table = upload(sorted.data(), nt, st);
      D.rank = upload(rank.data(), nt, st);
      p.kind = bb::kSvcCyclic;
      p.table = D.table.as<double>();
      p.n_table = (uint32_t)nt;
      p.key_domain = nt;
      break;
    }
  }
}

// -------------------------------------------------------- trace pipeline
struct DetailDev {
  DBuf tb, pb, batch, comp, bbin, bsize, bfirst, bformed, bstart, bfinish, bservice, members;
};

void fill_metrics(const bb::TraceResult& R, const SimSpec& c, bb_sim_metrics* m) {
  std::memset(m, 0, sizeof *m);
  m->throughput = R.throughput;
  m->makespan = R.makespan;
  m->latency_mean = R.latency_mean;
  m->latency_p50 = R.p50;
  m->latency_p99 = R.p99;
  m->server_busy_fraction = R.busy_fraction;
  m->n_completed = R.n_completed;
  m->n_batches = R.n_batches;
  m->k = c.k();
  for (uint64_t b = 0; b < c.k() && b < BB_MAX_BINS; ++b) m->per_bin_batch_counts[b] = R.per_bin[b];
  m->busy_time = R.busy;
  m->latency_sum = R.latency_sum;
}

// The bin edges and confusion rows of the last trace run on each device,
// kept resident: repeated runs with the same bins upload nothing (and keep
// one device address, which the pipeline's graph replay relies on less than
// on the arrays').  Callers hold the device's mutex; every trace run
// synchronises before it returns.
struct TraceParams {
  std::vector<double> edges, conf;
  double *d_edges = nullptr, *d_conf = nullptr;
};
TraceParams g_tparams[64];

const double* resident(std::vector<double>& have, double*& dev, const std::vector<double>& want, size_t cap,
                       cudaStream_t st) {
  if (!dev) CK(cudaMalloc((void**)&dev, cap * sizeof(double)));
  if (have != want) {
    have.clear();  // (stale if the copy below throws)
    h2d(dev, want.data(), want.size() * sizeof(double), st);
    have = want;
  }
  return dev;
}

// Runs the trace pipeline on device arrays; fills metrics and (optionally)
// the host detail.  `req_a/req_s` are host copies for the detail output.
void run_pipeline(const SimSpec& c, const double* a_dev, const double* s_dev, const double* u_dev,
                  const uint8_t* pred_dev, bb_sim_metrics* out, bb_sim_detail* det,
                  bool detail_on_device, cudaStream_t st) {
  const uint64_t n = c.n, k = c.k();
  int dev = 0;
  CK(cudaGetDevice(&dev));
  TraceParams& TP = g_tparams[dev & 63];
  const double* edges = resident(TP.edges, TP.d_edges, c.edges, BB_TRACE_MAX_BINS + 1, st);
  const double* conf = c.err_kind == BB_ERR_CONFUSION
                           ? resident(TP.conf, TP.d_conf, c.conf, BB_TRACE_MAX_BINS * BB_TRACE_MAX_BINS, st)
                           : nullptr;
  bb::TraceArgs A{};
  A.n = (uint32_t)n;
  A.B = (uint32_t)c.B;
  A.k = (uint32_t)k;
  A.n_servers = (uint32_t)c.S;
  A.flush = c.flush;
  A.err_kind = pred_dev ? 0 : (c.error_draws() ? c.err_kind : 0);
  A.p_error = c.p;
  A.edges = edges;
  A.conf = conf;
  A.a = a_dev;
  A.s = s_dev;
  A.u_err = u_dev;
  A.pred = pred_dev;
  A.max_batch_wait = c.mbw;
  if (A.err_kind && !u_dev) raise(BB_EINVAL, "trace arrays: the error model needs u_err (or pred_bin)");
  DetailDev D;
  const uint64_t cap = n;
  if (det && !detail_on_device) {
    if (det->req_true_bin) D.tb = DBuf(n, st), A.req_true_bin = D.tb.as<uint8_t>();
    if (det->req_batch) D.batch = DBuf(n * 4, st), A.req_batch = D.batch.as<uint32_t>();
    if (det->req_completion) D.comp = DBuf(n * 8, st), A.req_completion = D.comp.as<double>();
    if (det->bat_bin) D.bbin = DBuf(cap, st), A.bat_bin = D.bbin.as<uint8_t>();
    if (det->bat_size) D.bsize = DBuf(cap * 4, st), A.bat_size = D.bsize.as<uint32_t>();
    if (det->bat_first) D.bfirst = DBuf(cap * 4, st), A.bat_first = D.bfirst.as<uint32_t>();
    if (det->bat_formed) D.bformed = DBuf(cap * 8, st), A.bat_formed = D.bformed.as<double>();
    if (det->bat_start) D.bstart = DBuf(cap * 8, st), A.bat_start = D.bstart.as<double>();
    if (det->bat_finish) D.bfinish = DBuf(cap * 8, st), A.bat_finish = D.bfinish.as<double>();
    if (det->bat_service) D.bservice = DBuf(cap * 8, st), A.bat_service = D.bservice.as<double>();
    if (det->members) D.members = DBuf(n * 4, st), A.members = D.members.as<uint32_t>();
    if (det->req_pred_bin) D.pb = DBuf(n, st), A.req_pred_bin = D.pb.as<uint8_t>();
  } else if (det) {
    A.req_pred_bin = det->req_pred_bin;
    A.req_true_bin = det->req_true_bin;
    A.req_batch = det->req_batch;
    A.req_completion = det->req_completion;
    A.bat_bin = det->bat_bin;
    A.bat_size = det->bat_size;
    A.bat_first = det->bat_first;
    A.bat_formed = det->bat_formed;
    A.bat_start = det->bat_start;
    A.bat_finish = det->bat_finish;
    A.bat_service = det->bat_service;
    A.members = det->members;
  }
  bb::TraceResult R;
  bb::trace_run(A, &R, st);
  if (R.status != BB_OK) raise((bb_status)R.status, R.message);
  fill_metrics(R, c, out);
  g_ev_valid = false;
  g_trace_ms = R.ms_partition;
  g_ev_name = "partition_kernel";
  if (det && !detail_on_device) {
    const uint64_t nb = R.n_batches;
    auto dl = [&](void* h, const DBuf& d, size_t bytes) {
      if (h && d.p && bytes) d2h(h, d.p, bytes, st);
    };
    dl(det->req_true_bin, D.tb, n);
    dl(det->req_pred_bin, D.pb, n);
    dl(det->req_batch, D.batch, n * 4);
    dl(det->req_completion, D.comp, n * 8);
    dl(det->bat_bin, D.bbin, nb);
    dl(det->bat_size, D.bsize, nb * 4);
    dl(det->bat_first, D.bfirst, nb * 4);
    dl(det->bat_formed, D.bformed, nb * 8);
    dl(det->bat_start, D.bstart, nb * 8);
    dl(det->bat_finish, D.bfinish, nb * 8);
    dl(det->bat_service, D.bservice, nb * 8);
    dl(det->members, D.members, n * 4);
    CK(cudaStreamSynchronize(st));
  }
}

void run_single(const bb_sim_config* cfg, const double* lengths, uint64_t n_lengths,
                bb_sim_metrics* out, bb_sim_detail* det) {
  bb_sim_config c2 = *cfg;
  if (lengths) {
    c2.table = lengths;
    c2.n_table = n_lengths;
    if (c2.service_kind != BB_SVC_TRACE_CYCLIC && c2.service_kind != BB_SVC_TRACE_RESAMPLE)
      c2.service_kind = BB_SVC_TRACE_CYCLIC;  // SimConfig.trace_mode default (simulator.hpp:73)
  }
  SimSpec c = make_spec(&c2);
  const int dev = current_device(cfg->device);
  std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
  cudaStream_t st = ctx_stream(dev);
  const uint64_t n = c.n;
  DBuf a(n * 8, st), s(n * 8, st), u;
  HostStreams H;
  if (c.rng == BB_RNG_REFERENCE) {
    reference_streams(c, H);
    h2d(a.p, H.a.data(), n * 8, st);
    h2d(s.p, H.s.data(), n * 8, st);
    if (!H.u.empty()) u = upload(H.u.data(), n, st);
  } else {
    SvcDev sv;
    make_svc(c, sv, st);
    DBuf gap(n * 8, st);
    if (c.error_draws()) u = DBuf(n * 8, st);
    bb::MatArgs M{};
    M.n = (uint32_t)n;
    const uint64_t sw = smix(c.seed);
    M.c2 = (uint32_t)sw;
    M.c3 = (uint32_t)(sw >> 32);
    M.overload = std::isinf(c.lambda);
    M.inv_lambda = M.overload ? 0.0 : 1.0 / c.lambda;
    M.svc = sv.p;
    M.cyc_rank = sv.rank.as<uint32_t>();
    M.gap = gap.as<double>();
    M.s = s.as<double>();
    M.u_err = u.as<double>();
    CK(bb::materialize_streams(M, a.as<double>(), st));
  }
  run_pipeline(c, a.as<double>(), s.as<double>(), u.as<double>(), nullptr, out, det, false, st);
  if (det) {
    if (det->req_arrival) {
      if (!H.a.empty()) std::memcpy(det->req_arrival, H.a.data(), n * 8);
      else CK(cudaMemcpyAsync(det->req_arrival, a.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    if (det->req_service) {
      if (!H.s.empty()) std::memcpy(det->req_service, H.s.data(), n * 8);
      else CK(cudaMemcpyAsync(det->req_service, s.p, n * 8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
  }
}

// ------------------------------------------------------------ sweeps
struct Point {
  bb_run_template t;             // after overrides (pointers into the spec)
  std::vector<double> edges;
  SimSpec spec;                  // materialised (materialize, experiment.hpp:110-155)
};

SimSpec materialize(const bb_run_template& t, uint64_t seed) {
  bb_sim_config c{};
  c.arrival_rate = t.arrival_rate;
  c.n_requests = t.n_requests;
  c.batch_size = t.batch_size;
  c.n_servers = t.n_servers;
  c.seed = seed;
  c.flush_partial = t.flush_partial;
  c.has_max_batch_wait = t.has_max_batch_wait;
  c.max_batch_wait = t.max_batch_wait;
  c.error_kind = t.error_kind;
  c.p_error = t.p_error;
  c.confusion = t.confusion;
  c.confusion_k = t.confusion_k;
  std::vector<double> edges;
  switch (t.service) {
    case BB_KIND_UNIFORM:
      check_service(BB_SVC_UNIFORM, t.min_time, t.max_time, 0, nullptr, 0);
      c.service_kind = BB_SVC_UNIFORM;
      c.lo = t.min_time;
      c.hi = t.max_time;
      if (!t.edges) edges = uniform_edges(t.k, t.min_time, t.max_time);
      break;
    case BB_KIND_EXPONENTIAL:
      check_service(BB_SVC_EXPONENTIAL, 0, 0, t.rate, nullptr, 0);
      c.service_kind = BB_SVC_EXPONENTIAL;
      c.rate = t.rate;
      if (!t.edges) edges = exponential_edges(t.k, t.rate, t.batch_size);
      break;
    case BB_KIND_TRACE:
      check_service(BB_SVC_EMPIRICAL, 0, 0, 0, t.trace_times, t.n_trace);
      c.service_kind = t.trace_cyclic ? BB_SVC_TRACE_CYCLIC : BB_SVC_TRACE_RESAMPLE;
      c.table = t.trace_times;
      c.n_table = t.n_trace;
      if (!t.edges) edges = empirical_edges(t.k, t.trace_times, t.n_trace);
      break;
    case BB_KIND_LINEAR: {
      check_service(BB_SVC_LINEAR, t.min_time, t.max_time, 0, nullptr, 0);
      c.service_kind = BB_SVC_LINEAR;
      c.lo = t.min_time;
      c.hi = t.max_time;
      c.lin_a = t.lin_a;
      c.lin_b = t.lin_b;
      const double tlo = t.lin_b * t.min_time + t.lin_a, thi = t.lin_b * t.max_time + t.lin_a;
      if (!t.edges) edges = uniform_edges(t.k, tlo, thi);
      break;
    }
    case BB_KIND_LOGNORMAL:
      c.service_kind = BB_SVC_LOGNORMAL;
      c.mu = t.mu;
      c.sigma = t.sigma;
      if (!t.edges) edges = lognormal_edges(t.k, t.mu, t.sigma);
      break;
    default:
      raise(BB_EINVAL, "service type must be uniform, exponential or trace");
  }
  if (t.edges) {
    check_edges(t.edges, t.n_edges);
    edges.assign(t.edges, t.edges + t.n_edges);
  }
  c.edges = edges.data();
  c.n_edges = edges.size();
  c.rng = BB_RNG_PHILOX;
  SimSpec s = make_spec(&c, false);
  s.S = t.n_servers;
  return s;
}

uint64_t as_count(double v, const char* param) {  // experiment.hpp:202-206
  if (!(v >= 1) || v != std::floor(v) || !std::isfinite(v))
    raise(BB_EINVAL, std::string("sweep axis ") + param + ": values must be integers >= 1");
  return (uint64_t)v;
}

void apply_override(bb_run_template& t, int param, double v) {  // experiment.hpp:208-228
  switch (param) {
    case BB_AXIS_LAMBDA:
      if (!(v > 0)) raise(BB_EINVAL, "sweep axis lambda: values must be positive");
      t.arrival_rate = v;
      break;
    case BB_AXIS_K:
      if (t.edges) raise(BB_EINVAL, "cannot sweep k when explicit bin edges are given");
      t.k = as_count(v, "k");
      break;
    case BB_AXIS_B: t.batch_size = as_count(v, "B"); break;
    case BB_AXIS_N_SERVERS: t.n_servers = as_count(v, "n_servers"); break;
    case BB_AXIS_P_E:
      if (t.error_kind == BB_ERR_CONFUSION)
        raise(BB_EINVAL, "cannot sweep p_e over a confusion-matrix error model");
      t.error_kind = BB_ERR_SYMMETRIC;
      t.p_error = v;
      break;
    default: raise(BB_EINVAL, "unknown sweep parameter");
  }
}

std::vector<bb_run_template> expand(const bb_experiment_spec* spec) {
  if (!spec) raise(BB_EINVAL, "null experiment spec");
  if (spec->n_axes > 2) raise(BB_EINVAL, "experiment spec: at most 2 sweep axes");
  if (spec->replications < 1) raise(BB_EINVAL, "experiment spec: replications must be >= 1");
  std::vector<std::vector<double>> grid;
  for (uint64_t a = 0; a < spec->n_axes; ++a) {
    const bb_sweep_axis& ax = spec->axes[a];
    if (!ax.n_values || !ax.values) raise(BB_EINVAL, "experiment spec: sweep axis has no values");
    bb_run_template probe = spec->base;
    for (uint64_t i = 0; i < ax.n_values; ++i) apply_override(probe, ax.param, ax.values[i]);
    std::vector<double> v(ax.values, ax.values + ax.n_values);
    std::sort(v.begin(), v.end());
    grid.push_back(v);
  }
  std::vector<bb_run_template> pts;
  if (grid.empty()) pts.push_back(spec->base);
  else if (grid.size() == 1) {
    for (double v : grid[0]) {
      bb_run_template t = spec->base;
      apply_override(t, spec->axes[0].param, v);
      pts.push_back(t);
    }
  } else {
    for (double v0 : grid[0])
      for (double v1 : grid[1]) {
        bb_run_template t = spec->base;
        apply_override(t, spec->axes[0].param, v0);
        apply_override(t, spec->axes[1].param, v1);
        pts.push_back(t);
      }
  }
  return pts;
}

// run_experiment's failure wrapper (experiment.hpp:352-358): a point's error
// comes back as runtime_error "experiment '<name>': sweep point <i> failed: <what>".
struct PointFail {
  const char* name = nullptr;  // null: run_point semantics (no wrapping)
  [[noreturn]] void raise_at(size_t i, bb_status st, const std::string& what) const {
    if (!name) raise(st, what);
    raise(BB_ERUNTIME, std::string("experiment '") + name + "': sweep point " + std::to_string(i) +
                           " failed: " + what);
  }
};

// Build device GenPoints for a set of templates; group launches by template
// instantiation (error kind, cyclic, overload).
struct Sweep {
  std::vector<bb_run_template> tpl;
  std::vector<SimSpec> spec;
  std::vector<bb::GenPoint> gp;
  DBuf d_pts, d_edges, d_conf, d_table, d_rank;
};

struct SweepParams {
  uint64_t seed, replications;
};

// `generated`: the points run in the fused Philox kernel (its envelope is
// checked); reference-stream points run the trace pipeline per replication.
void build_sweep(std::vector<bb_run_template> tpl, Sweep& W, cudaStream_t st, bool generated = true,
                 const PointFail& pf = PointFail{}) {
  if (tpl.empty()) raise(BB_EINVAL, "sweep has no points");
  W.tpl = std::move(tpl);
  const size_t P = W.tpl.size();
  W.spec.reserve(P);
  for (size_t i = 0; i < P; ++i) {
    const bb_run_template& t = W.tpl[i];
    try {
      W.spec.push_back(materialize(t, 0));
    } catch (const BBError& e) {
      pf.raise_at(i, e.st, e.msg);
    }
    const SimSpec& s = W.spec.back();
    if (t.has_max_batch_wait && !(t.max_batch_wait > 0))  // simulator.hpp:160-161
      pf.raise_at(i, BB_EINVAL, "sim config: max_batch_wait must be positive");
    if (!generated) continue;
    if (s.S > 4096) raise(BB_EUNSUPPORTED, "more than 4096 servers is not supported");
    if (s.k() > BB_MAX_BINS) raise(BB_EUNSUPPORTED, "more than 64 bins is not supported");
    if (s.B > 2047) raise(BB_EUNSUPPORTED, "batch sizes above 2047 are not supported by the fused kernel");
    if (s.n >= (1ull << 32) - 1) raise(BB_EUNSUPPORTED, "n_requests must be < 2^32");
  }
  // edges and confusion thresholds, concatenated
  std::vector<double> edges;
  std::vector<uint64_t> eoff(P), coff(P);
  std::vector<uint64_t> conf;
  for (size_t i = 0; i < P; ++i) {
    eoff[i] = edges.size();
    edges.insert(edges.end(), W.spec[i].edges.begin(), W.spec[i].edges.end());
    coff[i] = conf.size();
    if (W.spec[i].err_kind == BB_ERR_CONFUSION) {
      const uint64_t k = W.spec[i].k();
      for (uint64_t r = 0; r < k; ++r) {
        double cum = 0.0;
        for (uint64_t j = 0; j < k; ++j) {
          cum += W.spec[i].conf[r * k + j];
          const double sc = cum * 0x1.0p53;  // u < cum <=> x < ceil(cum * 2^53)
          conf.push_back(sc >= 0x1.0p63 ? (1ull << 63) : (uint64_t)std::ceil(sc));
        }
      }
    }
  }
  W.d_edges = upload(edges.data(), edges.size(), st);
  W.d_conf = upload(conf.data(), conf.size(), st);
  // shared service table (the template's trace, identical for all points)
  SvcDev sv;
  make_svc(W.spec[0], sv, st);
  W.d_table = std::move(sv.table);
  W.d_rank = std::move(sv.rank);
  W.gp.resize(P);
  for (size_t i = 0; i < P; ++i) {
    const SimSpec& s = W.spec[i];
    bb::GenPoint g{};
    svc_params(s, g.svc);
    g.svc.table = W.d_table.as<double>();
    g.cyc_rank = W.d_rank.as<uint32_t>();
    g.inv_lambda = std::isinf(s.lambda) ? 0.0 : 1.0 / s.lambda;
    g.n = (uint32_t)s.n;
    g.B = (uint32_t)s.B;
    g.k = (uint32_t)s.k();
    g.flush = s.flush;
    g.err_kind = s.error_draws() ? (uint32_t)s.err_kind : 0u;
    g.gidx = (uint32_t)i;
    g.n_servers = (uint32_t)s.S;
    g.max_batch_wait = W.tpl[i].has_max_batch_wait ? W.tpl[i].max_batch_wait : 0.0;
    if (g.err_kind == 1) {
      g.e_t1 = (uint64_t)std::ceil(s.p * 0x1.0p53);
      g.e_t2 = (uint64_t)std::ceil((1.0 - s.p) * 0x1.0p53);
    }
    g.edges = W.d_edges.as<double>() + eoff[i];
    g.conf_thr = W.d_conf.as<uint64_t>() + coff[i];
    W.gp[i] = g;
  }
  W.d_pts = upload(W.gp.data(), P, st);
  CK(bb::gen_setup_thresholds(W.d_pts.as<bb::GenPoint>(), (uint32_t)P, st));
}

// the message of a device-side error of sweep point `pt` (support = its edges)
void raise_sweep_error(const bb::DevError& he, const std::pair<double, double>& support,
                       const PointFail& pf) {
  const size_t pt = (size_t)(he.packed >> 40);
  char buf[256];
  if (he.value > 0 && std::isfinite(he.value))  // binning.hpp:135-140
    snprintf(buf, sizeof buf, "assign_bin: length %g outside bin support [%g, %g]", he.value,
             support.first, support.second);
  else  // simulator.hpp:189-190
    snprintf(buf, sizeof buf, "simulation: drew a non-positive service time");
  pf.raise_at(pt, (bb_status)(he.packed & 0xFF), buf);
}

// out_reps/out_rep0: the output rows hold replications [out_rep0, out_rep0 +
// out_reps) (a shard's own slice; 0: the full [0, replications) rows).
// deferred: the device error flag to use, left unchecked (stream order kept).
void launch_sweep(const SweepParams* E, Sweep& W, uint64_t rep_begin, uint64_t rep_end,
                  double* rep_dev, cudaStream_t st, bool time_it, const PointFail& pf = PointFail{},
                  uint32_t out_reps = 0, uint32_t out_rep0 = 0, bb::DevError* deferred = nullptr) {
  const size_t P = W.tpl.size();
  // group points by kernel instantiation; each group's points are copied
  // (already threshold-resolved) into a contiguous device array
  struct Key {
    int err, cyc, ovl, track, ms, tm;
  };
  std::vector<Key> keys(P);
  for (size_t i = 0; i < P; ++i)
    keys[i] = Key{(int)W.gp[i].err_kind, (int)W.gp[i].svc.kind, W.gp[i].inv_lambda == 0.0,
                  W.gp[i].inv_lambda != 0.0 && !W.gp[i].flush, W.gp[i].n_servers > 1,
                  W.gp[i].max_batch_wait > 0.0};
  std::vector<bool> done(P, false);
  bool first = true;
  for (size_t i = 0; i < P; ++i) {
    if (done[i]) continue;
    std::vector<uint32_t> members;
    uint32_t kmax = 1, smax = 1, nmax = 1, nfmax = 1;
    uint64_t nbmax = 1;
    for (size_t j = i; j < P; ++j)
      if (!done[j] && keys[j].err == keys[i].err && keys[j].cyc == keys[i].cyc &&
          keys[j].ovl == keys[i].ovl && keys[j].track == keys[i].track &&
          keys[j].ms == keys[i].ms && keys[j].tm == keys[i].tm) {
        members.push_back((uint32_t)j);
        done[j] = true;
        kmax = std::max(kmax, W.gp[j].k);
        smax = std::max(smax, W.gp[j].n_servers);
        nbmax = std::max<uint64_t>(nbmax, W.gp[j].n / W.gp[j].B + W.gp[j].k + 1);
        nmax = std::max(nmax, W.gp[j].n);
        // batch ids per replication: n/B full + k partials, or up to n with timers
        nfmax = std::max(nfmax, W.gp[j].max_batch_wait > 0.0 ? W.gp[j].n + 1
                                                             : W.gp[j].n / W.gp[j].B + W.gp[j].k + 1);
      }
    const bb::GenPoint* base = W.d_pts.as<bb::GenPoint>();
    DBuf grp;
    const bb::GenPoint* ptr = base + members[0];
    bool contiguous = true;
    for (size_t q = 0; q < members.size(); ++q) contiguous &= members[q] == members[0] + q;
    if (!contiguous) {
      grp = DBuf(members.size() * sizeof(bb::GenPoint), st);
      for (size_t q = 0; q < members.size(); ++q)
        CK(cudaMemcpyAsync(grp.as<bb::GenPoint>() + q, base + members[q], sizeof(bb::GenPoint),
                           cudaMemcpyDeviceToDevice, st));
      ptr = grp.as<bb::GenPoint>();
    }
    bb::GenLaunch L{};
    L.pts_dev = ptr;
    L.n_points = (uint32_t)members.size();
    L.points_total = (uint32_t)P;
    L.k_max = kmax;
    L.s_max = smax;
    L.nb_max = (uint32_t)nbmax;
    L.master = E->seed;
    L.single_seed = 0;
    L.reps_total = (uint32_t)E->replications;
    L.rep_begin = (uint32_t)rep_begin;
    L.rep_end = (uint32_t)rep_end;
    L.err_kind = keys[i].err;
    L.cyclic = keys[i].cyc == bb::kSvcCyclic;
    L.svc_kind = keys[i].cyc;
    L.track = keys[i].track;
    L.overload = keys[i].ovl;
    L.out = rep_dev;
    L.out_reps = out_reps;
    L.out_rep0 = out_rep0;
    L.quant = bb::g_gen_quantiles.load() ? 1 : 0;
    L.timers = keys[i].tm;
    L.n_max = nmax;
    L.nf_max = nfmax;
    DBuf err;
    if (deferred) {
      L.err = deferred;
    } else {
      err = DBuf(sizeof(bb::DevError), st);
      CK(cudaMemsetAsync(err.p, 0xFF, 8, st));
      L.err = err.as<bb::DevError>();
    }
    if (time_it && first) {
      if (!g_ev[0]) {
        CK(cudaEventCreate(&g_ev[0]));
        CK(cudaEventCreate(&g_ev[1]));
      }
      CK(cudaEventRecord(g_ev[0], st));
    }
    const cudaError_t ge = bb::gen_run(L, st);
    if (ge == cudaErrorMemoryAllocation && L.quant) {
      cudaGetLastError();
      char buf[256];
      snprintf(buf, sizeof buf,
               "generated-mode quantiles keep a %u-request log per replication in flight "
               "(about 14 B per request): not even one block fits in free HBM; "
               "bb_set_generated_quantiles(0) runs without p50/p99", nmax);
      raise(BB_EUNSUPPORTED, buf);
    }
    CK(ge);
    if (time_it && first) {
      CK(cudaEventRecord(g_ev[1], st));
      g_ev_name = "gen_kernel";
      g_ev_valid = true;
      g_trace_ms = -1.0;
    }
    first = false;
    if (deferred) continue;
    bb::DevError he;
    d2h(&he, err.p, sizeof he, st);
    CK(cudaStreamSynchronize(st));
    if (he.packed != ~0ull) {  // packed = (point << 40 | request << 8 | code)
      const size_t pt = (size_t)(he.packed >> 40);
      const SimSpec& s = W.spec[pt < W.spec.size() ? pt : 0];
      raise_sweep_error(he, {s.edges.front(), s.edges.back()}, pf);
    }
  }
}

void fill_points(const SweepParams* E, const Sweep& W, const std::vector<double>& stats,
                 bb_point_result* out) {
  for (size_t i = 0; i < W.tpl.size(); ++i) {
    const bb_run_template& t = W.tpl[i];
    const SimSpec& s = W.spec[i];
    bb_point_result& r = out[i];
    std::memset(&r, 0, sizeof r);
    r.arrival_rate = t.arrival_rate;
    r.k = t.edges ? t.n_edges - 1 : t.k;
    r.batch_size = t.batch_size;
    r.n_servers = t.n_servers;
    r.error_kind = t.error_kind;
    r.p_error = t.error_kind == BB_ERR_SYMMETRIC ? t.p_error : 0.0;
    r.n_requests = t.n_requests;
    r.replications = E->replications;
    const double* st = &stats[i * 8];
    r.throughput_mean = st[0];
    r.throughput_std = st[1];
    r.latency_mean = st[2];
    r.latency_std = st[3];
    r.latency_p50 = st[4];
    r.latency_p99 = st[5];
    r.makespan_mean = st[6];
    r.busy_fraction_mean = st[7];
    // analytic columns, experiment.hpp:283-305
    const double nan = std::numeric_limits<double>::quiet_NaN();
    r.analytic_throughput = r.analytic_latency = r.analytic_max_throughput = nan;
    const double servers = (double)t.n_servers;
    double lo = nan, hi = nan;
    if (t.service == BB_KIND_UNIFORM) lo = t.min_time, hi = t.max_time;
    if (t.service == BB_KIND_LINEAR)  // uniform in time on [b*lo+a, b*hi+a]
      lo = t.lin_b * t.min_time + t.lin_a, hi = t.lin_b * t.max_time + t.lin_a;
    if (!std::isnan(lo) && !t.edges) {
      r.analytic_max_throughput = servers * ((double)t.batch_size / ((lo + hi) / 2.0));
      if (std::isinf(t.arrival_rate))
        r.analytic_throughput = servers * an_throughput(t.batch_size, r.k, lo, hi);
      else
        r.analytic_latency = an_latency(t.batch_size, r.k, lo, hi, t.arrival_rate);
    } else if (t.service == BB_KIND_EXPONENTIAL) {
      r.analytic_max_throughput = servers * (double)t.batch_size * t.rate;
    } else if (t.service == BB_KIND_TRACE && t.n_trace) {
      double sum = 0;
      for (uint64_t q = 0; q < t.n_trace; ++q) sum += t.trace_times[q];
      r.analytic_max_throughput = servers * (double)t.batch_size * (double)t.n_trace / sum;
    }
    (void)s;
  }
}

// Bit-exact replication loop (reference streams, trace pipeline per replica).
void reference_point_reps(const SweepParams* E, const Sweep& W, std::vector<double>& rep,
                          cudaStream_t st, const PointFail& pf = PointFail{}) {
  const size_t P = W.tpl.size();
  const uint64_t R = E->replications;
  rep.assign(BB_REP_FIELDS * P * R, 0.0);
  for (size_t i = 0; i < P; ++i) {
    SimSpec s = W.spec[i];
    if (s.S >= (1ull << 32)) raise(BB_EUNSUPPORTED, "n_servers must be < 2^32");
    if (s.k() > BB_TRACE_MAX_BINS) raise(BB_EUNSUPPORTED, "more than 32 bins in reference-stream mode");
    for (uint64_t r = 0; r < R; ++r) {
      s.seed = bb::replication_seed(E->seed, r);
      HostStreams H;
      reference_streams(s, H);
      DBuf a = upload(H.a.data(), s.n, st), sv = upload(H.s.data(), s.n, st), u;
      if (!H.u.empty()) u = upload(H.u.data(), s.n, st);
      bb_sim_metrics m;
      try {
        run_pipeline(s, a.as<double>(), sv.as<double>(), u.as<double>(), nullptr, &m, nullptr,
                     false, st);
      } catch (const BBError& e) {
        if (e.st == BB_EUNSUPPORTED) throw;
        pf.raise_at(i, e.st, e.msg);
      }
      const uint64_t o = i * R + r, stride = P * R;
      rep[BB_REP_THROUGHPUT * stride + o] = m.throughput;
      rep[BB_REP_LATENCY * stride + o] = m.latency_mean;
      rep[BB_REP_P50 * stride + o] = m.latency_p50;
      rep[BB_REP_P99 * stride + o] = m.latency_p99;
      rep[BB_REP_MAKESPAN * stride + o] = m.makespan;
      rep[BB_REP_BUSY * stride + o] = m.server_busy_fraction;
    }
  }
}

// Devices a sweep spreads over (bb_set_devices); empty: the current device.
std::mutex g_dev_mu;
std::vector<int> g_devices;

std::vector<int> sweep_devices() {
  std::lock_guard<std::mutex> lock(g_dev_mu);
  return g_devices;
}

// The sweep over several devices in one process (the reference's thread pool,
// experiment.hpp:342-368, one host thread per device): shard g of G runs
// replications [R g / G, R (g+1) / G) of every point on devs[g] and its
// kernels store the per-replication results straight into devs[0]'s gather
// array (peer stores over NVLink; a device-to-device copy when peer access is
// unavailable), in the shard's own [field][point][replication] block; devs[0]
// then reduces every point in replication order -- the same sums as one
// device, so the results are bit-identical for any device list.
void run_points_multi(std::vector<bb_run_template> tpl, SweepParams E, const std::vector<int>& devs,
                      bb_point_result* out, const PointFail& pf) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    raise(BB_ECUDA, "no CUDA device available (the engine has no CPU path)");
  for (int d : devs)
    if (d < 0 || d >= ndev) raise(BB_EINVAL, "bb_set_devices: device ordinal out of range");
  std::vector<int> uniq(devs);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int d : uniq) locks.emplace_back(g_ctx[d].mu);  // ascending order: no lock cycles
  const int d0 = devs[0];
  CK(cudaSetDevice(d0));
  cudaStream_t st0 = ctx_stream(d0);
  const uint64_t P = tpl.size(), R = E.replications, G = devs.size();
  if (R < G) raise(BB_EINVAL, "fewer replications than devices");
  DBuf rep(BB_REP_FIELDS * P * R * 8, st0), stats(P * 8 * 8, st0);
  CK(cudaStreamSynchronize(st0));  // the gather array exists before any shard writes it
  std::vector<char> peer(ndev, 0);
  for (int d : uniq) {
    if (d == d0) continue;
    int ok = 0;
    CK(cudaDeviceCanAccessPeer(&ok, d, d0));
    if (!ok) continue;
    CK(cudaSetDevice(d));
    const cudaError_t e = cudaDeviceEnablePeerAccess(d0, 0);
    if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) peer[d] = 1;
    cudaGetLastError();
  }
  std::vector<std::exception_ptr> errs(G);
  auto shard = [&](uint64_t g) {
    try {
      const int dev = devs[g];
      CK(cudaSetDevice(dev));
      cudaStream_t st;
      CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
        }
      } guard{st};
      const uint64_t lo = R * g / G, hi = R * (g + 1) / G;
      double* dst = rep.as<double>() + BB_REP_FIELDS * P * lo;  // the shard's block on d0
      Sweep W;
      build_sweep(tpl, W, st, true, pf);
      if (dev == d0 || peer[dev]) {
        launch_sweep(&E, W, lo, hi, dst, st, false, pf, (uint32_t)(hi - lo), (uint32_t)lo);
      } else {
        DBuf loc(BB_REP_FIELDS * P * (hi - lo) * 8, st);
        launch_sweep(&E, W, lo, hi, loc.as<double>(), st, false, pf, (uint32_t)(hi - lo), (uint32_t)lo);
        CK(cudaMemcpyAsync(dst, loc.p, BB_REP_FIELDS * P * (hi - lo) * 8, cudaMemcpyDefault, st));
      }
      CK(cudaStreamSynchronize(st));
    } catch (...) {
      errs[g] = std::current_exception();
    }
  };
  std::vector<std::thread> pool;
  for (uint64_t g = 1; g < G; ++g) pool.emplace_back(shard, g);
  shard(0);
  for (auto& t : pool) t.join();
  for (auto& e : errs)  // the lowest shard's error, as the reference's first failure
    if (e) std::rethrow_exception(e);
  CK(cudaSetDevice(d0));
  g_ev_valid = false;
  Sweep W;
  W.tpl = std::move(tpl);
  for (auto& t : W.tpl) W.spec.push_back(materialize(t, 0));
  CK(bb::gen_point_reduce(rep.as<double>(), (uint32_t)P, (uint32_t)R, stats.as<double>(), st0,
                          (uint32_t)G));
  std::vector<double> hs(P * 8);
  d2h(hs.data(), stats.p, hs.size() * 8, st0);
  CK(cudaStreamSynchronize(st0));
  fill_points(&E, W, hs, out);
}

void run_points_host(std::vector<bb_run_template> tpl, SweepParams E, int32_t rng,
                     bb_point_result* out, const PointFail& pf = PointFail{}) {
  const std::vector<int> devs = sweep_devices();
  if (rng != BB_RNG_REFERENCE && devs.size() > 1) {
    if (tpl.empty()) raise(BB_EINVAL, "sweep has no points");
    run_points_multi(std::move(tpl), E, devs, out, pf);
    return;
  }
  const int dev = current_device(devs.empty() ? -1 : devs[0]);
  std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
  cudaStream_t st = ctx_stream(dev);
  Sweep W;
  build_sweep(std::move(tpl), W, st, rng != BB_RNG_REFERENCE, pf);
  const uint64_t P = W.tpl.size(), R = E.replications;
  DBuf rep(BB_REP_FIELDS * P * R * 8, st), stats(P * 8 * 8, st);
  if (rng == BB_RNG_REFERENCE) {
    std::vector<double> h;
    reference_point_reps(&E, W, h, st, pf);
    CK(cudaMemcpyAsync(rep.p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
  } else {
    launch_sweep(&E, W, 0, R, rep.as<double>(), st, true, pf);
  }
  CK(bb::gen_point_reduce(rep.as<double>(), (uint32_t)P, (uint32_t)R, stats.as<double>(), st));
  std::vector<double> hs(P * 8);
  d2h(hs.data(), stats.p, hs.size() * 8, st);
  CK(cudaStreamSynchronize(st));
  fill_points(&E, W, hs, out);
}

// Stream-ordered shard (one process per GPU): no host synchronisation; a
// device-side error (out-of-support service) is left in the device's pending
// flag and raised by the next reduce on this device.
// local: rep_dev holds only [rep_begin, rep_end) ([field][point][its reps]),
// the block a gather of shard slices concatenates (bb_points_reduce_gathered_device).
void points_shard(std::vector<bb_run_template> tpl, SweepParams E, uint64_t rep_begin,
                  uint64_t rep_end, double* rep_dev, void* stream, bool local = false) {
  if (rep_end > E.replications || rep_begin > rep_end) raise(BB_EINVAL, "bad replication range");
  const int dev = current_device(-1);
  std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx_stream(dev);
  DevCtx& C = g_ctx[dev];
  if (!C.pending) {
    CK(cudaMalloc((void**)&C.pending, sizeof(bb::DevError)));
    CK(cudaMemsetAsync(C.pending, 0xFF, 8, st));
  }
  Sweep W;
  build_sweep(std::move(tpl), W, st);
  C.pending_support.clear();
  for (const SimSpec& sp : W.spec) C.pending_support.push_back({sp.edges.front(), sp.edges.back()});
  if (rep_end > rep_begin)
    launch_sweep(&E, W, rep_begin, rep_end, rep_dev, st, true, PointFail{},
                 local ? (uint32_t)(rep_end - rep_begin) : 0u, local ? (uint32_t)rep_begin : 0u,
                 C.pending);
}

// chunks > 1: rep_dev is a gather of `chunks` shard slices (see gen_point_reduce)
void points_reduce(std::vector<bb_run_template> tpl, SweepParams E, const double* rep_dev,
                   bb_point_result* out, void* stream, uint32_t chunks = 1) {
  const int dev = current_device(-1);
  std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx_stream(dev);
  DevCtx& C = g_ctx[dev];
  Sweep W;
  W.tpl = std::move(tpl);
  for (auto& t : W.tpl) W.spec.push_back(materialize(t, 0));
  const uint64_t P = W.tpl.size();
  DBuf stats(P * 8 * 8, st);
  CK(bb::gen_point_reduce(rep_dev, (uint32_t)P, (uint32_t)E.replications, stats.as<double>(), st,
                          chunks));
  std::vector<double> hs(P * 8);
  d2h(hs.data(), stats.p, hs.size() * 8, st);
  bb::DevError he{~0ull, 0.0, 0};
  if (C.pending) d2h(&he, C.pending, sizeof he, st);
  CK(cudaStreamSynchronize(st));
  if (he.packed != ~0ull) {  // a shard on this device failed: report it here
    CK(cudaMemsetAsync(C.pending, 0xFF, 8, st));
    CK(cudaStreamSynchronize(st));
    const size_t pt = (size_t)(he.packed >> 40);
    raise_sweep_error(he, pt < C.pending_support.size() ? C.pending_support[pt]
                                                         : std::pair<double, double>{0.0, 0.0},
                      PointFail{});
  }
  fill_points(&E, W, hs, out);
}

}  // namespace

namespace bb {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace bb

// =================================================================== C ABI
extern "C" {

const char* bb_last_error(void) { return g_err.c_str(); }
int bb_abi_version(void) { return BB_ABI_VERSION; }

bb_status bb_device_info(int32_t device, char* name, size_t name_len, int32_t* sm_count,
                         int32_t* cc_major, int32_t* cc_minor) {
  return guarded([&] {
    const int dev = current_device(device);
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    if (name && name_len) snprintf(name, name_len, "%s", p.name);
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
  });
}

bb_status bb_run_simulation(const bb_sim_config* cfg, bb_sim_metrics* out) {
  return guarded([&] { run_single(cfg, nullptr, 0, out, nullptr); });
}

bb_status bb_run_simulation_detailed(const bb_sim_config* cfg, bb_sim_metrics* out,
                                     bb_sim_detail* detail) {
  return guarded([&] { run_single(cfg, nullptr, 0, out, detail); });
}

bb_status bb_replay_trace(const bb_sim_config* cfg, const double* lengths, uint64_t n_lengths,
                          bb_sim_metrics* out) {
  return guarded([&] {
    if (!lengths || !n_lengths) raise(BB_EINVAL, "replay_trace: empty trace");
    run_single(cfg, lengths, n_lengths, out, nullptr);
  });
}

bb_status bb_replay_trace_detailed(const bb_sim_config* cfg, const double* lengths,
                                   uint64_t n_lengths, bb_sim_metrics* out,
                                   bb_sim_detail* detail) {
  return guarded([&] {
    if (!lengths || !n_lengths) raise(BB_EINVAL, "replay_trace: empty trace");
    run_single(cfg, lengths, n_lengths, out, detail);
  });
}

bb_status bb_run_trace(const bb_sim_config* cfg, const bb_trace_in* in, bb_sim_metrics* out,
                       bb_sim_detail* detail) {
  return guarded([&] {
    if (!in || !in->arrivals || !in->services) raise(BB_EINVAL, "trace arrays: arrivals and services are required");
    bb_sim_config c2 = *cfg;
    c2.service_kind = BB_SVC_UNIFORM;  // services come from the arrays; skip sampler checks
    c2.lo = 0;
    c2.hi = 1;
    SimSpec c = make_spec(&c2);
    c.svc = cfg->service_kind;
    const int dev = current_device(cfg->device);
    std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
    cudaStream_t st = ctx_stream(dev);
    const uint64_t n = c.n;
    DBuf a = upload(in->arrivals, n, st), s = upload(in->services, n, st), u, pr;
    if (in->u_err) u = upload(in->u_err, n, st);
    if (in->pred_bin) pr = upload(in->pred_bin, n, st);
    run_pipeline(c, a.as<double>(), s.as<double>(), u.as<double>(), pr.as<uint8_t>(), out, detail,
                 false, st);
    if (detail) {
      if (detail->req_arrival) std::memcpy(detail->req_arrival, in->arrivals, n * 8);
      if (detail->req_service) std::memcpy(detail->req_service, in->services, n * 8);
    }
  });
}

bb_status bb_run_trace_device(const bb_sim_config* cfg, const bb_trace_in* in, bb_sim_metrics* out,
                              bb_sim_detail* detail, void* stream) {
  return guarded([&] {
    if (!in || !in->arrivals || !in->services) raise(BB_EINVAL, "trace arrays: arrivals and services are required");
    bb_sim_config c2 = *cfg;
    c2.service_kind = BB_SVC_UNIFORM;
    c2.lo = 0;
    c2.hi = 1;
    SimSpec c = make_spec(&c2);
    const int dev = current_device(cfg->device);
    std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx_stream(dev);
    run_pipeline(c, in->arrivals, in->services, in->u_err, in->pred_bin, out, detail, true, st);
  });
}

uint64_t bb_replication_seed(uint64_t master, uint64_t rep) { return bb::replication_seed(master, rep); }

bb_status bb_experiment_points(const bb_experiment_spec* spec, uint64_t* n_points) {
  return guarded([&] { *n_points = expand(spec).size(); });
}

bb_status bb_run_experiment(const bb_experiment_spec* spec, unsigned jobs, bb_point_result* out,
                            uint64_t capacity, uint64_t* n_points) {
  (void)jobs;  // results never depend on the pool size (experiment.hpp:309-311)
  return guarded([&] {
    std::vector<bb_run_template> tpl = expand(spec);
    const uint64_t P = tpl.size();
    if (n_points) *n_points = P;
    if (!out) return;
    if (capacity < P) raise(BB_EINVAL, "bb_run_experiment: output capacity too small");
    PointFail pf;
    pf.name = spec->name ? spec->name : "experiment";
    run_points_host(std::move(tpl), SweepParams{spec->seed, spec->replications}, spec->rng, out, pf);
  });
}

bb_status bb_run_points(const bb_run_template* points, uint64_t n_points, uint64_t replications,
                        uint64_t seed, int32_t rng, bb_point_result* out) {
  return guarded([&] {
    if (!points || !n_points || !out) raise(BB_EINVAL, "bb_run_points: empty point list");
    if (replications < 1) raise(BB_EINVAL, "experiment spec: replications must be >= 1");
    run_points_host(std::vector<bb_run_template>(points, points + n_points),
                    SweepParams{seed, replications}, rng, out);
  });
}

bb_status bb_run_point(const bb_run_template* t, uint64_t master_seed, uint64_t replications,
                       bb_point_result* out) {
  // run_point (experiment.hpp:254): errors propagate unwrapped
  return guarded([&] {
    if (!t || !out) raise(BB_EINVAL, "bb_run_point: null template or output");
    if (replications < 1) raise(BB_EINVAL, "experiment spec: replications must be >= 1");
    run_points_host(std::vector<bb_run_template>(1, *t), SweepParams{master_seed, replications},
                    BB_RNG_PHILOX, out);
  });
}

bb_status bb_sweep_shard_device(const bb_experiment_spec* spec, uint64_t rep_begin,
                                uint64_t rep_end, double* rep_metrics_dev, void* stream) {
  return guarded([&] {
    std::vector<bb_run_template> tpl = expand(spec);
    points_shard(std::move(tpl), SweepParams{spec->seed, spec->replications}, rep_begin, rep_end,
                 rep_metrics_dev, stream);
  });
}

bb_status bb_points_shard_device(const bb_run_template* points, uint64_t n_points,
                                 uint64_t replications, uint64_t seed, uint64_t rep_begin,
                                 uint64_t rep_end, double* rep_metrics_dev, void* stream) {
  return guarded([&] {
    if (!points || !n_points) raise(BB_EINVAL, "empty point list");
    points_shard(std::vector<bb_run_template>(points, points + n_points),
                 SweepParams{seed, replications}, rep_begin, rep_end, rep_metrics_dev, stream);
  });
}

bb_status bb_points_shard_local_device(const bb_run_template* points, uint64_t n_points,
                                       uint64_t replications, uint64_t seed, uint64_t rep_begin,
                                       uint64_t rep_end, double* shard_dev, void* stream) {
  return guarded([&] {
    if (!points || !n_points) raise(BB_EINVAL, "empty point list");
    points_shard(std::vector<bb_run_template>(points, points + n_points),
                 SweepParams{seed, replications}, rep_begin, rep_end, shard_dev, stream, true);
  });
}

bb_status bb_points_reduce_gathered_device(const bb_run_template* points, uint64_t n_points,
                                           uint64_t replications, uint32_t n_shards,
                                           const double* gathered_dev, bb_point_result* out,
                                           void* stream) {
  return guarded([&] {
    if (!points || !n_points) raise(BB_EINVAL, "empty point list");
    if (n_shards < 1 || n_shards > replications) raise(BB_EINVAL, "bad shard count");
    points_reduce(std::vector<bb_run_template>(points, points + n_points),
                  SweepParams{0, replications}, gathered_dev, out, stream, n_shards);
  });
}

bb_status bb_set_devices(const int32_t* devices, uint32_t n) {
  return guarded([&] {
    if (n && !devices) raise(BB_EINVAL, "bb_set_devices: null device list");
    int ndev = 0;
    if (n && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0))
      raise(BB_ECUDA, "no CUDA device available (the engine has no CPU path)");
    for (uint32_t i = 0; i < n; ++i)
      if (devices[i] < 0 || devices[i] >= ndev) raise(BB_EINVAL, "bb_set_devices: device ordinal out of range");
    std::lock_guard<std::mutex> lock(g_dev_mu);
    g_devices.assign(devices, devices + n);
  });
}

bb_status bb_sweep_reduce_device(const bb_experiment_spec* spec, const double* rep_metrics_dev,
                                 bb_point_result* out, void* stream) {
  return guarded([&] {
    points_reduce(expand(spec), SweepParams{spec->seed, spec->replications}, rep_metrics_dev, out,
                  stream);
  });
}

bb_status bb_points_reduce_device(const bb_run_template* points, uint64_t n_points,
                                  uint64_t replications, const double* rep_metrics_dev,
                                  bb_point_result* out, void* stream) {
  return guarded([&] {
    if (!points || !n_points) raise(BB_EINVAL, "empty point list");
    points_reduce(std::vector<bb_run_template>(points, points + n_points),
                  SweepParams{0, replications}, rep_metrics_dev, out, stream);
  });
}

bb_status bb_uniform_boundaries(uint64_t k, double lo, double hi, double* out) {
  return guarded([&] {
    auto e = uniform_edges(k, lo, hi);
    std::memcpy(out, e.data(), e.size() * 8);
  });
}
bb_status bb_exponential_boundaries(uint64_t k, double rate, uint64_t B, double* out) {
  return guarded([&] {
    auto e = exponential_edges(k, rate, B);
    std::memcpy(out, e.data(), e.size() * 8);
  });
}
bb_status bb_empirical_boundaries(uint64_t k, const double* s, uint64_t n, double* out) {
  return guarded([&] {
    auto e = empirical_edges(k, s, n);
    std::memcpy(out, e.data(), e.size() * 8);
  });
}
double bb_analytic_throughput(uint64_t B, uint64_t k, double lo, double hi) {
  return an_throughput(B, k, lo, hi);
}
double bb_analytic_latency(uint64_t B, uint64_t k, double lo, double hi, double lam) {
  return an_latency(B, k, lo, hi, lam);
}

void bb_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint4 r = bb::philox4x32_10(make_uint4(ctr[0], ctr[1], ctr[2], ctr[3]), key[0], key[1]);
  out[0] = r.x;
  out[1] = r.y;
  out[2] = r.z;
  out[3] = r.w;
}

bb_status bb_exponential_variates(const uint64_t* keys, uint64_t n, int32_t table, double* out) {
  return guarded([&] {
    if (n && (!keys || !out)) raise(BB_EINVAL, "exponential variates: null buffer");
    for (uint64_t i = 0; i < n; ++i)
      if (keys[i] >= (1ull << 53)) raise(BB_EINVAL, "exponential variates: keys must be < 2^53");
    const int dev = current_device(-1);
    std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
    cudaStream_t st = ctx_stream(dev);
    DBuf x = upload(keys, n, st), y(n * 8, st);
    CK(bb::exp1_variates(x.as<uint64_t>(), n, table, y.as<double>(), st));
    d2h(out, y.p, n * 8, st);
    CK(cudaStreamSynchronize(st));
  });
}

bb_status bb_template_edges(const bb_run_template* t, double* out, uint64_t capacity,
                            uint64_t* n_edges) {
  return guarded([&] {
    if (!t) raise(BB_EINVAL, "null run template");
    const SimSpec s = materialize(*t, 0);
    if (n_edges) *n_edges = s.edges.size();
    if (!out) return;
    if (capacity < s.edges.size()) raise(BB_EINVAL, "bb_template_edges: capacity too small");
    std::memcpy(out, s.edges.data(), s.edges.size() * 8);
  });
}

bb_status bb_service_of_keys(const bb_run_template* t, const uint64_t* keys, uint64_t n,
                             double* out) {
  return guarded([&] {
    if (!t) raise(BB_EINVAL, "null run template");
    if (n && (!keys || !out)) raise(BB_EINVAL, "service keys: null buffer");
    const SimSpec c = materialize(*t, 0);
    const int dev = current_device(-1);
    std::lock_guard<std::mutex> lock(g_ctx[dev].mu);
    cudaStream_t st = ctx_stream(dev);
    SvcDev sv;
    make_svc(c, sv, st);
    DBuf x = upload(keys, n, st), y(n * 8, st);
    CK(bb::service_of_keys(sv.p, x.as<uint64_t>(), n, y.as<double>(), st));
    d2h(out, y.p, n * 8, st);
    CK(cudaStreamSynchronize(st));
  });
}

void bb_transfer_bytes(uint64_t* h2d_bytes, uint64_t* d2h_bytes, int reset) {
  if (h2d_bytes) *h2d_bytes = reset ? bb::g_h2d.exchange(0) : bb::g_h2d.load();
  if (d2h_bytes) *d2h_bytes = reset ? bb::g_d2h.exchange(0) : bb::g_d2h.load();
}

int bb_set_generated_quantiles(int on) { return bb::g_gen_quantiles.exchange(on ? 1 : 0); }

uint64_t bb_launch_count(int reset) {
  return reset ? bb::g_launches.exchange(0) : bb::g_launches.load();
}

void bb_trace_graph_stats(uint64_t* captures, uint64_t* replays, int reset) {
  bb::trace_graph_stats(captures, replays, reset != 0);
}

double bb_last_kernel_ms(const char** name) {
  if (name) *name = g_ev_name;
  if (!g_ev_valid) return g_trace_ms;
  float ms = 0;
  if (cudaEventSynchronize(g_ev[1]) != cudaSuccess) return -1.0;
  if (cudaEventElapsedTime(&ms, g_ev[0], g_ev[1]) != cudaSuccess) return -1.0;
  return ms;
}

}  // extern "C"
