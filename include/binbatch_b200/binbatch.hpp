#pragma once
// binbatch_b200/binbatch.hpp -- C++ drop-in for the reference simulator API.
//
// Replace   #include "binbatch/binbatch.hpp"      (reference, header-only)
// with      #include "binbatch_b200/binbatch.hpp" and link libbinbatch_b200.so.
//
// Same namespace, type and function names as the reference
// (/root/reference/proj/include/binbatch/{simulator,experiment,binning,
// service_dist,analytics}.hpp); every simulation forwards to the C ABI
// (include/binbatch_b200.h) and runs on the B200.  Status codes are rethrown
// as the reference's exception types.
//
// A reference program can also stay byte-for-byte unchanged: compile it with
// -I include/compat first on the include path (include/compat/binbatch/*.hpp
// forward every reference header name here) and link the library.
//
// Differences a caller can observe (documented in DESIGN.md):
//   * SimConfig::rng selects the random streams: Rng::reference reproduces the
//     reference's mt19937_64 streams (bit-exact per-request/per-batch records,
//     dispatch order, completions, makespan, throughput, p50/p99; the
//     Sigma-based latency_mean and busy fraction are tree sums, equal to the
//     reference's sequential sums within n * 2^-53 relative), Rng::philox (the
//     default for sweeps) draws counter-based streams on the device
//     (distribution-equal; every replication's p50/p99 is exact for its draws).
//   * > 32 bins (single runs), > 64 bins (sweeps) and n >= 2^32 throw
//     std::logic_error("...not supported").
//   * ServiceKind / ServiceSpec add the linear (tokens -> time) and log-normal
//     samplers of BASELINE configs 3 and 5; ServiceSpec::trace_times and
//     ErrorSpec::rows accept in-memory data in place of trace / matrix files.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <istream>
#include <limits>
#include <map>
#include <optional>
#include <ostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../binbatch_b200.h"

#if __has_include(<json.hpp>)
#include <json.hpp>
#define BINBATCH_B200_HAS_JSON 1
#endif

namespace binbatch {

constexpr double kOverload = std::numeric_limits<double>::infinity();
constexpr std::size_t kNoBatch = std::numeric_limits<std::size_t>::max();

namespace detail {
inline void check(bb_status st) {
  switch (st) {
    case BB_OK: return;
    case BB_EINVAL: throw std::invalid_argument(bb_last_error());
    case BB_EDOMAIN: throw std::domain_error(bb_last_error());
    case BB_EUNSUPPORTED: throw std::logic_error(bb_last_error());
    default: throw std::runtime_error(bb_last_error());
  }
}
template <class... Ts>
struct overloaded : Ts... {
  using Ts::operator()...;
};
template <class... Ts>
overloaded(Ts...) -> overloaded<Ts...>;

// rng.hpp:16-21
inline std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
}  // namespace detail

// ---------------------------------------------------------------- rng.hpp
// The reference's host stream (rng.hpp:28-53): std::mt19937_64 seeded
// through splitmix64.  Simulations never use it on the device path; it is
// here for callers that draw on the host (and it is the generator behind
// Rng::reference runs).
class RandomStream {
 public:
  explicit RandomStream(std::uint64_t seed) : engine_(detail::splitmix64(seed)) {}
  static RandomStream derive(std::uint64_t master_seed, std::uint64_t stream_id) {
    return RandomStream(detail::splitmix64(master_seed ^ (0x632BE59BD9B4E019ULL * (stream_id + 1))));
  }
  double uniform01() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  double exponential(double rate) { return -std::log1p(-uniform01()) / rate; }
  std::size_t index(std::size_t n) {
    if (n == 0) throw std::invalid_argument("RandomStream::index: n must be positive");
    return static_cast<std::size_t>(engine_() % n);
  }

 private:
  std::mt19937_64 engine_;
};

// ---------------------------------------------------------------- service_dist.hpp
struct Uniform { double min_time = 0, max_time = 0; };
struct Exponential { double rate = 0; };
struct Empirical { std::vector<double> samples; };
using ServiceDist = std::variant<Uniform, Exponential, Empirical>;

inline ServiceDist make_uniform(double lo, double hi) {
  if (!(lo >= 0) || !(lo < hi) || !std::isfinite(hi))
    throw std::invalid_argument("uniform service: need 0 <= min_time < max_time");
  return Uniform{lo, hi};
}
inline ServiceDist make_exponential(double rate) {
  if (!(rate > 0) || !std::isfinite(rate))
    throw std::invalid_argument("exponential service: rate must be positive");
  return Exponential{rate};
}
inline ServiceDist make_empirical(std::vector<double> s) {
  if (s.empty()) throw std::invalid_argument("empirical service: sample set is empty");
  for (double v : s)
    if (!(v > 0) || !std::isfinite(v))
      throw std::invalid_argument("empirical service: all samples must be positive");
  std::sort(s.begin(), s.end());
  return Empirical{std::move(s)};
}
inline double expected_max_uniform(std::size_t count, double lo, double hi) {
  if (count == 0) throw std::invalid_argument("expected_max_uniform: count must be >= 1");
  if (!(lo < hi)) throw std::invalid_argument("expected_max_uniform: need lo < hi");
  const double b = static_cast<double>(count);
  return (b * hi + lo) / (b + 1.0);
}
inline double harmonic_number(std::size_t n) {  // service_dist.hpp:82-87
  double h = 0;
  detail::check(bb_harmonic_number(n, &h));
  return h;
}
inline double mean(const ServiceDist& dist) {  // service_dist.hpp:65-72
  return std::visit(detail::overloaded{
                        [](const Uniform& u) { return (u.min_time + u.max_time) / 2.0; },
                        [](const Exponential& e) { return 1.0 / e.rate; },
                        [](const Empirical& e) {
                          double sum = 0.0;
                          for (double v : e.samples) sum += v;
                          return sum / static_cast<double>(e.samples.size());
                        },
                    },
                    dist);
}
// One host draw (service_dist.hpp:94-101).
inline double sample(const ServiceDist& dist, RandomStream& rng) {
  return std::visit(detail::overloaded{
                        [&](const Uniform& u) { return rng.uniform(u.min_time, u.max_time); },
                        [&](const Exponential& e) { return rng.exponential(e.rate); },
                        [&](const Empirical& e) { return e.samples[rng.index(e.samples.size())]; },
                    },
                    dist);
}

// ---------------------------------------------------------------- binning.hpp
struct BinConfig {
  std::vector<double> edges;
  std::size_t bin_count() const { return edges.size() - 1; }
  double lower() const { return edges.front(); }
  double upper() const { return edges.back(); }
};

inline BinConfig make_bin_config(std::vector<double> edges) {
  if (edges.size() < 2) throw std::invalid_argument("bin config: need at least two edges");
  for (std::size_t i = 0; i < edges.size(); ++i) {
    const bool last = i + 1 == edges.size();
    if (std::isnan(edges[i]) || (!last && !std::isfinite(edges[i])) ||
        (last && edges[i] == -std::numeric_limits<double>::infinity()))
      throw std::invalid_argument("bin config: only the top edge may be infinite");
  }
  for (std::size_t i = 1; i < edges.size(); ++i)
    if (!(edges[i - 1] < edges[i]))
      throw std::invalid_argument("bin config: edges must be strictly increasing");
  return BinConfig{std::move(edges)};
}

inline BinConfig uniform_boundaries(std::size_t k, double lo, double hi) {
  std::vector<double> e(k + 1);
  detail::check(bb_uniform_boundaries(k, lo, hi, e.data()));
  return BinConfig{std::move(e)};
}
inline BinConfig exponential_boundaries(std::size_t k, double rate, std::size_t batch_size) {
  std::vector<double> e(k + 1);
  detail::check(bb_exponential_boundaries(k, rate, batch_size, e.data()));
  return BinConfig{std::move(e)};
}
inline BinConfig empirical_boundaries(std::size_t k, const std::vector<double>& samples) {
  std::vector<double> e(k + 1);
  detail::check(bb_empirical_boundaries(k, samples.data(), samples.size(), e.data()));
  return BinConfig{std::move(e)};
}

namespace detail {
inline double interpolated_quantile(const std::vector<double>& sorted, double q) {  // :98-104
  const double pos = q * static_cast<double>(sorted.size() - 1);
  const auto idx = static_cast<std::size_t>(pos);
  if (idx + 1 >= sorted.size()) return sorted.back();
  const double frac = pos - static_cast<double>(idx);
  return sorted[idx] + frac * (sorted[idx + 1] - sorted[idx]);
}
}  // namespace detail

// [L_1 .. L_{k-1}], L_1 = H_B, L_m = 1 + ln L_{m-1} (binning.hpp:59-75)
inline std::vector<double> l_sequence(std::size_t k, std::size_t batch_size) {
  if (k == 0) throw std::invalid_argument("l_sequence: k must be >= 1");
  if (batch_size == 0) throw std::invalid_argument("l_sequence: batch size must be >= 1");
  std::vector<double> seq;
  if (k == 1) return seq;
  seq.push_back(harmonic_number(batch_size));
  while (seq.size() + 1 < k) {
    if (!(seq.back() > 0)) throw std::domain_error("l_sequence: non-positive term, log undefined");
    seq.push_back(1.0 + std::log(seq.back()));
  }
  return seq;
}

inline std::size_t assign_bin(const BinConfig& config, double length) {  // :133-144
  uint64_t b = 0;
  detail::check(bb_assign_bin(config.edges.data(), config.edges.size(), length, &b));
  return static_cast<std::size_t>(b);
}

struct Perfect {};
struct Symmetric { double p_error = 0; };
struct Confusion { std::vector<std::vector<double>> rows; };
using ErrorModel = std::variant<Perfect, Symmetric, Confusion>;

inline ErrorModel make_symmetric(double p) {
  if (!(p >= 0) || !(p <= 0.5))
    throw std::invalid_argument("symmetric error model: need 0 <= p_error <= 0.5");
  return Symmetric{p};
}
inline ErrorModel make_confusion(std::vector<std::vector<double>> rows) {
  if (rows.empty()) throw std::invalid_argument("confusion matrix: empty");
  for (const auto& r : rows) {
    if (r.size() != rows.size()) throw std::invalid_argument("confusion matrix: must be square");
    double sum = 0;
    for (double p : r) {
      if (!(p >= 0)) throw std::invalid_argument("confusion matrix: negative entry");
      sum += p;
    }
    if (std::abs(sum - 1.0) > 1e-9) throw std::invalid_argument("confusion matrix: row sum != 1");
  }
  return Confusion{std::move(rows)};
}

// Plain-text matrix, k lines of k probabilities (binning.hpp:191-223).
inline ErrorModel parse_confusion(std::istream& in, const std::string& name) {
  std::vector<std::vector<double>> rows;
  std::string line;
  std::size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    std::istringstream fields(line);
    std::vector<double> row;
    double v = 0;
    while (fields >> v) row.push_back(v);
    if (!fields.eof())
      throw std::runtime_error(name + " line " + std::to_string(line_no) + ": malformed probability");
    if (!row.empty()) rows.push_back(std::move(row));
  }
  if (rows.empty()) throw std::runtime_error(name + ": no matrix rows");
  for (std::size_t i = 0; i < rows.size(); ++i)
    if (rows[i].size() != rows.size())
      throw std::runtime_error(name + ": row " + std::to_string(i + 1) + " has " +
                               std::to_string(rows[i].size()) + " entries, expected " +
                               std::to_string(rows.size()));
  return make_confusion(std::move(rows));
}
inline ErrorModel load_confusion(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open confusion matrix file: " + path);
  return parse_confusion(in, path);
}

// Predicted bin on the host (binning.hpp:231-261); the device path applies
// the same rule in key space.
inline std::size_t predict_bin(const ErrorModel& model, std::size_t true_bin, std::size_t k,
                               RandomStream& rng) {
  if (true_bin < 1 || true_bin > k) throw std::invalid_argument("predict_bin: true bin out of range");
  if (const auto* s = std::get_if<Symmetric>(&model)) {
    if (k == 1 || s->p_error == 0) return true_bin;
    const double u = rng.uniform01();
    if (true_bin == 1) return u < s->p_error ? std::size_t{2} : true_bin;
    if (true_bin == k) return u < s->p_error ? k - 1 : true_bin;
    if (u < s->p_error) return true_bin - 1;
    if (u >= 1.0 - s->p_error) return true_bin + 1;
    return true_bin;
  }
  if (const auto* c = std::get_if<Confusion>(&model)) {
    if (c->rows.size() != k)
      throw std::invalid_argument("predict_bin: confusion matrix size does not match k");
    const auto& row = c->rows[true_bin - 1];
    const double u = rng.uniform01();
    double cum = 0.0;
    for (std::size_t j = 0; j < k; ++j) {
      cum += row[j];
      if (u < cum) return j + 1;
    }
    return k;
  }
  return true_bin;
}

// Exhaustive grid search of the batch-service objective (binning.hpp:268-351).
inline BinConfig brute_force_boundaries(std::size_t k, const ServiceDist& dist,
                                        std::size_t batch_size, std::size_t grid_points) {
  std::vector<double> e(k + 1 > 4 ? k + 1 : 4);
  if (const auto* u = std::get_if<Uniform>(&dist))
    detail::check(bb_brute_force_boundaries(k, 0, u->min_time, u->max_time, batch_size,
                                            grid_points, e.data()));
  else if (const auto* x = std::get_if<Exponential>(&dist))
    detail::check(bb_brute_force_boundaries(k, 1, x->rate, 0.0, batch_size, grid_points, e.data()));
  else
    detail::check(bb_brute_force_boundaries(k, 2, 0.0, 0.0, batch_size, grid_points, e.data()));
  e.resize(k + 1);
  return make_bin_config(std::move(e));
}

// ---------------------------------------------------------------- simulator.hpp
struct Request {
  std::size_t id = 0;
  double arrival_time = 0;
  double service_time = 0;
  std::size_t true_bin = 0;
  std::size_t predicted_bin = 0;
  std::size_t batch = kNoBatch;
  double completion_time = std::numeric_limits<double>::quiet_NaN();
};

struct BatchRecord {
  std::size_t bin = 0;
  std::vector<std::size_t> members;
  double formed_time = 0;
  double start_time = std::numeric_limits<double>::quiet_NaN();
  double finish_time = std::numeric_limits<double>::quiet_NaN();
  double service_time = 0;
};

enum class TraceMode { cyclic, resample };
enum class Rng { philox = BB_RNG_PHILOX, reference = BB_RNG_REFERENCE };

struct SimConfig {
  double arrival_rate = kOverload;
  std::size_t n_requests = 0;
  std::size_t batch_size = 1;
  BinConfig bins;
  ErrorModel error_model = Perfect{};
  std::size_t n_servers = 1;
  ServiceDist service = Uniform{1.0, 2.0};
  std::uint64_t seed = 0;
  bool flush_partial = true;
  std::optional<double> max_batch_wait;
  TraceMode trace_mode = TraceMode::cyclic;
  Rng rng = Rng::reference;  // a drop-in reproduces the reference's streams by default
  int device = -1;
};

struct SimMetrics {
  double throughput = 0;
  double makespan = 0;
  double latency_mean = 0;
  double latency_p50 = 0;
  double latency_p99 = 0;
  std::vector<std::size_t> per_bin_batch_counts;
  double server_busy_fraction = 0;
  std::size_t n_completed = 0;
  bool operator==(const SimMetrics&) const = default;
};

struct SimResult {
  SimMetrics metrics;
  std::vector<Request> requests;
  std::vector<BatchRecord> batches;
};

namespace detail {

struct CfgHolder {
  bb_sim_config c{};
  std::vector<double> conf, table;
};

inline CfgHolder to_c(const SimConfig& s) {
  CfgHolder h;
  bb_sim_config& c = h.c;
  c.arrival_rate = s.arrival_rate;
  c.n_requests = s.n_requests;
  c.batch_size = s.batch_size;
  c.n_servers = s.n_servers;
  c.seed = s.seed;
  c.flush_partial = s.flush_partial;
  c.has_max_batch_wait = s.max_batch_wait.has_value();
  c.max_batch_wait = s.max_batch_wait.value_or(0.0);
  c.edges = s.bins.edges.empty() ? nullptr : s.bins.edges.data();
  c.n_edges = s.bins.edges.size();
  if (const auto* sy = std::get_if<Symmetric>(&s.error_model)) {
    c.error_kind = BB_ERR_SYMMETRIC;
    c.p_error = sy->p_error;
  } else if (const auto* cf = std::get_if<Confusion>(&s.error_model)) {
    c.error_kind = BB_ERR_CONFUSION;
    const std::size_t ck = cf->rows.size();
    for (const auto& r : cf->rows) {
      if (r.size() != ck) throw std::invalid_argument("confusion matrix: must be square");
      h.conf.insert(h.conf.end(), r.begin(), r.end());
    }
    c.confusion = h.conf.empty() ? nullptr : h.conf.data();
    c.confusion_k = ck;
  }
  if (const auto* u = std::get_if<Uniform>(&s.service)) {
    c.service_kind = BB_SVC_UNIFORM;
    c.lo = u->min_time;
    c.hi = u->max_time;
  } else if (const auto* e = std::get_if<Exponential>(&s.service)) {
    c.service_kind = BB_SVC_EXPONENTIAL;
    c.rate = e->rate;
  } else if (const auto* em = std::get_if<Empirical>(&s.service)) {
    c.service_kind = BB_SVC_EMPIRICAL;
    h.table = em->samples;
  }
  c.rng = static_cast<int32_t>(s.rng);
  c.device = s.device;
  if (!h.table.empty()) {
    c.table = h.table.data();
    c.n_table = h.table.size();
  }
  return h;
}

inline SimMetrics from_c(const bb_sim_metrics& m) {
  SimMetrics r;
  r.throughput = m.throughput;
  r.makespan = m.makespan;
  r.latency_mean = m.latency_mean;
  r.latency_p50 = m.latency_p50;
  r.latency_p99 = m.latency_p99;
  r.per_bin_batch_counts.assign(m.per_bin_batch_counts, m.per_bin_batch_counts + m.k);
  r.server_busy_fraction = m.server_busy_fraction;
  r.n_completed = m.n_completed;
  return r;
}

struct DetailBufs {
  std::vector<double> arr, svc, comp, formed, start, finish, service;
  std::vector<uint8_t> tb, pb, bbin;
  std::vector<uint32_t> batch, bsize, bfirst, members;
  bb_sim_detail d{};
  explicit DetailBufs(std::size_t n)
      : arr(n), svc(n), comp(n), formed(n), start(n), finish(n), service(n), tb(n), pb(n),
        bbin(n), batch(n), bsize(n), bfirst(n), members(n) {
    d.req_arrival = arr.data();
    d.req_service = svc.data();
    d.req_true_bin = tb.data();
    d.req_pred_bin = pb.data();
    d.req_batch = batch.data();
    d.req_completion = comp.data();
    d.batch_capacity = n;
    d.bat_bin = bbin.data();
    d.bat_size = bsize.data();
    d.bat_first = bfirst.data();
    d.bat_formed = formed.data();
    d.bat_start = start.data();
    d.bat_finish = finish.data();
    d.bat_service = service.data();
    d.members = members.data();
  }
  SimResult result(const bb_sim_metrics& m) const {
    SimResult r;
    r.metrics = from_c(m);
    const std::size_t n = arr.size();
    r.requests.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
      Request& q = r.requests[i];
      q.id = i;
      q.arrival_time = arr[i];
      q.service_time = svc[i];
      q.true_bin = tb[i];
      q.predicted_bin = pb[i];
      q.batch = batch[i] == BB_NO_BATCH ? kNoBatch : batch[i];
      q.completion_time = comp[i];
    }
    r.batches.resize(m.n_batches);
    for (std::size_t j = 0; j < m.n_batches; ++j) {
      BatchRecord& b = r.batches[j];
      b.bin = bbin[j];
      b.members.assign(members.begin() + bfirst[j], members.begin() + bfirst[j] + bsize[j]);
      b.formed_time = formed[j];
      b.start_time = start[j];
      b.finish_time = finish[j];
      b.service_time = service[j];
    }
    return r;
  }
};

}  // namespace detail

inline SimResult run_simulation_detailed(const SimConfig& config) {
  auto h = detail::to_c(config);
  bb_sim_metrics m{};
  detail::DetailBufs d(config.n_requests);
  detail::check(bb_run_simulation_detailed(&h.c, &m, &d.d));
  return d.result(m);
}

inline SimMetrics run_simulation(const SimConfig& config) {
  auto h = detail::to_c(config);
  bb_sim_metrics m{};
  detail::check(bb_run_simulation(&h.c, &m));
  return detail::from_c(m);
}

inline SimResult replay_trace_detailed(const SimConfig& config, const std::vector<double>& lengths) {
  auto h = detail::to_c(config);
  h.c.service_kind = config.trace_mode == TraceMode::cyclic ? BB_SVC_TRACE_CYCLIC : BB_SVC_TRACE_RESAMPLE;
  bb_sim_metrics m{};
  detail::DetailBufs d(config.n_requests);
  detail::check(bb_replay_trace_detailed(&h.c, lengths.data(), lengths.size(), &m, &d.d));
  return d.result(m);
}

inline SimMetrics replay_trace(const SimConfig& config, const std::vector<double>& lengths) {
  auto h = detail::to_c(config);
  h.c.service_kind = config.trace_mode == TraceMode::cyclic ? BB_SVC_TRACE_CYCLIC : BB_SVC_TRACE_RESAMPLE;
  bb_sim_metrics m{};
  detail::check(bb_replay_trace(&h.c, lengths.data(), lengths.size(), &m));
  return detail::from_c(m);
}

// ---------------------------------------------------------------- analytics.hpp
struct SystemParams {
  std::size_t batch_size = 1;
  std::size_t bins = 1;
  ServiceDist service = Uniform{1.0, 2.0};
  std::optional<double> arrival_rate;
};
inline SystemParams make_system_params(std::size_t batch_size, std::size_t bins, ServiceDist service,
                                       std::optional<double> arrival_rate = {}) {
  if (batch_size == 0) throw std::invalid_argument("system params: batch size must be >= 1");
  if (bins == 0) throw std::invalid_argument("system params: bin count must be >= 1");
  if (arrival_rate && !(*arrival_rate > 0))
    throw std::invalid_argument("system params: arrival rate must be positive");
  return SystemParams{batch_size, bins, std::move(service), arrival_rate};
}
inline double expected_service_time(std::size_t B, std::size_t k, double lo, double hi) {
  double v = 0;
  detail::check(bb_expected_service_time(B, k, lo, hi, &v));
  return v;
}
inline double throughput(std::size_t B, std::size_t k, double lo, double hi) {
  double v = 0;
  detail::check(bb_throughput(B, k, lo, hi, &v));
  return v;
}
inline double max_throughput(std::size_t B, double lo, double hi) {
  double v = 0;
  detail::check(bb_max_throughput(B, lo, hi, &v));
  return v;
}
inline std::size_t min_bins_for_throughput(std::size_t B, double lo, double hi, double epsilon) {
  uint64_t k = 0;
  detail::check(bb_min_bins_for_throughput(B, lo, hi, epsilon, &k));
  return static_cast<std::size_t>(k);
}
inline double expected_latency(std::size_t B, std::size_t k, double lo, double hi, double lam) {
  double v = 0;
  detail::check(bb_expected_latency(B, k, lo, hi, lam, &v));
  return v;
}
inline double exponential_service_bound(std::size_t B, std::size_t k, double rate) {
  double v = 0;
  detail::check(bb_exponential_service_bound(B, k, rate, &v));
  return v;
}
inline double throughput(const SystemParams& p) {  // analytics.hpp:130-135
  const auto* u = std::get_if<Uniform>(&p.service);
  if (!u) throw std::invalid_argument("throughput: closed form requires uniform service");
  return throughput(p.batch_size, p.bins, u->min_time, u->max_time);
}
inline double expected_latency(const SystemParams& p) {  // analytics.hpp:137-144
  const auto* u = std::get_if<Uniform>(&p.service);
  if (!u) throw std::invalid_argument("expected_latency: closed form requires uniform service");
  if (!p.arrival_rate) throw std::invalid_argument("expected_latency: params carry no arrival rate");
  return expected_latency(p.batch_size, p.bins, u->min_time, u->max_time, *p.arrival_rate);
}

// ---------------------------------------------------------------- workload.hpp
// Token counts -> service times (the linear model of the paper's traces).
// Trace files are front-end I/O: CSV is parsed here, JSON lines need
// nlohmann/json on the include path (like the reference).
struct LinearTimeModel {
  double slope = 0;
  double intercept = 0;
};
inline LinearTimeModel make_linear_time_model(double slope, double intercept) {
  if (!(slope > 0) || !std::isfinite(slope))
    throw std::invalid_argument("linear time model: slope must be positive");
  if (!(intercept >= 0) || !std::isfinite(intercept))
    throw std::invalid_argument("linear time model: intercept must be non-negative");
  return LinearTimeModel{slope, intercept};
}
struct TraceEntry {
  std::int64_t id = 0;
  std::size_t token_count = 0;
  std::optional<double> measured_time;
};
struct Trace {
  std::vector<TraceEntry> entries;
};
enum class TraceFormat { csv, jsonl };

namespace detail {
inline std::runtime_error trace_error(const std::string& name, std::size_t line, const std::string& what) {
  return std::runtime_error(name + " line " + std::to_string(line) + ": " + what);
}
inline void check_entry(const TraceEntry& e, const std::string& name, std::size_t line) {
  if (e.token_count < 1) throw trace_error(name, line, "token_count must be >= 1");
  if (e.measured_time && !(*e.measured_time > 0))
    throw trace_error(name, line, "measured_time must be positive");
}
}  // namespace detail

// id,token_count[,measured_time]; one leading header line tolerated (workload.hpp:56-96)
inline Trace parse_trace_csv(std::istream& in, const std::string& name) {
  Trace trace;
  std::string line;
  std::size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    std::vector<std::string> f;
    {
      std::istringstream split(line);
      std::string cell;
      while (std::getline(split, cell, ',')) f.push_back(cell);
    }
    if (line_no == 1 && !f.empty() && f[0].find_first_not_of("0123456789+- \t") != std::string::npos)
      continue;
    if (f.size() < 2 || f.size() > 3)
      throw detail::trace_error(name, line_no, "expected id,token_count[,measured_time]");
    TraceEntry e;
    try {
      std::size_t used = 0;
      e.id = std::stoll(f[0], &used);
      if (used != f[0].size()) throw std::invalid_argument("trailing characters");
      const long long tokens = std::stoll(f[1], &used);
      if (used != f[1].size()) throw std::invalid_argument("trailing characters");
      if (tokens < 0) throw std::invalid_argument("negative token count");
      e.token_count = static_cast<std::size_t>(tokens);
      if (f.size() == 3) {
        e.measured_time = std::stod(f[2], &used);
        if (used != f[2].size()) throw std::invalid_argument("trailing characters");
      }
    } catch (const std::exception&) {
      throw detail::trace_error(name, line_no, "malformed field in '" + line + "'");
    }
    detail::check_entry(e, name, line_no);
    trace.entries.push_back(e);
  }
  if (trace.entries.empty()) throw std::runtime_error(name + ": no trace entries");
  return trace;
}

#ifdef BINBATCH_B200_HAS_JSON
// {"id":1,"token_count":100,"measured_time":2.5} per line (workload.hpp:98-128)
inline Trace parse_trace_jsonl(std::istream& in, const std::string& name) {
  Trace trace;
  std::string line;
  std::size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    nlohmann::json obj;
    try {
      obj = nlohmann::json::parse(line);
    } catch (const nlohmann::json::exception& ex) {
      throw detail::trace_error(name, line_no, ex.what());
    }
    if (!obj.contains("id") || !obj.contains("token_count"))
      throw detail::trace_error(name, line_no, "missing id or token_count");
    TraceEntry e;
    e.id = obj["id"].get<std::int64_t>();
    const auto tokens = obj["token_count"].get<std::int64_t>();
    if (tokens < 0) throw detail::trace_error(name, line_no, "negative token count");
    e.token_count = static_cast<std::size_t>(tokens);
    if (obj.contains("measured_time") && !obj["measured_time"].is_null())
      e.measured_time = obj["measured_time"].get<double>();
    detail::check_entry(e, name, line_no);
    trace.entries.push_back(e);
  }
  if (trace.entries.empty()) throw std::runtime_error(name + ": no trace entries");
  return trace;
}

inline void save_model(const LinearTimeModel& model, std::ostream& out) {  // :182-186
  nlohmann::json obj{{"slope", model.slope}, {"intercept", model.intercept}};
  out << obj.dump(2) << "\n";
}
inline void save_model(const LinearTimeModel& model, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open model file for writing: " + path);
  save_model(model, out);
}
inline LinearTimeModel load_model(std::istream& in) {
  const nlohmann::json obj = nlohmann::json::parse(in);
  return make_linear_time_model(obj.at("slope").get<double>(), obj.at("intercept").get<double>());
}
inline LinearTimeModel load_model(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open model file: " + path);
  return load_model(in);
}
#endif

inline Trace load_trace(const std::string& path, TraceFormat format) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trace file: " + path);
  if (format == TraceFormat::csv) return parse_trace_csv(in, path);
#ifdef BINBATCH_B200_HAS_JSON
  return parse_trace_jsonl(in, path);
#else
  throw std::runtime_error(path + ": JSON-lines traces need nlohmann/json (<json.hpp>)");
#endif
}

// Least squares of measured_time on token_count (workload.hpp:134-160).
inline LinearTimeModel fit_linear_model(const Trace& trace) {
  double sx = 0, sy = 0;
  std::size_t n = 0;
  for (const TraceEntry& e : trace.entries)
    if (e.measured_time) {
      sx += static_cast<double>(e.token_count);
      sy += *e.measured_time;
      ++n;
    }
  if (n < 2) throw std::invalid_argument("fit_linear_model: need at least 2 entries with measured times");
  const double mx = sx / static_cast<double>(n), my = sy / static_cast<double>(n);
  double sxx = 0, sxy = 0;
  for (const TraceEntry& e : trace.entries)
    if (e.measured_time) {
      const double dx = static_cast<double>(e.token_count) - mx;
      sxx += dx * dx;
      sxy += dx * (*e.measured_time - my);
    }
  if (sxx == 0) throw std::invalid_argument("fit_linear_model: all token counts equal, slope undefined");
  const double slope = sxy / sxx;
  return make_linear_time_model(slope, my - slope * mx);
}
inline double tokens_to_time(const LinearTimeModel& model, std::size_t tokens) {  // :162-165
  if (tokens == 0) throw std::invalid_argument("tokens_to_time: token count must be >= 1");
  return model.slope * static_cast<double>(tokens) + model.intercept;
}
inline std::vector<double> service_times(const Trace& trace,
                                         const std::optional<LinearTimeModel>& model = {}) {
  std::vector<double> t;
  t.reserve(trace.entries.size());
  for (const TraceEntry& e : trace.entries) {
    if (model) t.push_back(tokens_to_time(*model, e.token_count));
    else if (e.measured_time) t.push_back(*e.measured_time);
    else
      throw std::invalid_argument(
          "service_times: trace entry lacks measured_time and no time model was given");
  }
  return t;
}

// ---------------------------------------------------------------- experiment.hpp
// ServiceKind adds linear (t = slope * len + intercept, len ~ U[min_time,
// max_time]) and lognormal (exp(mu + sigma Z)) after the reference's kinds.
enum class ServiceKind { uniform, exponential, trace, linear, lognormal };
struct ServiceSpec {
  ServiceKind kind = ServiceKind::uniform;
  double min_time = 1.0;
  double max_time = 2.0;
  double rate = 1.0;
  std::string trace_path;
  TraceFormat trace_format = TraceFormat::csv;
  TraceMode trace_mode = TraceMode::resample;
  std::optional<LinearTimeModel> time_model;  // token counts -> times (experiment.hpp:44)
  std::vector<double> trace_times;  // in-memory resolved service times (instead of trace_path)
  double intercept = 0.5, slope = 0.03;  // linear
  double mu = 0.0, sigma = 1.0;          // lognormal
};
struct BinRule {
  std::size_t k = 1;
  std::vector<double> edges;
};
enum class ErrorKind { perfect, symmetric, confusion };
struct ErrorSpec {
  ErrorKind kind = ErrorKind::perfect;
  double p_error = 0;
  std::string matrix_path;
  std::vector<std::vector<double>> rows;  // in-memory matrix (instead of matrix_path)
};
struct RunTemplate {
  double arrival_rate = kOverload;
  std::size_t n_requests = 0;
  std::size_t batch_size = 1;
  std::size_t n_servers = 1;
  bool flush_partial = true;
  std::optional<double> max_batch_wait;
  ServiceSpec service;
  BinRule bins;
  ErrorSpec error;
};
struct SweepAxis {
  std::string param;
  std::vector<double> values;
};
struct ExperimentSpec {
  std::string name = "experiment";
  RunTemplate base;
  std::vector<SweepAxis> axes;
  std::size_t replications = 10;
  std::string output;
  std::uint64_t seed = 1;
  // The drop-in reproduces the reference's streams unless told otherwise:
  // Rng::reference (bit-exact per replication); Rng::philox selects the fused
  // counter-based kernel (distribution-equal, ~10^3x faster on big sweeps).
  Rng rng = Rng::reference;
};
struct PointResult {
  double arrival_rate = kOverload;
  std::size_t k = 1, batch_size = 1, n_servers = 1;
  std::string error_model = "perfect";
  double p_error = 0;
  std::size_t n_requests = 0, replications = 1;
  double throughput_mean = 0, throughput_std = 0;
  double latency_mean = 0, latency_std = 0;
  double latency_p50 = 0, latency_p99 = 0;
  double makespan_mean = 0, busy_fraction_mean = 0;
  double analytic_throughput = std::numeric_limits<double>::quiet_NaN();
  double analytic_latency = std::numeric_limits<double>::quiet_NaN();
  double analytic_max_throughput = std::numeric_limits<double>::quiet_NaN();
};

inline std::uint64_t replication_seed(std::uint64_t master, std::uint64_t rep) {
  return bb_replication_seed(master, rep);
}

// Files a template references, loaded once per experiment (experiment.hpp:95-108).
struct ResolvedWorkload {
  std::vector<double> trace_times;
  std::optional<ErrorModel> confusion;
};

inline ResolvedWorkload resolve_workload(const RunTemplate& t) {
  ResolvedWorkload w;
  if (t.service.kind == ServiceKind::trace) {
    if (!t.service.trace_times.empty()) w.trace_times = t.service.trace_times;
    else w.trace_times = service_times(load_trace(t.service.trace_path, t.service.trace_format),
                                       t.service.time_model);
  }
  if (t.error.kind == ErrorKind::confusion)
    w.confusion = t.error.rows.empty() ? load_confusion(t.error.matrix_path)
                                       : make_confusion(t.error.rows);
  return w;
}

// The SimConfig of one replication (experiment.hpp:110-155).  The linear and
// log-normal kinds have no reference ServiceDist: those templates run
// through run_point / run_experiment only.
inline SimConfig materialize(const RunTemplate& t, const ResolvedWorkload& w, std::uint64_t seed) {
  SimConfig cfg;
  cfg.arrival_rate = t.arrival_rate;
  cfg.n_requests = t.n_requests;
  cfg.batch_size = t.batch_size;
  cfg.n_servers = t.n_servers;
  cfg.flush_partial = t.flush_partial;
  cfg.max_batch_wait = t.max_batch_wait;
  cfg.seed = seed;
  cfg.trace_mode = t.service.trace_mode;
  switch (t.service.kind) {
    case ServiceKind::uniform: cfg.service = make_uniform(t.service.min_time, t.service.max_time); break;
    case ServiceKind::exponential: cfg.service = make_exponential(t.service.rate); break;
    case ServiceKind::trace: cfg.service = make_empirical(w.trace_times); break;
    default: throw std::logic_error("materialize: the linear / lognormal kinds have no SimConfig form");
  }
  if (!t.bins.edges.empty()) {
    cfg.bins = make_bin_config(t.bins.edges);
  } else if (t.service.kind == ServiceKind::uniform) {
    cfg.bins = uniform_boundaries(t.bins.k, t.service.min_time, t.service.max_time);
  } else if (t.service.kind == ServiceKind::exponential) {
    cfg.bins = exponential_boundaries(t.bins.k, t.service.rate, t.batch_size);
  } else {
    cfg.bins = empirical_boundaries(t.bins.k, w.trace_times);
  }
  switch (t.error.kind) {
    case ErrorKind::perfect: cfg.error_model = Perfect{}; break;
    case ErrorKind::symmetric: cfg.error_model = make_symmetric(t.error.p_error); break;
    case ErrorKind::confusion: cfg.error_model = *w.confusion; break;
  }
  return cfg;
}

// One replication with the reference's streams: bit-exact records (experiment.hpp:157-161).
inline SimResult run_template(const RunTemplate& t, const ResolvedWorkload& w, std::uint64_t seed) {
  const SimConfig cfg = materialize(t, w, seed);
  if (t.service.kind == ServiceKind::trace) return replay_trace_detailed(cfg, w.trace_times);
  return run_simulation_detailed(cfg);
}

namespace detail {
struct TemplateHolder {
  std::vector<double> conf;
  std::vector<double> trace;
};
inline bb_run_template to_c(const RunTemplate& t, const ResolvedWorkload& w, TemplateHolder& h) {
  bb_run_template c{};
  c.arrival_rate = t.arrival_rate;
  c.n_requests = t.n_requests;
  c.batch_size = t.batch_size;
  c.n_servers = t.n_servers;
  c.flush_partial = t.flush_partial;
  c.has_max_batch_wait = t.max_batch_wait.has_value();
  c.max_batch_wait = t.max_batch_wait.value_or(0.0);
  switch (t.service.kind) {
    case ServiceKind::uniform: c.service = BB_KIND_UNIFORM; break;
    case ServiceKind::exponential: c.service = BB_KIND_EXPONENTIAL; break;
    case ServiceKind::trace: c.service = BB_KIND_TRACE; break;
    case ServiceKind::linear: c.service = BB_KIND_LINEAR; break;
    case ServiceKind::lognormal: c.service = BB_KIND_LOGNORMAL; break;
  }
  c.trace_cyclic = t.service.trace_mode == TraceMode::cyclic;
  c.min_time = t.service.min_time;
  c.max_time = t.service.max_time;
  c.rate = t.service.rate;
  c.lin_a = t.service.intercept;
  c.lin_b = t.service.slope;
  c.mu = t.service.mu;
  c.sigma = t.service.sigma;
  h.trace = w.trace_times;
  c.trace_times = h.trace.empty() ? nullptr : h.trace.data();
  c.n_trace = h.trace.size();
  c.k = t.bins.k;
  c.edges = t.bins.edges.empty() ? nullptr : t.bins.edges.data();
  c.n_edges = t.bins.edges.size();
  c.error_kind = t.error.kind == ErrorKind::perfect ? BB_ERR_PERFECT
                 : t.error.kind == ErrorKind::symmetric ? BB_ERR_SYMMETRIC : BB_ERR_CONFUSION;
  c.p_error = t.error.p_error;
  if (t.error.kind == ErrorKind::confusion && w.confusion) {
    const auto& rows = std::get<Confusion>(*w.confusion).rows;
    for (const auto& r : rows) h.conf.insert(h.conf.end(), r.begin(), r.end());
    c.confusion = h.conf.empty() ? nullptr : h.conf.data();
    c.confusion_k = rows.size();
  }
  return c;
}
inline PointResult from_c(const bb_point_result& r) {
  PointResult p;
  p.arrival_rate = r.arrival_rate;
  p.k = r.k;
  p.batch_size = r.batch_size;
  p.n_servers = r.n_servers;
  p.error_model = r.error_kind == BB_ERR_SYMMETRIC ? "symmetric"
                  : r.error_kind == BB_ERR_CONFUSION ? "confusion" : "perfect";
  p.p_error = r.p_error;
  p.n_requests = r.n_requests;
  p.replications = r.replications;
  p.throughput_mean = r.throughput_mean;
  p.throughput_std = r.throughput_std;
  p.latency_mean = r.latency_mean;
  p.latency_std = r.latency_std;
  p.latency_p50 = r.latency_p50;
  p.latency_p99 = r.latency_p99;
  p.makespan_mean = r.makespan_mean;
  p.busy_fraction_mean = r.busy_fraction_mean;
  p.analytic_throughput = r.analytic_throughput;
  p.analytic_latency = r.analytic_latency;
  p.analytic_max_throughput = r.analytic_max_throughput;
  return p;
}
inline int axis_param(const std::string& p) {
  if (p == "lambda") return BB_AXIS_LAMBDA;
  if (p == "k") return BB_AXIS_K;
  if (p == "B") return BB_AXIS_B;
  if (p == "p_e") return BB_AXIS_P_E;
  if (p == "n_servers") return BB_AXIS_N_SERVERS;
  throw std::invalid_argument("unknown sweep parameter: " + p);
}
}  // namespace detail

// experiment.hpp:241-252: axis count, replications, every axis value applicable.
inline void validate_spec(const ExperimentSpec& spec) {
  if (spec.axes.size() > 2) throw std::invalid_argument("experiment spec: at most 2 sweep axes");
  if (spec.replications < 1) throw std::invalid_argument("experiment spec: replications must be >= 1");
  for (const SweepAxis& axis : spec.axes) {
    if (axis.values.empty())
      throw std::invalid_argument("experiment spec: sweep axis '" + axis.param + "' has no values");
    detail::axis_param(axis.param);
  }
  uint64_t n = 0;
  // the per-value override checks (apply_override, experiment.hpp:208-228) run in the library
  bb_experiment_spec e{};
  detail::TemplateHolder h;
  e.base = detail::to_c(spec.base, ResolvedWorkload{}, h);
  std::vector<std::vector<double>> vals;
  for (std::size_t i = 0; i < spec.axes.size(); ++i) {
    vals.push_back(spec.axes[i].values);
    e.axes[i].param = detail::axis_param(spec.axes[i].param);
    e.axes[i].values = vals.back().data();
    e.axes[i].n_values = vals.back().size();
  }
  e.n_axes = spec.axes.size();
  e.replications = spec.replications;
  detail::check(bb_experiment_points(&e, &n));
}

// run_point (experiment.hpp:254-307): R replications with seeds
// replication_seed(master_seed, r), one device launch.  `rng` picks the
// streams (Rng::reference: the reference's own, per replication bit-exact).
inline PointResult run_point(const RunTemplate& t, const ResolvedWorkload& w,
                             std::uint64_t master_seed, std::size_t replications,
                             Rng rng = Rng::reference) {
  detail::TemplateHolder h;
  const bb_run_template c = detail::to_c(t, w, h);
  bb_point_result out{};
  detail::check(bb_run_points(&c, 1, replications, master_seed, static_cast<int32_t>(rng), &out));
  return detail::from_c(out);
}
inline PointResult run_point(const RunTemplate& t, std::uint64_t master_seed, std::size_t replications,
                             Rng rng = Rng::reference) {
  return run_point(t, resolve_workload(t), master_seed, replications, rng);
}

// GPUs the sweeps below spread their replications over in this process (one
// host thread per device, results gathered on devices[0]; repeats allowed);
// empty: the current device.  Results never depend on the list.
inline void set_devices(const std::vector<int>& devices) {
  std::vector<int32_t> d(devices.begin(), devices.end());
  detail::check(bb_set_devices(d.empty() ? nullptr : d.data(), static_cast<uint32_t>(d.size())));
}

// run_experiment (experiment.hpp:312-370): every point x replication in one
// device launch; `jobs` is accepted and never changes results.  A failing
// point throws std::runtime_error("experiment '<name>': sweep point <i> failed: ...").
inline std::vector<PointResult> run_experiment(const ExperimentSpec& spec, unsigned jobs = 1) {
  validate_spec(spec);
  const ResolvedWorkload workload = resolve_workload(spec.base);
  detail::TemplateHolder h;
  bb_experiment_spec e{};
  e.base = detail::to_c(spec.base, workload, h);
  std::vector<std::vector<double>> vals;
  vals.reserve(spec.axes.size());
  for (std::size_t i = 0; i < spec.axes.size(); ++i) {
    vals.push_back(spec.axes[i].values);
    e.axes[i].param = detail::axis_param(spec.axes[i].param);
    e.axes[i].values = vals.back().data();
    e.axes[i].n_values = vals.back().size();
  }
  e.n_axes = spec.axes.size();
  e.replications = spec.replications;
  e.seed = spec.seed;
  e.rng = static_cast<int32_t>(spec.rng);
  e.name = spec.name.c_str();
  uint64_t n = 0;
  detail::check(bb_run_experiment(&e, jobs, nullptr, 0, &n));
  std::vector<bb_point_result> out(n);
  detail::check(bb_run_experiment(&e, jobs, out.data(), n, &n));
  std::vector<PointResult> r;
  r.reserve(out.size());
  for (const auto& p : out) r.push_back(detail::from_c(p));
  return r;
}

// ---------------------------------------------------------------- output formats
// Byte-identical to the reference's writers (a caller diffing files sees no
// change); formatting goes through snprintf: "%.17g" is what an ostream at
// precision 17 prints, "%.10g" the CSV cells.
namespace detail {
inline void put_g(std::string& s, const char* fmt, double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), fmt, v);
  s += buf;
}
inline std::string csv_number(double v) {  // experiment.hpp:374-380: NaN -> empty cell
  if (std::isnan(v)) return {};
  if (std::isinf(v)) return v < 0 ? "-inf" : "inf";
  std::string s;
  put_g(s, "%.10g", v);
  return s;
}
}  // namespace detail

// One JSON object per request (simulator.hpp:359-382); unserved requests
// (flush_partial = false) carry null batch fields.
inline void write_request_log(const SimResult& result, std::ostream& out) {
  std::string line;
  for (const Request& r : result.requests) {
    line.assign("{\"id\":").append(std::to_string(r.id));
    line += ",\"arrival\":";
    detail::put_g(line, "%.17g", r.arrival_time);
    line += ",\"service\":";
    detail::put_g(line, "%.17g", r.service_time);
    line.append(",\"true_bin\":").append(std::to_string(r.true_bin));
    line.append(",\"predicted_bin\":").append(std::to_string(r.predicted_bin));
    if (r.batch == kNoBatch) {
      line += ",\"batch\":null,\"start\":null,\"finish\":null}\n";
    } else {
      const BatchRecord& b = result.batches.at(r.batch);
      line.append(",\"batch\":").append(std::to_string(r.batch)).append(",\"start\":");
      detail::put_g(line, "%.17g", b.start_time);
      line += ",\"finish\":";
      detail::put_g(line, "%.17g", b.finish_time);
      line += "}\n";
    }
    out << line;
  }
}
inline void write_request_log(const SimResult& result, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("cannot open request log for writing: " + path);
  write_request_log(result, f);
}

// Sweep results CSV (experiment.hpp:382-414): one row per point, columns in
// the order below; empty cells for NaN.
namespace detail {
struct CsvColumn {
  const char* name;
  std::string (*cell)(const ExperimentSpec&, const PointResult&);
};
#define BB_NUM_COL(col, field) \
  {col, [](const ExperimentSpec&, const PointResult& r) { return csv_number(r.field); }}
#define BB_INT_COL(col, field) \
  {col, [](const ExperimentSpec&, const PointResult& r) { return std::to_string(r.field); }}
inline const std::vector<CsvColumn>& csv_columns() {
  static const std::vector<CsvColumn> cols = {
      {"name", [](const ExperimentSpec& s, const PointResult&) { return s.name; }},
      BB_NUM_COL("lambda", arrival_rate),
      BB_INT_COL("k", k),
      BB_INT_COL("B", batch_size),
      BB_INT_COL("n_servers", n_servers),
      {"error_model", [](const ExperimentSpec&, const PointResult& r) { return r.error_model; }},
      BB_NUM_COL("p_e", p_error),
      BB_INT_COL("n_requests", n_requests),
      BB_INT_COL("replications", replications),
      {"seed", [](const ExperimentSpec& s, const PointResult&) { return std::to_string(s.seed); }},
      BB_NUM_COL("throughput_mean", throughput_mean),
      BB_NUM_COL("throughput_std", throughput_std),
      BB_NUM_COL("latency_mean", latency_mean),
      BB_NUM_COL("latency_std", latency_std),
      BB_NUM_COL("latency_p50", latency_p50),
      BB_NUM_COL("latency_p99", latency_p99),
      BB_NUM_COL("makespan_mean", makespan_mean),
      BB_NUM_COL("server_busy_fraction", busy_fraction_mean),
      BB_NUM_COL("analytic_throughput", analytic_throughput),
      BB_NUM_COL("analytic_latency", analytic_latency),
      BB_NUM_COL("analytic_cmax", analytic_max_throughput),
  };
  return cols;
}
#undef BB_NUM_COL
#undef BB_INT_COL
}  // namespace detail

inline std::string results_csv_header_string() {
  std::string h;
  for (const auto& c : detail::csv_columns()) h.append(h.empty() ? "" : ",").append(c.name);
  return h;
}
inline const char* results_csv_header() {
  static const std::string h = results_csv_header_string();
  return h.c_str();
}
inline void write_results_csv(const ExperimentSpec& spec, const std::vector<PointResult>& results,
                              std::ostream& out) {
  const auto& cols = detail::csv_columns();
  out << results_csv_header() << '\n';
  for (const PointResult& r : results) {
    std::string row;
    for (std::size_t c = 0; c < cols.size(); ++c) {
      if (c) row += ',';
      row += cols[c].cell(spec, r);
    }
    out << row << '\n';
  }
}
inline void write_results_csv(const ExperimentSpec& spec, const std::vector<PointResult>& results,
                              const std::string& path) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("cannot open results file for writing: " + path);
  write_results_csv(spec, results, f);
}

// ---------------------------------------------------------------- measured vs analytic
// compare_results (experiment.hpp:418-495): every results-CSV row carrying an
// analytic prediction is checked against its measured mean.
struct CompareRow {
  std::size_t csv_line = 0;
  std::string label;
  std::string metric;  // throughput | latency
  double measured = 0;
  double analytic = 0;
  double rel_error = 0;
  bool pass = false;
};
struct CompareReport {
  std::vector<CompareRow> rows;
  std::size_t n_checked = 0;
  std::size_t n_failed = 0;
  bool ok() const { return n_failed == 0 && n_checked > 0; }
};

namespace detail {
inline std::vector<std::string> split_csv_line(const std::string& line) {
  std::vector<std::string> cells;
  std::istringstream in(line);
  std::string cell;
  while (std::getline(in, cell, ',')) cells.push_back(cell);
  return cells;
}
}  // namespace detail

inline CompareReport compare_results(std::istream& in, double tol_throughput = 0.02,
                                     double tol_latency = 0.05) {
  std::string header;
  if (!std::getline(in, header)) throw std::runtime_error("compare: empty results file");
  std::map<std::string, std::size_t> col;
  {
    const auto names = detail::split_csv_line(header);
    for (std::size_t i = 0; i < names.size(); ++i) col[names[i]] = i;
  }
  for (const char* need : {"name", "lambda", "k", "throughput_mean", "latency_mean",
                           "analytic_throughput", "analytic_latency"})
    if (!col.count(need)) throw std::runtime_error(std::string("compare: missing column ") + need);
  CompareReport rep;
  std::string line;
  std::size_t line_no = 1;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty()) continue;
    std::vector<std::string> cells = detail::split_csv_line(line);
    cells.resize(col.size());
    auto cell = [&](const char* name) -> const std::string& { return cells[col.at(name)]; };
    const std::string label = cell("name") + " lambda=" + cell("lambda") + " k=" + cell("k");
    auto check_pair = [&](const char* measured, const char* analytic, const char* metric,
                          double tol) {
      const std::string& a = cell(analytic);
      const std::string& m = cell(measured);
      if (a.empty() || m.empty()) return;
      CompareRow row;
      row.csv_line = line_no;
      row.label = label;
      row.metric = metric;
      row.measured = std::stod(m);
      row.analytic = std::stod(a);
      row.rel_error = std::abs(row.measured - row.analytic) / std::abs(row.analytic);
      row.pass = row.rel_error <= tol;
      ++rep.n_checked;
      if (!row.pass) ++rep.n_failed;
      rep.rows.push_back(std::move(row));
    };
    check_pair("throughput_mean", "analytic_throughput", "throughput", tol_throughput);
    check_pair("latency_mean", "analytic_latency", "latency", tol_latency);
  }
  return rep;
}
inline CompareReport compare_results_file(const std::string& path, double tol_throughput = 0.02,
                                          double tol_latency = 0.05) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open results file: " + path);
  return compare_results(in, tol_throughput, tol_latency);
}

#ifdef BINBATCH_B200_HAS_JSON
// ---------------------------------------------------------------- JSON specs
// parse_run_template / parse_experiment_spec / load_experiment_spec
// (experiment.hpp:497-608): the CLI's `simulate` / `sweep` inputs.
namespace detail {
inline double json_rate(const nlohmann::json& v, const char* what) {
  if (v.is_string()) {
    const std::string s = v.get<std::string>();
    if (s == "inf" || s == "overload") return kOverload;
    throw std::invalid_argument(std::string(what) + ": expected a number, \"inf\" or \"overload\"");
  }
  return v.get<double>();
}
inline ServiceSpec json_service(const nlohmann::json& o) {
  ServiceSpec s;
  const std::string type = o.at("type").get<std::string>();
  if (type == "uniform") {
    s.kind = ServiceKind::uniform;
    s.min_time = o.at("min_time").get<double>();
    s.max_time = o.at("max_time").get<double>();
  } else if (type == "exponential") {
    s.kind = ServiceKind::exponential;
    s.rate = o.at("rate").get<double>();
  } else if (type == "trace") {
    s.kind = ServiceKind::trace;
    s.trace_path = o.at("path").get<std::string>();
    if (o.contains("format"))
      s.trace_format = o["format"].get<std::string>() == "jsonl" ? TraceFormat::jsonl : TraceFormat::csv;
    if (o.contains("mode"))
      s.trace_mode = o["mode"].get<std::string>() == "cyclic" ? TraceMode::cyclic : TraceMode::resample;
    if (o.contains("time_model") && !o["time_model"].is_null())
      s.time_model = make_linear_time_model(o["time_model"].at("slope").get<double>(),
                                            o["time_model"].at("intercept").get<double>());
  } else {
    throw std::invalid_argument("service type must be uniform, exponential or trace");
  }
  return s;
}
}  // namespace detail

inline RunTemplate parse_run_template(const nlohmann::json& o) {
  RunTemplate t;
  t.arrival_rate = detail::json_rate(o.at("lambda"), "lambda");
  t.n_requests = o.at("n_requests").get<std::size_t>();
  t.batch_size = o.at("batch_size").get<std::size_t>();
  if (o.contains("n_servers")) t.n_servers = o["n_servers"].get<std::size_t>();
  if (o.contains("flush_partial")) t.flush_partial = o["flush_partial"].get<bool>();
  if (o.contains("max_batch_wait") && !o["max_batch_wait"].is_null())
    t.max_batch_wait = o["max_batch_wait"].get<double>();
  t.service = detail::json_service(o.at("service"));
  if (o.contains("bins")) {
    const auto& b = o["bins"];
    if (b.contains("edges")) t.bins.edges = b["edges"].get<std::vector<double>>();
    else t.bins.k = b.at("k").get<std::size_t>();
  }
  if (o.contains("error")) {
    const auto& e = o["error"];
    const std::string type = e.at("type").get<std::string>();
    if (type == "perfect") {
      t.error.kind = ErrorKind::perfect;
    } else if (type == "symmetric") {
      t.error.kind = ErrorKind::symmetric;
      t.error.p_error = e.at("p_error").get<double>();
    } else if (type == "confusion") {
      t.error.kind = ErrorKind::confusion;
      t.error.matrix_path = e.at("path").get<std::string>();
    } else {
      throw std::invalid_argument("error type must be perfect, symmetric or confusion");
    }
  }
  return t;
}

inline ExperimentSpec parse_experiment_spec(const nlohmann::json& o) {
  ExperimentSpec spec;
  if (o.contains("name")) spec.name = o["name"].get<std::string>();
  if (o.contains("seed")) spec.seed = o["seed"].get<std::uint64_t>();
  if (o.contains("replications")) spec.replications = o["replications"].get<std::size_t>();
  if (o.contains("output")) spec.output = o["output"].get<std::string>();
  spec.base = parse_run_template(o.at("base"));
  if (o.contains("sweep"))
    for (const auto& ax : o["sweep"])
      spec.axes.push_back(SweepAxis{ax.at("param").get<std::string>(),
                                    ax.at("values").get<std::vector<double>>()});
  validate_spec(spec);
  return spec;
}

inline ExperimentSpec load_experiment_spec(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open experiment spec: " + path);
  nlohmann::json o;
  try {
    o = nlohmann::json::parse(in);
  } catch (const nlohmann::json::exception& e) {
    throw std::runtime_error(path + ": " + e.what());
  }
  return parse_experiment_spec(o);
}
#endif  // BINBATCH_B200_HAS_JSON

}  // namespace binbatch
