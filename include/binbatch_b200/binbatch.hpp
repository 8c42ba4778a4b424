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
// Differences a caller can observe (documented in DESIGN.md):
//   * SimConfig::rng selects the random streams: Rng::reference reproduces the
//     reference's mt19937_64 streams (bit-exact SimResult), Rng::philox (the
//     default for sweeps) draws counter-based streams on the device
//     (distribution-equal; every replication's p50/p99 is exact for its draws).
//   * > 32 bins (single runs), > 64 bins (sweeps), n >= 2^32 and tie groups
//     of equal arrivals in given trace arrays (other than the overload case)
//     throw std::logic_error("...not supported yet").

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <limits>
#include <optional>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "binbatch_b200.h"

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
}  // namespace detail

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
    if (cf->rows.size() == s.bins.bin_count())
      for (const auto& r : cf->rows) h.conf.insert(h.conf.end(), r.begin(), r.end());
    c.confusion = h.conf.empty() ? nullptr : h.conf.data();
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
inline double throughput(std::size_t B, std::size_t k, double lo, double hi) {
  return bb_analytic_throughput(B, k, lo, hi);
}
inline double expected_latency(std::size_t B, std::size_t k, double lo, double hi, double lam) {
  return bb_analytic_latency(B, k, lo, hi, lam);
}

// ---------------------------------------------------------------- experiment.hpp
enum class ServiceKind { uniform, exponential, trace };
struct ServiceSpec {
  ServiceKind kind = ServiceKind::uniform;
  double min_time = 1.0;
  double max_time = 2.0;
  double rate = 1.0;
  std::vector<double> trace_times;  // resolved service times (the reference loads a file)
  TraceMode trace_mode = TraceMode::resample;
};
struct BinRule {
  std::size_t k = 1;
  std::vector<double> edges;
};
enum class ErrorKind { perfect, symmetric, confusion };
struct ErrorSpec {
  ErrorKind kind = ErrorKind::perfect;
  double p_error = 0;
  std::vector<std::vector<double>> rows;
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
  Rng rng = Rng::philox;
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

namespace detail {
struct SpecHolder {
  bb_experiment_spec e{};
  std::vector<double> conf;
  std::vector<std::vector<double>> axis_values;
};
inline bb_run_template to_c(const RunTemplate& t, std::vector<double>& conf) {
  bb_run_template c{};
  c.arrival_rate = t.arrival_rate;
  c.n_requests = t.n_requests;
  c.batch_size = t.batch_size;
  c.n_servers = t.n_servers;
  c.flush_partial = t.flush_partial;
  c.has_max_batch_wait = t.max_batch_wait.has_value();
  c.max_batch_wait = t.max_batch_wait.value_or(0.0);
  c.service = t.service.kind == ServiceKind::uniform ? BB_KIND_UNIFORM
              : t.service.kind == ServiceKind::exponential ? BB_KIND_EXPONENTIAL : BB_KIND_TRACE;
  c.trace_cyclic = t.service.trace_mode == TraceMode::cyclic;
  c.min_time = t.service.min_time;
  c.max_time = t.service.max_time;
  c.rate = t.service.rate;
  c.trace_times = t.service.trace_times.empty() ? nullptr : t.service.trace_times.data();
  c.n_trace = t.service.trace_times.size();
  c.k = t.bins.k;
  c.edges = t.bins.edges.empty() ? nullptr : t.bins.edges.data();
  c.n_edges = t.bins.edges.size();
  c.error_kind = t.error.kind == ErrorKind::perfect ? BB_ERR_PERFECT
                 : t.error.kind == ErrorKind::symmetric ? BB_ERR_SYMMETRIC : BB_ERR_CONFUSION;
  c.p_error = t.error.p_error;
  for (const auto& r : t.error.rows) conf.insert(conf.end(), r.begin(), r.end());
  c.confusion = conf.empty() ? nullptr : conf.data();
  return c;
}
inline int axis_param(const std::string& p) {
  if (p == "lambda") return BB_AXIS_LAMBDA;
  if (p == "k") return BB_AXIS_K;
  if (p == "B") return BB_AXIS_B;
  if (p == "p_e") return BB_AXIS_P_E;
  if (p == "n_servers") return BB_AXIS_N_SERVERS;
  throw std::invalid_argument("unknown sweep parameter: " + p);
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
}  // namespace detail

inline std::vector<PointResult> run_experiment(const ExperimentSpec& spec, unsigned jobs = 1) {
  if (spec.axes.size() > 2) throw std::invalid_argument("experiment spec: at most 2 sweep axes");
  detail::SpecHolder h;
  h.e.base = detail::to_c(spec.base, h.conf);
  h.axis_values.reserve(spec.axes.size());
  for (std::size_t i = 0; i < spec.axes.size(); ++i) {
    h.axis_values.push_back(spec.axes[i].values);
    h.e.axes[i].param = detail::axis_param(spec.axes[i].param);
    h.e.axes[i].values = h.axis_values.back().empty() ? nullptr : h.axis_values.back().data();
    h.e.axes[i].n_values = h.axis_values.back().size();
  }
  h.e.n_axes = spec.axes.size();
  h.e.replications = spec.replications;
  h.e.seed = spec.seed;
  h.e.rng = static_cast<int32_t>(spec.rng);
  uint64_t n = 0;
  detail::check(bb_run_experiment(&h.e, jobs, nullptr, 0, &n));
  std::vector<bb_point_result> out(n);
  detail::check(bb_run_experiment(&h.e, jobs, out.data(), n, &n));
  std::vector<PointResult> r;
  for (const auto& p : out) r.push_back(detail::from_c(p));
  return r;
}

inline PointResult run_point(const RunTemplate& t, std::uint64_t master_seed,
                             std::size_t replications) {
  ExperimentSpec spec;
  spec.base = t;
  spec.replications = replications;
  spec.seed = master_seed;
  return run_experiment(spec).front();
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

}  // namespace binbatch
