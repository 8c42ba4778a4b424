// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver around the UNMODIFIED reference headers
// (/root/reference/proj/include/binbatch/*.hpp, header-only C++20).  Built by
// oracle/Makefile into oracle/_ref/libbbref.so; nothing from the reference is
// copied into this repository -- the headers are #included where they lie.
//
// Uses:
//   * pins the C restatement (oracle/bb_oracle.c) bit-for-bit,
//   * generates the golden fixtures under tests/golden/,
//   * is the CPU reference arm of bench.py (cpu_baseline.kind = "reference").
//
// The two samplers the reference lacks (BASELINE configs 3 and 5: a linear
// tokens->time service and a log-normal service) are injected
// through the reference's own detail::Engine(cfg, sampler) hook
// (simulator.hpp:120-126), drawing from the reference's service stream.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <exception>
#include <fstream>
#include <functional>
#include <json.hpp>
#include <limits>
#include <map>
#include <mutex>
#include <numeric>
#include <optional>
#include <ostream>
#include <queue>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <variant>
#include <vector>

// Given arrival arrays (bbref_run_arrays, below) need the engine's own event
// loop with the arrivals scheduled from the array instead of its Poisson
// stream.  detail::Engine keeps schedule() and its handlers private, so the
// reference headers are read with private access opened (every standard and
// JSON header they use is included above, unaffected).  Nothing in the
// engine is changed: the same handlers run in the same event order.
#define private public
#include "binbatch/binbatch.hpp"
#undef private
#include "bb_oracle.h"

using namespace binbatch;

namespace {
thread_local std::string g_err;

int code_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return BBO_EDOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return BBO_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BBO_ERUNTIME;
  }
  return BBO_ERUNTIME;
}

SimConfig to_sim(const bbo_config* c) {
  SimConfig cfg;
  cfg.arrival_rate = c->arrival_rate;
  cfg.n_requests = c->n_requests;
  cfg.batch_size = c->batch_size;
  cfg.n_servers = c->n_servers;
  cfg.seed = c->seed;
  cfg.flush_partial = c->flush_partial != 0;
  if (c->has_max_batch_wait) cfg.max_batch_wait = c->max_batch_wait;
  if (c->edges && c->n_edges >= 2)
    cfg.bins = make_bin_config(std::vector<double>(c->edges, c->edges + c->n_edges));
  const std::size_t k = c->n_edges ? c->n_edges - 1 : 0;
  switch (c->error_kind) {
    case BBO_ERR_PERFECT: cfg.error_model = Perfect{}; break;
    case BBO_ERR_SYMMETRIC: cfg.error_model = make_symmetric(c->p_error); break;
    case BBO_ERR_CONFUSION: {
      std::vector<std::vector<double>> rows(k, std::vector<double>(k));
      for (std::size_t i = 0; i < k; ++i)
        for (std::size_t j = 0; j < k; ++j) rows[i][j] = c->confusion[i * k + j];
      cfg.error_model = make_confusion(rows);
      break;
    }
  }
  switch (c->service_kind) {
    case BBO_SVC_UNIFORM: cfg.service = make_uniform(c->lo, c->hi); break;
    case BBO_SVC_EXPONENTIAL: cfg.service = make_exponential(c->rate); break;
    case BBO_SVC_EMPIRICAL:
      cfg.service = make_empirical(std::vector<double>(c->table, c->table + c->n_table));
      break;
    case BBO_SVC_TRACE_CYCLIC: cfg.trace_mode = TraceMode::cyclic; break;
    case BBO_SVC_TRACE_RESAMPLE: cfg.trace_mode = TraceMode::resample; break;
    default: break;
  }
  return cfg;
}

SimResult run_one(const bbo_config* c, const SimConfig& cfg) {
  switch (c->service_kind) {
    case BBO_SVC_UNIFORM:
    case BBO_SVC_EXPONENTIAL:
    case BBO_SVC_EMPIRICAL: return run_simulation_detailed(cfg);
    case BBO_SVC_TRACE_CYCLIC:
    case BBO_SVC_TRACE_RESAMPLE:
      return replay_trace_detailed(cfg, std::vector<double>(c->table, c->table + c->n_table));
    case BBO_SVC_LINEAR: {
      const double lo = c->lo, hi = c->hi, a = c->lin_a, b = c->lin_b;
      detail::Engine eng(cfg, [=](std::size_t, RandomStream& rng) {
        const double len = rng.uniform(lo, hi);
        return b * len + a;  // tokens_to_time, workload.hpp:167-170
      });
      return eng.run();
    }
    case BBO_SVC_LOGNORMAL: {
      const double mu = c->mu, sigma = c->sigma;
      detail::Engine eng(cfg, [=](std::size_t, RandomStream& rng) {
        const double u1 = rng.uniform01(), u2 = rng.uniform01();
        const double z = std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(6.283185307179586 * u2);
        return std::exp(mu + sigma * z);
      });
      return eng.run();
    }
  }
  throw std::invalid_argument("ref shim: service kind not expressible through the reference API");
}

void fill(const SimResult& r, std::size_t k, bbo_metrics* m, bbo_detail* d) {
  std::memset(m, 0, sizeof *m);
  m->throughput = r.metrics.throughput;
  m->makespan = r.metrics.makespan;
  m->latency_mean = r.metrics.latency_mean;
  m->latency_p50 = r.metrics.latency_p50;
  m->latency_p99 = r.metrics.latency_p99;
  m->server_busy_fraction = r.metrics.server_busy_fraction;
  m->n_completed = r.metrics.n_completed;
  m->n_batches = r.batches.size();
  if (!d) return;
  for (std::size_t i = 0; i < r.requests.size(); ++i) {
    const Request& q = r.requests[i];
    if (d->req_arrival) d->req_arrival[i] = q.arrival_time;
    if (d->req_service) d->req_service[i] = q.service_time;
    if (d->req_true_bin) d->req_true_bin[i] = static_cast<uint32_t>(q.true_bin);
    if (d->req_pred_bin) d->req_pred_bin[i] = static_cast<uint32_t>(q.predicted_bin);
    if (d->req_batch) d->req_batch[i] = q.batch == kNoBatch ? UINT64_MAX : q.batch;
    if (d->req_completion) d->req_completion[i] = q.completion_time;
  }
  std::size_t off = 0;
  for (std::size_t j = 0; j < r.batches.size(); ++j) {
    const BatchRecord& b = r.batches[j];
    if (d->bat_bin) d->bat_bin[j] = static_cast<uint32_t>(b.bin);
    if (d->bat_size) d->bat_size[j] = b.members.size();
    if (d->bat_first) d->bat_first[j] = off;
    if (d->bat_formed) d->bat_formed[j] = b.formed_time;
    if (d->bat_start) d->bat_start[j] = b.start_time;
    if (d->bat_finish) d->bat_finish[j] = b.finish_time;
    if (d->bat_service) d->bat_service[j] = b.service_time;
    if (d->members)
      for (std::size_t t = 0; t < b.members.size(); ++t) d->members[off + t] = b.members[t];
    off += b.members.size();
  }
  if (d->per_bin_batch_counts)
    for (std::size_t b = 0; b < k; ++b) d->per_bin_batch_counts[b] = r.metrics.per_bin_batch_counts[b];
}
}  // namespace

extern "C" {

const char* bbref_last_error(void) { return g_err.c_str(); }

uint64_t bbref_replication_seed(uint64_t master, uint64_t rep) {
  return replication_seed(master, rep);  // experiment.hpp:90-92
}

void bbref_stream_uniform01(uint64_t seed, uint64_t stream_id, uint64_t n, double* out) {
  RandomStream s = RandomStream::derive(seed, stream_id);  // rng.hpp:33-35
  for (uint64_t i = 0; i < n; ++i) out[i] = s.uniform01();
}

int bbref_assign_bin(const double* edges, uint64_t n_edges, double len, uint32_t* bin) {
  try {
    const BinConfig cfg = make_bin_config(std::vector<double>(edges, edges + n_edges));
    *bin = static_cast<uint32_t>(assign_bin(cfg, len));
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// One run through the reference's public entry points (run_simulation_detailed,
// replay_trace_detailed) or detail::Engine for the injected samplers.
int bbref_run(const bbo_config* c, bbo_metrics* m, bbo_detail* d) {
  try {
    if (c->service_kind == BBO_SVC_ARRAYS)
      throw std::invalid_argument("ref shim: arrays mode has no reference entry point");
    const SimConfig cfg = to_sim(c);
    const SimResult r = run_one(c, cfg);
    fill(r, c->n_edges ? c->n_edges - 1 : 0, m, d);
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// Replications rep0 .. rep0+nrep-1 of one template with seeds
// replication_seed(master, rep) (run_point, experiment.hpp:254-265), spread
// over `threads` std::threads (the reference pool pattern, :342-368, applied
// to replicas).  out[i] = metrics of replication rep0+i.  Returns the
// elapsed wall seconds through *seconds.
int bbref_run_replicas(const bbo_config* c, uint64_t master, uint64_t rep0, uint64_t nrep,
                       int threads, bbo_metrics* out, double* seconds) {
  SimConfig base;
  try {
    base = to_sim(c);
  } catch (...) {
    return code_of(std::current_exception());
  }
  std::atomic<uint64_t> next{0};
  std::atomic<bool> failed{false};
  std::mutex mu;
  std::exception_ptr first;
  const auto t0 = std::chrono::steady_clock::now();
  auto worker = [&] {
    for (uint64_t i = next.fetch_add(1); i < nrep; i = next.fetch_add(1)) {
      if (failed.load()) return;
      try {
        SimConfig cfg = base;
        cfg.seed = replication_seed(master, rep0 + i);
        const SimResult r = run_one(c, cfg);
        fill(r, 0, &out[i], nullptr);
      } catch (...) {
        failed.store(true);
        std::lock_guard<std::mutex> lock(mu);
        if (!first) first = std::current_exception();
        return;
      }
    }
  };
  const int pool = threads < 1 ? 1 : threads;
  std::vector<std::thread> ts;
  for (int j = 1; j < pool; ++j) ts.emplace_back(worker);
  worker();
  for (auto& t : ts) t.join();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (first) return code_of(first);
  return BBO_OK;
}

// run_point (experiment.hpp:254-307) of the template the config describes:
// service uniform / exponential / trace (table = the resolved trace times,
// ResolvedWorkload, :95-108), bins from `edges` when given, else the rule's
// k (derived edges, :128-146).  out[] = the PointResult numbers in
// declaration order: throughput_mean, throughput_std, latency_mean,
// latency_std, latency_p50, latency_p99, makespan_mean, busy_fraction_mean,
// analytic_throughput, analytic_latency, analytic_max_throughput.
int bbref_run_point(const bbo_config* c, uint64_t k, uint64_t master, uint64_t reps, double* out) {
  try {
    RunTemplate t;
    ResolvedWorkload w;
    t.arrival_rate = c->arrival_rate;
    t.n_requests = c->n_requests;
    t.batch_size = c->batch_size;
    t.n_servers = c->n_servers;
    t.flush_partial = c->flush_partial != 0;
    if (c->has_max_batch_wait) t.max_batch_wait = c->max_batch_wait;
    switch (c->service_kind) {
      case BBO_SVC_UNIFORM:
        t.service.kind = ServiceKind::uniform;
        t.service.min_time = c->lo;
        t.service.max_time = c->hi;
        break;
      case BBO_SVC_EXPONENTIAL:
        t.service.kind = ServiceKind::exponential;
        t.service.rate = c->rate;
        break;
      case BBO_SVC_TRACE_CYCLIC:
      case BBO_SVC_TRACE_RESAMPLE:
        t.service.kind = ServiceKind::trace;
        t.service.trace_mode =
            c->service_kind == BBO_SVC_TRACE_CYCLIC ? TraceMode::cyclic : TraceMode::resample;
        w.trace_times.assign(c->table, c->table + c->n_table);
        break;
      default:
        throw std::invalid_argument("ref shim: run_point needs a uniform, exponential or trace service");
    }
    if (c->edges && c->n_edges >= 2) t.bins.edges.assign(c->edges, c->edges + c->n_edges);
    else t.bins.k = k;
    const std::size_t kk = t.bins.edges.empty() ? k : t.bins.edges.size() - 1;
    switch (c->error_kind) {
      case BBO_ERR_PERFECT: t.error.kind = ErrorKind::perfect; break;
      case BBO_ERR_SYMMETRIC:
        t.error.kind = ErrorKind::symmetric;
        t.error.p_error = c->p_error;
        break;
      case BBO_ERR_CONFUSION: {
        t.error.kind = ErrorKind::confusion;
        std::vector<std::vector<double>> rows(kk, std::vector<double>(kk));
        for (std::size_t i = 0; i < kk; ++i)
          for (std::size_t j = 0; j < kk; ++j) rows[i][j] = c->confusion[i * kk + j];
        w.confusion = make_confusion(rows);
        break;
      }
    }
    const PointResult r = run_point(t, w, master, reps);
    const double v[] = {r.throughput_mean, r.throughput_std, r.latency_mean, r.latency_std,
                        r.latency_p50, r.latency_p99, r.makespan_mean, r.busy_fraction_mean,
                        r.analytic_throughput, r.analytic_latency, r.analytic_max_throughput};
    std::memcpy(out, v, sizeof v);
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// The reference engine on GIVEN arrival times and service times
// (non-decreasing arrivals, e.g. quantised ones with tie groups of any size):
// Engine::run (simulator.hpp:128-150) with schedule_arrivals (:174-185)
// replaced by scheduling arrival i at arrivals[i]; services come through the
// engine's sampler hook (:120-126); predicted bins from the error model on
// the seed's stream 2, exactly as in a generated run.
int bbref_run_arrays(const bbo_config* c, const double* arrivals, const double* services,
                     bbo_metrics* m, bbo_detail* d) {
  try {
    SimConfig cfg = to_sim(c);
    detail::Engine e(cfg, [services](std::size_t id, RandomStream&) { return services[id]; });
    e.validate();
    const std::size_t k = e.cfg_.bins.bin_count();
    e.bin_queues_.assign(k + 1, {});
    e.batch_counts_.assign(k, 0);
    e.requests_.reserve(cfg.n_requests);
    e.idle_servers_ = cfg.n_servers;
    for (std::size_t i = 0; i < cfg.n_requests; ++i) e.schedule(arrivals[i], detail::EventKind::arrival, i);
    while (!e.events_.empty()) {
      const detail::Event ev = e.events_.top();
      e.events_.pop();
      e.now_ = ev.time;
      switch (ev.kind) {
        case detail::EventKind::batch_done: e.on_batch_done(ev.a); break;
        case detail::EventKind::arrival: e.on_arrival(ev.a); break;
        case detail::EventKind::formation: e.on_formation(ev.a); break;
        case detail::EventKind::flush_timer: e.on_flush_timer(ev.a, ev.b); break;
        case detail::EventKind::drain_bin: e.on_drain(ev.a); break;
      }
    }
    const SimResult r = e.finish();
    fill(r, k, m, d);
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// Closed forms (analytics.hpp), for the generated-mode parity tests.
double bbref_throughput(uint64_t B, uint64_t k, double lo, double hi) { return throughput(B, k, lo, hi); }
double bbref_expected_latency(uint64_t B, uint64_t k, double lo, double hi, double lam) {
  return expected_latency(B, k, lo, hi, lam);
}
double bbref_expected_max_uniform(uint64_t B, double lo, double hi) {
  return expected_max_uniform(B, lo, hi);
}

// Boundary constructors (binning.hpp:47-128) -- host-side edge formulas.
int bbref_uniform_boundaries(uint64_t k, double lo, double hi, double* out) {
  try {
    const BinConfig b = uniform_boundaries(k, lo, hi);
    std::memcpy(out, b.edges.data(), b.edges.size() * sizeof(double));
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int bbref_exponential_boundaries(uint64_t k, double rate, uint64_t B, double* out) {
  try {
    const BinConfig b = exponential_boundaries(k, rate, B);
    std::memcpy(out, b.edges.data(), b.edges.size() * sizeof(double));
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int bbref_empirical_boundaries(uint64_t k, const double* s, uint64_t n, double* out) {
  try {
    const BinConfig b = empirical_boundaries(k, std::vector<double>(s, s + n));
    std::memcpy(out, b.edges.data(), b.edges.size() * sizeof(double));
    return BBO_OK;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

}  // extern "C"
