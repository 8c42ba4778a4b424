// The reference's simulator unit tests (proj/tests/test_simulator.cpp) and
// acceptance criteria 1/2/7/8/10 (proj/tests/acceptance.cpp), rewritten
// against the C++ drop-in header: the only change a reference user makes is
// the include (binbatch_b200/binbatch.hpp) and the link line.  (The
// reference's own test programs also run unchanged: tests/cpp/Makefile.)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <string>
#include <vector>

#include "binbatch_b200/binbatch.hpp"

using namespace binbatch;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (cond) ++g_pass;                                                   \
    else {                                                                \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
    }                                                                     \
  } while (0)
#define CHECK_THROWS(expr, Ex)                                            \
  do {                                                                    \
    bool ok_ = false;                                                     \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const Ex&) {                                                 \
      ok_ = true;                                                         \
    } catch (...) {                                                       \
    }                                                                     \
    CHECK(ok_);                                                           \
  } while (0)

static bool approx(double a, double b, double rel) { return std::abs(a - b) <= rel * std::abs(b); }

static SimConfig overload_uniform(std::size_t n, std::size_t batch, std::size_t k, std::uint64_t seed) {
  SimConfig cfg;  // test_simulator.cpp:17-27
  cfg.arrival_rate = kOverload;
  cfg.n_requests = n;
  cfg.batch_size = batch;
  cfg.bins = uniform_boundaries(k, 1.0, 20.0);
  cfg.service = make_uniform(1.0, 20.0);
  cfg.n_servers = 1;
  cfg.seed = seed;
  return cfg;
}

int main() {
  {  // config validation rejects degenerate setups (:31-50)
    CHECK_THROWS(run_simulation(SimConfig{}), std::invalid_argument);
    SimConfig cfg = overload_uniform(100, 8, 2, 1);
    cfg.n_requests = 4;
    CHECK_THROWS(run_simulation(cfg), std::invalid_argument);
    cfg = overload_uniform(100, 8, 2, 1);
    cfg.n_servers = 0;
    CHECK_THROWS(run_simulation(cfg), std::invalid_argument);
    cfg = overload_uniform(100, 8, 2, 1);
    cfg.arrival_rate = 0.0;
    CHECK_THROWS(run_simulation(cfg), std::invalid_argument);
    cfg = overload_uniform(100, 8, 2, 1);
    cfg.max_batch_wait = 0.0;
    CHECK_THROWS(run_simulation(cfg), std::invalid_argument);
    cfg = overload_uniform(100, 8, 2, 1);
    cfg.error_model = make_confusion({{0.9, 0.1}, {0.1, 0.9}});
    bool ok = true;
    try {
      run_simulation(cfg);
    } catch (...) {
      ok = false;
    }
    CHECK(ok);
    cfg.bins = uniform_boundaries(3, 1.0, 20.0);
    CHECK_THROWS(run_simulation(cfg), std::invalid_argument);
  }
  {  // serial single-request batches serve at the mean (:52-58)
    const SimMetrics m = run_simulation(overload_uniform(10000, 1, 1, 99));
    CHECK(m.n_completed == 10000);
    CHECK(approx(m.throughput, 1.0 / 10.5, 0.02));
    CHECK(approx(m.server_busy_fraction, 1.0, 1e-9));
  }
  {  // changing the error model never perturbs arrivals or services (:85-100)
    SimConfig cfg = overload_uniform(800, 16, 4, 2024);
    cfg.arrival_rate = 6.0;
    const SimResult clean = run_simulation_detailed(cfg);
    cfg.error_model = make_symmetric(0.3);
    const SimResult noisy = run_simulation_detailed(cfg);
    std::size_t moved = 0;
    bool same = clean.requests.size() == noisy.requests.size();
    for (std::size_t i = 0; same && i < clean.requests.size(); ++i) {
      same &= clean.requests[i].arrival_time == noisy.requests[i].arrival_time;
      same &= clean.requests[i].service_time == noisy.requests[i].service_time;
      same &= clean.requests[i].true_bin == noisy.requests[i].true_bin;
      moved += clean.requests[i].predicted_bin != noisy.requests[i].predicted_bin;
    }
    CHECK(same);
    CHECK(moved > 0);
  }
  {  // identical configs produce bit-identical results (:102-112)
    SimConfig cfg = overload_uniform(2000, 32, 4, 12345);
    cfg.arrival_rate = 8.0;
    cfg.error_model = make_symmetric(0.1);
    const SimMetrics a = run_simulation(cfg), b = run_simulation(cfg);
    CHECK(a == b);
    cfg.seed = 54321;
    CHECK(!(a == run_simulation(cfg)));
  }
  {  // batch service time is the member maximum (:114-126)
    SimConfig cfg = overload_uniform(500, 8, 2, 3);
    cfg.arrival_rate = 3.0;
    const SimResult r = run_simulation_detailed(cfg);
    bool ok = true;
    for (const BatchRecord& b : r.batches) {
      double expected = 0;
      for (std::size_t id : b.members) expected = std::max(expected, r.requests[id].service_time);
      ok &= std::abs((b.finish_time - b.start_time) - expected) <= 1e-9;
      ok &= b.formed_time <= b.start_time && b.start_time <= b.finish_time;
    }
    CHECK(ok);
  }
  {  // batches start in formation order on a single server (:128-140)
    SimConfig cfg = overload_uniform(1200, 16, 3, 8);
    cfg.arrival_rate = 20.0;
    std::vector<BatchRecord> b = run_simulation_detailed(cfg).batches;
    std::sort(b.begin(), b.end(), [](const BatchRecord& x, const BatchRecord& y) {
      return x.formed_time < y.formed_time;
    });
    bool ok = true;
    double prev = -1.0;
    for (const BatchRecord& x : b) {
      ok &= x.start_time >= prev;
      prev = x.start_time;
    }
    CHECK(ok);
  }
  {  // perfect predictions keep batch members inside their bin (:142-153)
    SimConfig cfg = overload_uniform(2000, 16, 5, 21);
    const SimResult r = run_simulation_detailed(cfg);
    bool ok = true;
    for (const BatchRecord& b : r.batches)
      for (std::size_t id : b.members)
        ok &= r.requests[id].service_time >= cfg.bins.edges[b.bin - 1] &&
              r.requests[id].service_time <= cfg.bins.edges[b.bin];
    CHECK(ok);
  }
  {  // mispredicted requests serve with their true time (:155-175)
    SimConfig cfg = overload_uniform(3000, 16, 4, 33);
    cfg.error_model = make_symmetric(0.4);
    const SimResult r = run_simulation_detailed(cfg);
    std::size_t moved = 0;
    bool ok = true;
    for (const Request& q : r.requests) {
      const long long diff = (long long)q.predicted_bin - (long long)q.true_bin;
      ok &= std::llabs(diff) <= 1;
      moved += diff != 0;
    }
    for (const BatchRecord& b : r.batches)
      for (std::size_t id : b.members) ok &= r.requests[id].predicted_bin == b.bin;
    CHECK(ok);
    CHECK(moved > 0);
  }
  {  // overloaded single server never idles (:177-184)
    const SimResult r = run_simulation_detailed(overload_uniform(5 * 128, 128, 2, 77));
    double total = 0;
    for (const BatchRecord& b : r.batches) total += b.service_time;
    CHECK(approx(r.metrics.makespan, total, 1e-12));
    CHECK(approx(r.metrics.server_busy_fraction, 1.0, 1e-12));
  }
  {  // mean batch service time at one bin matches the order statistic (:186-200)
    const std::size_t batch = 8, nb = 1500;
    const SimResult r = run_simulation_detailed(overload_uniform(batch * nb, batch, 1, 13));
    CHECK(r.batches.size() == nb);
    double sum = 0, sq = 0;
    for (const BatchRecord& b : r.batches) {
      sum += b.service_time;
      sq += b.service_time * b.service_time;
    }
    const double mean = sum / nb;
    const double sd = std::sqrt((sq - nb * mean * mean) / (nb - 1));
    CHECK(std::abs(mean - expected_max_uniform(batch, 1.0, 20.0)) < 3 * sd / std::sqrt((double)nb));
  }
  {  // latency mean dominates the served mean service time (:220-229)
    SimConfig cfg = overload_uniform(2000, 32, 2, 55);
    cfg.arrival_rate = 6.0;
    const SimResult r = run_simulation_detailed(cfg);
    double ms = 0;
    for (const Request& q : r.requests) ms += q.service_time;
    ms /= r.requests.size();
    CHECK(r.metrics.latency_mean >= ms);
    CHECK(r.metrics.latency_p99 >= r.metrics.latency_p50);
  }
  {  // disabling the flush leaves only full batches (:231-242)
    SimConfig cfg = overload_uniform(1000, 16, 3, 9);
    cfg.flush_partial = false;
    const SimResult r = run_simulation_detailed(cfg);
    bool ok = true;
    for (const BatchRecord& b : r.batches) ok &= b.members.size() == 16;
    CHECK(ok);
    CHECK(r.metrics.n_completed == 16 * r.batches.size());
    CHECK(r.metrics.n_completed < 1000);
    std::size_t unserved = 0;
    for (const Request& q : r.requests) unserved += q.batch == kNoBatch;
    CHECK(unserved == 1000 - r.metrics.n_completed);
  }
  {  // service draws outside the bin support are an error (:265-275)
    SimConfig cfg;
    cfg.arrival_rate = kOverload;
    cfg.n_requests = 4;
    cfg.batch_size = 2;
    cfg.bins = make_bin_config({1.0, 3.5, 6.0});
    cfg.seed = 5;
    CHECK_THROWS(replay_trace(cfg, {1.0, 5.0, 2.0, 50.0}), std::domain_error);
    CHECK_THROWS(replay_trace(cfg, {}), std::invalid_argument);
    CHECK_THROWS(replay_trace(cfg, {1.0, -2.0}), std::invalid_argument);
  }
  {  // splitting a two-length trace (:293-311) and the 1/5/2/6 example (:313-328)
    SimConfig cfg;
    cfg.arrival_rate = kOverload;
    cfg.n_requests = 8;
    cfg.batch_size = 2;
    cfg.seed = 1;
    cfg.trace_mode = TraceMode::cyclic;
    cfg.bins = make_bin_config({1.0, 6.0});
    const double mixed = replay_trace(cfg, {1.0, 6.0}).makespan;
    cfg.bins = make_bin_config({1.0, 3.5, 6.0});
    const double split = replay_trace(cfg, {1.0, 6.0}).makespan;
    CHECK(split < mixed);
    CHECK(mixed == 24.0);
    CHECK(split == 14.0);
    cfg.n_requests = 4;
    cfg.seed = 2;
    cfg.bins = make_bin_config({1.0, 6.0});
    CHECK(replay_trace(cfg, {1.0, 5.0, 2.0, 6.0}).makespan == 11.0);
    cfg.bins = make_bin_config({1.0, 3.5, 6.0});
    CHECK(replay_trace(cfg, {1.0, 5.0, 2.0, 6.0}).makespan == 8.0);
  }
  {  // all requests complete and appear in exactly one batch, 2 servers (:60-83)
    SimConfig cfg = overload_uniform(1003, 16, 3, 7);
    cfg.arrival_rate = 5.0;
    cfg.n_servers = 2;
    cfg.flush_partial = true;
    const SimResult result = run_simulation_detailed(cfg);
    CHECK(result.metrics.n_completed == 1003);
    std::set<std::size_t> seen;
    std::size_t total = 0;
    bool sizes_ok = true, complete_ok = true;
    for (const BatchRecord& b : result.batches) {
      total += b.members.size();
      for (const std::size_t id : b.members) seen.insert(id);
      sizes_ok &= b.members.size() <= 16;
    }
    for (const Request& r : result.requests)
      complete_ok &= r.batch != kNoBatch && r.completion_time >= r.arrival_time;
    CHECK(sizes_ok && complete_ok);
    CHECK(total == 1003 && seen.size() == 1003);
    std::size_t batch_sum = 0;
    for (const std::size_t c : result.metrics.per_bin_batch_counts) batch_sum += c;
    CHECK(batch_sum == result.batches.size());
  }
  {  // latency matches the closed form when servers are plentiful (:202-218)
    SimConfig cfg;
    cfg.arrival_rate = 2.0;
    cfg.n_requests = 6400;
    cfg.batch_size = 16;
    cfg.bins = uniform_boundaries(2, 1.0, 20.0);
    cfg.service = make_uniform(1.0, 20.0);
    cfg.n_servers = 500;
    double total = 0;
    for (int rep = 0; rep < 5; ++rep) {
      cfg.seed = 400 + rep;
      total += run_simulation(cfg).latency_mean;
    }
    const double predicted = expected_latency(16, 2, 1.0, 20.0, 2.0);
    CHECK(std::abs(total / 5 - predicted) / predicted < 0.05);
  }
  {  // equal-length traces remove all batching inefficiency, 2 servers (:277-291)
    SimConfig cfg;
    cfg.arrival_rate = kOverload;
    cfg.n_requests = 64;
    cfg.batch_size = 16;
    cfg.bins = make_bin_config({0.5, 1.5});
    cfg.n_servers = 2;
    cfg.seed = 31;
    cfg.trace_mode = TraceMode::cyclic;
    const SimResult result = replay_trace_detailed(cfg, {1.0});
    bool svc_ok = true;
    for (const BatchRecord& b : result.batches) svc_ok &= b.service_time == 1.0;
    CHECK(svc_ok);
    CHECK(approx(result.metrics.makespan, 2.0, 1e-12));
    CHECK(approx(result.metrics.throughput, 64.0 / 2.0, 1e-12));
  }
  {  // a batch-wait cap bounds in-bin waiting (test_simulator.cpp:244-263)
    SimConfig cfg;
    cfg.arrival_rate = 2.0;
    cfg.n_requests = 400;
    cfg.batch_size = 10;
    cfg.bins = uniform_boundaries(4, 1.0, 20.0);
    cfg.service = make_uniform(1.0, 20.0);
    cfg.n_servers = 8;
    cfg.seed = 70;
    cfg.max_batch_wait = 1.5;
    const SimResult result = run_simulation_detailed(cfg);
    CHECK(result.metrics.n_completed == 400);
    bool any_undersized = false, waits_ok = true;
    for (const BatchRecord& b : result.batches) {
      any_undersized = any_undersized || b.members.size() < 10;
      for (const std::size_t id : b.members)
        waits_ok &= b.formed_time - result.requests[id].arrival_time <= 1.5 + 1e-9;
    }
    CHECK(any_undersized);
    CHECK(waits_ok);
  }
  {  // acceptance criteria 1, 2, 7: capacity protocol (B=128, U[1,20], overload, 10 seeds)
    ExperimentSpec spec;
    spec.name = "overload-capacity";
    spec.seed = 1001;
    spec.replications = 10;
    spec.base.arrival_rate = kOverload;
    spec.base.n_requests = 12800;
    spec.base.batch_size = 128;
    spec.base.flush_partial = false;
    spec.base.service = {ServiceKind::uniform, 1.0, 20.0};
    spec.axes = {{"k", {1.0, 2.0, 3.0, 5.0}}};
    spec.rng = Rng::reference;  // the reference's own streams: its published numbers
    const auto pts = run_experiment(spec, 4);
    const double want[] = {6.447, 8.438, 9.392, 10.34};  // proj/test_output.txt:17
    bool ok = pts.size() == 4;
    double prev = 0;
    for (std::size_t i = 0; ok && i < pts.size(); ++i) {
      char buf[32];
      std::snprintf(buf, sizeof buf, "%.4g", pts[i].throughput_mean);
      ok &= std::abs(std::atof(buf) - want[i]) < 1e-9 * want[i] + 1e-12;
      ok &= approx(pts[i].throughput_mean, throughput(128, pts[i].k, 1.0, 20.0), 0.02);
      ok &= pts[i].throughput_mean > prev;
      prev = pts[i].throughput_mean;
    }
    CHECK(ok);
    spec.rng = Rng::philox;  // generated mode: same criteria statistically (2%)
    spec.replications = 200;
    const auto gpts = run_experiment(spec);
    ok = true;
    for (const auto& p : gpts) ok &= approx(p.throughput_mean, throughput(128, p.k, 1.0, 20.0), 0.02);
    CHECK(ok);
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 2 : 0;
}
