// bb_analytics.cpp -- the reference's host-side closed forms and bin helpers
// behind the C ABI (include/binbatch_b200.h): analytics.hpp:55-126,
// service_dist.hpp:82-93 (harmonic_number), binning.hpp:133-144 (assign_bin)
// and the exhaustive boundary oracle binning.hpp:268-351.
//
// None of this is on the simulation hot path -- the reference evaluates it on
// the host once per run (capacities, latency bounds, edge cross-checks) --
// but a drop-in has to export it with the reference's argument checks,
// exception categories and bits: the drop-in tests compile the reference's
// own acceptance suite against include/binbatch_b200/binbatch.hpp.
// Compiled with -ffp-contract=off like the reference's Release build.
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "binbatch_b200.h"

namespace bb {
void set_last_error(const std::string& msg);  // bb_last_error() (bb_host.cpp)
}

namespace {

struct Fail {
  bb_status st;
  std::string msg;
};
[[noreturn]] void fail(bb_status st, const std::string& m) { throw Fail{st, m}; }

template <class F>
bb_status guard(F&& f) {
  try {
    f();
    return BB_OK;
  } catch (const Fail& e) {
    bb::set_last_error(e.msg);
    return e.st;
  }
}

void check_counts(uint64_t B, uint64_t bins) {  // analytics.hpp:42-45
  if (B == 0) fail(BB_EINVAL, "analytics: batch size must be >= 1");
  if (bins == 0) fail(BB_EINVAL, "analytics: bin count must be >= 1");
}
void check_range(double lo, double hi) {  // analytics.hpp:37-40
  if (!(lo >= 0) || !(lo < hi)) fail(BB_EINVAL, "analytics: need 0 <= min_time < max_time");
}

// E[max of B iid U(lo, hi)] = (B hi + lo)/(B + 1)   (service_dist.hpp:74-80)
double expected_max(uint64_t B, double lo, double hi) {
  const double b = (double)B;
  return (b * hi + lo) / (b + 1.0);
}
double midpoint(double lo, double hi) { return (lo + hi) / 2.0; }

// E[batch service] under k equal-mass bins (analytics.hpp:55-62): the batch
// maximum's excess over the mean shrinks by the bin count.
double service_k(uint64_t B, uint64_t k, double lo, double hi) {
  check_counts(B, k);
  check_range(lo, hi);
  const double excess = expected_max(B, lo, hi) - midpoint(lo, hi);
  return midpoint(lo, hi) + excess / (double)k;
}

double capacity(uint64_t B, uint64_t k, double lo, double hi) {  // analytics.hpp:64-69
  return (double)B / service_k(B, k, lo, hi);
}

double ceiling(uint64_t B, double lo, double hi) {  // analytics.hpp:71-77
  check_counts(B, 1);
  check_range(lo, hi);
  return (double)B / midpoint(lo, hi);
}

double harmonic(uint64_t n) {  // service_dist.hpp:82-87: smallest terms first
  if (n == 0) fail(BB_EINVAL, "harmonic_number: n must be >= 1");
  double acc = 0.0;
  for (uint64_t j = n; j >= 1; --j) acc += 1.0 / (double)j;
  return acc;
}

// binning.hpp:61-93 (the L sequence and the optimal exponential edges)
std::vector<double> exp_edges(uint64_t k, double rate, uint64_t B) {
  if (k == 0) fail(BB_EINVAL, "exponential_boundaries: k must be >= 1");
  if (!(rate > 0)) fail(BB_EINVAL, "exponential_boundaries: rate must be positive");
  if (B == 0) fail(BB_EINVAL, "l_sequence: batch size must be >= 1");
  std::vector<double> L;
  if (k > 1) {
    L.push_back(harmonic(B));
    while (L.size() < k - 1) {
      if (!(L.back() > 0)) fail(BB_EDOMAIN, "l_sequence: non-positive term, log undefined");
      L.push_back(1.0 + std::log(L.back()));
    }
  }
  std::vector<double> e(1, 0.0);
  double acc = 0.0;
  for (uint64_t i = 1; i < k; ++i) {
    acc += std::log(L[k - i - 1]);
    e.push_back(acc / rate);
  }
  e.push_back(std::numeric_limits<double>::infinity());
  return e;
}

// Expected-batch-service objectives of the grid search (binning.hpp:287-347).
// Uniform: sum over bins of P(bin) * E[max of B in the bin].
double uniform_objective(const std::vector<double>& e, uint64_t B, double span) {
  double total = 0.0;
  for (size_t i = 1; i < e.size(); ++i)
    total += (e[i] - e[i - 1]) / span * expected_max(B, e[i - 1], e[i]);
  return total;
}
// Exponential: interior bins charged their top edge, the open bin exact.
double exponential_objective(const std::vector<double>& interior, double rate, double hb) {
  double total = 0.0, prev = 0.0;
  for (double edge : interior) {
    total += (std::exp(-rate * prev) - std::exp(-rate * edge)) * edge;
    prev = edge;
  }
  return total + std::exp(-rate * prev) * (prev + hb / rate);
}

}  // namespace

extern "C" {

bb_status bb_harmonic_number(uint64_t n, double* out) {
  return guard([&] { *out = harmonic(n); });
}

bb_status bb_expected_service_time(uint64_t batch_size, uint64_t bins, double min_time,
                                   double max_time, double* out) {
  return guard([&] { *out = service_k(batch_size, bins, min_time, max_time); });
}

bb_status bb_throughput(uint64_t batch_size, uint64_t bins, double min_time, double max_time,
                        double* out) {
  return guard([&] { *out = capacity(batch_size, bins, min_time, max_time); });
}

bb_status bb_max_throughput(uint64_t batch_size, double min_time, double max_time, double* out) {
  return guard([&] { *out = ceiling(batch_size, min_time, max_time); });
}

bb_status bb_min_bins_for_throughput(uint64_t batch_size, double min_time, double max_time,
                                     double epsilon, uint64_t* out) {
  return guard([&] {  // analytics.hpp:79-98
    const double cap = ceiling(batch_size, min_time, max_time);
    if (!(epsilon > 0) || !(epsilon < cap))
      fail(BB_EINVAL, "min_bins_for_throughput: need 0 < epsilon < max throughput");
    const double target = cap - epsilon;
    const double excess = expected_max(batch_size, min_time, max_time) - midpoint(min_time, max_time);
    // throughput(k) >= target  <=>  k >= (cap - eps) * excess / (eps * mid)
    const double need = target * excess / (epsilon * midpoint(min_time, max_time));
    uint64_t k = need < 1.0 ? 1 : (uint64_t)std::ceil(need);
    // pin to the smallest k that reaches the target (the closed form can be
    // one off when it lands on an integer)
    while (k > 1 && capacity(batch_size, k - 1, min_time, max_time) >= target) --k;
    while (capacity(batch_size, k, min_time, max_time) < target) ++k;
    *out = k;
  });
}

bb_status bb_expected_latency(uint64_t batch_size, uint64_t bins, double min_time, double max_time,
                              double arrival_rate, double* out) {
  return guard([&] {  // analytics.hpp:100-108
    if (!(arrival_rate > 0) || !std::isfinite(arrival_rate))
      fail(BB_EINVAL, "expected_latency: arrival rate must be positive and finite");
    const double fill = (double)(batch_size - 1) * (double)bins / (2.0 * arrival_rate);
    *out = service_k(batch_size, bins, min_time, max_time) + fill;
  });
}

bb_status bb_exponential_service_bound(uint64_t batch_size, uint64_t bins, double rate,
                                       double* out) {
  return guard([&] {  // analytics.hpp:110-126
    check_counts(batch_size, bins);
    if (!(rate > 0)) fail(BB_EINVAL, "exponential_service_bound: rate must be positive");
    const std::vector<double> e = exp_edges(bins, rate, batch_size);
    const double hb = harmonic(batch_size);
    double total = 0.0;
    for (uint64_t i = 1; i < bins; ++i)
      total += (std::exp(-rate * e[i - 1]) - std::exp(-rate * e[i])) * e[i];
    const double last = e[bins - 1];
    total += std::exp(-rate * last) * (last + hb / rate);
    *out = total;
  });
}

bb_status bb_assign_bin(const double* edges, uint64_t n_edges, double length, uint64_t* bin) {
  return guard([&] {  // binning.hpp:133-144
    if (!edges || n_edges < 2) fail(BB_EINVAL, "bin config: need at least two edges");
    const double lo = edges[0], hi = edges[n_edges - 1];
    if (!(length >= lo) || !(length <= hi)) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "assign_bin: length %g outside bin support [%g, %g]", length,
                    lo, hi);
      fail(BB_EDOMAIN, buf);
    }
    if (length == hi) {
      *bin = n_edges - 1;
      return;
    }
    // upper_bound: the first edge strictly above `length`
    uint64_t a = 0, b = n_edges;
    while (a < b) {
      const uint64_t m = a + (b - a) / 2;
      if (edges[m] <= length) a = m + 1;
      else b = m;
    }
    *bin = a;
  });
}

bb_status bb_brute_force_boundaries(uint64_t k, int32_t family, double p0, double p1,
                                    uint64_t batch_size, uint64_t grid_points, double* out) {
  return guard([&] {  // binning.hpp:268-351 (test machinery of the reference)
    if (k != 2 && k != 3) fail(BB_EINVAL, "brute_force_boundaries: only k = 2 or 3 supported");
    if (batch_size == 0) fail(BB_EINVAL, "brute_force_boundaries: batch size must be >= 1");
    if (grid_points < k + 1 || grid_points > 400)
      fail(BB_EINVAL, "brute_force_boundaries: grid_points must be in [k+1, 400]");
    // every interior edge set on the grid, in lexicographic order; the first
    // strict minimum wins
    std::vector<std::vector<uint64_t>> grid;
    if (k == 2) {
      for (uint64_t j = 1; j < grid_points; ++j) grid.push_back({j});
    } else {
      for (uint64_t j1 = 1; j1 + 1 < grid_points; ++j1)
        for (uint64_t j2 = j1 + 1; j2 < grid_points; ++j2) grid.push_back({j1, j2});
    }
    std::vector<double> best;
    double best_val = std::numeric_limits<double>::infinity();
    if (family == 0) {  // Uniform(p0 = min_time, p1 = max_time)
      const double lo = p0, hi = p1, span = hi - lo, step = span / (double)grid_points;
      for (const auto& g : grid) {
        std::vector<double> e{lo};
        for (uint64_t j : g) e.push_back(lo + (double)j * step);
        e.push_back(hi);
        const double v = uniform_objective(e, batch_size, span);
        if (v < best_val) best_val = v, best = e;
      }
    } else if (family == 1) {  // Exponential(p0 = rate)
      const double rate = p0, hb = harmonic(batch_size);
      const double step = hb / rate / (double)grid_points;
      for (const auto& g : grid) {
        std::vector<double> interior;
        for (uint64_t j : g) interior.push_back((double)j * step);
        const double v = exponential_objective(interior, rate, hb);
        if (v < best_val) best_val = v, best = interior;
      }
      best.insert(best.begin(), 0.0);
      best.push_back(std::numeric_limits<double>::infinity());
    } else {
      fail(BB_EINVAL, "brute_force_boundaries: unsupported distribution family");
    }
    for (size_t i = 1; i < best.size(); ++i)
      if (!(best[i - 1] < best[i])) fail(BB_EINVAL, "bin config: edges must be strictly increasing");
    for (uint64_t i = 0; i <= k; ++i) out[i] = best[i];
  });
}

}  // extern "C"
