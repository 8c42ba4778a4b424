// Output-format parity: the same program is compiled against the reference
// headers (-DBB_AGAINST_REFERENCE, only where /root/reference exists) and
// against this repo's drop-in header; tests/test_cpp_dropin.py diffs the two
// outputs byte for byte. The values exercise NaN/inf cells, integral doubles,
// 17-digit round trips and unserved requests.
#include <cmath>
#include <iostream>
#include <limits>
#include <sstream>

#ifdef BB_AGAINST_REFERENCE
#include <binbatch/experiment.hpp>
#include <binbatch/simulator.hpp>
#else
#include <binbatch_b200/binbatch.hpp>
#endif

int main() {
  using namespace binbatch;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  const double inf = std::numeric_limits<double>::infinity();

  SimResult res;
  const double arrivals[] = {0.0, 0.1 + 0.2, 1.0 / 3.0, 12345.678901234567, 2.0e-310, 7.0};
  const double services[] = {1.0, 20.0, 0.53000000000000003, 31.22, 1e300, 5.5};
  for (std::size_t i = 0; i < 6; ++i) {
    Request r;
    r.id = i;
    r.arrival_time = arrivals[i];
    r.service_time = services[i];
    r.true_bin = 1 + i % 3;
    r.predicted_bin = 1 + (i + 1) % 3;
    r.batch = i < 4 ? i / 2 : kNoBatch;
    res.requests.push_back(r);
  }
  for (std::size_t b = 0; b < 2; ++b) {
    BatchRecord br;
    br.bin = b + 1;
    br.members = {2 * b, 2 * b + 1};
    br.formed_time = arrivals[2 * b + 1];
    br.start_time = b ? 21.000000000000004 : 0.3;
    br.finish_time = br.start_time + services[2 * b + 1];
    res.batches.push_back(br);
  }
  write_request_log(res, std::cout);

  ExperimentSpec spec;
  spec.name = "fmt";
  spec.seed = 18446744073709551615ull;
  std::vector<PointResult> rows(3);
  rows[0].arrival_rate = inf;
  rows[0].k = 16;
  rows[0].batch_size = 32;
  rows[0].throughput_mean = 1.0 / 7.0;
  rows[0].latency_mean = nan;
  rows[1].arrival_rate = 0.95 * 6.447481452557596;
  rows[1].error_model = "symmetric";
  rows[1].p_error = 0.05;
  rows[1].n_requests = 100000;
  rows[1].replications = 10000;
  rows[1].throughput_std = -inf;
  rows[1].latency_p99 = 1e-7;
  rows[1].makespan_mean = 123456789012.5;
  rows[1].busy_fraction_mean = 0.999999999949;
  rows[1].analytic_throughput = 10.347161298408322;
  rows[1].analytic_latency = 26.202713178294573;
  rows[1].analytic_max_throughput = 1e21;
  rows[2].n_servers = 4;
  rows[2].latency_std = 0.0;
  rows[2].latency_p50 = -0.0;
  write_results_csv(spec, rows, std::cout);
  return 0;
}
