// Test driver (test infrastructure): the reference-facing drop-in end to end —
// load_config_file -> run_experiment (shim/sim_gpu.cpp: the B200 DES) ->
// write_outputs (the reference's own writer over the refilled collector).
// tests/test_gpu_reports.py compares the four CSVs with the reference's.
//   usage: run_outputs <config.json> <out_dir>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "sbsim/config.h"
#include "sbsim/simulation.h"

int main(int argc, char** argv) {
  if (argc >= 7 && std::string(argv[1]) == "peak") {  // peak <cfg> slo min max res
    try {
      sbsim::ExperimentConfig cfg = sbsim::load_config_file(argv[2]);
      sbsim::PeakResult r = sbsim::find_peak_qps(cfg, std::atof(argv[3]), std::atof(argv[4]),
                                                 std::atof(argv[5]), std::atof(argv[6]));
      std::printf("peak %.17g %d\n", r.peak_qps, r.attainable ? 1 : 0);
      for (const auto& p : r.probes)
        std::printf("probe %.17g %.17g %llu %d\n", p.rate_qps, p.ttft_mean_s,
                    (unsigned long long)p.window_requests, p.feasible ? 1 : 0);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "run_outputs: %s\n", e.what());
      return 1;
    }
    return 0;
  }
  if (argc < 3) return 2;
  try {
    sbsim::ExperimentConfig cfg = sbsim::load_config_file(argv[1]);
    sbsim::SimulationResult r = sbsim::run_experiment(cfg);
    sbsim::write_outputs(cfg, r, argv[2]);
    std::printf("kv_samples %zu passes %zu dispatches %zu\n", r.metrics.kv_samples().size(),
                r.metrics.pass_samples().size(), r.metrics.dispatch_log().size());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "run_outputs: %s\n", e.what());
    return 1;
  }
  return 0;
}
