// Dev probe: per-call cost of the shim entry points on the GPU.
#include <chrono>
#include <cstdio>
#include "sbsim/config.h"
#include "sbsim/prefill_alloc.h"
#include "sbsim/simulation.h"
using namespace sbsim;
static double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  std::vector<Request> st(6);
  for (int i = 0; i < 6; ++i) { st[i].id = i; st[i].prompt_len = 1 + i % 5; }
  std::vector<Request*> pend{&st[0], &st[1]}, fresh{&st[2], &st[3], &st[4], &st[5]};
  { std::vector<DpPlan> w(3); for (int d = 0; d < 3; ++d) { w[d].dp_index = d; w[d].c_avail = 7; }
    allocate_batch(pend, fresh, w, 2, AllocMode::kBasic); }  // context + module warm-up
  double t0 = now_s();
  int n = 20000;
  for (int k = 0; k < n; ++k) {
    std::vector<DpPlan> dps(3);
    for (int d = 0; d < 3; ++d) { dps[d].dp_index = d; dps[d].c_avail = 7; }
    for (auto& r : st) r.wait_cycles = 0;
    allocate_batch(pend, fresh, dps, 2, AllocMode::kBasic);
  }
  double t1 = now_s();
  std::printf("allocate_batch: %.1f us/call\n", 1e6 * (t1 - t0) / n);
  std::fflush(stdout);
  ExperimentConfig cfg = load_config_file(argv[1]);
  double t2 = now_s();
  SimulationResult r = run_experiment(cfg);
  double t3 = now_s();
  std::printf("run_experiment short_3k: %.3f s, completed %zu ttft %.6f\n", t3 - t2, r.aggregates.completed, r.aggregates.ttft_mean_s);
  std::fflush(stdout);
  cfg.policy = SchedulerPolicy::kImmediate;
  double t4 = now_s();
  PeakResult p = find_peak_qps(cfg, 0.70, 50.0, 900.0, 2.0);
  double t5 = now_s();
  std::printf("find_peak_qps immediate: %.3f s peak %.3f probes %zu\n", t5 - t4, p.peak_qps, p.probes.size());
  std::fflush(stdout);
  cfg.policy = SchedulerPolicy::kSbs;
  t4 = now_s();
  p = find_peak_qps(cfg, 0.58, 50.0, 900.0, 2.0);
  t5 = now_s();
  std::printf("find_peak_qps sbs: %.3f s peak %.3f probes %zu\n", t5 - t4, p.peak_qps, p.probes.size());
  return 0;
}
