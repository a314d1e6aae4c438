// Drop-in replacement for the reference's simulation.cpp (proj/src), built
// against the reference's own headers.  run_experiment (simulation.h:33) runs
// the replica on the B200 through the C-ABI (sbs_sim_*), and find_peak_qps
// (simulation.h:66-67) evaluates the bisection tree of candidate rates five
// levels at a time as multi-replica launches and replays the reference's
// sequential search over those results — same probes, same peak.
//
// SimulationResult.metrics is refilled from the GPU run records through the
// collector's public record_* methods (dispatch log, passes, control samples,
// decode steps, and record_kv with the per-unit KV loads of every decode step,
// SBS_FLAG_KV_LOADS), so write_outputs produces the reference's four CSVs.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <map>
#include <stdexcept>
#include <thread>
#include <tuple>
#include <vector>

#include "sbs_b200.h"
#include "sbsim/simulation.h"
#include "sbsim/workload.h"

namespace sbsim {
namespace {

void throw_rc(int rc) {
  if (rc == SBS_OK) return;
  if (rc == SBS_ERR_CONFIG) throw ConfigError(sbs_last_error());
  if (rc == SBS_ERR_INVARIANT) throw std::logic_error(sbs_last_error());
  throw std::runtime_error(std::string("sbs_b200: ") + sbs_last_error());
}

sbs_length_spec to_c(const LengthSpec& s) {
  sbs_length_spec o{};
  o.dist = s.dist == LengthDist::kConstant ? SBS_LEN_CONSTANT
         : s.dist == LengthDist::kUniformInt ? SBS_LEN_UNIFORM : SBS_LEN_LOGNORMAL;
  o.value = s.value;
  o.min = s.min;
  o.max = s.max;
  o.mu = s.mu;
  o.sigma = s.sigma;
  return o;
}

// ExperimentConfig (config.h:66-75) -> sbs_experiment; fault arrays owned by `h`.
struct CExp {
  sbs_experiment x{};
  std::vector<int64_t> probes;
  std::vector<sbs_drop_fault> drops;
  std::vector<sbs_dead_fault> deads;
  std::vector<sbs_topology_fault> topo;
};

CExp to_c(const ExperimentConfig& cfg) {
  CExp h;
  const ClusterConfig& c = cfg.cluster;
  sbs_cluster& o = h.x.cluster;
  o.n_instances_prefill = c.n_instances_prefill;
  o.n_instances_decode = c.n_instances_decode;
  o.dp_degree = c.dp_degree;
  o.dp_degree_decode = c.dp_degree_decode;
  o.c_chunk = c.c_chunk;
  o.t_default_s = c.t_default_s;
  o.w_size = static_cast<int64_t>(c.w_size);
  o.l_net_s = c.l_net_s;
  o.n_limit = c.n_limit;
  o.decode_max_batch_per_dp = c.decode_max_batch_per_dp;
  o.iqr_k = c.iqr_k;
  o.watchdog_multiplier = c.watchdog_multiplier;
  o.prefill_base_s = c.engine.prefill_base_s;
  o.prefill_per_token_s = c.engine.prefill_per_token_s;
  o.decode_base_s = c.engine.decode_base_s;
  o.decode_per_request_s = c.engine.decode_per_request_s;
  o.decode_per_kv_token_s = c.engine.decode_per_kv_token_s;
  o.decode_tokens_per_step = c.decode_tokens_per_step;
  o.cache_enabled = c.cache.enabled ? 1 : 0;
  h.probes.assign(c.cache.probe_lens.begin(), c.cache.probe_lens.end());
  o.cache_n_probes = (int32_t)h.probes.size();
  o.cache_budget_tokens = c.cache.budget_tokens;
  const WorkloadSpec& w = cfg.workload;
  sbs_workload& ow = h.x.workload;
  ow.process = w.process == ArrivalProcess::kPoisson ? SBS_ARRIVAL_POISSON
             : w.process == ArrivalProcess::kUniform ? SBS_ARRIVAL_UNIFORM
                                                     : SBS_ARRIVAL_UNIFORM_JITTER;
  ow.initial_burst = w.initial_burst;
  ow.rate_qps = w.rate_qps;
  ow.duration_s = w.duration_s;
  ow.prompt = to_c(w.prompt);
  ow.output = to_c(w.output);
  ow.shared_prefix_fraction = w.shared_prefix_fraction;
  ow.prefix_pool = w.prefix_pool;
  ow.prefix_len = w.prefix_len;
  h.x.policy = cfg.policy == SchedulerPolicy::kSbs ? SBS_POLICY_SBS
             : cfg.policy == SchedulerPolicy::kImmediate ? SBS_POLICY_IMMEDIATE
             : cfg.policy == SchedulerPolicy::kRoundRobin ? SBS_POLICY_ROUND_ROBIN
                                                           : SBS_POLICY_LEAST_OUTSTANDING;
  h.x.prefill_mode = cfg.prefill_mode == AllocMode::kBasic ? SBS_ALLOC_BASIC : SBS_ALLOC_CACHE_AWARE;
  h.x.decode_policy = cfg.decode_policy == DecodePolicy::kIqr ? SBS_DECODE_IQR
                    : cfg.decode_policy == DecodePolicy::kRandom ? SBS_DECODE_RANDOM
                                                                 : SBS_DECODE_ROUND_ROBIN;
  h.x.seed = cfg.sim.seed;
  h.x.warmup_fraction = cfg.sim.warmup_fraction;
  for (const auto& f : cfg.faults.drop_end_forward) h.drops.push_back({f.instance, 0, f.from_s, f.until_s});
  for (const auto& f : cfg.faults.dead) h.deads.push_back({f.instance, 0, f.time_s});
  for (const auto& f : cfg.faults.topology) h.topo.push_back({f.instance, f.healthy ? 1 : 0, f.time_s});
  h.x.drops = h.drops.data();
  h.x.n_drops = (int32_t)h.drops.size();
  h.x.deads = h.deads.data();
  h.x.n_deads = (int32_t)h.deads.size();
  h.x.topology = h.topo.data();
  h.x.n_topology = (int32_t)h.topo.size();
  h.x.cluster.cache_probe_lens = h.probes.empty() ? nullptr : h.probes.data();
  return h;
}

struct CTrace {
  std::vector<int64_t> arr;
  std::vector<int32_t> prompt, output, pool, psize;
  uint64_t digest = 0;
  sbs_trace view() const {
    return sbs_trace{arr.data(), prompt.data(), output.data(), (int64_t)arr.size(), digest,
                     pool.empty() ? nullptr : pool.data(), psize.empty() ? nullptr : psize.data()};
  }
};

CTrace make_trace(const sbs_experiment& x) {
  CTrace t;
  int64_t n = 0;
  throw_rc(sbs_generate_workload(&x.workload, x.seed, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                 &n, &t.digest));
  const bool pfx = x.workload.shared_prefix_fraction > 0;
  t.arr.resize((size_t)std::max<int64_t>(n, 1));
  t.prompt.resize(t.arr.size());
  t.output.resize(t.arr.size());
  if (pfx) {
    t.pool.resize(t.arr.size());
    t.psize.resize(t.arr.size());
  }
  throw_rc(sbs_generate_workload(&x.workload, x.seed, t.arr.data(), t.prompt.data(),
                                 t.output.data(), pfx ? t.pool.data() : nullptr,
                                 pfx ? t.psize.data() : nullptr, n, &n, &t.digest));
  t.arr.resize((size_t)n);
  t.prompt.resize((size_t)n);
  t.output.resize((size_t)n);
  if (pfx) {
    t.pool.resize((size_t)n);
    t.psize.resize((size_t)n);
  }
  return t;
}

Aggregates to_agg(const sbs_aggregates& a) {
  Aggregates g;
  g.generated = a.generated;
  g.completed = a.completed;
  g.throttled = a.throttled;
  g.in_flight = a.in_flight;
  g.window_requests = a.window_requests;
  g.ttft_mean_s = a.ttft_mean_s;
  g.ttft_p50_s = a.ttft_p50_s;
  g.ttft_p95_s = a.ttft_p95_s;
  g.scheduler_wait_mean_s = a.scheduler_wait_mean_s;
  g.device_wait_mean_s = a.device_wait_mean_s;
  g.total_wait_mean_s = a.total_wait_mean_s;
  g.passes = a.passes;
  g.chunk_util_mean = a.chunk_util_mean;
  g.decode_steps = a.decode_steps;
  g.output_tokens = a.output_tokens;
  g.output_tokens_per_s = a.output_tokens_per_s;
  g.kv_mean_time_avg = a.kv_mean_time_avg;
  g.kv_sigma_time_avg = a.kv_sigma_time_avg;
  g.completed_per_s = a.completed_per_s;
  g.watchdog_fires = a.watchdog_fires;
  g.dropped_end_forwards = a.dropped_end_forwards;
  g.rejected_samples = a.rejected_samples;
  g.deferrals = a.deferrals;
  g.flow_control_events = a.flow_control_events;
  g.mask_events = a.mask_events;
  g.fallback_events = a.fallback_events;
  g.warmup_cutoff_s = a.warmup_cutoff_s;
  g.duration_s = a.duration_s;
  return g;
}

// Many configs, one launch (one warp per replica).  Errors stay per config:
// err[i] is the SBS_* code of config i (its trace generation or its replica),
// msg[i] the message; the caller raises only for the configs it consumes.
struct ManyResult {
  std::vector<sbs_aggregates> agg;
  std::vector<int> err;
  std::vector<std::string> msg;
};

ManyResult run_many(const std::vector<ExperimentConfig>& cfgs) {
  ManyResult out;
  const size_t n = cfgs.size();
  out.agg.assign(n, sbs_aggregates{});
  out.err.assign(n, SBS_OK);
  out.msg.assign(n, std::string());
  std::vector<CExp> xs(n);
  std::vector<CTrace> tr(n);
  for (size_t i = 0; i < n; ++i) {
    try {
      validate(cfgs[i].cluster);
      xs[i] = to_c(cfgs[i]);
    } catch (const ConfigError& e) {
      out.err[i] = SBS_ERR_CONFIG;
      out.msg[i] = e.what();
    }
  }
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i; (i = next.fetch_add(1)) < n;) {
      if (out.err[i]) continue;
      int64_t cnt = 0;
      uint64_t dg = 0;
      int rc = sbs_generate_workload(&xs[i].x.workload, xs[i].x.seed, nullptr, nullptr, nullptr,
                                     nullptr, nullptr, 0, &cnt, &dg);
      if (rc != SBS_OK) {
        out.err[i] = rc;
        out.msg[i] = sbs_last_error();
        continue;
      }
      try {
        tr[i] = make_trace(xs[i].x);
      } catch (const std::exception& e) {
        out.err[i] = SBS_ERR_CONFIG;
        out.msg[i] = e.what();
      }
    }
  };
  std::vector<std::thread> pool;
  unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), (unsigned)n));
  for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work);
  for (auto& t : pool) t.join();
  std::vector<size_t> live;
  std::vector<sbs_experiment> px;
  std::vector<sbs_trace> pt;
  for (size_t i = 0; i < n; ++i) {
    if (out.err[i]) continue;
    live.push_back(i);
    px.push_back(xs[i].x);
    pt.push_back(tr[i].view());
  }
  if (px.empty()) return out;
  sbs_sim* sim = nullptr;
  int rc = sbs_sim_create(px.data(), (int32_t)px.size(), pt.data(), (int32_t)pt.size(), nullptr, 0, 0,
                          &sim);
  if (rc != SBS_OK) {  // a create failure is not attributable to one config
    for (size_t i : live) {
      out.err[i] = rc;
      out.msg[i] = sbs_last_error();
    }
    return out;
  }
  std::vector<sbs_aggregates> agg(px.size());
  rc = sbs_sim_launch(sim, nullptr);
  if (rc == SBS_OK) rc = sbs_sim_results(sim, agg.data(), nullptr, nullptr);
  const std::string m = sbs_last_error();
  sbs_sim_destroy(sim);
  for (size_t k = 0; k < live.size(); ++k) {
    const size_t i = live[k];
    out.agg[i] = agg[k];
    if (agg[k].error) {
      out.err[i] = agg[k].error;
      out.msg[i] = "replica failed with code " + std::to_string(agg[k].error);
    } else if (rc != SBS_OK && rc != agg[k].error) {
      // launch-level failure (CUDA error): every replica of the launch failed
      bool any = false;
      for (auto& a : agg) any |= a.error != 0;
      if (!any) {
        out.err[i] = rc;
        out.msg[i] = m;
      }
    }
  }
  return out;
}

}  // namespace

SimulationResult run_experiment(const ExperimentConfig& config) {
  validate(config.cluster);
  CExp x = to_c(config);
  CTrace tr = make_trace(x.x);
  sbs_trace tv = tr.view();
  sbs_sim* sim = nullptr;
  throw_rc(sbs_sim_create(&x.x, 1, &tv, 1, nullptr,
                          SBS_FLAG_PER_REQUEST | SBS_FLAG_LOGS | SBS_FLAG_KV_LOADS, 0, &sim));
  struct Guard {
    sbs_sim* s;
    ~Guard() { sbs_sim_destroy(s); }
  } guard{sim};
  sbs_aggregates agg{};
  throw_rc(sbs_sim_launch(sim, nullptr));
  throw_rc(sbs_sim_results(sim, &agg, nullptr, nullptr));
  const size_t n = tr.arr.size();
  std::vector<int64_t> disp(n), ps(n), ft(n), comp(n);
  std::vector<int8_t> st(n);
  if (n) throw_rc(sbs_sim_requests(sim, 0, disp.data(), ps.data(), ft.data(), comp.data(), st.data()));
  int64_t nw = 0;
  throw_rc(sbs_sim_log(sim, 0, nullptr, 0, &nw));
  std::vector<int64_t> log((size_t)std::max<int64_t>(nw, 1));
  throw_rc(sbs_sim_log(sim, 0, log.data(), nw, &nw));

  SimulationResult res;
  res.aggregates = to_agg(agg);
  res.workload_digest = tr.digest;
  res.horizon = seconds_to_ns(config.workload.duration_s);
  res.requests.resize(n);
  auto opt = [](int64_t v) { return v < 0 ? std::optional<TimeNs>() : std::optional<TimeNs>(v); };
  for (size_t i = 0; i < n; ++i) {
    Request& r = res.requests[i];
    r.id = i;
    r.arrival_time = tr.arr[i];
    r.prompt_len = tr.prompt[i];
    r.output_len = tr.output[i];
    r.status = static_cast<RequestStatus>(st[i]);
    r.dispatch_time = opt(disp[i]);
    r.prefill_start = opt(ps[i]);
    r.first_token_time = opt(ft[i]);
    r.completion_time = opt(comp[i]);
    if (r.dispatch_time) r.compute_total = std::max<Tokens>(1, r.prompt_len);
    if (r.first_token_time) r.compute_done = r.compute_total;
    if (r.status == RequestStatus::kCompleted) r.decode_done = r.decode_target();
  }
  // run records -> collector (public API)
  for (int64_t i = 0; i < nw;) {
    const int kind = (int)(log[(size_t)i] & 0xff);
    const int64_t len = log[(size_t)i] >> 8;
    const int64_t* p = log.data() + i + 1;
    if (kind == 1) {
      res.metrics.record_dispatch(p[0], (int)p[1]);
    } else if (kind == 2) {
      SchedulerState s;
      s.i_opt = p[1];
      s.t_fwd_bar = p[2];
      s.n_active = (int)p[3];
      res.metrics.record_control(p[0], s);
    } else if (kind == 3) {
      PassBegin b;
      b.time = p[0];
      b.instance_id = (int)p[1];
      b.dp_assigned.assign(p + 2, p + len);
      res.metrics.record_pass(b, config.cluster.c_chunk);
    } else if (kind == 4) {
      res.metrics.record_step(p[0], p[1]);
    } else if (kind == 6) {  // record_kv_snapshot (simulation.cpp:486-495)
      res.metrics.record_kv(p[0], std::span<const Tokens>(p + 1, (size_t)(len - 1)));
    }
    i += 1 + len;
  }
  return res;
}

nlohmann::ordered_json aggregates_json(const Aggregates& a) {
  nlohmann::ordered_json o;
  o["generated"] = a.generated; o["completed"] = a.completed; o["throttled"] = a.throttled;
  o["in_flight"] = a.in_flight; o["window_requests"] = a.window_requests;
  o["ttft_mean_s"] = a.ttft_mean_s; o["ttft_p50_s"] = a.ttft_p50_s; o["ttft_p95_s"] = a.ttft_p95_s;
  o["scheduler_wait_mean_s"] = a.scheduler_wait_mean_s;
  o["device_wait_mean_s"] = a.device_wait_mean_s; o["total_wait_mean_s"] = a.total_wait_mean_s;
  o["passes"] = a.passes; o["chunk_util_mean"] = a.chunk_util_mean;
  o["decode_steps"] = a.decode_steps; o["output_tokens"] = a.output_tokens;
  o["output_tokens_per_s"] = a.output_tokens_per_s; o["kv_mean_time_avg"] = a.kv_mean_time_avg;
  o["kv_sigma_time_avg"] = a.kv_sigma_time_avg; o["completed_per_s"] = a.completed_per_s;
  o["watchdog_fires"] = a.watchdog_fires; o["dropped_end_forwards"] = a.dropped_end_forwards;
  o["rejected_samples"] = a.rejected_samples; o["deferrals"] = a.deferrals;
  o["flow_control_events"] = a.flow_control_events; o["mask_events"] = a.mask_events;
  o["fallback_events"] = a.fallback_events; o["warmup_cutoff_s"] = a.warmup_cutoff_s;
  o["duration_s"] = a.duration_s;
  return o;
}

nlohmann::ordered_json summary_json(const ExperimentConfig& config, const SimulationResult& r) {
  nlohmann::ordered_json o;
  o["config"] = resolved_json(config);
  o["workload_digest"] = digest_hex(r.workload_digest);
  o["aggregates"] = aggregates_json(r.aggregates);
  return o;
}

void write_outputs(const ExperimentConfig& config, const SimulationResult& result,
                   const std::string& out_dir) {
  namespace fs = std::filesystem;
  fs::create_directories(out_dir);
  auto put = [&](const char* name, const std::string& text) {
    std::ofstream f(fs::path(out_dir) / name, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("cannot write ") + name);
    f << text;
  };
  put("requests.csv", MetricsCollector::requests_csv(result.requests));
  put("passes.csv", result.metrics.passes_csv());
  put("kvband.csv", result.metrics.kvband_csv());
  put("control.csv", result.metrics.control_csv());
  put("summary.json", summary_json(config, result).dump(2) + "\n");
}

PeakResult find_peak_qps(const ExperimentConfig& base, double slo_ttft_s, double rate_min,
                         double rate_max, double resolution) {
  if (slo_ttft_s <= 0) throw ConfigError("peak: slo_ttft must be > 0");
  if (rate_min <= 0 || rate_max < rate_min || resolution <= 0)
    throw ConfigError("peak: invalid rate search bounds");
  // Speculative batches: every launch evaluates the next kLevels levels of
  // the bisection tree under the current interval (2^kLevels - 1 midpoints,
  // plus both ends in the first launch); the reference's sequential search
  // (simulation.cpp:608-644) is then replayed over the results, launching the
  // next subtree only when the path leaves the evaluated one.  An error is
  // raised only for a probe the sequential search actually makes.
  constexpr int kLevels = 5;
  std::map<double, std::pair<sbs_aggregates, std::pair<int, std::string>>> done;
  auto evaluate = [&](std::vector<double> rates) {
    std::vector<ExperimentConfig> cfgs;
    std::vector<double> todo;
    std::sort(rates.begin(), rates.end());
    rates.erase(std::unique(rates.begin(), rates.end()), rates.end());
    for (double r : rates)
      if (!done.count(r)) {
        ExperimentConfig c = base;
        c.workload.rate_qps = r;
        cfgs.push_back(c);
        todo.push_back(r);
      }
    if (cfgs.empty()) return;
    ManyResult m = run_many(cfgs);
    for (size_t i = 0; i < todo.size(); ++i)
      done.emplace(todo[i], std::make_pair(m.agg[i], std::make_pair(m.err[i], m.msg[i])));
  };
  auto subtree = [&](double lo, double hi, std::vector<double>& out) {
    std::vector<std::tuple<double, double, int>> st{{lo, hi, 0}};
    while (!st.empty()) {
      auto [a, b, d] = st.back();
      st.pop_back();
      if (d >= kLevels || !(b - a > resolution)) continue;
      const double mid = 0.5 * (a + b);
      out.push_back(mid);
      st.push_back({mid, b, d + 1});
      st.push_back({a, mid, d + 1});
    }
  };
  PeakResult result;
  auto probe = [&](double rate, double lo, double hi) {
    if (!done.count(rate)) {
      std::vector<double> rs{rate};
      subtree(lo, hi, rs);
      evaluate(rs);
    }
    const auto& [a, e] = done.at(rate);
    if (e.first == SBS_ERR_CONFIG) throw ConfigError(e.second);
    if (e.first == SBS_ERR_INVARIANT) throw std::logic_error(e.second);
    if (e.first != SBS_OK) throw std::runtime_error("sbs_b200: " + e.second);
    PeakProbe p;
    p.rate_qps = rate;
    p.ttft_mean_s = a.ttft_mean_s;
    p.window_requests = a.window_requests;
    p.feasible = p.window_requests >= 10 && p.ttft_mean_s <= slo_ttft_s;
    result.probes.push_back(p);
    return p.feasible;
  };
  {  // first launch: both ends and the top of the tree
    std::vector<double> rs{rate_min, rate_max};
    subtree(rate_min, rate_max, rs);
    evaluate(rs);
  }
  if (!probe(rate_min, rate_min, rate_max)) return result;
  result.attainable = true;
  if (probe(rate_max, rate_min, rate_max)) {
    result.peak_qps = rate_max;
    return result;
  }
  double lo = rate_min, hi = rate_max;
  while (hi - lo > resolution) {
    double mid = 0.5 * (lo + hi);
    if (probe(mid, lo, hi)) lo = mid;
    else hi = mid;
  }
  result.peak_qps = lo;
  return result;
}

}  // namespace sbsim
