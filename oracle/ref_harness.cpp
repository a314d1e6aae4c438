// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// C-ABI harness around the *unmodified* reference sources
// (/root/reference/proj/src/*.cpp), compiled in place by oracle/Makefile into
// oracle/_ref/libsbsim_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it.
//
// Two reference functions are interposed (never edited): prefill_alloc.cpp is
// compiled with -Dallocate_batch=ref_impl_allocate_batch and decode_alloc.cpp
// with -Dselect_decode_unit=ref_impl_select_decode_unit, so the wrappers below
// (which carry the original names) can count and optionally record every
// allocation window and decode placement that the reference Runner makes
// (simulation.cpp:287-289 and :459-460) without changing its behaviour.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "sbsim/config.h"
#include "sbsim/decode_alloc.h"
#include "sbsim/metrics.h"
#include "sbsim/prefill_alloc.h"
#include "sbsim/simulation.h"
#include "sbsim/workload.h"

namespace sbsim {
// Renamed reference implementations (see file header).
AllocationResult ref_impl_allocate_batch(std::span<Request* const> q_pending,
                                         std::span<Request* const> q_new,
                                         std::vector<DpPlan>& dps, int n_limit,
                                         AllocMode mode);
int ref_impl_select_decode_unit(const std::vector<DecodeUnitPlan>& units,
                                double k, std::uint64_t request_id,
                                const DecodeObserver& observe);
}  // namespace sbsim

namespace {

using namespace sbsim;

// Flat window record: [n_pending, n_new, D, n_limit,
//   pending (id,len,wait)*, new (id,len,wait)*, caps_in*D,
//   n_map, (id,dp)*, n_def, (id,wait)*, n_thr, id*, caps_out*D, flow]
struct Recorder {
  bool windows = false;
  bool decodes = false;
  std::vector<std::int64_t> win;
  std::vector<std::int64_t> dec;  // U, (B,K)*U, selected, fallback
  std::int64_t alloc_calls = 0;
  std::int64_t decode_selects = 0;
};

thread_local Recorder* g_rec = nullptr;

thread_local std::string g_err;

}  // namespace

namespace sbsim {

AllocationResult allocate_batch(std::span<Request* const> q_pending,
                                std::span<Request* const> q_new,
                                std::vector<DpPlan>& dps, int n_limit,
                                AllocMode mode) {
  Recorder* r = g_rec;
  if (r == nullptr)
    return ref_impl_allocate_batch(q_pending, q_new, dps, n_limit, mode);
  r->alloc_calls += 1;
  if (!r->windows)
    return ref_impl_allocate_batch(q_pending, q_new, dps, n_limit, mode);
  auto& w = r->win;
  w.push_back(static_cast<std::int64_t>(q_pending.size()));
  w.push_back(static_cast<std::int64_t>(q_new.size()));
  w.push_back(static_cast<std::int64_t>(dps.size()));
  w.push_back(n_limit);
  for (auto* q : {&q_pending, &q_new})
    for (Request* req : *q) {
      w.push_back(static_cast<std::int64_t>(req->id));
      w.push_back(req->prompt_len);
      w.push_back(req->wait_cycles);
    }
  for (const DpPlan& d : dps) w.push_back(d.c_avail);
  AllocationResult res =
      ref_impl_allocate_batch(q_pending, q_new, dps, n_limit, mode);
  w.push_back(static_cast<std::int64_t>(res.mapping.size()));
  for (auto& [req, dp] : res.mapping) {
    w.push_back(static_cast<std::int64_t>(req->id));
    w.push_back(dp);
  }
  w.push_back(static_cast<std::int64_t>(res.deferred.size()));
  for (Request* req : res.deferred) {
    w.push_back(static_cast<std::int64_t>(req->id));
    w.push_back(req->wait_cycles);
  }
  w.push_back(static_cast<std::int64_t>(res.throttled.size()));
  for (Request* req : res.throttled) w.push_back(static_cast<std::int64_t>(req->id));
  for (const DpPlan& d : dps) w.push_back(d.c_avail);
  w.push_back(res.flow_control ? 1 : 0);
  return res;
}

int select_decode_unit(const std::vector<DecodeUnitPlan>& units, double k,
                       std::uint64_t request_id, const DecodeObserver& observe) {
  Recorder* r = g_rec;
  if (r == nullptr || !r->decodes) {
    if (r != nullptr) r->decode_selects += 1;
    return ref_impl_select_decode_unit(units, k, request_id, observe);
  }
  r->decode_selects += 1;
  bool fb = false;
  auto wrapped = [&](const DecodePlacementInfo& info) {
    fb = info.fallback;
    if (observe) observe(info);
  };
  int pos = ref_impl_select_decode_unit(units, k, request_id, wrapped);
  auto& d = r->dec;
  d.push_back(static_cast<std::int64_t>(units.size()));
  for (const auto& u : units) {
    d.push_back(u.batch);
    d.push_back(u.kv);
  }
  d.push_back(pos);
  d.push_back(fb ? 1 : 0);
  return pos;
}

}  // namespace sbsim

namespace {

// Aggregates in aggregates_json order (simulation.cpp:545-576).
constexpr int kAggFields = 28;

void fill_agg(const Aggregates& a, double* out) {
  double v[kAggFields] = {
      double(a.generated), double(a.completed), double(a.throttled),
      double(a.in_flight), double(a.window_requests), a.ttft_mean_s,
      a.ttft_p50_s, a.ttft_p95_s, a.scheduler_wait_mean_s,
      a.device_wait_mean_s, a.total_wait_mean_s, double(a.passes),
      a.chunk_util_mean, double(a.decode_steps), double(a.output_tokens),
      a.output_tokens_per_s, a.kv_mean_time_avg, a.kv_sigma_time_avg,
      a.completed_per_s, double(a.watchdog_fires),
      double(a.dropped_end_forwards), double(a.rejected_samples),
      double(a.deferrals), double(a.flow_control_events),
      double(a.mask_events), double(a.fallback_events), a.warmup_cutoff_s,
      a.duration_s};
  std::memcpy(out, v, sizeof(v));
}

int status_code(RequestStatus s) { return static_cast<int>(s); }

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_agg_fields(void) { return kAggFields; }

// Runs one experiment from JSON text exactly as `sbsim run` would
// (config.cpp:405 parse_config -> simulation.cpp:537 run_experiment).
//   agg: kAggFields doubles.   meta: [digest, alloc_calls, decode_selects,
//   n_requests, horizon_ns].
//   per_req (nullable, cap rows x 8): arrival, prompt, output, status,
//   dispatch, prefill_start, first_token, completion (-1 when unset).
//   windows/decodes (nullable): recorder outputs; *_len in/out (capacity in,
//   used out; if capacity is too small returns 4 and sets used).
//   csv (nullable): requests|passes|kvband|control joined by '\x1e'.
int ref_run_json(const char* json_text, double* agg, std::int64_t* meta,
                 std::int64_t* per_req, std::int64_t per_req_cap,
                 std::int64_t* windows, std::int64_t* windows_len,
                 std::int64_t* decodes, std::int64_t* decodes_len, char* csv,
                 std::int64_t* csv_len) {
  try {
    ExperimentConfig cfg = parse_config(json_text, "<ref_run_json>");
    Recorder rec;
    rec.windows = windows != nullptr;
    rec.decodes = decodes != nullptr;
    g_rec = &rec;
    SimulationResult res;
    try {
      res = run_experiment(cfg);
    } catch (...) {
      g_rec = nullptr;
      throw;
    }
    g_rec = nullptr;
    if (agg) fill_agg(res.aggregates, agg);
    if (meta) {
      meta[0] = static_cast<std::int64_t>(res.workload_digest);
      meta[1] = rec.alloc_calls;
      meta[2] = rec.decode_selects;
      meta[3] = static_cast<std::int64_t>(res.requests.size());
      meta[4] = res.horizon;
    }
    int rc = 0;
    if (per_req) {
      if (static_cast<std::int64_t>(res.requests.size()) > per_req_cap) {
        rc = 4;
      } else {
        std::int64_t* p = per_req;
        for (const Request& r : res.requests) {
          p[0] = r.arrival_time;
          p[1] = r.prompt_len;
          p[2] = r.output_len;
          p[3] = status_code(r.status);
          p[4] = r.dispatch_time ? *r.dispatch_time : -1;
          p[5] = r.prefill_start ? *r.prefill_start : -1;
          p[6] = r.first_token_time ? *r.first_token_time : -1;
          p[7] = r.completion_time ? *r.completion_time : -1;
          p += 8;
        }
      }
    }
    auto copy_out = [&rc](const std::vector<std::int64_t>& src,
                          std::int64_t* dst, std::int64_t* len) {
      if (dst == nullptr) return;
      std::int64_t cap = *len;
      *len = static_cast<std::int64_t>(src.size());
      if (*len > cap) {
        rc = 4;
        return;
      }
      std::memcpy(dst, src.data(), src.size() * sizeof(std::int64_t));
    };
    copy_out(rec.win, windows, windows_len);
    copy_out(rec.dec, decodes, decodes_len);
    if (csv) {
      std::string all = MetricsCollector::requests_csv(res.requests);
      all += '\x1e';
      all += res.metrics.passes_csv();
      all += '\x1e';
      all += res.metrics.kvband_csv();
      all += '\x1e';
      all += res.metrics.control_csv();
      std::int64_t cap = *csv_len;
      *csv_len = static_cast<std::int64_t>(all.size());
      if (*csv_len + 1 > cap)
        rc = 4;
      else
        std::memcpy(csv, all.c_str(), all.size() + 1);
    }
    return rc;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// generate_workload (workload.cpp:67-142) for the config's workload+seed.
// out: cap rows x 3 (arrival_ns, prompt_len, output_len). meta: [n, digest].
int ref_generate_workload(const char* json_text, std::int64_t* out,
                          std::int64_t cap, std::int64_t* meta) {
  try {
    ExperimentConfig cfg = parse_config(json_text, "<ref_generate_workload>");
    std::vector<Request> reqs = generate_workload(cfg.workload, cfg.sim.seed);
    meta[0] = static_cast<std::int64_t>(reqs.size());
    meta[1] = static_cast<std::int64_t>(workload_digest(reqs));
    if (out == nullptr) return 0;
    if (static_cast<std::int64_t>(reqs.size()) > cap) return 4;
    for (const Request& r : reqs) {
      out[0] = r.arrival_time;
      out[1] = r.prompt_len;
      out[2] = r.output_len;
      out += 3;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// allocate_batch (prefill_alloc.cpp:61-88), Basic mode, on plain arrays.
// pend/fresh: rows of (id, prompt_len, wait_cycles).
// out_map: (id, dp) pairs; out_def: (id, wait) pairs; out_thr: ids;
// counts[3] = n_map, n_def, n_thr; caps updated in place; returns flow flag.
int ref_allocate_batch(const std::int64_t* pend, std::int64_t n_pend,
                       const std::int64_t* fresh, std::int64_t n_fresh,
                       std::int64_t* caps, std::int64_t n_dp, int n_limit,
                       std::int64_t* out_map, std::int64_t* out_def,
                       std::int64_t* out_thr, std::int64_t* counts) {
  std::vector<Request> storage(static_cast<std::size_t>(n_pend + n_fresh));
  std::vector<Request*> pv, nv;
  for (std::int64_t i = 0; i < n_pend + n_fresh; ++i) {
    const std::int64_t* row = i < n_pend ? pend + 3 * i : fresh + 3 * (i - n_pend);
    Request& r = storage[static_cast<std::size_t>(i)];
    r.id = static_cast<std::uint64_t>(row[0]);
    r.prompt_len = row[1];
    r.wait_cycles = static_cast<int>(row[2]);
    (i < n_pend ? pv : nv).push_back(&r);
  }
  std::vector<DpPlan> dps(static_cast<std::size_t>(n_dp));
  for (std::int64_t d = 0; d < n_dp; ++d) {
    dps[static_cast<std::size_t>(d)].dp_index = static_cast<int>(d);
    dps[static_cast<std::size_t>(d)].c_avail = caps[d];
  }
  AllocationResult res = ref_impl_allocate_batch(
      {pv.data(), pv.size()}, {nv.data(), nv.size()}, dps, n_limit,
      AllocMode::kBasic);
  for (std::size_t i = 0; i < res.mapping.size(); ++i) {
    out_map[2 * i] = static_cast<std::int64_t>(res.mapping[i].first->id);
    out_map[2 * i + 1] = res.mapping[i].second;
  }
  for (std::size_t i = 0; i < res.deferred.size(); ++i) {
    out_def[2 * i] = static_cast<std::int64_t>(res.deferred[i]->id);
    out_def[2 * i + 1] = res.deferred[i]->wait_cycles;
  }
  for (std::size_t i = 0; i < res.throttled.size(); ++i)
    out_thr[i] = static_cast<std::int64_t>(res.throttled[i]->id);
  counts[0] = static_cast<std::int64_t>(res.mapping.size());
  counts[1] = static_cast<std::int64_t>(res.deferred.size());
  counts[2] = static_cast<std::int64_t>(res.throttled.size());
  for (std::int64_t d = 0; d < n_dp; ++d) caps[d] = dps[static_cast<std::size_t>(d)].c_avail;
  return res.flow_control ? 1 : 0;
}

// allocate_batch in cache-aware mode with a given Len_hit(r, d) matrix
// (hits: row-major n x n_dp, rows in pending-then-new order).  The hits are
// realised through the reference's own PrefixCache: request r gets unique
// prefix tokens of length max_d hit(r, d); DP d's cache holds r's prefix cut to
// hit(r, d); the probe set is every distinct positive hit; the budget never
// evicts.  Requires hit(r, d) <= prompt_len(r).  Outputs as ref_allocate_batch.
int ref_allocate_batch_ca(const std::int64_t* pend, std::int64_t n_pend,
                          const std::int64_t* fresh, std::int64_t n_fresh,
                          std::int64_t* caps, std::int64_t n_dp, int n_limit,
                          const std::int64_t* hits, std::int64_t* out_map,
                          std::int64_t* out_def, std::int64_t* out_thr,
                          std::int64_t* counts) {
  const std::int64_t n = n_pend + n_fresh;
  std::vector<Request> storage(static_cast<std::size_t>(n));
  std::vector<Request*> pv, nv;
  std::vector<Tokens> probes;
  for (std::int64_t i = 0; i < n * n_dp; ++i)
    if (hits[i] > 0) probes.push_back(hits[i]);
  std::sort(probes.begin(), probes.end());
  probes.erase(std::unique(probes.begin(), probes.end()), probes.end());
  for (std::int64_t i = 0; i < n; ++i) {
    const std::int64_t* row = i < n_pend ? pend + 3 * i : fresh + 3 * (i - n_pend);
    Request& r = storage[static_cast<std::size_t>(i)];
    r.id = static_cast<std::uint64_t>(row[0]);
    r.prompt_len = row[1];
    r.wait_cycles = static_cast<int>(row[2]);
    Tokens mx = 0;
    for (std::int64_t d = 0; d < n_dp; ++d) mx = std::max<Tokens>(mx, hits[i * n_dp + d]);
    for (Tokens t = 0; t < mx; ++t)
      r.prefix_tokens.push_back(static_cast<std::int32_t>((i * 1000003 + t * 7919 + 1) & 0x7fffffff));
    (i < n_pend ? pv : nv).push_back(&r);
  }
  std::vector<PrefixCache> cache;
  for (std::int64_t d = 0; d < n_dp; ++d) cache.emplace_back(probes, Tokens(1) << 60);
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t d = 0; d < n_dp; ++d) {
      const Tokens h = hits[i * n_dp + d];
      if (h <= 0) continue;
      const Request& r = storage[static_cast<std::size_t>(i)];
      std::vector<std::int32_t> cut(r.prefix_tokens.begin(), r.prefix_tokens.begin() + h);
      cache[static_cast<std::size_t>(d)].insert(cut, h);
    }
  std::vector<DpPlan> dps(static_cast<std::size_t>(n_dp));
  for (std::int64_t d = 0; d < n_dp; ++d) {
    dps[static_cast<std::size_t>(d)].dp_index = static_cast<int>(d);
    dps[static_cast<std::size_t>(d)].c_avail = caps[d];
    dps[static_cast<std::size_t>(d)].cache = &cache[static_cast<std::size_t>(d)];
  }
  AllocationResult res = ref_impl_allocate_batch(
      {pv.data(), pv.size()}, {nv.data(), nv.size()}, dps, n_limit,
      AllocMode::kCacheAware);
  for (std::size_t i = 0; i < res.mapping.size(); ++i) {
    out_map[2 * i] = static_cast<std::int64_t>(res.mapping[i].first->id);
    out_map[2 * i + 1] = res.mapping[i].second;
  }
  for (std::size_t i = 0; i < res.deferred.size(); ++i) {
    out_def[2 * i] = static_cast<std::int64_t>(res.deferred[i]->id);
    out_def[2 * i + 1] = res.deferred[i]->wait_cycles;
  }
  for (std::size_t i = 0; i < res.throttled.size(); ++i)
    out_thr[i] = static_cast<std::int64_t>(res.throttled[i]->id);
  counts[0] = static_cast<std::int64_t>(res.mapping.size());
  counts[1] = static_cast<std::int64_t>(res.deferred.size());
  counts[2] = static_cast<std::int64_t>(res.throttled.size());
  for (std::int64_t d = 0; d < n_dp; ++d) caps[d] = dps[static_cast<std::size_t>(d)].c_avail;
  return res.flow_control ? 1 : 0;
}

// select_decode_unit (decode_alloc.cpp:38-81) on (B, K) arrays.
int ref_select_decode_unit(const std::int64_t* batch, const std::int64_t* kv,
                           std::int64_t n, double k, int* fallback,
                           double* threshold) {
  std::vector<DecodeUnitPlan> units(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i)
    units[static_cast<std::size_t>(i)] =
        DecodeUnitPlan{static_cast<int>(i), static_cast<int>(batch[i]), kv[i]};
  bool fb = false;
  double th = 0.0;
  int pos = ref_impl_select_decode_unit(
      units, k, 0, [&](const DecodePlacementInfo& info) {
        fb = info.fallback;
        th = info.threshold;
      });
  if (fallback) *fallback = fb ? 1 : 0;
  if (threshold) *threshold = th;
  return pos;
}

// schedule_decode_batch (decode_alloc.cpp:83-106), the reference's own
// function: cand rows (request_id, sort_len, kv_len); out rows (request_id,
// unit position) in placement order, plus the observer's threshold/fallback
// per placement; batch/kv updated in place.
int ref_schedule_decode_batch(const std::int64_t* cand, std::int64_t n_cand,
                              std::int64_t* batch, std::int64_t* kv, std::int64_t n_units,
                              double k, std::int64_t* out, double* th_out, int* fb_out) {
  try {
    std::vector<DecodeCandidate> cands(static_cast<std::size_t>(n_cand));
    for (std::int64_t i = 0; i < n_cand; ++i)
      cands[static_cast<std::size_t>(i)] = DecodeCandidate{
          static_cast<std::uint64_t>(cand[3 * i]), cand[3 * i + 1], cand[3 * i + 2]};
    std::vector<DecodeUnitPlan> units(static_cast<std::size_t>(n_units));
    for (std::int64_t i = 0; i < n_units; ++i)
      units[static_cast<std::size_t>(i)] =
          DecodeUnitPlan{static_cast<int>(i), static_cast<int>(batch[i]), kv[i]};
    std::size_t j = 0;
    auto res = schedule_decode_batch(cands, units, k, [&](const DecodePlacementInfo& info) {
      th_out[j] = info.threshold;
      fb_out[j] = info.fallback ? 1 : 0;
      ++j;
    });
    for (std::size_t i = 0; i < res.size(); ++i) {
      out[2 * i] = static_cast<std::int64_t>(res[i].first);
      out[2 * i + 1] = res[i].second;
    }
    for (std::int64_t i = 0; i < n_units; ++i) {
      batch[i] = units[static_cast<std::size_t>(i)].batch;
      kv[i] = units[static_cast<std::size_t>(i)].kv;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// find_peak_qps (simulation.cpp:608-644), the reference's own search: probes
// as rows (rate, ttft_mean, window_requests, feasible); returns the probe count
// (-1 on error), *peak / *attainable.
int ref_find_peak_qps(const char* json_text, double slo, double rmin, double rmax, double res,
                      double* probes, int cap, double* peak, int* attainable) {
  try {
    ExperimentConfig cfg = parse_config(json_text, "<test>");
    PeakResult r = find_peak_qps(cfg, slo, rmin, rmax, res);
    int n = 0;
    for (const auto& p : r.probes) {
      if (n < cap) {
        probes[4 * n] = p.rate_qps;
        probes[4 * n + 1] = p.ttft_mean_s;
        probes[4 * n + 2] = static_cast<double>(p.window_requests);
        probes[4 * n + 3] = p.feasible ? 1.0 : 0.0;
      }
      ++n;
    }
    *peak = r.peak_qps;
    *attainable = r.attainable ? 1 : 0;
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double ref_percentile(const double* v, std::int64_t n, double p) {
  return percentile(std::vector<double>(v, v + n), p);
}

double ref_outlier_threshold(const std::int64_t* kv, std::int64_t n, double k) {
  return outlier_threshold(std::span<const Tokens>(kv, static_cast<std::size_t>(n)), k);
}

// CPU baseline: run_experiment over n configs on a pool of `threads` std::threads
// (independent runs may be concurrent). Returns wall seconds in
// *wall_s; agg_out holds n x kAggFields; meta_out n x 3 (digest, alloc_calls,
// decode_selects).
int ref_run_batch(const char* const* json_texts, std::int64_t n, int threads,
                  double* agg_out, std::int64_t* meta_out, double* wall_s) {
  std::atomic<std::int64_t> next{0};
  std::atomic<int> rc{0};
  auto worker = [&]() {
    for (;;) {
      std::int64_t i = next.fetch_add(1);
      if (i >= n) return;
      std::int64_t meta[5];
      int r = ref_run_json(json_texts[i], agg_out + i * kAggFields, meta,
                           nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                           nullptr, nullptr);
      if (r != 0) rc = r;
      if (meta_out) {
        meta_out[3 * i] = meta[0];
        meta_out[3 * i + 1] = meta[1];
        meta_out[3 * i + 2] = meta[2];
      }
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  int nt = std::max(1, threads);
  for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rc.load();
}

// CPU baseline of the allocation step alone: the reference's allocate_batch
// (Basic mode) over `n` recorded windows (flat Recorder records, see above),
// `reps` passes per window, on a pool of `threads` std::threads.  Each call
// starts from the recorded inputs (c_avail snapshot, wait_cycles), as the
// Runner's perform_dispatch does (simulation.cpp:277-289).  Returns wall
// seconds; *checksum folds the placements (so nothing is optimised away).
int ref_bench_allocate(const std::int64_t* rec, std::int64_t rec_len, int threads, int reps,
                       double* wall_s, std::int64_t* n_windows, std::int64_t* checksum) {
  struct Win {
    std::vector<Request> req;
    std::vector<Request*> pend, fresh;
    std::vector<std::int64_t> caps;
    std::vector<int> waits;
    int n_limit = 0;
  };
  std::vector<Win> wins;
  std::int64_t i = 0;
  while (i < rec_len) {
    const std::int64_t np = rec[i], nn = rec[i + 1], D = rec[i + 2];
    Win w;
    w.n_limit = static_cast<int>(rec[i + 3]);
    i += 4;
    w.req.resize(static_cast<std::size_t>(np + nn));
    for (std::int64_t r = 0; r < np + nn; ++r) {
      Request& q = w.req[static_cast<std::size_t>(r)];
      q.id = static_cast<std::uint64_t>(rec[i]);
      q.prompt_len = rec[i + 1];
      q.wait_cycles = static_cast<int>(rec[i + 2]);
      w.waits.push_back(q.wait_cycles);
      i += 3;
    }
    for (std::int64_t r = 0; r < np + nn; ++r)
      (r < np ? w.pend : w.fresh).push_back(&w.req[static_cast<std::size_t>(r)]);
    for (std::int64_t d = 0; d < D; ++d) w.caps.push_back(rec[i + d]);
    i += D;
    const std::int64_t nm = rec[i];
    i += 1 + 2 * nm;
    const std::int64_t nd = rec[i];
    i += 1 + 2 * nd;
    const std::int64_t nt = rec[i];
    i += 1 + nt + D + 1;
    wins.push_back(std::move(w));
  }
  *n_windows = static_cast<std::int64_t>(wins.size());
  std::atomic<std::int64_t> next{0}, sum{0};
  const std::int64_t total = static_cast<std::int64_t>(wins.size()) * std::max(1, reps);
  auto worker = [&]() {
    std::vector<DpPlan> dps;
    std::int64_t local = 0;
    for (;;) {
      const std::int64_t j = next.fetch_add(64);
      if (j >= total) break;
      for (std::int64_t t = j; t < std::min(total, j + 64); ++t) {
        Win& w = wins[static_cast<std::size_t>(t % static_cast<std::int64_t>(wins.size()))];
        // (per-thread copies of the mutable request state)
        std::vector<Request> req = w.req;
        std::vector<Request*> pv, nv;
        for (std::size_t r = 0; r < req.size(); ++r)
          (r < w.pend.size() ? pv : nv).push_back(&req[r]);
        dps.resize(w.caps.size());
        for (std::size_t d = 0; d < w.caps.size(); ++d) {
          dps[d].dp_index = static_cast<int>(d);
          dps[d].c_avail = w.caps[d];
          dps[d].cache = nullptr;
        }
        AllocationResult res = ref_impl_allocate_batch({pv.data(), pv.size()}, {nv.data(), nv.size()},
                                                       dps, w.n_limit, AllocMode::kBasic);
        local += static_cast<std::int64_t>(res.mapping.size()) + (res.flow_control ? 1 : 0);
      }
    }
    sum += local;
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *checksum = sum.load();
  return 0;
}

// CPU baseline of the decode placement alone: the reference's
// select_decode_unit over `n` recorded calls (Recorder decode records), `reps`
// passes, on `threads` threads.
int ref_bench_select(const std::int64_t* rec, std::int64_t rec_len, double k, int threads, int reps,
                     double* wall_s, std::int64_t* n_calls, std::int64_t* checksum) {
  std::vector<std::vector<DecodeUnitPlan>> calls;
  std::int64_t i = 0;
  while (i < rec_len) {
    const std::int64_t U = rec[i];
    std::vector<DecodeUnitPlan> u(static_cast<std::size_t>(U));
    for (std::int64_t x = 0; x < U; ++x)
      u[static_cast<std::size_t>(x)] =
          DecodeUnitPlan{static_cast<int>(x), static_cast<int>(rec[i + 1 + 2 * x]), rec[i + 2 + 2 * x]};
    i += 1 + 2 * U + 2;
    calls.push_back(std::move(u));
  }
  *n_calls = static_cast<std::int64_t>(calls.size());
  std::atomic<std::int64_t> next{0}, sum{0};
  const std::int64_t total = static_cast<std::int64_t>(calls.size()) * std::max(1, reps);
  auto worker = [&]() {
    std::int64_t local = 0;
    for (;;) {
      const std::int64_t j = next.fetch_add(64);
      if (j >= total) break;
      for (std::int64_t t = j; t < std::min(total, j + 64); ++t)
        local += ref_impl_select_decode_unit(
            calls[static_cast<std::size_t>(t % static_cast<std::int64_t>(calls.size()))], k, 0, nullptr);
    }
    sum += local;
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *checksum = sum.load();
  return 0;
}

}  // extern "C"
