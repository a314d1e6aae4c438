// Drop-in replacement for the reference's prefill_alloc.cpp and decode_alloc.cpp
// (proj/src), built against the reference's own headers (proj/include/sbsim).
// Link this translation unit *instead of* those two files and every caller —
// Runner::perform_dispatch (simulation.cpp:287-289), Runner::
// drain_decode_admissions (:459-460), the acceptance audits — runs the
// allocation on the B200 through the C-ABI (include/sbs_b200.h):
//   allocate_batch / greedy_dispatch -> sbs_prefill_allocate (PBAA kernel)
//   select_decode_unit -> sbs_decode_select (IQR kernel)
//   schedule_decode_batch -> sbs_decode_schedule_batch (one sched_kernel launch
//                            per batch: order + every placement on the device)
//   outlier_threshold -> the IQR kernel's threshold output
// percentile / lex_less are scalar helpers the reference's own metrics TU
// calls per finalize (metrics.cpp:151-152); they stay host math.
//
// Cache-aware PBAA (AllocMode::kCacheAware): Len_hit(r, d) is resolved on the
// host against the PrefixCache objects the caller's DpPlans borrow and shipped
// with the window; the kernel does the argmax / guard / update.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "sbs_b200.h"
#include "sbsim/decode_alloc.h"
#include "sbsim/prefill_alloc.h"

namespace {

// Per-thread device staging: one pinned host block and one device block,
// grown on demand, one stream.  Each call is a single H2D copy, one kernel and
// a single D2H copy.
struct Staging {
  cudaStream_t stream = nullptr;
  unsigned char* host = nullptr;
  unsigned char* dev = nullptr;
  size_t cap = 0;

  void ensure(size_t bytes) {
    if (stream == nullptr) check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (bytes <= cap) return;
    size_t n = std::max(bytes, cap * 2);
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    check(cudaMallocHost(&host, n));
    check(cudaMalloc(&dev, n));
    cap = n;
  }
  static void check(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("sbs_b200 shim: ") + cudaGetErrorString(e));
  }
  ~Staging() {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    if (stream) cudaStreamDestroy(stream);
  }
};
thread_local Staging g_st;

size_t align8(size_t v) { return (v + 7) & ~size_t(7); }

void throw_rc(int rc) {
  if (rc == SBS_OK) return;
  if (rc == SBS_ERR_CONFIG) throw sbsim::ConfigError(sbs_last_error());
  if (rc == SBS_ERR_INVARIANT) throw std::logic_error(sbs_last_error());
  throw std::runtime_error(std::string("sbs_b200: ") + sbs_last_error());
}

struct WindowOut {
  std::vector<int32_t> dp, rank, wait;
  std::vector<int64_t> caps;
  bool flow = false;
};

// One cluster-window through the PBAA kernel (sbs_prefill_allocate_one: small
// Basic windows travel in the kernel parameters, one launch per call).
WindowOut run_window(std::span<sbsim::Request* const> pending,
                     std::span<sbsim::Request* const> fresh,
                     const std::vector<sbsim::DpPlan>& dps, int n_limit, sbsim::AllocMode mode) {
  const size_t n = pending.size() + fresh.size(), D = dps.size();
  // cache-aware: Len_hit(r, d) resolved against the caller's caches (the
  // PrefixCache objects the DpPlans borrow, prefill_alloc.h:22)
  const bool ca = mode == sbsim::AllocMode::kCacheAware;
  thread_local std::vector<int64_t> rows, hits;
  rows.resize(3 * n);
  hits.resize(ca ? n * D : 0);
  size_t i = 0;
  for (auto* q : {&pending, &fresh})
    for (sbsim::Request* r : *q) {
      rows[3 * i] = (int64_t)r->id;
      rows[3 * i + 1] = r->prompt_len;
      rows[3 * i + 2] = r->wait_cycles;
      if (ca)
        for (size_t d = 0; d < D; ++d) hits[i * D + d] = sbsim::cache_hit_len(*r, dps[d]);
      ++i;
    }
  WindowOut w;
  w.dp.resize(n);
  w.rank.resize(n);
  w.wait.resize(n);
  w.caps.resize(D);
  for (size_t d = 0; d < D; ++d) w.caps[d] = dps[d].c_avail;
  uint8_t flow = 0;
  throw_rc(sbs_prefill_allocate_one(rows.data(), (int32_t)pending.size(), (int32_t)fresh.size(),
                                    w.caps.data(), (int32_t)D, n_limit, ca ? hits.data() : nullptr,
                                    w.dp.data(), w.rank.data(), w.wait.data(), &flow));
  w.flow = flow != 0;
  return w;
}

}  // namespace

namespace sbsim {

Tokens cache_hit_len(const Request& req, const DpPlan& dp) {
  if (dp.cache == nullptr) return 0;
  return dp.cache->longest_hit(req.prefix_tokens, req.prompt_len);
}

Tokens capacity_after(const Request& req, const DpPlan& dp, AllocMode mode) {
  Tokens charge = req.prompt_len;
  if (mode == AllocMode::kCacheAware) charge -= cache_hit_len(req, dp);
  return dp.c_avail - charge;
}

void greedy_dispatch(std::span<Request* const> queue, std::vector<DpPlan>& dps, AllocMode mode,
                     std::vector<Placement>& mapping, std::vector<Request*>& deferred) {
  // one phase == a window whose whole queue is "pending", never throttled
  WindowOut w = run_window(queue, {}, dps, std::numeric_limits<int>::max(), mode);
  std::vector<std::pair<int32_t, size_t>> placed;
  for (size_t i = 0; i < queue.size(); ++i) {
    if (w.dp[i] >= 0) placed.emplace_back(w.rank[i], i);
    else deferred.push_back(queue[i]);
  }
  std::sort(placed.begin(), placed.end());
  for (auto& [rk, i] : placed) mapping.emplace_back(queue[i], dps[(size_t)w.dp[i]].dp_index);
  for (size_t d = 0; d < dps.size(); ++d) dps[d].c_avail = w.caps[d];
}

AllocationResult allocate_batch(std::span<Request* const> q_pending,
                                std::span<Request* const> q_new, std::vector<DpPlan>& dps,
                                int n_limit, AllocMode mode) {
  AllocationResult res;
  WindowOut w = run_window(q_pending, q_new, dps, n_limit, mode);
  const size_t n = q_pending.size() + q_new.size();
  auto req = [&](size_t i) { return i < q_pending.size() ? q_pending[i] : q_new[i - q_pending.size()]; };
  std::vector<std::pair<int32_t, size_t>> placed;
  for (size_t i = 0; i < n; ++i) {
    Request* r = req(i);
    if (w.dp[i] >= 0) {
      placed.emplace_back(w.rank[i], i);
    } else {
      r->wait_cycles = w.wait[i];
      (w.dp[i] == -2 ? res.throttled : res.deferred).push_back(r);
    }
  }
  std::sort(placed.begin(), placed.end());
  for (auto& [rk, i] : placed) res.mapping.emplace_back(req(i), dps[(size_t)w.dp[i]].dp_index);
  for (size_t d = 0; d < dps.size(); ++d) dps[d].c_avail = w.caps[d];
  res.flow_control = w.flow;
  return res;
}

double percentile(std::vector<double> values, double p) {
  if (values.empty()) throw std::logic_error("percentile: empty input");
  p = std::clamp(p, 0.0, 100.0);
  std::sort(values.begin(), values.end());
  double rank = (static_cast<double>(values.size()) - 1.0) * p / 100.0;
  auto lo = static_cast<std::size_t>(std::floor(rank));
  auto hi = static_cast<std::size_t>(std::ceil(rank));
  if (lo == hi) return values[lo];
  return values[lo] + (rank - static_cast<double>(lo)) * (values[hi] - values[lo]);
}

double outlier_threshold(std::span<const Tokens> kv_loads, double k) {
  // Q3 + k (Q3 - Q1) from the IQR kernel (the threshold it masks with)
  const size_t U = kv_loads.size();
  if (U == 0) throw std::logic_error("percentile: empty input");
  if (U > 16384)  // the IQR kernel's envelope (= the simulator's decode-unit limit); no host fallback
    throw std::runtime_error("outlier_threshold: more than 16384 decode units (GPU envelope)");
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align8(off + bytes); return o; };
  const size_t o_off = take(16), o_b = take(4 * U), o_k = take(8 * U), o_err = take(8),
               o_pos = take(4), o_fb = take(8), o_th = take(8);
  g_st.ensure(off + 64);
  unsigned char* h = g_st.host;
  int64_t uo[2] = {0, (int64_t)U};
  std::memcpy(h + o_off, uo, 16);
  for (size_t i = 0; i < U; ++i) {
    ((int32_t*)(h + o_b))[i] = 0;
    ((int64_t*)(h + o_k))[i] = kv_loads[i];
  }
  *(int32_t*)(h + o_err) = 0;
  unsigned char* g = g_st.dev;
  Staging::check(cudaMemcpyAsync(g, h, o_pos, cudaMemcpyHostToDevice, g_st.stream));
  sbs_decode_batch b{};
  b.n_calls = 1;
  b.max_units = (int32_t)std::min<size_t>(U, 1 << 30);
  b.unit_off = (const int64_t*)(g + o_off);
  b.batch = (const int32_t*)(g + o_b);
  b.kv = (const int64_t*)(g + o_k);
  b.k = k;
  b.pos_out = (int32_t*)(g + o_pos);
  b.fallback_out = (uint8_t*)(g + o_fb);
  b.threshold_out = (double*)(g + o_th);
  throw_rc(sbs_decode_select_async(&b, (int32_t*)(g + o_err), g_st.stream));
  Staging::check(cudaMemcpyAsync(h + o_err, g + o_err, off - o_err, cudaMemcpyDeviceToHost,
                                 g_st.stream));
  Staging::check(cudaStreamSynchronize(g_st.stream));
  if (int e = *(int32_t*)(h + o_err)) throw_rc(e == 3 ? SBS_ERR_INVARIANT : SBS_ERR_OVERFLOW);
  return *(double*)(h + o_th);
}

bool lex_less(const std::pair<int, Tokens>& a, const std::pair<int, Tokens>& b) {
  return a.first != b.first ? a.first < b.first : a.second < b.second;
}

int select_decode_unit(const std::vector<DecodeUnitPlan>& units, double k,
                       std::uint64_t request_id, const DecodeObserver& observe) {
  if (units.empty()) throw std::logic_error("select_decode_unit: no units");
  const size_t U = units.size();
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align8(off + bytes); return o; };
  const size_t o_off = take(16), o_b = take(4 * U), o_k = take(8 * U), o_err = take(8),
               o_pos = take(4), o_fb = take(8), o_th = take(8);
  g_st.ensure(off + 64);
  unsigned char* h = g_st.host;
  int64_t uo[2] = {0, (int64_t)U};
  std::memcpy(h + o_off, uo, 16);
  for (size_t i = 0; i < U; ++i) {
    ((int32_t*)(h + o_b))[i] = units[i].batch;
    ((int64_t*)(h + o_k))[i] = units[i].kv;
  }
  *(int32_t*)(h + o_err) = 0;
  unsigned char* g = g_st.dev;
  Staging::check(cudaMemcpyAsync(g, h, o_pos, cudaMemcpyHostToDevice, g_st.stream));
  sbs_decode_batch b{};
  b.n_calls = 1;
  b.max_units = (int32_t)std::min<size_t>(U, 1 << 30);
  b.unit_off = (const int64_t*)(g + o_off);
  b.batch = (const int32_t*)(g + o_b);
  b.kv = (const int64_t*)(g + o_k);
  b.k = k;
  b.pos_out = (int32_t*)(g + o_pos);
  b.fallback_out = (uint8_t*)(g + o_fb);
  b.threshold_out = (double*)(g + o_th);
  throw_rc(sbs_decode_select_async(&b, (int32_t*)(g + o_err), g_st.stream));
  Staging::check(cudaMemcpyAsync(h + o_err, g + o_err, off - o_err, cudaMemcpyDeviceToHost,
                                 g_st.stream));
  Staging::check(cudaStreamSynchronize(g_st.stream));
  if (int e = *(int32_t*)(h + o_err)) throw_rc(e == 3 ? SBS_ERR_INVARIANT : SBS_ERR_OVERFLOW);
  int pos = *(int32_t*)(h + o_pos);
  if (observe) {
    DecodePlacementInfo info;
    info.request_id = request_id;
    info.threshold = *(double*)(h + o_th);
    info.fallback = h[o_fb] != 0;
    for (size_t i = 0; i < U; ++i) {
      info.kv_snapshot.push_back(units[i].kv);
      if (info.fallback || static_cast<double>(units[i].kv) <= info.threshold)
        info.safe.push_back((int)i);
    }
    info.selected = pos;
    observe(info);
  }
  return pos;
}

std::vector<std::pair<std::uint64_t, int>> schedule_decode_batch(
    std::vector<DecodeCandidate> candidates, std::vector<DecodeUnitPlan>& units, double k,
    const DecodeObserver& observe) {
  // The whole batch is one sched_kernel launch (sbs_decode_schedule_batch):
  // stable order + one select_decode_unit per candidate on the device.
  std::vector<std::pair<std::uint64_t, int>> out;
  const size_t M = candidates.size(), U = units.size();
  if (M == 0) return out;
  if (U == 0) throw std::logic_error("select_decode_unit: no units");
  if (M > 4096 || U > 4096) throw std::runtime_error("sbs_b200 shim: decode batch above 4096");
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align8(off + bytes); return o; };
  const size_t o_co = take(16), o_id = take(8 * M), o_sl = take(8 * M), o_kl = take(8 * M),
               o_uo = take(16), o_err = take(8), o_b = take(4 * U), o_k = take(8 * U),
               o_ord = take(4 * M), o_pos = take(4 * M), o_fb = take(M), o_th = take(8 * M);
  g_st.ensure(off + 64);
  unsigned char* h = g_st.host;
  const int64_t co[2] = {0, (int64_t)M}, uo[2] = {0, (int64_t)U};
  std::memcpy(h + o_co, co, 16);
  std::memcpy(h + o_uo, uo, 16);
  for (size_t i = 0; i < M; ++i) {
    ((uint64_t*)(h + o_id))[i] = candidates[i].request_id;
    ((int64_t*)(h + o_sl))[i] = candidates[i].sort_len;
    ((int64_t*)(h + o_kl))[i] = candidates[i].kv_len;
  }
  *(int32_t*)(h + o_err) = 0;
  for (size_t u = 0; u < U; ++u) {
    ((int32_t*)(h + o_b))[u] = units[u].batch;
    ((int64_t*)(h + o_k))[u] = units[u].kv;
  }
  unsigned char* g = g_st.dev;
  Staging::check(cudaMemcpyAsync(g, h, o_ord, cudaMemcpyHostToDevice, g_st.stream));
  sbs_decode_schedule b{};
  b.n_batches = 1;
  b.max_candidates = (int32_t)M;
  b.max_units = (int32_t)U;
  b.cand_off = (const int64_t*)(g + o_co);
  b.request_id = (const uint64_t*)(g + o_id);
  b.sort_len = (const int64_t*)(g + o_sl);
  b.kv_len = (const int64_t*)(g + o_kl);
  b.unit_off = (const int64_t*)(g + o_uo);
  b.batch = (int32_t*)(g + o_b);
  b.kv = (int64_t*)(g + o_k);
  b.k = k;
  b.order_out = (int32_t*)(g + o_ord);
  b.pos_out = (int32_t*)(g + o_pos);
  b.fallback_out = (uint8_t*)(g + o_fb);
  b.threshold_out = (double*)(g + o_th);
  throw_rc(sbs_decode_schedule_batch_async(&b, (int32_t*)(g + o_err), g_st.stream));
  Staging::check(cudaMemcpyAsync(h + o_err, g + o_err, off - o_err, cudaMemcpyDeviceToHost,
                                 g_st.stream));
  Staging::check(cudaStreamSynchronize(g_st.stream));
  if (int e = *(int32_t*)(h + o_err)) throw_rc(e == 3 ? SBS_ERR_INVARIANT : SBS_ERR_OVERFLOW);
  out.reserve(M);
  for (size_t j = 0; j < M; ++j) {
    const DecodeCandidate& c = candidates[(size_t)((int32_t*)(h + o_ord))[j]];
    const int pos = ((int32_t*)(h + o_pos))[j];
    if (observe) {  // the observer sees the units as they were before this placement
      DecodePlacementInfo info;
      info.request_id = c.request_id;
      info.threshold = ((double*)(h + o_th))[j];
      info.fallback = h[o_fb + j] != 0;
      for (size_t i = 0; i < U; ++i) {
        info.kv_snapshot.push_back(units[i].kv);
        if (info.fallback || static_cast<double>(units[i].kv) <= info.threshold)
          info.safe.push_back((int)i);
      }
      info.selected = pos;
      observe(info);
    }
    units[(size_t)pos].batch += 1;
    units[(size_t)pos].kv += c.kv_len;
    out.emplace_back(c.request_id, units[(size_t)pos].unit_index);
  }
  // the device's final B/K are the same sums; keep the host copy authoritative
  return out;
}

}  // namespace sbsim
