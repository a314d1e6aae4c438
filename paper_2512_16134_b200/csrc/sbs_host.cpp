// Host side of the B200 SBS hot path: the C-ABI declared in include/sbs_b200.h.
//
//  * sbs_generate_workload: restates generate_workload / workload_digest
//    (workload.cpp:19-162) with the same libstdc++ mt19937_64 and glibc libm
//    calls, so traces are bit-identical to the reference's on this image.
//  * sbs_sim_*: validates experiments like validate() (core.cpp:79-114) and
//    setup_faults() (simulation.cpp:93-120), lays out one HBM arena per
//    replica, uploads traces once per unique trace, launches the persistent
//    DES kernel, and turns the device counters into Aggregates with the same
//    formulas as MetricsCollector::finalize (metrics.cpp:103-190).
//  * sbs_prefill_allocate / sbs_decode_select: batched allocation kernels.
//
// Built with -ffp-contract=off: every FP64 expression that feeds an integer
// timestamp must round exactly like the reference's x86-64 build.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sbs_b200.h"
#include "des_types.h"

namespace sbs {
cudaError_t launch_des(int variant, const DevPoint* d_pts, int n_pts, int* d_counter,
                       DevResult* d_res, int smem_per_warp, int warps_per_block, int n_blocks,
                       int min_smem, cudaStream_t st);
cudaError_t launch_des_pair3(int variant, const DevPoint* d_pts, int n_pts, DevResult* d_res, int slice_pf,
                             int slice_dc, int n_psm, int wp, int n_dsm, int wd, int* sync,
                             cudaStream_t st_pf, cudaStream_t st_dc, bool simple_decode, bool simple_prefill);
cudaError_t launch_des_cluster(int variant, const DevPoint* d_pts, int n_pts, DevResult* d_res,
                               int smem_per_rep, cudaStream_t st);
cudaError_t launch_finalize(const DevPoint* d_pts, int n_pts, DevResult* d_res, cudaStream_t st);
cudaError_t launch_reset(const DevPoint* d_pts, int n_pts, DevResult* d_res, cudaStream_t st);
struct CopySeg {
  const unsigned char* src;
  unsigned char* dst;
  int64_t bytes;
};
cudaError_t launch_gather(const CopySeg* d_segs, int n_segs, int64_t n_blocks, cudaStream_t st);
struct PbaaArgs {
  int32_t n_windows;
  int32_t max_req, max_dp;
  const int64_t* req_off;
  const int32_t* n_pending;
  const int64_t* dp_off;
  const int32_t* n_limit;
  const int64_t* req_id;
  const int64_t* prompt_len;
  const int32_t* wait_in;
  int64_t* caps;
  int32_t* out_dp;
  int32_t* out_rank;
  int32_t* wait_out;
  uint8_t* flow;
  int32_t* error;
  const int64_t* hit_off;  // cache-aware mode (NULL: Basic)
  const int64_t* hit;
};
struct IqrArgs {
  int32_t n_calls;
  int32_t max_units;
  const int64_t* unit_off;
  const int32_t* batch;
  const int64_t* kv;
  double k;
  int32_t* pos_out;
  uint8_t* fallback_out;
  double* threshold_out;
  int32_t* error;
};
cudaError_t launch_pbaa(const PbaaArgs& a, cudaStream_t st);
cudaError_t launch_pbaa_one(const int64_t* rows, int n_pending, int n_new, const int64_t* caps,
                            int n_dp, int n_limit, int32_t* mapped_out, cudaStream_t st);
cudaError_t launch_iqr(const IqrArgs& a, cudaStream_t st);
struct SchedArgs {
  int32_t n_batches, max_cands, max_units;
  const int64_t* cand_off;
  const uint64_t* request_id;
  const int64_t* sort_len;
  const int64_t* kv_len;
  const int64_t* unit_off;
  int32_t* batch;
  int64_t* kv;
  double k;
  int32_t* order_out;
  int32_t* pos_out;
  uint8_t* fallback_out;
  double* threshold_out;
  int32_t* error;
};
cudaError_t launch_sched(const SchedArgs& a, cudaStream_t st);
cudaError_t launch_gen(const sbs_gen_job* d_jobs, int n_jobs, const uint64_t* d_seeds, int want_digest,
                       cudaStream_t st);
}  // namespace sbs

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct Error {
  int code;
  std::string msg;
};

#define CUDA_OR_THROW(x)                                                              \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw Error{SBS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)};     \
  } while (0)

int64_t seconds_to_ns(double s) { return static_cast<int64_t>(std::llround(s * 1e9)); }

// ------------------------- workload (workload.cpp) -------------------------
constexpr double kTwoPi = 6.283185307179586476925286766559;

inline double u01(std::mt19937_64& rng) {
  return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}
inline double standard_normal(std::mt19937_64& rng) {
  double a = u01(rng);
  double b = u01(rng);
  double r = std::sqrt(-2.0 * std::log(1.0 - a));
  return r * std::cos(kTwoPi * b);
}
inline double exponential(std::mt19937_64& rng, double rate) {
  return -std::log(1.0 - u01(rng)) / rate;
}
int64_t sample_length(const sbs_length_spec& s, std::mt19937_64& rng) {
  switch (s.dist) {
    case SBS_LEN_CONSTANT:
      return std::max<int64_t>(1, s.value);
    case SBS_LEN_UNIFORM: {
      int64_t lo = std::max<int64_t>(1, s.min);
      int64_t hi = std::max(lo, s.max);
      double span = static_cast<double>(hi - lo + 1);
      int64_t off = static_cast<int64_t>(u01(rng) * span);
      return lo + std::min(off, hi - lo);
    }
    case SBS_LEN_LOGNORMAL: {
      double v = std::exp(s.mu + s.sigma * standard_normal(rng));
      int64_t t = static_cast<int64_t>(std::llround(v));
      return std::clamp(t, std::max<int64_t>(1, s.min), s.max);
    }
  }
  throw Error{SBS_ERR_INVARIANT, "sample_length: unknown distribution"};
}

void check_workload(const sbs_workload& w) {
  if (!(w.rate_qps > 0)) throw Error{SBS_ERR_CONFIG, "workload rate_qps must be > 0"};
  if (!(w.duration_s > 0)) throw Error{SBS_ERR_CONFIG, "workload duration_s must be > 0"};
  if (w.shared_prefix_fraction < 0 || w.shared_prefix_fraction > 1)
    throw Error{SBS_ERR_CONFIG, "shared_prefix_fraction must be in [0, 1]"};
  if (w.shared_prefix_fraction > 0 && (w.prefix_pool <= 0 || w.prefix_len <= 0))
    throw Error{SBS_ERR_CONFIG,
                "prefix_pool and prefix_len must be positive when shared prefixes are enabled"};
  if (w.initial_burst < 0) throw Error{SBS_ERR_CONFIG, "workload initial_burst must be >= 0"};
}

struct HostTrace {
  std::vector<int64_t> arr;
  std::vector<int32_t> prompt, output;
  std::vector<int32_t> pool, psize;  // empty when no request has a shared prefix
  uint64_t digest = 0;
};

// Deterministic token id for position i of pool prefix p (workload.cpp:30-37).
int32_t prefix_token(int pool_id, int64_t i) {
  uint64_t h = 1469598103934665603ull;
  h ^= static_cast<uint64_t>(pool_id) * 0x9e3779b97f4a7c15ull;
  h ^= static_cast<uint64_t>(i) + 0x632be59bd9b4e019ull;
  h *= 1099511628211ull;
  return static_cast<int32_t>(h & 0x7fffffff);
}

// PrefixCache::hash_prefix (core.cpp:18-31) of the first k tokens of pool p.
uint64_t hash_pool_prefix(int pool_id, int64_t k) {
  uint64_t h = 14695981039346656037ull ^ static_cast<uint64_t>(k);
  for (int64_t i = 0; i < k; ++i) {
    const uint32_t v = static_cast<uint32_t>(prefix_token(pool_id, i));
    for (int b = 0; b < 4; ++b) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 1099511628211ull;
    }
  }
  return h;
}

void mix_digest(uint64_t& h, uint64_t v) {
  for (int b = 0; b < 8; ++b) {
    h ^= (v >> (8 * b)) & 0xff;
    h *= 1099511628211ull;
  }
}

// generate_workload (workload.cpp:67-142) + workload_digest (:144-162).
void generate(const sbs_workload& spec, uint64_t seed, HostTrace& out) {
  check_workload(spec);
  std::mt19937_64 rng(seed);
  const int64_t horizon = seconds_to_ns(spec.duration_s);
  const double slot = 1.0 / spec.rate_qps;
  std::vector<double> arrivals(static_cast<size_t>(spec.initial_burst), 0.0);
  switch (spec.process) {
    case SBS_ARRIVAL_POISSON: {
      double t = exponential(rng, spec.rate_qps);
      while (t < spec.duration_s) {
        arrivals.push_back(t);
        t += exponential(rng, spec.rate_qps);
      }
      break;
    }
    case SBS_ARRIVAL_UNIFORM:
      for (size_t n = 0;; ++n) {
        double t = static_cast<double>(n) * slot;
        if (t >= spec.duration_s) break;
        arrivals.push_back(t);
      }
      break;
    case SBS_ARRIVAL_UNIFORM_JITTER:
      for (size_t n = 0;; ++n) {
        double base = static_cast<double>(n) * slot;
        if (base >= spec.duration_s) break;
        double t = base + u01(rng) * slot;
        if (t < spec.duration_s) arrivals.push_back(t);
      }
      break;
    default:
      throw Error{SBS_ERR_CONFIG, "workload.process must be poisson, uniform, or uniform_jitter"};
  }
  const size_t n = arrivals.size();
  out.arr.resize(n);
  out.prompt.resize(n);
  out.output.resize(n);
  const bool prefixes = spec.shared_prefix_fraction > 0;
  out.pool.assign(prefixes ? n : 0, -1);
  out.psize.assign(prefixes ? n : 0, 0);
  uint64_t h = 14695981039346656037ull;
  for (size_t i = 0; i < n; ++i) {
    int64_t at = std::min(seconds_to_ns(arrivals[i]), horizon - 1);
    int64_t p = sample_length(spec.prompt, rng);
    int64_t o = spec.output.dist == SBS_LEN_CONSTANT ? std::max<int64_t>(0, spec.output.value)
                                                      : sample_length(spec.output, rng);
    if (p > 0x3fffffff || o > 0x3fffffff)
      throw Error{SBS_ERR_CONFIG, "request lengths above 2^30 tokens are not supported"};
    out.arr[i] = at;
    out.prompt[i] = static_cast<int32_t>(p);
    out.output[i] = static_cast<int32_t>(o);
    // shared prefix (workload.cpp:129-138): the tokens are a pure function of
    // (pool, position), so (pool id, length) stands for Request::prefix_tokens
    int64_t plen = 0;
    int32_t pool_id = -1;
    if (prefixes && u01(rng) < spec.shared_prefix_fraction) {
      int pid = static_cast<int>(u01(rng) * static_cast<double>(spec.prefix_pool));
      pool_id = std::min(pid, spec.prefix_pool - 1);
      plen = std::max<int64_t>(0, std::min<int64_t>(spec.prefix_len, p));  // empty vector if <= 0
      out.pool[i] = plen > 0 ? pool_id : -1;
      out.psize[i] = static_cast<int32_t>(plen);
    }
    mix_digest(h, static_cast<uint64_t>(at));
    mix_digest(h, static_cast<uint64_t>(p));
    mix_digest(h, static_cast<uint64_t>(o));
    mix_digest(h, plen == 0 ? 0 : static_cast<uint64_t>(prefix_token(pool_id, 0)) + 1);
    mix_digest(h, static_cast<uint64_t>(plen));
  }
  out.digest = h;
}

// ------------------------- validation (core.cpp:79-114) ---------------------
void validate(const sbs_experiment& x) {
  const sbs_cluster& c = x.cluster;
  auto require = [](bool ok, const char* what) {
    if (!ok) throw Error{SBS_ERR_CONFIG, what};
  };
  require(c.n_instances_prefill >= 1, "n_instances_prefill must be >= 1");
  require(c.n_instances_decode >= 1, "n_instances_decode must be >= 1");
  require(c.dp_degree >= 1, "dp_degree must be >= 1");
  require(c.dp_degree_decode >= 0, "dp_degree_decode must be >= 0");
  require(c.c_chunk >= 1, "c_chunk must be >= 1");
  require(c.t_default_s > 0, "t_default_s must be > 0");
  require(c.w_size >= 1, "w_size must be >= 1");
  require(c.l_net_s >= 0, "l_net_s must be >= 0");
  require(c.n_limit >= 0, "n_limit must be >= 0");
  require(c.iqr_k >= 0, "iqr_k must be >= 0");
  require(c.watchdog_multiplier > 0, "watchdog_multiplier must be > 0");
  require(c.prefill_base_s >= 0, "prefill_base_s must be >= 0");
  require(c.prefill_per_token_s >= 0, "prefill_per_token_s must be >= 0");
  require(c.decode_base_s >= 0, "decode_base_s must be >= 0");
  require(c.decode_per_request_s >= 0, "decode_per_request_s must be >= 0");
  require(c.decode_per_kv_token_s >= 0, "decode_per_kv_token_s must be >= 0");
  require(c.decode_tokens_per_step >= 1, "decode_tokens_per_step must be >= 1");
  require(c.decode_max_batch_per_dp >= 0, "decode_max_batch_per_dp must be >= 0");
  require(x.warmup_fraction >= 0.0 && x.warmup_fraction < 1.0,
          "sim.warmup_fraction must be in [0, 1)");
  if (c.cache_enabled) {  // core.cpp:106-113
    require(c.cache_n_probes >= 1 && c.cache_probe_lens != nullptr,
            "cache.probe_lens must be non-empty when the cache is enabled");
    for (int i = 0; i < c.cache_n_probes; ++i)
      require(c.cache_probe_lens[i] >= 1, "cache.probe_lens entries must be >= 1");
    require(c.cache_budget_tokens >= 1, "cache.budget_tokens must be >= 1 when the cache is enabled");
  }
  require(x.prefill_mode == SBS_ALLOC_BASIC || x.prefill_mode == SBS_ALLOC_CACHE_AWARE,
          "scheduler.prefill_mode must be basic or cache_aware");
  // GPU-path envelope (documented in DESIGN.md)
  if (c.cache_enabled && x.prefill_mode == SBS_ALLOC_CACHE_AWARE) {
    std::vector<int64_t> pr(c.cache_probe_lens, c.cache_probe_lens + c.cache_n_probes);
    std::sort(pr.begin(), pr.end());
    pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
    require(pr.size() <= (size_t)sbs::kMaxProbes, "GPU path supports at most 32 distinct probe lengths");
  }
  require(c.n_instances_prefill <= sbs::kMaxInstances && c.n_instances_decode <= sbs::kMaxInstances,
          "GPU path supports at most 32 prefill and 32 decode instances");
  require(c.dp_degree <= sbs::kMaxPrefillDp, "GPU path supports dp_degree <= 128");
  require(c.c_chunk <= 0x7fffffff, "GPU path supports c_chunk < 2^31");
  require(c.decode_tokens_per_step < (1 << 17), "GPU path supports decode_tokens_per_step < 2^17");
  require(c.w_size <= sbs::kMaxWSize, "GPU path supports w_size <= 1024");
  require(x.policy >= 0 && x.policy <= 3, "scheduler.policy out of range");
  require(x.decode_policy >= 0 && x.decode_policy <= 2, "scheduler.decode_policy out of range");
  int dd = c.dp_degree_decode > 0 ? c.dp_degree_decode : c.dp_degree;
  require((int64_t)dd * c.n_instances_decode <= 16384, "GPU path supports <= 16384 decode units");
  const int n_inst = c.n_instances_prefill + c.n_instances_decode;
  for (int i = 0; i < x.n_deads; ++i)
    if (x.deads[i].instance < 0 || x.deads[i].instance >= n_inst)
      throw Error{SBS_ERR_CONFIG, "faults.dead: instance out of range"};
  for (int i = 0; i < x.n_topology; ++i) {
    if (x.topology[i].instance < 0 || x.topology[i].instance >= n_inst)
      throw Error{SBS_ERR_CONFIG, "faults.topology: instance out of range"};
    if (seconds_to_ns(x.topology[i].time_s) < 0)
      throw Error{SBS_ERR_INVARIANT, "SimClock::schedule: event time is before now"};
  }
  for (int i = 0; i < x.n_drops; ++i)
    if (x.drops[i].instance != -1 && (x.drops[i].instance < 0 || x.drops[i].instance >= n_inst))
      throw Error{SBS_ERR_CONFIG, "faults.drop_end_forward: instance out of range"};
}

int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

struct TraceDev {
  int64_t* arr = nullptr;
  int32_t* prompt = nullptr;
  int32_t* output = nullptr;
  int32_t* pool = nullptr;   // shared-prefix pool id per request (-1: none), or NULL
  int32_t* psize = nullptr;  // prefix tokens per request
  // second trace buffer set (sbs_sim_enable_trace_slots(2)): the next step's
  // traces go up while the current step runs
  int64_t* arr1 = nullptr;
  int32_t* prompt1 = nullptr;
  int32_t* output1 = nullptr;
  int32_t* pool1 = nullptr;
  int32_t* psize1 = nullptr;
  int64_t n = 0;              // length (host traces) or capacity (generated traces)
  int32_t max_output = 0;
  int32_t max_prompt = 0;
  int32_t n_pools = 0;       // 1 + max pool id
  int64_t max_psize = 0;
  uint64_t digest = 0;
  // device-generated traces (sbs_sim_create_generated): the (workload, seed)
  // they come from, per-slot generation stats on the device (n first: the
  // DES kernels read the length from there) and their host copies
  bool gen = false;
  sbs_workload spec{};
  uint64_t seed = 0;
  sbs_gen_stats* d_stats = nullptr;  // [2]
  sbs_gen_stats h_stats[2] = {};
};

struct PointHost {
  sbs_experiment x;  // copy (fault pointers re-pointed into owned vectors)
  std::vector<sbs_drop_fault> drops;
  std::vector<sbs_dead_fault> deads;
  std::vector<sbs_topology_fault> topo;
  std::vector<int64_t> probes;  // cache.probe_lens (owned copy)
  int trace = 0;
  // capacities (grown on overflow)
  int32_t F = 0, QP = 0, QW = 0, BC = 0, QD = 0;
  int64_t LOG = 0;
  int32_t split = 1;  // two-warp replica (cleared for an exact one-warp rerun)
  bool prefill_only = false;  // every output_len <= 1: no request reaches the decode side
  void* arena = nullptr;
  size_t arena_bytes = 0;
  void* fault_buf = nullptr;
  sbs::DevPoint dp{};
  double cost = 0;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct sbs_sim {
  int device = 0;
  uint32_t flags = 0;
  std::vector<PointHost> pts;
  std::vector<TraceDev> traces;
  std::vector<int> order;  // device slot -> point index (grouped by variant, cost-descending)
  static constexpr int kVariants = 14;
  int group_begin[kVariants + 1] = {};  // slots of kernel variant v: [group_begin[v], group_begin[v+1])
  sbs::DevPoint* d_pts = nullptr;
  sbs::DevResult* d_res = nullptr;
  int* d_counter = nullptr;
  std::vector<sbs::DevResult> h_res;
  int smem_per_warp = 0;
  int warps_per_block = 4;
  int n_blocks = 0;
  int n_launches = 0;
  int64_t device_bytes = 0;
  int sm_count = 148;
  // two-warp replicas: 1 = one CTA, 2 = a 2-CTA cluster, 3 = two kernels
  // (default; clusters when the group shares the launch or overflows one
  // round, or when the kernels turn out not co-resident) — SBS_SPLIT
  int pair_mode = 3;
  int* d_sync = nullptr;  // pair mode 3: [0] CTAs checked in, [1] gave up (not co-resident)
  int pair3_used = 0;     // the last launch ran a two-kernel group
  cudaEvent_t ev_des[2] = {nullptr, nullptr};  // around the DES kernels of the last launch
  // one stream per kernel variant: the variant groups run side by side
  cudaStream_t vstream[kVariants] = {};
  cudaStream_t vstream2[kVariants] = {};  // pair mode 3: the decode kernel's stream
  cudaEvent_t ev_join[kVariants] = {};
  // trace re-upload in one gather launch (segment table, pinned host + device)
  sbs::CopySeg* h_segs = nullptr;
  sbs::CopySeg* d_segs = nullptr;
  int seg_cap = 0;
  cudaEvent_t ev_segs = nullptr;  // the previous gather has consumed h_segs
  bool generated = false;          // traces are generated on the device
  sbs_gen_job* d_jobs[2] = {};     // per slot, one job per trace
  uint64_t* d_seeds[2] = {};
  uint64_t* h_seeds[2] = {};       // pinned staging for the next seeds
  cudaEvent_t ev_seeds[2] = {};    // the staged seeds of a slot were consumed
  int gen_slot_valid[2] = {};      // h_stats of the slot are current
  int n_slots = 1;                 // trace buffer sets
  int cur_slot = 0;                // the set the last launch read
  sbs::DevPoint* d_pts1 = nullptr; // point descriptors pointing at set 1
};

namespace {

void free_point(PointHost& p) {
  if (p.arena) cudaFree(p.arena);
  if (p.fault_buf) cudaFree(p.fault_buf);
  p.arena = nullptr;
  p.fault_buf = nullptr;
}

// Shared-memory carve for one replica (must match des.cu).
void layout_smem(sbs::DevPoint& d) {
  size_t off = 0;
  const size_t PD = (size_t)d.P * d.D, U = (size_t)d.U;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 16);
    return (int32_t)o;
  };
  // prefill warp's fields first (a prefix: the slice of a prefill-only CTA)
  d.sm_pf_out = take(8 * PD);
  d.sm_pf_head = take(4 * PD);
  d.sm_pf_tail = take(4 * PD);
  d.sm_pf_rel = take(4 * PD);
  d.sm_pf_part = take(PD);
  d.sm_wring = take(8 * (size_t)d.w_size);
  d.sm_wkeys = take(8 * (size_t)sbs::kSmemWinKeys);
  d.sm_cnt = take(256);
  // then the decode warp's (the slice of a decode-only CTA)
  d.sm_dec_begin = (int32_t)off;
  d.sm_dPK = take(8 * U);
  d.sm_dR = take(8 * U);
  d.sm_dS = take(4 * U);
  d.sm_dT = take(4 * U);
  d.sm_dnst = take(4 * U);
  d.sm_ulist = take(2 * U);
  d.sm_bcnt = take(2 * (size_t)d.Dn * d.R);
  d.sm_hist = take(4 * 256);
  d.sm_stage = take(16 * (size_t)sbs::kStageEntries * d.Dn);
  d.sm_cnt2 = take(256);
  d.sm_dec_end = (int32_t)off;
  d.sm_chan = take(sizeof(sbs::Chan));
  d.sm_bytes = (int32_t)off;
}

// Upper bounds of sample_length (workload.cpp:52-65) over a LengthSpec.
int64_t length_bound(const sbs_length_spec& l, bool output) {
  switch (l.dist) {
    case SBS_LEN_CONSTANT:
      return output ? std::max<int64_t>(0, l.value) : std::max<int64_t>(1, l.value);
    case SBS_LEN_UNIFORM:
      return std::max(std::max<int64_t>(1, l.min), l.max);
    default:
      return l.max;  // clamp(t, lo, max) = min(max(t, lo), max)
  }
}

// Shape bounds of every trace generate_workload can produce for `w`: what the
// arenas of a generated trace are sized by (a host trace uses its own maxima).
void bound_trace_shape(TraceDev& t, const sbs_workload& w) {
  t.max_output = (int32_t)std::min<int64_t>(std::max<int64_t>(0, length_bound(w.output, true)), 0x3fffffff);
  t.max_prompt = (int32_t)std::min<int64_t>(std::max<int64_t>(0, length_bound(w.prompt, false)), 0x3fffffff);
  if (w.shared_prefix_fraction > 0) {
    t.n_pools = w.prefix_pool;
    t.max_psize = std::max<int64_t>(0, std::min<int64_t>(w.prefix_len, length_bound(w.prompt, false)));
  }
}

// Requests in the trace the point's last launch read.
int64_t live_n(const sbs_sim& s, const PointHost& p) {
  const TraceDev& t = s.traces[p.trace];
  return t.gen ? t.h_stats[s.cur_slot].n : t.n;
}

void build_point(sbs_sim& s, PointHost& p) {
  const sbs_experiment& x = p.x;
  const sbs_cluster& c = x.cluster;
  const TraceDev& t = s.traces[p.trace];
  sbs::DevPoint& d = p.dp;
  std::memset(&d, 0, sizeof(d));
  d.P = c.n_instances_prefill;
  d.Dn = c.n_instances_decode;
  d.D = c.dp_degree;
  d.Dd = c.dp_degree_decode > 0 ? c.dp_degree_decode : c.dp_degree;
  d.U = d.Dn * d.Dd;
  d.policy = x.policy == SBS_POLICY_ROUND_ROBIN ? sbs::kImmediate : x.policy;
  d.decode_policy = x.decode_policy;
  d.n_limit = c.n_limit;
  d.cap_batch = c.decode_max_batch_per_dp;
  d.w_size = (int32_t)c.w_size;
  d.per_request = (s.flags & SBS_FLAG_PER_REQUEST) ? 1 : 0;
  d.log_kv_loads = ((s.flags & SBS_FLAG_LOGS) && (s.flags & SBS_FLAG_KV_LOADS)) ? 1 : 0;
  {
    const char* e = std::getenv("SBS_SPLIT");
    const bool allow = e == nullptr || std::atoi(e) != 0;
    // two-warp replicas (cache-aware points included: kernel variants 10/11
    // compile the cache into the prefill warp) whenever the trace has decode
    // work; run records (SBS_FLAG_LOGS) are kept by the one-warp kernels only
    d.split = (allow && p.split && !(s.flags & SBS_FLAG_LOGS) && t.max_output > 1) ? 1 : 0;
    p.prefill_only = t.max_output <= 1;
  }
  d.c_chunk = c.c_chunk;
  d.t_default = seconds_to_ns(c.t_default_s);
  d.l_net = seconds_to_ns(c.l_net_s);
  d.tps = c.decode_tokens_per_step;
  d.horizon = seconds_to_ns(x.workload.duration_s);
  d.warmup = seconds_to_ns(x.workload.duration_s * x.warmup_fraction);
  d.iqr_k = c.iqr_k;
  d.wd_mult = c.watchdog_multiplier;
  d.pf_base = c.prefill_base_s;
  d.pf_tok = c.prefill_per_token_s;
  d.dc_base = c.decode_base_s;
  d.dc_req = c.decode_per_request_s;
  d.dc_kv = c.decode_per_kv_token_s;
  d.rng_seed = x.seed ^ 0x9E3779B97F4A7C15ULL;
  d.N = t.n;
  d.n_dev = t.gen ? &t.d_stats[0].n : nullptr;
  d.arr = t.arr;
  d.prompt = t.prompt;
  d.output = t.output;
  // cache-aware PBAA (simulation.cpp:267-268: mode cache_aware AND cache on)
  d.cache_on = (x.prefill_mode == SBS_ALLOC_CACHE_AWARE && c.cache_enabled && t.pool != nullptr &&
                t.n_pools > 0) ? 1 : 0;
  if (d.cache_on) {
    // probe lengths ascending (core.cpp:15); a repeated length only re-touches
    // the entry it just inserted, which leaves the LRU order unchanged
    std::vector<int64_t> pr = p.probes;
    std::sort(pr.begin(), pr.end());
    pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
    d.n_probes = (int32_t)pr.size();
    for (size_t j = 0; j < pr.size(); ++j)
      d.probe_k[j] = (int32_t)std::min<int64_t>(pr[j], (int64_t)1 << 30);
    d.n_pools = t.n_pools;
    d.cache_budget = c.cache_budget_tokens;
    d.pfx_pool = t.pool;
    d.pfx_size = t.psize;
    // entries are keyed by (pool, probe); the reference keys them by a 64-bit
    // FNV hash of the tokens (core.cpp:18-31): refuse the (never observed)
    // case of two distinct prefixes hashing alike
    std::vector<uint64_t> hs;
    for (int pool = 0; pool < t.n_pools; ++pool)
      for (int64_t k : pr)
        if (k <= t.max_psize) hs.push_back(hash_pool_prefix(pool, k));
    std::sort(hs.begin(), hs.end());
    if (std::adjacent_find(hs.begin(), hs.end()) != hs.end())
      throw Error{SBS_ERR_CONFIG, "prefix hash collision between distinct cache keys"};
    if ((int64_t)t.n * d.n_probes >= ((int64_t)1 << 31))
      throw Error{SBS_ERR_CONFIG, "GPU path: requests x probe lengths must stay below 2^31"};
  }
  // decode completion ring: strictly more buckets than steps a request lives
  int64_t max_target = std::max<int64_t>(1, (int64_t)t.max_output - 1);
  int64_t max_steps = (max_target + c.decode_tokens_per_step - 1) / c.decode_tokens_per_step;
  d.R = (int32_t)next_pow2(max_steps + 1);
  if ((int64_t)d.R * d.Dn > (1 << 16)) throw Error{SBS_ERR_CONFIG, "decode ring too large"};
  // decode waiter key fields: length bits + id bits + output bits <= 64, else
  // the unpacked 32/32 layout (output and prompt then read from the trace)
  {
    auto bits = [](int64_t v) { int b = 0; while (b < 63 && (v >> b) != 0) ++b; return b; };
    const int64_t lmax = (int64_t)t.max_prompt + t.max_output;
    const int lb = bits(lmax), ib = std::max(1, bits(std::max<int64_t>(t.n, 1) - 1)),
              ob = std::max(1, bits(t.max_output));
    if (lb + ib + ob <= 64 && lmax <= 0xffffffffLL) {
      d.kq_ob = ob; d.kq_ib = ib; d.kq_lmax = (uint32_t)lmax;
    } else {
      d.kq_ob = 0; d.kq_ib = 32; d.kq_lmax = 0xffffffffu;
    }
  }

  // faults: deaths (min over entries), topology sorted by (time, order), drops
  const int n_inst = d.P + d.Dn;
  for (int i = 0; i < 2 * sbs::kMaxInstances; ++i) d.death[i] = INT64_MAX;
  for (auto& f : p.deads) {
    int64_t tt = seconds_to_ns(f.time_s);
    // instance ids: prefill 0..P-1 map to lanes 0..P-1, decode P.. map to slots P..
    d.death[f.instance] = std::min(d.death[f.instance], tt);
  }
  (void)n_inst;
  // remap decode deaths into slot P + j (already, since id = P + j)
  std::vector<std::pair<int64_t, int>> topo;
  for (size_t i = 0; i < p.topo.size(); ++i) topo.emplace_back(seconds_to_ns(p.topo[i].time_s), (int)i);
  std::stable_sort(topo.begin(), topo.end(),
                   [](auto& a, auto& b) { return a.first < b.first; });
  d.n_topo = (int32_t)topo.size();
  d.n_drops = (int32_t)p.drops.size();
  size_t fb = 8 * topo.size() + 8 * topo.size() + 16 * p.drops.size() + 8 * p.drops.size() + 64;
  if (p.fault_buf == nullptr) CUDA_OR_THROW(cudaMalloc(&p.fault_buf, fb));
  std::vector<unsigned char> hb(fb, 0);
  size_t off = 0;
  auto put = [&](const void* src, size_t bytes) {
    size_t o = off;
    std::memcpy(hb.data() + o, src, bytes);
    off = align_up(off + bytes, 8);
    return (unsigned char*)p.fault_buf + o;
  };
  std::vector<int64_t> tt(topo.size());
  std::vector<int32_t> ti(topo.size()), th(topo.size());
  for (size_t i = 0; i < topo.size(); ++i) {
    tt[i] = topo[i].first;
    ti[i] = p.topo[topo[i].second].instance;
    th[i] = p.topo[topo[i].second].healthy ? 1 : 0;
  }
  std::vector<int64_t> dfrom(p.drops.size()), duntil(p.drops.size());
  std::vector<int32_t> dinst(p.drops.size());
  for (size_t i = 0; i < p.drops.size(); ++i) {
    dfrom[i] = seconds_to_ns(p.drops[i].from_s);
    duntil[i] = std::isfinite(p.drops[i].until_s) ? seconds_to_ns(p.drops[i].until_s) : INT64_MAX;
    dinst[i] = p.drops[i].instance;
  }
  d.topo_time = (const int64_t*)put(tt.data(), 8 * tt.size());
  d.topo_inst = (const int32_t*)put(ti.data(), 4 * ti.size());
  d.topo_healthy = (const int32_t*)put(th.data(), 4 * th.size());
  d.drop_from = (const int64_t*)put(dfrom.data(), 8 * dfrom.size());
  d.drop_until = (const int64_t*)put(duntil.data(), 8 * duntil.size());
  d.drop_inst = (const int32_t*)put(dinst.data(), 4 * dinst.size());
  CUDA_OR_THROW(cudaMemcpy(p.fault_buf, hb.data(), fb, cudaMemcpyHostToDevice));

  // arena
  const int64_t N = std::max<int64_t>(t.n, 1);
  const int64_t PD = (int64_t)d.P * d.D;
  d.F = p.F;
  d.QP = p.QP;
  d.QW = p.QW;
  d.BC = p.BC;
  d.QD = p.QD;
  size_t sz = 0;
  auto carve = [&](size_t bytes) {
    size_t o = sz;
    sz = align_up(sz + bytes, 256);
    return o;
  };
  size_t o_disp = carve(8 * N), o_ps = carve(8 * N), o_ft = carve(8 * N);
  size_t o_comp = carve(8 * N);  // completion stamps (finalize_kernel reads them)
  size_t o_st = d.per_request ? carve(N) : 0;
  size_t o_ttft = carve(8 * N);
  size_t o_pk0 = carve(8 * (size_t)p.QP), o_pk1 = carve(8 * (size_t)p.QP);
  size_t o_pw0 = carve(4 * (size_t)p.QP), o_pw1 = carve(4 * (size_t)p.QP);
  size_t o_ws = carve(8 * (size_t)p.QW);
  size_t o_fifo = carve(8 * (size_t)PD * p.F);
  size_t o_bk = carve(16 * (size_t)d.Dn * d.R * p.BC);
  size_t o_dw = carve(8 * (size_t)p.QD);
  size_t o_mt = carve(8 * 312);
  size_t o_th = carve(8 * sbs::kHistBins);
  // two-warp replicas: the hand-off channel and the two warps' counters in HBM
  // (used when the pair runs as two kernels, pair mode 3)
  size_t o_gch = d.split ? carve(sizeof(sbs::Chan)) : 0;
  size_t o_gcn = d.split ? carve(512) : 0;
  const size_t n_keys = d.cache_on ? (size_t)d.n_pools * d.n_probes : 0;
  size_t o_cs = d.cache_on ? carve(4 * (size_t)PD * n_keys) : 0;
  size_t o_cu = d.cache_on ? carve(8 * (size_t)PD) : 0;
  size_t o_cc = d.cache_on ? carve(4 * (size_t)PD) : 0;
  const bool logs = (s.flags & SBS_FLAG_LOGS) != 0;
  size_t o_log = logs ? carve(8 * (size_t)p.LOG) : 0;
  if (p.arena == nullptr || p.arena_bytes < sz) {
    if (p.arena) cudaFree(p.arena);
    p.arena = nullptr;
    CUDA_OR_THROW(cudaMalloc(&p.arena, sz));
    p.arena_bytes = sz;
  }
  unsigned char* b = (unsigned char*)p.arena;
  d.o_dispatch = (int64_t*)(b + o_disp);
  d.o_pstart = (int64_t*)(b + o_ps);
  d.o_ftok = (int64_t*)(b + o_ft);
  d.o_comp = (int64_t*)(b + o_comp);
  d.o_status = d.per_request ? (int8_t*)(b + o_st) : nullptr;
  d.ttft = (int64_t*)(b + o_ttft);
  d.pend_key[0] = (uint64_t*)(b + o_pk0);
  d.pend_key[1] = (uint64_t*)(b + o_pk1);
  d.pend_wait[0] = (int32_t*)(b + o_pw0);
  d.pend_wait[1] = (int32_t*)(b + o_pw1);
  d.wscr = (uint64_t*)(b + o_ws);
  d.fifo = (int2*)(b + o_fifo);
  d.buckets = (int4*)(b + o_bk);
  d.dwait = (uint64_t*)(b + o_dw);
  d.mt = (uint64_t*)(b + o_mt);
  d.tpot_hist = (int64_t*)(b + o_th);
  d.gchan = d.split ? (sbs::Chan*)(b + o_gch) : nullptr;
  d.gcnt = d.split ? (int64_t*)(b + o_gcn) : nullptr;
  d.c_stamp = d.cache_on ? (int32_t*)(b + o_cs) : nullptr;
  d.c_used = d.cache_on ? (int64_t*)(b + o_cu) : nullptr;
  d.c_clock = d.cache_on ? (int32_t*)(b + o_cc) : nullptr;
  d.log = logs ? (int64_t*)(b + o_log) : nullptr;
  d.log_cap = logs ? p.LOG : 0;
  layout_smem(d);
  const double n_exp = t.gen ? t.spec.rate_qps * t.spec.duration_s + t.spec.initial_burst : (double)t.n;
  p.cost = n_exp * (1.0 + (double)d.U / 64.0) * (1.0 + (double)(d.P * d.D) / 256.0);
}

// Per-run reset of the parts of the arena the kernel reads before writing.
void reset_point(const PointHost& p, cudaStream_t st) {
  const sbs::DevPoint& d = p.dp;
  if (d.cache_on) {  // empty prefix caches
    const size_t PD = (size_t)d.P * d.D;
    CUDA_OR_THROW(cudaMemsetAsync(d.c_stamp, 0, 4 * PD * (size_t)d.n_pools * d.n_probes, st));
    CUDA_OR_THROW(cudaMemsetAsync(d.c_used, 0, 8 * PD, st));
    CUDA_OR_THROW(cudaMemsetAsync(d.c_clock, 0, 4 * PD, st));
  }
  if (d.per_request) {
    CUDA_OR_THROW(cudaMemsetAsync(d.o_dispatch, 0xff, 8 * (size_t)d.N, st));
    CUDA_OR_THROW(cudaMemsetAsync(d.o_pstart, 0xff, 8 * (size_t)d.N, st));
    CUDA_OR_THROW(cudaMemsetAsync(d.o_ftok, 0xff, 8 * (size_t)d.N, st));
    CUDA_OR_THROW(cudaMemsetAsync(d.o_status, 0, (size_t)d.N, st));
  }
}

void initial_caps(PointHost& p, const TraceDev& t) {
  const sbs_cluster& c = p.x.cluster;
  const int64_t PD = (int64_t)c.n_instances_prefill * c.dp_degree;
  if (p.x.policy == SBS_POLICY_SBS) {
    p.F = 256;
  } else {
    int64_t share = t.n / std::max<int64_t>(PD, 1) + 2;
    p.F = (int32_t)next_pow2(std::max<int64_t>(64, std::min<int64_t>(share * 2, 1 << 20)));
  }
  p.QP = 4096;
  p.QW = 4096;
  p.BC = 64;
  p.QD = 1024;
  // run records: ~ a pass + a step + a control sample per few requests
  p.LOG = std::max<int64_t>(1 << 16, t.n * (16 + 2 * (int64_t)c.dp_degree / 8));
}

void grow_caps(PointHost& p) {
  p.F = std::min<int32_t>(p.F * 2, 1 << 24);
  p.QP = std::min<int32_t>(p.QP * 2, 1 << 28);
  p.QW = std::min<int32_t>(p.QW * 2, 1 << 28);
  p.BC = std::min<int32_t>(p.BC * 2, 32768);
  p.QD = std::min<int32_t>(p.QD * 2, 1 << 28);
  p.LOG = std::min<int64_t>(p.LOG * 2, (int64_t)1 << 34);
}

int variant_of(const PointHost& p) {
  if (p.dp.split) return (4 | (p.dp.D > 32 ? 1 : 0)) + (p.dp.cache_on ? 6 : 0);
  // prefill-only SBS replicas without faults: the one-warp kernel with the
  // decode side and the baseline / fault paths compiled out (variants 12|13)
  if (p.prefill_only && p.dp.log == nullptr && !p.dp.cache_on && p.dp.policy == SBS_POLICY_SBS &&
      p.dp.n_drops == 0 && p.dp.n_topo == 0 && std::getenv("SBS_NO_PO") == nullptr) {
    bool alive = true;
    for (int q = 0; q < p.dp.P; ++q) alive = alive && p.dp.death[q] == INT64_MAX;
    if (alive) return 12 + (p.dp.D > 32 ? 1 : 0);
  }
  return (p.dp.D > 32 ? 1 : 0) + (p.dp.log != nullptr ? 2 : 0) + (p.dp.cache_on ? 6 : 0);
}

void order_points(sbs_sim& s) {
  const int n = (int)s.pts.size();
  s.order.resize(n);
  for (int i = 0; i < n; ++i) s.order[i] = i;
  std::stable_sort(s.order.begin(), s.order.end(), [&](int a, int b) {
    int va = variant_of(s.pts[a]), vb = variant_of(s.pts[b]);
    if (va != vb) return va < vb;
    return s.pts[a].cost > s.pts[b].cost;
  });
  for (int v = 0; v <= sbs_sim::kVariants; ++v) s.group_begin[v] = 0;
  for (int i = 0; i < n; ++i) s.group_begin[variant_of(s.pts[s.order[i]]) + 1] += 1;
  for (int v = 1; v <= sbs_sim::kVariants; ++v) s.group_begin[v] += s.group_begin[v - 1];
}

// Kernel variants whose replicas are warp pairs (prefill warp + decode warp).
bool is_pair_variant(int v) { return v == 4 || v == 5 || v == 10 || v == 11; }

// Pair mode 3: the group's prefill warps in one kernel on n_psm SMs (wp warps
// each: the prefill role idles about half the time), their decode warps in
// another on the remaining SMs (fewer decode warps per SM than a 2-CTA
// cluster gives), the channel in HBM.  Only when the group is the whole
// launch (the two kernels must be co-resident on every SM) and the slices
// fit; else the caller falls back to clusters.
bool launch_pair3(sbs_sim& s, int v, const sbs::DevPoint* dp, int b, int e, cudaStream_t vs) {
  for (int w = 0; w < sbs_sim::kVariants; ++w)
    if (w != v && s.group_begin[w + 1] > s.group_begin[w]) {
      if (std::getenv("SBS_DEBUG")) std::fprintf(stderr, "sbs: pair mode 3: other kernel groups, clusters\n");
      return false;
    }
  const int n = e - b;
  int slice_pf = 0, slice_dc = 0;
  bool simple = std::getenv("SBS_NO_SD") == nullptr;
  bool simple_p = std::getenv("SBS_NO_SP") == nullptr;
  for (int i = b; i < e; ++i) {
    const sbs::DevPoint& d = s.pts[s.order[i]].dp;
    slice_pf = std::max(slice_pf, d.sm_dec_begin);
    slice_dc = std::max(slice_dc, d.sm_dec_end - d.sm_dec_begin);
    // the specialised decode kernel: one decode instance, IQR, no cap, one
    // token per step, no decode topology events or deaths
    bool sd = d.Dn == 1 && d.decode_policy == sbs::kIqr && d.cap_batch <= 0 && d.tps == 1 &&
              d.death[d.P] == INT64_MAX && d.U <= 512;
    for (const auto& f : s.pts[s.order[i]].topo) sd = sd && f.instance < d.P;
    simple = simple && sd;
    // the specialised prefill kernel: SBS, no drops, no topology events, no prefill deaths
    bool sp = d.policy == SBS_POLICY_SBS && d.n_drops == 0 && d.n_topo == 0;
    for (int q = 0; q < d.P; ++q) sp = sp && d.death[q] == INT64_MAX;
    simple_p = simple_p && sp;
  }
  slice_pf = (int)align_up((size_t)slice_pf, 128);
  slice_dc = (int)align_up((size_t)slice_dc, 128);
  const char* ew = std::getenv("SBS_WP");
  // 10 prefill warps per prefill SM measured best on the cfg5 slice (512 pairs
  // on 52 + 96 SMs: 155.7 vs 146.3 M sim-req/s as clusters; 12 per SM makes
  // the prefill side the limit, `profiles/r02_pair3_geometry.txt`)
  int wp = ew ? std::atoi(ew) : 10;
  while (wp > 1 && (size_t)wp * slice_pf > 227 * 1024) --wp;
  int n_psm = (n + wp - 1) / wp;
  if (const char* es = std::getenv("SBS_PSM")) {  // (dev: explicit prefill SM count)
    n_psm = std::max(1, std::atoi(es));
    wp = (n + n_psm - 1) / n_psm;
    if (wp > 12 || (size_t)wp * slice_pf > 227 * 1024) return false;
  }
  if (n_psm >= s.sm_count) return false;
  const int n_dsm = s.sm_count - n_psm;
  int wd = std::min(8, (n + n_dsm - 1) / n_dsm);
  while (wd > 1 && (size_t)wd * slice_dc > 227 * 1024) --wd;
  if (s.d_sync == nullptr) CUDA_OR_THROW(cudaMalloc(&s.d_sync, 2 * sizeof(int)));
  cudaStream_t st2 = s.vstream2[v];
  CUDA_OR_THROW(cudaStreamWaitEvent(st2, s.ev_des[0], 0));
  const cudaError_t err = sbs::launch_des_pair3(v, dp + b, n, s.d_res + b, slice_pf, slice_dc, n_psm, wp,
                                                n_dsm, wd, s.d_sync, vs, st2, simple, simple_p);
  if (std::getenv("SBS_DEBUG"))
    std::fprintf(stderr, "sbs: pair mode 3: %d replicas, prefill %d SMs x %d warps (slice %d B), decode %d SMs x %d warps (slice %d B): %s\n",
                 n, n_psm, wp, slice_pf, n_dsm, wd, slice_dc, cudaGetErrorString(err));
  if (err == cudaErrorInvalidValue) return false;
  CUDA_OR_THROW(err);
  // join the decode kernel's stream into the group's
  cudaEvent_t ev;
  CUDA_OR_THROW(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_OR_THROW(cudaEventRecord(ev, st2));
  CUDA_OR_THROW(cudaStreamWaitEvent(vs, ev, 0));
  CUDA_OR_THROW(cudaEventDestroy(ev));
  s.pair3_used = 1;
  s.n_launches += 1;  // (two kernels for the group)
  return true;
}

void launch_all(sbs_sim& s, cudaStream_t st) {
  s.n_launches = 0;
  s.pair3_used = 0;
  const sbs::DevPoint* dp = s.cur_slot ? s.d_pts1 : s.d_pts;
  if (s.ev_des[0] == nullptr) {
    CUDA_OR_THROW(cudaEventCreate(&s.ev_des[0]));
    CUDA_OR_THROW(cudaEventCreate(&s.ev_des[1]));
    for (int v = 0; v < sbs_sim::kVariants; ++v) {
      CUDA_OR_THROW(cudaStreamCreateWithFlags(&s.vstream[v], cudaStreamNonBlocking));
      CUDA_OR_THROW(cudaStreamCreateWithFlags(&s.vstream2[v], cudaStreamNonBlocking));
      CUDA_OR_THROW(cudaEventCreateWithFlags(&s.ev_join[v], cudaEventDisableTiming));
    }
  }
  // Geometry of the one-warp-per-replica groups: when all their CTAs fit one
  // per SM, reserve enough shared memory that no SM takes two (the block
  // scheduler would otherwise pack them and leave SMs idle).
  int total_blocks = 0;
  for (int v = 0; v < sbs_sim::kVariants; ++v) {
    const int n = s.group_begin[v + 1] - s.group_begin[v];
    if (n <= 0 || (is_pair_variant(v) && s.pair_mode >= 2)) continue;
    const int per = is_pair_variant(v) ? std::max(1, std::min(4, (n + s.sm_count - 1) / s.sm_count))
                                       : s.warps_per_block;
    total_blocks += (n + per - 1) / per;
  }
  const int min_smem = total_blocks <= s.sm_count ? 116 * 1024 : 0;
  // completion stamps := unset, every replica in one launch (finalize_kernel
  // derives the completion-based aggregates from them)
  CUDA_OR_THROW(sbs::launch_reset(dp, (int)s.order.size(), s.d_res, st));
  s.n_launches += 1;
  CUDA_OR_THROW(cudaEventRecord(s.ev_des[0], st));
  int used[sbs_sim::kVariants] = {};
  for (int v = 0; v < sbs_sim::kVariants; ++v) {
    const int b = s.group_begin[v], e = s.group_begin[v + 1];
    if (e <= b) continue;
    // fork: each variant group on its own stream after everything queued on st
    cudaStream_t vs = s.vstream[v];
    CUDA_OR_THROW(cudaStreamWaitEvent(vs, s.ev_des[0], 0));
    used[v] = 1;
    int wpb = s.warps_per_block, per_block = wpb;
    bool done = false;
    if (is_pair_variant(v) && s.pair_mode == 3) done = launch_pair3(s, v, dp, b, e, vs);
    if (done) {
      // (launched)
    } else if (is_pair_variant(v) && s.pair_mode >= 2) {  // replica = a CTA pair of a 2-CTA cluster
      CUDA_OR_THROW(sbs::launch_des_cluster(v, dp + b, e - b, s.d_res + b, s.smem_per_warp, vs));
    } else {
      if (is_pair_variant(v)) {  // two warps per replica; up to four replicas per block
        int rpb = std::max(1, std::min(4, (e - b + s.sm_count - 1) / s.sm_count));
        while (rpb > 1 && (size_t)rpb * s.smem_per_warp > 227 * 1024) --rpb;
        wpb = 2 * rpb;
        per_block = rpb;
      }
      const int blocks = std::max(1, (e - b + per_block - 1) / per_block);
      CUDA_OR_THROW(sbs::launch_des(v, dp + b, e - b, s.d_counter + v, s.d_res + b,
                                    s.smem_per_warp, wpb, blocks, min_smem, vs));
    }
    CUDA_OR_THROW(cudaEventRecord(s.ev_join[v], vs));
    s.n_launches += 1;
  }
  for (int v = 0; v < sbs_sim::kVariants; ++v)  // join
    if (used[v]) CUDA_OR_THROW(cudaStreamWaitEvent(st, s.ev_join[v], 0));
  CUDA_OR_THROW(cudaEventRecord(s.ev_des[1], st));
  CUDA_OR_THROW(sbs::launch_finalize(dp, (int)s.order.size(), s.d_res, st));
  s.n_launches += 1;
}

void upload_points(sbs_sim& s) {
  std::vector<sbs::DevPoint> h(s.order.size());
  int smem = 0;
  for (size_t i = 0; i < s.order.size(); ++i) {
    h[i] = s.pts[s.order[i]].dp;
    smem = std::max(smem, h[i].sm_bytes);
  }
  s.smem_per_warp = (int)align_up((size_t)smem, 128);
  CUDA_OR_THROW(cudaMemcpy(s.d_pts, h.data(), sizeof(sbs::DevPoint) * h.size(),
                           cudaMemcpyHostToDevice));
  if (s.n_slots == 2) {  // the same points reading trace set 1
    for (size_t i = 0; i < h.size(); ++i) {
      const TraceDev& t = s.traces[s.pts[s.order[i]].trace];
      h[i].arr = t.arr1;
      h[i].prompt = t.prompt1;
      h[i].output = t.output1;
      if (t.gen) h[i].n_dev = &t.d_stats[1].n;
      if (h[i].cache_on) {
        h[i].pfx_pool = t.pool1;
        h[i].pfx_size = t.psize1;
      }
    }
    CUDA_OR_THROW(cudaMemcpy(s.d_pts1, h.data(), sizeof(sbs::DevPoint) * h.size(),
                             cudaMemcpyHostToDevice));
  }
  // occupancy: warps per block 4 unless shared memory forces fewer
  const int max_smem_block = 227 * 1024;
  // spread replicas over every SM first: warps of one SM share its issue
  // slots, L1.5 instruction cache and shared-memory pipe (4 per SM at most)
  const int n_rep = (int)s.order.size();
  int wpb = std::max(1, std::min(4, (n_rep + s.sm_count - 1) / std::max(1, s.sm_count)));
  if (const char* e = std::getenv("SBS_WARPS_PER_BLOCK")) wpb = std::max(1, std::min(4, std::atoi(e)));
  while (wpb > 1 && wpb * s.smem_per_warp > max_smem_block) wpb >>= 1;
  if (s.smem_per_warp > max_smem_block)
    throw Error{SBS_ERR_CONFIG, "replica state exceeds shared memory"};
  s.warps_per_block = wpb;
  int blocks_per_sm = std::max(1, std::min(16, (228 * 1024) / std::max(1, wpb * s.smem_per_warp + 1024)));
  int max_blocks = s.sm_count * blocks_per_sm;
  int need = (int)((s.order.size() + wpb - 1) / wpb);
  s.n_blocks = std::max(1, std::min(need, max_blocks));
}

// Host source readable by the device (pinned memory under unified addressing)?
bool device_readable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

// One gather launch when every source is pinned host memory; false otherwise.
bool upload_traces_gather(sbs_sim& s, const sbs_trace* traces, int slot, cudaStream_t st) {
  std::vector<sbs::CopySeg> segs;
  for (size_t i = 0; i < s.traces.size(); ++i) {
    const TraceDev& t = s.traces[i];
    if (t.n == 0) continue;
    const void* src[5] = {traces[i].arrival_ns, traces[i].prompt_len, traces[i].output_len,
                          traces[i].prefix_pool_id, traces[i].prefix_size};
    void* dst[5] = {slot ? (void*)t.arr1 : t.arr, slot ? (void*)t.prompt1 : t.prompt,
                    slot ? (void*)t.output1 : t.output, slot ? (void*)t.pool1 : t.pool,
                    slot ? (void*)t.psize1 : t.psize};
    const int64_t bytes[5] = {8 * t.n, 4 * t.n, 4 * t.n, 4 * t.n, 4 * t.n};
    for (int k = 0; k < 5; ++k) {
      if (dst[k] == nullptr) continue;
      if (!device_readable(src[k])) return false;
      segs.push_back({(const unsigned char*)src[k], (unsigned char*)dst[k], bytes[k]});
    }
  }
  if (segs.empty()) return true;
  // the previous gather has finished reading its host sources and table (the
  // Python wrapper keeps those host buffers alive until this returns)
  if (s.ev_segs) CUDA_OR_THROW(cudaEventSynchronize(s.ev_segs));
  if ((int)segs.size() > s.seg_cap) {
    if (s.h_segs) cudaFreeHost(s.h_segs);
    if (s.d_segs) cudaFree(s.d_segs);
    s.seg_cap = (int)segs.size();
    CUDA_OR_THROW(cudaMallocHost(&s.h_segs, sizeof(sbs::CopySeg) * s.seg_cap));
    CUDA_OR_THROW(cudaMalloc(&s.d_segs, sizeof(sbs::CopySeg) * s.seg_cap));
    if (s.ev_segs == nullptr) CUDA_OR_THROW(cudaEventCreateWithFlags(&s.ev_segs, cudaEventDisableTiming));
  }
  int64_t blocks = 0;
  for (size_t k = 0; k < segs.size(); ++k) {
    s.h_segs[k] = segs[k];
    blocks += (segs[k].bytes + (1 << 16) - 1) >> 16;
  }
  CUDA_OR_THROW(cudaMemcpyAsync(s.d_segs, s.h_segs, sizeof(sbs::CopySeg) * segs.size(),
                                cudaMemcpyHostToDevice, st));
  CUDA_OR_THROW(sbs::launch_gather(s.d_segs, (int)segs.size(), blocks, st));
  CUDA_OR_THROW(cudaEventRecord(s.ev_segs, st));
  return true;
}

int parallel_threads();

// A re-uploaded trace must fit what the points' arenas were sized for at
// create time: its length, the completion ring (max output), the prefix-cache
// key space (pool ids, prefix sizes).  Anything else is refused, never wrapped.
void check_reupload(const TraceDev& t, const sbs_trace& tr) {
  if (tr.n != t.n) throw Error{SBS_ERR_CONFIG, "trace shape changed (length)"};
  if ((tr.prefix_pool_id != nullptr) != (t.pool != nullptr))
    throw Error{SBS_ERR_CONFIG, "trace shape changed (shared prefixes)"};
  int32_t mo = 0, mp = 0;
  for (int64_t k = 0; k < tr.n; ++k) mo = std::max(mo, tr.output_len[k]);
  for (int64_t k = 0; k < tr.n; ++k) mp = std::max(mp, tr.prompt_len[k]);
  if (mo > t.max_output || mp > t.max_prompt)
    throw Error{SBS_ERR_CONFIG, "re-uploaded trace has longer prompts or outputs than the one the "
                                "simulator was created with (completion ring, waiter keys); create a "
                                "new simulator"};
  if (tr.prefix_pool_id != nullptr) {
    for (int64_t k = 0; k < tr.n; ++k) {
      const int32_t pid = tr.prefix_pool_id[k], ps = tr.prefix_size[k];
      if (ps < 0 || (ps > 0 && pid < 0) || ps > tr.prompt_len[k])
        throw Error{SBS_ERR_CONFIG, "trace prefix sizes out of range"};
      if (ps > 0 && (pid >= t.n_pools || ps > t.max_psize))
        throw Error{SBS_ERR_CONFIG, "re-uploaded trace uses prefix pools / sizes beyond the "
                                    "create-time trace (prefix-cache key space)"};
    }
  }
}

void do_upload_traces(sbs_sim& s, const sbs_trace* traces, cudaStream_t st, int slot = 0,
                      bool check = true) {
  if (s.generated) throw Error{SBS_ERR_CONFIG, "traces of this simulator are generated on the device"};
  if (check) {  // one O(n) scan per trace, traces spread over the host threads
    const size_t nt = s.traces.size();
    const int nth = (int)std::min<size_t>(nt, (size_t)parallel_threads());
    std::vector<std::string> errs(nt);
    std::atomic<size_t> next{0};
    auto work = [&] {
      for (size_t i; (i = next.fetch_add(1)) < nt;) {
        try {
          check_reupload(s.traces[i], traces[i]);
        } catch (const Error& e) {
          errs[i] = e.msg;
        }
      }
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nth; ++k) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw Error{SBS_ERR_CONFIG, e};
  }
  if (slot < 0 || slot >= s.n_slots) throw Error{SBS_ERR_CONFIG, "trace slot out of range"};
  if (s.traces.size() > 1 && upload_traces_gather(s, traces, slot, st)) return;
  for (size_t i = 0; i < s.traces.size(); ++i) {
    TraceDev& t = s.traces[i];
    if (t.n == 0) continue;
    CUDA_OR_THROW(cudaMemcpyAsync(slot ? t.arr1 : t.arr, traces[i].arrival_ns, 8 * t.n,
                                  cudaMemcpyHostToDevice, st));
    CUDA_OR_THROW(cudaMemcpyAsync(slot ? t.prompt1 : t.prompt, traces[i].prompt_len, 4 * t.n,
                                  cudaMemcpyHostToDevice, st));
    CUDA_OR_THROW(cudaMemcpyAsync(slot ? t.output1 : t.output, traces[i].output_len, 4 * t.n,
                                  cudaMemcpyHostToDevice, st));
    if (t.pool) {
      CUDA_OR_THROW(cudaMemcpyAsync(slot ? t.pool1 : t.pool, traces[i].prefix_pool_id, 4 * t.n,
                                    cudaMemcpyHostToDevice, st));
      CUDA_OR_THROW(cudaMemcpyAsync(slot ? t.psize1 : t.psize, traces[i].prefix_size, 4 * t.n,
                                    cudaMemcpyHostToDevice, st));
    }
  }
}

void finish_aggregates(const PointHost& p, const sbs::DevResult& r, sbs_aggregates& a, int64_t N) {
  std::memset(&a, 0, sizeof(a));
  const sbs::DevPoint& d = p.dp;
  a.generated = (uint64_t)N;
  a.completed = (uint64_t)r.completed;
  a.throttled = (uint64_t)r.throttled;
  a.in_flight = (uint64_t)(N - r.completed - r.throttled);
  a.window_requests = (uint64_t)r.wr;
  a.warmup_cutoff_s = (double)d.warmup / 1e9;
  a.duration_s = (double)d.horizon / 1e9;
  if (r.wr > 0) {
    const double n = (double)r.wr;
    a.ttft_mean_s = ((double)r.ttft_sum / 1e9) / n;
    a.scheduler_wait_mean_s = ((double)r.sched_sum / 1e9) / n;
    a.device_wait_mean_s = ((double)r.dev_sum / 1e9) / n;
    a.total_wait_mean_s = ((double)r.sched_sum / 1e9 + (double)r.dev_sum / 1e9) / n;
    // percentile (decode_alloc.cpp:13-23) from exact order statistics
    auto pct = [&](int which, double pv) {
      double rank = (n - 1.0) * pv / 100.0;
      size_t lo = (size_t)std::floor(rank), hi = (size_t)std::ceil(rank);
      double vlo = (double)r.ttft_sel[2 * which] / 1e9;
      if (lo == hi) return vlo;
      double vhi = (double)r.ttft_sel[2 * which + 1] / 1e9;
      double frac = rank - (double)lo;
      return vlo + frac * (vhi - vlo);
    };
    a.ttft_p50_s = pct(0, 50.0);
    a.ttft_p95_s = pct(1, 95.0);
  }
  a.passes = (uint64_t)r.passes;
  if (r.passes > 0) a.chunk_util_mean = r.util_sum / (double)r.passes;
  a.decode_steps = (uint64_t)r.steps;
  a.output_tokens = (uint64_t)r.out_tokens;
  double window_s = (double)(d.horizon - d.warmup) / 1e9;
  if (window_s > 0) {
    a.output_tokens_per_s = (double)a.output_tokens / window_s;
    a.completed_per_s = (double)r.cw / window_s;
  }
  if (r.kv_n > 0) {
    a.kv_mean_time_avg = r.kv_mean_sum / (double)r.kv_n;
    a.kv_sigma_time_avg = r.kv_sigma_sum / (double)r.kv_n;
  }
  a.watchdog_fires = (uint64_t)r.wd_fires;
  a.dropped_end_forwards = (uint64_t)r.dropped;
  a.rejected_samples = (uint64_t)r.rejected;
  a.deferrals = (uint64_t)r.deferrals;
  a.flow_control_events = (uint64_t)r.flow;
  a.mask_events = (uint64_t)r.mask;
  a.fallback_events = (uint64_t)r.fallback;
  a.alloc_calls = (uint64_t)r.alloc_calls;
  a.decode_selects = (uint64_t)r.dec_selects;
  a.events = (uint64_t)r.events;
  a.tpot_count = (uint64_t)r.tpot_n;
  if (r.tpot_n > 0) a.tpot_mean_s = r.tpot_sum / (double)r.tpot_n;
  a.ttft_sum_ns = r.ttft_sum;
  a.sched_sum_ns = r.sched_sum;
  a.device_sum_ns = r.dev_sum;
  a.error = r.error;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SBS_ERR_OVERFLOW;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SBS_ERR_INVARIANT;
  }
}

int parallel_threads() {
  unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, hc);
}

// Per-thread, per-device error flag for the allocation kernels (allocated
// once: a per-call cudaMallocAsync costs milliseconds once the pool trims).
struct Scratch {
  int device = -1;
  int32_t* d_err = nullptr;
  int32_t* h_err = nullptr;
};
Scratch& scratch() {
  thread_local Scratch sc[16];
  int dev = 0;
  CUDA_OR_THROW(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) throw Error{SBS_ERR_CUDA, "device ordinal above 15"};
  Scratch& s = sc[dev];
  if (s.d_err == nullptr) {
    CUDA_OR_THROW(cudaMalloc(&s.d_err, sizeof(int32_t)));
    CUDA_OR_THROW(cudaMallocHost(&s.h_err, sizeof(int32_t)));
    s.device = dev;
  }
  return s;
}

}  // namespace

extern "C" {

const char* sbs_last_error(void) { return g_err.c_str(); }
const char* sbs_version(void) { return "sbs_b200 0.1 (sm_100a)"; }

int sbs_generate_workload(const sbs_workload* spec, uint64_t seed, int64_t* arrival_ns,
                          int32_t* prompt_len, int32_t* output_len, int32_t* prefix_pool_id,
                          int32_t* prefix_size, int64_t cap, int64_t* n_out, uint64_t* digest) {
  return guarded([&] {
    HostTrace t;
    generate(*spec, seed, t);
    if (n_out) *n_out = (int64_t)t.arr.size();
    if (digest) *digest = t.digest;
    if (arrival_ns == nullptr) return SBS_OK;
    if ((int64_t)t.arr.size() > cap) return fail(SBS_ERR_OVERFLOW, "trace capacity too small");
    std::memcpy(arrival_ns, t.arr.data(), 8 * t.arr.size());
    std::memcpy(prompt_len, t.prompt.data(), 4 * t.prompt.size());
    std::memcpy(output_len, t.output.data(), 4 * t.output.size());
    const size_t n = t.arr.size();
    for (size_t i = 0; i < n; ++i) {
      if (prefix_pool_id) prefix_pool_id[i] = t.pool.empty() ? -1 : t.pool[i];
      if (prefix_size) prefix_size[i] = t.psize.empty() ? 0 : t.psize[i];
    }
    return SBS_OK;
  });
}

int64_t sbs_workload_capacity(const sbs_workload* w) {
  const double burst = w->initial_burst > 0 ? (double)w->initial_burst : 0.0;
  const double slots = std::ceil(w->duration_s * w->rate_qps);
  double cap;
  if (w->process == SBS_ARRIVAL_POISSON)
    cap = burst + slots + 8.0 * std::sqrt(slots) + 64.0;
  else
    cap = burst + slots + 2.0;
  if (!(cap < 2147483647.0)) return (int64_t)1 << 31;
  return (int64_t)cap;
}

int sbs_generate_workload_device(const sbs_gen_job* jobs, int32_t n_jobs, const uint64_t* seeds,
                                 int32_t want_digest, void* stream) {
  return guarded([&] {
    if (n_jobs <= 0) return SBS_OK;
    for (int i = 0; i < n_jobs; ++i) {
      check_workload(jobs[i].spec);
      const sbs_workload& w = jobs[i].spec;
      if (w.process < 0 || w.process > SBS_ARRIVAL_UNIFORM_JITTER)
        return fail(SBS_ERR_CONFIG, "workload.process must be poisson, uniform, or uniform_jitter");
      if (w.shared_prefix_fraction > 0 && (!jobs[i].prefix_pool_id || !jobs[i].prefix_size))
        return fail(SBS_ERR_CONFIG, "shared prefixes need prefix_pool_id / prefix_size arrays");
      if (!jobs[i].arrival_ns || !jobs[i].prompt_len || !jobs[i].output_len || !jobs[i].stats)
        return fail(SBS_ERR_CONFIG, "sbs_gen_job: NULL output array");
    }
    cudaStream_t st = (cudaStream_t)stream;
    sbs_gen_job* d_jobs = nullptr;
    const size_t bytes = sizeof(sbs_gen_job) * (size_t)n_jobs;
    CUDA_OR_THROW(cudaMallocAsync((void**)&d_jobs, bytes, st));
    CUDA_OR_THROW(cudaMemcpyAsync(d_jobs, jobs, bytes, cudaMemcpyHostToDevice, st));
    CUDA_OR_THROW(sbs::launch_gen(d_jobs, n_jobs, seeds, want_digest, st));
    CUDA_OR_THROW(cudaFreeAsync(d_jobs, st));
    return SBS_OK;
  });
}

}  // extern "C"

namespace {

void open_device(sbs_sim* s, const sbs_experiment* points, int32_t n_points, uint32_t flags,
                 int32_t device) {
  if (n_points < 1) throw Error{SBS_ERR_CONFIG, "no points"};
  for (int i = 0; i < n_points; ++i) {
    validate(points[i]);
    check_workload(points[i].workload);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error{SBS_ERR_CUDA, "no CUDA device visible (the GPU path has no CPU fallback)"};
  if (device < 0 || device >= ndev) throw Error{SBS_ERR_CONFIG, "device index out of range"};
  s->device = device;
  s->flags = flags;
  CUDA_OR_THROW(cudaSetDevice(device));
  CUDA_OR_THROW(cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, device));
  if (const char* e = std::getenv("SBS_SPLIT")) {
    const int m = std::atoi(e);
    s->pair_mode = m == 1 ? 1 : m == 2 ? 2 : 3;
  }
}

void alloc_trace(sbs_sim* s, TraceDev& t, bool prefixes) {
  const size_t n = (size_t)std::max<int64_t>(t.n, 1);
  CUDA_OR_THROW(cudaMalloc(&t.arr, 8 * n));
  CUDA_OR_THROW(cudaMalloc(&t.prompt, 4 * n));
  CUDA_OR_THROW(cudaMalloc(&t.output, 4 * n));
  s->device_bytes += (int64_t)(16 * n);
  if (prefixes) {
    CUDA_OR_THROW(cudaMalloc(&t.pool, 4 * n));
    CUDA_OR_THROW(cudaMalloc(&t.psize, 4 * n));
    s->device_bytes += (int64_t)(8 * n);
  }
}

void init_points(sbs_sim* s, const sbs_experiment* points, int32_t n_points,
                 const int32_t* trace_of_point, int32_t n_traces) {
  s->pts.resize(n_points);
  for (int i = 0; i < n_points; ++i) {
    PointHost& p = s->pts[i];
    p.x = points[i];
    p.drops.assign(points[i].drops, points[i].drops + points[i].n_drops);
    p.deads.assign(points[i].deads, points[i].deads + points[i].n_deads);
    p.topo.assign(points[i].topology, points[i].topology + points[i].n_topology);
    if (p.x.cluster.cache_enabled)
      p.probes.assign(points[i].cluster.cache_probe_lens,
                      points[i].cluster.cache_probe_lens + points[i].cluster.cache_n_probes);
    p.x.cluster.cache_probe_lens = p.probes.empty() ? nullptr : p.probes.data();
    p.trace = trace_of_point ? trace_of_point[i] : i;
    if (p.trace < 0 || p.trace >= n_traces) throw Error{SBS_ERR_CONFIG, "trace index out of range"};
    initial_caps(p, s->traces[p.trace]);
    build_point(*s, p);
    s->device_bytes += (int64_t)p.arena_bytes;
  }
  order_points(*s);
  CUDA_OR_THROW(cudaMalloc(&s->d_pts, sizeof(sbs::DevPoint) * n_points));
  CUDA_OR_THROW(cudaMalloc(&s->d_res, sizeof(sbs::DevResult) * n_points));
  CUDA_OR_THROW(cudaMalloc(&s->d_counter, sbs_sim::kVariants * sizeof(int)));
  s->h_res.resize(n_points);
  upload_points(*s);
}

// The generation jobs of one trace slot (device array, seeds from d_seeds).
void upload_gen_jobs(sbs_sim* s, int slot) {
  std::vector<sbs_gen_job> jobs(s->traces.size());
  for (size_t i = 0; i < s->traces.size(); ++i) {
    TraceDev& t = s->traces[i];
    sbs_gen_job& j = jobs[i];
    std::memset(&j, 0, sizeof(j));
    j.spec = t.spec;
    j.seed = t.seed;
    j.cap = t.n;
    j.arrival_ns = slot ? t.arr1 : t.arr;
    j.prompt_len = slot ? t.prompt1 : t.prompt;
    j.output_len = slot ? t.output1 : t.output;
    j.prefix_pool_id = slot ? t.pool1 : t.pool;
    j.prefix_size = slot ? t.psize1 : t.psize;
    j.stats = &t.d_stats[slot];
  }
  if (s->d_jobs[slot] == nullptr) {
    CUDA_OR_THROW(cudaMalloc(&s->d_jobs[slot], sizeof(sbs_gen_job) * jobs.size()));
    CUDA_OR_THROW(cudaMalloc(&s->d_seeds[slot], sizeof(uint64_t) * jobs.size()));
    CUDA_OR_THROW(cudaMallocHost(&s->h_seeds[slot], sizeof(uint64_t) * jobs.size()));
    CUDA_OR_THROW(cudaEventCreateWithFlags(&s->ev_seeds[slot], cudaEventDisableTiming));
    CUDA_OR_THROW(cudaEventRecord(s->ev_seeds[slot], 0));
  }
  CUDA_OR_THROW(cudaMemcpy(s->d_jobs[slot], jobs.data(), sizeof(sbs_gen_job) * jobs.size(),
                           cudaMemcpyHostToDevice));
}

void generate_slot(sbs_sim* s, const uint64_t* seeds, int slot, int want_digest, cudaStream_t st) {
  const size_t n = s->traces.size();
  CUDA_OR_THROW(cudaEventSynchronize(s->ev_seeds[slot]));  // staging buffer free again
  for (size_t i = 0; i < n; ++i) s->h_seeds[slot][i] = seeds ? seeds[i] : s->traces[i].seed;
  CUDA_OR_THROW(cudaMemcpyAsync(s->d_seeds[slot], s->h_seeds[slot], sizeof(uint64_t) * n,
                                cudaMemcpyHostToDevice, st));
  CUDA_OR_THROW(cudaEventRecord(s->ev_seeds[slot], st));
  CUDA_OR_THROW(sbs::launch_gen(s->d_jobs[slot], (int)n, s->d_seeds[slot], want_digest, st));
  s->gen_slot_valid[slot] = 0;
}

}  // namespace

extern "C" {

int sbs_sim_create(const sbs_experiment* points, int32_t n_points, const sbs_trace* traces,
                   int32_t n_traces, const int32_t* trace_of_point, uint32_t flags,
                   int32_t device, sbs_sim** out) {
  *out = nullptr;
  sbs_sim* s = new sbs_sim();
  int rc = guarded([&] {
    open_device(s, points, n_points, flags, device);
    s->traces.resize(n_traces);
    for (int i = 0; i < n_traces; ++i) {
      TraceDev& t = s->traces[i];
      t.n = traces[i].n;
      t.digest = traces[i].digest;
      if (t.n >= (int64_t)1 << 31) throw Error{SBS_ERR_CONFIG, "trace longer than 2^31 requests"};
      for (int64_t k = 0; k < t.n; ++k) t.max_output = std::max(t.max_output, traces[i].output_len[k]);
      for (int64_t k = 0; k < t.n; ++k) t.max_prompt = std::max(t.max_prompt, traces[i].prompt_len[k]);
      const bool prefixes = traces[i].prefix_pool_id != nullptr && traces[i].prefix_size != nullptr;
      if (prefixes) {
        for (int64_t k = 0; k < t.n; ++k) {
          const int32_t pid = traces[i].prefix_pool_id[k], ps = traces[i].prefix_size[k];
          if (ps < 0 || (ps > 0 && pid < 0) || ps > traces[i].prompt_len[k])
            throw Error{SBS_ERR_CONFIG, "trace prefix sizes out of range"};
          if (ps > 0) {
            t.n_pools = std::max(t.n_pools, pid + 1);
            t.max_psize = std::max<int64_t>(t.max_psize, ps);
          }
        }
      }
      alloc_trace(s, t, prefixes);
    }
    do_upload_traces(*s, traces, 0, 0, false);
    CUDA_OR_THROW(cudaDeviceSynchronize());
    init_points(s, points, n_points, trace_of_point, n_traces);
    return SBS_OK;
  });
  if (rc != SBS_OK) {
    sbs_sim_destroy(s);
    return rc;
  }
  *out = s;
  return SBS_OK;
}

int sbs_sim_create_generated(const sbs_experiment* points, int32_t n_points,
                             const int32_t* trace_of_point, int32_t n_traces, uint32_t flags,
                             int32_t device, sbs_sim** out) {
  *out = nullptr;
  sbs_sim* s = new sbs_sim();
  int rc = guarded([&] {
    open_device(s, points, n_points, flags, device);
    if (trace_of_point == nullptr) n_traces = n_points;
    if (n_traces < 1) throw Error{SBS_ERR_CONFIG, "no traces"};
    s->generated = true;
    s->traces.resize(n_traces);
    std::vector<int> first(n_traces, -1);
    for (int i = 0; i < n_points; ++i) {
      const int t = trace_of_point ? trace_of_point[i] : i;
      if (t < 0 || t >= n_traces) throw Error{SBS_ERR_CONFIG, "trace index out of range"};
      if (first[t] < 0) first[t] = i;
      else if (std::memcmp(&points[i].workload, &points[first[t]].workload, sizeof(sbs_workload)) != 0 ||
               points[i].seed != points[first[t]].seed)
        throw Error{SBS_ERR_CONFIG, "points sharing a trace must share workload and seed"};
    }
    for (int i = 0; i < n_traces; ++i) {
      if (first[i] < 0) throw Error{SBS_ERR_CONFIG, "a trace no point uses"};
      TraceDev& t = s->traces[i];
      t.gen = true;
      t.spec = points[first[i]].workload;
      t.seed = points[first[i]].seed;
      t.n = sbs_workload_capacity(&t.spec);
      if (t.n >= (int64_t)1 << 31) throw Error{SBS_ERR_CONFIG, "trace longer than 2^31 requests"};
      bound_trace_shape(t, t.spec);
      alloc_trace(s, t, t.spec.shared_prefix_fraction > 0);
      CUDA_OR_THROW(cudaMalloc(&t.d_stats, 2 * sizeof(sbs_gen_stats)));
      CUDA_OR_THROW(cudaMemset(t.d_stats, 0, 2 * sizeof(sbs_gen_stats)));
    }
    upload_gen_jobs(s, 0);
    init_points(s, points, n_points, trace_of_point, n_traces);
    generate_slot(s, nullptr, 0, 0, 0);
    CUDA_OR_THROW(cudaDeviceSynchronize());
    return SBS_OK;
  });
  if (rc != SBS_OK) {
    sbs_sim_destroy(s);
    return rc;
  }
  *out = s;
  return SBS_OK;
}

int sbs_sim_generate_slot(sbs_sim* s, const uint64_t* seeds, int32_t slot, int32_t want_digest,
                          void* stream) {
  return guarded([&] {
    if (!s->generated) throw Error{SBS_ERR_CONFIG, "simulator traces are host-uploaded"};
    if (slot < 0 || slot >= s->n_slots) throw Error{SBS_ERR_CONFIG, "trace slot out of range"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    if (seeds)
      for (size_t i = 0; i < s->traces.size(); ++i) s->traces[i].seed = seeds[i];
    generate_slot(s, seeds, slot, want_digest, (cudaStream_t)stream);
    return SBS_OK;
  });
}

int sbs_sim_trace_stats(sbs_sim* s, int32_t trace, int32_t slot, sbs_gen_stats* out) {
  return guarded([&] {
    if (trace < 0 || trace >= (int)s->traces.size()) throw Error{SBS_ERR_CONFIG, "trace out of range"};
    if (slot < 0 || slot >= s->n_slots) throw Error{SBS_ERR_CONFIG, "trace slot out of range"};
    TraceDev& t = s->traces[trace];
    if (!t.gen) throw Error{SBS_ERR_CONFIG, "trace was uploaded from the host"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    CUDA_OR_THROW(cudaDeviceSynchronize());
    CUDA_OR_THROW(cudaMemcpy(out, &t.d_stats[slot], sizeof(sbs_gen_stats), cudaMemcpyDeviceToHost));
    return SBS_OK;
  });
}

int sbs_sim_trace_arrays(sbs_sim* s, int32_t trace, int32_t slot, int64_t* arrival_ns,
                         int32_t* prompt_len, int32_t* output_len, int32_t* prefix_pool_id,
                         int32_t* prefix_size, int64_t cap, int64_t* n_out) {
  return guarded([&] {
    if (trace < 0 || trace >= (int)s->traces.size()) throw Error{SBS_ERR_CONFIG, "trace out of range"};
    if (slot < 0 || slot >= s->n_slots) throw Error{SBS_ERR_CONFIG, "trace slot out of range"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    CUDA_OR_THROW(cudaDeviceSynchronize());
    TraceDev& t = s->traces[trace];
    int64_t n = t.n;
    if (t.gen) {
      sbs_gen_stats st{};
      CUDA_OR_THROW(cudaMemcpy(&st, &t.d_stats[slot], sizeof(st), cudaMemcpyDeviceToHost));
      n = st.n;
    }
    if (n_out) *n_out = n;
    if (arrival_ns == nullptr || n == 0) return SBS_OK;
    if (n > cap) return fail(SBS_ERR_OVERFLOW, "trace buffer too small");
    CUDA_OR_THROW(cudaMemcpy(arrival_ns, slot ? t.arr1 : t.arr, 8 * n, cudaMemcpyDeviceToHost));
    CUDA_OR_THROW(cudaMemcpy(prompt_len, slot ? t.prompt1 : t.prompt, 4 * n, cudaMemcpyDeviceToHost));
    CUDA_OR_THROW(cudaMemcpy(output_len, slot ? t.output1 : t.output, 4 * n, cudaMemcpyDeviceToHost));
    if (prefix_pool_id && t.pool)
      CUDA_OR_THROW(cudaMemcpy(prefix_pool_id, slot ? t.pool1 : t.pool, 4 * n, cudaMemcpyDeviceToHost));
    if (prefix_size && t.psize)
      CUDA_OR_THROW(cudaMemcpy(prefix_size, slot ? t.psize1 : t.psize, 4 * n, cudaMemcpyDeviceToHost));
    return SBS_OK;
  });
}

int sbs_sim_upload_traces(sbs_sim* s, const sbs_trace* traces, void* stream) {
  return guarded([&] {
    CUDA_OR_THROW(cudaSetDevice(s->device));
    do_upload_traces(*s, traces, (cudaStream_t)stream);
    return SBS_OK;
  });
}

int sbs_sim_launch_slot(sbs_sim* s, int32_t slot, void* stream) {
  return guarded([&] {
    if (slot < 0 || slot >= s->n_slots) throw Error{SBS_ERR_CONFIG, "trace slot out of range"};
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_OR_THROW(cudaSetDevice(s->device));
    s->cur_slot = slot;
    for (auto& p : s->pts) reset_point(p, st);
    launch_all(*s, st);
    return SBS_OK;
  });
}

int sbs_sim_launch(sbs_sim* s, void* stream) { return sbs_sim_launch_slot(s, 0, stream); }

int sbs_sim_upload_traces_slot(sbs_sim* s, const sbs_trace* traces, int32_t slot, void* stream) {
  return guarded([&] {
    CUDA_OR_THROW(cudaSetDevice(s->device));
    do_upload_traces(*s, traces, (cudaStream_t)stream, slot);
    return SBS_OK;
  });
}

int sbs_sim_enable_trace_slots(sbs_sim* s, int32_t n) {
  return guarded([&] {
    if (n != 1 && n != 2) throw Error{SBS_ERR_CONFIG, "trace slots must be 1 or 2"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    if (n == 2 && s->n_slots == 1) {
      for (auto& t : s->traces) {
        const size_t m = (size_t)std::max<int64_t>(t.n, 1);
        CUDA_OR_THROW(cudaMalloc(&t.arr1, 8 * m));
        CUDA_OR_THROW(cudaMalloc(&t.prompt1, 4 * m));
        CUDA_OR_THROW(cudaMalloc(&t.output1, 4 * m));
        s->device_bytes += (int64_t)(16 * m);
        if (t.pool) {
          CUDA_OR_THROW(cudaMalloc(&t.pool1, 4 * m));
          CUDA_OR_THROW(cudaMalloc(&t.psize1, 4 * m));
          s->device_bytes += (int64_t)(8 * m);
        }
      }
      CUDA_OR_THROW(cudaMalloc(&s->d_pts1, sizeof(sbs::DevPoint) * s->pts.size()));
      s->n_slots = 2;
      upload_points(*s);
      if (s->generated) upload_gen_jobs(s, 1);
    }
    return SBS_OK;
  });
}

int32_t sbs_sim_launches_per_run(const sbs_sim* s) {
  // the kernels of the last launch: reset_kernel, the DES kernel(s) of each
  // variant group (two for a two-kernel pair group), finalize_kernel
  if (s->n_launches > 0) return s->n_launches;
  int n = 2;
  for (int v = 0; v < sbs_sim::kVariants; ++v) n += s->group_begin[v + 1] > s->group_begin[v] ? 1 : 0;
  return n;
}

int64_t sbs_sim_device_bytes(const sbs_sim* s) { return s->device_bytes; }

int sbs_sim_des_ms(sbs_sim* s, double* ms) {
  return guarded([&] {
    if (s->ev_des[0] == nullptr) throw Error{SBS_ERR_INVARIANT, "no launch recorded"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    CUDA_OR_THROW(cudaEventSynchronize(s->ev_des[1]));
    float f = 0.f;
    CUDA_OR_THROW(cudaEventElapsedTime(&f, s->ev_des[0], s->ev_des[1]));
    *ms = (double)f;
    return SBS_OK;
  });
}

int sbs_sim_results(sbs_sim* s, sbs_aggregates* out, sbs_histograms* hist, void* stream) {
  return guarded([&] {
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_OR_THROW(cudaSetDevice(s->device));
    const int n = (int)s->order.size();
    for (int attempt = 0;; ++attempt) {
      CUDA_OR_THROW(cudaMemcpyAsync(s->h_res.data(), s->d_res, sizeof(sbs::DevResult) * n,
                                    cudaMemcpyDeviceToHost, st));
      CUDA_OR_THROW(cudaStreamSynchronize(st));
      if (s->generated && !s->gen_slot_valid[s->cur_slot]) {
        for (auto& t : s->traces)
          CUDA_OR_THROW(cudaMemcpy(&t.h_stats[s->cur_slot], &t.d_stats[s->cur_slot],
                                   sizeof(sbs_gen_stats), cudaMemcpyDeviceToHost));
        s->gen_slot_valid[s->cur_slot] = 1;
      }
      if (s->pair3_used) {  // the two kernels were not co-resident: rerun the launch as clusters
        int sync[2] = {0, 0};
        CUDA_OR_THROW(cudaMemcpy(sync, s->d_sync, sizeof(sync), cudaMemcpyDeviceToHost));
        if (sync[1] != 0) {
          if (std::getenv("SBS_DEBUG")) std::fprintf(stderr, "sbs: pair mode 3 not co-resident, clusters\n");
          s->pair_mode = 2;
          for (auto& p : s->pts) reset_point(p, st);
          launch_all(*s, st);
          continue;
        }
      }
      bool overflow = false;
      for (int i = 0; i < n; ++i) {
        const int err = s->h_res[i].error;
        if (err != SBS_ERR_OVERFLOW && err != sbs::kErrSplitTie) continue;
        overflow = true;
        PointHost& p = s->pts[s->order[i]];
        if (err == SBS_ERR_OVERFLOW) grow_caps(p);
        else p.split = 0;  // exact one-warp rerun of this replica
        s->device_bytes -= (int64_t)p.arena_bytes;
        build_point(*s, p);
        s->device_bytes += (int64_t)p.arena_bytes;
      }
      if (!overflow) break;
      if (std::getenv("SBS_DEBUG")) {
        int nt = 0, no = 0;
        for (int i = 0; i < n; ++i) {
          nt += s->h_res[i].error == sbs::kErrSplitTie;
          no += s->h_res[i].error == SBS_ERR_OVERFLOW;
        }
        std::fprintf(stderr, "sbs: rerun attempt %d: %d split ties, %d overflows of %d\n", attempt, nt,
                     no, n);
      }
      if (attempt >= 12) throw Error{SBS_ERR_OVERFLOW, "device arena overflow persists"};
      order_points(*s);
      upload_points(*s);
      for (auto& p : s->pts) reset_point(p, st);
      launch_all(*s, st);
    }
    int rc = SBS_OK;
    if (hist) std::memset(hist, 0, sizeof(*hist));
    std::vector<int64_t> th(sbs::kHistBins);
    for (int i = 0; i < n; ++i) {
      const PointHost& p = s->pts[s->order[i]];
      const TraceDev& t = s->traces[p.trace];
      if (t.gen && t.h_stats[s->cur_slot].error != 0) {
        rc = t.h_stats[s->cur_slot].error;
        g_err = "device trace generation failed for trace " + std::to_string(p.trace) + " (code " +
                std::to_string(rc) + ")";
      }
      finish_aggregates(p, s->h_res[i], out[s->order[i]], live_n(*s, p));
      if (s->h_res[i].error != 0) {
        rc = s->h_res[i].error;
        g_err = "replica " + std::to_string(s->order[i]) + " failed with code " + std::to_string(rc) +
                (rc == SBS_ERR_ENVELOPE
                     ? " (integer envelope: decode unit B >= 2^15 or K >= 2^32, or 2^32 scheduled events)"
                     : "");
      }
      if (hist) {
        CUDA_OR_THROW(cudaMemcpy(th.data(), p.dp.tpot_hist, 8 * sbs::kHistBins, cudaMemcpyDeviceToHost));
        for (int b = 0; b < sbs::kHistBins; ++b) {
          hist->ttft[b] += s->h_res[i].ttft_hist[b];
          hist->tpot[b] += th[b];
        }
      }
    }
    return rc;
  });
}

int sbs_sim_requests(sbs_sim* s, int32_t point, int64_t* dispatch_ns, int64_t* prefill_start_ns,
                     int64_t* first_token_ns, int64_t* completion_ns, int8_t* status) {
  return guarded([&] {
    if (!(s->flags & SBS_FLAG_PER_REQUEST))
      throw Error{SBS_ERR_CONFIG, "simulator was created without SBS_FLAG_PER_REQUEST"};
    if (point < 0 || point >= (int)s->pts.size()) throw Error{SBS_ERR_CONFIG, "point out of range"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    const sbs::DevPoint& d = s->pts[point].dp;
    size_t n = (size_t)live_n(*s, s->pts[point]);
    if (n == 0) return SBS_OK;
    if (dispatch_ns) CUDA_OR_THROW(cudaMemcpy(dispatch_ns, d.o_dispatch, 8 * n, cudaMemcpyDeviceToHost));
    if (prefill_start_ns) CUDA_OR_THROW(cudaMemcpy(prefill_start_ns, d.o_pstart, 8 * n, cudaMemcpyDeviceToHost));
    if (first_token_ns) CUDA_OR_THROW(cudaMemcpy(first_token_ns, d.o_ftok, 8 * n, cudaMemcpyDeviceToHost));
    if (completion_ns) CUDA_OR_THROW(cudaMemcpy(completion_ns, d.o_comp, 8 * n, cudaMemcpyDeviceToHost));
    if (status) CUDA_OR_THROW(cudaMemcpy(status, d.o_status, n, cudaMemcpyDeviceToHost));
    return SBS_OK;
  });
}

int sbs_sim_log(sbs_sim* s, int32_t point, int64_t* words, int64_t cap, int64_t* n_out) {
  return guarded([&] {
    if (!(s->flags & SBS_FLAG_LOGS))
      throw Error{SBS_ERR_CONFIG, "simulator was created without SBS_FLAG_LOGS"};
    if (point < 0 || point >= (int)s->pts.size()) throw Error{SBS_ERR_CONFIG, "point out of range"};
    CUDA_OR_THROW(cudaSetDevice(s->device));
    int slot = -1;
    for (size_t i = 0; i < s->order.size(); ++i)
      if (s->order[i] == point) slot = (int)i;
    const int64_t n = s->h_res[slot].log_n;
    if (n_out) *n_out = n;
    if (words == nullptr) return SBS_OK;
    if (n > cap) return fail(SBS_ERR_OVERFLOW, "log buffer too small");
    CUDA_OR_THROW(cudaMemcpy(words, s->pts[point].dp.log, 8 * (size_t)n, cudaMemcpyDeviceToHost));
    return SBS_OK;
  });
}

int sbs_sim_profile_counters(const sbs_sim* s, int64_t* out) {
  for (int i = 0; i < SBS_PROF_COUNTERS; ++i) out[i] = 0;
  for (const auto& r : s->h_res)
    for (int i = 0; i < SBS_PROF_COUNTERS; ++i) out[i] += r.prof[i];
  return SBS_OK;
}

void sbs_sim_destroy(sbs_sim* s) {
  if (s == nullptr) return;
  cudaSetDevice(s->device);
  for (auto& p : s->pts) free_point(p);
  for (auto& t : s->traces) {
    if (t.arr) cudaFree(t.arr);
    if (t.prompt) cudaFree(t.prompt);
    if (t.output) cudaFree(t.output);
    if (t.pool) cudaFree(t.pool);
    if (t.psize) cudaFree(t.psize);
    for (void* q : {(void*)t.arr1, (void*)t.prompt1, (void*)t.output1, (void*)t.pool1, (void*)t.psize1})
      if (q) cudaFree(q);
    if (t.d_stats) cudaFree(t.d_stats);
  }
  for (int k = 0; k < 2; ++k) {
    if (s->d_jobs[k]) cudaFree(s->d_jobs[k]);
    if (s->d_seeds[k]) cudaFree(s->d_seeds[k]);
    if (s->h_seeds[k]) cudaFreeHost(s->h_seeds[k]);
    if (s->ev_seeds[k]) cudaEventDestroy(s->ev_seeds[k]);
  }
  if (s->d_pts) cudaFree(s->d_pts);
  if (s->d_pts1) cudaFree(s->d_pts1);
  if (s->d_res) cudaFree(s->d_res);
  if (s->d_counter) cudaFree(s->d_counter);
  if (s->d_sync) cudaFree(s->d_sync);
  for (auto& e : s->ev_des)
    if (e) cudaEventDestroy(e);
  for (int v = 0; v < sbs_sim::kVariants; ++v) {
    if (s->vstream[v]) cudaStreamDestroy(s->vstream[v]);
    if (s->vstream2[v]) cudaStreamDestroy(s->vstream2[v]);
    if (s->ev_join[v]) cudaEventDestroy(s->ev_join[v]);
  }
  if (s->h_segs) cudaFreeHost(s->h_segs);
  if (s->d_segs) cudaFree(s->d_segs);
  if (s->ev_segs) cudaEventDestroy(s->ev_segs);
  delete s;
}

int sbs_run_experiments(const sbs_experiment* points, int32_t n_points, sbs_aggregates* out,
                        int32_t device) {
  return guarded([&] {
    // unique (workload, seed) traces, generated on host threads
    std::vector<HostTrace> tr;
    std::vector<int32_t> map(n_points);
    std::map<std::string, int> seen;
    for (int i = 0; i < n_points; ++i) {
      std::string key(reinterpret_cast<const char*>(&points[i].workload), sizeof(sbs_workload));
      key.append(reinterpret_cast<const char*>(&points[i].seed), sizeof(uint64_t));
      auto it = seen.find(key);
      if (it == seen.end()) {
        map[i] = (int)tr.size();
        seen.emplace(key, (int)tr.size());
        tr.emplace_back();
      } else {
        map[i] = it->second;
      }
    }
    std::vector<int> first(tr.size(), -1);
    for (int i = 0; i < n_points; ++i)
      if (first[map[i]] < 0) first[map[i]] = i;
    std::atomic<size_t> next{0};
    std::atomic<bool> bad{false};
    Error firsterr{0, ""};
    auto work = [&]() {
      for (;;) {
        size_t k = next.fetch_add(1);
        if (k >= tr.size()) return;
        try {
          generate(points[first[k]].workload, points[first[k]].seed, tr[k]);
        } catch (const Error& e) {
          if (!bad.exchange(true)) firsterr = e;
        }
      }
    };
    std::vector<std::thread> pool;
    int nt = std::min<int>(parallel_threads(), (int)tr.size());
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    if (bad) throw firsterr;
    std::vector<sbs_trace> st(tr.size());
    for (size_t k = 0; k < tr.size(); ++k)
      st[k] = sbs_trace{tr[k].arr.data(), tr[k].prompt.data(), tr[k].output.data(),
                        (int64_t)tr[k].arr.size(), tr[k].digest,
                        tr[k].pool.empty() ? nullptr : tr[k].pool.data(),
                        tr[k].psize.empty() ? nullptr : tr[k].psize.data()};
    sbs_sim* s = nullptr;
    int rc = sbs_sim_create(points, n_points, st.data(), (int32_t)st.size(), map.data(), 0, device, &s);
    if (rc != SBS_OK) return rc;
    rc = sbs_sim_launch(s, nullptr);
    if (rc == SBS_OK) rc = sbs_sim_results(s, out, nullptr, nullptr);
    std::string msg = g_err;
    sbs_sim_destroy(s);
    g_err = msg;
    return rc;
  });
}

int sbs_prefill_allocate(const sbs_window_batch* b, void* stream) {
  return guarded([&] {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch& sc = scratch();
    CUDA_OR_THROW(cudaMemsetAsync(sc.d_err, 0, sizeof(int32_t), st));
    sbs::PbaaArgs a{b->n_windows, b->max_requests, b->max_dp, b->req_off, b->n_pending, b->dp_off,
                    b->n_limit, b->req_id, b->prompt_len, b->wait_in, b->caps, b->out_dp,
                    b->out_rank, b->wait_out, b->flow, sc.d_err, b->hit_off, b->hit};
    CUDA_OR_THROW(sbs::launch_pbaa(a, st));
    CUDA_OR_THROW(cudaMemcpyAsync(sc.h_err, sc.d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_OR_THROW(cudaStreamSynchronize(st));
    if (*sc.h_err) throw Error{*sc.h_err, "window exceeds the kernel's shared-memory envelope"};
    return SBS_OK;
  });
}

// One window from host arrays (the reference's allocate_batch call shape).
// Small Basic-mode windows travel in the kernel parameters and come back
// through mapped pinned memory: one launch and one synchronisation per call.
// Larger or cache-aware windows use a per-thread device staging block.
struct OneWindow {
  int device = -1;
  cudaStream_t stream = nullptr;
  int32_t* mapped = nullptr;             // pinned, device-visible outputs
  unsigned char* host = nullptr;         // staged path
  unsigned char* dev = nullptr;
  size_t cap = 0;
};
// One staging block per (thread, device), like scratch(): a device switch
// never reuses another device's stream or staging memory.
OneWindow& one_window() {
  thread_local OneWindow ws[16];
  int dev = 0;
  CUDA_OR_THROW(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 16) throw Error{SBS_ERR_CUDA, "device ordinal above 15"};
  OneWindow& w = ws[dev];
  if (w.device != dev) {
    CUDA_OR_THROW(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
    CUDA_OR_THROW(cudaHostAlloc(&w.mapped, 4096, cudaHostAllocMapped));
    w.device = dev;
  }
  return w;
}

int sbs_prefill_allocate_one(const int64_t* rows, int32_t n_pending, int32_t n_new, int64_t* caps,
                             int32_t n_dp, int32_t n_limit, const int64_t* hits, int32_t* out_dp,
                             int32_t* out_rank, int32_t* wait_out, uint8_t* flow) {
  return guarded([&] {
    const int n = n_pending + n_new;
    if (n_dp < 1 || n_pending < 0 || n_new < 0) throw Error{SBS_ERR_CONFIG, "bad window shape"};
    OneWindow& w = one_window();
    if (hits == nullptr && n <= 32 && n_dp <= 32) {
      int32_t* o = nullptr;
      CUDA_OR_THROW(cudaHostGetDevicePointer((void**)&o, w.mapped, 0));
      CUDA_OR_THROW(sbs::launch_pbaa_one(rows, n_pending, n_new, caps, n_dp, n_limit, o, w.stream));
      CUDA_OR_THROW(cudaStreamSynchronize(w.stream));
      const int32_t* m = w.mapped;
      if (m[3 * n + 1]) throw Error{SBS_ERR_OVERFLOW, "window exceeds the kernel envelope"};
      std::memcpy(out_dp, m, 4 * (size_t)n);
      std::memcpy(out_rank, m + n, 4 * (size_t)n);
      std::memcpy(wait_out, m + 2 * n, 4 * (size_t)n);
      *flow = (uint8_t)m[3 * n];
      std::memcpy(caps, (const int64_t*)(m + ((3 * n + 3) & ~1)), 8 * (size_t)n_dp);
      return SBS_OK;
    }
    // staged: [req_off 2][n_pending][dp_off 2][n_limit][ids][lens][waits][caps][hit_off 2][hits]
    //         [dp][rank][wait_out][flow][err]
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 7) & ~size_t(7); return o; };
    const size_t o_roff = take(16), o_np = take(4), o_doff = take(16), o_nl = take(4),
                 o_id = take(8 * (size_t)n), o_len = take(8 * (size_t)n), o_win = take(4 * (size_t)n),
                 o_caps = take(8 * (size_t)n_dp), o_hoff = take(16),
                 o_hit = take(hits ? 8 * (size_t)n * n_dp : 0), o_dp = take(4 * (size_t)n),
                 o_rank = take(4 * (size_t)n), o_wout = take(4 * (size_t)n), o_flow = take(8),
                 o_err = take(8);
    if (off > w.cap) {
      if (w.host) cudaFreeHost(w.host);
      if (w.dev) cudaFree(w.dev);
      w.cap = std::max(off, 2 * w.cap);
      CUDA_OR_THROW(cudaMallocHost(&w.host, w.cap));
      CUDA_OR_THROW(cudaMalloc(&w.dev, w.cap));
    }
    unsigned char* h = w.host;
    const int64_t roff[2] = {0, n}, doff[2] = {0, n_dp}, hoff[2] = {0, (int64_t)n * n_dp};
    std::memcpy(h + o_roff, roff, 16);
    std::memcpy(h + o_np, &n_pending, 4);
    std::memcpy(h + o_doff, doff, 16);
    std::memcpy(h + o_nl, &n_limit, 4);
    for (int i = 0; i < n; ++i) {
      ((int64_t*)(h + o_id))[i] = rows[3 * i];
      ((int64_t*)(h + o_len))[i] = rows[3 * i + 1];
      ((int32_t*)(h + o_win))[i] = (int32_t)rows[3 * i + 2];
    }
    std::memcpy(h + o_caps, caps, 8 * (size_t)n_dp);
    std::memcpy(h + o_hoff, hoff, 16);
    if (hits) std::memcpy(h + o_hit, hits, 8 * (size_t)n * n_dp);
    *(int32_t*)(h + o_err) = 0;
    unsigned char* g = w.dev;
    CUDA_OR_THROW(cudaMemcpyAsync(g, h, off, cudaMemcpyHostToDevice, w.stream));
    sbs::PbaaArgs a{1, n, n_dp, (const int64_t*)(g + o_roff), (const int32_t*)(g + o_np),
                    (const int64_t*)(g + o_doff), (const int32_t*)(g + o_nl),
                    (const int64_t*)(g + o_id), (const int64_t*)(g + o_len),
                    (const int32_t*)(g + o_win), (int64_t*)(g + o_caps), (int32_t*)(g + o_dp),
                    (int32_t*)(g + o_rank), (int32_t*)(g + o_wout), (uint8_t*)(g + o_flow),
                    (int32_t*)(g + o_err), hits ? (const int64_t*)(g + o_hoff) : nullptr,
                    hits ? (const int64_t*)(g + o_hit) : nullptr};
    CUDA_OR_THROW(sbs::launch_pbaa(a, w.stream));
    CUDA_OR_THROW(cudaMemcpyAsync(h + o_dp, g + o_dp, off - o_dp, cudaMemcpyDeviceToHost, w.stream));
    CUDA_OR_THROW(cudaMemcpyAsync(h + o_caps, g + o_caps, 8 * (size_t)n_dp, cudaMemcpyDeviceToHost,
                                  w.stream));
    CUDA_OR_THROW(cudaStreamSynchronize(w.stream));
    if (*(int32_t*)(h + o_err)) throw Error{SBS_ERR_OVERFLOW, "window exceeds the kernel envelope"};
    std::memcpy(out_dp, h + o_dp, 4 * (size_t)n);
    std::memcpy(out_rank, h + o_rank, 4 * (size_t)n);
    std::memcpy(wait_out, h + o_wout, 4 * (size_t)n);
    *flow = h[o_flow];
    std::memcpy(caps, h + o_caps, 8 * (size_t)n_dp);
    return SBS_OK;
  });
}

int sbs_decode_select(const sbs_decode_batch* b, void* stream) {
  return guarded([&] {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch& sc = scratch();
    CUDA_OR_THROW(cudaMemsetAsync(sc.d_err, 0, sizeof(int32_t), st));
    sbs::IqrArgs a{b->n_calls, b->max_units, b->unit_off, b->batch, b->kv, b->k, b->pos_out,
                   b->fallback_out, b->threshold_out, sc.d_err};
    CUDA_OR_THROW(sbs::launch_iqr(a, st));
    CUDA_OR_THROW(cudaMemcpyAsync(sc.h_err, sc.d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_OR_THROW(cudaStreamSynchronize(st));
    if (*sc.h_err == 3) throw Error{SBS_ERR_INVARIANT, "select_decode_unit: no units"};
    if (*sc.h_err) throw Error{*sc.h_err, "decode call exceeds the kernel's shared-memory envelope"};
    return SBS_OK;
  });
}

int sbs_prefill_allocate_async(const sbs_window_batch* b, int32_t* error_out, void* stream) {
  return guarded([&] {
    sbs::PbaaArgs a{b->n_windows, b->max_requests, b->max_dp, b->req_off, b->n_pending, b->dp_off,
                    b->n_limit, b->req_id, b->prompt_len, b->wait_in, b->caps, b->out_dp,
                    b->out_rank, b->wait_out, b->flow, error_out, b->hit_off, b->hit};
    CUDA_OR_THROW(sbs::launch_pbaa(a, (cudaStream_t)stream));
    return SBS_OK;
  });
}

int sbs_decode_select_async(const sbs_decode_batch* b, int32_t* error_out, void* stream) {
  return guarded([&] {
    sbs::IqrArgs a{b->n_calls, b->max_units, b->unit_off, b->batch, b->kv, b->k, b->pos_out,
                   b->fallback_out, b->threshold_out, error_out};
    CUDA_OR_THROW(sbs::launch_iqr(a, (cudaStream_t)stream));
    return SBS_OK;
  });
}

namespace {
sbs::SchedArgs sched_args(const sbs_decode_schedule* b, int32_t* err) {
  if (b->max_candidates < 0 || b->max_candidates > 4096 || b->max_units < 1 || b->max_units > 4096)
    throw Error{SBS_ERR_CONFIG, "sbs_decode_schedule: max_candidates / max_units must be <= 4096"};
  sbs::SchedArgs a{};
  a.n_batches = b->n_batches;
  a.max_cands = std::max(1, b->max_candidates);
  a.max_units = b->max_units;
  a.cand_off = b->cand_off;
  a.request_id = b->request_id;
  a.sort_len = b->sort_len;
  a.kv_len = b->kv_len;
  a.unit_off = b->unit_off;
  a.batch = b->batch;
  a.kv = b->kv;
  a.k = b->k;
  a.order_out = b->order_out;
  a.pos_out = b->pos_out;
  a.fallback_out = b->fallback_out;
  a.threshold_out = b->threshold_out;
  a.error = err;
  return a;
}
}  // namespace

int sbs_decode_schedule_batch_async(const sbs_decode_schedule* b, int32_t* error_out, void* stream) {
  return guarded([&] {
    CUDA_OR_THROW(sbs::launch_sched(sched_args(b, error_out), (cudaStream_t)stream));
    return SBS_OK;
  });
}

int sbs_decode_schedule_batch(const sbs_decode_schedule* b, void* stream) {
  return guarded([&] {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch& sc = scratch();
    CUDA_OR_THROW(cudaMemsetAsync(sc.d_err, 0, sizeof(int32_t), st));
    CUDA_OR_THROW(sbs::launch_sched(sched_args(b, sc.d_err), st));
    CUDA_OR_THROW(cudaMemcpyAsync(sc.h_err, sc.d_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_OR_THROW(cudaStreamSynchronize(st));
    if (*sc.h_err == 3) return fail(SBS_ERR_INVARIANT, "select_decode_unit: no units");
    if (*sc.h_err) return fail(SBS_ERR_OVERFLOW, "decode batch beyond max_candidates / max_units");
    return SBS_OK;
  });
}

}  // extern "C"
