// Device-side replica descriptors shared by sbs_host.cpp and des.cu.
//
// One DevPoint describes one independent replica (= one run_experiment call of
// the reference, simulation.cpp:537): its cluster and engine constants, its
// trace (SoA, shared between replicas with the same (seed, workload)), its
// fault plan, and its private HBM arena.  Layout in HBM per replica:
//   per-request timestamps   3 x int64 x N  (dispatch, prefill_start, first_token)
//   [parity] completion int64 x N, status int8 x N
//   TTFT window buffer       int64 x N      (exact p50/p95 order statistics)
//   q_pending double buffer  2 x (u64 key + i32 wait) x QP
//   window scratch           u64 x QW       (only when a window exceeds smem)
//   prefill DP FIFOs         (P*D) x F x int2 {request id, tokens left}
//   decode completion ring   Dn x R x BC x int4 {id, unit, kv release, excess}
//   decode waiters           u64 x QD
//   mt19937_64 state         312 x u64      (decode policy "random" only)
#pragma once
#include <stdint.h>

namespace sbs {

constexpr int kMaxInstances = 32;   // per pool (one lane per instance)
constexpr int kMaxPrefillDp = 128;  // 4 DP units per lane
constexpr int kMaxWSize = 1024;     // exec-window ring in shared memory
constexpr int kSmemWinKeys = 256;   // window keys kept in shared memory
constexpr int kHistBins = 64;
constexpr int kChanRecs = 32;       // prefill->decode hand-off records in flight
constexpr int kChanKeys = 1024;     // hand-off waiter keys in flight
constexpr int kMaxProbes = 32;      // distinct prefix-cache probe lengths
constexpr int kStageEntries = 32;   // completion-bucket entries staged in smem per decode step
constexpr int kErrSplitTie = 7;     // two-warp replica met an unresolvable tie: rerun serially

// Prefill-warp -> decode-warp hand-off channel of a two-warp replica (shared
// memory).  One record per EndForward event: its time, the time its pass was
// scheduled (= pass start), the prefill-warp index of the handler event that
// scheduled it and of the EndForward event itself, and the decode-bound
// requests it finished (waiter keys in a ring).
struct ChanRec {
  long long t, ts;
  int ef_idx;    // prefill-warp event index of this EndForward
  int h_idx;     // prefill-warp event index of the handler that scheduled it
  int h_ext;     // that handler was an arrival/topology event (seq below internals)
  int nk, k0, pad;
};
struct Chan {
  volatile long long p_done;  // every prefill-warp event with time < p_done is processed
  volatile int tail, head;    // records written / consumed
  volatile int ktail, khead;  // keys written / consumed
  volatile int abort;         // decode warp met an unresolvable tie
  int pad_;
  ChanRec rec[kChanRecs];
  unsigned long long keys[kChanKeys];
};

enum Policy : int32_t { kSbs = 0, kImmediate = 1, kRoundRobin = 2, kLeastOutstanding = 3 };
enum DecodePolicy : int32_t { kIqr = 0, kRandom = 1, kDecRoundRobin = 2 };
enum Status : int8_t {
  kStPending = 0, kStDispatched = 1, kStPrefilling = 2, kStDecoding = 3,
  kStCompleted = 4, kStThrottled = 5
};

struct DevPoint {
  // ---- dimensions
  int32_t P, Dn, D, Dd, U;  // prefill inst, decode inst, prefill DP, decode DP, Dn*Dd
  int32_t policy, decode_policy, n_limit, cap_batch;
  int32_t n_topo, n_drops, w_size;
  int32_t per_request;      // parity mode: also write completion + status
  int32_t split;            // run as a prefill warp + decode warp pair
  int32_t log_kv_loads;     // run records also keep the per-unit KV loads per step
  // decode waiter key (simulation.cpp:446-453 order): (kq_lmax - len) << (kq_ib + kq_ob)
  // | id << kq_ob | output_len, ascending == (prompt+output desc, id asc); the
  // low field carries output_len (prompt = len - output) so the decode side
  // never reads the trace.  kq_ob = 0 (no room): 32-bit fields, lengths loaded.
  int32_t kq_ob, kq_ib;
  uint32_t kq_lmax;
  int32_t _pad0;
  // ---- constants (integer ns, FP64 engine coefficients)
  int64_t c_chunk, t_default, l_net, tps, horizon, warmup;
  double iqr_k, wd_mult, pf_base, pf_tok, dc_base, dc_req, dc_kv;
  uint64_t rng_seed;
  int64_t N;             // trace length, or its capacity when n_dev is set
  const int64_t* n_dev;  // device-generated trace: its length (sbs_gen_stats::n), else NULL
  // ---- trace (SoA)
  const int64_t* arr;
  const int32_t* prompt;
  const int32_t* output;
  // ---- prefix caches (cache-aware PBAA, core.cpp:13-75): per prefill DP unit
  // an LRU over keys (pool, probe) kept as last-use stamps (0 = absent)
  int32_t cache_on, n_probes, n_pools, _pc;
  int64_t cache_budget;
  int32_t probe_k[kMaxProbes];  // ascending, distinct
  const int32_t* pfx_pool;      // per request, -1 = no prefix
  const int32_t* pfx_size;      // per request prefix tokens
  int32_t* c_stamp;             // [P*D][n_pools*n_probes]
  int64_t* c_used;              // [P*D] cached tokens
  int32_t* c_clock;             // [P*D] stamps issued
  // ---- faults
  const int64_t* topo_time;  // sorted by (time, config order)
  const int32_t* topo_inst;
  const int32_t* topo_healthy;
  const int64_t* drop_from;
  const int64_t* drop_until;
  const int32_t* drop_inst;
  int64_t death[2 * kMaxInstances];  // by instance id, INT64_MAX = never
  // ---- arena
  int64_t* o_dispatch;
  int64_t* o_pstart;
  int64_t* o_ftok;
  int64_t* o_comp;     // parity only
  int8_t* o_status;    // parity only
  int64_t* ttft;
  uint64_t* pend_key[2];
  int32_t* pend_wait[2];
  uint64_t* wscr;
  int2* fifo;
  int4* buckets;
  uint64_t* dwait;
  uint64_t* mt;
  int64_t* tpot_hist;  // kHistBins
  // two-kernel pairs (pair mode 3): the hand-off channel in HBM and each
  // warp's counters (2 x 256 B) for finalize_kernel to combine
  struct Chan* gchan;
  int64_t* gcnt;
  int64_t* log;        // optional run records (parity / report files), LOG_* below
  int64_t log_cap;     // words
  int32_t QP, QW, F, R, BC, QD;
  // ---- shared-memory carve (bytes, relative to the warp's slice)
  int32_t sm_pf_out, sm_pf_head, sm_pf_tail, sm_pf_rel, sm_pf_part;
  int32_t sm_dPK, sm_dR, sm_dS, sm_dT, sm_dnst, sm_ulist, sm_bcnt, sm_hist, sm_wring, sm_wkeys, sm_cnt, sm_cnt2, sm_chan;
  int32_t sm_stage;  // per decode instance: the completion bucket of its step in progress
  int32_t sm_bytes;
  // the prefill warp's fields come first, [0, sm_dec_begin); the decode
  // warp's are [sm_dec_begin, sm_dec_end); the channel follows
  int32_t sm_dec_begin, sm_dec_end;
  int32_t _pad1;
};

// Run-record log (MetricsCollector records, metrics.h:107-152), one stream of
// int64 words per replica: header = kind | (payload words << 8), then payload.
enum LogKind : int32_t {
  LOG_DISPATCH = 1,  // time, instance                      (record_dispatch)
  LOG_CONTROL = 2,   // time, i_opt, t_fwd_bar, n_active      (record_control)
  LOG_PASS = 3,      // time, instance, assigned[D]           (record_pass)
  LOG_STEP = 4,      // time, generated                       (record_step)
  LOG_KV = 5,        // time, mean bits, sigma bits, min, max (record_kv / kv_band)
  LOG_KVLOADS = 6,   // time, K of every healthy live decode unit (record_kv's span)
};

struct DevResult {
  int64_t completed, throttled, cw, wr, passes, steps, out_tokens;
  int64_t wd_fires, dropped, rejected, deferrals, flow, mask, fallback;
  int64_t alloc_calls, dec_selects, events, n_ttft;
  int64_t ttft_sum, sched_sum, dev_sum;
  double util_sum, kv_mean_sum, kv_sigma_sum, tpot_sum;
  int64_t kv_n, tpot_n;
  int64_t ttft_sel[4];  // order statistics at ranks lo50, hi50, lo95, hi95
  int64_t ttft_hist[kHistBins];
  int64_t log_n;        // words written (== log_cap + 1 on overflow)
  int64_t prof[24];     // SBS_PROF builds only: clock64 cycles per region
  int32_t error;
  int32_t _pad;
};

}  // namespace sbs
