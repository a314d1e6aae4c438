// Persistent discrete-event simulator of the SBS cluster: one warp per
// replica, or a prefill warp + a decode warp per replica (two-warp replicas,
// default for points with decode work, see the channel notes at the event
// loop and DESIGN.md §3.8).
//
// Reproduces reference Runner::run (simulation.cpp:136-169) event for event:
// every event fires in the reference's (time, seq) order, every allocation
// window is decided exactly as allocate_batch (prefill_alloc.cpp:61-88), every
// decode placement as select_decode_unit (decode_alloc.cpp:38-81), with the
// same integer-ns rounding and FP64 expressions (compiled with -fmad=false and
// explicit __d*_rn so no FMA contraction changes a timestamp).
//
// Restructuring vs the reference (results identical):
//  * Event queue (simclock.cpp:24-45): arrivals are streamed from the SoA
//    trace (seq = n_topo + id, always below internal events); topology events
//    are a pre-sorted list; every internal event kind has at most one *live*
//    instance per (kind, instance) — stale ticks / watchdogs are no-ops in the
//    reference (simulation.cpp:241, interval_control.cpp:93-95) — so live
//    events live in lane registers (lane p = instance p) with an explicit
//    (time, seq) and the seq counter is advanced for every schedule() call,
//    stale or not.
//  * q_new is the contiguous id range [new_begin, next_id); q_pending is kept
//    sorted by the PBAA key (prompt desc, id asc).  Its order is otherwise
//    unobservable: greedy_dispatch re-sorts every queue by a total order.
//  * Basic-mode PBAA argmax of c_avail - prompt == argmax c_avail, and a
//    deferral only happens once max c_avail <= 0, so each phase places a
//    prefix of its sorted queue.
//  * u_flight/r_queued are only ever observed as their sum (c_avail,
//    least_outstanding), so a DP unit keeps one `outstanding` counter and a
//    FIFO of {id, tokens left}.
//  * Decode residents are not scanned per step (engine_model.cpp:181-217):
//    with every resident stamped at step begin, a request admitted while the
//    instance is at step s completes at step s + ceil(target/tps); it is
//    pushed into a completion ring bucket and K grows by tps * B_at_begin
//    minus the last-step excess of completers.
//  * A decode unit is one packed u64 (B << 48 | K) in shared memory, so the
//    lexicographic (B, K) minimum is a u64 minimum.  IQR quartiles read a
//    sorted K multiset, updated in O(U/32) per admission and re-sorted by a
//    warp LSD radix sort after a decode step.  Step begin is O(1): resident
//    count and max_u(per_req*B + per_kv*K) are maintained incrementally; the
//    KV band uses exact per-instance sums of K and K^2.  A step's completion
//    bucket is final when the step begins and is staged into shared memory
//    by cp.async while the step runs.
//  * Cache-aware PBAA (prefill_alloc.cpp:12-21): per prefill DP unit the
//    PrefixCache LRU is a table of last-use stamps (compiled in only for the
//    CA kernel variants).
//  * The hot loops are instruction-cache bound: warp loops stay rolled, cold
//    paths carry branch hints or sit out of line, and warp reductions use
//    32-bit REDUX where the operands allow.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "des_types.h"
#include "mt19937.cuh"
#include "warp.cuh"

namespace sbs {

namespace {

constexpr int kErrOverflow = 4;
constexpr int kErrInvariant = 3;

// Event kinds in the lane-resident table.
constexpr int kEvEF = 2, kEvWD = 3, kEvDS = 5;

// prefill instance flags
constexpr int F_BUSY = 1, F_DEAD = 2, F_HEALTHY = 4, F_EFSEEN = 8, F_WDFIRED = 16, F_HASDL = 32;
// decode instance flags
constexpr int G_STEP = 1, G_DEAD = 2, G_HEALTHY = 4;

__device__ __forceinline__ int64_t llround_ns(double s) {
  // seconds_to_ns (core.h:26-28): llround(s * 1e9)
  return (int64_t)llround(__dmul_rn(s, 1e9));
}

__device__ __forceinline__ uint64_t pbaa_key(int32_t prompt, int64_t id) {
  // ascending order == (prompt_len desc, id asc) (prefill_alloc.cpp:28-35)
  return ((uint64_t)(0x7fffffffu - (uint32_t)prompt) << 32) | (uint64_t)(uint32_t)id;
}
__device__ __forceinline__ int32_t key_len(uint64_t k) {
  return (int32_t)(0x7fffffffu - (uint32_t)(k >> 32));
}
__device__ __forceinline__ int64_t key_id(uint64_t k) { return (int64_t)(k & 0xffffffffu); }

__device__ __forceinline__ int hist_bin(int64_t v) {
  if (v <= 0) return 0;
  int b = 63 - __clzll(v);
  return b < kHistBins ? b : kHistBins - 1;
}

__device__ __noinline__ void mt_twist_ool(uint64_t* mt) { mt_twist(mt); }


}  // namespace

// ---------------------------------------------------------------------------
// One replica, executed by one warp.
// ---------------------------------------------------------------------------
constexpr uint64_t kBOne = 1ull << 48;       // packed decode unit: B << 48 | K
constexpr uint64_t kKMask = kBOne - 1;
constexpr int kErrEnvelope = 6;               // B >= 2^15 or K >= 2^32 on a decode unit, or seq wrap
// The event seq counter is 32-bit (the reference's is 64-bit, simclock.h:63):
// a replica stops with kErrEnvelope before it can wrap.  One handler makes far
// fewer than 2^16 schedule() calls, so checking once per event is enough.
constexpr uint32_t kSeqLimit = 0xFFFF0000u;

// Per-replica counters and FP sums (metrics.h:107-152 state), in shared memory
// and written by lane 0 only: they are rarely read, so they should not occupy
// 50 replicated registers per lane.  FP sums stay sequential in event order.
struct Counters {
  long long completed, throttled, cw, wr, passes, steps, outtok, wdf, drop, rej, def, flow,
      mask, fb, alloc, dsel, events, ttft, sched, dev, kv_n, n_ttft, tpot_n, err;
  double util, kv_mean, kv_sig, tpot;
};

// Development instrumentation: -DSBS_PROF accumulates clock64() cycles per
// region (inclusive) into DevResult::prof.  Compiled out by default.
// Branch hints: cold paths leave the hot instruction stream (block layout).
#define SBS_LIKELY(x) __builtin_expect(!!(x), 1)
#define SBS_UNLIKELY(x) __builtin_expect(!!(x), 0)

// Checked build (-DSBS_CHECK, build.py SBS_CHECK=1): every index into the
// per-replica shared-memory and HBM arrays is bounds-checked on the device;
// a violation prints the site and traps (the run fails loudly).  Compiled out
// of the product build.
#ifdef SBS_CHECK
#define SBS_ASSERT(c) \
  do { if (!(c)) { printf("SBS_CHECK %s:%d: %s\n", __FILE__, __LINE__, #c); __trap(); } } while (0)
#else
#define SBS_ASSERT(c) do { } while (0)
#endif

#ifdef SBS_PROF
#define PROF_BEGIN(r) const long long _pt##r = clock64()
#define PROF_END(r) prof_acc[r] += clock64() - _pt##r
#else
#define PROF_BEGIN(r)
#define PROF_END(r)
#endif

// Ordering of the two-warp channel (CM = channel mode): 0 = both warps in one
// CTA (CTA scope), 1 = the two CTAs of a cluster (cluster scope, DSMEM),
// 2 = the two warps in different kernels (GPU scope, the channel in HBM).
template <int CM>
__device__ __forceinline__ void chan_fence() {
  if constexpr (CM == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  else if constexpr (CM == 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
  else __threadfence_block();
}
// acquire load of a channel word from this warp's own copy
template <int CM>
__device__ __forceinline__ long long chan_ld(const volatile long long* p) {
  long long v;
  if constexpr (CM == 2) {
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  } else if constexpr (CM == 1) {
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void*)p);
    asm volatile("ld.acquire.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  } else {
    v = *p;
    __threadfence_block();
  }
  return v;
}
template <int CM>
__device__ __forceinline__ int chan_ld(const volatile int* p) {
  int v;
  if constexpr (CM == 2) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  } else if constexpr (CM == 1) {
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void*)p);
    asm volatile("ld.acquire.cluster.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  } else {
    v = *p;
    __threadfence_block();
  }
  return v;
}

// kv_band (metrics.cpp:50-72) over every healthy, live decode unit, out of
// line (the single-instance sweep path computes the band in the step loop):
// the mean from the exact integer sum (bit-identical to the reference, whose
// partial sums are exact integers), then the reference's second pass
// sum (v - mean)^2 in FP64: lane partials + tree (<= 1e-15 rel.), or, when run
// records are kept (seq), sequentially in unit order (bit-exact).  Warp-wide.
__device__ __forceinline__ void kv_band_general_impl(const uint64_t* s_PK, int U, int Dd, int Dn,
                                             unsigned live, bool seq, double* band,
                                             int64_t* out_min, int64_t* out_max) {
  const int lane = lane_id();
  const bool all = live == (Dn == 32 ? 0xffffffffu : ((1u << Dn) - 1u));
  int64_t s1 = 0, cnt = 0, vmin = kInf64, vmax = -1;
#pragma unroll 1
  for (int u = lane; u < U; u += 32) {
    if (all || ((live >> (u / Dd)) & 1u)) {
      const int64_t v = (int64_t)(s_PK[u] & kKMask);
      s1 += v;
      cnt += 1;
      vmin = v < vmin ? v : vmin;
      vmax = v > vmax ? v : vmax;
    }
  }
  s1 = warp_sum_i64(s1);
  cnt = __reduce_add_sync(kFull, (unsigned)cnt);
  const double n_d = (double)cnt;
  const double mean = __ddiv_rn((double)s1, n_d);
  double var = 0.0;
  if (seq) {
    if (lane == 0)
      for (int u = 0; u < U; ++u)
        if (all || ((live >> (u / Dd)) & 1u)) {
          const double dv = __dsub_rn((double)(int64_t)(s_PK[u] & kKMask), mean);
          var = __dadd_rn(var, __dmul_rn(dv, dv));
        }
    var = __shfl_sync(kFull, var, 0);
  } else {
#pragma unroll 1
    for (int u = lane; u < U; u += 32) {
      if (all || ((live >> (u / Dd)) & 1u)) {
        const double dv = __dsub_rn((double)(int64_t)(s_PK[u] & kKMask), mean);
        var = __dadd_rn(var, __dmul_rn(dv, dv));
      }
    }
    var = warp_sum_f64(var);
  }
  band[0] = mean;
  band[1] = sqrt(__ddiv_rn(var, n_d));
  *out_min = warp_min_i64(vmin);
  *out_max = warp_max_i64(vmax);
}
// Out-of-line copy for the decode warp of a two-warp replica (its hot loop is
// instruction-cache bound); the one-warp kernels keep it inline (a call site
// costs them more in register allocation than the code it moves out).
__device__ __noinline__ void kv_band_general_ool(const uint64_t* s_PK, int U, int Dd, int Dn,
                                                 unsigned live, bool seq, double* band,
                                                 int64_t* out_min, int64_t* out_max) {
  kv_band_general_impl(s_PK, U, Dd, Dn, live, seq, band, out_min, out_max);
}

// KD: prefill DP units per lane, 1 (dp_degree <= 32) or 4 (<= 128).
// LOG: keep run records (compiled out of the sweep kernel).
// ROLE: 0 = the whole replica on one warp; 1 = the prefill warp and 2 = the
// decode warp of a two-warp replica (see the channel notes at the event loop).
// SD (decode warp only): the replica has one decode instance, the IQR
// policy, no batch cap, one token per step and no decode faults; those
// runtime parameters become constants, so the decode warp's code carries only
// the paths it can take (a smaller instruction-cache working set).
// SP (prefill warp only): SBS policy, no EndForward drops, no topology
// events and no prefill deaths, as constants (the prefill kernel's code
// carries only the SBS paths).
// PO (one-warp replica only): a prefill-only trace (every output_len <= 1,
// so no request ever reaches the decode side) with the SP constants: the
// decode code is compiled out of the one-warp kernel.
template <int KD, bool LOG, int ROLE, int CL, bool CA = false, bool SD = false, bool SP = false,
          bool PO = false>
__device__ void run_replica(const DevPoint& pt, DevResult& res, unsigned char* sm,
                            unsigned char* sm_peer) {
  static_assert(!(LOG && ROLE != 0), "run records are kept by the one-warp replica only");
  constexpr bool kPre = ROLE != 2;  // this warp runs the prefill side
  constexpr bool kDec = ROLE == 2 || (ROLE == 0 && !PO);  // this warp runs the decode side
  const int lane = lane_id();
  const unsigned lt_mask = lanemask_lt();

  // ---- constants hoisted out of the (global) descriptor
  static_assert(!SD || ROLE == 2, "SD specialises the decode warp");
  static_assert(!SP || ROLE != 2, "SP specialises the prefill side");
  static_assert(!PO || (ROLE == 0 && SP && !LOG), "PO: one-warp, simple, prefill-only");
  const int P = pt.P, Dn = SD ? 1 : pt.Dn, D = pt.D, Dd = pt.Dd, U = SD ? pt.Dd : pt.U;
  const int PD = P * D;
  const bool sbs = SP || pt.policy == kSbs;
  const int policy = SP ? (int)kSbs : pt.policy, dec_policy = SD ? (int)kIqr : pt.decode_policy;
  const int64_t c_chunk = pt.c_chunk;
  const int64_t N = pt.n_dev ? *pt.n_dev : pt.N;
  const int64_t horizon = pt.horizon, warmup = pt.warmup;
  const int F = pt.F, Fm = pt.F - 1, R = pt.R, BC = pt.BC;
  const int n_limit = pt.n_limit, cap_batch = SD ? 0 : pt.cap_batch, n_drops = SP ? 0 : pt.n_drops;
  const int n_topo = SP ? 0 : pt.n_topo, w_size = pt.w_size, QD = pt.QD, QP = pt.QP, QW = pt.QW;
  const bool per_req = pt.per_request != 0;
  const int64_t tps = SD ? 1 : pt.tps, t_default = pt.t_default;
  const double inv_dd = 1.0 / (double)(pt.Dd > 0 ? pt.Dd : 1);
  const double pf_base = pt.pf_base, pf_tok = pt.pf_tok, dc_base = pt.dc_base, dc_req = pt.dc_req,
               dc_kv = pt.dc_kv, iqr_k = pt.iqr_k, wd_mult = pt.wd_mult;
  const int64_t* __restrict__ g_arr = pt.arr;
  const int32_t* __restrict__ g_prompt = pt.prompt;
  const int32_t* __restrict__ g_output = pt.output;
  int64_t* const o_dispatch = pt.o_dispatch;
  int64_t* const o_pstart = pt.o_pstart;
  int64_t* const o_ftok = pt.o_ftok;
  int64_t* const o_comp = pt.o_comp;
  int8_t* const o_status = pt.o_status;
  int2* const g_fifo = pt.fifo;
  int4* const g_buckets = pt.buckets;
  uint64_t* const g_dwait = pt.dwait;
  int64_t* const g_log = LOG ? pt.log : nullptr;
  const int64_t log_cap = LOG ? pt.log_cap : 0;
  int64_t log_n = 0;

  // ---- shared-memory carve
  int64_t* s_out = (int64_t*)(sm + pt.sm_pf_out);
  int32_t* s_head = (int32_t*)(sm + pt.sm_pf_head);
  int32_t* s_tail = (int32_t*)(sm + pt.sm_pf_tail);
  int32_t* s_rel = (int32_t*)(sm + pt.sm_pf_rel);
  uint8_t* s_part = (uint8_t*)(sm + pt.sm_pf_part);
  uint64_t* s_PK = (uint64_t*)(sm + pt.sm_dPK);   // B << 48 | K per decode unit
  uint64_t* s_R = (uint64_t*)(sm + pt.sm_dR);     // completers this step: n << 48 | kv release
  uint32_t* s_S = (uint32_t*)(sm + pt.sm_dS);     // sorted K multiset over the unit list (K < 2^32)
  uint32_t* s_T = (uint32_t*)(sm + pt.sm_dT);     // radix-sort scratch
  int32_t* s_nst = (int32_t*)(sm + pt.sm_dnst);   // residents stamped at the next/current step
  int16_t* s_ul = (int16_t*)(sm + pt.sm_ulist);
  uint16_t* s_bcnt = (uint16_t*)(sm + pt.sm_bcnt);
  uint32_t* s_hist = (uint32_t*)(sm + pt.sm_hist);
  int4* s_stage = (int4*)(sm + pt.sm_stage);     // step-in-progress completers, per instance
  int64_t* s_wr = (int64_t*)(sm + pt.sm_wring);
  uint64_t* s_wk = (uint64_t*)(sm + pt.sm_wkeys);
  Counters* cn = (Counters*)(sm + (ROLE == 2 ? pt.sm_cnt2 : pt.sm_cnt));
  // two-warp replicas: every channel word is read from this warp's own copy
  // (chL) and written into the peer's (chR); one CTA (CL false): the same
  // struct; a CTA pair of a cluster (CL true): the peer CTA's shared memory
  Chan* const chL = CL == 2 ? pt.gchan : (Chan*)(sm + pt.sm_chan);
  Chan* const chR = CL == 2 ? pt.gchan : (Chan*)((CL ? sm_peer : sm) + pt.sm_chan);
  if (lane == 0) {
    long long* z = (long long*)cn;
    for (int i = 0; i < (int)(sizeof(Counters) / 8); ++i) z[i] = 0;
  }

  if (kPre)
#pragma unroll 1
    for (int g = lane; g < PD; g += 32) {
      s_out[g] = 0; s_head[g] = 0; s_tail[g] = 0; s_rel[g] = 0; s_part[g] = 0;
    }
  if (kDec) {
#pragma unroll 1
    for (int u = lane; u < U; u += 32) { s_PK[u] = 0; s_R[u] = 0; s_nst[u] = 0; }
#pragma unroll 1
    for (int b = lane; b < Dn * R; b += 32) s_bcnt[b] = 0;
  }
  __syncwarp();

  // ---- lane-resident instance state (lane p <-> prefill instance p,
  //      lane j <-> decode instance j; core.h:164-193)
  int pflags = (lane < P) ? F_HEALTHY : 0;
  int64_t p_started = 0, p_deadline = 0;
  int32_t p_td = 0;
  int64_t ef_t = kInf64, wd_t = kInf64;
  uint32_t ef_s = 0xffffffffu, wd_s = 0xffffffffu;
  const int64_t p_death = (!SP && lane < P) ? pt.death[lane] : kInf64;
  int32_t imm_dp = 0;  // RotationCursor::next_dp (baselines.h:17-20)
  int32_t ef_hidx = 0, ef_hext = 0;  // ROLE 1: handler that scheduled the live EndForward

  // SD (one decode instance): the instance's state is kept warp-uniform (every
  // lane applies every update), so reading it needs no shuffle
  constexpr bool UNI = SD;
  static_assert(!SD || ROLE == 2, "SD is the decode role's specialisation");
  int dflags = (UNI || lane < Dn) ? G_HEALTHY : 0;
  int64_t d_step = 0;
  int64_t ds_t = kInf64;
  uint32_t ds_s = 0xffffffffu;
  const int64_t d_death = (!SD && lane < Dn) ? pt.death[P + lane] : kInf64;
  int64_t d_res = 0;            // residents over the instance's units
  double d_worst = 0.0;         // max_u decode_per_request*B + decode_per_kv*K
  int64_t d_res_begin = 0;      // residents stamped at the running step
  int64_t ds_ts = 0;            // ROLE 2: scheduling time of the live decode step,
  int32_t ds_hk = 1, ds_hi = 0;  // its handler: 0 = EndForward #ds_hi, 1 = a decode step

  // ---- scheduler state (SchedulerState, core.h:197-218; new_cluster core.cpp:162-168)
  int64_t now = 0;
  const int64_t l_net = pt.l_net;
  int64_t t_bar = t_default;
  int32_t n_active = P;
  int64_t i_opt = (t_bar + l_net) / n_active;  // no max(1) initially (core.cpp:167)
  bool has_ld = false;
  int64_t last_disp = 0;
  int32_t last_inst = -1;
  int32_t win_n = 0, win_head = 0;
  int64_t win_sum = 0;
  int64_t tick_t = kInf64;
  uint32_t tick_s = 0;
  uint32_t seq = 0;
  int64_t next_id = 0, new_begin = 0;
  int32_t np = 0, pcur = 0;
  int32_t ndw = 0;
  int32_t topo_idx = 0;
  int32_t imm_next = 0;
  int64_t dec_rr = 0;
  int32_t mti = 312;
  // SD: every decode unit stays listed (no caps, deaths or topology)
  bool S_valid = false, ul_dirty = !SD, ul_ident = SD;
  bool S_gathered = false;      // s_S holds the unit Ks (unsorted) after a step
  // IQR fast path (one decode instance, every unit listed, U <= 1024): lane l
  // keeps the minimum of (B << 48 | K << 16 | u) over its units u = l mod 32
  bool lmin_ok = false;
  uint64_t lmin = UINT64_MAX;
  uint64_t S_mx = 0;
  // percentile ranks (decode_alloc.cpp:17-20) depend only on the unit count
  int pc_n = -1, lo25 = 0, hi25 = 0, lo75 = 0, hi75 = 0;
  double fr25 = 0.0, fr75 = 0.0;
  int32_t nul = SD ? pt.U : 0;
  int error = 0;
  int32_t pidx = 0, cur_ext = 0;   // ROLE 1: prefill-warp event index, handler is arrival/topology
  int32_t d_hk = 1, d_hi = 0;      // ROLE 2: handler of the decode event being processed
  int32_t ktail = 0;               // ROLE 1: hand-off keys written
  bool wreg = false;               // ROLE 2: the ndw (<= 32) waiters' sorted keys are in rkey
  uint64_t rkey = 0;

  // other-event cache (EF/WD/DS min)
  bool odirty = true;
  int64_t o_t = kInf64;
  uint32_t o_s = 0;
  int o_k = 0, o_i = 0;

  // ---- counters (shared memory, lane 0; the per-admission ones in registers)
  int64_t n_fb = 0, n_mask = 0, n_dsel = 0, n_events = 0, n_steps = 0, n_outtok = 0;
#ifdef SBS_PROF
  long long prof_acc[24] = {0};
  const long long prof_t0 = clock64();
#endif
#define CNT(f, v) do { if (lane == 0) cn->f += (v); } while (0)
  // append one fixed-size record (lane 0); overflow is reported, never silent
  auto log_rec = [&](int kind, int nw, int64_t a, int64_t b, int64_t c, int64_t d, int64_t e) {
    if (log_n + 1 + nw > log_cap) { log_n = log_cap + 1; error = kErrOverflow; return; }
    if (lane == 0) {
      int64_t* w = g_log + log_n;
      w[0] = kind | ((int64_t)nw << 8);
      if (nw > 0) w[1] = a;
      if (nw > 1) w[2] = b;
      if (nw > 2) w[3] = c;
      if (nw > 3) w[4] = d;
      if (nw > 4) w[5] = e;
    }
    log_n += 1 + nw;
  };

  // random decode policy: mt19937_64(seed ^ 0x9E3779B97F4A7C15) (simulation.cpp:42)
  if (dec_policy == kRandom) {
    if (lane == 0) {
      mt_seed_lane0(pt.mt, pt.rng_seed);
    }
    __syncwarp();
  }

  // ---- arrival stream: lane l holds arrival[abase + l]
  int64_t abase = 0;
  int64_t abuf = (lane < N) ? __ldg(g_arr + lane) : kInf64;
  int64_t anext = (32 + lane < N) ? __ldg(g_arr + 32 + lane) : kInf64;

  // =======================================================================
  // helpers (all warp-uniform)
  // =======================================================================
  auto p_flag = [&](int p, int f) -> bool { return (bcast(pflags, p) & f) != 0; };
  auto ib = [&](auto v, int j) { if constexpr (UNI) return v; else return bcast(v, j); };
  auto d_flag = [&](int j, int f) -> bool { return (ib(dflags, j) & f) != 0; };

  // maybe_die (simulation.cpp:122-126)
  auto maybe_die_p = [&](int p) {
    if constexpr (SP) return;  // (no prefill deaths)
    if (lane == p && !(pflags & F_DEAD) && now >= p_death) pflags |= F_DEAD;
  };
  auto maybe_die_d = [&](int j) {
    if constexpr (SD) return;  // (no decode deaths)
    bool died = false;
    if (lane == j && !(dflags & G_DEAD) && now >= d_death) { dflags |= G_DEAD; died = true; }
    if (__any_sync(kFull, died)) { ul_dirty = true; S_valid = false; S_gathered = false; }
  };

  auto arm_tick = [&](int64_t at) {  // simulation.cpp:234-238
    tick_t = at > now ? at : now;
    tick_s = seq++;
  };

  // recompute_interval (interval_control.cpp:18-24)
  auto recompute_interval = [&]() {
    t_bar = (win_n == 0) ? t_default : win_sum / (int64_t)win_n;
    if (n_active <= 0) return;
    int64_t v = (t_bar + l_net) / (int64_t)n_active;
    i_opt = v > 1 ? v : 1;
  };

  auto recompute_other = [&]() {
    if (ROLE == 2 && Dn == 1) {  // decode warp, one instance: its step is the only other event
      o_t = ib(ds_t, 0); o_s = ib(ds_s, 0); o_k = kEvDS; o_i = 0;
      odirty = false;
      return;
    }
    int64_t lt = ef_t;
    uint32_t ls = ef_s;
    int lk = kEvEF;
    if (wd_t < lt || (wd_t == lt && wd_s < ls)) { lt = wd_t; ls = wd_s; lk = kEvWD; }
    if (ds_t < lt || (ds_t == lt && ds_s < ls)) { lt = ds_t; ls = ds_s; lk = kEvDS; }
    int64_t m = warp_min_nonneg_i64(lt);  // event times are >= 0 (kInf64 when none)
    uint32_t cs = (lt == m) ? ls : 0xffffffffu;
    uint32_t ms = __reduce_min_sync(kFull, cs);
    unsigned who = __ballot_sync(kFull, lt == m && ls == ms);
    int src = __ffs(who) - 1;
    o_t = m; o_s = ms; o_k = bcast(lk, src); o_i = src;
    odirty = false;
  };

  // ---- prefix caches (cache-aware mode only): PrefixCache (core.cpp:13-75)
  // per prefill DP unit g as last-use stamps over keys pool * n_probes + j;
  // a larger stamp = nearer the front of the reference's LRU list.
  // (nothing is hoisted into registers: the Basic-mode loop must not pay)
  // longest_hit (core.cpp:33-41): the longest probe k <= prefix size cached on g
  auto cache_hit = [&](int g, int pool, int ps) -> int32_t {
    const int n_probes = pt.n_probes;
    int32_t best = 0;
    const int32_t* st = pt.c_stamp + (int64_t)g * pt.n_pools * n_probes + pool * n_probes;
    for (int j = 0; j < n_probes; ++j) {  // (no shuffles: callers may diverge)
      const int32_t k = pt.probe_k[j];
      if (k > ps) break;
      if (st[j] != 0) best = k;
    }
    return best;
  };
  // insert + evict_to_budget (core.cpp:43-75), warp-wide, lane j = probe j:
  // probe j takes stamp clock + j + 1 (touch and new alike), new entries add
  // k_j tokens; then the oldest entries go until the budget holds.
  auto cache_insert = [&](int g, int pool, int ps) {
    const int n_probes = pt.n_probes, n_keys = pt.n_pools * pt.n_probes;
    const int32_t my_probe = lane < n_probes ? pt.probe_k[lane] : 0x7fffffff;
    int32_t* const g_cstamp = pt.c_stamp;
    int64_t* const g_cused = pt.c_used;
    int32_t* const g_cclock = pt.c_clock;
    const bool act = my_probe <= ps;  // a prefix of the lanes (probes ascend)
    const unsigned m = __ballot_sync(kFull, act);
    if (m == 0) return;
    int32_t* st = g_cstamp + (int64_t)g * n_keys;
    const int32_t clk = g_cclock[g];
    int64_t add = 0;
    if (act) {
      const int key = pool * n_probes + lane;
      if (st[key] == 0) add = my_probe;
      st[key] = clk + lane + 1;
    }
    int64_t used = g_cused[g] + warp_sum_i64(add);
    __syncwarp();
    while (used > pt.cache_budget) {
      uint32_t best = 0xffffffffu;
      int bi = 0;
      for (int i = lane; i < n_keys; i += 32) {
        const uint32_t v = (uint32_t)st[i];
        if (v != 0 && v < best) { best = v; bi = i; }
      }
      const uint32_t mn = __reduce_min_sync(kFull, best);
      if (mn == 0xffffffffu) break;  // the list is empty
      const int victim = (int)__reduce_max_sync(kFull, best == mn ? (uint32_t)bi : 0u);
      used -= __shfl_sync(kFull, my_probe, victim % n_probes);
      __syncwarp();
      if (lane == 0) st[victim] = 0;
      __syncwarp();
    }
    if (lane == 0) {
      g_cclock[g] = clk + __popc(m);
      g_cused[g] = used;
    }
    __syncwarp();
  };

  // ---- completion (metrics.cpp:117-153 inputs): the loop only stamps the
  //      completion time; TTFT / scheduler / device waits, the window TTFT
  //      buffer, TPOT and the completion counts are derived from the
  //      per-request arrays by finalize_kernel after the run (deferred
  //      accounting: no gathers on the event chains).
  auto complete_req = [&](bool has, int64_t id, int64_t t_done) {
    if (has) {
      SBS_ASSERT(id >= 0 && id < N);
      o_comp[id] = t_done;
      if (per_req) o_status[id] = kStCompleted;
    }
  };

  // Pair mode 3 (the two warps in different kernels): a hand-off wait that
  // exceeds ~8 s of clock means the partner cannot make progress; the replica
  // stops with an invariant error instead of hanging the GPU.
  auto wait_expired = [&](long long& t0) -> bool {
    if constexpr (CL != 2) {
      return false;
    } else {
      const long long t = clock64();
      if (t0 == 0) { t0 = t; return false; }
      return t - t0 > 16000000000ll;
    }
  };

  // decode waiter key (DevPoint::kq_*): ascending == (prompt+output desc, id
  // asc) (simulation.cpp:446-453), carrying output_len when there is room
  auto wait_key = [&](int32_t prompt, int32_t out, int64_t id) -> uint64_t {
    const int ob = pt.kq_ob, ib = pt.kq_ib;
    const uint64_t len = (uint64_t)(int64_t)prompt + (uint64_t)(int64_t)out;
    return (((uint64_t)pt.kq_lmax - len) << (ib + ob)) | ((uint64_t)id << ob) |
           (ob ? (uint64_t)(uint32_t)out : 0ull);
  };

  // ---- decode unit list over healthy, live decode instances, skipping
  //      capped units (simulation.cpp:432-442)
  auto rebuild_ulist = [&]() {
    int cnt = 0;
#pragma unroll 1
    for (int base = 0; base < U; base += 32) {
      int u = base + lane;
      int fl = __shfl_sync(kFull, dflags, (u < U ? u / Dd : 0) & 31);
      bool in = u < U && (fl & G_HEALTHY) && !(fl & G_DEAD) &&
                (cap_batch <= 0 || (int64_t)(s_PK[u] >> 48) < cap_batch);
      unsigned m = __ballot_sync(kFull, in);
      if (in) s_ul[cnt + __popc(m & lt_mask)] = (int16_t)u;
      cnt += __popc(m);
    }
    __syncwarp();
    nul = cnt;
    ul_ident = cnt == U;
    ul_dirty = false;
    lmin_ok = false;  // per-lane minima are rebuilt by the next decode step
    S_valid = false;
    S_gathered = false;
  };

  // sorted K multiset (for Q1/Q3) by warp radix sort
  auto rebuild_S = [&]() {
#ifdef SBS_PROF
    prof_acc[18] += 1;  // sorts
#endif
    uint64_t mx = S_mx;
    if (!S_gathered) {
      mx = 0;
      if (ul_ident) {
#pragma unroll 1
        for (int i = lane; i < nul; i += 32) {
          uint64_t k = s_PK[i] & kKMask;
          s_S[i] = (uint32_t)k;
          mx = k > mx ? k : mx;
        }
      } else {
#pragma unroll 1
        for (int i = lane; i < nul; i += 32) {
          uint64_t k = s_PK[s_ul[i]] & kKMask;
          s_S[i] = (uint32_t)k;
          mx = k > mx ? k : mx;
        }
      }
      mx = (uint64_t)__reduce_max_sync(kFull, (uint32_t)mx);  // K < 2^32
    }
    S_gathered = false;
    __syncwarp();
    if (nul <= 64) warp_sort_reg_u32<2>(s_S, nul, lane);
    else if (SD || nul <= 512) warp_sort_reg_u32<16>(s_S, nul, lane);  // (SD: U <= 512)
    else warp_radix_sort<uint32_t>(s_S, s_T, s_hist, nul, mx ? 64 - __clzll((long long)mx) : 0, lane, lt_mask);
    S_valid = true;
  };

  // try_begin_decode_step (engine_model.cpp:153-179).  Every resident is
  // stamped (s_nst tracks them), the step time uses the maintained max.
  auto try_begin_step = [&](int j) {
    int fl = ib(dflags, j);
    if ((fl & G_STEP) || (fl & G_DEAD)) return;
    if (ib(d_res, j) == 0) return;
    double dur = __dadd_rn(dc_base, ib(d_worst, j));
    int64_t t_end = now + llround_ns(dur);
    if (UNI || lane == j) {
      d_step += 1;
      dflags |= G_STEP;
      ds_t = t_end;
      ds_s = seq;
      d_res_begin = d_res;
      ds_ts = now;
      ds_hk = d_hk;
      ds_hi = d_hi;
    }
    seq++;
    odirty = true;
    // This step's completion bucket is final now (requests admitted from here
    // on complete at a later step): copy its head into shared memory while the
    // step runs, so finish_step reads it without a global round trip.
    {
      const int64_t s1 = ib(d_step, j);
      const int bb = j * R + (int)(s1 & (R - 1));
      const int nb = s_bcnt[bb];
      if (lane < nb && lane < kStageEntries) {
        SBS_ASSERT(j >= 0 && j < Dn && bb >= 0 && bb < Dn * R);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(s_stage + j * kStageEntries + lane);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst),
                     "l"(g_buckets + (int64_t)bb * BC + lane) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };

  // IQR select over the unit list (decode_alloc.cpp:38-81); returns position.
  auto iqr_select = [&]() -> int {
    PROF_BEGIN(7);
    if (!S_valid) rebuild_S();
    PROF_END(7);
    PROF_BEGIN(5);
    if (SBS_UNLIKELY(pc_n != nul)) {
      const double r25 = __ddiv_rn(__dmul_rn((double)nul - 1.0, 25.0), 100.0);
      const double r75 = __ddiv_rn(__dmul_rn((double)nul - 1.0, 75.0), 100.0);
      lo25 = (int)floor(r25); hi25 = (int)ceil(r25); fr25 = __dsub_rn(r25, (double)lo25);
      lo75 = (int)floor(r75); hi75 = (int)ceil(r75); fr75 = __dsub_rn(r75, (double)lo75);
      pc_n = nul;
    }
    // the lex-min over all units (fast path) is reduced while the quartile
    // loads and the FP64 threshold chain are in flight
    uint32_t gh = 0xffffffffu, gl = 0xffffffffu;
    if (lmin_ok) {
      gh = __reduce_min_sync(kFull, (uint32_t)(lmin >> 32));
      gl = __reduce_min_sync(kFull, (uint32_t)(lmin >> 32) == gh ? (uint32_t)lmin : 0xffffffffu);
    }
    const uint32_t smin = s_S[0], smax = s_S[nul - 1];
    const double a1 = (double)s_S[lo25], b1 = (double)s_S[hi25];
    const double a3 = (double)s_S[lo75], b3 = (double)s_S[hi75];
    const double q1 = lo25 == hi25 ? a1 : __dadd_rn(a1, __dmul_rn(fr25, __dsub_rn(b1, a1)));
    const double q3 = lo75 == hi75 ? a3 : __dadd_rn(a3, __dmul_rn(fr75, __dsub_rn(b3, a3)));
    const double th = __dadd_rn(q3, __dmul_rn(iqr_k, __dsub_rn(q3, q1)));
    // (double)K <= th  <=>  K <= floor(th) for integer K < 2^53
    const double fth = floor(th);
    const int64_t thi = fth >= 281474976710656.0 ? (int64_t)kKMask : (fth < 0.0 ? -1 : (int64_t)fth);
    // safe set empty <=> min K > th (fallback); a proper subset <=> max K > th
    // (mask): both read off the sorted multiset, so the scan needs no count
    const bool fallback = (int64_t)smin > thi;
    n_fb += fallback ? 1 : 0;
    n_mask += (!fallback && (int64_t)smax > thi) ? 1 : 0;
    // lexicographic (B, K, position) as one u64: B << 48 | K << 16 | position
    // (K < 2^32, position < 2^16).  Fast path: the lex-min over all units is
    // the answer whenever it is safe (or the safe set is empty): the minimum
    // over a superset that lies in the set.
    if (lmin_ok) {
      const uint64_t gm = ((uint64_t)gh << 32) | gl;
      if (SBS_LIKELY(fallback || (int64_t)((gm >> 16) & 0xffffffffull) <= thi)) {
        PROF_END(5);
        return (int)(gm & 0xffffu);
      }
    }
    uint64_t best = UINT64_MAX;
    if (ul_ident) {
      // rolled, with the next unit's load issued ahead (hides the smem latency)
      uint64_t k = lane < nul ? s_PK[lane] : 0;
#pragma unroll 1
      for (int i = lane; i < nul; i += 32) {
        const uint64_t kn = i + 32 < nul ? s_PK[i + 32] : 0;
        const uint64_t c = (k & ~kKMask) | ((k & kKMask) << 16) | (uint64_t)i;
        if ((fallback || (int64_t)(k & kKMask) <= thi) && c < best) best = c;
        k = kn;
      }
    } else {
#pragma unroll 1
      for (int i = lane; i < nul; i += 32) {
        const uint64_t k = s_PK[s_ul[i]];
        const uint64_t c = (k & ~kKMask) | ((k & kKMask) << 16) | (uint64_t)i;
        if ((fallback || (int64_t)(k & kKMask) <= thi) && c < best) best = c;
      }
    }
    const uint32_t hi = (uint32_t)(best >> 32);
    const uint32_t mh = __reduce_min_sync(kFull, hi);
    const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? (uint32_t)best : 0xffffffffu);
    const int sel = (int)(ml & 0xffffu);
    PROF_END(5);
    return sel;
  };

  // S multiset: replace one copy of `oldv` by `newv` (> oldv).
  auto S_update = [&](uint64_t oldv, uint64_t newv) {
    const uint32_t o = (uint32_t)oldv, nv = (uint32_t)newv;
    int c_old, c_new;
    warp_lower_bound2<uint32_t>(s_S, nul, o, nv, lane, c_old, c_new);
    SBS_ASSERT(c_old >= 0 && c_old < c_new && c_new <= nul && s_S[c_old] == o);
    // shift S[c_old+1 .. c_new-1] left by one (128 per round: every load of a
    // round is issued before its stores), then S[c_new-1] = newv
#pragma unroll 1
    for (int base = c_old; base < c_new - 1; base += 128) {
      uint32_t v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = base + lane + 32 * q;
        v[q] = i < c_new - 1 ? s_S[i + 1] : 0u;
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = base + lane + 32 * q;
        if (i < c_new - 1) s_S[i] = v[q];
      }
      __syncwarp();
    }
    if (lane == 0) s_S[c_new - 1] = nv;
    __syncwarp();
  };

  // drain_decode_admissions (simulation.cpp:413-484)
  // then_j >= 0: the decode step just finished on instance then_j, whose
  // handler calls try_begin_decode_step after the drain (simulation.cpp:511);
  // it joins the drain's own begins (a second begin of a touched instance is
  // a no-op), so try_begin_step has a single call site.
  auto drain_decode = [&](int then_j) {
    uint32_t touched = 0;
    int32_t order_lane = -1;  // lane t holds the t-th instance to begin
    int ntouched = 0;
    if (ndw > 0) {
#ifdef SBS_PROF
    prof_acc[15] += 1;  // drains with waiters
#endif
    for (int j = 0; j < Dn; ++j) maybe_die_d(j);
    if (!wreg) warp_sort_buf<true>(g_dwait, ndw, lane);
    int wi = 0;
    int64_t w_id = 0;
    int32_t w_prompt = 0, w_out = 0;
    const int kq_ob = pt.kq_ob, kq_ib = pt.kq_ib;
    while (wi < ndw) {
      if (SBS_UNLIKELY(ul_dirty)) rebuild_ulist();
      if (nul == 0) break;
      if ((wi & 31) == 0) {  // next 32 waiters: ids + lengths decoded in parallel
        const bool v = wi + lane < ndw;
        const uint64_t w_key = wreg ? rkey : (v ? g_dwait[wi + lane] : 0);
        w_id = (int64_t)((w_key >> kq_ob) & ((1ull << kq_ib) - 1));
        if (SBS_LIKELY(kq_ob != 0)) {  // lengths travel in the key
          w_out = (int32_t)(w_key & ((1ull << kq_ob) - 1));
          w_prompt = (int32_t)((int64_t)pt.kq_lmax - (int64_t)(w_key >> (kq_ib + kq_ob)) - w_out);
        } else {
          w_prompt = v ? __ldg(g_prompt + w_id) : 0;
          w_out = v ? __ldg(g_output + w_id) : 0;
        }
      }
      const int64_t id = bcast(w_id, wi & 31);
      const int32_t prompt = bcast(w_prompt, wi & 31);
      const int32_t out = bcast(w_out, wi & 31);
      int pos;
      if (SBS_LIKELY(dec_policy == kIqr)) {
        pos = iqr_select();
      } else if (dec_policy == kRandom) {
        if (mti >= 312) {
          if constexpr (ROLE == 2) mt_twist_ool(pt.mt); else mt_twist(pt.mt);
          mti = 0;
        }
        uint64_t y = mt_temper(pt.mt[mti]);
        mti += 1;
        double u01 = (double)(y >> 11) * 0x1.0p-53;
        int64_t q = (int64_t)__dmul_rn(u01, (double)nul);
        pos = (int)(q < nul - 1 ? q : nul - 1);
      } else {
        pos = (int)(dec_rr % nul);
        dec_rr += 1;
      }
      n_dsel += 1;
#ifdef SBS_PROF
      const long long pa0 = clock64();
#endif
      const int u = ul_ident ? pos : s_ul[pos];
      const int j = Dn == 1 ? 0 : u / Dd;
      // admit_decode (engine_model.cpp:145-151): B += 1, K += prompt_len
      SBS_ASSERT(u >= 0 && u < U && j >= 0 && j < Dn && id >= 0 && id < N && prompt >= 1 && out > 1);
      const uint64_t k0 = s_PK[u];
      const uint64_t K0 = k0 & kKMask, B0 = k0 >> 48;
      const uint64_t K1 = K0 + (uint64_t)prompt;
      if (SBS_UNLIKELY(B0 + 1 >= (1u << 15) || K1 >= (1ull << 32))) { error = kErrEnvelope; return; }
      const bool stepping = d_flag(j, G_STEP);
      __syncwarp();
      if (lane == 0) {
        s_PK[u] = k0 + kBOne + (uint64_t)prompt;
        if (!stepping) s_nst[u] += 1;  // stamped by the step that begins next
        if (per_req) o_status[id] = kStDecoding;
      }
      if (UNI || lane == j) {
        d_res += 1;
        double t = __dadd_rn(__dmul_rn(dc_req, (double)(B0 + 1)), __dmul_rn(dc_kv, (double)K1));
        d_worst = t > d_worst ? t : d_worst;
      }
      __syncwarp();
      if (lmin_ok) {  // unit u's owner lane re-takes its minimum (all lanes load one unit each)
        const int ow = u & 31, v = ow + 32 * lane;
        uint64_t c = UINT64_MAX;
        if (v < U) {
          const uint64_t k = s_PK[v];
          c = (k & ~kKMask) | ((k & kKMask) << 16) | (uint64_t)v;
        }
        const uint32_t h = __reduce_min_sync(kFull, (uint32_t)(c >> 32));
        const uint32_t l = __reduce_min_sync(kFull, (uint32_t)(c >> 32) == h ? (uint32_t)c : 0xffffffffu);
        if (lane == ow) lmin = ((uint64_t)h << 32) | l;
      }
      PROF_BEGIN(6);
      if (S_valid) S_update(K0, K1);
      PROF_END(6);
      if (SBS_UNLIKELY(cap_batch > 0 && (int64_t)B0 + 1 >= cap_batch)) ul_dirty = true;
      // completion ring: finishes at step d_step + ceil(target/tps)
      const int64_t target = (int64_t)out - 1;
      const int64_t nsteps = tps == 1 ? target : (target + tps - 1) / tps;
      const int64_t excess = nsteps * tps - target;
      const int64_t c = ib(d_step, j) + nsteps;
      const int b = j * R + (int)(c & (R - 1));
      const int cnt = s_bcnt[b];
      if (SBS_UNLIKELY(cnt >= BC)) { error = kErrOverflow; return; }
      if (lane == 0) {
        SBS_ASSERT(b >= 0 && b < Dn * R && cnt >= 0 && cnt < BC && u >= 0 && u < U);
        g_buckets[(int64_t)b * BC + cnt] =
            make_int4((int)id, u, (int)(prompt + target + excess), (int)excess);
        s_bcnt[b] = (uint16_t)(cnt + 1);
      }
      __syncwarp();
      if (!(touched & (1u << j))) {
        touched |= 1u << j;
        if (lane == ntouched) order_lane = j;
        ntouched += 1;
      }
#ifdef SBS_PROF
      prof_acc[19] += clock64() - pa0;  // admission bookkeeping (incl. S_update)
#endif
      wi += 1;
    }
    // keep unadmitted waiters (still sorted)
    if (wreg) {
      if (lane >= wi && lane < ndw) g_dwait[lane - wi] = rkey;
      __syncwarp();
      wreg = false;
    } else if (wi > 0 && wi < ndw) {
#pragma unroll 1
      for (int base = 0; base < ndw - wi; base += 32) {
        int i = base + lane;
        uint64_t v = (i < ndw - wi) ? g_dwait[wi + i] : 0;
        __syncwarp();
        if (i < ndw - wi) g_dwait[i] = v;
        __syncwarp();
      }
    }
    ndw -= wi;
    }
    if (then_j >= 0 && !(touched & (1u << then_j))) {
      if (lane == ntouched) order_lane = then_j;
      ntouched += 1;
    }
    PROF_BEGIN(10);
    for (int t = 0; t < ntouched; ++t) try_begin_step(Dn == 1 ? 0 : bcast(order_lane, t));
    PROF_END(10);
  };

  // try_begin_prefill_pass (engine_model.cpp:51-116) + record_pass
  auto try_start_pass = [&](int p) {
    int fl = bcast(pflags, p);
    if ((fl & F_BUSY) || (fl & F_DEAD)) return;
    const int g0 = p * D;
    bool any = false;
    for (int d = lane; d < D; d += 32) any |= s_head[g0 + d] != s_tail[g0 + d];
    if (!__any_sync(kFull, any)) return;
    int64_t amax = 0;
    double terms[KD];
    int64_t asg[KD];
#pragma unroll
    for (int k = 0; k < KD; ++k) {
      terms[k] = 0.0;
      int d = lane + 32 * k;
      if (d >= D) continue;
      int g = g0 + d;
      int32_t h = s_head[g], t = s_tail[g];
      bool part = s_part[g] != 0;
      int64_t outv = s_out[g];
      int64_t room = c_chunk;
      int2* fq = g_fifo + (int64_t)g * F;
      while (room > 0 && h != t) {
        int2 e = fq[h & Fm];
        int64_t take = (int64_t)e.y < room ? (int64_t)e.y : room;
        room -= take;
        if (!part) {
          o_pstart[e.x] = now;
          if (per_req) o_status[e.x] = kStPrefilling;
        }
        outv -= take;
        if (take == e.y) { h += 1; part = false; }
        else { fq[h & Fm].y = e.y - (int)take; part = true; }
      }
      s_head[g] = h;
      s_part[g] = part ? 1 : 0;
      s_out[g] = outv;
      int64_t assigned = c_chunk - room;
      asg[k] = assigned;
      amax = assigned > amax ? assigned : amax;
      // min(a, c) / c (metrics.cpp:199-200); exact shortcuts for full/empty units
      terms[k] = assigned >= c_chunk ? 1.0
               : assigned == 0 ? 0.0 : __ddiv_rn((double)assigned, (double)c_chunk);
    }
    amax = (int64_t)__reduce_max_sync(kFull, (uint32_t)amax);  // 0 <= assigned <= c_chunk < 2^31
    if (g_log) {  // record_pass (simulation.cpp:229, metrics.cpp:76-86)
      if (log_n + 3 + D > log_cap) {
        log_n = log_cap + 1;
        error = kErrOverflow;
      } else {
        if (lane == 0) {
          g_log[log_n] = LOG_PASS | ((int64_t)(2 + D) << 8);
          g_log[log_n + 1] = now;
          g_log[log_n + 2] = p;
        }
#pragma unroll
        for (int k = 0; k < KD; ++k)
          if (lane + 32 * k < D) g_log[log_n + 3 + lane + 32 * k] = asg[k];
        log_n += 3 + D;
      }
    }
    double dur = __dadd_rn(pf_base, __dmul_rn(pf_tok, (double)amax));
    int64_t t_end = now + llround_ns(dur);
    if (now >= warmup) {
      // chunk_utilization (metrics.cpp:193-202): sequential sum in DP order
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < KD; ++k) {
        if (32 * k >= D) break;
        for (int l = 0; l < 32 && 32 * k + l < D; ++l)
          sum = __dadd_rn(sum, __shfl_sync(kFull, terms[k], l));
      }
      if (lane == 0) {
        cn->util = __dadd_rn(cn->util, __ddiv_rn(sum, (double)D));
        cn->passes += 1;
      }
    }
    if (lane == p) {
      pflags |= F_BUSY;
      p_started = now;
      ef_t = t_end;
      ef_s = seq;
      ef_hidx = pidx;
      ef_hext = cur_ext;
    }
    seq++;
    odirty = true;
    __syncwarp();
  };

  // finish_prefill_pass (engine_model.cpp:118-141) + hand_off_finished
  // (simulation.cpp:397-411).  Finished order is unobservable (see header).
  auto finish_pass = [&](int p) {
    const int g0 = p * D;
    int d = lane;
    int32_t idx = 0, end = 0;
    if (d < D) { idx = s_rel[g0 + d]; end = s_head[g0 + d]; }
    for (;;) {
      while (d < D && idx == end) {
        s_rel[g0 + d] = end;
        d += 32;
        if (d < D) { idx = s_rel[g0 + d]; end = s_head[g0 + d]; }
      }
      bool has = d < D;
      if (!__any_sync(kFull, has)) break;
      int64_t id = 0;
      int32_t out = 0;
      if (has) {
        id = g_fifo[(int64_t)(g0 + d) * F + (idx & Fm)].x;
        SBS_ASSERT(g0 + d < PD && id >= 0 && id < N);
        idx += 1;
        out = __ldg(g_output + id);
        o_ftok[id] = now;
      }
      bool done = has && out <= 1;   // decode_target() == 0
      bool wait = !PO && has && out > 1;  // (PO: every output_len <= 1)
      complete_req(done, id, now);
      unsigned m = __ballot_sync(kFull, wait);
      if (ROLE == 1) {
        // hand-off ring: wait for room (the decode warp consumes independently);
        // one EndForward's keys must fit the ring whole, else run on one warp
        if (m && ndw + 32 > kChanKeys) { error = kErrSplitTie; break; }
        if (m) {
#ifdef SBS_PROF
          const long long pk0 = clock64();
#endif
          long long w0 = 0;
          for (;;) {
            const int kh = chL->khead;
            if (ktail + 32 - kh <= kChanKeys) break;
            if (SBS_UNLIKELY(wait_expired(w0))) { error = kErrInvariant; break; }
            __nanosleep(100);
          }
#ifdef SBS_PROF
          prof_acc[17] += clock64() - pk0;
#endif
          chan_fence<CL>();
          if (wait) {
            int32_t prompt = __ldg(g_prompt + id);
            chR->keys[(ktail + __popc(m & lt_mask)) % kChanKeys] = wait_key(prompt, out, id);
          }
          ktail += __popc(m);
          ndw += __popc(m);  // keys of this EndForward
        }
      } else {
        if (wait) {
          int32_t prompt = __ldg(g_prompt + id);
          SBS_ASSERT(ndw + __popc(m & lt_mask) < QD);
          g_dwait[ndw + __popc(m & lt_mask)] = wait_key(prompt, out, id);
        }
        ndw += __popc(m);
        if (ndw > QD - 32) { error = kErrOverflow; break; }
      }
    }
    if (lane == p) pflags &= ~F_BUSY;
    __syncwarp();
  };

  // FIFO push (dispatch_prefill, engine_model.cpp:37-49), by the owning lane.
  auto fifo_push = [&](int g, int64_t id, int32_t tokens) -> bool {
    int32_t t = s_tail[g];
    if (t - s_rel[g] >= F) return false;
    SBS_ASSERT(g >= 0 && g < PD && id >= 0 && id < N);
    g_fifo[(int64_t)g * F + (t & Fm)] = make_int2((int)id, tokens);
    s_tail[g] = t + 1;
    s_out[g] += tokens;
    return true;
  };

  // ---------------- perform_dispatch (simulation.cpp:265-342) ----------------
  // Returns p when requests were dispatched (the caller then runs maybe_die,
  // try_start_pass and the trailing tick, simulation.cpp:338-341), else -1.
  auto perform_dispatch = [&](int p) -> int {
    const int g0 = p * D;
    int64_t cap[KD];
#pragma unroll
    for (int k = 0; k < KD; ++k) {
      int d = lane + 32 * k;
      cap[k] = d < D ? c_chunk - s_out[g0 + d] : INT64_MIN;
    }
    // q_new keys, sorted
    const int nn = (int)(next_id - new_begin);
    uint64_t* nk = (nn <= kSmemWinKeys) ? s_wk : pt.wscr;
    if (nn > QW) { error = kErrOverflow; return -1; }
    for (int i = lane; i < nn; i += 32) {
      int64_t id = new_begin + i;
      nk[i] = pbaa_key(__ldg(g_prompt + id), id);
    }
    __syncwarp();
    warp_sort_buf(nk, nn, lane);
    uint64_t* pk = pt.pend_key[pcur];
    int32_t* pw = pt.pend_wait[pcur];
#ifdef SBS_PROF
    prof_acc[22] += np;
    prof_acc[23] += nn;
#endif
    bool ovf = false;
    constexpr uint64_t kPlaced = ~0ull;  // cache-aware mode: a placed queue entry

    // greedy phase over a sorted queue; returns number placed (a prefix)
    auto greedy = [&](const uint64_t* q, int n, bool& stopped) -> int {
      int i = 0;
      uint64_t kreg = 0;
      stopped = false;
      while (i < n) {
        if ((i & 31) == 0) kreg = (i + lane < n) ? q[i + lane] : 0;
        uint64_t key = bcast(kreg, i & 31);
        int32_t len = key_len(key);
        // argmax c_avail (== argmax capacity_after in Basic mode), lowest index
        uint32_t lv = 0;
        int ld = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < KD; ++k) {
          int64_t c = cap[k];
          uint32_t v = c > 0 ? (uint32_t)c : 0u;
          if (v > lv) { lv = v; ld = lane + 32 * k; }
        }
        uint32_t m = __reduce_max_sync(kFull, lv);
        if (m == 0) { stopped = true; break; }  // guard c_avail > 0 fails for all
        int best = (int)__reduce_min_sync(kFull, lv == m ? (uint32_t)ld : 0x7fffffffu);
        int64_t id = key_id(key);
        int32_t tokens = len > 1 ? len : 1;  // max(1, prompt - hit)
        if (lane == (best & 31)) {
#pragma unroll
          for (int k = 0; k < KD; ++k)
            if (k == (best >> 5)) cap[k] -= len;
          if (!fifo_push(g0 + best, id, tokens)) ovf = true;
          o_dispatch[id] = now;
          if (per_req) o_status[id] = kStDispatched;
        }
        i += 1;
      }
      return i;
    };
    // cache-aware greedy (capacity_after with Len_hit, prefill_alloc.cpp:12-21):
    // the argmax differs per request, so a guard failure defers only this
    // request; placed entries are marked and the deferred ones kept in order
    auto greedy_cache = [&](uint64_t* q, int n) -> int {
      int placed = 0;
      uint64_t kreg = 0;
      int32_t preg = -1, sreg = 0;
      for (int i = 0; i < n; ++i) {
        if ((i & 31) == 0) {
          kreg = (i + lane < n) ? q[i + lane] : 0;
          const int64_t qid = key_id(kreg);
          preg = (i + lane < n) ? __ldg(pt.pfx_pool + qid) : -1;
          sreg = (i + lane < n) ? __ldg(pt.pfx_size + qid) : 0;
        }
        const uint64_t key = bcast(kreg, i & 31);
        const int pool = bcast(preg, i & 31), ps = bcast(sreg, i & 31);
        const int32_t len = key_len(key);
        int64_t ba = INT64_MIN;
        int bd = 0x7fffffff;
        int32_t bh = 0;
        bool room = false;
#pragma unroll
        for (int k = 0; k < KD; ++k) {
          const int d = lane + 32 * k;
          if (d >= D) continue;
          const int32_t hit = pool >= 0 ? cache_hit(g0 + d, pool, ps) : 0;
          const int64_t after = cap[k] - (int64_t)(len - hit);
          if (after > ba) { ba = after; bd = d; bh = hit; }
          room |= cap[k] > 0;
        }
        if (!__any_sync(kFull, room)) break;  // no unit has headroom: the rest defer
        const int64_t mx = warp_max_i64(ba);
        const int best = (int)__reduce_min_sync(kFull, ba == mx ? (uint32_t)bd : 0x7fffffffu);
        int64_t cb = 0;
#pragma unroll
        for (int k = 0; k < KD; ++k)
          if (k == (best >> 5)) cb = cap[k];
        cb = __shfl_sync(kFull, cb, best & 31);
        if (cb <= 0) continue;  // guard on the argmax unit: deferred
        if (lane == (best & 31)) {
#pragma unroll
          for (int k = 0; k < KD; ++k)
            if (k == (best >> 5)) cap[k] = mx;
          const int64_t id = key_id(key);
          const int32_t tokens = len - bh > 1 ? len - bh : 1;  // max(1, prompt - hit)
          if (!fifo_push(g0 + best, id, tokens)) ovf = true;
          o_dispatch[id] = now;
          if (per_req) o_status[id] = kStDispatched;
        }
        if (lane == 0) q[i] = kPlaced;
        placed += 1;
      }
      __syncwarp();
      return placed;
    };
    int k1 = 0, k2 = 0, nplaced = 0;
    int32_t tail0[KD];  // per-DP FIFO tails before this dispatch
    int nn_left = nn;
    if constexpr (CA) {
#pragma unroll
      for (int k = 0; k < KD; ++k) {
        const int d = lane + 32 * k;
        tail0[k] = d < D ? s_tail[g0 + d] : 0;
      }
      nplaced = greedy_cache(pk, np);
      nplaced += greedy_cache(nk, nn);
      // keep the unplaced new keys, in order, at the front of nk
      int kept = 0;
      for (int base = 0; base < nn; base += 32) {
        const int i = base + lane;
        const uint64_t v = i < nn ? nk[i] : kPlaced;
        const bool keep = v != kPlaced;
        const unsigned km = __ballot_sync(kFull, keep);
        __syncwarp();
        if (keep) nk[kept + __popc(km & lt_mask)] = v;
        kept += __popc(km);
        __syncwarp();
      }
      nn_left = kept;
    } else {
      bool stopped = false;
      k1 = greedy(pk, np, stopped);
      if (!stopped) k2 = greedy(nk, nn, stopped);
      nplaced = k1 + k2;
      nn_left = nn - k2;
    }
    if (__any_sync(kFull, ovf)) { error = kErrOverflow; return -1; }
    CNT(alloc, 1);

    // aging (prefill_alloc.cpp:70-87): pending suffix then new suffix
    int na = 0, thr = 0;
    for (int base = k1; base < np; base += 32) {
      int i = base + lane;
      SBS_ASSERT(np <= QP);
      uint64_t key = i < np ? pk[i] : 0;
      bool valid = i < np && key != kPlaced;
      int32_t w = valid ? pw[i] + 1 : 0;
      bool th = valid && w > n_limit;
      bool keep = valid && !th;
      if (th && per_req) o_status[key_id(key)] = kStThrottled;
      unsigned m = __ballot_sync(kFull, keep);
      int pos = na + __popc(m & lt_mask);
      __syncwarp();
      if (keep) { pk[pos] = key; pw[pos] = w; }
      na += __popc(m);
      thr += __popc(__ballot_sync(kFull, th));
      __syncwarp();
    }
    int nb = nn_left;
    int nbk = nb;
    if (nb > 0 && 1 > n_limit) {
      for (int i = lane; i < nb; i += 32)
        if (per_req) o_status[key_id(nk[k2 + i])] = kStThrottled;
      thr += nb;
      nbk = 0;
    }
    CNT(def, na + nbk);
    CNT(throttled, thr);
    if (thr > 0) CNT(flow, 1);
    if (na + nbk > QP) { error = kErrOverflow; return -1; }
    if (nbk > 0) {
      if (na == 0) {
        for (int i = lane; i < nbk; i += 32) { pk[i] = nk[k2 + i]; pw[i] = 1; }
      } else {
        uint64_t* ok = pt.pend_key[pcur ^ 1];
        int32_t* ow = pt.pend_wait[pcur ^ 1];
        const uint64_t* bk = nk + k2;
        for (int i = lane; i < na; i += 32) {
          uint64_t x = pk[i];
          int pos = i + lower_bound_u64(bk, nbk, x);
          ok[pos] = x; ow[pos] = pw[i];
        }
        for (int j = lane; j < nbk; j += 32) {
          uint64_t y = bk[j];
          int pos = j + lower_bound_u64(pk, na, y);
          ok[pos] = y; ow[pos] = 1;
        }
        pcur ^= 1;
      }
    }
    __syncwarp();
    np = na + nbk;
    new_begin = next_id;  // q_new.clear()

    if (nplaced == 0) {
      if (np > 0) arm_tick(now + i_opt);
      return -1;
    }
    if constexpr (CA) {
      // register the dispatched prefixes (simulation.cpp:319-326) after every
      // hit was resolved; per DP unit in mapping order (= its FIFO order)
      for (int d = 0; d < D; ++d) {
        const int g = g0 + d;
        int32_t t0 = 0;
#pragma unroll
        for (int k = 0; k < KD; ++k)
          if (k == (d >> 5)) t0 = tail0[k];
        t0 = __shfl_sync(kFull, t0, d & 31);
        const int32_t te = s_tail[g];
        for (int32_t t = t0; t < te; ++t) {
          const int rid = g_fifo[(int64_t)g * F + (t & Fm)].x;
          const int pool = __ldg(pt.pfx_pool + rid);
          if (pool >= 0) cache_insert(g, pool, __ldg(pt.pfx_size + rid));
        }
      }
    }
    has_ld = true;
    last_disp = now;
    last_inst = p;
    // arm_watchdog (interval_control.cpp:76-86)
    int64_t deadline = now + (int64_t)llround(__dmul_rn(wd_mult, (double)t_bar));
    if (lane == p) {
      p_td += 1;
      pflags &= ~(F_EFSEEN | F_WDFIRED);
      pflags |= F_HASDL;
      p_deadline = deadline;
      wd_t = deadline;
      wd_s = seq;
    }
    seq++;
    odirty = true;
    if (g_log) {  // simulation.cpp:335-336
      log_rec(LOG_DISPATCH, 2, now, p, 0, 0, 0);
      log_rec(LOG_CONTROL, 4, now, i_opt, t_bar, n_active, 0);
    }
    return p;
  };

  // ---------------- try_dispatch (simulation.cpp:245-263) ----------------
  auto try_dispatch = [&]() -> int {
    if (np + (next_id - new_begin) == 0) return -1;
    if (n_active <= 0) return -1;
    if (has_ld && now < last_disp + i_opt) { arm_tick(last_disp + i_opt); return -1; }
    // select_ready_instance (interval_control.cpp:50-74)
    unsigned hm = __ballot_sync(kFull, lane < P && (pflags & F_HEALTHY));
    unsigned gt = last_inst < 0 ? 0xffffffffu : (unsigned)(~((2ull << last_inst) - 1ull));
    unsigned cand = hm & gt;
    int target = cand ? __ffs(cand) - 1 : (hm ? __ffs(hm) - 1 : -1);
    bool r = (p_td == 0 && !(pflags & F_BUSY)) || (pflags & F_EFSEEN) || (pflags & F_WDFIRED) ||
             ((pflags & F_HASDL) && now >= p_deadline);
    bool ready = __shfl_sync(kFull, (int)r, target < 0 ? 0 : target) != 0 && target >= 0;
    if (!ready) { arm_tick(now + i_opt); return -1; }
    return perform_dispatch(target);
  };

  // ---------------- baseline_dispatch (simulation.cpp:206-223) ----------------
  auto baseline_dispatch = [&](int64_t id) -> int {
    int tp = -1, tdp = -1;
    if (policy == kLeastOutstanding) {
      // least_outstanding (baselines.cpp:28-45)
      int64_t bv = kInf64;
      int bg = 0x7fffffff;
      for (int base = 0; base < PD; base += 32) {
        int g = base + lane;
        int inst = g < PD ? g / D : 0;
        int fl = __shfl_sync(kFull, pflags, inst & 31);
        if (g < PD && (fl & F_HEALTHY) && !(fl & F_DEAD)) {
          int64_t v = s_out[g];
          if (v < bv) { bv = v; bg = g; }
        }
      }
      int64_t mv = warp_min_nonneg_i64(bv);  // outstanding tokens >= 0 (kInf64 when none)
      int g = (int)__reduce_min_sync(kFull, bv == mv ? (uint32_t)bg : 0x7fffffffu);
      if (mv != kInf64) { tp = g / D; tdp = g % D; }
    } else {
      // immediate_dispatch (baselines.cpp:9-26)
      for (int tries = 0; tries < P; ++tries) {
        int pos = imm_next % P;
        imm_next = (pos + 1) % P;
        int fl = bcast(pflags, pos);
        if (!(fl & F_HEALTHY) || (fl & F_DEAD)) continue;
        int dp = bcast(imm_dp, pos) % D;
        if (lane == pos) imm_dp = (dp + 1) % D;
        tp = pos; tdp = dp;
        break;
      }
    }
    if (tp < 0) return -1;  // stays pending
    int32_t prompt = __ldg(g_prompt + id);
    bool ok = true;
    if (lane == 0) {
      o_dispatch[id] = now;
      if (per_req) o_status[id] = kStDispatched;
      ok = fifo_push(tp * D + tdp, id, prompt);
    }
    if (!bcast((int)ok, 0)) { error = kErrOverflow; return -1; }
    __syncwarp();
    if (g_log) log_rec(LOG_DISPATCH, 2, now, tp, 0, 0, 0);  // simulation.cpp:219
    return tp;
  };

  // finish_decode_step (engine_model.cpp:181-217), record_step and
  // record_kv_snapshot (simulation.cpp:486-512, metrics.cpp:50-72, 99-101)
  auto finish_step = [&](int j) {
    const int u0 = j * Dd;
    const int64_t s = ib(d_step, j);
    const int b = j * R + (int)(s & (R - 1));
    const int n = s_bcnt[b];
    const int4* ent = g_buckets + (int64_t)b * BC;
    SBS_ASSERT(j >= 0 && j < Dn && b >= 0 && b < Dn * R && n <= BC);
    const int4* stg = s_stage + j * kStageEntries;  // entries < kStageEntries (lane-owned copies)
    asm volatile("cp.async.wait_all;" ::: "memory");
    int64_t exc = 0;
    PROF_BEGIN(11);
#pragma unroll 1
    for (int base = 0; base < n; base += 32) {
      const int e = base + lane;
      if (e < n) {
        const int4 v = e < kStageEntries ? stg[e] : ent[e];
        SBS_ASSERT(v.y >= u0 && v.y < u0 + Dd && v.x >= 0 && v.x < N);
        complete_req(true, v.x, now);
        atomicAdd((unsigned long long*)&s_R[v.y], (unsigned long long)(kBOne | (uint64_t)(uint32_t)v.z));
        exc += v.w;
      }
    }
    __syncwarp();
    if (lane == 0) s_bcnt[b] = 0;
    PROF_END(11);
    PROF_BEGIN(12);
    // every stamped resident produced tps tokens (minus the last-step excess
    // of completers); completers release B and prompt + decode_done of K
    const bool gather = ul_ident && Dn == 1;  // s_S order == unit order
    // 32-bit unit arithmetic: K < 2^32 (decode-unit envelope, checked here:
    // a carry out of K + tps * stamped sets kErrEnvelope), B < 2^15, and
    // tps * stamped < 2^32 (tps < 2^17, host check)
    uint32_t mx = 0, ovf = 0;
    uint64_t s1 = 0, s2lo = 0, s2hi = 0;  // sum K, sum K^2 (128-bit)
    const bool band_fast = !LOG && Dn == 1 && now >= warmup;
    // step-time maximum over non-negative doubles == maximum of their bit
    // patterns (u64 compare: no FP64 compare on the loop-carried chain)
    uint64_t worst_b = 0;
    uint64_t lm = UINT64_MAX;
    const uint32_t tps32 = (uint32_t)tps;
    // software-pipelined: the next unit's three loads are issued before this
    // unit's stores, so their shared-memory latency overlaps this iteration
    uint64_t k = 0, r = 0;
    uint32_t st = 0;
    if (lane < Dd) { k = s_PK[u0 + lane]; r = s_R[u0 + lane]; st = (uint32_t)s_nst[u0 + lane]; }
#pragma unroll 1
    for (int d = lane; d < Dd; d += 32) {
      const int u = u0 + d;
      uint64_t k_nx = 0, r_nx = 0;
      uint32_t st_nx = 0;
      if (d + 32 < Dd) { k_nx = s_PK[u + 32]; r_nx = s_R[u + 32]; st_nx = (uint32_t)s_nst[u + 32]; }
      const uint32_t kk = (uint32_t)k, rk = (uint32_t)r;
      const uint32_t grown = kk + tps32 * st;
      ovf |= grown < kk;
      const uint32_t K = grown - rk;
      const uint32_t B = (uint32_t)(k >> 48) - (uint32_t)(r >> 48);
      s_PK[u] = ((uint64_t)B << 48) | K;
      const uint64_t c = ((uint64_t)((B << 16) | (K >> 16)) << 32) | ((K << 16) | (uint32_t)u);
      lm = c < lm ? c : lm;
      s_nst[u] = (int32_t)B;
      if (r) s_R[u] = 0;
      if (gather) s_S[u] = K;
      mx = K > mx ? K : mx;
      s1 += K;
      const uint64_t k2 = (uint64_t)K * K;
      s2lo += k2;
      s2hi += s2lo < k2;
      const double t = __dadd_rn(__dmul_rn(dc_req, (double)B), __dmul_rn(dc_kv, (double)K));
      const uint64_t tb = (uint64_t)__double_as_longlong(t);
      worst_b = tb > worst_b ? tb : worst_b;
      k = k_nx; r = r_nx; st = st_nx;
    }
    if (SBS_UNLIKELY(__any_sync(kFull, ovf != 0))) error = kErrEnvelope;
    double worst;
    PROF_END(12);
    PROF_BEGIN(13);
    // per-step reductions as independent 32-bit REDUX: the step time's max
    // over non-negative doubles is the max of their bit patterns; the exact
    // sums are split into chunks whose 32-lane sums cannot overflow 32 bits
    // (lane partials: sum K < 2^36, sum K^2 < 2^68)
    {
      const uint64_t wb = worst_b;
      const uint32_t wh = __reduce_max_sync(kFull, (uint32_t)(wb >> 32));
      const uint32_t wl = __reduce_max_sync(kFull, (uint32_t)(wb >> 32) == wh ? (uint32_t)wb : 0u);
      worst = __longlong_as_double((long long)(((uint64_t)wh << 32) | wl));
    }
    if (band_fast) {
      const uint32_t a_hi = __reduce_add_sync(kFull, (uint32_t)(s1 >> 16));
      const uint32_t a_lo = __reduce_add_sync(kFull, (uint32_t)(s1 & 0xffffu));
      const uint32_t c0 = __reduce_add_sync(kFull, (uint32_t)(s2lo & 0xffffffu));
      const uint32_t c1 = __reduce_add_sync(kFull, (uint32_t)((s2lo >> 24) & 0xffffffu));
      const uint32_t c2 = __reduce_add_sync(kFull, (uint32_t)(((s2lo >> 48) | (s2hi << 16)) & 0xffffffu));
      s1 = ((uint64_t)a_hi << 16) + a_lo;
      typedef unsigned __int128 u128;
      const u128 sq = (u128)c0 + ((u128)c1 << 24) + ((u128)c2 << 48);
      s2lo = (uint64_t)sq;
      s2hi = (uint64_t)(sq >> 64);
    }
    // (completers' excess <= n * tps and K < 2^32: single 32-bit REDUX each)
    exc = (int64_t)__reduce_add_sync(kFull, (uint32_t)exc);
    const int64_t stamped = ib(d_res_begin, j);
    const int64_t gen = tps * stamped - exc;
    if (UNI || lane == j) {
      d_res -= n;
      d_worst = worst;
      dflags &= ~G_STEP;
    }
    S_valid = false;
    lmin = lm;
    lmin_ok = SD || (dec_policy == kIqr && Dn == 1 && U <= 1024 && ul_ident && !ul_dirty);
    if (gather) {
      S_gathered = true;
      S_mx = (uint64_t)__reduce_max_sync(kFull, mx);
    }
    if (cap_batch > 0 && n > 0) ul_dirty = true;
    __syncwarp();
    if (now >= warmup) {
      if constexpr (ROLE == 2) { n_steps += 1; n_outtok += gen; }
      else { CNT(steps, 1); CNT(outtok, gen); }
    }
    if (g_log) log_rec(LOG_STEP, 2, now, gen, 0, 0, 0);  // record_step (simulation.cpp:507)
    PROF_END(13);
    PROF_BEGIN(14);
    if (SBS_LIKELY(band_fast)) {
      // single decode instance: the band comes from the step loop's exact sums
      // mean = sum/n (bit-identical); sum (v-mean)^2 = (n*sum v^2 - (sum v)^2)/n
      if (d_flag(0, G_HEALTHY) && !d_flag(0, G_DEAD) && lane == 0) {
        typedef unsigned __int128 u128;
        const double n_d = (double)Dd;
        const u128 sq = ((u128)s2hi << 64) | s2lo;
        const u128 x = (u128)(uint64_t)Dd * sq - (u128)s1 * (u128)s1;
        const double xd = __dadd_rn(__dmul_rn((double)(uint64_t)(x >> 64), 18446744073709551616.0),
                                    (double)(uint64_t)x);
        const double mean = __ddiv_rn((double)s1, n_d);  // == reference mean (exact sum)
        const double sigma = __dmul_rn(sqrt(xd), inv_dd);  // sqrt(sum (v-mean)^2 / n), ~1e-16
        cn->kv_mean = __dadd_rn(cn->kv_mean, mean);
        cn->kv_sig = __dadd_rn(cn->kv_sig, sigma);
        cn->kv_n += 1;
      }
    } else if (now >= warmup || g_log) {
      // kv_band (metrics.cpp:50-72) over every healthy, live decode unit:
      // the mean from the exact integer sum (bit-identical to the reference,
      // whose partial sums are exact integers), then the reference's second
      // pass sum (v - mean)^2 in FP64: lane partials + tree (<= 1e-15 rel.),
      // or, when run records are kept, sequentially in unit order (bit-exact).
      unsigned live = __ballot_sync(kFull, lane < Dn && (dflags & G_HEALTHY) && !(dflags & G_DEAD));
      if (live) {
        double band[2];
        int64_t vmin, vmax;
        if constexpr (ROLE == 2)
          kv_band_general_ool(s_PK, U, Dd, Dn, live, g_log != nullptr, band, &vmin, &vmax);
        else
          kv_band_general_impl(s_PK, U, Dd, Dn, live, g_log != nullptr, band, &vmin, &vmax);
        const double mean = band[0], sigma = band[1];
        if (g_log) {
          log_rec(LOG_KV, 5, now, __double_as_longlong(mean), __double_as_longlong(sigma), vmin, vmax);
          if (pt.log_kv_loads) {
            // the loads record_kv_snapshot hands to record_kv (simulation.cpp:486-495):
            // K of every unit of the healthy, live decode instances, in unit order
            const int nl = __popc(live) * Dd;
            if (log_n + 2 + nl > log_cap) {
              log_n = log_cap + 1;
              error = kErrOverflow;
            } else {
              if (lane == 0) {
                g_log[log_n] = LOG_KVLOADS | ((int64_t)(1 + nl) << 8);
                g_log[log_n + 1] = now;
              }
#pragma unroll 1
              for (int u = lane; u < U; u += 32) {
                const int inst = u / Dd;
                if ((live >> inst) & 1u)
                  g_log[log_n + 2 + __popc(live & ((1u << inst) - 1u)) * Dd + (u - inst * Dd)] =
                      (int64_t)(s_PK[u] & kKMask);
              }
              log_n += 2 + nl;
            }
          }
        }
        if (now >= warmup && lane == 0) {
          cn->kv_mean = __dadd_rn(cn->kv_mean, mean);
          cn->kv_sig = __dadd_rn(cn->kv_sig, sigma);
          cn->kv_n += 1;
        }
      }
    }
    PROF_END(14);
  };

  // drop_matches (simulation.cpp:128-134)
  auto drop_matches = [&](int p) -> bool {
    for (int i = 0; i < n_drops; ++i) {
      int inst = pt.drop_inst[i];
      if ((inst == -1 || inst == p) && now >= pt.drop_from[i] && now < pt.drop_until[i]) return true;
    }
    return false;
  };

  // =======================================================================
  // event loop (SimClock::run_until, simclock.cpp:32-45).  Each handler only
  // decides *which* actions run; the actions themselves have one call site
  // each (instruction-cache footprint) and run in the reference's order:
  //   finish_pass/finish_step -> drain_decode_admissions -> begin decode step
  //   -> try_start_pass -> [SBS EndForward ack] -> try_dispatch ->
  //   try_start_pass(target) -> trailing tick.
  // =======================================================================
  if constexpr (ROLE == 2) {
    // ===================================================================
    // Decode warp of a two-warp replica.  The decode side never feeds back
    // into the prefill side; it sees (a) its own decode steps, (b) topology
    // events of decode instances, (c) one record per EndForward from the
    // prefill warp (simulation.cpp:397-411 hand-off).  They are merged in the
    // reference's (time, seq) order: topology < EndForward/step by seq; an
    // EndForward/step tie at the same ns is ordered by their scheduling
    // times, then by the prefill-warp index of the scheduling handlers (an
    // EndForward's drain schedules steps before its own restart/dispatch),
    // then arrival/topology handlers before internal ones; anything deeper is
    // reported (kErrSplitTie) and the host reruns the replica on one warp.
    // The prefill warp publishes p_done = time of the next event it will
    // process, so a decode event at time c is safe once p_done > c.
    // ===================================================================
    int rhead = 0, khead = 0, dtopo = 0, pub_head = 0;
    int tail_seen = 0;  // records known published (re-read only once all are consumed)
    long long dwait0 = 0;  // start of the current wait on the prefill warp (pair mode 3 guard)
    bool aborted = false;
    auto next_dtopo = [&]() -> int64_t {
      while (dtopo < n_topo && pt.topo_inst[dtopo] < P) ++dtopo;
      return dtopo < n_topo ? pt.topo_time[dtopo] : kInf64;
    };
    int64_t dt_t = SD ? kInf64 : next_dtopo();  // (SD: no decode topology events)
    for (;;) {
      if (SBS_UNLIKELY(seq > kSeqLimit) && !aborted) { error = kErrEnvelope; aborted = true; }
      if (odirty) recompute_other();
      const int64_t td = o_t <= horizon ? o_t : kInf64;
      const int64_t tt = dt_t <= horizon ? dt_t : kInf64;
      // The queue first: a published record later than the next decode
      // event already proves that event safe (records come in time order),
      // so the progress word is read only when no record is known; then
      // progress before the queue (a record below the progress seen is
      // published before it).  Each acquire load is a round trip (HBM in
      // pair mode 3).
      long long pdone = 0;
      if (rhead >= tail_seen) {
        pdone = chan_ld<CL>(&chL->p_done);
        tail_seen = chan_ld<CL>(&chL->tail);
      }
      const bool have = rhead < tail_seen;
      const ChanRec* rc = &chL->rec[rhead % kChanRecs];
      const int64_t th = have ? rc->t : kInf64;
      if (SBS_UNLIKELY(aborted)) {  // keep the prefill warp unblocked until it finishes
        if (have) {
          rhead += 1;
          khead += rc->nk;
          chan_fence<CL>();
          __syncwarp();
          if (lane == 0) { chR->head = rhead; chR->khead = khead; }
          continue;
        }
        if (pdone == kInf64) break;
        if (SBS_UNLIKELY(wait_expired(dwait0))) break;
        __nanosleep(128);
        continue;
      }
      const int64_t c = td < tt ? td : tt;
      if (!have) {
        if (c == kInf64 && pdone == kInf64) break;  // all done
        if (pdone <= c) {  // an EndForward <= c may still come
#ifdef SBS_PROF
          prof_acc[16] += 164;  // ~cycles of one wait round (nanosleep 64 + polling)
#endif
          if (pub_head != rhead) {  // exact release before waiting on the prefill warp
            chan_fence<CL>();
            __syncwarp();
            if (lane == 0) { chR->head = rhead; chR->khead = khead; }
            pub_head = rhead;
          }
          if (SBS_UNLIKELY(wait_expired(dwait0))) { error = kErrInvariant; aborted = true; }
          __nanosleep(64);
          continue;
        }
      }
      dwait0 = 0;
      int kind;  // 0 record, 1 step, 2 topology
      if (tt <= th && tt <= td) {
        kind = 2;
      } else if (th < td) {
        kind = 0;
      } else if (th == td) {
        const int j = o_i;
        const int64_t tsd = ib(ds_ts, j);
        const int hk = ib(ds_hk, j), hi = ib(ds_hi, j);
        int ef_first;
        if (rc->ts != tsd) ef_first = rc->ts < tsd;
        else if (hk == 0) ef_first = rc->h_idx < hi;
        else if (rc->h_ext) ef_first = 1;
        else { error = kErrSplitTie; aborted = true; continue; }
        kind = ef_first ? 0 : 1;
      } else {
        kind = 1;
      }
      int step_j = -1;  // decode step handled: begin its next step after the drain
      if (kind == 0) {
        // ---- hand_off_finished (simulation.cpp:397-411) of one EndForward
        now = th;
        const int nk = rc->nk, k0 = rc->k0;
        d_hk = 0;
        d_hi = rc->ef_idx;
        if (SBS_UNLIKELY(ndw + nk + 32 > QD)) { error = kErrOverflow; aborted = true; continue; }
        // release the previous record's slots (its reads are long complete; this
        // record's are released at the next one, or exactly before a wait)
        if (lane == 0) { chR->head = rhead; chR->khead = khead; }
        pub_head = rhead;
        if (ndw == 0 && nk <= 32) {
          // the usual case: this record's waiters only, sorted in registers
          rkey = lane < nk ? chL->keys[(k0 + lane) % kChanKeys] : UINT64_MAX;
          if (nk > 1) rkey = warp_sort32_n(rkey, lane, nk);  // (lanes >= nk: UINT64_MAX)
          wreg = true;
        } else {
#pragma unroll 1
          for (int i = lane; i < nk; i += 32) {
            SBS_ASSERT(ndw + i < QD);
            g_dwait[ndw + i] = chL->keys[(k0 + i) % kChanKeys];
          }
        }
        ndw += nk;
        rhead += 1;
        khead += nk;
      } else if (kind == 1) {
        // ---- on_decode_step (simulation.cpp:497-512)
        now = td;
        n_events += 1;  // (ROLE 2: a register, flushed at the end)
        const int j = o_i;
        if (UNI || lane == j) ds_t = kInf64;
        odirty = true;
        maybe_die_d(j);
        if (d_flag(j, G_DEAD)) continue;
        PROF_BEGIN(3);
        finish_step(j);
        PROF_END(3);
        d_hk = 1;
        step_j = j;
      } else {
        // ---- on_topology for a decode instance (simulation.cpp:382-388)
        now = tt;
        const int inst = pt.topo_inst[dtopo];
        const bool h = pt.topo_healthy[dtopo] != 0;
        dtopo += 1;
        dt_t = next_dtopo();
        if (lane == inst - P) dflags = h ? (dflags | G_HEALTHY) : (dflags & ~G_HEALTHY);
        ul_dirty = true;
        S_valid = false;
        S_gathered = false;
      }
      if (kind != 2) {  // one call site: drain_decode is the largest inlined body
        PROF_BEGIN(4);
        drain_decode(step_j);
        PROF_END(4);
      }
      if (error) aborted = true;
    }
#ifdef SBS_PROF
    prof_acc[20] += clock64() - prof_t0;
#endif
  } else {
  int64_t topo_t = (n_topo > 0) ? pt.topo_time[0] : kInf64;
  int ch_tail = 0;
  if (g_log && sbs) log_rec(LOG_CONTROL, 4, 0, i_opt, t_bar, n_active, 0);  // simulation.cpp:152
  while (error == 0) {
    PROF_BEGIN(0);
    if (SBS_UNLIKELY(seq > kSeqLimit)) { error = kErrEnvelope; break; }
    if (odirty) recompute_other();
    // live internal minimum: tick vs other
    int64_t it = o_t;
    uint32_t is = o_s;
    int ik = o_k;
    if (tick_t < it || (tick_t == it && tick_s < is)) { it = tick_t; is = tick_s; ik = 1; }
    const int64_t at = (next_id < N) ? bcast(abuf, (int)(next_id - abase)) : kInf64;
    int kind;
    int64_t et;
    if (topo_t <= at && topo_t <= it) { kind = 4; et = topo_t; }  // topology (lowest seq)
    else if (at <= it) { kind = 0; et = at; }                      // arrival
    else { kind = ik; et = it; }
    if (et == kInf64 || et > horizon) break;
    now = et;
    PROF_END(0);
    CNT(events, 1);
    if (ROLE == 1) {
      // progress for the decode warp: every event before `et` is processed.
      // (Ordered after every earlier record by the fence that follows each
      // record publish; a stale value only makes the decode warp wait.)
      if (lane == 0) chR->p_done = et;
      pidx += 1;
      cur_ext = (kind == 0 || kind == 4) ? 1 : 0;
    }

    int start_p = -1;      // try_start_pass before the dispatch stage
    int step_j = -1;       // decode instance whose step finished
    int ef_p = -1;         // SBS EndForward acknowledgement
    int64_t measured = 0;
    bool dispatch = false;
    if (kind == 0) {
      // ---- on_arrival (simulation.cpp:196-204)
      const int64_t id = next_id;
      next_id += 1;
      if (next_id - abase == 32) {
        abase += 32;
        abuf = anext;
        anext = (abase + 32 + lane < N) ? __ldg(g_arr + abase + 32 + lane) : kInf64;
      }
      if (sbs) {
        dispatch = true;
      } else {
        start_p = baseline_dispatch(id);  // simulation.cpp:206-223
        if (start_p >= 0) maybe_die_p(start_p);
      }
    } else if (kind == 1) {
      // ---- on_tick (simulation.cpp:240-243): only the live tick reaches here
      tick_t = kInf64;
      dispatch = true;
    } else if (kind == kEvEF) {
      // ---- on_end_forward (simulation.cpp:346-372)
      const int p = o_i;
      if (lane == p) ef_t = kInf64;
      odirty = true;
      maybe_die_p(p);
      if (p_flag(p, F_DEAD)) continue;
      measured = now - bcast(p_started, p);
      PROF_BEGIN(2);
      finish_pass(p);
      PROF_END(2);
      if (ROLE == 1) {
        // hand-off record for the decode warp (one per EndForward)
        const int32_t hidx = bcast(ef_hidx, p), hext = bcast(ef_hext, p);
#ifdef SBS_PROF
        const long long pw0 = clock64();
#endif
        long long w0 = 0;
        for (;;) {
          const int hd = chL->head;
          if (ch_tail - hd < kChanRecs) break;
          if (SBS_UNLIKELY(wait_expired(w0))) { error = kErrInvariant; break; }
          __nanosleep(100);
        }
#ifdef SBS_PROF
        prof_acc[17] += clock64() - pw0;  // cycles waiting for record room
#endif
        chan_fence<CL>();
        if (lane == 0) {
          ChanRec& r = chR->rec[ch_tail % kChanRecs];
          r.t = now;
          r.ts = now - measured;  // pass start == when this EndForward was scheduled
          r.ef_idx = pidx;
          r.h_idx = hidx;
          r.h_ext = hext;
          r.nk = ndw;
          r.k0 = ktail - ndw;
        }
        chan_fence<CL>();  // every lane's key / record writes precede the publish
        __syncwarp();
        if (lane == 0) chR->tail = ch_tail + 1;
        chan_fence<CL>();  // the record precedes any later progress word
        ch_tail += 1;
        ndw = 0;
      }
      start_p = p;
      if (sbs) ef_p = p;
    } else if (kind == kEvWD) {
      // ---- on_watchdog (simulation.cpp:374-380) via watchdog_expired
      const int p = o_i;
      if (lane == p) {
        wd_t = kInf64;
        pflags |= F_WDFIRED;
        pflags &= ~F_HASDL;
        p_td = 0;
      }
      odirty = true;
      CNT(wdf, 1);
      dispatch = sbs;
    } else if (kind == kEvDS) {
      // ---- on_decode_step (simulation.cpp:497-512)
      const int j = o_i;
      if (lane == j) ds_t = kInf64;
      odirty = true;
      maybe_die_d(j);
      if (d_flag(j, G_DEAD)) continue;
      PROF_BEGIN(3);
      finish_step(j);
      PROF_END(3);
      step_j = j;
    } else {
      // ---- on_topology (simulation.cpp:382-393)
      const int inst = pt.topo_inst[topo_idx];
      const bool h = pt.topo_healthy[topo_idx] != 0;
      topo_idx += 1;
      topo_t = (topo_idx < n_topo) ? pt.topo_time[topo_idx] : kInf64;
      if (inst < P) {
        if (lane == inst) pflags = h ? (pflags | F_HEALTHY) : (pflags & ~F_HEALTHY);
      } else {
        if (lane == inst - P) dflags = h ? (dflags | G_HEALTHY) : (dflags & ~G_HEALTHY);
        ul_dirty = true;
        S_valid = false;
        S_gathered = false;
      }
      int32_t na_ = __popc(__ballot_sync(kFull, lane < P && (pflags & F_HEALTHY)));
      if (sbs) {
        n_active = na_;
        recompute_interval();
        if (g_log) log_rec(LOG_CONTROL, 4, now, i_opt, t_bar, n_active, 0);  // simulation.cpp:391
        dispatch = true;
      }
    }

    // ---- decode hand-off: hand_off_finished / on_decode_step tail
    if (ROLE == 0 && !PO && (kind == kEvEF || kind == kEvDS)) {
      PROF_BEGIN(4);
      drain_decode(step_j);
      PROF_END(4);
      if (error) break;
    }
    PROF_BEGIN(9);
    // ---- prefill passes and the SBS dispatch chain
    for (int stage = 0; stage < 2; ++stage) {
      PROF_BEGIN(8);
      if (start_p >= 0) try_start_pass(start_p);
      PROF_END(8);
      if (stage == 1) {
        if (start_p >= 0 && np > 0) arm_tick(now + i_opt);  // simulation.cpp:341
        break;
      }
      if (ef_p >= 0) {
        if (n_drops > 0 && drop_matches(ef_p)) {
          CNT(drop, 1);  // scheduler view stays stale (simulation.cpp:359-362)
        } else {
          // on_end_forward_sample (interval_control.cpp:26-36)
          if (measured <= 0) {
            CNT(rej, 1);
          } else {
            if (win_n < w_size) {
              s_wr[(win_head + win_n) % w_size] = measured;
              win_n += 1;
              win_sum += measured;
            } else {
              win_sum += measured - s_wr[win_head];
              s_wr[win_head] = measured;
              win_head = (win_head + 1) % w_size;
            }
            __syncwarp();
            recompute_interval();
          }
          if (lane == ef_p) {
            p_td = p_td > 0 ? p_td - 1 : 0;
            pflags |= F_EFSEEN;
            pflags &= ~F_HASDL;  // disarm_watchdog
            wd_t = kInf64;
          }
          if (g_log) log_rec(LOG_CONTROL, 4, now, i_opt, t_bar, n_active, 0);  // simulation.cpp:370
          dispatch = true;
        }
      }
      start_p = -1;
      if (!dispatch) break;
      start_p = try_dispatch();
      if (error) break;
      if (start_p < 0) break;
      maybe_die_p(start_p);
    }
    PROF_END(9);
  }
  if (ROLE == 1) {
    chan_fence<CL>();
    __syncwarp();
    if (lane == 0) chR->p_done = kInf64;
#ifdef SBS_PROF
    prof_acc[21] += clock64() - prof_t0;
#endif
  }
  }  // ROLE != 2

  asm volatile("cp.async.wait_all;" ::: "memory");  // staged buckets: nothing in flight
  // ---- results (completion-derived fields: finalize_kernel)
  if (lane == 0) {
    cn->fb += n_fb; cn->mask += n_mask; cn->dsel += n_dsel;
    if constexpr (ROLE == 2) { cn->events += n_events; cn->steps += n_steps; cn->outtok += n_outtok; }
  }
  __syncwarp();
#ifdef SBS_PROF
  if (ROLE == 0) prof_acc[21] += clock64() - prof_t0;
#endif
  __syncwarp();
  if (ROLE != 0) {
    if (lane == 0) {
      cn->err = error;
      if constexpr (CL == 2) {  // two kernels: finalize_kernel combines the counters from HBM
        const long long* src = (const long long*)cn;
        long long* dst = (long long*)(pt.gcnt + (ROLE == 1 ? 0 : 32));
        for (int i = 0; i < (int)(sizeof(Counters) / 8); ++i) dst[i] = src[i];
        if (ROLE == 1) pt.gcnt[63] = 3;  // marker: finalize_kernel combines this replica
      }
#ifdef SBS_PROF
      for (int i = 0; i < 24; ++i) atomicAdd((unsigned long long*)&res.prof[i], (unsigned long long)prof_acc[i]);
#endif
    }
    __syncwarp();
    return;
  }
  if (lane == 0) {
    res.throttled = cn->throttled;
    res.passes = cn->passes;
    res.steps = cn->steps;
    res.out_tokens = cn->outtok;
    res.wd_fires = cn->wdf;
    res.dropped = cn->drop;
    res.rejected = cn->rej;
    res.deferrals = cn->def;
    res.flow = cn->flow;
    res.mask = cn->mask;
    res.fallback = cn->fb;
    res.alloc_calls = cn->alloc;
    res.dec_selects = cn->dsel;
    res.events = cn->events;
    res.util_sum = cn->util;
    res.kv_mean_sum = cn->kv_mean;
    res.kv_sigma_sum = cn->kv_sig;
    res.kv_n = cn->kv_n;
    res.log_n = log_n;
    res.error = error;
#ifdef SBS_PROF
    for (int i = 0; i < 24; ++i) res.prof[i] = prof_acc[i];
#endif
  }
#undef CNT
  (void)kErrInvariant;
}

// Persistent kernel: each warp grabs replicas until none are left (the host
// orders replicas by estimated cost, longest first).  One instantiation per
// (prefill DP units per lane, run records) so each keeps its own registers and
// instruction footprint.
template <int KD, bool LOG, bool CA = false, bool PO = false>
__global__ void __launch_bounds__(128) des_kernel(const DevPoint* __restrict__ pts, int n_pts,
                                                  int* __restrict__ next_point,
                                                  DevResult* __restrict__ res, int smem_per_warp) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* my = smem + (threadIdx.x >> 5) * smem_per_warp;
  for (;;) {
    int pi = 0;
    if (lane_id() == 0) pi = atomicAdd(next_point, 1);
    pi = bcast(pi, 0);
    if (pi >= n_pts) return;
    run_replica<KD, LOG, 0, false, CA, false, PO, PO>(pts[pi], res[pi], my, my);
    __syncwarp();
  }
}

// Channel reset before a replica (one warp).
__device__ void chan_init(Chan* ch, int lane) {
  if (lane == 0) {
    ch->p_done = 0;
    ch->tail = 0; ch->head = 0; ch->ktail = 0; ch->khead = 0; ch->abort = 0;
  }
  __syncwarp();
}

// Two-warp replicas: the prefill warp folds both warps' counters into the
// replica's DevResult (a: prefill warp, b: decode warp).
__device__ void combine_pair(const DevPoint& pt, DevResult& res, const Counters* a,
                             const Counters* b) {
  const int lane = lane_id();
  (void)pt;
  if (lane == 0) {
    DevResult& r = res;
    r.throttled = a->throttled;
    r.passes = a->passes;
    r.steps = b->steps;
    r.out_tokens = b->outtok;
    r.wd_fires = a->wdf;
    r.dropped = a->drop;
    r.rejected = a->rej;
    r.deferrals = a->def;
    r.flow = a->flow;
    r.mask = b->mask;
    r.fallback = b->fb;
    r.alloc_calls = a->alloc;
    r.dec_selects = b->dsel;
    r.events = a->events + b->events;
    r.util_sum = a->util;
    r.kv_mean_sum = b->kv_mean;
    r.kv_sigma_sum = b->kv_sig;
    r.kv_n = b->kv_n;
    r.log_n = 0;
    const long long e = b->err ? b->err : a->err;
    r.error = (int)e;
  }
}

// Two-warp replicas in one CTA (SBS_SPLIT=1): the prefill and decode warps of
// a pair share a shared-memory slice and the hand-off channel, synchronised
// by a named barrier per pair.
__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
}

// Warps [0, R) are the prefill warps and [R, 2R) the decode warps of R pairs,
// so with R = 4 every scheduler partition (warp % 4) holds one decode warp.
template <int KD, bool CA = false>
__global__ void __launch_bounds__(256) des_split_kernel(const DevPoint* __restrict__ pts, int n_pts,
                                                        int* __restrict__ next_point,
                                                        DevResult* __restrict__ res,
                                                        int smem_per_pair) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_pi[4];
  const int npairs = blockDim.x >> 6;
  const int warp = threadIdx.x >> 5, pair = warp % npairs, role = warp / npairs, lane = lane_id();
  unsigned char* my = smem + pair * smem_per_pair;
  for (;;) {
    if (role == 0 && lane == 0) s_pi[pair] = atomicAdd(next_point, 1);
    pair_sync(pair);
    const int pi = s_pi[pair];
    if (pi >= n_pts) return;
    const DevPoint& pt = pts[pi];
    Chan* ch = (Chan*)(my + pt.sm_chan);
    if (role == 0) chan_init(ch, lane);
    if (role == 0 && lane == 0)
      for (int i = 0; i < 24; ++i) res[pi].prof[i] = 0;
    pair_sync(pair);
    if (role == 0) run_replica<KD, false, 1, false, CA>(pt, res[pi], my, my);
    else run_replica<KD, false, 2, false>(pt, res[pi], my, my);
    pair_sync(pair);
    if (role == 0)
      combine_pair(pt, res[pi], (const Counters*)(my + pt.sm_cnt), (const Counters*)(my + pt.sm_cnt2));
    pair_sync(pair);
  }
}

// Cluster pairs: the two warps of a replica sit in the two CTAs of a 2-CTA
// cluster, CTA rank 0 holding W prefill warps and rank 1 their W decode
// warps, one CTA per SM (the launch reserves enough shared memory), so each
// SM runs one side's code only: the two sides' instruction working sets no
// longer share an SM's instruction cache.  Every channel word is polled in
// the reader's own shared memory and written remotely (DSMEM) by the other
// side.  Replicas go round-robin over clusters, rounds separated by a
// cluster barrier.
template <int KD, bool CA = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256)
    des_cluster_kernel(const DevPoint* __restrict__ pts, int n_pts, int* __restrict__ unused,
                       DevResult* __restrict__ res, int smem_per_rep) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = lane_id();
  unsigned crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  unsigned char* my = smem + warp * smem_per_rep;
  // generic address of the same slice in the peer CTA
  unsigned char* peer;
  {
    const unsigned long long mine = (unsigned long long)my;
    unsigned long long rp;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(rp) : "l"(mine), "r"(crank ^ 1u));
    peer = (unsigned char*)rp;
  }
  for (int base = 0; base < n_pts; base += ncl * nw) {
    const int pi = base + warp * ncl + cid;
    const bool active = pi < n_pts;
    if (active) chan_init((Chan*)(my + pts[pi].sm_chan), lane);
    if (active && crank == 0 && lane == 0)
      for (int i = 0; i < 24; ++i) res[pi].prof[i] = 0;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (active) {
      if (crank == 0) run_replica<KD, false, 1, true, CA>(pts[pi], res[pi], my, peer);
      else run_replica<KD, false, 2, true>(pts[pi], res[pi], my, peer);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (active && crank == 0)
      combine_pair(pts[pi], res[pi], (const Counters*)(my + pts[pi].sm_cnt),
                   (const Counters*)(peer + pts[pi].sm_cnt2));
    // the decode CTA's counters stay untouched until they are folded in
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

// Two-kernel pairs (pair mode 3): the prefill warps of all replicas in one
// kernel on a minority of SMs (the prefill role idles about half the time, so
// many share an SM), their decode warps in another on the rest (fewer decode
// warps per SM: each runs faster), the hand-off channel in HBM (GPU-scope
// acquire/release).  Slot s of both kernels runs replicas s, s + S, s + 2S...
// in the same order, so a warp only ever waits on the partner working on the
// same replica.  The pair must be co-resident: every CTA checks in on entry
// and waits (bounded) until all CTAs of both kernels have; otherwise both
// kernels give up (sync[1] = 1) and the host reruns the replicas as clusters.
__device__ bool pair3_checkin(int* sync, int total) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    atomicAdd(sync, 1);
    const long long t0 = clock64();
    int v = 0;
    for (;;) {
      v = *(volatile int*)sync;
      if (v >= total || *(volatile int*)(sync + 1) != 0) break;
      if (clock64() - t0 > 4000000000ll) { atomicExch(sync + 1, 1); break; }  // ~2 s
      __nanosleep(1000);
    }
    ok = v >= total && *(volatile int*)(sync + 1) == 0;
  }
  __syncthreads();
  return ok != 0;
}

template <int KD, bool CA = false, bool SP = false>
__global__ void __launch_bounds__(384) des_pf_kernel(const DevPoint* __restrict__ pts, int n_pts, int S,
                                                     int* __restrict__ sync, int total,
                                                     DevResult* __restrict__ res, int slice) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (!pair3_checkin(sync, total)) return;
  const int warp = threadIdx.x >> 5;
  const int slot = warp * gridDim.x + blockIdx.x;
  if (slot >= S) return;
  unsigned char* my = smem + (size_t)warp * slice;
  for (int pi = slot; pi < n_pts; pi += S) run_replica<KD, false, 1, 2, CA, false, SP>(pts[pi], res[pi], my, my);
}

template <int KD, bool SD = false>
__global__ void __launch_bounds__(256) des_dc_kernel(const DevPoint* __restrict__ pts, int n_pts, int S,
                                                     int* __restrict__ sync, int total,
                                                     DevResult* __restrict__ res, int slice) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (!pair3_checkin(sync, total)) return;
  const int warp = threadIdx.x >> 5;
  const int slot = warp * gridDim.x + blockIdx.x;
  if (slot >= S) return;
  unsigned char* my = smem + (size_t)warp * slice;
  for (int pi = slot; pi < n_pts; pi += S) {
    // the decode fields sit at [sm_dec_begin, sm_dec_end) of the replica layout
    unsigned char* base = my - pts[pi].sm_dec_begin;
    run_replica<KD, false, 2, 2, false, SD>(pts[pi], res[pi], base, base);
  }
}

// ---------------------------------------------------------------------------
// Finalize (MetricsCollector::finalize, metrics.cpp:103-190), one CTA per
// replica, after the event loops.  Deferred accounting: the loops only stamp
// per-request times; this kernel derives every completion-based field from
// the per-request arrays in one coalesced pass over the trace —
//   completed / completed-in-window counts (metrics.cpp:117-121, 174-176),
//   window TTFT / scheduler / device sums over completed requests with
//   arrival >= warmup (metrics.cpp:122-136; exact int64 ns),
//   TPOT = (completion - first_token) / (output_len - 1) per completed decode
//   request (one IEEE division; not in the reference), its FP64 sum in a fixed
//   thread/tree order and its log2 histogram,
// and compacts the window TTFTs into the replica's buffer; then the exact
// p50/p95 order statistics (percentile, decode_alloc.cpp:13-23, as used by
// metrics.cpp:151-152) by 8-bit MSB radix select, four ranks at once, plus
// the log2 TTFT histogram.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) reset_kernel(const DevPoint* __restrict__ pts, int n_pts,
                                                    DevResult* __restrict__ res) {
  // completion stamps of every replica := -1 (unset), one launch for all
  for (int pi = blockIdx.y; pi < n_pts; pi += gridDim.y) {
    const DevPoint& pt = pts[pi];
    const int64_t n = pt.N;
    int4* c = (int4*)pt.o_comp;  // 256-byte aligned carve
    const int64_t n16 = n >> 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
      c[i] = make_int4(-1, -1, -1, -1);
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) pt.o_comp[n - 1] = -1;
    if (pt.gcnt != nullptr && blockIdx.x == 0 && threadIdx.x == 0) pt.gcnt[63] = 0;
#ifdef SBS_PROF
    if (blockIdx.x == 0 && threadIdx.x < 24) res[pi].prof[threadIdx.x] = 0;  // (pair mode 3 accumulates)
#endif
    if (pt.gchan != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {  // pair mode 3's channel
      Chan* ch = pt.gchan;
      ch->p_done = 0;
      ch->tail = 0; ch->head = 0; ch->ktail = 0; ch->khead = 0; ch->abort = 0;
    }
  }
}

__global__ void __launch_bounds__(256) finalize_kernel(const DevPoint* __restrict__ pts,
                                                       DevResult* __restrict__ res) {
  const DevPoint& pt = pts[blockIdx.x];
  DevResult& r = res[blockIdx.x];
  __shared__ unsigned int hist[4][256];
  __shared__ unsigned long long hbin[kHistBins];
  __shared__ unsigned long long tbin[kHistBins];
  __shared__ uint64_t prefix[4];
  __shared__ int64_t want[4];
  __shared__ long long red[8][7];
  __shared__ double redf[8];
  __shared__ unsigned long long n_win;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < kHistBins) { hbin[tid] = 0; tbin[tid] = 0; }
  if (tid == 0) n_win = 0;
  // two-kernel pairs: fold the two warps' counters into the replica's result
  if (pt.gcnt != nullptr && pt.split && *(const volatile int*)&pt.gcnt[63] == 3 && tid < 32)
    combine_pair(pt, r, (const Counters*)pt.gcnt, (const Counters*)(pt.gcnt + 32));
  __syncthreads();

  // ---- pass 1: completion-derived sums (deferred accounting)
  {
    const int64_t N = pt.n_dev ? *pt.n_dev : pt.N;
    const int64_t warmup = pt.warmup;
    const int64_t* __restrict__ comp = pt.o_comp;
    long long done = 0, cw = 0, wr = 0, s_ttft = 0, s_sched = 0, s_dev = 0, tpn = 0;
    double tps = 0.0;
    for (int64_t b0 = 0; b0 < N; b0 += blockDim.x) {  // warp-uniform trip count (ballot below)
      const int64_t i = b0 + tid;
      const int64_t c = i < N ? comp[i] : -1;
      const bool has = c >= 0;
      int64_t ttft = 0;
      bool win = false;
      if (has) {
        done += 1;
        cw += c >= warmup;
        const int64_t arr = __ldg(pt.arr + i), ft = pt.o_ftok[i];
        const int32_t out = __ldg(pt.output + i);
        if (arr >= warmup) {
          const int64_t disp = pt.o_dispatch[i], ps = pt.o_pstart[i];
          win = true;
          ttft = ft - arr;
          wr += 1;
          s_ttft += ttft;
          s_sched += disp - arr;
          s_dev += ps - disp;
        }
        if (out > 1) {
          const double per = __ddiv_rn((double)(c - ft), (double)(out - 1));
          tps = __dadd_rn(tps, per);
          tpn += 1;
          atomicAdd(&tbin[hist_bin((int64_t)per)], 1ull);
        }
      }
      // compact the window TTFTs (their order is irrelevant to the select)
      const unsigned m = __ballot_sync(kFull, win);
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(&n_win, (unsigned long long)__popc(m));
      base = __shfl_sync(kFull, base, m ? __ffs(m) - 1 : 0);
      if (win) pt.ttft[base + __popc(m & ((1u << lane) - 1u))] = ttft;
    }
    long long v[7] = {done, cw, wr, s_ttft, s_sched, s_dev, tpn};
#pragma unroll
    for (int k = 0; k < 7; ++k) v[k] = warp_sum_i64(v[k]);
    tps = warp_sum_f64(tps);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 7; ++k) red[wid][k] = v[k];
      redf[wid] = tps;
    }
    __syncthreads();
    if (tid == 0) {
      long long t[7] = {0, 0, 0, 0, 0, 0, 0};
      double f = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        for (int k = 0; k < 7; ++k) t[k] += red[w][k];
        f = __dadd_rn(f, redf[w]);
      }
      r.completed = t[0]; r.cw = t[1]; r.wr = t[2]; r.n_ttft = t[2];
      r.ttft_sum = t[3]; r.sched_sum = t[4]; r.dev_sum = t[5];
      r.tpot_n = t[6]; r.tpot_sum = f / 1e9;
    }
    if (tid < kHistBins) pt.tpot_hist[tid] = (int64_t)tbin[tid];
  }
  __syncthreads();
  const int64_t n = (int64_t)n_win;
  if (tid < 4) {
    prefix[tid] = 0;
    int64_t k = 0;
    if (n > 0) {
      double p = (tid < 2) ? 50.0 : 95.0;
      double rank = __ddiv_rn(__dmul_rn((double)n - 1.0, p), 100.0);
      k = (tid & 1) ? (int64_t)ceil(rank) : (int64_t)floor(rank);
    }
    want[tid] = k;
  }
  __syncthreads();
  if (n == 0) {
    if (tid < 4) r.ttft_sel[tid] = 0;
    if (tid < kHistBins) r.ttft_hist[tid] = 0;
    return;
  }
  const uint64_t* v = (const uint64_t*)pt.ttft;
  for (int pass = 7; pass >= 0; --pass) {
    const int shift = pass * 8;
    for (int i = tid; i < 4 * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
    uint64_t pf[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) pf[t] = prefix[t];
    for (int64_t i = tid; i < n; i += blockDim.x) {
      uint64_t x = v[i];
      if (pass == 7) atomicAdd(&hbin[hist_bin((int64_t)x)], 1ull);
      uint64_t hi = (pass == 7) ? 0 : (x >> (shift + 8));
      unsigned dgt = (unsigned)(x >> shift) & 0xff;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (hi == pf[t]) atomicAdd(&hist[t][dgt], 1u);
    }
    __syncthreads();
    if (tid < 4) {
      int64_t k = want[tid];
      unsigned acc = 0;
      int dsel = 255;
      for (int d = 0; d < 256; ++d) {
        unsigned c = hist[tid][d];
        if (k < (int64_t)(acc + c)) { dsel = d; break; }
        acc += c;
      }
      want[tid] = k - acc;
      prefix[tid] = (prefix[tid] << 8) | (uint64_t)dsel;
    }
    __syncthreads();
  }
  if (tid < 4) r.ttft_sel[tid] = (int64_t)prefix[tid];
  if (tid < kHistBins) r.ttft_hist[tid] = (int64_t)hbin[tid];
}

}  // namespace sbs

// ---------------------------------------------------------------------------
// host-callable launchers (C++ linkage, used by sbs_host.cpp)
// ---------------------------------------------------------------------------
namespace sbs {
// variant: bit 0 = dp_degree > 32 (KD 4), bit 1 = run records, 4|5 = two-warp
// replicas (smem_per_warp is then the per-pair slice, warps_per_block even),
// 6..9 = 0..3 and 10|11 = 4|5 with the cache-aware dispatch compiled in
cudaError_t launch_des(int variant, const DevPoint* d_pts, int n_pts, int* d_counter,
                       DevResult* d_res, int smem_per_warp, int warps_per_block, int n_blocks,
                       int min_smem, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  // one-warp variants: a slice per warp; two-warp variants: a slice per pair
  const bool pairs = variant == 4 || variant == 5 || variant == 10 || variant == 11;
  size_t smem = (size_t)smem_per_warp * (pairs ? warps_per_block / 2 : warps_per_block);
  void (*k)(const DevPoint*, int, int*, DevResult*, int) =
      variant == 0 ? des_kernel<1, false> : variant == 1 ? des_kernel<4, false>
    : variant == 2 ? des_kernel<1, true> : variant == 3 ? des_kernel<4, true>
    : variant == 6 ? des_kernel<1, false, true> : variant == 7 ? des_kernel<4, false, true>
    : variant == 8 ? des_kernel<1, true, true> : variant == 9 ? des_kernel<4, true, true>
    : variant == 4 ? des_split_kernel<1> : variant == 5 ? des_split_kernel<4>
    : variant == 10 ? des_split_kernel<1, true> : variant == 11 ? des_split_kernel<4, true>
    : variant == 12 ? des_kernel<1, false, false, true> : des_kernel<4, false, false, true>;
  if (min_smem > 0 && smem < (size_t)min_smem) smem = (size_t)min_smem;  // CTAs per SM cap
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<n_blocks, 32 * warps_per_block, smem, st>>>(d_pts, n_pts, d_counter, d_res, smem_per_warp);
  return cudaGetLastError();
}

// Two-warp replicas on 2-CTA clusters (variant 4|5 points).  Geometry: one
// CTA per SM (reserved shared memory above half an SM's), as many clusters as
// are co-resident, W replicas per cluster with W = ceil(n / clusters) <= 8.
cudaError_t launch_des_cluster(int variant, const DevPoint* d_pts, int n_pts, DevResult* d_res,
                               int smem_per_rep, cudaStream_t st) {
  void (*k)(const DevPoint*, int, int*, DevResult*, int) =
      variant == 4 ? des_cluster_kernel<1> : variant == 5 ? des_cluster_kernel<4>
    : variant == 10 ? des_cluster_kernel<1, true> : des_cluster_kernel<4, true>;
  constexpr int kMaxSmem = 227 * 1024, kOnePerSm = 120 * 1024;
  int wmax = 8;
  while (wmax > 1 && wmax * smem_per_rep > kMaxSmem) --wmax;
  if (smem_per_rep > kMaxSmem) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  if (e != cudaSuccess) return e;
  // co-resident clusters, per (device, kernel, block size): the grid is one
  // CTA per SM of the current device (its SM count, not a constant)
  int dev = 0;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  static int cache[16][4][9] = {};
  const int vi = variant == 4 ? 0 : variant == 5 ? 1 : variant == 10 ? 2 : 3;
  int& max_clusters = cache[dev][vi][wmax];
  if (max_clusters == 0) {
    int n_sm = 0;
    e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_sm & ~1), 1, 1);
    cfg.blockDim = dim3(32 * wmax, 1, 1);
    cfg.dynamicSmemBytes = kOnePerSm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    if (e != cudaSuccess) return e;
    max_clusters = n > 0 ? n : 1;
  }
  int w = (n_pts + max_clusters - 1) / max_clusters;
  w = w < 1 ? 1 : (w > wmax ? wmax : w);
  const int ncl = (n_pts + w - 1) / w < max_clusters ? (n_pts + w - 1) / w : max_clusters;
  size_t smem = (size_t)w * smem_per_rep;
  if (smem < (size_t)kOnePerSm) smem = kOnePerSm;
  k<<<2 * ncl, 32 * w, smem, st>>>(d_pts, n_pts, nullptr, d_res, smem_per_rep);
  return cudaGetLastError();
}

// Two-kernel pairs (variant 4|5|10|11 points, pair mode 3).  Geometry: the
// prefill kernel on n_psm SMs with wp warps each, the decode kernel on the
// other n_dsm with wd warps each, one CTA per SM (reserved shared memory
// above half an SM), S = min(n_psm * wp, n_dsm * wd) slots.  `sync` is two
// device ints (zeroed here).  Returns cudaErrorInvalidValue when the
// geometry does not fit (the caller then uses cluster pairs).
cudaError_t launch_des_pair3(int variant, const DevPoint* d_pts, int n_pts, DevResult* d_res, int slice_pf,
                             int slice_dc, int n_psm, int wp, int n_dsm, int wd, int* sync,
                             cudaStream_t st_pf, cudaStream_t st_dc, bool simple_decode, bool simple_prefill) {
  void (*kp)(const DevPoint*, int, int, int*, int, DevResult*, int) =
      variant == 4 ? (simple_prefill ? des_pf_kernel<1, false, true> : des_pf_kernel<1>)
    : variant == 5 ? (simple_prefill ? des_pf_kernel<4, false, true> : des_pf_kernel<4>)
    : variant == 10 ? des_pf_kernel<1, true> : des_pf_kernel<4, true>;
  void (*kd)(const DevPoint*, int, int, int*, int, DevResult*, int) =
      (variant == 4 || variant == 10) ? (simple_decode ? des_dc_kernel<1, true> : des_dc_kernel<1>)
                                      : (simple_decode ? des_dc_kernel<4, true> : des_dc_kernel<4>);
  constexpr int kMaxSmem = 227 * 1024, kOnePerSm = 120 * 1024;
  if (wp < 1 || wp > 12 || wd < 1 || wd > 8 || n_psm < 1 || n_dsm < 1) return cudaErrorInvalidValue;
  const size_t sp = std::max<size_t>((size_t)wp * slice_pf, kOnePerSm);
  const size_t sd = std::max<size_t>((size_t)wd * slice_dc, kOnePerSm);
  // (the kernels' own static shared memory - the check-in flag - leaves 1 KB)
  if (sp > (size_t)kMaxSmem - 1024 || sd > (size_t)kMaxSmem - 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sd);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(sync, 0, 2 * sizeof(int), st_pf);
  if (e != cudaSuccess) return e;
  cudaEvent_t ev;
  e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;
  cudaEventRecord(ev, st_pf);
  cudaStreamWaitEvent(st_dc, ev, 0);  // the decode kernel after the zeroed check-in counter
  cudaEventDestroy(ev);
  const int S = std::min(n_psm * wp, n_dsm * wd);
  // (SBS_PAIR3_NOT_CORESIDENT: test hook, the check-in can never complete)
  const int total = n_psm + n_dsm + (std::getenv("SBS_PAIR3_NOT_CORESIDENT") ? 1 : 0);
  kp<<<n_psm, 32 * wp, sp, st_pf>>>(d_pts, n_pts, S, sync, total, d_res, slice_pf);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  kd<<<n_dsm, 32 * wd, sd, st_dc>>>(d_pts, n_pts, S, sync, total, d_res, slice_dc);
  return cudaGetLastError();
}

// Trace upload in one launch: every (host source, device destination, bytes)
// segment is copied by the device straight from pinned host memory (mapped
// under unified addressing), one CTA per segment slice, 16-byte accesses when
// both ends are aligned.  Replaces one cudaMemcpyAsync per trace array.
struct CopySeg {
  const unsigned char* src;
  unsigned char* dst;
  int64_t bytes;
};
__global__ void __launch_bounds__(256) gather_kernel(const CopySeg* __restrict__ segs, int n_segs) {
  const int64_t chunk = 1 << 16;  // bytes per CTA
  int64_t b = blockIdx.x;
  for (int s = 0; s < n_segs; ++s) {
    const int64_t nb = (segs[s].bytes + chunk - 1) / chunk;
    if (b >= nb) { b -= nb; continue; }
    const unsigned char* src = segs[s].src + b * chunk;
    unsigned char* dst = segs[s].dst + b * chunk;
    const int64_t n = min(chunk, segs[s].bytes - b * chunk);
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
      const int64_t n16 = n >> 4;
      for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
        ((int4*)dst)[i] = __ldcs(((const int4*)src) + i);
      for (int64_t i = (n16 << 4) + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    } else {
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    }
    return;
  }
}
cudaError_t launch_gather(const CopySeg* d_segs, int n_segs, int64_t n_blocks, cudaStream_t st) {
  if (n_segs == 0 || n_blocks == 0) return cudaSuccess;
  gather_kernel<<<(unsigned)n_blocks, 256, 0, st>>>(d_segs, n_segs);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const DevPoint* d_pts, int n_pts, DevResult* d_res, cudaStream_t st) {
  if (n_pts == 0) return cudaSuccess;
  finalize_kernel<<<n_pts, 256, 0, st>>>(d_pts, d_res);
  return cudaGetLastError();
}
cudaError_t launch_reset(const DevPoint* d_pts, int n_pts, DevResult* d_res, cudaStream_t st) {
  if (n_pts == 0) return cudaSuccess;
  reset_kernel<<<dim3(16, n_pts < 65535 ? n_pts : 65535), 256, 0, st>>>(d_pts, n_pts, d_res);
  return cudaGetLastError();
}
}  // namespace sbs
