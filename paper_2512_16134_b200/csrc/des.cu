// Persistent discrete-event simulator of the SBS cluster, one warp per replica.
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
//  * IQR quartiles read a sorted K multiset kept in shared memory, updated in
//    O(U/32) per admission and re-sorted after a decode step.
#include <cuda_runtime.h>

#include <cstdint>

#include "des_types.h"
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

__device__ __forceinline__ uint64_t decode_key(int64_t len, int64_t id) {
  // ascending == (prompt+output desc, id asc) (simulation.cpp:446-453)
  return ((uint64_t)(0xffffffffu - (uint32_t)len) << 32) | (uint64_t)(uint32_t)id;
}

__device__ __forceinline__ int hist_bin(int64_t v) {
  if (v <= 0) return 0;
  int b = 63 - __clzll(v);
  return b < kHistBins ? b : kHistBins - 1;
}

// percentile (decode_alloc.cpp:13-23) over a sorted int64 multiset.
__device__ __forceinline__ double pct_sorted(const int64_t* S, int n, double p) {
  double rank = __ddiv_rn(__dmul_rn((double)n - 1.0, p), 100.0);
  double fl = floor(rank), ce = ceil(rank);
  int lo = (int)fl, hi = (int)ce;
  double vlo = (double)S[lo];
  if (lo == hi) return vlo;
  double frac = __dsub_rn(rank, (double)lo);
  return __dadd_rn(vlo, __dmul_rn(frac, __dsub_rn((double)S[hi], vlo)));
}

// mt19937_64 (std::mersenne_twister_engine<uint64_t,64,312,156,31,...>).
__device__ void mt_twist(uint64_t* mt) {
  const int lane = lane_id();
  constexpr uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  constexpr uint64_t MA = 0xB5026F5AA96619E9ull;
  // phase 1: i in [0,156): reads old mt[i+1], old mt[i+156]
  for (int base = 0; base < 156; base += 32) {
    int i = base + lane;
    uint64_t nv = 0;
    if (i < 156) {
      uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
      uint64_t xa = (x >> 1) ^ ((x & 1) ? MA : 0);
      nv = mt[i + 156] ^ xa;
    }
    __syncwarp();
    if (i < 156) mt[i] = nv;
    __syncwarp();
  }
  // phase 2: i in [156,311): reads old mt[i+1], new mt[i-156]
  for (int base = 156; base < 311; base += 32) {
    int i = base + lane;
    uint64_t nv = 0;
    if (i < 311) {
      uint64_t x = (mt[i] & UM) | (mt[i + 1] & LM);
      uint64_t xa = (x >> 1) ^ ((x & 1) ? MA : 0);
      nv = mt[i - 156] ^ xa;
    }
    __syncwarp();
    if (i < 311) mt[i] = nv;
    __syncwarp();
  }
  if (lane == 0) {
    uint64_t x = (mt[311] & UM) | (mt[0] & LM);
    uint64_t xa = (x >> 1) ^ ((x & 1) ? MA : 0);
    mt[311] = mt[155] ^ xa;
  }
  __syncwarp();
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

}  // namespace

// ---------------------------------------------------------------------------
// One replica, executed by one warp.
// ---------------------------------------------------------------------------
__device__ void run_replica(const DevPoint& pt, DevResult& res, unsigned char* sm) {
  const int lane = lane_id();
  const unsigned lt_mask = lanemask_lt();

  // ---- constants
  const int P = pt.P, Dn = pt.Dn, D = pt.D, Dd = pt.Dd, U = pt.U;
  const int PD = P * D;
  const bool sbs = pt.policy == kSbs;
  const int64_t c_chunk = pt.c_chunk;
  const int64_t N = pt.N;
  const int64_t horizon = pt.horizon, warmup = pt.warmup;
  const int F = pt.F, Fm = pt.F - 1, R = pt.R, BC = pt.BC;

  // ---- shared-memory carve
  int64_t* s_out = (int64_t*)(sm + pt.sm_pf_out);
  int32_t* s_head = (int32_t*)(sm + pt.sm_pf_head);
  int32_t* s_tail = (int32_t*)(sm + pt.sm_pf_tail);
  int32_t* s_rel = (int32_t*)(sm + pt.sm_pf_rel);
  uint8_t* s_part = (uint8_t*)(sm + pt.sm_pf_part);
  int64_t* s_K = (int64_t*)(sm + pt.sm_dK);
  int64_t* s_S = (int64_t*)(sm + pt.sm_dS);
  int32_t* s_B = (int32_t*)(sm + pt.sm_dB);
  int32_t* s_nst = (int32_t*)(sm + pt.sm_dnst);
  int16_t* s_ul = (int16_t*)(sm + pt.sm_ulist);
  uint16_t* s_bcnt = (uint16_t*)(sm + pt.sm_bcnt);
  int64_t* s_wr = (int64_t*)(sm + pt.sm_wring);
  uint64_t* s_wk = (uint64_t*)(sm + pt.sm_wkeys);

  for (int g = lane; g < PD; g += 32) {
    s_out[g] = 0; s_head[g] = 0; s_tail[g] = 0; s_rel[g] = 0; s_part[g] = 0;
  }
  for (int u = lane; u < U; u += 32) { s_K[u] = 0; s_B[u] = 0; s_nst[u] = 0; }
  for (int b = lane; b < Dn * R; b += 32) s_bcnt[b] = 0;
  __syncwarp();

  // ---- lane-resident instance state (lane p <-> prefill instance p,
  //      lane j <-> decode instance j; core.h:164-193)
  int pflags = (lane < P) ? F_HEALTHY : 0;
  int64_t p_started = 0, p_deadline = 0;
  int32_t p_td = 0;
  int64_t ef_t = kInf64, wd_t = kInf64;
  uint32_t ef_s = 0xffffffffu, wd_s = 0xffffffffu;
  const int64_t p_death = (lane < P) ? pt.death[lane] : kInf64;
  int32_t imm_dp = 0;  // RotationCursor::next_dp (baselines.h:17-20)

  int dflags = (lane < Dn) ? G_HEALTHY : 0;
  int64_t d_step = 0;
  int64_t ds_t = kInf64;
  uint32_t ds_s = 0xffffffffu;
  const int64_t d_death = (lane < Dn) ? pt.death[P + lane] : kInf64;

  // ---- scheduler state (SchedulerState, core.h:197-218; new_cluster core.cpp:162-168)
  int64_t now = 0;
  const int64_t l_net = pt.l_net;
  int64_t t_bar = pt.t_default;
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
  bool S_valid = false, ul_dirty = true;
  int32_t nul = 0;
  int error = 0;

  // other-event cache (EF/WD/DS min)
  bool odirty = true;
  int64_t o_t = kInf64;
  uint32_t o_s = 0;
  int o_k = 0, o_i = 0;

  // ---- counters
  int64_t c_completed = 0, c_throttled = 0, c_cw = 0, c_wr = 0, c_passes = 0, c_steps = 0,
          c_outtok = 0, c_wdf = 0, c_drop = 0, c_rej = 0, c_def = 0, c_flow = 0, c_mask = 0,
          c_fb = 0, c_alloc = 0, c_dsel = 0, c_events = 0, n_ttft = 0, s_ttft = 0, s_sched = 0,
          s_dev = 0, kv_n = 0, tpot_n = 0;
  double util_sum = 0.0, kv_mean_sum = 0.0, kv_sig_sum = 0.0, tpot_sum = 0.0;

  // random decode policy: mt19937_64(seed ^ 0x9E3779B97F4A7C15) (simulation.cpp:42)
  if (pt.decode_policy == kRandom) {
    if (lane == 0) {
      uint64_t x = pt.rng_seed;
      pt.mt[0] = x;
      for (int i = 1; i < 312; ++i) {
        x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
        pt.mt[i] = x;
      }
    }
    __syncwarp();
  }

  // ---- arrival stream: lane l holds arrival[abase + l]
  int64_t abase = 0;
  int64_t abuf = (lane < N) ? __ldg(pt.arr + lane) : kInf64;
  int64_t anext = (32 + lane < N) ? __ldg(pt.arr + 32 + lane) : kInf64;

  // =======================================================================
  // helpers (all warp-uniform)
  // =======================================================================
  auto p_flag = [&](int p, int f) -> bool { return (bcast(pflags, p) & f) != 0; };
  auto d_flag = [&](int j, int f) -> bool { return (bcast(dflags, j) & f) != 0; };

  // maybe_die (simulation.cpp:122-126)
  auto maybe_die_p = [&](int p) {
    if (lane == p && !(pflags & F_DEAD) && now >= p_death) pflags |= F_DEAD;
  };
  auto maybe_die_d = [&](int j) {
    bool died = false;
    if (lane == j && !(dflags & G_DEAD) && now >= d_death) { dflags |= G_DEAD; died = true; }
    if (__any_sync(kFull, died)) { ul_dirty = true; S_valid = false; }
  };

  auto arm_tick = [&](int64_t at) {  // simulation.cpp:234-238
    tick_t = at > now ? at : now;
    tick_s = seq++;
  };

  auto n_active_count = [&]() -> int32_t {
    return __popc(__ballot_sync(kFull, lane < P && (pflags & F_HEALTHY)));
  };

  // recompute_interval (interval_control.cpp:18-24)
  auto recompute_interval = [&]() {
    t_bar = (win_n == 0) ? pt.t_default : win_sum / (int64_t)win_n;
    if (n_active <= 0) return;
    int64_t v = (t_bar + l_net) / (int64_t)n_active;
    i_opt = v > 1 ? v : 1;
  };

  auto recompute_other = [&]() {
    int64_t lt = ef_t;
    uint32_t ls = ef_s;
    int lk = kEvEF;
    if (wd_t < lt || (wd_t == lt && wd_s < ls)) { lt = wd_t; ls = wd_s; lk = kEvWD; }
    if (ds_t < lt || (ds_t == lt && ds_s < ls)) { lt = ds_t; ls = ds_s; lk = kEvDS; }
    int64_t m = warp_min_i64(lt);
    uint32_t cs = (lt == m) ? ls : 0xffffffffu;
    uint32_t ms = __reduce_min_sync(kFull, cs);
    unsigned who = __ballot_sync(kFull, lt == m && ls == ms);
    int src = __ffs(who) - 1;
    o_t = m; o_s = ms; o_k = bcast(lk, src); o_i = src;
    odirty = false;
  };

  // ---- completion accounting (metrics.cpp:117-153), called by the lanes
  //      holding a completed request; all lanes must call (ballots inside).
  int64_t l_cw = 0, l_wr = 0, l_ttft = 0, l_sched = 0, l_dev = 0, l_done = 0;
  auto complete_lanes = [&](bool has, int64_t id, int64_t ftok, bool decode) {
    int64_t ttft = 0;
    bool inwin = false;
    if (has) {
      l_done += 1;
      if (now >= warmup) l_cw += 1;
      int64_t arr = __ldg(pt.arr + id);
      if (pt.per_request) {
        pt.o_comp[id] = now;
        pt.o_status[id] = kStCompleted;
      }
      if (decode) {
        int32_t out = __ldg(pt.output + id);
        int64_t dt = now - ftok;
        tpot_sum = __dadd_rn(tpot_sum, __ddiv_rn(__ddiv_rn((double)dt, 1e9), (double)(out - 1)));
        tpot_n += 1;
        int64_t per = dt / (int64_t)(out - 1);
        atomicAdd((unsigned long long*)&pt.tpot_hist[hist_bin(per)], 1ull);
      }
      if (arr >= warmup) {
        inwin = true;
        int64_t disp = pt.o_dispatch[id];
        int64_t ps = pt.o_pstart[id];
        ttft = ftok - arr;
        l_wr += 1;
        l_ttft += ttft;
        l_sched += disp - arr;
        l_dev += ps - disp;
      }
    }
    unsigned m = __ballot_sync(kFull, inwin);
    if (inwin) pt.ttft[n_ttft + __popc(m & lt_mask)] = ttft;
    n_ttft += __popc(m);
  };
  auto flush_lanes = [&]() {
    c_completed += warp_sum_i64(l_done);
    c_cw += warp_sum_i64(l_cw);
    c_wr += warp_sum_i64(l_wr);
    s_ttft += warp_sum_i64(l_ttft);
    s_sched += warp_sum_i64(l_sched);
    s_dev += warp_sum_i64(l_dev);
    l_done = l_cw = l_wr = l_ttft = l_sched = l_dev = 0;
  };

  // ---- decode unit list over healthy, live decode instances, skipping
  //      capped units (simulation.cpp:432-442)
  auto rebuild_ulist = [&]() {
    int cnt = 0;
    for (int base = 0; base < U; base += 32) {
      int u = base + lane;
      bool in = false;
      if (u < U) {
        int j = u / Dd;
        int fl = __shfl_sync(kFull, dflags, j & 31);
        in = (fl & G_HEALTHY) && !(fl & G_DEAD) &&
             (pt.cap_batch <= 0 || s_B[u] < pt.cap_batch);
      } else {
        (void)__shfl_sync(kFull, dflags, 0);
      }
      unsigned m = __ballot_sync(kFull, in);
      if (in) s_ul[cnt + __popc(m & lt_mask)] = (int16_t)u;
      cnt += __popc(m);
    }
    __syncwarp();
    nul = cnt;
    ul_dirty = false;
    S_valid = false;
  };

  auto rebuild_S = [&]() {
    for (int i = lane; i < nul; i += 32) s_S[i] = s_K[s_ul[i]];
    __syncwarp();
    warp_sort_buf((uint64_t*)s_S, nul);  // K >= 0: unsigned order == signed order
    S_valid = true;
  };

  // try_begin_decode_step (engine_model.cpp:153-179)
  auto try_begin_step = [&](int j) {
    int fl = bcast(dflags, j);
    if ((fl & G_STEP) || (fl & G_DEAD)) return;
    const int u0 = j * Dd;
    bool any = false;
    for (int d = lane; d < Dd; d += 32) any |= s_B[u0 + d] > 0;
    if (!__any_sync(kFull, any)) return;
    double worst = 0.0;
    for (int d = lane; d < Dd; d += 32) {
      int32_t b = s_B[u0 + d];
      s_nst[u0 + d] = b;
      double t = __dadd_rn(__dmul_rn(pt.dc_req, (double)b), __dmul_rn(pt.dc_kv, (double)s_K[u0 + d]));
      worst = t > worst ? t : worst;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double w = __shfl_xor_sync(kFull, worst, o);
      worst = w > worst ? w : worst;
    }
    double dur = __dadd_rn(pt.dc_base, worst);
    int64_t t_end = now + llround_ns(dur);
    if (lane == j) {
      d_step += 1;
      dflags |= G_STEP;
      ds_t = t_end;
      ds_s = seq;
    }
    seq++;
    odirty = true;
    __syncwarp();
  };

  // IQR select over the unit list (decode_alloc.cpp:38-81); returns position.
  auto iqr_select = [&]() -> int {
    if (!S_valid) rebuild_S();
    double q1 = pct_sorted(s_S, nul, 25.0);
    double q3 = pct_sorted(s_S, nul, 75.0);
    double th = __dadd_rn(q3, __dmul_rn(pt.iqr_k, __dsub_rn(q3, q1)));
    // pass 1: safe count
    int nsafe = 0;
    for (int i = lane; i < nul; i += 32) nsafe += ((double)s_K[s_ul[i]] <= th) ? 1 : 0;
    nsafe = __reduce_add_sync(kFull, nsafe);
    bool fallback = nsafe == 0;
    if (fallback) c_fb += 1;
    else if (nsafe < nul) c_mask += 1;
    // lex-min (B, K), lowest position
    int32_t bb = 0x7fffffff;
    int64_t bk = kInf64;
    int bp = 0x7fffffff;
    for (int i = lane; i < nul; i += 32) {
      int u = s_ul[i];
      int64_t kv = s_K[u];
      if (!fallback && !((double)kv <= th)) continue;
      int32_t b = s_B[u];
      if (b < bb || (b == bb && kv < bk)) { bb = b; bk = kv; bp = i; }
    }
    uint32_t mb = __reduce_min_sync(kFull, (uint32_t)bb);
    int64_t ck = ((uint32_t)bb == mb) ? bk : kInf64;
    int64_t mk = warp_min_i64(ck);
    uint32_t cp = ((uint32_t)bb == mb && bk == mk) ? (uint32_t)bp : 0xffffffffu;
    return (int)__reduce_min_sync(kFull, cp);
  };

  // S multiset: replace one copy of `oldv` by `newv` (> oldv).
  auto S_update = [&](int64_t oldv, int64_t newv) {
    int c_old = 0, c_new = 0;
    for (int i = lane; i < nul; i += 32) {
      int64_t v = s_S[i];
      c_old += v < oldv;
      c_new += v < newv;
    }
    c_old = __reduce_add_sync(kFull, c_old);
    c_new = __reduce_add_sync(kFull, c_new);
    // shift S[c_old+1 .. c_new-1] left by one, then S[c_new-1] = newv
    for (int base = c_old; base < c_new - 1; base += 32) {
      int i = base + lane;
      int64_t v = (i < c_new - 1) ? s_S[i + 1] : 0;
      __syncwarp();
      if (i < c_new - 1) s_S[i] = v;
      __syncwarp();
    }
    if (lane == 0) s_S[c_new - 1] = newv;
    __syncwarp();
  };

  // drain_decode_admissions (simulation.cpp:413-484)
  auto drain_decode = [&]() {
    if (ndw == 0) return;
    for (int j = 0; j < Dn; ++j) maybe_die_d(j);
    warp_sort_buf(pt.dwait, ndw);
    uint32_t touched = 0;
    int32_t order_lane = -1;  // lane t holds the t-th touched instance
    int ntouched = 0;
    int wi = 0;
    const int64_t tps = pt.tps;
    while (wi < ndw) {
      if (ul_dirty) rebuild_ulist();
      if (nul == 0) break;
      uint64_t key = pt.dwait[wi];
      int64_t id = key_id(key);
      int32_t prompt = __ldg(pt.prompt + id);
      int32_t out = __ldg(pt.output + id);
      int pos;
      if (pt.decode_policy == kIqr) {
        pos = iqr_select();
      } else if (pt.decode_policy == kRandom) {
        if (mti >= 312) { mt_twist(pt.mt); mti = 0; }
        uint64_t y = mt_temper(pt.mt[mti]);
        mti += 1;
        double u01 = (double)(y >> 11) * 0x1.0p-53;
        int64_t q = (int64_t)__dmul_rn(u01, (double)nul);
        pos = (int)(q < nul - 1 ? q : nul - 1);
      } else {
        pos = (int)(dec_rr % nul);
        dec_rr += 1;
      }
      c_dsel += 1;
      int u = s_ul[pos];
      int j = u / Dd;
      int64_t oldK = s_K[u];
      int64_t newK = oldK + prompt;
      __syncwarp();
      if (lane == 0) { s_B[u] += 1; s_K[u] = newK; }
      if (pt.per_request && lane == 0) pt.o_status[id] = kStDecoding;
      __syncwarp();
      if (S_valid) S_update(oldK, newK);
      if (pt.cap_batch > 0 && s_B[u] >= pt.cap_batch) ul_dirty = true;
      // completion ring: finishes at step d_step + ceil(target/tps)
      int64_t target = (int64_t)out - 1;
      int64_t nsteps = (target + tps - 1) / tps;
      int64_t excess = nsteps * tps - target;
      int64_t c = bcast(d_step, j) + nsteps;
      int b = j * R + (int)(c & (R - 1));
      int cnt = s_bcnt[b];
      if (cnt >= BC) { error = kErrOverflow; return; }
      if (lane == 0) {
        pt.buckets[(int64_t)b * BC + cnt] =
            make_int4((int)id, u, (int)(prompt + target + excess), (int)excess);
        s_bcnt[b] = (uint16_t)(cnt + 1);
      }
      __syncwarp();
      if (!(touched & (1u << j))) {
        touched |= 1u << j;
        if (lane == ntouched) order_lane = j;
        ntouched += 1;
      }
      wi += 1;
    }
    // keep unadmitted waiters (still sorted)
    if (wi > 0 && wi < ndw) {
      for (int base = 0; base < ndw - wi; base += 32) {
        int i = base + lane;
        uint64_t v = (i < ndw - wi) ? pt.dwait[wi + i] : 0;
        __syncwarp();
        if (i < ndw - wi) pt.dwait[i] = v;
        __syncwarp();
      }
    }
    ndw -= wi;
    for (int t = 0; t < ntouched; ++t) try_begin_step(bcast(order_lane, t));
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
    double terms[kMaxPrefillDp / 32];
#pragma unroll
    for (int k = 0; k < kMaxPrefillDp / 32; ++k) {
      terms[k] = 0.0;
      int d = lane + 32 * k;
      if (d >= D) continue;
      int g = g0 + d;
      int32_t h = s_head[g], t = s_tail[g];
      bool part = s_part[g] != 0;
      int64_t outv = s_out[g];
      int64_t room = c_chunk;
      int2* fq = pt.fifo + (int64_t)g * F;
      while (room > 0 && h != t) {
        int2 e = fq[h & Fm];
        int64_t take = (int64_t)e.y < room ? (int64_t)e.y : room;
        room -= take;
        if (!part) {
          pt.o_pstart[e.x] = now;
          if (pt.per_request) pt.o_status[e.x] = kStPrefilling;
        }
        outv -= take;
        if (take == e.y) { h += 1; part = false; }
        else { fq[h & Fm].y = e.y - (int)take; part = true; }
      }
      s_head[g] = h;
      s_part[g] = part ? 1 : 0;
      s_out[g] = outv;
      int64_t assigned = c_chunk - room;
      amax = assigned > amax ? assigned : amax;
      int64_t mn = assigned < c_chunk ? assigned : c_chunk;
      terms[k] = __ddiv_rn((double)mn, (double)c_chunk);
    }
    amax = warp_max_i64(amax);
    double dur = __dadd_rn(pt.pf_base, __dmul_rn(pt.pf_tok, (double)amax));
    int64_t t_end = now + llround_ns(dur);
    if (now >= warmup) {
      // chunk_utilization (metrics.cpp:193-202): sequential sum in DP order
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < kMaxPrefillDp / 32; ++k) {
        if (32 * k >= D) break;
        for (int l = 0; l < 32 && 32 * k + l < D; ++l)
          sum = __dadd_rn(sum, __shfl_sync(kFull, terms[k], l));
      }
      util_sum = __dadd_rn(util_sum, __ddiv_rn(sum, (double)D));
      c_passes += 1;
    }
    if (lane == p) {
      pflags |= F_BUSY;
      p_started = now;
      ef_t = t_end;
      ef_s = seq;
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
        id = pt.fifo[(int64_t)(g0 + d) * F + (idx & Fm)].x;
        idx += 1;
        out = __ldg(pt.output + id);
        pt.o_ftok[id] = now;
      }
      bool done = has && out <= 1;   // decode_target() == 0
      bool wait = has && out > 1;
      complete_lanes(done, id, now, false);
      unsigned m = __ballot_sync(kFull, wait);
      if (wait) {
        int32_t prompt = __ldg(pt.prompt + id);
        pt.dwait[ndw + __popc(m & lt_mask)] = decode_key((int64_t)prompt + out, id);
      }
      ndw += __popc(m);
      if (ndw > pt.QD - 32) { error = kErrOverflow; }
    }
    flush_lanes();
    if (lane == p) pflags &= ~F_BUSY;
    __syncwarp();
  };

  // FIFO push (dispatch_prefill, engine_model.cpp:37-49), by the owning lane.
  auto fifo_push = [&](int g, int64_t id, int32_t tokens) -> bool {
    int32_t t = s_tail[g];
    if (t - s_rel[g] >= F) return false;
    pt.fifo[(int64_t)g * F + (t & Fm)] = make_int2((int)id, tokens);
    s_tail[g] = t + 1;
    s_out[g] += tokens;
    return true;
  };

  // ---------------- perform_dispatch (simulation.cpp:265-342) ----------------
  auto perform_dispatch = [&](int p) {
    const int g0 = p * D;
    int64_t cap[kMaxPrefillDp / 32];
#pragma unroll
    for (int k = 0; k < kMaxPrefillDp / 32; ++k) {
      int d = lane + 32 * k;
      cap[k] = d < D ? c_chunk - s_out[g0 + d] : INT64_MIN;
    }
    // q_new keys, sorted
    const int nn = (int)(next_id - new_begin);
    uint64_t* nk = (nn <= kSmemWinKeys) ? s_wk : pt.wscr;
    if (nn > pt.QW) { error = kErrOverflow; return; }
    for (int i = lane; i < nn; i += 32) {
      int64_t id = new_begin + i;
      nk[i] = pbaa_key(__ldg(pt.prompt + id), id);
    }
    __syncwarp();
    warp_sort_buf(nk, nn);
    uint64_t* pk = pt.pend_key[pcur];
    int32_t* pw = pt.pend_wait[pcur];
    bool ovf = false;

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
        for (int k = 0; k < kMaxPrefillDp / 32; ++k) {
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
          for (int k = 0; k < kMaxPrefillDp / 32; ++k)
            if (k == (best >> 5)) cap[k] -= len;
          if (!fifo_push(g0 + best, id, tokens)) ovf = true;
          pt.o_dispatch[id] = now;
          if (pt.per_request) pt.o_status[id] = kStDispatched;
        }
        i += 1;
      }
      return i;
    };
    bool stopped = false;
    int k1 = greedy(pk, np, stopped);
    int k2 = 0;
    if (!stopped) k2 = greedy(nk, nn, stopped);
    if (__any_sync(kFull, ovf)) { error = kErrOverflow; return; }
    c_alloc += 1;

    // aging (prefill_alloc.cpp:70-87): pending suffix then new suffix
    int na = 0, thr = 0;
    for (int base = k1; base < np; base += 32) {
      int i = base + lane;
      bool valid = i < np;
      uint64_t key = valid ? pk[i] : 0;
      int32_t w = valid ? pw[i] + 1 : 0;
      bool th = valid && w > pt.n_limit;
      bool keep = valid && !th;
      if (th && pt.per_request) pt.o_status[key_id(key)] = kStThrottled;
      unsigned m = __ballot_sync(kFull, keep);
      int pos = na + __popc(m & lt_mask);
      __syncwarp();
      if (keep) { pk[pos] = key; pw[pos] = w; }
      na += __popc(m);
      thr += __popc(__ballot_sync(kFull, th));
      __syncwarp();
    }
    int nb = nn - k2;
    int nbk = nb;
    if (nb > 0 && 1 > pt.n_limit) {
      for (int i = lane; i < nb; i += 32)
        if (pt.per_request) pt.o_status[key_id(nk[k2 + i])] = kStThrottled;
      thr += nb;
      nbk = 0;
    }
    c_def += na + nbk;
    c_throttled += thr;
    if (thr > 0) c_flow += 1;
    if (na + nbk > pt.QP) { error = kErrOverflow; return; }
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

    if (k1 + k2 == 0) {
      if (np > 0) arm_tick(now + i_opt);
      return;
    }
    has_ld = true;
    last_disp = now;
    last_inst = p;
    // arm_watchdog (interval_control.cpp:76-86)
    int64_t deadline = now + (int64_t)llround(__dmul_rn(pt.wd_mult, (double)t_bar));
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
    maybe_die_p(p);
    try_start_pass(p);
    if (np > 0) arm_tick(now + i_opt);
  };

  // ---------------- try_dispatch (simulation.cpp:245-263) ----------------
  auto try_dispatch = [&]() {
    if (np + (next_id - new_begin) == 0) return;
    if (n_active <= 0) return;
    if (has_ld && now < last_disp + i_opt) { arm_tick(last_disp + i_opt); return; }
    // select_ready_instance (interval_control.cpp:50-74)
    unsigned hm = __ballot_sync(kFull, lane < P && (pflags & F_HEALTHY));
    unsigned gt = last_inst < 0 ? 0xffffffffu : (unsigned)(~((2ull << last_inst) - 1ull));
    unsigned cand = hm & gt;
    int target = cand ? __ffs(cand) - 1 : (hm ? __ffs(hm) - 1 : -1);
    bool ready = false;
    if (target >= 0) {
      bool r = (p_td == 0 && !(pflags & F_BUSY)) || (pflags & F_EFSEEN) || (pflags & F_WDFIRED) ||
               ((pflags & F_HASDL) && now >= p_deadline);
      ready = bcast((int)r, target) != 0;
    } else {
      (void)bcast(0, 0);
    }
    if (!ready) { arm_tick(now + i_opt); return; }
    perform_dispatch(target);
  };

  // ---------------- baseline_dispatch (simulation.cpp:206-223) ----------------
  auto baseline_dispatch = [&](int64_t id) {
    int tp = -1, tdp = -1;
    if (pt.policy == kLeastOutstanding) {
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
      int64_t mv = warp_min_i64(bv);
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
    if (tp < 0) return;  // stays pending
    int32_t prompt = __ldg(pt.prompt + id);
    bool ok = true;
    if (lane == 0) {
      pt.o_dispatch[id] = now;
      if (pt.per_request) pt.o_status[id] = kStDispatched;
      ok = fifo_push(tp * D + tdp, id, prompt);
    }
    if (!bcast((int)ok, 0)) { error = kErrOverflow; return; }
    __syncwarp();
    maybe_die_p(tp);
    try_start_pass(tp);
  };

  // finish_decode_step (engine_model.cpp:181-217) + on_decode_step bookkeeping
  auto finish_step = [&](int j) {
    const int u0 = j * Dd;
    const int64_t tps = pt.tps;
    int64_t gen = 0;
    for (int d = lane; d < Dd; d += 32) {
      int64_t add = tps * (int64_t)s_nst[u0 + d];
      s_K[u0 + d] += add;
      gen += add;
    }
    __syncwarp();
    const int64_t s = bcast(d_step, j);
    const int b = j * R + (int)(s & (R - 1));
    const int n = s_bcnt[b];
    const int4* ent = pt.buckets + (int64_t)b * BC;
    for (int base = 0; base < n; base += 32) {
      int e = base + lane;
      bool has = e < n;
      int64_t id = 0, ft = 0;
      if (has) {
        int4 v = ent[e];
        id = v.x;
        atomicAdd((unsigned long long*)&s_K[v.y], (unsigned long long)(-(int64_t)v.z));
        atomicSub(&s_B[v.y], 1);
        gen -= v.w;
        ft = pt.o_ftok[id];
      }
      complete_lanes(has, id, ft, true);
    }
    __syncwarp();
    flush_lanes();
    if (lane == 0) s_bcnt[b] = 0;
    gen = warp_sum_i64(gen);
    if (lane == j) dflags &= ~G_STEP;
    S_valid = false;
    if (pt.cap_batch > 0 && n > 0) ul_dirty = true;
    __syncwarp();
    // record_step (metrics.cpp:99-101)
    if (now >= warmup) { c_steps += 1; c_outtok += gen; }
    // record_kv_snapshot (simulation.cpp:486-495) -> kv_band (metrics.cpp:50-72)
    if (now >= warmup) {
      int64_t sum = 0;
      int cnt = 0;
      for (int u = lane; u < U; u += 32) {
        int fl = __shfl_sync(kFull, dflags, (u / Dd) & 31);
        if ((fl & G_HEALTHY) && !(fl & G_DEAD)) { sum += s_K[u]; cnt += 1; }
      }
      // (lanes beyond U still take part in the shuffles above via loop bound)
      sum = warp_sum_i64(sum);
      cnt = __reduce_add_sync(kFull, cnt);
      if (cnt > 0) {
        double mean = __ddiv_rn((double)sum, (double)cnt);
        double var = 0.0;
        for (int u = lane; u < U; u += 32) {
          int fl = __shfl_sync(kFull, dflags, (u / Dd) & 31);
          if ((fl & G_HEALTHY) && !(fl & G_DEAD)) {
            double dv = __dsub_rn((double)s_K[u], mean);
            var = __dadd_rn(var, __dmul_rn(dv, dv));
          }
        }
        var = warp_sum_f64(var);
        double sigma = sqrt(__ddiv_rn(var, (double)cnt));
        kv_mean_sum = __dadd_rn(kv_mean_sum, mean);
        kv_sig_sum = __dadd_rn(kv_sig_sum, sigma);
        kv_n += 1;
      }
    }
  };

  // drop_matches (simulation.cpp:128-134)
  auto drop_matches = [&](int p) -> bool {
    for (int i = 0; i < pt.n_drops; ++i) {
      int inst = pt.drop_inst[i];
      if ((inst == -1 || inst == p) && now >= pt.drop_from[i] && now < pt.drop_until[i]) return true;
    }
    return false;
  };

  // =======================================================================
  // event loop (SimClock::run_until, simclock.cpp:32-45)
  // =======================================================================
  while (error == 0) {
    if (odirty) recompute_other();
    // live internal minimum: tick vs other
    int64_t it = o_t;
    uint32_t is = o_s;
    int ik = o_k;
    if (tick_t < it || (tick_t == it && tick_s < is)) { it = tick_t; is = tick_s; ik = 1; }
    const int64_t at = (next_id < N) ? bcast(abuf, (int)(next_id - abase)) : kInf64;
    const int64_t tt = (topo_idx < pt.n_topo) ? pt.topo_time[topo_idx] : kInf64;
    int kind;
    int64_t et;
    if (tt <= at && tt <= it) { kind = 4; et = tt; }      // topology (lowest seq)
    else if (at <= it) { kind = 0; et = at; }             // arrival
    else { kind = ik; et = it; }
    if (et == kInf64 || et > horizon) break;
    now = et;
    c_events += 1;

    if (kind == 0) {
      // ---- on_arrival (simulation.cpp:196-204)
      const int64_t id = next_id;
      next_id += 1;
      if (next_id - abase == 32) {
        abase += 32;
        abuf = anext;
        anext = (abase + 32 + lane < N) ? __ldg(pt.arr + abase + 32 + lane) : kInf64;
      }
      if (sbs) try_dispatch();
      else baseline_dispatch(id);
    } else if (kind == 1) {
      // ---- on_tick (simulation.cpp:240-243): only the live tick reaches here
      tick_t = kInf64;
      try_dispatch();
    } else if (kind == kEvEF) {
      // ---- on_end_forward (simulation.cpp:346-372)
      const int p = o_i;
      if (lane == p) ef_t = kInf64;
      odirty = true;
      maybe_die_p(p);
      if (p_flag(p, F_DEAD)) continue;
      const int64_t measured = now - bcast(p_started, p);
      finish_pass(p);
      drain_decode();
      if (error) break;
      try_start_pass(p);
      if (!sbs) continue;
      if (drop_matches(p)) { c_drop += 1; continue; }
      // on_end_forward_sample (interval_control.cpp:26-36)
      if (measured <= 0) {
        c_rej += 1;
      } else {
        if (win_n < pt.w_size) {
          s_wr[(win_head + win_n) % pt.w_size] = measured;
          win_n += 1;
          win_sum += measured;
        } else {
          win_sum += measured - s_wr[win_head];
          s_wr[win_head] = measured;
          win_head = (win_head + 1) % pt.w_size;
        }
        __syncwarp();
        recompute_interval();
      }
      if (lane == p) {
        p_td = p_td > 0 ? p_td - 1 : 0;
        pflags |= F_EFSEEN;
        pflags &= ~F_HASDL;  // disarm_watchdog
        wd_t = kInf64;
      }
      try_dispatch();
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
      c_wdf += 1;
      if (sbs) try_dispatch();
    } else if (kind == kEvDS) {
      // ---- on_decode_step (simulation.cpp:497-512)
      const int j = o_i;
      if (lane == j) ds_t = kInf64;
      odirty = true;
      maybe_die_d(j);
      if (d_flag(j, G_DEAD)) continue;
      finish_step(j);
      drain_decode();
      if (error) break;
      try_begin_step(j);
    } else {
      // ---- on_topology (simulation.cpp:382-393)
      const int inst = pt.topo_inst[topo_idx];
      const bool h = pt.topo_healthy[topo_idx] != 0;
      topo_idx += 1;
      if (inst < P) {
        if (lane == inst) pflags = h ? (pflags | F_HEALTHY) : (pflags & ~F_HEALTHY);
      } else {
        if (lane == inst - P) dflags = h ? (dflags | G_HEALTHY) : (dflags & ~G_HEALTHY);
        ul_dirty = true;
        S_valid = false;
      }
      int32_t na_ = n_active_count();
      if (!sbs) continue;
      n_active = na_;
      recompute_interval();
      try_dispatch();
    }
  }

  // ---- results
  if (lane == 0) {
    res.completed = c_completed;
    res.throttled = c_throttled;
    res.cw = c_cw;
    res.wr = c_wr;
    res.passes = c_passes;
    res.steps = c_steps;
    res.out_tokens = c_outtok;
    res.wd_fires = c_wdf;
    res.dropped = c_drop;
    res.rejected = c_rej;
    res.deferrals = c_def;
    res.flow = c_flow;
    res.mask = c_mask;
    res.fallback = c_fb;
    res.alloc_calls = c_alloc;
    res.dec_selects = c_dsel;
    res.events = c_events;
    res.n_ttft = n_ttft;
    res.ttft_sum = s_ttft;
    res.sched_sum = s_sched;
    res.dev_sum = s_dev;
    res.util_sum = util_sum;
    res.kv_mean_sum = kv_mean_sum;
    res.kv_sigma_sum = kv_sig_sum;
    res.tpot_sum = tpot_sum;
    res.kv_n = kv_n;
    res.tpot_n = tpot_n;
    res.error = error;
  }
  (void)kErrInvariant;
}

// Persistent kernel: each warp grabs replicas until none are left (the host
// orders replicas by estimated cost, longest first).
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
    run_replica(pts[pi], res[pi], my);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Finalize: exact TTFT order statistics (percentile, decode_alloc.cpp:13-23,
// as used by metrics.cpp:151-152) by 8-bit MSB radix select over the replica's
// window TTFT buffer, four ranks at once, plus the log2 TTFT histogram.
// One CTA per replica.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) finalize_kernel(const DevPoint* __restrict__ pts,
                                                       DevResult* __restrict__ res) {
  const DevPoint& pt = pts[blockIdx.x];
  DevResult& r = res[blockIdx.x];
  const int64_t n = r.n_ttft;
  __shared__ unsigned int hist[4][256];
  __shared__ unsigned long long hbin[kHistBins];
  __shared__ uint64_t prefix[4];
  __shared__ int64_t want[4];
  const int tid = threadIdx.x;
  if (tid < kHistBins) hbin[tid] = 0;
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
cudaError_t launch_des(const DevPoint* d_pts, int n_pts, int* d_counter, DevResult* d_res,
                       int smem_per_warp, int warps_per_block, int n_blocks, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  size_t smem = (size_t)smem_per_warp * warps_per_block;
  e = cudaFuncSetAttribute(des_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  des_kernel<<<n_blocks, 32 * warps_per_block, smem, st>>>(d_pts, n_pts, d_counter, d_res,
                                                           smem_per_warp);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  finalize_kernel<<<n_pts, 256, 0, st>>>(d_pts, d_res);
  return cudaGetLastError();
}
}  // namespace sbs
