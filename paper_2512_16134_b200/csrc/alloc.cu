// Batched allocation kernels — the allocation step as its own sm_100a kernel.
//
//  pbaa_kernel   : allocate_batch (prefill_alloc.cpp:61-88) over a CSR batch
//                  of cluster-windows, one warp per window.  Windows of <= 32
//                  requests and <= 32 DP units (Basic mode) run on registers:
//                  lane i holds request i and DP unit i, one in-register
//                  bitonic sort orders (phase, prompt_len desc, id asc, input
//                  position) — pending before new, stable like std::stable_sort
//                  — and each placement is a REDUX argmax over the lanes'
//                  capacities (lowest index on ties), guarded by c_avail > 0.
//                  Larger or cache-aware windows sort in a shared-memory slice
//                  sized from the batch's bounds and take a warp max over
//                  capacity_after = c_avail - (prompt - hit).
//  iqr_kernel    : select_decode_unit (decode_alloc.cpp:38-81), one warp per
//                  call: for <= 512 units K is sorted in registers (16 per
//                  lane), else in shared memory; Q1/Q3 by the reference's
//                  FP64 interpolation, IQR mask, lex-min (B, K).
//  sched_kernel  : schedule_decode_batch (decode_alloc.cpp:83-106), one warp
//                  per candidate batch: stable order (sort_len desc, id asc),
//                  then one select_decode_unit per candidate on units kept in
//                  shared memory — the sorted K multiset is updated in place
//                  (one O(U/32) shift per placement), B/K written back.
//
// No tensor cores: this is integer sorting/selection, HBM/latency bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "warp.cuh"

namespace sbs {

constexpr int kAllocWarps = 4;
constexpr int kAllocMaxReq = 1024;  // per window (shared-memory sort)
constexpr int kAllocMaxDp = 1024;
constexpr int kIqrMaxUnits = 16384;     // = the simulator's decode-unit envelope
constexpr int kIqrDefaultUnits = 2048;  // bound assumed when the caller gives none
constexpr int kOneMax = 32;  // pbaa_one_kernel: requests / DP units by value

// Lexicographic ascending sort of (a, b) pairs in shared memory by a warp.
__device__ void warp_sort_pairs(uint64_t* a, uint64_t* b, int* idx, int n) {
  const int lane = lane_id();
  if (n <= 1) return;
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + lane; i < m; i += 32) { a[i] = UINT64_MAX; b[i] = UINT64_MAX; idx[i] = -1; }
  __syncwarp();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < (m >> 1); i += 32) {
        int x = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        int y = x | j;
        bool up = (x & k) == 0;
        uint64_t ax = a[x], ay = a[y], bx = b[x], by = b[y];
        bool gt = ax > ay || (ax == ay && bx > by);
        if (gt == up) {
          a[x] = ay; a[y] = ax; b[x] = by; b[y] = bx;
          int t = idx[x]; idx[x] = idx[y]; idx[y] = t;
        }
      }
      __syncwarp();
    }
  }
}

struct PbaaArgs {
  int32_t n_windows;
  int32_t max_req, max_dp;  // slice bounds of the shared-memory path (<= 1024 each)
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
  const int64_t* hit_off;  // cache-aware: Len_hit per (request, DP), NULL = Basic
  const int64_t* hit;
};

// Shared-memory slice of one warp on the general path: sort keys (2 x u64),
// positions (i32) for a power-of-two padded queue, then the DP capacities.
__host__ __device__ inline int pbaa_pow2(int n) {
  int m = 1;
  while (m < n) m <<= 1;
  return m;
}
__host__ __device__ inline size_t pbaa_slice_bytes(int max_req, int max_dp) {
  const size_t q = (size_t)pbaa_pow2(max_req < 1 ? 1 : max_req);
  return ((q * 20 + 15) & ~(size_t)15) + 8 * (size_t)(max_dp < 1 ? 1 : max_dp);
}

// One cluster-window by one warp; `my` is its shared-memory slice
// (pbaa_slice_bytes(A.max_req, A.max_dp)).
__device__ void pbaa_window(const PbaaArgs& A, int w, unsigned char* my) {
  const int lane = lane_id();
  const int QP = pbaa_pow2(A.max_req < 1 ? 1 : A.max_req);
  uint64_t* ka = (uint64_t*)my;
  uint64_t* kb = ka + QP;
  int* ki = (int*)(kb + QP);
  int64_t* cap = (int64_t*)(my + ((QP * 20 + 15) & ~15));

  const int64_t r0 = A.req_off[w], r1 = A.req_off[w + 1];
  const int n = (int)(r1 - r0);
  const int npend = A.n_pending[w];
  const int64_t c0 = A.dp_off[w];
  const int D = (int)(A.dp_off[w + 1] - c0);
  const int nlim = A.n_limit[w];
  if (n > A.max_req || D > A.max_dp || npend > n || D < 1) {
    if (lane == 0) atomicExch(A.error, 4);
    return;
  }
  for (int d = lane; d < D; d += 32) cap[d] = A.caps[c0 + d];
  __syncwarp();

  int rank = 0;
  bool stopped = false;
  bool any_thr = false;
  const int64_t* hrow = A.hit != nullptr ? A.hit + A.hit_off[w] : nullptr;
  for (int phase = 0; phase < 2; ++phase) {
    const int q0 = phase == 0 ? 0 : npend;
    const int qn = phase == 0 ? npend : n - npend;
    for (int i = lane; i < qn; i += 32) {
      int64_t r = r0 + q0 + i;
      ka[i] = (uint64_t)(INT64_MAX - A.prompt_len[r]);  // prompt desc
      kb[i] = (uint64_t)A.req_id[r];                    // id asc
      ki[i] = q0 + i;
    }
    __syncwarp();
    warp_sort_pairs(ka, kb, ki, qn);
    for (int i = 0; i < qn && !stopped; ++i) {
      int pos = ki[i];
      int64_t len = A.prompt_len[r0 + pos];
      // argmax capacity_after over D, lowest index on ties
      int64_t bv = INT64_MIN;
      int bd = 0x7fffffff;
      bool room = false;
      for (int d = lane; d < D; d += 32) {
        const int64_t c = cap[d];
        const int64_t after = c - (len - (hrow ? hrow[(int64_t)pos * D + d] : 0));
        if (after > bv) { bv = after; bd = d; }
        room |= c > 0;
      }
      // no unit with headroom: nothing in this phase (or the next) fits
      if (!__any_sync(kFull, room)) { stopped = true; break; }
      int64_t mv = warp_max_i64(bv);
      int best = (int)__reduce_min_sync(kFull, bv == mv ? (uint32_t)bd : 0x7fffffffu);
      if (cap[best] <= 0) continue;  // guard on the chosen unit: deferred
      __syncwarp();
      if (lane == 0) {
        cap[best] = mv;
        A.out_dp[r0 + pos] = best;
        A.out_rank[r0 + pos] = rank;
        A.wait_out[r0 + pos] = A.wait_in[r0 + pos];
        ki[i] = -1;  // placed
      }
      __syncwarp();
      rank += 1;
    }
    // deferred (every unplaced request): age; throttle beyond n_limit
    for (int j = lane; j < qn; j += 32) {
      int pos = ki[j];
      if (pos < 0) continue;
      int wv = A.wait_in[r0 + pos] + 1;
      bool thr = wv > nlim;
      A.out_dp[r0 + pos] = thr ? -2 : -1;
      A.out_rank[r0 + pos] = -1;
      A.wait_out[r0 + pos] = wv;
      any_thr |= thr;
    }
    __syncwarp();
  }
  any_thr = __any_sync(kFull, any_thr);
  for (int d = lane; d < D; d += 32) A.caps[c0 + d] = cap[d];
  if (lane == 0) A.flow[w] = any_thr ? 1 : 0;
}

// Register path: <= 32 requests, <= 32 DP units, Basic mode, 0 <= id < 2^27,
// 0 <= prompt_len < 2^31.  Lane i loads request i and DP unit i.  One u64 key
// per request — phase (pending 0 / new 1) | 0x7fffffff - prompt | id | input
// position — sorts both queues at once in the order greedy_dispatch visits
// them (prefill_alloc.cpp:28-35, std::stable_sort: the position breaks full
// ties).  In Basic mode argmax(c_avail - prompt) == argmax c_avail, and once
// the maximum is <= 0 nothing later fits (capacities only fall), so the loop
// stops there; every unplaced request is deferred or throttled
// (prefill_alloc.cpp:71-86).  Returns false (nothing written) when the window
// is outside this envelope.
__device__ bool pbaa_window_reg(const PbaaArgs& A, int w, int lane) {
  const int64_t r0 = A.req_off[w];
  const int n = (int)(A.req_off[w + 1] - r0);
  const int npend = A.n_pending[w];
  const int64_t c0 = A.dp_off[w];
  const int D = (int)(A.dp_off[w + 1] - c0);
  if (n > 32 || D > 32 || D < 1 || npend > n || A.hit != nullptr) return false;
  const bool has = lane < n;
  const int64_t id = has ? A.req_id[r0 + lane] : 0;
  const int64_t len = has ? A.prompt_len[r0 + lane] : 0;
  const int64_t cap0 = lane < D ? A.caps[c0 + lane] : 0;
  const bool ok = !has || (id >= 0 && id < (1ll << 27) && len >= 0 && len < (1ll << 31));
  if (!__all_sync(kFull, ok)) return false;
  uint64_t key = has ? ((uint64_t)(lane >= npend) << 63) | ((uint64_t)(0x7fffffffu - (uint32_t)len) << 32) |
                           ((uint64_t)id << 5) | (uint64_t)lane
                     : UINT64_MAX;
  key = warp_sort32<true>(key, lane);  // lane j: the j-th request visited
  const int src = (int)(key & 31u);
  const int64_t my_len = (int64_t)(0x7fffffffu - (uint32_t)((key >> 32) & 0x7fffffffu));
  // capacities: 32-bit REDUX when they fit (a placed unit keeps c - len >
  // -2^31 because c > 0 and len < 2^31, so they keep fitting), else 64-bit
  const bool small = __all_sync(kFull, lane >= D || (cap0 >= INT32_MIN && cap0 <= INT32_MAX));
  int64_t cap = lane < D ? cap0 : INT64_MIN;
  int my_dp = -1, my_rank = -1, rank = 0;
  for (int j = 0; j < n; ++j) {
    const int64_t L = __shfl_sync(kFull, my_len, j);
    int64_t mv;
    int best;
    if (small) {
      const uint32_t bv = (uint32_t)(int32_t)(lane < D ? cap : (int64_t)INT32_MIN) ^ 0x80000000u;
      const uint32_t m = __reduce_max_sync(kFull, bv);
      best = (int)__reduce_min_sync(kFull, bv == m ? (uint32_t)lane : 32u);
      mv = (int64_t)(int32_t)(m ^ 0x80000000u);
    } else {
      const uint64_t bv = (uint64_t)cap ^ 0x8000000000000000ull;
      const uint32_t h = __reduce_max_sync(kFull, (uint32_t)(bv >> 32));
      const uint32_t l = __reduce_max_sync(kFull, (uint32_t)(bv >> 32) == h ? (uint32_t)bv : 0u);
      const uint64_t m = ((uint64_t)h << 32) | l;
      best = (int)__reduce_min_sync(kFull, bv == m ? (uint32_t)lane : 32u);
      mv = (int64_t)(m ^ 0x8000000000000000ull);
    }
    if (mv <= 0) break;  // guard on the chosen unit fails here and for everything after
    if (lane == best) cap -= L;
    if (lane == j) { my_dp = best; my_rank = rank; }
    rank += 1;
  }
  bool thr = false;
  if (has) {
    const int32_t wv = A.wait_in[r0 + src];
    if (my_dp >= 0) {
      A.out_dp[r0 + src] = my_dp;
      A.out_rank[r0 + src] = my_rank;
      A.wait_out[r0 + src] = wv;
    } else {
      thr = wv + 1 > A.n_limit[w];
      A.out_dp[r0 + src] = thr ? -2 : -1;
      A.out_rank[r0 + src] = -1;
      A.wait_out[r0 + src] = wv + 1;
    }
  }
  if (lane < D) A.caps[c0 + lane] = cap;
  thr = __any_sync(kFull, thr);
  if (lane == 0) A.flow[w] = thr ? 1 : 0;
  return true;
}

__global__ void __launch_bounds__(256) pbaa_kernel(PbaaArgs A, int slice) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + warp;
  if (w >= A.n_windows) return;
  if (pbaa_window_reg(A, w, lane)) return;
  pbaa_window(A, w, smem + (size_t)warp * slice);
}

// A single small window passed by value in the kernel parameters (no input
// copy), results written straight into mapped pinned host memory (no output
// copy): one launch per call for the reference's one-window interface.
struct PbaaOne {
  int32_t n, n_pending, n_dp, n_limit;
  int64_t req_id[kOneMax];
  int64_t prompt_len[kOneMax];
  int32_t wait_in[kOneMax];
  int64_t caps[kOneMax];
  int32_t* out;  // mapped host: dp[n], rank[n], wait[n], flow, error; then caps (int64, 8-aligned)
};
__global__ void __launch_bounds__(32) pbaa_one_kernel(PbaaOne P) {
  __shared__ __align__(16) unsigned char slice[kOneMax * 20 + kOneMax * 8];
  __shared__ int64_t s_id[kOneMax], s_len[kOneMax], s_caps[kOneMax], s_off[4];
  __shared__ int32_t s_wait[kOneMax], s_dp[kOneMax], s_rank[kOneMax], s_wout[kOneMax], s_misc[4];
  __shared__ uint8_t s_flow;
  __shared__ int32_t s_err;
  const int lane = lane_id();
  for (int i = lane; i < P.n; i += 32) {
    s_id[i] = P.req_id[i];
    s_len[i] = P.prompt_len[i];
    s_wait[i] = P.wait_in[i];
  }
  for (int d = lane; d < P.n_dp; d += 32) s_caps[d] = P.caps[d];
  if (lane == 0) {
    s_off[0] = 0; s_off[1] = P.n; s_off[2] = 0; s_off[3] = P.n_dp;
    s_misc[0] = P.n_pending; s_misc[1] = P.n_limit;
    s_err = 0;
  }
  __syncwarp();
  PbaaArgs A{1, kOneMax, kOneMax, s_off, s_misc, s_off + 2, s_misc + 1, s_id, s_len, s_wait, s_caps,
             s_dp, s_rank, s_wout, &s_flow, &s_err, nullptr, nullptr};
  if (!pbaa_window_reg(A, 0, lane)) pbaa_window(A, 0, slice);
  __syncwarp();
  int32_t* o = P.out;
  for (int i = lane; i < P.n; i += 32) {
    o[i] = s_dp[i];
    o[P.n + i] = s_rank[i];
    o[2 * P.n + i] = s_wout[i];
  }
  int64_t* oc = (int64_t*)(o + ((3 * P.n + 2 + 1) & ~1));
  for (int d = lane; d < P.n_dp; d += 32) oc[d] = s_caps[d];
  if (lane == 0) {
    o[3 * P.n] = s_flow;
    o[3 * P.n + 1] = s_err;
  }
}

struct IqrArgs {
  int32_t n_calls;
  int32_t max_units;  // bound over the calls (<= 16384); <= 512: no shared memory
  const int64_t* unit_off;
  const int32_t* batch;
  const int64_t* kv;
  double k;
  int32_t* pos_out;
  uint8_t* fallback_out;
  double* threshold_out;
  int32_t* error;
};

__device__ __forceinline__ double pct_sorted_f(const int64_t* S, int n, double p) {
  double rank = __ddiv_rn(__dmul_rn((double)n - 1.0, p), 100.0);
  int lo = (int)floor(rank), hi = (int)ceil(rank);
  double vlo = (double)S[lo];
  if (lo == hi) return vlo;
  double frac = __dsub_rn(rank, (double)lo);
  return __dadd_rn(vlo, __dmul_rn(frac, __dsub_rn((double)S[hi], vlo)));
}

// Safe-set lex-min (B, K) with the first position on ties over the call's
// units (decode_alloc.cpp:46-68), given the threshold; writes the outputs.
__device__ __forceinline__ void iqr_finish(const IqrArgs& A, int c, int lane, int64_t u0, int n, double th,
                                           bool fallback) {
  int32_t bb = 0x7fffffff;
  int64_t bk = kInf64;
  int bp = 0x7fffffff;
  for (int i = lane; i < n; i += 32) {
    const int64_t kv = A.kv[u0 + i];
    if (!fallback && !((double)kv <= th)) continue;
    const int32_t b = A.batch[u0 + i];
    if (b < bb || (b == bb && kv < bk)) { bb = b; bk = kv; bp = i; }
  }
  const uint32_t ob = (uint32_t)bb ^ 0x80000000u;
  const uint32_t mb = __reduce_min_sync(kFull, ob);
  const int64_t mk = warp_min_i64(ob == mb ? bk : kInf64);
  const int pos = (int)__reduce_min_sync(kFull, (ob == mb && bk == mk) ? (uint32_t)bp : 0xffffffffu);
  if (lane == 0) {
    A.pos_out[c] = pos;
    if (A.fallback_out) A.fallback_out[c] = fallback ? 1 : 0;
    if (A.threshold_out) A.threshold_out[c] = th;
  }
}

// <= 512 units: K (offset by 2^63, so signed order == unsigned order) sorted
// in registers, 16 per lane; quartiles read by shuffles; no shared memory.
__device__ void iqr_call_reg(const IqrArgs& A, int c, int lane, int64_t u0, int n) {
  constexpr int KP = 16;
  uint64_t x[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) {
    const int p = KP * lane + i;
    x[i] = p < n ? (uint64_t)A.kv[u0 + p] ^ 0x8000000000000000ull : UINT64_MAX;
  }
  warp_bitonic_regs<uint64_t, KP>(x, lane);
  auto at = [&](int p) -> double {
    return (double)(int64_t)(warp_regs_at<uint64_t, KP>(x, p) ^ 0x8000000000000000ull);
  };
  auto pct = [&](double p) -> double {  // percentile (decode_alloc.cpp:13-23) on the sorted K
    const double rank = __ddiv_rn(__dmul_rn((double)n - 1.0, p), 100.0);
    const int lo = (int)floor(rank), hi = (int)ceil(rank);
    const double vlo = at(lo);
    if (lo == hi) return vlo;
    return __dadd_rn(vlo, __dmul_rn(__dsub_rn(rank, (double)lo), __dsub_rn(at(hi), vlo)));
  };
  const double q1 = pct(25.0), q3 = pct(75.0);
  const double th = __dadd_rn(q3, __dmul_rn(A.k, __dsub_rn(q3, q1)));
  const bool fallback = !(at(0) <= th);  // no K <= th
  iqr_finish(A, c, lane, u0, n, th, fallback);
}

__global__ void __launch_bounds__(256) iqr_kernel(IqrArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= A.n_calls) return;
  const int64_t u0 = A.unit_off[c];
  const int n = (int)(A.unit_off[c + 1] - u0);
  if (n < 1 || n > A.max_units) {
    if (lane == 0) atomicExch(A.error, n < 1 ? 3 : 4);
    return;
  }
  if (n <= 512) {
    iqr_call_reg(A, c, lane, u0, n);
    return;
  }
  int64_t* S = (int64_t*)(smem + (size_t)warp * pbaa_pow2(A.max_units) * 8);
  // K -> double is monotone, so sorting int64 K == sorting the doubles.
  // Keys are offset by 2^63 so negative K would also order correctly.
  for (int i = lane; i < n; i += 32) S[i] = A.kv[u0 + i];
  __syncwarp();
  uint64_t* SU = (uint64_t*)S;
  for (int i = lane; i < n; i += 32) SU[i] ^= 0x8000000000000000ull;
  __syncwarp();
  warp_sort_buf(SU, n);
  for (int i = lane; i < n; i += 32) SU[i] ^= 0x8000000000000000ull;
  __syncwarp();
  double q1 = pct_sorted_f(S, n, 25.0);
  double q3 = pct_sorted_f(S, n, 75.0);
  double th = __dadd_rn(q3, __dmul_rn(A.k, __dsub_rn(q3, q1)));
  int nsafe = 0;
  for (int i = lane; i < n; i += 32) nsafe += ((double)A.kv[u0 + i] <= th) ? 1 : 0;
  nsafe = __reduce_add_sync(kFull, nsafe);
  iqr_finish(A, c, lane, u0, n, th, nsafe == 0);
}

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

__device__ __forceinline__ uint64_t enc_k(int64_t v) { return (uint64_t)v ^ 0x8000000000000000ull; }
__device__ __forceinline__ int64_t dec_k(uint64_t v) { return (int64_t)(v ^ 0x8000000000000000ull); }

// std::stable_sort order of schedule_decode_batch (decode_alloc.cpp:88-93):
// sort_len desc, request_id asc, then input position.
__device__ __forceinline__ bool cand_before(const SchedArgs& A, int64_t c0, int x, int y) {
  if (x < 0) return false;
  if (y < 0) return true;
  const int64_t lx = A.sort_len[c0 + x], ly = A.sort_len[c0 + y];
  if (lx != ly) return lx > ly;
  const uint64_t ix = A.request_id[c0 + x], iy = A.request_id[c0 + y];
  if (ix != iy) return ix < iy;
  return x < y;
}

__device__ __forceinline__ int lb_enc(const uint64_t* S, int n, uint64_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ double pct_enc(const uint64_t* S, int lo, int hi, double frac) {
  const double vlo = (double)dec_k(S[lo]);
  if (lo == hi) return vlo;
  return __dadd_rn(vlo, __dmul_rn(frac, __dsub_rn((double)dec_k(S[hi]), vlo)));
}

__global__ void __launch_bounds__(32) sched_kernel(SchedArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = lane_id();
  const int bidx = blockIdx.x;
  const int64_t c0 = A.cand_off[bidx], u0 = A.unit_off[bidx];
  const int M = (int)(A.cand_off[bidx + 1] - c0), U = (int)(A.unit_off[bidx + 1] - u0);
  if (M == 0) return;
  if (U < 1 || M > A.max_cands || U > A.max_units) {
    if (lane == 0) atomicExch(A.error, U < 1 ? 3 : 4);  // "select_decode_unit: no units"
    return;
  }
  int Mp = 1;
  while (Mp < M) Mp <<= 1;
  int32_t* ord = (int32_t*)smem;
  int32_t* sB = ord + ((A.max_cands + 1) & ~1) * 2;  // ord has room for the padded pow2
  int64_t* sK = (int64_t*)(sB + ((A.max_units + 1) & ~1));
  uint64_t* S = (uint64_t*)(sK + A.max_units);
  uint64_t* T = S + A.max_units;
  for (int i = lane; i < Mp; i += 32) ord[i] = i < M ? i : -1;
  for (int u = lane; u < U; u += 32) {
    sB[u] = A.batch[u0 + u];
    sK[u] = A.kv[u0 + u];
    S[u] = enc_k(sK[u]);
  }
  __syncwarp();
  warp_sort_buf(S, U);
  // candidates: bitonic network over positions with the stable comparator
  for (int k2 = 2; k2 <= Mp; k2 <<= 1)
    for (int j = k2 >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < (Mp >> 1); i += 32) {
        const int x = ((i & ~(j - 1)) << 1) | (i & (j - 1)), y = x | j;
        const bool up = (x & k2) == 0;
        const int ox = ord[x], oy = ord[y];
        if (cand_before(A, c0, oy, ox) == up) { ord[x] = oy; ord[y] = ox; }
      }
      __syncwarp();
    }
  // percentile ranks (decode_alloc.cpp:17-20) depend on U only
  const double r25 = __ddiv_rn(__dmul_rn((double)U - 1.0, 25.0), 100.0);
  const double r75 = __ddiv_rn(__dmul_rn((double)U - 1.0, 75.0), 100.0);
  const int lo25 = (int)floor(r25), hi25 = (int)ceil(r25), lo75 = (int)floor(r75), hi75 = (int)ceil(r75);
  const double f25 = __dsub_rn(r25, (double)lo25), f75 = __dsub_rn(r75, (double)lo75);
  for (int j = 0; j < M; ++j) {
    const int ci = ord[j];
    const double q1 = pct_enc(S, lo25, hi25, f25), q3 = pct_enc(S, lo75, hi75, f75);
    const double th = __dadd_rn(q3, __dmul_rn(A.k, __dsub_rn(q3, q1)));
    int nsafe = 0;
    for (int u = lane; u < U; u += 32) nsafe += ((double)sK[u] <= th) ? 1 : 0;
    nsafe = __reduce_add_sync(kFull, nsafe);
    const bool fallback = nsafe == 0;
    int32_t bb = 0x7fffffff;
    int64_t bk = kInf64;
    int bp = 0x7fffffff;
    for (int u = lane; u < U; u += 32) {
      const int64_t kv = sK[u];
      if (!fallback && !((double)kv <= th)) continue;
      const int32_t b = sB[u];
      if (b < bb || (b == bb && kv < bk)) { bb = b; bk = kv; bp = u; }
    }
    const uint32_t ob = (uint32_t)bb ^ 0x80000000u;
    const uint32_t mb = __reduce_min_sync(kFull, ob);
    const int64_t mk = warp_min_i64(ob == mb ? bk : kInf64);
    const int pos = (int)__reduce_min_sync(kFull, (ob == mb && bk == mk) ? (uint32_t)bp : 0xffffffffu);
    const int64_t old_k = sK[pos];
    const int64_t new_k = old_k + A.kv_len[c0 + ci];
    if (lane == 0) {
      A.order_out[c0 + j] = ci;
      A.pos_out[c0 + j] = pos;
      if (A.fallback_out) A.fallback_out[c0 + j] = fallback ? 1 : 0;
      if (A.threshold_out) A.threshold_out[c0 + j] = th;
      sB[pos] += 1;
      sK[pos] = new_k;
    }
    // sorted multiset: replace one old_k by new_k (ping-pong shift)
    const uint64_t a = enc_k(old_k), b = enc_k(new_k);
    if (a != b) {
      const int i = lb_enc(S, U, a);
      if (b > a) {
        const int q = lb_enc(S, U, b) - 1;
        for (int p = lane; p < U; p += 32) T[p] = (p < i || p > q) ? S[p] : (p == q ? b : S[p + 1]);
      } else {
        const int q = lb_enc(S, U, b);
        for (int p = lane; p < U; p += 32) T[p] = (p < q || p > i) ? S[p] : (p == q ? b : S[p - 1]);
      }
      __syncwarp();
      uint64_t* t = S; S = T; T = t;
    } else {
      __syncwarp();
    }
  }
  for (int u = lane; u < U; u += 32) {
    A.batch[u0 + u] = sB[u];
    A.kv[u0 + u] = sK[u];
  }
}

size_t sched_smem_bytes(int max_cands, int max_units) {
  int mp = 1;
  while (mp < max_cands) mp <<= 1;
  const size_t ord = 4 * (size_t)std::max(mp, ((max_cands + 1) & ~1) * 2);
  return ord + 4 * (size_t)((max_units + 1) & ~1) + 8 * (size_t)max_units * 3;
}

cudaError_t launch_sched(const SchedArgs& a, cudaStream_t st) {
  if (a.n_batches <= 0) return cudaSuccess;
  const size_t smem = sched_smem_bytes(a.max_cands, a.max_units);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(sched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sched_kernel<<<a.n_batches, 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pbaa_one(const int64_t* rows, int n_pending, int n_new, const int64_t* caps,
                            int n_dp, int n_limit, int32_t* mapped_out, cudaStream_t st) {
  const int n = n_pending + n_new;
  if (n > kOneMax || n_dp > kOneMax || n_dp < 1) return cudaErrorInvalidValue;
  PbaaOne P;
  P.n = n; P.n_pending = n_pending; P.n_dp = n_dp; P.n_limit = n_limit;
  for (int i = 0; i < n; ++i) {
    P.req_id[i] = rows[3 * i];
    P.prompt_len[i] = rows[3 * i + 1];
    P.wait_in[i] = (int32_t)rows[3 * i + 2];
  }
  for (int d = 0; d < n_dp; ++d) P.caps[d] = caps[d];
  P.out = mapped_out;
  pbaa_one_kernel<<<1, 32, 0, st>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_pbaa(const PbaaArgs& a0, cudaStream_t st) {
  PbaaArgs a = a0;
  if (a.n_windows <= 0) return cudaSuccess;
  // bounds: 0 = unknown -> the envelope.  Every warp keeps a slice sized from
  // them: a window inside the register envelope by shape can still need the
  // shared-memory path (ids >= 2^27, prompt lengths >= 2^31).
  a.max_req = a.max_req > 0 ? std::min(a.max_req, kAllocMaxReq) : kAllocMaxReq;
  a.max_dp = a.max_dp > 0 ? std::min(a.max_dp, kAllocMaxDp) : kAllocMaxDp;
  const int slice = (int)pbaa_slice_bytes(a.max_req, a.max_dp);
  int warps = 8;  // per CTA
  while (warps > 1 && (size_t)warps * slice > 200 * 1024) warps >>= 1;
  const int smem = warps * slice;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pbaa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const int blocks = (a.n_windows + warps - 1) / warps;
  pbaa_kernel<<<blocks, 32 * warps, smem, st>>>(a, slice);
  return cudaGetLastError();
}

cudaError_t launch_iqr(const IqrArgs& a0, cudaStream_t st) {
  IqrArgs a = a0;
  if (a.n_calls <= 0) return cudaSuccess;
  a.max_units = a.max_units > 0 ? std::min(a.max_units, kIqrMaxUnits) : kIqrDefaultUnits;
  // <= 512 units: registers only, 8 warps per CTA; else one power-of-two
  // shared-memory slice per warp (the bitonic sort pads to it), <= 4 per CTA
  const size_t slice = a.max_units <= 512 ? 0 : (size_t)pbaa_pow2(a.max_units) * 8;
  int warps = slice == 0 ? 8 : kAllocWarps;
  while (warps > 1 && (size_t)warps * slice > 200 * 1024) warps >>= 1;
  const int smem = (int)(warps * slice);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(iqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  const int blocks = (a.n_calls + warps - 1) / warps;
  iqr_kernel<<<blocks, 32 * warps, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sbs
