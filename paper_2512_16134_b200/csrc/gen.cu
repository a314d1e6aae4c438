// Device trace generation: generate_workload (workload.cpp:67-142) and
// workload_digest (:144-162) on the GPU, bit-identical to the host (glibc)
// run of the reference on the same (spec, seed).
//
// One warp per trace.  The reference draws everything from one
// mt19937_64 stream in a fixed order: first the arrival process (Poisson:
// one exponential per arrival plus the draw that crosses the horizon;
// uniform_jitter: one per slot), then per request in id order the prompt
// length (lognormal: 2 draws, uniform: 1, constant: 0), the output length,
// and the shared-prefix draws (1, plus 1 when the request gets a prefix).
// The warp produces the stream 312 words at a time (mt19937.cuh) into a
// 1024-word ring in shared memory and consumes it in chunks of 32 arrivals /
// requests, one per lane:
//  * Poisson arrival times are a sequential FP64 sum (t += e, left to right,
//    as the reference adds them); the 32 exponentials of a chunk are
//    computed lane-parallel, the sum is a 32-step shuffle chain.
//  * A request's draw offset is i * (draws per request) without shared
//    prefixes; with them lane 0 walks the chunk once (the prefix coin decides
//    whether a second draw follows).
//  * log/cos/exp are glibc's own algorithms (glibc_libm.cuh), sqrt and the
//    arithmetic are IEEE-rounded single ops: every value is the host's.
// Algorithmic bytes: 16 B written per request (+8 with shared prefixes).
#include <cuda_runtime.h>

#include <cstdint>

#include "glibc_libm.cuh"
#include "mt19937.cuh"
#include "sbs_b200.h"
#include "warp.cuh"

namespace sbs {

namespace {

constexpr int kRing = 1024;  // draws buffered per warp (a chunk needs <= 32 * 6)
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr int kGenWarps = 4;

struct GenSmem {
  uint64_t mt[312];
  uint64_t ring[kRing];
  int32_t offs[32];
  int32_t end, _pad;
};

// glibc llround on x86-64 (s_llround.c): half away from zero; out of range
// and NaN end in a (long long) conversion, i.e. INT64_MIN.
__device__ __forceinline__ int64_t llround_glibc(double v) {
  if (!(glibc::f_abs(v) < 9223372036854775808.0)) return INT64_MIN;
  return (int64_t)llround(v);
}

__device__ __forceinline__ int64_t seconds_to_ns(double s) {  // core.h:26-28
  return llround_glibc(__dmul_rn(s, 1e9));
}

struct Stream {
  GenSmem* w;
  int64_t produced = 0;  // draws written into the ring so far
  __device__ void ensure(int64_t end) {
    const int lane = lane_id();
    while (produced < end) {
      mt_twist(w->mt);
      for (int i = lane; i < 312; i += 32) w->ring[(produced + i) & (kRing - 1)] = mt_temper(w->mt[i]);
      __syncwarp();
      produced += 312;
    }
  }
  __device__ __forceinline__ double u(int64_t i) const { return u01_of(w->ring[i & (kRing - 1)]); }
};

__device__ __forceinline__ int draws_of(const sbs_length_spec& s) {
  return s.dist == SBS_LEN_LOGNORMAL ? 2 : s.dist == SBS_LEN_UNIFORM ? 1 : 0;
}

// standard_normal (workload.cpp:19-25): Box-Muller on two draws.
__device__ __forceinline__ double standard_normal(double a, double b) {
  const double r = __dsqrt_rn(__dmul_rn(-2.0, glibc::log(__dsub_rn(1.0, a))));
  return __dmul_rn(r, glibc::cos(__dmul_rn(kTwoPi, b)));
}

// sample_length (workload.cpp:52-65) reading its draws from the ring at `off`.
__device__ int64_t sample_length(const sbs_length_spec& s, const Stream& st, int64_t off) {
  switch (s.dist) {
    case SBS_LEN_CONSTANT:
      return s.value > 1 ? s.value : 1;
    case SBS_LEN_UNIFORM: {
      const int64_t lo = s.min > 1 ? s.min : 1;
      const int64_t hi = s.max > lo ? s.max : lo;
      const double span = (double)(hi - lo + 1);
      const int64_t o = (int64_t)__dmul_rn(st.u(off), span);
      return lo + (o < hi - lo ? o : hi - lo);
    }
    default: {  // lognormal, clamped: std::clamp = min(max(t, lo), hi) (libstdc++)
      const double z = standard_normal(st.u(off), st.u(off + 1));
      const double v = glibc::exp(__dadd_rn(s.mu, __dmul_rn(s.sigma, z)));
      const int64_t t = llround_glibc(v);
      const int64_t lo = s.min > 1 ? s.min : 1;
      const int64_t m = t > lo ? t : lo;
      return m < s.max ? m : s.max;
    }
  }
}

// prefix_token(pool, 0) (workload.cpp:30-37)
__device__ __forceinline__ int32_t prefix_token0(int pool_id) {
  uint64_t h = 1469598103934665603ull;
  h ^= (uint64_t)pool_id * 0x9e3779b97f4a7c15ull;
  h ^= 0x632be59bd9b4e019ull;
  h *= 1099511628211ull;
  return (int32_t)(h & 0x7fffffff);
}

__device__ __forceinline__ void mix(uint64_t& h, uint64_t v) {  // workload.cpp:146-152
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    h ^= (v >> (8 * b)) & 0xff;
    h *= 1099511628211ull;
  }
}

__global__ void __launch_bounds__(32 * kGenWarps)
gen_kernel(const sbs_gen_job* __restrict__ jobs, int n_jobs, const uint64_t* __restrict__ seeds,
           int want_digest) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int j = blockIdx.x * kGenWarps + warp;
  if (j >= n_jobs) return;
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  GenSmem* w = (GenSmem*)(smem + (size_t)warp * sizeof(GenSmem));
  const sbs_gen_job& job = jobs[j];
  const sbs_workload& sp = job.spec;
  const uint64_t seed = seeds ? seeds[j] : job.seed;
  const int64_t cap = job.cap;
  int64_t* __restrict__ o_arr = job.arrival_ns;
  int32_t* __restrict__ o_prompt = job.prompt_len;
  int32_t* __restrict__ o_output = job.output_len;
  int32_t* __restrict__ o_pool = job.prefix_pool_id;
  int32_t* __restrict__ o_psize = job.prefix_size;

  if (lane == 0) mt_seed_lane0(w->mt, seed);
  __syncwarp();
  Stream st{w, 0};
  int64_t c = 0;  // next unconsumed draw
  int error = 0;

  const int64_t horizon = seconds_to_ns(sp.duration_s);
  const double dur = sp.duration_s;
  const double rate = sp.rate_qps;

  // ---- arrivals (workload.cpp:89-118); initial_burst zeros first
  const int64_t burst = sp.initial_burst;
  int64_t n = 0;
  if (burst > cap) error = SBS_ERR_OVERFLOW;
  else {
    for (int64_t i = lane; i < burst; i += 32) o_arr[i] = 0;  // min(seconds_to_ns(0), horizon-1)
    n = burst;
  }
  auto put_arrival = [&](bool push, double t) -> int {
    const unsigned m = __ballot_sync(kFull, push);
    const int cnt = __popc(m);
    if (n + cnt > cap) { error = SBS_ERR_OVERFLOW; return cnt; }
    if (push) {
      const int64_t at = seconds_to_ns(t);
      o_arr[n + __popc(m & lt)] = at < horizon - 1 ? at : horizon - 1;
    }
    n += cnt;
    return cnt;
  };
  if (!error) {
    if (sp.process == SBS_ARRIVAL_POISSON) {
      double t = 0.0;  // t = e0, then t += e_k (0.0 + e0 == e0, incl. the -0.0 case's ns)
      for (;;) {
        st.ensure(c + 32);
        const double e = __ddiv_rn(glibc::f_neg(glibc::log(__dsub_rn(1.0, st.u(c + lane)))), rate);
        double mine = 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          t = __dadd_rn(t, __shfl_sync(kFull, e, k));
          if (k == lane) mine = t;
        }
        const bool in = mine < dur;  // t is non-decreasing: a prefix of the lanes
        const int cnt = put_arrival(in, mine);
        if (error) break;
        if (cnt < 32) { c += cnt + 1; break; }
        c += 32;
      }
    } else if (sp.process == SBS_ARRIVAL_UNIFORM) {
      const double slot = __ddiv_rn(1.0, rate);
      for (int64_t n0 = 0;; n0 += 32) {
        const double t = __dmul_rn((double)(n0 + lane), slot);
        const bool in = t < dur;
        const int cnt = put_arrival(in, t);
        if (error || cnt < 32) break;
      }
    } else {  // uniform_jitter: one draw per slot whose base is inside the horizon
      const double slot = __ddiv_rn(1.0, rate);
      for (int64_t n0 = 0;; n0 += 32) {
        st.ensure(c + 32);
        const double base = __dmul_rn((double)(n0 + lane), slot);
        const bool live = base < dur;
        const int nlive = __popc(__ballot_sync(kFull, live));
        const double t = __dadd_rn(base, __dmul_rn(st.u(c + lane), slot));
        put_arrival(live && t < dur, t);
        c += nlive;
        if (error || nlive < 32) break;
      }
    }
  }

  // ---- per-request lengths and prefixes (workload.cpp:120-140)
  const int dp = draws_of(sp.prompt);
  const bool out_const = sp.output.dist == SBS_LEN_CONSTANT;
  const int dfix = dp + (out_const ? 0 : draws_of(sp.output));
  const bool prefixes = sp.shared_prefix_fraction > 0;
  const double frac = sp.shared_prefix_fraction;
  uint64_t h = 14695981039346656037ull;
  int32_t mx_prompt = INT32_MIN, mx_output = INT32_MIN, mx_pool = -1, mx_psize = 0;
  for (int64_t i0 = 0; !error && i0 < n; i0 += 32) {
    const int m = (int)(n - i0 < 32 ? n - i0 : 32);
    st.ensure(c + 32 * (dfix + 2));
    int64_t rel, used;
    if (!prefixes) {
      rel = (int64_t)lane * dfix;
      used = (int64_t)m * dfix;
    } else {  // the prefix coin decides whether a pool draw follows
      if (lane == 0) {
        int32_t o = 0;
        for (int k = 0; k < m; ++k) {
          w->offs[k] = o;
          o += dfix + 1 + (st.u(c + o + dfix) < frac ? 1 : 0);
        }
        w->end = o;
      }
      __syncwarp();
      rel = lane < m ? w->offs[lane] : 0;
      used = w->end;
      __syncwarp();
    }
    const int64_t off = c + rel;
    c += used;
    int64_t p = 0, o = 0, plen = 0;
    int32_t pool_id = -1;
    bool bad = false;
    if (lane < m) {
      p = sample_length(sp.prompt, st, off);
      o = out_const ? (sp.output.value > 0 ? sp.output.value : 0)
                    : sample_length(sp.output, st, off + dp);
      if (prefixes && st.u(off + dfix) < frac) {
        const int pid = (int)__dmul_rn(st.u(off + dfix + 1), (double)sp.prefix_pool);
        pool_id = pid < sp.prefix_pool - 1 ? pid : sp.prefix_pool - 1;
        plen = sp.prefix_len < p ? sp.prefix_len : p;
        if (plen < 0) plen = 0;  // an empty prefix_tokens vector
      }
      bad = p > 0x3fffffff || o > 0x3fffffff;
      const int64_t i = i0 + lane;
      o_prompt[i] = (int32_t)p;
      o_output[i] = (int32_t)o;
      if (prefixes) {
        o_pool[i] = plen > 0 ? pool_id : -1;
        o_psize[i] = (int32_t)plen;
      }
      mx_prompt = max(mx_prompt, (int32_t)p);
      mx_output = max(mx_output, (int32_t)o);
      if (plen > 0) {
        mx_pool = max(mx_pool, pool_id);
        mx_psize = max(mx_psize, (int32_t)plen);
      }
    }
    if (__any_sync(kFull, bad)) error = SBS_ERR_CONFIG;
    if (want_digest) {  // workload_digest, sequential in id order (all lanes alike)
      const int64_t at = lane < m ? o_arr[i0 + lane] : 0;
      const uint64_t tok = plen == 0 ? 0 : (uint64_t)prefix_token0(pool_id) + 1;
      for (int k = 0; k < m; ++k) {
        mix(h, (uint64_t)__shfl_sync(kFull, at, k));
        mix(h, (uint64_t)__shfl_sync(kFull, p, k));
        mix(h, (uint64_t)__shfl_sync(kFull, o, k));
        mix(h, __shfl_sync(kFull, tok, k));
        mix(h, (uint64_t)__shfl_sync(kFull, plen, k));
      }
    }
  }
  mx_prompt = __reduce_max_sync(kFull, mx_prompt);
  mx_output = __reduce_max_sync(kFull, mx_output);
  mx_pool = __reduce_max_sync(kFull, mx_pool);
  mx_psize = __reduce_max_sync(kFull, mx_psize);
  if (lane == 0) {
    sbs_gen_stats* s = job.stats;
    s->n = error ? 0 : n;
    s->digest = want_digest ? h : 0;
    s->max_prompt = mx_prompt;
    s->max_output = mx_output;
    s->n_pools = mx_pool + 1;
    s->max_psize = mx_psize;
    s->error = error;
    s->draws = c;
  }
}

}  // namespace

cudaError_t launch_gen(const sbs_gen_job* d_jobs, int n_jobs, const uint64_t* d_seeds, int want_digest,
                       cudaStream_t st) {
  if (n_jobs <= 0) return cudaSuccess;
  const size_t smem = kGenWarps * sizeof(GenSmem);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int blocks = (n_jobs + kGenWarps - 1) / kGenWarps;
  gen_kernel<<<blocks, 32 * kGenWarps, smem, st>>>(d_jobs, n_jobs, d_seeds, want_digest);
  return cudaGetLastError();
}

}  // namespace sbs
