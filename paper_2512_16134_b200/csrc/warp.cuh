// Warp-level building blocks for the sm_100a SBS kernels.
//
// The simulator runs one warp per replica: scalar control is executed
// warp-uniformly (every lane holds the same value), and the per-unit loops of
// the reference (DP intake, argmax/argmin, KV bands, sorts) are spread over the
// 32 lanes with shuffles, REDUX and ballots.  Nothing here touches tensor
// cores: this is integer / index work.
#pragma once
#include <cstdint>

namespace sbs {

constexpr unsigned kFull = 0xffffffffu;
constexpr int64_t kInf64 = INT64_MAX;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T bcast(T v, int src) {
  return __shfl_sync(kFull, v, src);
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(kFull, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// min of non-negative int64 values by two 32-bit REDUX (high word, then the
// low word among the lanes holding the minimal high word)
__device__ __forceinline__ int64_t warp_min_nonneg_i64(int64_t v) {
  const uint32_t hi = (uint32_t)((uint64_t)v >> 32), lo = (uint32_t)v;
  const uint32_t mh = __reduce_min_sync(kFull, hi);
  const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? lo : 0xffffffffu);
  return (int64_t)(((uint64_t)mh << 32) | ml);
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// In-register bitonic sort of one uint64 key per lane, ascending by lane.
// ROLLED: loops kept rolled where the caller is instruction-cache bound.
__device__ __forceinline__ uint64_t bitonic_step(uint64_t x, int lane, int k, int j) {
  const uint64_t y = __shfl_xor_sync(kFull, x, j);
  const bool up = (lane & k) == 0;
  const bool lower = (lane & j) == 0;
  // lower lane keeps min when ascending block, max when descending
  const bool take_min = (lower == up);
  const uint64_t mn = x < y ? x : y, mx = x < y ? y : x;
  return take_min ? mn : mx;
}
template <bool ROLLED = false>
__device__ __forceinline__ uint64_t warp_sort32(uint64_t x) {
  const int lane = lane_id();
  if constexpr (ROLLED) {
#pragma unroll 1
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll 1
      for (int j = k >> 1; j > 0; j >>= 1) x = bitonic_step(x, lane, k, j);
  } else {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) x = bitonic_step(x, lane, k, j);
  }
  return x;
}

// Warp bitonic sort of n keys (ascending) in a buffer of capacity >= pow2(n)
// (generic pointer: shared or global).  Pads with UINT64_MAX.
template <bool ROLLED = false>
__device__ __forceinline__ void warp_sort_buf(uint64_t* buf, int n) {
  const int lane = lane_id();
  if (n <= 1) return;
  if (n <= 32) {
    uint64_t x = lane < n ? buf[lane] : UINT64_MAX;
    x = warp_sort32<ROLLED>(x);
    if (lane < n) buf[lane] = x;
    __syncwarp();
    return;
  }
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + lane; i < m; i += 32) buf[i] = UINT64_MAX;
  __syncwarp();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < (m >> 1); i += 32) {
        // pair index i -> (a, b) with b = a ^ j, a has bit j clear
        int a = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        int b = a | j;
        bool up = (a & k) == 0;
        uint64_t xa = buf[a], xb = buf[b];
        if ((xa > xb) == up) {
          buf[a] = xb;
          buf[b] = xa;
        }
      }
      __syncwarp();
    }
  }
}

// lower_bound over a sorted buffer (all lanes may search different keys).
__device__ __forceinline__ int lower_bound_u64(const uint64_t* a, int n, uint64_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace sbs

namespace sbs {

// Stable LSD radix sort (8-bit digits) of n uint64 keys with at most `nbits`
// significant bits, by one warp, ascending.  a: keys (in/out), t: scratch of
// n keys, hist: 256 x u32 (all shared memory).  Per pass: shared-memory
// histogram, warp exclusive scan, then a stable scatter of 32-key chunks where
// __match_any_sync groups equal digits and popc(peers & lanemask_lt) ranks
// each key inside its group.
template <typename Key>
__device__ __forceinline__ void warp_radix_sort(Key* a, Key* t, uint32_t* hist, int n, int nbits) {
  const int lane = lane_id();
  const unsigned lt = lanemask_lt();
  const int passes = (nbits + 7) >> 3;
  Key* src = a;
  Key* dst = t;
  for (int p = 0; p < passes; ++p) {
    const int sh = 8 * p;
#pragma unroll 1
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
#pragma unroll 1
    for (int i = lane; i < n; i += 32) atomicAdd(&hist[(unsigned)(src[i] >> sh) & 255u], 1u);
    __syncwarp();
    uint32_t v[8];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { v[k] = hist[8 * lane + k]; s += v[k]; }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t run = incl - s;
#pragma unroll
    for (int k = 0; k < 8; ++k) { hist[8 * lane + k] = run; run += v[k]; }
    __syncwarp();
#pragma unroll 1
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool valid = i < n;
      const Key x = valid ? src[i] : 0;
      const unsigned dg = valid ? ((unsigned)(x >> sh) & 255u) : 256u + lane;
      const unsigned peers = __match_any_sync(kFull, dg);
      unsigned off = 0;
      if (valid) {
        off = hist[dg];
        dst[off + __popc(peers & lt)] = x;
      }
      __syncwarp();
      if (valid && (peers >> lane) == 1u) hist[dg] = off + __popc(peers);
      __syncwarp();
    }
    Key* tmp = src; src = dst; dst = tmp;
  }
  if (passes & 1) {
    for (int i = lane; i < n; i += 32) a[i] = t[i];
    __syncwarp();
  }
}

}  // namespace sbs

namespace sbs {

// Number of elements < x in a sorted array (a lower bound), by a warp: one
// 32-ary partition round per 32x narrowing, then a ballot over the last <= 32.
template <typename Key>
__device__ __forceinline__ int warp_lower_bound(const Key* a, int n, Key x) {
  const int lane = lane_id();
  int lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const bool lt = idx < hi && a[idx] < x;
    const int k = __popc(__ballot_sync(kFull, lt));  // pivots < x (ascending)
    if (k == 0) return lo;
    const int nlo = lo + (k - 1) * step + 1;
    const int nhi = lo + k * step;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  const int idx = lo + lane;
  return lo + __popc(__ballot_sync(kFull, idx < hi && a[idx] < x));
}

}  // namespace sbs
