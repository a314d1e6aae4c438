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

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// In-register bitonic sort of one uint64 key per lane, ascending by lane.
__device__ __forceinline__ uint64_t warp_sort32(uint64_t x) {
  const int lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      uint64_t y = __shfl_xor_sync(kFull, x, j);
      bool up = (lane & k) == 0;
      bool lower = (lane & j) == 0;
      // lower lane keeps min when ascending block, max when descending
      bool take_min = (lower == up);
      uint64_t mn = x < y ? x : y, mx = x < y ? y : x;
      x = take_min ? mn : mx;
    }
  }
  return x;
}

// Warp bitonic sort of n keys (ascending) in a buffer of capacity >= pow2(n)
// (generic pointer: shared or global).  Pads with UINT64_MAX.
__device__ __forceinline__ void warp_sort_buf(uint64_t* buf, int n) {
  const int lane = lane_id();
  if (n <= 1) return;
  if (n <= 32) {
    uint64_t x = lane < n ? buf[lane] : UINT64_MAX;
    x = warp_sort32(x);
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
