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
// (callers that hold the lane index pass it: lane_id() is an S2R whose
// latency shows up when the compiler rematerialises it inside hot loops)
template <bool ROLLED = false>
__device__ __forceinline__ uint64_t warp_sort32(uint64_t x, int lane) {
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
template <bool ROLLED = false>
__device__ __forceinline__ uint64_t warp_sort32(uint64_t x) { return warp_sort32<ROLLED>(x, lane_id()); }

// Ascending sort of lanes 0..n-1 (1 < n <= 32) when lanes >= n hold
// UINT64_MAX: only the bitonic stages up to the next power of two >= n
// (partners never leave their block of that size; the padding stays on top).
__device__ __forceinline__ uint64_t warp_sort32_n(uint64_t x, int lane, int n) {
  const int m = 1 << (32 - __clz(n - 1));
#pragma unroll 1
  for (int k = 2; k <= m; k <<= 1)
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) x = bitonic_step(x, lane, k, j);
  return x;
}

// Warp bitonic sort of n keys (ascending) in a buffer of capacity >= pow2(n)
// (generic pointer: shared or global).  Pads with UINT64_MAX.
template <bool ROLLED = false>
__device__ __forceinline__ void warp_sort_buf(uint64_t* buf, int n, int lane) {
  if (n <= 1) return;
  if (n <= 32) {
    uint64_t x = lane < n ? buf[lane] : UINT64_MAX;
    x = warp_sort32<ROLLED>(x, lane);
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
template <bool ROLLED = false>
__device__ __forceinline__ void warp_sort_buf(uint64_t* buf, int n) { warp_sort_buf<ROLLED>(buf, n, lane_id()); }

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
__device__ __forceinline__ void warp_radix_sort(Key* a, Key* t, uint32_t* hist, int n, int nbits, int lane,
                                                unsigned lt) {
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

// Ascending sort of n <= 32*KP uint32 keys a[0..n) (shared memory) by one
// warp in registers: lane l holds positions KP*l .. KP*l+KP-1 (padding
// 0xffffffff) and a bitonic network runs over all 32*KP positions.  Phases up
// to KP stay inside a lane (register compare-exchanges); later phases
// exchange whole registers with the partner lane (one shuffle + one min/max
// per register), then finish inside the lane.  A descending block is merged
// as an ascending one on complemented keys (bitonic sequences stay bitonic),
// so every compare-exchange is a plain min/max pair.  Replaces two 8-bit
// radix passes (smem histogram + match_any scatter per 32 keys) for the
// sorted-K multiset of <= 512 decode units.
template <typename Key, int KP>
__device__ __forceinline__ void warp_bitonic_regs(Key (&x)[KP], int lane) {
  static_assert(KP >= 2 && KP <= 16 && (KP & (KP - 1)) == 0, "KP: power of two in [2, 16]");
  auto cas_up = [&](Key& lo, Key& hi) {
    const Key a0 = lo, b0 = hi;
    lo = a0 < b0 ? a0 : b0;
    hi = a0 < b0 ? b0 : a0;
  };
  // phases k < KP: directions follow the register index only
#pragma unroll
  for (int k = 2; k < KP; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < KP; ++i)
        if ((i & j) == 0) {
          if ((i & k) == 0) cas_up(x[i], x[i | j]);
          else cas_up(x[i | j], x[i]);
        }
  // phases k >= KP: direction per lane ((KP*lane) & k), first the cross-lane
  // stages (j >= KP), then the in-lane ones
#pragma unroll 1
  for (int k = KP; k <= 32 * KP; k <<= 1) {
    const Key flip = ((KP * lane) & k) ? (Key)~(Key)0 : (Key)0;
#pragma unroll
    for (int i = 0; i < KP; ++i) x[i] ^= flip;
#pragma unroll 1
    for (int j = k >> 1; j >= KP; j >>= 1) {
      const int m = j / KP;
      const bool lower = (lane & m) == 0;
#pragma unroll
      for (int i = 0; i < KP; ++i) {
        const Key y = __shfl_xor_sync(kFull, x[i], m);
        x[i] = lower ? (x[i] < y ? x[i] : y) : (x[i] < y ? y : x[i]);
      }
    }
#pragma unroll
    for (int j = KP >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < KP; ++i)
        if ((i & j) == 0) cas_up(x[i], x[i | j]);
#pragma unroll
    for (int i = 0; i < KP; ++i) x[i] ^= flip;
  }
}

// Register i of lane o holds position KP*o + i after warp_bitonic_regs:
// the key at position p (warp-uniform p), every lane gets it.
template <typename Key, int KP>
__device__ __forceinline__ Key warp_regs_at(const Key (&x)[KP], int p) {
  const int r = p % KP;
  Key v = x[0];
#pragma unroll
  for (int i = 1; i < KP; ++i) v = i == r ? x[i] : v;
  return __shfl_sync(kFull, v, p / KP);
}

template <int KP>
__device__ __forceinline__ void warp_sort_reg_u32(uint32_t* a, int n, int lane) {
  uint32_t x[KP];
#pragma unroll
  for (int i = 0; i < KP; ++i) {
    const int p = KP * lane + i;
    x[i] = p < n ? a[p] : 0xffffffffu;
  }
  warp_bitonic_regs<uint32_t, KP>(x, lane);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < KP; ++i) {
    const int p = KP * lane + i;
    if (p < n) a[p] = x[i];
  }
  __syncwarp();
}

}  // namespace sbs

namespace sbs {

// Number of elements < x in a sorted array (a lower bound), by a warp: one
// 32-ary partition round per 32x narrowing, then a ballot over the last <= 32.
template <typename Key>
__device__ __forceinline__ int warp_lower_bound(const Key* a, int n, Key x, int lane) {
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

// Two lower bounds over one sorted array (x0 < x1) with shared probe rounds:
// one 32-ary pivot round serves both keys, then lanes 0-15 finish x0 and lanes
// 16-31 finish x1 when each window holds <= 16 elements (n <= 512); larger
// arrays take two single searches.
template <typename Key>
__device__ __forceinline__ void warp_lower_bound2(const Key* a, int n, Key x0, Key x1, int lane, int& r0,
                                                  int& r1) {
  if (n > 512) {
    r0 = warp_lower_bound<Key>(a, n, x0, lane);
    r1 = warp_lower_bound<Key>(a, n, x1, lane);
    return;
  }
  int lo0 = 0, hi0 = n, lo1 = 0, hi1 = n;
  if (n > 16) {
    const int step = (n + 31) >> 5;  // <= 16
    const int idx = lane * step;
    const Key v = idx < n ? a[idx] : Key(0);
    const int k0 = __popc(__ballot_sync(kFull, idx < n && v < x0));
    const int k1 = __popc(__ballot_sync(kFull, idx < n && v < x1));
    // answer for x in [(k-1)*step + 1, min(k*step, n)], or 0 when k == 0
    lo0 = k0 == 0 ? 0 : (k0 - 1) * step + 1;
    hi0 = k0 == 0 ? 0 : min(k0 * step, n);
    lo1 = k1 == 0 ? 0 : (k1 - 1) * step + 1;
    hi1 = k1 == 0 ? 0 : min(k1 * step, n);
  }
  const bool second = lane >= 16;
  const int idx = (second ? lo1 : lo0) + (lane & 15);
  const int hi = second ? hi1 : hi0;
  const Key x = second ? x1 : x0;
  const unsigned m = __ballot_sync(kFull, idx < hi && a[idx] < x);
  r0 = lo0 + __popc(m & 0xffffu);
  r1 = lo1 + __popc(m >> 16);
}

}  // namespace sbs
