// std::mt19937_64 (mersenne_twister_engine<uint64_t, 64, 312, 156, 31,
// 0xB5026F5AA96619E9, 29, 0x5555555555555555, 17, 0x71D67FFFEDA60000, 37,
// 0xFFF7EEE000000000, 43, 6364136223846793005>) on one warp.  The state lives
// in memory the warp shares (global or shared); the twist is split into its
// two data-parallel halves (outputs [0,156) read only old words, [156,311)
// read the new words of the first half), so 312 outputs cost ~10 warp steps.
// Used by the random decode policy (simulation.cpp:42, 463-466) and by the
// device trace generator (workload.cpp:67-142).
#pragma once
#include <cstdint>

namespace sbs {

// seed_seq-free constructor: mt[0] = seed, mt[i] = f * (mt[i-1] ^ mt[i-1] >> 62) + i.
__device__ __forceinline__ void mt_seed_lane0(uint64_t* mt, uint64_t seed) {
  uint64_t x = seed;
  mt[0] = x;
  for (int i = 1; i < 312; ++i) {
    x = 6364136223846793005ull * (x ^ (x >> 62)) + (uint64_t)i;
    mt[i] = x;
  }
}

__device__ __forceinline__ void mt_twist(uint64_t* mt) {
  const int lane = threadIdx.x & 31;
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

// u01 (workload.cpp:47-50): 53 random bits mapped to [0, 1), exact.
__device__ __forceinline__ double u01_of(uint64_t draw) {
  return __dmul_rn(__ull2double_rn(draw >> 11), 0x1.0p-53);
}

}  // namespace sbs
