// xxh64.cuh — XXH64 of one chained KV block on the device (reading A1):
//   H_j = XXH64( le64(H_{j-1}) || le32(tok_j[0]) || ... || le32(tok_j[n-1]), seed 0 )
// The byte string is consumed as 64-bit little-endian lanes: lane 0 = H_{j-1},
// lane i>=1 = tok[2i-2] | tok[2i-1] << 32, plus a trailing 4-byte word when n is odd.
#pragma once
#include <cstdint>

namespace sae {
namespace xx {

constexpr uint64_t P1 = 0x9E3779B185EBCA87ull;
constexpr uint64_t P2 = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t P3 = 0x165667B19E3779F9ull;
constexpr uint64_t P4 = 0x85EBCA77C2B2AE63ull;
constexpr uint64_t P5 = 0x27D4EB2F165667C5ull;

__device__ __forceinline__ uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__device__ __forceinline__ uint64_t rnd(uint64_t acc, uint64_t v) { return rotl(acc + v * P2, 31) * P1; }
__device__ __forceinline__ uint64_t merge(uint64_t acc, uint64_t v) { return (acc ^ rnd(0, v)) * P1 + P4; }

// n in [1, 16]; tok is 4-byte aligned global memory.
__device__ __forceinline__ uint64_t block(uint64_t prev, const uint32_t* __restrict__ tok, int n) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = i < n ? __ldg(tok + i) : 0u;
  auto lane = [&](int i) -> uint64_t {  // i >= 1
    return (uint64_t)w[2 * i - 2] | ((uint64_t)w[2 * i - 1] << 32);
  };
  const int len = 8 + 4 * n;
  const int lanes = len >> 3;            // 1 + n/2
  int l = 0;
  uint64_t h;
  if (len >= 32) {
    uint64_t v1 = P1 + P2, v2 = P2, v3 = 0, v4 = 0 - P1;
    const int ns = len >> 5;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s < ns) {
        const int b = 4 * s;
        v1 = rnd(v1, b == 0 ? prev : lane(b));
        v2 = rnd(v2, lane(b + 1));
        v3 = rnd(v3, lane(b + 2));
        v4 = rnd(v4, lane(b + 3));
      }
    }
    l = 4 * ns;
    h = rotl(v1, 1) + rotl(v2, 7) + rotl(v3, 12) + rotl(v4, 18);
    h = merge(h, v1); h = merge(h, v2); h = merge(h, v3); h = merge(h, v4);
  } else {
    h = P5;
  }
  h += (uint64_t)len;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    if (i >= l && i < lanes) {
      h ^= rnd(0, i == 0 ? prev : lane(i));
      h = rotl(h, 27) * P1 + P4;
    }
  }
  if (n & 1) {
    uint32_t last = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) last = (k == n - 1) ? w[k] : last;
    h ^= (uint64_t)last * P1;
    h = rotl(h, 23) * P2 + P3;
  }
  h ^= h >> 33; h *= P2;
  h ^= h >> 29; h *= P3;
  h ^= h >> 32;
  return h;
}

}  // namespace xx
}  // namespace sae
