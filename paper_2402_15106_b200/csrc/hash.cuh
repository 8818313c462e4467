// hash.cuh - device-side counter hash (R9/R10).
// splitmix64 output function: smx(x) = mix64(x + 0x9E3779B97F4A7C15),
// mix64(z) = z ^= z>>30, z *= 0xBF58476D1CE4E5B9; z ^= z>>27,
// z *= 0x94D049BB133111EB; z ^= z>>31  (all mod 2^64).
#pragma once
#include <stdint.h>

namespace dsmpnn {

__host__ __device__ __forceinline__ uint64_t smx(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// key_node(seed, g) = smx(smx(seed) ^ g); caller passes s0 = smx(seed).
__host__ __device__ __forceinline__ uint64_t key_node(uint64_t s0, uint64_t g) { return smx(s0 ^ g); }

// key_edge(seed, gi, gj) = smx(smx(smx(seed) ^ gi) ^ gj); caller passes si = smx(smx(seed) ^ gi).
__host__ __device__ __forceinline__ uint64_t key_edge(uint64_t si, uint64_t gj) { return smx(si ^ gj); }

}  // namespace dsmpnn
