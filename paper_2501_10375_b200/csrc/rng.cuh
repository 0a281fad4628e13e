// Counter-based random-init generator (device side).
//
// Bit-identical to oracle/rng.py: every weight is a pure function of
// (seed, tag, flat index), so the 90 GB Mixtral-8x7B-shaped expert set is
// generated in place in HBM (or in the pinned host pool) and the CPU oracle
// regenerates exactly the experts it checks.  The reference has no weights at
// all (pkg/README.md:16-18); this is builder defined.
#pragma once
#include <stdint.h>

namespace daop {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t tag) {
  return mix64((seed * kGolden) ^ mix64(tag + kGolden));
}

// uniform in [-1, 1): exact dyadic float32 (24 random bits)
__device__ __forceinline__ float uniform_pm1(uint64_t key, uint64_t index) {
  uint64_t b = mix64(key + (index + 1ull) * kGolden);
  float u = static_cast<float>(static_cast<uint32_t>(b >> 40));
  return __fsub_rn(__fmul_rn(u, 1.1920928955078125e-07f /* 2^-23 */), 1.0f);
}

constexpr uint64_t kKindExpert = 1, kKindGate = 2, kKindNorm = 3, kKindInput = 4;

__host__ __device__ __forceinline__ uint64_t make_tag(uint64_t kind, uint64_t layer, uint64_t expert,
                                                      uint64_t matrix) {
  return (kind << 56) | (layer << 32) | (expert << 16) | matrix;
}

}  // namespace daop
