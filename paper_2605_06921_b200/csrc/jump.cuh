// jump.cuh -- xoshiro256** jump-ahead for replaying reference draws in
// parallel.  The state update of rng.hpp:20-30 is linear over GF(2)^256, so
// advancing a stream by d draws is a 256x256 bit-matrix product.  The host
// builds M_e = T^(kSeg * 2^e) once; a device thread that owns draws
// [t*kSeg, (t+1)*kSeg) of a chain's section reaches its start with
// popcount(t) matrix-vector products, then draws sequentially.
#pragma once

#include <cstdint>

#include "rng.cuh"

namespace mqo_b200 {

constexpr int kSeg = 256;       // draws per thread segment
constexpr int kJumpLevels = 24;  // segments up to 2^24 * 256 draws per section

// Column-major 256x256 GF(2) matrix: col[j] = M * e_j as 4 words.
struct JumpMatrix {
  uint64_t col[256][4];
};

// Device table of M_e, e = 0..kJumpLevels-1 (built lazily per device).
const JumpMatrix* jump_table(int device);

// out = M * s
__device__ __forceinline__ void jump_apply(const JumpMatrix* __restrict__ M, uint64_t (&s)[4]) {
  uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll 1
  for (int w = 0; w < 4; ++w) {
    uint64_t word = s[w];
    while (word) {
      const int j = w * 64 + __ffsll(static_cast<long long>(word)) - 1;
      word &= word - 1;
      const uint64_t* c = M->col[j];
      o0 ^= c[0];
      o1 ^= c[1];
      o2 ^= c[2];
      o3 ^= c[3];
    }
  }
  s[0] = o0;
  s[1] = o1;
  s[2] = o2;
  s[3] = o3;
}

// State after skipping `seg * kSeg` draws from `s`.
__device__ __forceinline__ void jump_segments(const JumpMatrix* __restrict__ table, uint64_t seg,
                                              uint64_t (&s)[4]) {
  for (int e = 0; seg; ++e, seg >>= 1)
    if (seg & 1) jump_apply(table + e, s);
}

}  // namespace mqo_b200
