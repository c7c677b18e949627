// rng.cuh -- xoshiro256** + splitmix64 (reference: rng.hpp:13-86), usable
// on host and device.  Streams are bit-identical to mqo::Rng.  The device
// side also needs jump-ahead (the xoshiro state transition is linear over
// GF(2)^256, so advancing by any count is a 256x256 bit-matrix product);
// see reset.cu for the matrix tables.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define MQO_HD __host__ __device__ __forceinline__
#else
#define MQO_HD inline
#endif

namespace mqo_b200 {

struct Xoshiro {
  uint64_t s[4];
};

MQO_HD uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

MQO_HD uint64_t splitmix64(uint64_t& s) {  // rng.hpp:71-76
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

MQO_HD Xoshiro xoshiro_seed(uint64_t seed) {  // rng.hpp:15-18
  Xoshiro r;
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r.s[i] = splitmix64(s);
  return r;
}

MQO_HD uint64_t xoshiro_next(Xoshiro& r) {  // rng.hpp:20-30
  const uint64_t result = rotl64(r.s[1] * 5, 7) * 9;
  const uint64_t t = r.s[1] << 17;
  r.s[2] ^= r.s[0];
  r.s[3] ^= r.s[1];
  r.s[1] ^= r.s[2];
  r.s[0] ^= r.s[3];
  r.s[2] ^= t;
  r.s[3] = rotl64(r.s[3], 45);
  return result;
}

MQO_HD double u01_of(uint64_t r) { return static_cast<double>(r >> 11) * 0x1.0p-53; }  // rng.hpp:33

// uniform_index rejection threshold (rng.hpp:41): draws below it are
// rejected and redrawn.
MQO_HD uint64_t index_threshold(uint64_t n) { return (0 - n) % n; }

MQO_HD uint64_t xoshiro_index(Xoshiro& r, uint64_t n) {  // rng.hpp:40-46
  const uint64_t threshold = index_threshold(n);
  for (;;) {
    const uint64_t x = xoshiro_next(r);
    if (x >= threshold) return x % n;
  }
}

MQO_HD uint64_t derive_seed(uint64_t master, uint64_t stream) {  // rng.hpp:80-86
  uint64_t s = master ^ (0x9e3779b97f4a7c15ULL + stream * 0xd1342543de82ef95ULL);
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace mqo_b200
