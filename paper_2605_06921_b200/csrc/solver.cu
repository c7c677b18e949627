// solver.cu -- the per-round kernels around the PGA loop.
//
//   K3 init_states     init_state (solver.cpp:30-46), Rng::normal (rng.hpp:49-62)
//   K4 reset           pool pick (solver.cpp:302), encode_solution (147-160),
//                      global_reset (48-63)
//   K5 harvest         extract_solution / cut_value / is_independent
//                      (objectives.cpp:143-180), harvest (solver.cpp:166-175)
//   K6 greedy          greedy_maximalize (localsearch.cpp:35-56)
//
// Every chain replays its own reference stream (Rng(derive_seed(seed, b+1)),
// solver.cpp:234-236).  Draws are data-independent except for the
// uniform_index rejection (probability < n / 2^64 per draw) and the
// Box-Muller u1 <= 0 redraw (2^-53): the parallel kernels generate segments
// of the stream with GF(2) jump-ahead, detect either event and the chain is
// then replayed by an exact sequential kernel -- results never depend on
// which path ran.
#include <algorithm>
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "glibc_math.cuh"
#include "jump.cuh"
#include "rng.cuh"

using namespace mqo_b200;

namespace mqo_b200 {

// ------------------------------------------------------- jump tables
namespace jump_detail {

// T: the xoshiro256** state transition as a column-major GF(2) matrix.
void transition_matrix(JumpMatrix& T) {
  for (int j = 0; j < 256; ++j) {
    Xoshiro x{{0, 0, 0, 0}};
    x.s[j >> 6] = 1ull << (j & 63);
    xoshiro_next(x);
    for (int w = 0; w < 4; ++w) T.col[j][w] = x.s[w];
  }
}

void mat_vec(const JumpMatrix& M, const uint64_t* s, uint64_t* out) {
  uint64_t o[4] = {0, 0, 0, 0};
  for (int j = 0; j < 256; ++j)
    if ((s[j >> 6] >> (j & 63)) & 1)
      for (int w = 0; w < 4; ++w) o[w] ^= M.col[j][w];
  for (int w = 0; w < 4; ++w) out[w] = o[w];
}

void mat_mul(const JumpMatrix& A, const JumpMatrix& B, JumpMatrix& C) {  // C = A*B
  for (int j = 0; j < 256; ++j) mat_vec(A, B.col[j], C.col[j]);
}

}  // namespace jump_detail

const JumpMatrix* jump_table(int device) {
  using namespace jump_detail;
  static std::mutex mu;
  static const JumpMatrix* tables[64] = {nullptr};
  std::lock_guard<std::mutex> lock(mu);
  if (tables[device]) return tables[device];
  std::vector<JumpMatrix> host(kJumpLevels);
  JumpMatrix P;
  transition_matrix(P);
  for (int i = 0; (1 << i) < kSeg; ++i) {  // P = T^kSeg
    JumpMatrix Q;
    mat_mul(P, P, Q);
    P = Q;
  }
  host[0] = P;
  for (int e = 1; e < kJumpLevels; ++e) mat_mul(host[e - 1], host[e - 1], host[e]);
  JumpMatrix* d = nullptr;
  MQO_CUDA(cudaMalloc(&d, sizeof(JumpMatrix) * kJumpLevels));
  MQO_CUDA(cudaMemcpy(d, host.data(), sizeof(JumpMatrix) * kJumpLevels, cudaMemcpyHostToDevice));
  tables[device] = d;
  return d;
}

}  // namespace mqo_b200

namespace {

constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi (exact doubling)

__device__ __forceinline__ Xoshiro load_state(const ChainRng& r) {
  return Xoshiro{{r.s[0], r.s[1], r.s[2], r.s[3]}};
}

// ------------------------------------------------------------- K3 init
// Thread (segment t, chain b): Box-Muller pairs [t*128, t*128+128) of the
// (log / sincos: glibc_math.cuh, identical bits to the reference's libm calls)
// chain's init section; warps span 32 consecutive chains so the writes of a
// vertex row are coalesced.
__global__ void k_init_normals(const int64_t* __restrict__ off, int32_t n, int32_t dmax,
                               int32_t mis, double sigma, ChainRng* rng,
                               const ChainRng* __restrict__ saved, int32_t B, int32_t Bp,
                               double* __restrict__ X, const JumpMatrix* __restrict__ table,
                               int64_t segments) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int groups = (B + 31) / 32;
  const int64_t t = gw / groups;
  const int b = static_cast<int>(gw % groups) * 32 + lane;
  if (t >= segments || b >= B) return;
  const ChainRng r0 = saved[b];  // stream position at the start of init
  const int32_t s0 = r0.has_spare ? 1 : 0;
  const int64_t m = n - s0;                 // normals still to draw in pairs
  const int64_t pairs = (m + 1) / 2;
  constexpr int kPairs = kSeg / 2;
  const int64_t p_begin = t * kPairs, p_end = (pairs < p_begin + kPairs ? pairs : p_begin + kPairs);
  const double dm = static_cast<double>(dmax);
  auto base_of = [&](int64_t v) {
    const double ratio = 1.0 - static_cast<double>(off[v + 1] - off[v]) / dm;
    return mis ? ratio : ex_sub(ex_mul(2.0, ratio), 1.0);
  };
  const double lo = mis ? 0.0 : -1.0;
  if (t == 0 && s0) {  // vertex 0 takes the cached spare: mean + stddev * spare_
    const double nv = ex_add(0.0, ex_mul(sigma, r0.spare));
    X[b] = clamp_box(ex_add(base_of(0), nv), lo);
  }
  if (p_begin >= p_end) {
    if (t == 0 && pairs == 0) rng[b].has_spare = 0;  // n == s0: spare consumed, no draws
    return;
  }
  uint64_t s[4] = {r0.s[0], r0.s[1], r0.s[2], r0.s[3]};
  jump_segments(table, static_cast<uint64_t>(t), s);
  Xoshiro x{{s[0], s[1], s[2], s[3]}};
  bool rejected = false;
  double last_sin = 0.0;
  for (int64_t p = p_begin; p < p_end; ++p) {
    const double u1 = u01_of(xoshiro_next(x));
    const double u2 = u01_of(xoshiro_next(x));
    if (u1 <= 0.0) rejected = true;  // rng.hpp:56 redraw -> exact replay
    const double rad = __dsqrt_rn(ex_mul(-2.0, mqo_glibc::glibc_log(u1)));
    const double theta = ex_mul(kTwoPi, u2);
    double sn, cs;
    mqo_glibc::glibc_sincos(theta, &sn, &cs);
    const int64_t v = s0 + 2 * p;
    const double first = ex_add(0.0, ex_mul(ex_mul(sigma, rad), cs));
    X[v * Bp + b] = clamp_box(ex_add(base_of(v), first), lo);
    const double spare = ex_mul(rad, sn);
    if (v + 1 < n) {
      const double second = ex_add(0.0, ex_mul(sigma, spare));
      X[(v + 1) * Bp + b] = clamp_box(ex_add(base_of(v + 1), second), lo);
    } else {
      last_sin = spare;
    }
  }
  if (rejected) atomicOr(&rng[b].flags, 1);
  if (p_end == pairs) {  // the thread holding the last pair owns the end state
    ChainRng& o = rng[b];
    o.s[0] = x.s[0];
    o.s[1] = x.s[1];
    o.s[2] = x.s[2];
    o.s[3] = x.s[3];
    if (m & 1) {
      o.spare = last_sin;
      o.has_spare = 1;
    } else {
      o.has_spare = 0;
    }
  }
}

// Exact sequential replay of init_state for the chains flagged above (and
// the reference path when sigma draws must follow the redraw loop).
__global__ void k_init_sequential(const int64_t* __restrict__ off, int32_t n, int32_t dmax,
                                  int32_t mis, double sigma, ChainRng* rng, const ChainRng* saved,
                                  int32_t B, int32_t Bp, double* __restrict__ X, int32_t only_flagged) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (only_flagged && !(rng[b].flags & 1)) return;
  ChainRng r = saved[b];
  Xoshiro x = load_state(r);
  const double dm = static_cast<double>(dmax);
  const double lo = mis ? 0.0 : -1.0;
  for (int64_t v = 0; v < n; ++v) {
    const double ratio = 1.0 - static_cast<double>(off[v + 1] - off[v]) / dm;
    double base = mis ? ratio : ex_sub(ex_mul(2.0, ratio), 1.0);
    double nv;
    if (r.has_spare) {
      r.has_spare = 0;
      nv = ex_add(0.0, ex_mul(sigma, r.spare));
    } else {
      double u1 = u01_of(xoshiro_next(x));
      const double u2 = u01_of(xoshiro_next(x));
      while (u1 <= 0.0) u1 = u01_of(xoshiro_next(x));
      const double rad = __dsqrt_rn(ex_mul(-2.0, mqo_glibc::glibc_log(u1)));
      const double theta = ex_mul(kTwoPi, u2);
      double sn, cs;
      mqo_glibc::glibc_sincos(theta, &sn, &cs);
      r.spare = ex_mul(rad, sn);
      r.has_spare = 1;
      nv = ex_add(0.0, ex_mul(ex_mul(sigma, rad), cs));
    }
    X[v * Bp + b] = clamp_box(ex_add(base, nv), lo);
  }
  for (int w = 0; w < 4; ++w) r.s[w] = x.s[w];
  r.flags = 0;
  rng[b] = r;
}

// init without noise / init_constant: x = Pi(base) or Pi(c) (solver.cpp:283-287)
__global__ void k_init_plain(const int64_t* __restrict__ off, int32_t n, int32_t dmax, int32_t mis,
                             int32_t use_const, double c, int32_t B, int32_t Bp,
                             double* __restrict__ X) {
  const int64_t total = static_cast<int64_t>(n) * Bp;
  const double lo = mis ? 0.0 : -1.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i / Bp;
    const int b = static_cast<int>(i % Bp);
    if (b >= B) continue;
    double val;
    if (use_const) {
      val = c;
    } else {
      const double ratio = 1.0 - static_cast<double>(off[v + 1] - off[v]) / static_cast<double>(dmax);
      val = mis ? ratio : ex_sub(ex_mul(2.0, ratio), 1.0);
    }
    X[i] = clamp_box(val, lo);
  }
}

// -------------------------------------------------------------- K4 reset
// One thread per chain: the pool pick (solver.cpp:302) -- uniform_index
// with its exact rejection loop.
__global__ void k_reset_pick(ChainRng* rng, int32_t B, uint64_t pool_size, int32_t* pick) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Xoshiro x = load_state(rng[b]);
  pick[b] = static_cast<int32_t>(xoshiro_index(x, pool_size));
  for (int w = 0; w < 4; ++w) rng[b].s[w] = x.s[w];
  rng[b].flags = 0;
}

// encode_solution (solver.cpp:147-160) of each chain's picked pool body.
__global__ void k_encode(const uint64_t* __restrict__ pool, int64_t W, const int32_t* __restrict__ pick,
                         int32_t n, int32_t B, int32_t Bp, int32_t mis, double* __restrict__ X) {
  const int64_t total = static_cast<int64_t>(n) * Bp;
  const double zero = mis ? 0.0 : -1.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i / Bp;
    const int b = static_cast<int>(i % Bp);
    if (b >= B) continue;
    const uint64_t w = __ldg(pool + static_cast<int64_t>(pick[b]) * W + (v >> 6));
    X[i] = ((w >> (63 - (v & 63))) & 1) ? 1.0 : zero;
  }
}

// Fisher-Yates draws j_i = i + uniform_index(n - i), i < k, segment-parallel.
__global__ void k_reset_draw(ChainRng* rng, const ChainRng* __restrict__ saved, int32_t B,
                             int32_t n, int32_t k,
                             int32_t* __restrict__ jdraw, const JumpMatrix* __restrict__ table,
                             int64_t segments) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int groups = (B + 31) / 32;
  const int64_t t = gw / groups;
  const int b = static_cast<int>(gw % groups) * 32 + lane;
  if (t >= segments || b >= B) return;
  const int64_t i0 = t * kSeg, i1 = (static_cast<int64_t>(k) < i0 + kSeg ? static_cast<int64_t>(k) : i0 + kSeg);
  uint64_t s[4] = {saved[b].s[0], saved[b].s[1], saved[b].s[2], saved[b].s[3]};
  jump_segments(table, static_cast<uint64_t>(t), s);
  Xoshiro x{{s[0], s[1], s[2], s[3]}};
  bool rejected = false;
  int32_t* jd = jdraw + static_cast<int64_t>(b) * n;
  for (int64_t i = i0; i < i1; ++i) {
    const uint64_t N = static_cast<uint64_t>(n - i);
    const uint64_t r = xoshiro_next(x);
    if (r < index_threshold(N)) rejected = true;
    jd[i] = static_cast<int32_t>(i + static_cast<int64_t>(r % N));
  }
  if (rejected) atomicOr(&rng[b].flags, 1);
  if (i1 == k) {  // end of the section: the chain's next stream position
    rng[b].s[0] = x.s[0];
    rng[b].s[1] = x.s[1];
    rng[b].s[2] = x.s[2];
    rng[b].s[3] = x.s[3];
  }
}

// lastw[j_i] = max{i : j_i != i}
__global__ void k_reset_scatter(const int32_t* __restrict__ jdraw, int32_t* lastw, int32_t B,
                                int32_t n, int32_t k) {
  const int64_t total = static_cast<int64_t>(B) * k;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / k, i = q % k;
    const int32_t j = jdraw[b * n + i];
    if (j != i) atomicMax(lastw + b * n + j, static_cast<int32_t>(i));
  }
}

// Value finally resting at position p >= k: the value carried there by its
// last writer (pointer chase through earlier writers), or p itself.  Those
// n-k values are exactly the vertices NOT chosen; mark them (state8 = 1).
__global__ void k_reset_keep(const int32_t* __restrict__ lastw, int32_t B, int32_t Bp, int32_t n,
                             int32_t k, uint8_t* __restrict__ keep) {
  const int64_t span = n - k;
  const int64_t total = static_cast<int64_t>(B) * span;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / span, p = k + q % span;
    const int32_t* lw = lastw + b * n;
    int32_t t = lw[p];
    int64_t val = p;
    if (t >= 0) {
      while (lw[t] >= 0) t = lw[t];
      val = t;
    }
    keep[val * Bp + b] = 1;
  }
}

__global__ void k_reset_zero(const uint8_t* __restrict__ keep, int32_t n, int32_t B, int32_t Bp,
                             const ChainRng* __restrict__ rng, double* __restrict__ X) {
  const int64_t total = static_cast<int64_t>(n) * Bp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(i % Bp);
    if (b < B && !keep[i] && !(rng[b].flags & 1)) X[i] = 0.0;
  }
}

__global__ void k_clear_flags(ChainRng* rng, int32_t Bp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < Bp) rng[b].flags = 0;
}

// Exact sequential global_reset for flagged chains (rejection happened):
// a literal partial Fisher-Yates on an order array (solver.cpp:53-61).
__global__ void k_reset_sequential(ChainRng* rng, const ChainRng* saved, int32_t B, int32_t Bp,
                                   int32_t n, int32_t k, int32_t* order_scratch,
                                   double* __restrict__ X) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !(rng[b].flags & 1)) return;
  Xoshiro x = load_state(saved[b]);
  int32_t* order = order_scratch + static_cast<int64_t>(b) * n;
  for (int32_t v = 0; v < n; ++v) order[v] = v;
  for (int32_t i = 0; i < k; ++i) {
    const int32_t j = i + static_cast<int32_t>(xoshiro_index(x, static_cast<uint64_t>(n - i)));
    const int32_t tmp = order[i];
    order[i] = order[j];
    order[j] = tmp;
  }
  for (int32_t i = 0; i < k; ++i) X[static_cast<int64_t>(order[i]) * Bp + b] = 0.0;
  for (int w = 0; w < 4; ++w) rng[b].s[w] = x.s[w];
  rng[b].flags = 0;
}

// ----------------------------------------------------------- K5/K6 harvest
enum : uint8_t { kOut = 0, kIn = 1, kFree = 2, kJoined = 3 };

// MIS: threshold (x > 0.5), tightness, independence, free set.
__global__ void k_mis_prepare(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                              int32_t n, int32_t B, int32_t Bp, const double* __restrict__ X,
                              uint8_t* __restrict__ st, int32_t* __restrict__ dependent) {
  const int64_t total = static_cast<int64_t>(n) * Bp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i / Bp;
    const int b = static_cast<int>(i % Bp);
    if (b >= B) {
      st[i] = kOut;
      continue;
    }
    const bool sel = X[i] > 0.5;  // objectives.cpp:150
    int cnt = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) cnt += X[static_cast<int64_t>(nbr[e]) * Bp + b] > 0.5;
    if (sel && cnt) dependent[b] = 1;  // is_independent fails (objectives.cpp:173-180)
    st[i] = sel ? kIn : (cnt == 0 ? kFree : kOut);
  }
}

// One round of the parallel lexicographically-first greedy over the free
// set with priority (degree, id) -- the same set greedy_maximalize
// (localsearch.cpp:45-53) builds sequentially: v joins once every
// higher-priority free neighbour is excluded; it is excluded as soon as a
// neighbour joined.  Decisions are final, so in-place updates are safe.
__global__ void k_mis_greedy_round(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                   int32_t n, int32_t B, int32_t Bp, uint8_t* st,
                                   const int32_t* __restrict__ dependent, int32_t* changed,
                                   int32_t* undecided) {
  const int64_t total = static_cast<int64_t>(n) * Bp;
  int my_changed = 0, my_und = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (st[i] != kFree) continue;
    const int64_t v = i / Bp;
    const int b = static_cast<int>(i % Bp);
    if (dependent[b]) {
      st[i] = kOut;
      continue;
    }
    const int64_t dv = off[v + 1] - off[v];
    bool wait = false, excluded = false;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      const int32_t u = nbr[e];
      const uint8_t su = *(volatile const uint8_t*)(st + static_cast<int64_t>(u) * Bp + b);
      if (su == kJoined) {
        excluded = true;
        break;
      }
      if (su == kFree) {
        const int64_t du = off[u + 1] - off[u];
        if (du < dv || (du == dv && u < v)) wait = true;
      }
    }
    if (excluded) {
      st[i] = kOut;
      ++my_changed;
    } else if (!wait) {
      st[i] = kJoined;
      ++my_changed;
    } else {
      ++my_und;
    }
  }
  if (my_changed) atomicAdd(changed, my_changed);
  if (my_und) atomicAdd(undecided, my_und);
}

// Score + packed body per chain from a state array (MIS: in|joined) or
// from x (MaxCut: side = x > 0, objectives.cpp:154).  One warp per
// (chain, 64-vertex word): lane l handles vertices 2l, 2l+1 of the word.
__global__ void k_pack(const uint8_t* __restrict__ st, const double* __restrict__ X, int32_t mis,
                       int32_t n, int32_t B, int32_t Bp, uint64_t* __restrict__ bodies,
                       int64_t W, int64_t* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (gw >= W * B) return;
  const int64_t w = gw / B;
  const int b = static_cast<int>(gw % B);
  uint64_t bits = 0;
  for (int h = 0; h < 2; ++h) {
    const int64_t v = w * 64 + lane * 2 + h;
    bool on = false;
    if (v < n) {
      const int64_t i = v * Bp + b;
      on = mis ? (st[i] == kIn || st[i] == kJoined) : (X[i] > 0.0);
    }
    if (on) bits |= 1ull << (63 - (lane * 2 + h));
  }
  for (int o = 16; o; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
  if (lane == 0) {
    bodies[static_cast<int64_t>(b) * W + w] = bits;
    if (mis && bits) atomicAdd(reinterpret_cast<unsigned long long*>(count + b),
                               static_cast<unsigned long long>(__popcll(bits)));
  }
}

// cut_value (objectives.cpp:163-171) for all chains at once, vertex-major.
// K5a: side bits chain-minor -- one ballot per (vertex, 32 chains) over a
// coalesced row of X (side_v = [x_v > 0], objectives.cpp:153-157, the same
// predicate k_pack uses); words per vertex padded to a multiple of 4 so a
// 128-chain slice is one 16-byte load.
__global__ void k_side_bits(const double* __restrict__ X, int32_t n, int32_t B, int32_t Bp,
                            int32_t words, uint32_t* __restrict__ sides) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  if (Bp < 32) {
    // 32 / Bp rows per ballot (Bp is 4, 8 or 16 here): lane l reads chain
    // l % Bp of row v0 + l / Bp; the words past the chains stay zero (the
    // buffer is cleared when allocated)
    const int per = 32 / Bp;
    for (int64_t v0 = w0 * per; v0 < n; v0 += nw * per) {
      const int64_t v = v0 + lane / Bp;
      const int c = lane % Bp;
      const bool on = v < n && c < B && X[v * Bp + c] > 0.0;
      const uint32_t bits = __ballot_sync(0xffffffffu, on);
      if (lane < per && v0 + lane < n)
        sides[(v0 + lane) * words] = (bits >> (lane * Bp)) & ((1u << Bp) - 1u);
    }
    return;
  }
  const int used = (B + 31) / 32;  // words holding chains; the others stay zero
  const int64_t total = static_cast<int64_t>(n) * used;
  for (int64_t q = w0; q < total; q += nw) {
    const int64_t v = q / used;
    const int wd = static_cast<int>(q % used);
    const int c = wd * 32 + lane;
    const bool on = c < B && X[v * Bp + c] > 0.0;
    const uint32_t bits = __ballot_sync(0xffffffffu, on);
    if (lane == 0) sides[v * words + wd] = bits;
  }
}

// K5b: one warp per row v (grid-stride), 128 chains per pass: lane l counts
// chains l, l+32, l+64, l+96.  The row's neighbour ids are loaded 32 at a
// time (coalesced) and broadcast by shuffle; every edge (v, u > v) costs one
// 16-byte broadcast load of u's side bits and an XOR -- the CSR is read
// once per 128 chains instead of once per chain.
__global__ void k_cut_vm(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                         int32_t n, int32_t B, int32_t words, const uint32_t* __restrict__ sides,
                         int64_t* __restrict__ cut) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int c4 = 0; c4 < words; c4 += 4) {
    uint32_t cnt[4] = {0, 0, 0, 0};
    for (int64_t v = warp; v < n; v += nwarps) {
      const uint4 sv = __ldg(reinterpret_cast<const uint4*>(sides + v * words + c4));
      // each edge counted once, from its higher endpoint: the lower
      // neighbours are a row prefix (rows ascend), and a hub's lower row is
      // short -- counted from the lower endpoint, one warp walked a hub's
      // thousands of neighbours while the grid waited
      const int64_t e0 = off[v], e1 = off[v + 1];
      for (int64_t base = e0; base < e1; base += 32) {
        const int32_t mine = base + lane < e1 ? __ldg(nbr + base + lane) : INT_MAX;
        const unsigned below = __ballot_sync(0xffffffffu, mine < v);
        if (!below) break;  // the rest of the row is above v
        const int k = __popc(below);  // a prefix of the chunk
#pragma unroll 8
        for (int j = 0; j < k; ++j) {
          const int32_t u = __shfl_sync(0xffffffffu, mine, j);
          const uint4 su = __ldg(reinterpret_cast<const uint4*>(sides + int64_t(u) * words + c4));
          cnt[0] += ((sv.x ^ su.x) >> lane) & 1u;
          cnt[1] += ((sv.y ^ su.y) >> lane) & 1u;
          cnt[2] += ((sv.z ^ su.z) >> lane) & 1u;
          cnt[3] += ((sv.w ^ su.w) >> lane) & 1u;
        }
        if (k < 32) break;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int chain = (c4 + k) * 32 + lane;
      if (chain < B && cnt[k])
        atomicAdd(reinterpret_cast<unsigned long long*>(cut + chain),
                  static_cast<unsigned long long>(cnt[k]));
    }
  }
}

// K5b for up to 32 chains (one side word per vertex), edge-parallel: a warp
// takes 32 consecutive CSR entries (the whole grid strides over the entry
// range, so hub rows spread over many warps), finds each entry's row among
// the chunk's few rows (crow[q] = the row holding entry 32q, a per-graph
// index; the offsets of rows crow[q]..crow[q+1] are shuffled between lanes),
// keeps the edge when its neighbour is lower (each edge once) and XORs the
// two side words; per chain c the warp sums bit c over its lanes with one
// ballot.  (k_cut_vm, a warp walking a row's neighbours one broadcast load
// at a time: 0.41 ms at C4 x 16; row blocks per warp: hub blocks 1.4 ms.)
__global__ void k_cut_edges(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                            const int32_t* __restrict__ crow, int64_t nnz, int32_t B,
                            int32_t words, const uint32_t* __restrict__ sides,
                            int64_t* __restrict__ cut) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t chunks = (nnz + 31) / 32;
  uint32_t cnt = 0;  // chain `lane`
  for (int64_t q = w0; q < chunks; q += nw) {
    const int32_t r0 = crow[q], r1 = crow[q + 1];  // rows r0..r1 hold the chunk
    const int span = r1 - r0 + 1;
    const int64_t ent = q * 32 + lane;
    int32_t v = r0;
    if (span <= 32) {
      const int64_t my_off = lane < span ? off[r0 + lane] : INT64_MAX;
      int r = 0;  // the last of the span's offsets <= ent
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int64_t o = __shfl_sync(0xffffffffu, my_off, r + step < 32 ? r + step : 31);
        if (r + step < span && o <= ent) r += step;
      }
      v = r0 + r;
    } else if (ent < nnz) {  // many empty / one-entry rows: search the offsets
      int32_t lo = r0, hi = r1;
      while (lo < hi) {
        const int32_t mid = lo + (hi - lo + 1) / 2;
        if (off[mid] <= ent) lo = mid; else hi = mid - 1;
      }
      v = lo;
    }
    uint32_t x = 0;
    if (ent < nnz) {
      const int32_t u = nbr[ent];
      if (u < v) x = sides[int64_t(v) * words] ^ sides[int64_t(u) * words];
    }
    for (int ch = 0; ch < B; ++ch) {
      const uint32_t bits = __ballot_sync(0xffffffffu, (x >> ch) & 1u);
      if (lane == ch) cnt += __popc(bits);
    }
  }
  if (lane < B && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(cut + lane),
                                 static_cast<unsigned long long>(cnt));
}

// crow[q] = the row holding CSR entry 32q (q < chunks), crow[chunks] = the
// row of the last entry
__global__ void k_chunk_rows(const int64_t* __restrict__ off, int32_t n, int64_t nnz,
                             int32_t* __restrict__ crow) {
  const int64_t chunks = (nnz + 31) / 32;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q <= chunks;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ent = q < chunks ? q * 32 : nnz - 1;
    int32_t lo = 0, hi = n - 1;  // the last row with off[row] <= ent
    while (lo < hi) {
      const int32_t mid = lo + (hi - lo + 1) / 2;
      if (off[mid] <= ent) lo = mid; else hi = mid - 1;
    }
    crow[q] = lo;
  }
}

int grid_for(int64_t work, int threads = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, 148 * 32)));
}

// the chunk -> row index of k_cut_edges, built once per graph
void ensure_chunk_rows(mqo_graph* g, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g->lazy_mu);
  if (g->d_crow) return;
  const int64_t chunks = (2 * g->m + 31) / 32;
  void* p = nullptr;
  const cudaStream_t ms = mem_stream(g->device);
  MQO_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * (chunks + 1), ms));
  MQO_CUDA(cudaStreamSynchronize(ms));
  auto* crow = static_cast<int32_t*>(p);
  k_chunk_rows<<<grid_for(chunks + 1), 256, 0, st>>>(g->d_off, g->n, 2 * g->m, crow);
  MQO_CUDA(cudaGetLastError());
  MQO_CUDA(cudaStreamSynchronize(st));
  g->d_crow = crow;
}

// Cut values of the current iterates into d_scores (zeroed by the caller).
void launch_cut(mqo_batch* b, const double* X) {
  const mqo_graph* g = b->g;
  const int32_t words = ((b->B + 31) / 32 + 3) / 4 * 4;
  if (!b->d_sides) {  // zeroed once: k_side_bits writes only the words holding chains
    const size_t bytes = sizeof(uint32_t) * std::max<int64_t>(1, int64_t(g->n) * words);
    dalloc(b, &b->d_sides, bytes);
    MQO_CUDA(cudaMemsetAsync(b->d_sides, 0, bytes, b->stream));
  }
  const int64_t rows_per_warp = b->Bp < 32 ? 32 / b->Bp : 1;
  k_side_bits<<<grid_for(int64_t(g->n) * ((b->B + 31) / 32) * 32 / rows_per_warp), 256, 0, b->stream>>>(
      X, g->n, b->B, b->Bp, words, b->d_sides);
  MQO_CUDA(cudaGetLastError());
  const int64_t nnz = 2 * g->m;
  if (b->B <= 32 && nnz > 0) {
    ensure_chunk_rows(const_cast<mqo_graph*>(g), b->stream);
    k_cut_edges<<<grid_for((nnz + 31) / 32 * 32), 256, 0, b->stream>>>(
        g->d_off, g->d_nbr, g->d_crow, nnz, b->B, words, b->d_sides, b->d_scores);
  } else
    k_cut_vm<<<148 * 8, 256, 0, b->stream>>>(g->d_off, g->d_nbr, g->n, b->B, words, b->d_sides,
                                             b->d_scores);
  MQO_CUDA(cudaGetLastError());
}

void ensure_solver_buffers(mqo_batch* b) {
  const mqo_graph* g = b->g;
  const int64_t W = body_words(g->n);
  if (!b->d_rng) {
    dalloc(b, &b->d_rng, sizeof(ChainRng) * b->Bp * 2);  // [0]: live, [Bp]: saved
    // on the batch stream: a legacy-stream memset is not ordered with the
    // (non-blocking) batch stream and could land after the seeding copy
    MQO_CUDA(cudaMemsetAsync(b->d_rng, 0, sizeof(ChainRng) * b->Bp * 2, b->stream));
  }
  if (!b->d_bodies) {
    dalloc(b, &b->d_bodies, sizeof(uint64_t) * std::max<int64_t>(1, W * b->Bp));
    dalloc(b, &b->d_scores, sizeof(int64_t) * b->Bp);
    dalloc(b, &b->d_valid, sizeof(int32_t) * b->Bp);
    dalloc(b, &b->d_pick, sizeof(int32_t) * b->Bp);
    dalloc(b, &b->d_counter, sizeof(int32_t) * 4);
  }
  if (!b->d_state8)
    dalloc(b, &b->d_state8, std::max<int64_t>(1, int64_t(g->n) * b->Bp));
}

void ensure_reset_buffers(mqo_batch* b) {
  const int64_t cells = std::max<int64_t>(1, int64_t(b->g->n) * b->B);
  if (!b->d_lastw) {
    dalloc(b, &b->d_lastw, sizeof(int32_t) * cells);
    dalloc(b, &b->d_jdraw, sizeof(int32_t) * cells);
  }
}

}  // namespace

namespace mqo_b200 {

void free_solver_buffers(mqo_batch* b) {
  dfree(b, b->d_rng);
  dfree(b, b->d_pool);
  dfree(b, b->d_bodies);
  dfree(b, b->d_scores);
  dfree(b, b->d_valid);
  dfree(b, b->d_pick);
  dfree(b, b->d_state8);
  dfree(b, b->d_sides);
  dfree(b, b->d_lastw);
  dfree(b, b->d_jdraw);
  dfree(b, b->d_counter);
}

// K3 on the device; Box-Muller's log / sincos are the bit-exact replays of
// the host glibc routines (glibc_math.cuh), so x matches init_state bit for bit.
void init_states_device(mqo_batch* b, int32_t problem, double sigma) {
  mqo_graph* g = b->g;
  ensure_solver_buffers(b);
  double* X = b->d_x[b->cur];
  const int mis = problem == MQO_PROBLEM_MIS;
  if (g->n == 0) return;
  if (!(sigma > 0.0)) {
    k_init_plain<<<grid_for(int64_t(g->n) * b->Bp), 256, 0, b->stream>>>(
        g->d_off, g->n, g->max_degree, mis, 0, 0.0, b->B, b->Bp, X);
    MQO_CUDA(cudaGetLastError());
    return;
  }
  ChainRng* saved = b->d_rng + b->Bp;
  k_clear_flags<<<(b->Bp + 255) / 256, 256, 0, b->stream>>>(b->d_rng, b->Bp);
  MQO_CUDA(cudaMemcpyAsync(saved, b->d_rng, sizeof(ChainRng) * b->Bp, cudaMemcpyDeviceToDevice,
                           b->stream));
  const int64_t pairs = (int64_t(g->n) + 1) / 2 + 1;
  const int64_t segments = (pairs + kSeg / 2 - 1) / (kSeg / 2);
  const int groups = (b->B + 31) / 32;
  const int64_t threads = segments * groups * 32;
  k_init_normals<<<static_cast<int>((threads + 255) / 256), 256, 0, b->stream>>>(
      g->d_off, g->n, g->max_degree, mis, sigma, b->d_rng, saved, b->B, b->Bp, X,
      jump_table(g->device), segments);
  MQO_CUDA(cudaGetLastError());
  k_init_sequential<<<(b->B + 127) / 128, 128, 0, b->stream>>>(
      g->d_off, g->n, g->max_degree, mis, sigma, b->d_rng, saved, b->B, b->Bp, X, 1);
  MQO_CUDA(cudaGetLastError());
}

void init_states_constant(mqo_batch* b, int32_t problem, double c) {
  mqo_graph* g = b->g;
  if (g->n == 0) return;
  k_init_plain<<<grid_for(int64_t(g->n) * b->Bp), 256, 0, b->stream>>>(
      g->d_off, g->n, g->max_degree, problem == MQO_PROBLEM_MIS, 1, c, b->B, b->Bp,
      b->d_x[b->cur]);
  MQO_CUDA(cudaGetLastError());
}

// global_reset on the current x of every chain (no pool pick).
void global_reset_device(mqo_batch* b, double rho) {
  mqo_graph* g = b->g;
  ensure_solver_buffers(b);
  const int32_t n = g->n;
  const int32_t k = static_cast<int32_t>(std::floor(rho * n));  // solver.cpp:51
  ChainRng* saved = b->d_rng + b->Bp;
  k_clear_flags<<<(b->Bp + 255) / 256, 256, 0, b->stream>>>(b->d_rng, b->Bp);
  MQO_CUDA(cudaMemcpyAsync(saved, b->d_rng, sizeof(ChainRng) * b->Bp, cudaMemcpyDeviceToDevice,
                           b->stream));
  if (k <= 0 || n == 0) return;
  ensure_reset_buffers(b);
  double* X = b->d_x[b->cur];
  const int64_t cells = int64_t(n) * b->B;
  MQO_CUDA(cudaMemsetAsync(b->d_lastw, 0xFF, sizeof(int32_t) * cells, b->stream));
  MQO_CUDA(cudaMemsetAsync(b->d_state8, 0, int64_t(n) * b->Bp, b->stream));
  const int64_t segments = (int64_t(k) + kSeg - 1) / kSeg;
  const int groups = (b->B + 31) / 32;
  const int64_t threads = segments * groups * 32;
  k_reset_draw<<<static_cast<int>((threads + 255) / 256), 256, 0, b->stream>>>(
      b->d_rng, saved, b->B, n, k, b->d_jdraw, jump_table(g->device), segments);
  MQO_CUDA(cudaGetLastError());
  k_reset_scatter<<<grid_for(int64_t(b->B) * k), 256, 0, b->stream>>>(b->d_jdraw, b->d_lastw,
                                                                      b->B, n, k);
  MQO_CUDA(cudaGetLastError());
  k_reset_keep<<<grid_for(int64_t(b->B) * (n - k)), 256, 0, b->stream>>>(b->d_lastw, b->B, b->Bp,
                                                                        n, k, b->d_state8);
  MQO_CUDA(cudaGetLastError());
  k_reset_zero<<<grid_for(int64_t(n) * b->Bp), 256, 0, b->stream>>>(b->d_state8, n, b->B, b->Bp,
                                                                    b->d_rng, X);
  MQO_CUDA(cudaGetLastError());
  k_reset_sequential<<<(b->B + 127) / 128, 128, 0, b->stream>>>(b->d_rng, saved, b->B, b->Bp, n,
                                                                k, b->d_lastw, X);
  MQO_CUDA(cudaGetLastError());
}

// Pool pick + encode + global_reset (solver.cpp:301-303).
void reset_from_pool(mqo_batch* b, int32_t problem, double rho) {
  mqo_graph* g = b->g;
  ensure_solver_buffers(b);
  if (b->pool_size < 1) throw std::logic_error("reset: empty pool");
  k_reset_pick<<<(b->B + 127) / 128, 128, 0, b->stream>>>(b->d_rng, b->B,
                                                         static_cast<uint64_t>(b->pool_size),
                                                         b->d_pick);
  MQO_CUDA(cudaGetLastError());
  if (g->n)
    k_encode<<<grid_for(int64_t(g->n) * b->Bp), 256, 0, b->stream>>>(
        b->d_pool, body_words(g->n), b->d_pick, g->n, b->B, b->Bp, problem == MQO_PROBLEM_MIS,
        b->d_x[b->cur]);
  MQO_CUDA(cudaGetLastError());
  global_reset_device(b, rho);
}

// K5/K6: harvest every chain's current x into d_scores / d_valid /
// d_bodies (solver.cpp:166-175).
void harvest_device(mqo_batch* b, int32_t problem) {
  mqo_graph* g = b->g;
  ensure_solver_buffers(b);
  const int32_t n = g->n;
  const int64_t W = body_words(n);
  const int64_t cells = int64_t(n) * b->Bp;
  double* X = b->d_x[b->cur];
  MQO_CUDA(cudaMemsetAsync(b->d_scores, 0, sizeof(int64_t) * b->Bp, b->stream));
  MQO_CUDA(cudaMemsetAsync(b->d_valid, 0, sizeof(int32_t) * b->Bp, b->stream));
  if (problem == MQO_PROBLEM_MIS) {
    // d_valid doubles as the "dependent" flag until the end
    k_mis_prepare<<<grid_for(cells), 256, 0, b->stream>>>(g->d_off, g->d_nbr, n, b->B, b->Bp, X,
                                                          b->d_state8, b->d_valid);
    MQO_CUDA(cudaGetLastError());
    for (int round = 0;; ++round) {
      MQO_CUDA(cudaMemsetAsync(b->d_counter, 0, sizeof(int32_t) * 2, b->stream));
      k_mis_greedy_round<<<grid_for(cells), 256, 0, b->stream>>>(
          g->d_off, g->d_nbr, n, b->B, b->Bp, b->d_state8, b->d_valid, b->d_counter,
          b->d_counter + 1);
      MQO_CUDA(cudaGetLastError());
      MQO_CUDA(cudaMemcpyAsync(b->h_flag, b->d_counter, sizeof(int32_t) * 2,
                               cudaMemcpyDeviceToHost, b->stream));
      MQO_CUDA(cudaStreamSynchronize(b->stream));
      MQO_TRACE("greedy round %d: changed %d undecided %d", round, b->h_flag[0], b->h_flag[1]);
      if (b->h_flag[1] == 0) break;
      if (b->h_flag[0] == 0) throw std::logic_error("greedy_maximalize: no progress");
    }
  }
  if (n) {
    const int64_t warps = W * b->B;
    k_pack<<<static_cast<int>((warps * 32 + 255) / 256), 256, 0, b->stream>>>(
        b->d_state8, X, problem == MQO_PROBLEM_MIS, n, b->B, b->Bp, b->d_bodies, W, b->d_scores);
    MQO_CUDA(cudaGetLastError());
    if (problem == MQO_PROBLEM_MAXCUT) launch_cut(b, X);
  }
}

}  // namespace mqo_b200

// ------------------------------------------------------------------ C ABI
extern "C" int mqo_batch_seed_streams(mqo_batch* b, uint64_t master_seed, uint64_t first_stream) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_batch_seed_streams: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    ensure_solver_buffers(b);
    std::vector<ChainRng> h(b->Bp);
    for (int i = 0; i < b->Bp; ++i) {
      const Xoshiro x = xoshiro_seed(derive_seed(master_seed, first_stream + i));
      h[i] = ChainRng{{x.s[0], x.s[1], x.s[2], x.s[3]}, 0.0, 0, 0};
    }
    MQO_CUDA(cudaMemcpyAsync(b->d_rng, h.data(), sizeof(ChainRng) * b->Bp, cudaMemcpyHostToDevice,
                             b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
  });
}

extern "C" int mqo_batch_get_streams(mqo_batch* b, mqo_rng_state* out) {
  return guard([&] {
    if (!b || !out) throw std::invalid_argument("mqo_batch_get_streams: null argument");
    MQO_CUDA(cudaSetDevice(b->g->device));
    ensure_solver_buffers(b);
    static_assert(sizeof(ChainRng) == sizeof(mqo_rng_state), "layout");
    MQO_CUDA(cudaMemcpyAsync(out, b->d_rng, sizeof(ChainRng) * b->B, cudaMemcpyDeviceToHost,
                             b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
  });
}

extern "C" int mqo_batch_set_streams(mqo_batch* b, const mqo_rng_state* in) {
  return guard([&] {
    if (!b || !in) throw std::invalid_argument("mqo_batch_set_streams: null argument");
    MQO_CUDA(cudaSetDevice(b->g->device));
    ensure_solver_buffers(b);
    MQO_CUDA(cudaMemcpyAsync(b->d_rng, in, sizeof(ChainRng) * b->B, cudaMemcpyHostToDevice,
                             b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
  });
}

extern "C" int mqo_init_states(mqo_batch* b, int32_t problem, double sigma) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_init_states: null batch");
    if (b->g->n == 0) throw std::invalid_argument("init_state: empty graph");
    if (b->g->max_degree < 1)
      throw std::invalid_argument("init_state: edgeless graph (strip isolated vertices upstream)");
    MQO_CUDA(cudaSetDevice(b->g->device));
    init_states_device(b, problem, sigma);
  });
}

extern "C" int mqo_init_constant(mqo_batch* b, int32_t problem, double c) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_init_constant: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    init_states_constant(b, problem, c);
  });
}

extern "C" int mqo_global_reset(mqo_batch* b, double rho) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_global_reset: null batch");
    if (rho < 0.0 || rho >= 1.0) throw std::invalid_argument("global_reset: rho must be in [0, 1)");
    MQO_CUDA(cudaSetDevice(b->g->device));
    global_reset_device(b, rho);
  });
}

extern "C" int mqo_set_pool(mqo_batch* b, int32_t count, const uint64_t* packed) {
  return guard([&] {
    if (!b || count < 0 || (count && !packed)) throw std::invalid_argument("mqo_set_pool: bad arguments");
    MQO_CUDA(cudaSetDevice(b->g->device));
    const int64_t W = body_words(b->g->n);
    if (count > b->pool_cap) {
      dfree(b, b->d_pool);
      b->d_pool = nullptr;
      dalloc(b, &b->d_pool, sizeof(uint64_t) * std::max<int64_t>(1, W * count));
      b->pool_cap = count;
    }
    if (count)
      MQO_CUDA(cudaMemcpyAsync(b->d_pool, packed, sizeof(uint64_t) * W * count,
                               cudaMemcpyHostToDevice, b->stream));
    b->pool_size = count;
  });
}

extern "C" int mqo_reset_from_pool(mqo_batch* b, int32_t problem, double rho, int32_t* picks) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_reset_from_pool: null batch");
    if (rho < 0.0 || rho >= 1.0) throw std::invalid_argument("global_reset: rho must be in [0, 1)");
    MQO_CUDA(cudaSetDevice(b->g->device));
    reset_from_pool(b, problem, rho);
    if (picks) {
      MQO_CUDA(cudaMemcpyAsync(picks, b->d_pick, sizeof(int32_t) * b->B, cudaMemcpyDeviceToHost,
                               b->stream));
      MQO_CUDA(cudaStreamSynchronize(b->stream));
    }
  });
}

extern "C" int mqo_harvest(mqo_batch* b, int32_t problem, int64_t* scores, int32_t* valid,
                           uint64_t* packed) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_harvest: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    harvest_device(b, problem);
    std::vector<int32_t> dep(b->B);
    MQO_CUDA(cudaMemcpyAsync(dep.data(), b->d_valid, sizeof(int32_t) * b->B, cudaMemcpyDeviceToHost,
                             b->stream));
    if (scores)
      MQO_CUDA(cudaMemcpyAsync(scores, b->d_scores, sizeof(int64_t) * b->B, cudaMemcpyDeviceToHost,
                               b->stream));
    if (packed)
      MQO_CUDA(cudaMemcpyAsync(packed, b->d_bodies, sizeof(uint64_t) * body_words(b->g->n) * b->B,
                               cudaMemcpyDeviceToHost, b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
    // MIS: d_valid held "dependent"; MaxCut: every state is a valid cut
    if (valid)
      for (int i = 0; i < b->B; ++i) valid[i] = problem == MQO_PROBLEM_MIS ? (dep[i] ? 0 : 1) : 1;
  });
}

namespace {
__global__ void k_threshold_mis(const double* __restrict__ X, int64_t total, int32_t B, int32_t Bp,
                                uint8_t* __restrict__ st) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    st[i] = (static_cast<int>(i % Bp) < B && X[i] > 0.5) ? 1 : 0;  // objectives.cpp:150
}
}  // namespace

// extract_solution (objectives.cpp:143-161) without repair: MIS members
// x > 0.5 (score = |I|, independent[b] = is_independent), MaxCut sides
// x > 0 (score = cut_value).
extern "C" int mqo_extract(mqo_batch* b, int32_t problem, int64_t* scores, int32_t* independent,
                           uint64_t* packed) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_extract: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    ensure_solver_buffers(b);
    mqo_graph* g = b->g;
    const int32_t n = g->n;
    const int64_t W = body_words(n), cells = int64_t(n) * b->Bp;
    double* X = b->d_x[b->cur];
    MQO_CUDA(cudaMemsetAsync(b->d_scores, 0, sizeof(int64_t) * b->Bp, b->stream));
    MQO_CUDA(cudaMemsetAsync(b->d_valid, 0, sizeof(int32_t) * b->Bp, b->stream));
    if (n) {
      if (problem == MQO_PROBLEM_MIS) {
        k_mis_prepare<<<grid_for(cells), 256, 0, b->stream>>>(g->d_off, g->d_nbr, n, b->B, b->Bp,
                                                              X, b->d_state8, b->d_valid);
        k_threshold_mis<<<grid_for(cells), 256, 0, b->stream>>>(X, cells, b->B, b->Bp, b->d_state8);
      }
      const int64_t warps = W * b->B;
      k_pack<<<static_cast<int>((warps * 32 + 255) / 256), 256, 0, b->stream>>>(
          b->d_state8, X, problem == MQO_PROBLEM_MIS, n, b->B, b->Bp, b->d_bodies, W, b->d_scores);
      if (problem == MQO_PROBLEM_MAXCUT) launch_cut(b, X);
      MQO_CUDA(cudaGetLastError());
    }
    std::vector<int32_t> dep(b->B);
    MQO_CUDA(cudaMemcpyAsync(dep.data(), b->d_valid, sizeof(int32_t) * b->B, cudaMemcpyDeviceToHost,
                             b->stream));
    if (scores)
      MQO_CUDA(cudaMemcpyAsync(scores, b->d_scores, sizeof(int64_t) * b->B, cudaMemcpyDeviceToHost,
                               b->stream));
    if (packed)
      MQO_CUDA(cudaMemcpyAsync(packed, b->d_bodies, sizeof(uint64_t) * W * b->B,
                               cudaMemcpyDeviceToHost, b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
    if (independent)
      for (int i = 0; i < b->B; ++i) independent[i] = dep[i] ? 0 : 1;
  });
}
