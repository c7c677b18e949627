// ls.cu -- K7/K8 discrete local search with the reference's exact
// sequential semantics (localsearch.cpp).
//
//   MaxCut  build_gain_table / apply_flip / one_flip_pass / two_flip_pass /
//           one_two_flip            localsearch.cpp:17-33, 139-190
//   MIS     build_tightness / greedy_maximalize / swap_pair_for /
//           one_two_swap            localsearch.cpp:9-15, 35-137
//
// The reference scans vertices in index order and commits every improving
// move immediately, so a move's legality depends on every earlier commit.
// Gains are built by a grid-parallel kernel.  1-flip passes are decided
// grid-parallel in rounds (a vertex's turn only depends on its lower
// neighbours' decisions; see k_flip_round).  2-flip sweeps test candidates
// grid-parallel and commit on one warp per solution that jumps from
// candidate to candidate with ballots and applies each move's neighbourhood
// update across the lanes -- identical commits in identical order.
// (1,2)-swap restarts from vertex 0 after every swap (localsearch.cpp:167-
// 199); the warp instead keeps the scanned prefix clean and re-examines
// only the 2-hop neighbourhood a swap can change ("dirty" list), which
// finds exactly the vertex the restarted scan would find.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <set>
#include <utility>

#include "common.cuh"

using namespace mqo_b200;

namespace {

constexpr int kLsWarps = 4;  // solutions per CTA (one warp each)
constexpr int64_t kSwapSmemMax = 227 * 1024;  // opt-in dynamic SMEM per CTA
// MQO_LS_SMEM=0 disables the SMEM-resident local-search variants (A/B runs)
const bool g_swap_smem = [] {
  const char* e = std::getenv("MQO_LS_SMEM");
  return !(e && *e == '0');
}();
// MQO_SWAP_CTA=0: (1,2)-swap on one warp per body (k_mis_swap)
const bool g_swap_cta = [] {
  const char* e = std::getenv("MQO_SWAP_CTA");
  return !(e && *e == '0');
}();
// 2-flip sweep look-ahead: warps per body (MQO_SCAN_CTA=8|16|32; 0 = one
// warp per body without look-ahead)
const int g_scan_cta = [] {
  const char* e = std::getenv("MQO_SCAN_CTA");
  return e ? std::atoi(e) : 16;
}();

// MQO_SCAN_MULTI=0: the 2-flip sweep commits one move per step
// (k_two_scan_cta) instead of every independent move of a window
// (k_two_scan_multi)
const bool g_scan_multi = [] {
  const char* e = std::getenv("MQO_SCAN_MULTI");
  return !(e && *e == '0');
}();

// MQO_FLIP_CLOSURE=0: the grid 1-flip passes round over every vertex and
// rebuild the gain table (A/B runs)
const bool g_flip_closure = [] {
  const char* e = std::getenv("MQO_FLIP_CLOSURE");
  return !(e && *e == '0');
}();

// lanes per candidate in the multi-commit sweep's simulation (MQO_SCAN_G =
// 8 | 16 | 32; with 32, MQO_SCAN_C picks the window).  8: BA(1e6)
// one_two_flip x 8 0.136 -> 0.131 s (scripts/ls_bench.py); the step is bound
// by its barriers after the commit phase, not by the row simulation.
const int g_scan_g = [] {
  const char* e = std::getenv("MQO_SCAN_G");
  return e && *e ? std::atoi(e) : 8;
}();
const int g_scan_c = [] {
  const char* e = std::getenv("MQO_SCAN_C");
  return e ? std::atoi(e) : 8;
}();

__device__ __forceinline__ int warp_first(unsigned mask) { return __ffs(mask) - 1; }

// ---------------------------------------------------------------- MaxCut
// build_gain_table (localsearch.cpp:17-26) for `count` solutions.
// Rows longer than kGainWarpDeg are summed by a warp each (k_gain_heavy):
// one thread walking a 3350-neighbour hub row set the table's critical path.
constexpr int64_t kGainWarpDeg = 64;

__global__ void k_gain(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr, int32_t n,
                       int32_t count, const uint8_t* __restrict__ side, int32_t* __restrict__ delta) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / n, v = q % n;
    if (off[v + 1] - off[v] > kGainWarpDeg) continue;  // k_gain_heavy
    const uint8_t* sd = side + s * n;
    const uint8_t sv = sd[v];
    int32_t same = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) same += sd[nbr[e]] == sv ? 1 : -1;
    delta[q] = same;
  }
}

// the long rows (a prefix of the degree-descending order), a warp per
// (body, row); integer sums, so the lane split does not change the value
__global__ void k_gain_heavy(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                             const int32_t* __restrict__ order, int32_t heavy, int32_t n,
                             int32_t count, const uint8_t* __restrict__ side,
                             int32_t* __restrict__ delta) {
  const int lane = threadIdx.x & 31;
  const int64_t total = static_cast<int64_t>(count) * heavy;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < total;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t s = w / heavy;
    const int32_t v = order[w - s * heavy];
    const uint8_t* sd = side + s * n;
    const uint8_t sv = sd[v];
    int32_t same = 0;
    for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) same += sd[nbr[e]] == sv ? 1 : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) same += __shfl_xor_sync(0xffffffffu, same, o);
    if (lane == 0) delta[s * n + v] = same;
  }
}

// apply_flip (localsearch.cpp:28-33) by a whole warp.
__device__ __forceinline__ void warp_flip(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                          uint8_t* side, int32_t* delta, int32_t v, int lane,
                                          int32_t& dmax) {
  int32_t local_max = INT_MIN;
  if (lane == 0) {
    side[v] ^= 1;
    delta[v] = -delta[v];
    local_max = delta[v];
  }
  __syncwarp();
  const uint8_t sv = side[v];
  for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
    const int32_t u = nbr[e];
    const int32_t nd = delta[u] + (side[u] == sv ? 2 : -2);
    delta[u] = nd;
    local_max = max(local_max, nd);
  }
  for (int o = 16; o; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  dmax = max(dmax, local_max);
  __syncwarp();
}

// ---- round-parallel one_flip_pass (localsearch.cpp:139-157) -------------
// Within a pass the reference flips v iff delta_v > 0 at v's turn.  At that
// turn the only changes to delta_v since the pass began come from flips of
// its LOWER neighbours (higher ones are scanned later): a flip of u < v adds
// c_u(v) = -2 if u and v started the pass on the same side, else +2.  So v's
// decision is fixed once its lower neighbours' are, and rounds can decide in
// parallel every vertex whose outcome interval
//   [d0_v + sum_{u flipped} c + sum_{u undecided} min(0, c),
//    d0_v + sum_{u flipped} c + sum_{u undecided} max(0, c)]
// lies entirely above 0 (flip) or at or below 0 (keep) -- exactly the
// sequential scan's decisions, typically in ~10 rounds (BA(1e6, 5)) instead
// of n dependent steps.  Decisions are final, so reading a neighbour decided
// earlier in the same round is safe; state bytes are 0 undecided, 1 keep,
// 2 flip (one byte: a reader never sees a half-written decision).
__global__ void k_flip_round(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                             const int32_t* __restrict__ lo_cnt, int32_t n, int32_t count,
                             const uint8_t* __restrict__ side_all,
                             const int32_t* __restrict__ d0_all, uint8_t* st_all,
                             const int32_t* __restrict__ live, int32_t* undecided) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / n;
    const int32_t v = static_cast<int32_t>(q - s * n);
    volatile uint8_t* st = st_all + s * n;
    if (!live[s] || st[v]) continue;
    const uint8_t* side = side_all + s * n;
    const uint8_t sv = side[v];
    int32_t base = d0_all[q], lo = 0, hi = 0;
    // rows ascend: the lower neighbours are a prefix, of known length, so
    // the walk is a counted loop with four loads in flight
    const int64_t e0 = off[v];
    const int32_t L = lo_cnt[v];
#pragma unroll 4
    for (int32_t k = 0; k < L; ++k) {
      const int32_t u = nbr[e0 + k];
      const int32_t c = side[u] == sv ? -2 : 2;
      const uint8_t su = st[u];
      if (su == 2)
        base += c;
      else if (su == 0)
        (c < 0 ? lo : hi) += c;
    }
    if (base + lo > 0)
      st[v] = 2;
    else if (base + hi <= 0)
      st[v] = 1;
    else
      undecided[s] = 1;
  }
}

// Gain of the pass: sum over flipped v of delta_v at its turn
// (d0_v + sum of c_u(v) over flipped lower neighbours), per body.
__global__ void k_flip_commit(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                              const int32_t* __restrict__ lo_cnt, int32_t n, int32_t count,
                              const uint8_t* __restrict__ side_all,
                              const int32_t* __restrict__ d0_all, const uint8_t* __restrict__ st_all,
                              const int32_t* __restrict__ live, unsigned long long* gain) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q0 = blockIdx.x * static_cast<int64_t>(blockDim.x); q0 < total;
       q0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = q0 + threadIdx.x;
    int64_t s = -1;
    int64_t g = 0;
    if (q < total) {
      s = q / n;
      const int32_t v = static_cast<int32_t>(q - s * n);
      const uint8_t* st = st_all + s * n;
      if (live[s] && st[v] == 2) {
        const uint8_t* side = side_all + s * n;
        const uint8_t sv = side[v];
        int32_t at = d0_all[q];
        const int64_t e0 = off[v];
        const int32_t L = lo_cnt[v];
#pragma unroll 4
        for (int32_t k = 0; k < L; ++k) {
          const int32_t u = nbr[e0 + k];
          if (st[u] == 2) at += side[u] == sv ? -2 : 2;
        }
        g = at;
      }
    }
    // bodies are contiguous in q: reduce runs of equal s within the warp
    const int lane = threadIdx.x & 31;
    const int64_t s0 = __shfl_sync(0xffffffffu, s, 0);
    const bool uniform = __all_sync(0xffffffffu, s == s0);
    if (uniform) {
      for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
      if (lane == 0 && g && s0 >= 0) atomicAdd(gain + s0, static_cast<unsigned long long>(g));
    } else if (g && s >= 0) {
      atomicAdd(gain + s, static_cast<unsigned long long>(g));
    }
  }
}

__global__ void k_flip_apply(int32_t n, int32_t count, uint8_t* side_all,
                             const uint8_t* __restrict__ st_all, const int32_t* __restrict__ live) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (st_all[q] == 2 && live[q / n]) side_all[q] ^= 1;
  }
}

// ---- 1-flip passes over the vertices that can flip (grid version) --------
// The closure P of cta_one_flip_closure for many large bodies: seeds are the
// positive pass-start gains, each member raises its favourable upper
// neighbours' counters, a counter crossing zero admits its vertex once; the
// rest are "keep" (st = 1) before the rounds, so a round's work is P's.  The
// gain table is then updated from the pass's flips (k_flip_update) instead of
// rebuilt.  Per body: len / fa / fb (list length, frontier [fa, fb)).
__global__ void k_flip_seed(int32_t n, int32_t count, const int32_t* __restrict__ delta_all,
                            uint8_t* st_all, int32_t* cnt_all, int32_t* list_all, int32_t* len,
                            const int32_t* __restrict__ live) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / n;
    if (!live[s]) continue;
    const int32_t d = delta_all[q];
    cnt_all[q] = d;
    if (d > 0) {
      st_all[q] = 0;
      list_all[s * n + atomicAdd(len + s, 1)] = static_cast<int32_t>(q - s * n);
    } else {
      st_all[q] = 1;
    }
  }
}

// next frontier: [fa, fb) = [fb, len)
__global__ void k_flip_front(int32_t count, const int32_t* __restrict__ len, int32_t* fa,
                             int32_t* fb) {
  for (int s = threadIdx.x; s < count; s += blockDim.x) {
    fa[s] = fb[s];
    fb[s] = len[s];
  }
}

// one closure step, a warp per frontier vertex (hub rows are long)
__global__ void k_flip_close(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                             const int32_t* __restrict__ lo_cnt, int32_t n, int32_t count,
                             const uint8_t* __restrict__ side_all, uint8_t* st_all,
                             int32_t* cnt_all, int32_t* list_all, int32_t* len,
                             const int32_t* __restrict__ fa, const int32_t* __restrict__ fb,
                             const int32_t* __restrict__ live) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int32_t s = 0; s < count; ++s) {
    if (!live[s]) continue;
    const int64_t base = int64_t(s) * n;
    const uint8_t* side = side_all + base;
    for (int64_t i = fa[s] + w0; i < fb[s]; i += nw) {
      const int32_t u = list_all[base + i];
      const uint8_t su = side[u];
      for (int64_t e = off[u] + lo_cnt[u] + lane, e1 = off[u + 1]; e < e1; e += 32) {
        const int32_t v = nbr[e];
        if (side[v] == su) continue;
        const int32_t old = atomicAdd(cnt_all + base + v, 2);
        if (old <= 0 && old > -2) {  // crossed zero: v joins P
          st_all[base + v] = 0;
          list_all[base + atomicAdd(len + s, 1)] = v;
        }
      }
    }
  }
}

// the gain table after the pass's flips (sides already applied), a warp per
// listed vertex: a flipped row recomputed, its unflipped neighbours +-2
// (apply_flip, localsearch.cpp:28-33)
__global__ void k_flip_update(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                              int32_t n, int32_t count, const uint8_t* __restrict__ side_all,
                              const uint8_t* __restrict__ st_all, int32_t* delta_all,
                              const int32_t* __restrict__ list_all, const int32_t* __restrict__ len,
                              const int32_t* __restrict__ live) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int32_t s = 0; s < count; ++s) {
    if (!live[s]) continue;
    const int64_t base = int64_t(s) * n;
    const uint8_t* side = side_all + base;
    const uint8_t* st = st_all + base;
    for (int64_t i = w0; i < len[s]; i += nw) {
      const int32_t v = list_all[base + i];
      if (st[v] != 2) continue;  // warp-uniform
      const uint8_t sv = side[v];
      int32_t same = 0;
      for (int64_t e = off[v] + lane, e1 = off[v + 1]; e < e1; e += 32) {
        const int32_t u = nbr[e];
        const bool eq = side[u] == sv;
        same += eq ? 1 : -1;
        if (st[u] != 2) atomicAdd(delta_all + base + u, eq ? 2 : -2);
      }
      for (int o = 16; o; o >>= 1) same += __shfl_xor_sync(0xffffffffu, same, o);
      if (lane == 0) delta_all[base + v] = same;
    }
  }
}

// ---- one_flip_pass in one CTA per body (small graphs) -------------------
// The round-parallel pass above, with side / pass-start gains / decision
// bytes of one body in shared memory (6n bytes), every round separated by a
// CTA barrier instead of a kernel launch and a host round trip, and the
// passes repeated inside the kernel until one flips nothing
// (localsearch.cpp:139-157).  Leaves side and the gain table of the final
// state in global memory (one_two_flip's 2-flip sweep reads it).
constexpr int kFlipCtaThreads = 1024;
constexpr int64_t kFlipCtaSmemMax = 226 * 1024;  // + static SMEM stays under the 227 KB cap
// d0 [n] int32, lo [n] int32 (lower-neighbour count per row), side [n], decision [n]
__host__ __device__ inline int64_t flip_cta_smem(int32_t n) { return (10 * int64_t(n) + 15) / 16 * 16; }
__host__ __device__ inline int64_t flip_cta_smem_csr(int32_t n, int64_t nnz) {
  return flip_cta_smem(n) + (8 * (int64_t(n) + 1) + 15) / 16 * 16 + 4 * nnz;
}

// one CTA per body: when the body state fits SMEM, and the graph is small or
// there are enough bodies to spread over the SMs (one large body runs faster
// on the grid-wide rounds)
inline bool one_flip_cta_fits(int32_t n, int32_t count) {
  return g_swap_smem && flip_cta_smem(n) <= kFlipCtaSmemMax && (n <= 8192 || count >= 16);
}

// one_flip_pass (localsearch.cpp:139-157) as CTA decision rounds on the
// SMEM state of one body: sd[n] sides (in/out), lo_cnt[n] (lower-neighbour
// counts, built here), d0[n] (left = the gain table of the final state),
// st[n] decision bytes.  Returns the gain (the same on every thread).
__device__ long long cta_one_flip_pass(const int64_t* off, const int32_t* nbr, int32_t n,
                                       uint8_t* sd, int32_t* d0, int32_t* lo_cnt,
                                       volatile uint8_t* st) {
  __shared__ long long s_part[32];
  // lower neighbours are a row prefix (rows ascend): their count, so the
  // round and commit walks below are counted loops the compiler can unroll
  // (independent loads in flight) instead of break-terminated chains
  for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
    int64_t a = off[v], b = off[v + 1];
    const int64_t e0 = a;
    while (a < b) {  // first entry >= v
      const int64_t mid = (a + b) >> 1;
      if (nbr[mid] < v) a = mid + 1; else b = mid;
    }
    lo_cnt[v] = static_cast<int32_t>(a - e0);
  }
  __syncthreads();
  long long total = 0;
  for (;;) {
    // build_gain_table (localsearch.cpp:17-26) of the pass-start sides
    for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
      const uint8_t sv = sd[v];
      int32_t same = 0;
      const int64_t e0 = off[v];
      const int32_t deg = static_cast<int32_t>(off[v + 1] - e0);
#pragma unroll 4
      for (int32_t k = 0; k < deg; ++k) same += sd[nbr[e0 + k]] == sv ? 1 : -1;
      d0[v] = same;
      st[v] = 0;
    }
    __syncthreads();
    // decision rounds (k_flip_round)
    for (;;) {
      int und = 0;
      for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
        if (st[v]) continue;
        const uint8_t sv = sd[v];
        int32_t base = d0[v], lo = 0, hi = 0;
        const int64_t e0 = off[v];
        const int32_t L = lo_cnt[v];
#pragma unroll 4
        for (int32_t k = 0; k < L; ++k) {
          const int32_t u = nbr[e0 + k];
          const int32_t c = sd[u] == sv ? -2 : 2;
          const uint8_t su = st[u];
          if (su == 2)
            base += c;
          else if (su == 0)
            (c < 0 ? lo : hi) += c;
        }
        if (base + lo > 0)
          st[v] = 2;
        else if (base + hi <= 0)
          st[v] = 1;
        else
          und = 1;
      }
      if (!__syncthreads_or(und)) break;
    }
    // the pass's gain (k_flip_commit), then apply its flips
    long long g = 0;
    int flips = 0;
    for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
      if (st[v] != 2) continue;
      ++flips;
      const uint8_t sv = sd[v];
      int32_t at = d0[v];
      const int64_t e0 = off[v];
      const int32_t L = lo_cnt[v];
#pragma unroll 4
      for (int32_t k = 0; k < L; ++k) {
        const int32_t u = nbr[e0 + k];
        if (st[u] == 2) at += sd[u] == sv ? -2 : 2;
      }
      g += at;
    }
    // warp sums, then one partial per warp (a 64-bit shared atomicAdd is a
    // CAS loop: 1024 contending threads serialised the pass)
    for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = g;
    const bool any = __syncthreads_or(flips) != 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total += s_part[w];
    for (int32_t v = threadIdx.x; v < n; v += blockDim.x)
      if (st[v] == 2) sd[v] ^= 1;
    __syncthreads();
    if (!any) break;  // a pass without a flip ends one_flip_pass
  }
  return total;
}

// `csr`: the CSR is staged in shared memory too (it fits next to the body
// state); every row walk is then ~30-cycle SMEM loads instead of L2 trips.
// CSR as a template parameter: the row walks then compile to LDS instead of
// generic loads.
template <bool CSR>
__global__ void __launch_bounds__(kFlipCtaThreads, 1)
    k_one_flip_cta(const int64_t* __restrict__ off_g, const int32_t* __restrict__ nbr_g, int32_t n,
                   uint8_t* side_all, int32_t* delta_all, const int32_t* __restrict__ live,
                   int64_t* __restrict__ gains) {
  extern __shared__ __align__(16) unsigned char sm[];
  int32_t* d0 = reinterpret_cast<int32_t*>(sm);
  int32_t* lo_cnt = d0 + n;
  uint8_t* sd = sm + 8 * int64_t(n);
  volatile uint8_t* st = sd + n;
  int64_t* o = reinterpret_cast<int64_t*>(sm + flip_cta_smem(n));
  int32_t* nb = reinterpret_cast<int32_t*>(sm + flip_cta_smem(n) + (8 * (int64_t(n) + 1) + 15) / 16 * 16);
  const int64_t* off = CSR ? o : off_g;
  const int32_t* nbr = CSR ? nb : nbr_g;
  // live == nullptr: every body is live
  if (CSR && (!live || live[blockIdx.x])) {
    const int64_t nnz = off_g[n];
    for (int64_t i = threadIdx.x; i <= n; i += blockDim.x) o[i] = off_g[i];
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < nnz; i += blockDim.x) nb[i] = nbr_g[i];
  }
  const int s = blockIdx.x;
  uint8_t* side = side_all + int64_t(s) * n;
  int32_t* delta = delta_all + int64_t(s) * n;
  if (live && !live[s]) {
    if (threadIdx.x == 0) gains[s] = 0;
    return;
  }
  __syncthreads();  // CSR staged
  for (int32_t v = threadIdx.x; v < n; v += blockDim.x) sd[v] = side[v];
  __syncthreads();
  const long long total = cta_one_flip_pass(off, nbr, n, sd, d0, lo_cnt, st);
  // write back the sides and the gain table of the final state (after the
  // last pass flipped nothing, d0 is that table)
  for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
    side[v] = sd[v];
    delta[v] = d0[v];
  }
  if (threadIdx.x == 0) gains[s] = total;
}

// Once per device (the attribute is per device and context; setting it to
// the cap on every call cost two driver calls per one_flip_pass).
void set_flip_cta_smem_attr() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  MQO_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && done[dev]) return;
  MQO_CUDA(cudaFuncSetAttribute(k_one_flip_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kFlipCtaSmemMax)));
  MQO_CUDA(cudaFuncSetAttribute(k_one_flip_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kFlipCtaSmemMax)));
  if (dev < 64) done[dev] = true;
}

// ---- host-driven 2-flip sweeps (localsearch.cpp:159-181) --------------
// cand(v) = exists u in N(v), u > v, opposite side, delta_v + delta_u + 2 > 0:
// the exact "v acts in this sweep if nothing before it changes" test,
// computed for every vertex of every body in one grid pass.  The warp then
// visits candidates only.  A joint flip of (v, u) can change cand(w) for a
// later vertex w only if delta or side changed at some y in
// Z = {v,u} U N(v) U N(u) with y = w or y in N(w), y > w -- those w > v are
// re-marked (a superset, resolved by the exact evaluation at the visit).
// (Resolving a chunk's marks lane-parallel and re-evaluating exactly at
// marking time were both tried: slower, as each lane then walks rows
// serially.)
// hmax[v] = the largest degree among v's higher neighbours bounds delta_u
// (delta_u <= deg u), so delta_v + hmax[v] + 2 <= 0 rules v out without
// reading its row -- hubs of a locally optimal cut are skipped in O(1).
__device__ __forceinline__ bool two_cand(const int64_t* __restrict__ off,
                                         const int32_t* __restrict__ nbr, const int32_t* hmax,
                                         const uint8_t* side, const int32_t* delta, int32_t v) {
  const int32_t dv = *reinterpret_cast<const volatile int32_t*>(delta + v);
  if (dv + hmax[v] + 2 <= 0) return false;
  const uint8_t sv = *reinterpret_cast<const volatile uint8_t*>(side + v);
  for (int64_t e = off[v + 1] - 1, e0 = off[v]; e >= e0; --e) {  // u > v lie at the row's end
    const int32_t u = nbr[e];
    if (u <= v) break;
    if (*reinterpret_cast<const volatile uint8_t*>(side + u) != sv &&
        dv + *reinterpret_cast<const volatile int32_t*>(delta + u) + 2 > 0)
      return true;
  }
  return false;
}

// Rows longer than this are tested by a whole warp (k_two_cand_heavy): a
// thread walking a hub's 3350 upper neighbours one dependent load at a time
// took milliseconds and set the sweep's critical path.
constexpr int64_t kCandWarpDeg = 64;

__global__ void k_two_cand(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                           const int32_t* __restrict__ hmax, int32_t n, int32_t count,
                           const uint8_t* __restrict__ side_all, const int32_t* __restrict__ delta_all,
                           const int32_t* __restrict__ live, uint8_t* __restrict__ cand_all,
                           const uint8_t* __restrict__ mask_all) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / n;
    const int32_t v = static_cast<int32_t>(q - s * n);
    if (!live[s]) continue;
    // mask (may be null): only vertices the last sweep's commits touched can
    // have become candidates; the rest keep their "no move" (tested before
    // the row is read; k_two_cand_heavy, launched after, rewrites long rows)
    if (mask_all && !mask_all[q]) {
      cand_all[q] = 0;
      continue;
    }
    if (off[v + 1] - off[v] > kCandWarpDeg) continue;  // k_two_cand_heavy
    cand_all[q] = two_cand(off, nbr, hmax, side_all + s * n, delta_all + s * n, v) ? 1 : 0;
  }
}

// The long rows (a prefix of the degree-descending order): a warp per
// (body, row), lanes over the upper neighbours.
__global__ void k_two_cand_heavy(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                 const int32_t* __restrict__ hmax,
                                 const int32_t* __restrict__ order, int32_t heavy, int32_t n,
                                 int32_t count, const uint8_t* __restrict__ side_all,
                                 const int32_t* __restrict__ delta_all,
                                 const int32_t* __restrict__ live, uint8_t* __restrict__ cand_all,
                                 const uint8_t* __restrict__ mask_all) {
  const int lane = threadIdx.x & 31;
  const int64_t total = static_cast<int64_t>(count) * heavy;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < total;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t s = w / heavy;
    if (!live[s]) continue;
    const int32_t v = order[w - s * heavy];
    const uint8_t* side = side_all + s * n;
    const int32_t* delta = delta_all + s * n;
    const int32_t dv = delta[v];
    bool found = false;
    if ((!mask_all || mask_all[s * n + v]) && dv + hmax[v] + 2 > 0) {  // uniform per warp
      const uint8_t sv = side[v];
      const int64_t e0 = off[v], e1 = off[v + 1];
      for (int64_t top = e1 - 1; top >= e0; top -= 32) {  // u > v lie at the row's end
        const int64_t e = top - lane;
        const int32_t u = e >= e0 ? nbr[e] : -1;
        const bool ok = u > v && side[u] != sv && dv + delta[u] + 2 > 0;
        found = __any_sync(0xffffffffu, ok);
        if (found || __all_sync(0xffffffffu, u <= v)) break;
      }
    }
    if (lane == 0) cand_all[s * n + v] = found ? 1 : 0;
  }
}

// hmax (above), once per graph; rows longer than 64 by k_hmax_heavy
__global__ void k_hmax_heavy(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                             const int32_t* __restrict__ order, int32_t heavy,
                             int32_t* __restrict__ hmax) {
  const int lane = threadIdx.x & 31;
  for (int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; w < heavy;
       w += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int32_t v = order[w];
    int32_t h = 0;
    for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
      const int32_t u = nbr[e];
      if (u > v) h = max(h, static_cast<int32_t>(off[u + 1] - off[u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h = max(h, __shfl_xor_sync(0xffffffffu, h, o));
    if (lane == 0) hmax[v] = h;
  }
}

__global__ void k_hmax(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr, int32_t n,
                       int32_t* __restrict__ hmax) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (off[v + 1] - off[v] > 64) continue;  // k_hmax_heavy
    int32_t h = 0;
    for (int64_t e = off[v + 1] - 1, e0 = off[v]; e >= e0; --e) {
      const int32_t u = nbr[e];
      if (u <= v) break;
      h = max(h, static_cast<int32_t>(off[u + 1] - off[u]));
    }
    hmax[v] = h;
  }
}

__device__ void warp_mark_after_flip(const int64_t* off, const int32_t* nbr, uint8_t* cand,
                                     int32_t t, int32_t v, int lane) {
  // y over {t} U N(t); mark y and its smaller neighbours w (w > v only)
  const int64_t e0 = off[t], e1 = off[t + 1];
  for (int64_t a = e0 - 1 + lane; a < e1; a += 32) {
    const int32_t y = a < e0 ? t : nbr[a];
    if (y > v) cand[y] = 1;
    for (int64_t c = off[y]; c < off[y + 1]; ++c) {
      const int32_t w = nbr[c];
      if (w >= y) break;  // rows ascending: only w < y
      if (w > v) cand[w] = 1;
    }
  }
  __syncwarp();
}

__global__ void k_two_scan(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                           const int32_t* __restrict__ hmax, int32_t n, int32_t count, uint8_t* side_all, int32_t* delta_all,
                           uint8_t* cand_all, int32_t* live, int64_t* gains) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * kLsWarps + (threadIdx.x >> 5);
  if (s >= count || !live[s]) return;
  uint8_t* side = side_all + static_cast<int64_t>(s) * n;
  int32_t* delta = delta_all + static_cast<int64_t>(s) * n;
  uint8_t* cand = cand_all + static_cast<int64_t>(s) * n;
  int64_t total = 0;
  int32_t dmax = INT_MIN;  // unused bound for warp_flip
  for (int32_t sb = 0; sb < n; sb += 512) {
    // 512 marks per warp step (16 independent byte loads per lane; a body's
    // marks need not be aligned): empty stretches cost one round trip
    bool any16 = false;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int32_t q = sb + 16 * lane + k;
      any16 |= q < n && *reinterpret_cast<const volatile uint8_t*>(cand + q) != 0;
    }
    if (!__any_sync(0xffffffffu, any16)) continue;
    for (int32_t cb = sb; cb < min(n, sb + 512); cb += 32) {
      bool f = cb + lane < n && *reinterpret_cast<volatile uint8_t*>(cand + cb + lane);
      unsigned mask = __ballot_sync(0xffffffffu, f);
      while (mask) {
        const int i = warp_first(mask);
        const int32_t v = cb + i;
        const int64_t e1 = off[v + 1];
        int64_t e = off[v];
        // delta_u <= hmax[v] for every higher neighbour u: skip hopeless rows
        if (*reinterpret_cast<volatile int32_t*>(delta + v) + hmax[v] + 2 <= 0) e = e1;
        while (e < e1) {
          const int64_t my = e + lane;
          bool ok = false;
          int32_t u = 0, joint = 0;
          if (my < e1) {
            u = nbr[my];
            const uint8_t sv = *reinterpret_cast<volatile uint8_t*>(side + v);
            if (u > v && *reinterpret_cast<volatile uint8_t*>(side + u) != sv) {
              joint = *reinterpret_cast<volatile int32_t*>(delta + v) +
                      *reinterpret_cast<volatile int32_t*>(delta + u) + 2;
              ok = joint > 0;
            }
          }
          const unsigned hit = __ballot_sync(0xffffffffu, ok);
          if (!hit) {
            e += 32;
            continue;
          }
          const int j = warp_first(hit);
          const int32_t uu = __shfl_sync(0xffffffffu, u, j);
          const int32_t jj = __shfl_sync(0xffffffffu, joint, j);
          warp_flip(off, nbr, side, delta, v, lane, dmax);
          warp_flip(off, nbr, side, delta, uu, lane, dmax);
          total += jj;
          warp_mark_after_flip(off, nbr, cand, v, v, lane);
          warp_mark_after_flip(off, nbr, cand, uu, v, lane);
          e += j + 1;
        }
        f = cb + lane < n && *reinterpret_cast<volatile uint8_t*>(cand + cb + lane);
        mask = __ballot_sync(0xffffffffu, f) & (i == 31 ? 0u : (~0u << (i + 1)));
      }
    }
  }
  if (lane == 0) {
    gains[s] += total;
    live[s] = total > 0 ? 1 : 0;  // improved: sweep again
  }
}


// The same sweep with speculative look-ahead: a CTA of kScanWarps warps per
// body.  Warp 0 collects the next kScanWarps candidates in scan order (the
// current vertex, resumed after its last joint flip, then the following
// marked vertices); warp k evaluates candidate k against the current state
// -- the first u in its row with opposite side and delta_v + delta_u + 2 > 0
// -- all in parallel; then the first candidate with a hit is committed and
// the batch ends there.  Every candidate before it saw exactly the state the
// sequential scan would have shown it (nothing was committed in between), so
// the commits and their order are the reference's; the serial chain of
// dependent loads is paid once per batch instead of once per candidate.
// apply_flip (localsearch.cpp:28-33) by a whole CTA; ends with a barrier.
__device__ __forceinline__ void cta_flip(const int64_t* __restrict__ off,
                                         const int32_t* __restrict__ nbr, uint8_t* side,
                                         int32_t* delta, int32_t v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    side[v] ^= 1;
    delta[v] = -delta[v];
  }
  __syncthreads();
  const uint8_t sv = side[v];
  for (int64_t e = off[v] + threadIdx.x, e1 = off[v + 1]; e < e1; e += blockDim.x) {
    const int32_t u = nbr[e];
    delta[u] += side[u] == sv ? 2 : -2;
  }
  __syncthreads();
}

// warp_mark_after_flip by a whole CTA: warps over y in {t} U N(t), lanes
// over y's lower neighbours w (marks y and w when > v).
__device__ __forceinline__ void cta_mark_after_flip(const int64_t* off, const int32_t* nbr,
                                                    uint8_t* cand, int32_t t, int32_t v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t e0 = off[t], e1 = off[t + 1];
  for (int64_t a = e0 - 1 + warp; a < e1; a += nw) {
    const int32_t y = a < e0 ? t : nbr[a];
    if (lane == 0 && y > v) cand[y] = 1;
    for (int64_t c = off[y] + lane, c1 = off[y + 1]; c < c1; c += 32) {
      const int32_t w = nbr[c];
      if (w >= y) break;  // rows ascending: only w < y
      if (w > v) cand[w] = 1;
    }
  }
}

template <int kScanWarps>
__global__ void __launch_bounds__(32 * kScanWarps)
    k_two_scan_cta(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                   const int32_t* __restrict__ hmax, int32_t n, int32_t count, uint8_t* side_all,
                   int32_t* delta_all, uint8_t* cand_all, int32_t* live, int64_t* gains) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = blockIdx.x;
  if (s >= count || !live[s]) return;
  uint8_t* side = side_all + static_cast<int64_t>(s) * n;
  int32_t* delta = delta_all + static_cast<int64_t>(s) * n;
  uint8_t* cand = cand_all + static_cast<int64_t>(s) * n;
  __shared__ int32_t c_v[kScanWarps], r_u[kScanWarps], r_joint[kScanWarps];
  __shared__ int64_t c_e0[kScanWarps], r_e[kScanWarps];
  __shared__ int32_t s_k, s_pos;
  __shared__ int64_t s_epos;
  int64_t total = 0;
  if (threadIdx.x == 0) {
    s_pos = 0;
    s_epos = -1;
  }
  __syncthreads();
  for (;;) {
    // A. collect the batch (warp 0)
    if (warp == 0) {
      int k = 0;
      int32_t from = s_pos;
      if (s_epos >= 0) {  // resume the current vertex's row
        if (lane == 0) {
          c_v[0] = s_pos;
          c_e0[0] = s_epos;
        }
        k = 1;
        from = s_pos + 1;
      }
      for (int32_t cb = from; cb < n && k < kScanWarps; cb += 32) {
        if (((cb - from) & 511) == 0) {  // empty 512-mark stretches cost one round trip
          bool any16 = false;
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int32_t q = cb + 16 * lane + t;
            any16 |= q < n && *reinterpret_cast<const volatile uint8_t*>(cand + q) != 0;
          }
          if (!__any_sync(0xffffffffu, any16)) {
            cb += 512 - 32;
            continue;
          }
        }
        const bool f = cb + lane < n && *reinterpret_cast<volatile uint8_t*>(cand + cb + lane);
        unsigned mask = __ballot_sync(0xffffffffu, f);
        while (mask && k < kScanWarps) {
          const int i = warp_first(mask);
          if (lane == 0) {
            c_v[k] = cb + i;
            c_e0[k] = -1;
          }
          ++k;
          mask &= mask - 1;
        }
      }
      if (lane == 0) s_k = k;
    }
    __syncthreads();
    const int K = s_k;
    if (K == 0) break;
    // B. evaluate candidate `warp` against the current state (read only)
    if (warp < K) {
      const int32_t v = c_v[warp];
      const int64_t e1 = off[v + 1];
      int64_t e = c_e0[warp] >= 0 ? c_e0[warp] : off[v];
      const int32_t dv = delta[v];
      const uint8_t sv = side[v];
      int32_t hit_u = -1, hit_j = 0;
      int64_t hit_e = -1;
      if (dv + hmax[v] + 2 <= 0) e = e1;  // delta_u <= hmax[v] for every higher u
      while (e < e1) {
        const int64_t my = e + lane;
        bool ok = false;
        int32_t u = 0, joint = 0;
        if (my < e1) {
          u = nbr[my];
          if (u > v && side[u] != sv) {
            joint = dv + delta[u] + 2;
            ok = joint > 0;
          }
        }
        const unsigned hit = __ballot_sync(0xffffffffu, ok);
        if (hit) {
          const int j = warp_first(hit);
          hit_u = __shfl_sync(0xffffffffu, u, j);
          hit_j = __shfl_sync(0xffffffffu, joint, j);
          hit_e = e + j;
          break;
        }
        e += 32;
      }
      if (lane == 0) {
        r_u[warp] = hit_u;
        r_joint[warp] = hit_j;
        r_e[warp] = hit_e;
      }
    }
    __syncthreads();
    // C. commit the first hit with the whole CTA, advance
    int first = -1;
    for (int k = 0; k < K; ++k)
      if (r_u[k] >= 0) {
        first = k;
        break;
      }
    if (first < 0) {
      if (threadIdx.x == 0) {
        s_pos = c_v[K - 1] + 1;
        s_epos = -1;
      }
    } else {
      const int32_t v = c_v[first], u = r_u[first];
      const int64_t ehit = r_e[first];
      total += r_joint[first];
      cta_flip(off, nbr, side, delta, v);
      cta_flip(off, nbr, side, delta, u);
      cta_mark_after_flip(off, nbr, cand, v, v);
      cta_mark_after_flip(off, nbr, cand, u, v);
      __syncthreads();
      if (threadIdx.x == 0) {
        s_pos = v;
        s_epos = ehit + 1;
      }
    }
    __syncthreads();
    if (s_pos >= n) break;
  }
  if (threadIdx.x == 0) {
    gains[s] += total;
    live[s] = total > 0 ? 1 : 0;  // improved: sweep again
  }
}

// ---- 2-flip sweep with many commits per step ---------------------------
// The reference scan (localsearch.cpp:159-181) visits v ascending and, for
// each u in N(v), u > v, on the other side with delta_v + delta_u + 2 > 0,
// flips both at once and carries on along v's row with the new state.  What
// the decision at vertex w reads is R(w) = {w} U {u in N(w): u > w} (side
// and delta of each); a joint flip of v with partners F changes sides in
// {v} U F and deltas in C = {v} U F U N(v) U N(F), so it can change the
// decision at w only if R(w) meets C, i.e. w in C or w a lower neighbour of
// some y in C.  Let m(v) be the smallest such w above v.
//
// A CTA per body takes K marked vertices at a time and every warp
// simulates whole rows of its candidates against the current state --
// including the row's later hits after v has flipped (delta of a later u
// shifts by +-2 for every flip of v and of each partner adjacent to u) --
// and computes m(v) for rows with a hit.  The sequential scan would then
// reach candidate k in exactly the state the snapshot shows as long as
// c_k < M = min m over the hits committed before it; so every hit below M
// is committed in one step (their flipped sets are pairwise non-adjacent,
// the shared neighbours' delta updates commute), and the next step starts
// at M (or after the window).  Commits, their order and the gain are the
// reference's; what changes is that a step commits every independent hit of
// the window instead of one.
constexpr int kMultiMaxFlips = 8;  // partners simulated per row and step

// first index in the sorted row [b, e) holding a value > x
__device__ __forceinline__ int64_t row_upper(const int32_t* __restrict__ nbr, int64_t b,
                                             int64_t e, int32_t x) {
  while (b < e) {
    const int64_t mid = (b + e) >> 1;
    if (nbr[mid] <= x) b = mid + 1; else e = mid;
  }
  return b;
}

__device__ __forceinline__ bool row_has(const int32_t* __restrict__ nbr, int64_t b, int64_t e,
                                        int32_t x) {
  const int64_t i = row_upper(nbr, b, e, x - 1);
  return i < e && nbr[i] == x;
}

// min over y in {t} U N(t), y > v, of y and of the smallest lower neighbour
// w of y with v < w < y (this lane's share; the caller reduces).  A smaller
// value is always safe (the step just stops earlier), so rows longer than
// kMultiScanRow -- hubs, whose 2-hop walk would stall the whole step --
// answer v + 1.
constexpr int64_t kMultiScanRow = 256;
template <int G = 32>
__device__ __forceinline__ int32_t affected_min(const int64_t* __restrict__ off,
                                                const int32_t* __restrict__ nbr, int32_t t,
                                                int32_t v, int lane) {
  int32_t m = INT_MAX;
  const int64_t e0 = off[t], e1 = off[t + 1];
  if (e1 - e0 > kMultiScanRow) return v + 1;
  for (int64_t a = e0 - 1 + lane; a < e1; a += G) {
    const int32_t y = a < e0 ? t : nbr[a];
    if (y <= v) continue;
    m = min(m, y);
    const int64_t yb = off[y], ye = off[y + 1];
    const int64_t i = row_upper(nbr, yb, ye, v);
    if (i < ye && nbr[i] < y) m = min(m, nbr[i]);
  }
  return m;
}

// warp_mark_after_flip that also records every affected position -- above
// and below v -- in `next`: the next sweep's candidates (a vertex whose read
// set no commit touched after its turn keeps the "no move" it had)
__device__ void warp_mark_after_flip2(const int64_t* off, const int32_t* nbr, uint8_t* cand,
                                      uint8_t* next, int32_t t, int32_t v, int lane) {
  const int64_t e0 = off[t], e1 = off[t + 1];
  for (int64_t a = e0 - 1 + lane; a < e1; a += 32) {
    const int32_t y = a < e0 ? t : nbr[a];
    if (y > v) cand[y] = 1;
    next[y] = 1;
    // y's lower neighbours (a row prefix: rows ascend), four loads in
    // flight instead of one load per step of a break-terminated chain
    for (int64_t c = off[y], c1 = off[y + 1]; c < c1; c += 4) {
      int32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = c + q < c1 ? nbr[c + q] : INT_MAX;
      bool stop = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (w[q] < y) {
          if (w[q] > v) cand[w[q]] = 1;
          next[w[q]] = 1;
        } else {
          stop = true;
        }
      }
      if (stop) break;
    }
  }
  __syncwarp();
}

template <int NW, int C, int G>
__global__ void __launch_bounds__(32 * NW, 1)
    k_two_scan_multi(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                     const int32_t* __restrict__ hmax, int32_t n, int32_t count,
                     uint8_t* side_all, int32_t* delta_all, uint8_t* cand_all,
                     uint8_t* next_all, int32_t* live, int64_t* gains, int64_t* stats) {
  constexpr int K = NW * C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = blockIdx.x;
  if (s >= count || !live[s]) return;
  uint8_t* side = side_all + static_cast<int64_t>(s) * n;
  int32_t* delta = delta_all + static_cast<int64_t>(s) * n;
  uint8_t* cand = cand_all + static_cast<int64_t>(s) * n;
  uint8_t* next_marks = next_all + static_cast<int64_t>(s) * n;
  __shared__ int32_t c_v[K];
  __shared__ int64_t c_e[K];                 // row start (resumed rows: after the last flip)
  __shared__ int32_t r_m[K], r_gain[K], r_nf[K];
  __shared__ int64_t r_resume[K];            // >= 0: row not finished (too many flips)
  __shared__ int32_t r_part[K][kMultiMaxFlips];
  __shared__ uint8_t r_commit[K];
  __shared__ int32_t s_k, s_pos, s_span;
  __shared__ int64_t s_epos;
  __shared__ long long s_total;
  __shared__ int32_t w_cnt[NW], w_tot;
  __shared__ int32_t s_steps, s_commits;
  __shared__ long long s_cyc[4];  // MQO_TRACE: cycles in phases A-D
  // per-group simulation scratch: partner rows [pb, pe) and sides after flip
  constexpr int GPW = 32 / G;  // candidate groups per warp
  __shared__ int64_t w_pb[NW * GPW][kMultiMaxFlips], w_pe[NW * GPW][kMultiMaxFlips];
  __shared__ uint8_t w_pside[NW * GPW][kMultiMaxFlips];
  if (threadIdx.x == 0) {
    s_pos = 0;
    s_epos = -1;
    s_total = 0;
    s_steps = 0;
    s_commits = 0;
    s_cyc[0] = s_cyc[1] = s_cyc[2] = s_cyc[3] = 0;
  }
  __syncthreads();
  for (;;) {
    long long t_a = clock64();
    // A. the next K marked vertices from s_pos, collected by the whole CTA:
    // warp w scans 1024 positions (32 per lane), per-lane masks, warp and
    // CTA prefix counts, positions written in order; s_span = last
    // position examined
    if (threadIdx.x == 0) {
      s_k = 0;
      s_span = n - 1;
      if (s_epos >= 0) {  // resume the current vertex's row first
        c_v[0] = s_pos;
        c_e[0] = s_epos;
        s_k = 1;
      }
    }
    __syncthreads();
    const int32_t start = s_epos >= 0 ? s_pos + 1 : s_pos;
    // 16-byte aligned windows (the body's marks need not be aligned)
    const int32_t skew = static_cast<int32_t>(reinterpret_cast<uintptr_t>(cand + start) & 15);
    for (int32_t from = start - skew; from < n; from += NW * 1024) {
      const int32_t base = from + warp * 1024 + lane * 32;
      unsigned bits = 0;
      if (base < n) {
        const uint4 w0 = __ldcg(reinterpret_cast<const uint4*>(cand + base));
        const uint4 w1 = __ldcg(reinterpret_cast<const uint4*>(cand + base) + 1);
        const uint32_t wd[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if ((wd[t >> 2] >> (8 * (t & 3))) & 0xffu) bits |= 1u << t;
        // positions outside [start, n)
        if (base < start) bits &= start - base >= 32 ? 0u : ~0u << (start - base);
        if (base + 32 > n) bits &= n - base >= 32 ? ~0u : (1u << (n - base)) - 1u;
      }
      const int cnt = __popc(bits);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) w_cnt[warp] = incl;
      __syncthreads();
      if (warp == 0) {  // exclusive prefix over the warps
        int c = lane < NW ? w_cnt[lane] : 0, pre = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += t;
        }
        if (lane < NW) w_cnt[lane] = pre - c;
        if (lane == 31) w_tot = pre;
      }
      __syncthreads();
      const int k0 = s_k;
      int k = k0 + w_cnt[warp] + incl - cnt;
      while (bits && k < K) {
        const int t = __ffs(bits) - 1;
        bits &= bits - 1;
        c_v[k] = base + t;
        c_e[k] = -1;
        if (k == K - 1) s_span = base + t;
        ++k;
      }
      __syncthreads();
      const int total = w_tot;
      if (threadIdx.x == 0) s_k = min(K, k0 + total);
      __syncthreads();
      if (s_k >= K) break;
    }
    __syncthreads();
    const int Kc = s_k;
    if (Kc == 0) break;
    long long t_b = clock64();
    // B. simulate each candidate's row against the current state (read
    // only): a candidate per G-lane group, 32/G groups of a warp side by side
    // (rows are mostly short, and each candidate is a chain of dependent L2
    // trips: candidates in parallel, not lanes idling on one row)
    {
      const int grp = lane / G, gl = lane % G;
      const int gid = warp * GPW + grp;
      const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << (grp * G);
      for (int kb = warp * GPW; kb < Kc; kb += NW * GPW) {  // warp-uniform
        const int k = kb + grp;
        const bool valid = k < Kc;
        int32_t v = 0, dv = 0, gain = 0;
        int64_t e = 0, e1 = 0, resume = -1;
        uint8_t sv = 0;
        int nf = 0, flips_v = 0;
        bool done = !valid;
        int32_t* part = r_part[valid ? k : 0];  // partners (SMEM: indexed at run time)
        if (valid) {
          v = c_v[k];
          e1 = off[v + 1];
          const bool resumed = c_e[k] >= 0;
          e = resumed ? c_e[k] : off[v];
          dv = delta[v];
          sv = side[v];
          if (!resumed && dv + hmax[v] + 2 <= 0) e = e1;  // delta_u <= hmax[v]: no hit in the row
        }
        for (;;) {
          const bool act = !done && e < e1;
          if (!__any_sync(0xffffffffu, act)) break;
          const int64_t my = e + gl;
          bool ok = false;
          int32_t u = -1, du = 0;
          if (act && my < e1) {
            u = nbr[my];
            if (u > v) {
              const uint8_t su = side[u];
              if (su != sv) {
                du = delta[u];
                // v flipped an odd number of times: the net +-2 of its flips
                if (flips_v & 1) du += su == sv ? 2 : -2;
                for (int f = 0; f < nf; ++f)
                  if (row_has(nbr, w_pb[gid][f], w_pe[gid][f], u))
                    du += su == w_pside[gid][f] ? 2 : -2;
                ok = dv + du + 2 > 0;
              }
            }
          }
          const unsigned hit = __ballot_sync(0xffffffffu, ok) & gmask;
          const int j = hit ? __ffs(hit) - 1 : grp * G;  // lane of the group's first hit
          const int32_t uh = __shfl_sync(0xffffffffu, u, j);
          const int32_t dh = __shfl_sync(0xffffffffu, du, j);
          if (act) {
            if (!hit) {
              e += G;
            } else if (nf == kMultiMaxFlips) {  // partner list full: finish the row next step
              resume = e + (j - grp * G);
              done = true;
            } else {
              gain += dv + dh + 2;
              // apply_flip(v), then apply_flip(uh) as seen from v (localsearch.cpp:28-33)
              sv ^= 1;
              dv = -dv;
              ++flips_v;
              const uint8_t su_new = side[uh] ^ 1;
              dv += sv == su_new ? 2 : -2;
              if (gl == 0) {
                part[nf] = uh;
                w_pside[gid][nf] = su_new;
                w_pb[gid][nf] = off[uh];
                w_pe[gid][nf] = off[uh + 1];
              }
              ++nf;
              e = e + (j - grp * G) + 1;
            }
          }
          __syncwarp();
        }
        // m(v): smallest position above v whose decision the flips can change
        int32_t m = INT_MAX;
        if (valid && nf > 0) {
          m = affected_min<G>(off, nbr, v, v, gl);
          for (int f = 0; f < nf; ++f) m = min(m, affected_min<G>(off, nbr, part[f], v, gl));
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (valid && gl == 0) {
          r_m[k] = m;
          r_gain[k] = gain;
          r_nf[k] = nf;
          r_resume[k] = resume;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    long long t_c = clock64();
    // C. commit every hit below M (warp 0; lane l owns candidates
    // [l*L, l*L + L)): a scan of the lanes' minima of m gives each lane the M
    // its first candidate sees, the lane walks its L candidates, and the
    // first stop over the warp ends the step
    if (warp == 0) {
      constexpr int L = K / 32;
      int32_t loc = INT_MAX;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const int k = lane * L + i;
        if (k < Kc && r_nf[k] > 0) loc = min(loc, r_m[k]);
      }
      int32_t pre = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre = min(pre, t);
      }
      int32_t running = __shfl_up_sync(0xffffffffu, pre, 1);
      if (lane == 0) running = INT_MAX;
      const int32_t all_min = __shfl_sync(0xffffffffu, pre, 31);
      // key 2k: stop before candidate k; 2k + 1: stop right after k
      int32_t key = INT_MAX, stop_next = -1;
      int64_t stop_e = -1;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const int k = lane * L + i;
        if (k >= Kc || key != INT_MAX) break;
        const int32_t v = c_v[k];
        if (v >= running) {  // a committed hit before k touched k's decision
          key = 2 * k;
          stop_next = running;
          break;
        }
        if (r_nf[k] > 0) {
          if (r_resume[k] >= 0) {  // row not finished: resume it next step
            key = 2 * k + 1;
            stop_next = v;
            stop_e = r_resume[k];
            break;
          }
          running = min(running, r_m[k]);
        }
      }
      int32_t gkey = key;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gkey = min(gkey, __shfl_xor_sync(0xffffffffu, gkey, o));
      long long add = 0;
      int commits = 0;
#pragma unroll
      for (int i = 0; i < L; ++i) {
        const int k = lane * L + i;
        if (k >= Kc) break;
        const bool commit = r_nf[k] > 0 && 2 * k < gkey;
        r_commit[k] = commit ? 1 : 0;
        if (commit) {
          add += r_gain[k];
          ++commits;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        add += __shfl_xor_sync(0xffffffffu, add, o);
        commits += __shfl_xor_sync(0xffffffffu, commits, o);
      }
      const unsigned owner = __ballot_sync(0xffffffffu, key == gkey && key != INT_MAX);
      int32_t next;
      int64_t next_e = -1;
      if (owner) {
        const int src = warp_first(owner);
        next = __shfl_sync(0xffffffffu, stop_next, src);
        next_e = __shfl_sync(0xffffffffu, stop_e, src);
      } else {
        next = min(all_min, s_span + 1);
      }
      if (lane == 0) {
        ++s_steps;
        s_commits += commits;
        s_total += add;
        s_pos = next;
        s_epos = next_e;
      }
    }
    __syncthreads();
    long long t_d = clock64();
    // D. apply the committed rows (warp per row): flips in the scan's
    // order v, u1, v, u2, ... then the re-marks of the changed set
    for (int k = warp; k < Kc; k += NW) {
      if (!r_commit[k]) continue;
      const int32_t v = c_v[k];
      const int nf = r_nf[k];
      if (nf == 1) {
        // one joint flip (v, u), u in N(v): the sequential pair apply_flip(v),
        // apply_flip(u) in closed form -- the two rows' neighbour updates
        // commute (no other commit of the step is adjacent to v or u, so
        // every other side read here is final), only the v-u edge terms
        // depend on the order -- so both rows and both mark walks run in
        // one pass instead of two chains of dependent L2 trips
        const int32_t u = r_part[k][0];
        const uint8_t svn = side[v] ^ 1, sun = side[u] ^ 1, su = sun ^ 1;
        const int64_t vb = off[v], ve = off[v + 1], ub = off[u], ue = off[u + 1];
        __syncwarp();  // every lane has read the old sides
        if (lane == 0) {
          side[v] = svn;
          side[u] = sun;
          const int32_t dv0 = delta[v], du0 = delta[u];
          delta[v] = -dv0 + (svn == sun ? 2 : -2);
          delta[u] = -(du0 + (su == svn ? 2 : -2));
        }
        const int64_t nv = ve - vb, tot = nv + (ue - ub);
        for (int64_t i = lane; i < tot; i += 32) {
          const bool in_v = i < nv;
          const int32_t y = in_v ? nbr[vb + i] : nbr[ub + (i - nv)];
          if (y == (in_v ? u : v)) continue;  // the v-u edge: done above
          atomicAdd(delta + y, side[y] == (in_v ? svn : sun) ? 2 : -2);
        }
        __syncwarp();
        // the re-marks of both changed sets: y over {v} U N(v) U {u} U N(u)
        for (int64_t i = lane; i < tot + 2; i += 32) {
          const int32_t y = i == 0 ? v : i <= nv ? nbr[vb + i - 1] : i == nv + 1 ? u : nbr[ub + (i - nv - 2)];
          if (y > v) cand[y] = 1;
          next_marks[y] = 1;
          for (int64_t c = off[y], c1 = off[y + 1]; c < c1; c += 4) {
            int32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = c + q < c1 ? nbr[c + q] : INT_MAX;
            bool stop = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (w[q] < y) {
                if (w[q] > v) cand[w[q]] = 1;
                next_marks[w[q]] = 1;
              } else {
                stop = true;
              }
            }
            if (stop) break;
          }
        }
        __syncwarp();
        continue;
      }
      for (int f = 0; f < nf; ++f) {
        for (int step = 0; step < 2; ++step) {
          const int32_t t = step == 0 ? v : r_part[k][f];
          if (lane == 0) {
            side[t] ^= 1;
            delta[t] = -delta[t];
          }
          __syncwarp();
          const uint8_t st = side[t];
          for (int64_t e = off[t] + lane, e1 = off[t + 1]; e < e1; e += 32) {
            const int32_t y = nbr[e];
            atomicAdd(delta + y, side[y] == st ? 2 : -2);
          }
          __syncwarp();
        }
      }
      warp_mark_after_flip2(off, nbr, cand, next_marks, v, v, lane);
      for (int f = 0; f < nf; ++f)
        warp_mark_after_flip2(off, nbr, cand, next_marks, r_part[k][f], v, lane);
    }
    __syncthreads();
    if (stats && threadIdx.x == 0) {
      const long long t_e = clock64();
      s_cyc[0] += t_b - t_a;
      s_cyc[1] += t_c - t_b;
      s_cyc[2] += t_d - t_c;
      s_cyc[3] += t_e - t_d;
    }
    if (s_pos >= n) break;
  }
  if (threadIdx.x == 0) {
    gains[s] += s_total;
    live[s] = s_total > 0 ? 1 : 0;  // improved: sweep again
    if (stats) {  // MQO_TRACE: steps and commits of this sweep
      atomicAdd(reinterpret_cast<unsigned long long*>(stats), static_cast<unsigned long long>(s_steps));
      atomicAdd(reinterpret_cast<unsigned long long*>(stats + 1),
                static_cast<unsigned long long>(s_commits));
      for (int q = 0; q < 4; ++q)
        atomicAdd(reinterpret_cast<unsigned long long*>(stats + 2 + q),
                  static_cast<unsigned long long>(s_cyc[q]));
    }
  }
}

}  // namespace

namespace {

// ------------------------------------------------------------------- MIS
// build_tightness (localsearch.cpp:9-15) + the require_maximal_is checks
// (76-84): flags[s] bit 0 = not independent, bit 1 = not maximal.
__global__ void k_tight(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr, int32_t n,
                        int32_t count, const uint8_t* __restrict__ sel, int32_t* __restrict__ tight,
                        int32_t* __restrict__ flags) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / n, v = q % n;
    const uint8_t* sd = sel + s * n;
    int32_t t = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) t += sd[nbr[e]];
    tight[q] = t;
    if (sd[v] && t) atomicOr(flags + s, 1);
    if (!sd[v] && t == 0) atomicOr(flags + s, 2);
  }
}

__device__ __forceinline__ bool has_edge(const int64_t* off, const int32_t* nbr, int32_t u, int32_t v) {
  int64_t lo = off[u], hi = off[u + 1];  // graph.cpp:58-61 (binary search)
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (nbr[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < off[u + 1] && nbr[lo] == v;
}

// swap_pair_for (localsearch.cpp:60-74) evaluated by one lane: the first
// pair (c_i, c_j), i < j, of unselected 1-tight neighbours of x in CSR
// order that are non-adjacent.
__device__ bool lane_swap_pair(const int64_t* off, const int32_t* nbr, const uint8_t* sel,
                               const int32_t* tight, int32_t x, int32_t& pu, int32_t& pw) {
  if (!*reinterpret_cast<const volatile uint8_t*>(sel + x)) return false;
  const int64_t e0 = off[x], e1 = off[x + 1];
  for (int64_t a = e0; a < e1; ++a) {
    const int32_t ca = nbr[a];
    if (*reinterpret_cast<const volatile uint8_t*>(sel + ca) ||
        *reinterpret_cast<const volatile int32_t*>(tight + ca) != 1)
      continue;
    for (int64_t c = a + 1; c < e1; ++c) {
      const int32_t cb = nbr[c];
      if (*reinterpret_cast<const volatile uint8_t*>(sel + cb) ||
          *reinterpret_cast<const volatile int32_t*>(tight + cb) != 1)
        continue;
      if (!has_edge(off, nbr, ca, cb)) {
        pu = ca;
        pw = cb;
        return true;
      }
    }
  }
  return false;
}

// lane_swap_pair without the dependent chain per neighbour: the row is
// read four entries at a time (four independent selection/tightness loads in
// flight), the first four candidates are kept in registers, and their six
// pairs are tested together (independent binary searches), the first
// non-adjacent one in (i, j) order winning.  Rows with more than four
// candidates whose first four are pairwise adjacent (rare: two random
// neighbours are adjacent with probability ~ degree / n) fall back to the
// exact serial search.  Callers order every access to sel / tight with
// barriers (no concurrent writer), so the loads are plain.
__device__ __forceinline__ bool lane_swap_pair_fast(const int64_t* off, const int32_t* nbr, const uint8_t* sel,
                                    const int32_t* tight, int32_t x, int32_t& pu, int32_t& pw) {
  if (!sel[x]) return false;
  const int64_t e0 = off[x], e1 = off[x + 1];
  int32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;  // the first four candidates
  int k = 0;
  bool more = false;  // a fifth candidate may exist (scan stopped at four)
  for (int64_t a = e0; a < e1; a += 4) {
    if (k >= 4) {
      more = true;
      break;
    }
    int32_t u[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = a + q < e1 ? nbr[a + q] : -1;
#pragma unroll
    for (int q = 0; q < 4; ++q) ok[q] = u[q] >= 0 && !sel[u[q]] && tight[u[q]] == 1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (ok[q]) {
        if (k == 0) c0 = u[q];
        if (k == 1) c1 = u[q];
        if (k == 2) c2 = u[q];
        if (k == 3) c3 = u[q];
        if (k == 4) more = true;
        ++k;
      }
    }
  }
  if (k < 2) return false;
  // the pairs among the first four in swap_pair_for's (i, j) order, tested
  // together: (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
  const bool t02 = k >= 3, t03 = k >= 4;
  const bool a01 = has_edge(off, nbr, c0, c1);
  const bool a02 = t02 ? has_edge(off, nbr, c0, c2) : true;
  const bool a03 = t03 ? has_edge(off, nbr, c0, c3) : true;
  const bool a12 = t02 ? has_edge(off, nbr, c1, c2) : true;
  if (!a01) { pu = c0; pw = c1; return true; }
  if (!a02) { pu = c0; pw = c2; return true; }
  if (!a03) { pu = c0; pw = c3; return true; }
  if (more) return lane_swap_pair(off, nbr, sel, tight, x, pu, pw);  // (0, j >= 4) come next
  if (!a12) { pu = c1; pw = c2; return true; }
  if (t03) {
    if (!has_edge(off, nbr, c1, c3)) { pu = c1; pw = c3; return true; }
    if (!has_edge(off, nbr, c2, c3)) { pu = c2; pw = c3; return true; }
  }
  return false;
}

// Adds vertex z to the set: sel[z] = 1, tight[N(z)] += 1 (warp-parallel).
__device__ __forceinline__ void warp_select(const int64_t* off, const int32_t* nbr, uint8_t* sel,
                                            int32_t* tight, int32_t z, int delta, int lane) {
  if (lane == 0) sel[z] = delta > 0 ? 1 : 0;
  for (int64_t e = off[z] + lane; e < off[z + 1]; e += 32) tight[nbr[e]] += delta;
  __syncwarp();
}

// Marks the selected vertices below the frontier whose swap_pair_for may
// have changed: 2-hop neighbourhood of a changed vertex t.
__device__ void warp_mark_dirty(const int64_t* off, const int32_t* nbr, const uint8_t* sel,
                                uint8_t* dflag, int32_t* dlist, int32_t* dcount, int32_t t,
                                int32_t frontier, int lane) {
  // s ranges over {t} U N(t); y over {s} U N(s)
  const int64_t e0 = off[t], e1 = off[t + 1];
  for (int64_t a = e0 - 1 + lane; a < e1; a += 32) {
    const int32_t s = a < e0 ? t : nbr[a];
    for (int64_t c = off[s] - 1; c < off[s + 1]; ++c) {
      const int32_t y = c < off[s] ? s : nbr[c];
      if (y >= frontier || !*reinterpret_cast<const volatile uint8_t*>(sel + y)) continue;
      // byte flag claim via 32-bit CAS on the containing word
      unsigned* word = reinterpret_cast<unsigned*>(reinterpret_cast<uintptr_t>(dflag + y) & ~uintptr_t(3));
      const unsigned shift = (reinterpret_cast<uintptr_t>(dflag + y) & 3) * 8;
      const unsigned old = atomicOr(word, 1u << shift);
      if (!((old >> shift) & 0xFF)) dlist[atomicAdd(dcount, 1)] = y;
    }
  }
  __syncwarp();
}

// Applies the (1,2)-swap at x (localsearch.cpp:174-196) and marks dirt.
__device__ void warp_apply_swap(const int64_t* off, const int32_t* nbr, const int32_t* deg_unused,
                                uint8_t* sel, int32_t* tight, uint8_t* dflag, int32_t* dlist,
                                int32_t* dcount, int32_t* freed, int32_t x, int32_t u, int32_t w,
                                int32_t frontier, int lane) {
  (void)deg_unused;
  warp_select(off, nbr, sel, tight, x, -1, lane);
  warp_select(off, nbr, sel, tight, u, +1, lane);
  warp_select(off, nbr, sel, tight, w, +1, lane);
  // freed neighbours of x, greedily re-added in ascending (degree, id)
  int32_t nf = 0;
  if (lane == 0) {
    for (int64_t e = off[x]; e < off[x + 1]; ++e) {
      const int32_t z = nbr[e];
      if (!sel[z] && tight[z] == 0) {
        // insertion sort by (deg, id)
        const int64_t dz = off[z + 1] - off[z];
        int32_t k = nf++;
        while (k > 0) {
          const int32_t p = freed[k - 1];
          const int64_t dp = off[p + 1] - off[p];
          if (dp < dz || (dp == dz && p < z)) break;
          freed[k] = p;
          --k;
        }
        freed[k] = z;
      }
    }
  }
  nf = __shfl_sync(0xffffffffu, nf, 0);
  __syncwarp();
  for (int32_t i = 0; i < nf; ++i) {
    const int32_t z = freed[i];
    const bool add = !*reinterpret_cast<volatile uint8_t*>(sel + z) &&
                     *reinterpret_cast<volatile int32_t*>(tight + z) == 0;
    if (add) warp_select(off, nbr, sel, tight, z, +1, lane);
    if (add) warp_mark_dirty(off, nbr, sel, dflag, dlist, dcount, z, frontier, lane);
  }
  warp_mark_dirty(off, nbr, sel, dflag, dlist, dcount, x, frontier, lane);
  warp_mark_dirty(off, nbr, sel, dflag, dlist, dcount, u, frontier, lane);
  warp_mark_dirty(off, nbr, sel, dflag, dlist, dcount, w, frontier, lane);
}

// The sequential part of a (1,2)-swap on one warp (selects, freed
// neighbours re-added greedily in (degree, id) order); the re-added vertices
// are left in freed[0..*nadd).  The dirty marking is done afterwards by the
// whole CTA (cta_mark_dirty), against the final selection: only selected
// vertices need re-examination, and every vertex whose swap pair could
// have changed is within two hops of x, u, w or a re-added vertex.
__device__ __forceinline__ void warp_swap_core(const int64_t* off, const int32_t* nbr, uint8_t* sel,
                               int32_t* tight, int32_t* freed, int32_t x, int32_t u, int32_t w,
                               int lane, int32_t* nadd) {
  warp_select(off, nbr, sel, tight, x, -1, lane);
  warp_select(off, nbr, sel, tight, u, +1, lane);
  warp_select(off, nbr, sel, tight, w, +1, lane);
  int32_t nf = 0;
  if (lane == 0) {
    for (int64_t e = off[x]; e < off[x + 1]; ++e) {
      const int32_t z = nbr[e];
      if (!sel[z] && tight[z] == 0) {
        const int64_t dz = off[z + 1] - off[z];
        int32_t k = nf++;
        while (k > 0) {
          const int32_t p = freed[k - 1];
          const int64_t dp = off[p + 1] - off[p];
          if (dp < dz || (dp == dz && p < z)) break;
          freed[k] = p;
          --k;
        }
        freed[k] = z;
      }
    }
  }
  nf = __shfl_sync(0xffffffffu, nf, 0);
  __syncwarp();
  int32_t na = 0;
  for (int32_t i = 0; i < nf; ++i) {
    const int32_t z = freed[i];
    const bool add = !*reinterpret_cast<volatile uint8_t*>(sel + z) &&
                     *reinterpret_cast<volatile int32_t*>(tight + z) == 0;
    if (add) {
      warp_select(off, nbr, sel, tight, z, +1, lane);
      if (lane == 0) freed[na] = z;  // na <= i: compaction in place
      ++na;
    }
  }
  __syncwarp();
  if (lane == 0) *nadd = na;
}

// Dirty marks for the 2-hop neighbourhood of t by the whole CTA: warps over
// s in {t} U N(t), lanes over y in {s} U N(s).
__device__ __forceinline__ void cta_mark_dirty(const int64_t* off, const int32_t* nbr, const uint8_t* sel,
                               uint8_t* dflag, int32_t* dlist, int32_t* dcount, int32_t t,
                               int32_t frontier) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t e0 = off[t], e1 = off[t + 1];
  for (int64_t a = e0 - 1 + warp; a < e1; a += nw) {
    const int32_t sv = a < e0 ? t : nbr[a];
    const int64_t c0 = off[sv], c1 = off[sv + 1];
    for (int64_t c = c0 - 1 + lane; c < c1; c += 32) {
      const int32_t y = c < c0 ? sv : nbr[c];
      if (y >= frontier || !*reinterpret_cast<const volatile uint8_t*>(sel + y)) continue;
      unsigned* word = reinterpret_cast<unsigned*>(reinterpret_cast<uintptr_t>(dflag + y) & ~uintptr_t(3));
      const unsigned shift = (reinterpret_cast<uintptr_t>(dflag + y) & 3) * 8;
      const unsigned old = atomicOr(word, 1u << shift);
      if (!((old >> shift) & 0xFF)) dlist[atomicAdd(dcount, 1)] = y;
    }
  }
}

// A full swap by the CTA: the core on warp 0, then the marks by everyone.
__device__ __forceinline__ void cta_apply_swap(const int64_t* off, const int32_t* nbr, uint8_t* sel, int32_t* tight,
                               uint8_t* dflag, int32_t* dlist, int32_t* dcount, int32_t* freed,
                               int32_t x, int32_t u, int32_t w, int32_t frontier, int32_t* s_nadd) {
  if ((threadIdx.x >> 5) == 0)
    warp_swap_core(off, nbr, sel, tight, freed, x, u, w, threadIdx.x & 31, s_nadd);
  __syncthreads();
  const int32_t na = *s_nadd;
  cta_mark_dirty(off, nbr, sel, dflag, dlist, dcount, x, frontier);
  cta_mark_dirty(off, nbr, sel, dflag, dlist, dcount, u, frontier);
  cta_mark_dirty(off, nbr, sel, dflag, dlist, dcount, w, frontier);
  for (int32_t i = 0; i < na; ++i)
    cta_mark_dirty(off, nbr, sel, dflag, dlist, dcount, freed[i], frontier);
  __syncthreads();
}

// Bytes of the SMEM-resident variant of k_mis_swap: the CSR and one body's
// state (one warp per CTA); 16-byte aligned sections.
__host__ __device__ inline int64_t swap_smem_bytes(int32_t n, int64_t nnz, int32_t max_degree) {
  auto al = [](int64_t b) { return (b + 15) / 16 * 16; };
  return al(8 * (int64_t(n) + 1)) + al(4 * nnz) + al(4 * int64_t(n)) + al(4 * int64_t(n)) +
         al(4 * (int64_t(max_degree) + 1)) + al(int64_t(n)) + al(int64_t(n) + 4) + 16;
}

__device__ __forceinline__ void cta_copy(void* dst, const void* src, int64_t bytes) {
  // bytes and both pointers 4-byte aligned; 16-byte moves where both allow
  const int64_t head = (reinterpret_cast<uintptr_t>(src) & 15) == 0 ? bytes / 16 : 0;
  const int4* s16 = static_cast<const int4*>(src);
  int4* d16 = static_cast<int4*>(dst);
  for (int64_t i = threadIdx.x; i < head; i += blockDim.x) d16[i] = __ldg(s16 + i);
  const int32_t* s4 = static_cast<const int32_t*>(src);
  int32_t* d4 = static_cast<int32_t*>(dst);
  for (int64_t i = head * 4 + threadIdx.x; i < bytes / 4; i += blockDim.x) d4[i] = s4[i];
}

// one_two_swap (localsearch.cpp:88-137) on one warp per solution.  With
// `smem` (graphs whose CSR + one body's state fit shared memory; one warp
// per CTA) the CSR, selection, tightness and dirty list are staged in SMEM
// first: the scan is a chain of dependent loads, ~30-cycle SMEM latency
// instead of ~300+ for L2.  Generic pointers serve both placements.
// one_two_swap's scan (localsearch.cpp:88-137) on one warp: the lowest
// swappable vertex among the dirty ones, else the next from the frontier;
// returns the number of swaps.
__device__ int64_t warp_swap_loop(const int64_t* off, const int32_t* nbr, uint8_t* sel,
                                  int32_t* tight, uint8_t* dflag, int32_t* dlist,
                                  int32_t* dcount, int32_t* freed, int32_t n, int lane) {
  int32_t frontier = 0;
  int64_t swaps = 0;
  for (;;) {
    // 1. lowest swappable vertex among the dirty ones below the frontier
    __syncwarp();
    const int32_t nd = *reinterpret_cast<volatile int32_t*>(dcount);
    int32_t best = INT_MAX, bu = 0, bw = 0;
    int32_t keep = 0;
    for (int32_t k0 = 0; k0 < nd; k0 += 32) {
      const int32_t k = k0 + lane;
      int32_t x = -1, pu = 0, pw = 0;
      bool ok = false;
      if (k < nd) {
        x = dlist[k];
        ok = lane_swap_pair_fast(off, nbr, sel, tight, x, pu, pw);
      }
      if (ok && x < best) {
        best = x;
        bu = pu;
        bw = pw;
      }
      // compact: keep swappable ones (they must be re-checked after the
      // next swap), drop the rest
      const unsigned km = __ballot_sync(0xffffffffu, ok);
      const int pos = __popc(km & ((1u << lane) - 1));
      __syncwarp();
      if (ok) dlist[keep + pos] = x;
      if (!ok && k < nd) dflag[x] = 0;
      keep += __popc(km);
      __syncwarp();
    }
    if (lane == 0) *dcount = keep;
    // warp min of best
    for (int o = 16; o; o >>= 1) {
      const int32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int32_t ou = __shfl_xor_sync(0xffffffffu, bu, o);
      const int32_t ow = __shfl_xor_sync(0xffffffffu, bw, o);
      if (ob < best) {
        best = ob;
        bu = ou;
        bw = ow;
      }
    }
    __syncwarp();
    if (best != INT_MAX) {
      warp_apply_swap(off, nbr, nullptr, sel, tight, dflag, dlist, dcount, freed, best, bu, bw,
                      frontier, lane);
      ++swaps;
      continue;
    }
    // 2. scan forward from the frontier
    int32_t found = -1, fu = 0, fw = 0;
    for (int32_t cb = frontier; cb < n; cb += 32) {
      const int32_t x = cb + lane;
      int32_t pu = 0, pw = 0;
      const bool ok = x < n && lane_swap_pair_fast(off, nbr, sel, tight, x, pu, pw);
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (m) {
        const int i = warp_first(m);
        found = cb + i;
        fu = __shfl_sync(0xffffffffu, pu, i);
        fw = __shfl_sync(0xffffffffu, pw, i);
        break;
      }
    }
    if (found < 0) break;
    frontier = found + 1;
    warp_apply_swap(off, nbr, nullptr, sel, tight, dflag, dlist, dcount, freed, found, fu, fw,
                    frontier, lane);
    ++swaps;
  }
  return swaps;
}

__global__ void k_mis_swap(const int64_t* __restrict__ off_g, const int32_t* __restrict__ nbr_g,
                           int32_t n, int32_t count, uint8_t* sel_all, int32_t* tight_all,
                           uint8_t* dflag_all, int32_t* dlist_all, int32_t* freed_all,
                           int32_t* dcount_all, int32_t max_degree, int64_t* swaps_out,
                           int32_t smem) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31;
  const int s = smem ? blockIdx.x : blockIdx.x * kLsWarps + (threadIdx.x >> 5);
  if (s >= count) return;
  uint8_t* sel_g = sel_all + static_cast<int64_t>(s) * n;
  const int64_t* off = off_g;
  const int32_t* nbr = nbr_g;
  uint8_t* sel = sel_g;
  int32_t* tight = tight_all + static_cast<int64_t>(s) * n;
  uint8_t* dflag = dflag_all + static_cast<int64_t>(s) * (n + 4);
  int32_t* dlist = dlist_all + static_cast<int64_t>(s) * n;
  int32_t* freed = freed_all + static_cast<int64_t>(s) * (max_degree + 1);
  int32_t* dcount = dcount_all + s;
  if (smem) {
    auto al = [](int64_t b) { return (b + 15) / 16 * 16; };
    const int64_t nnz = off_g[n];
    unsigned char* p = sm;
    int64_t* o = reinterpret_cast<int64_t*>(p);
    p += al(8 * (int64_t(n) + 1));
    int32_t* nb = reinterpret_cast<int32_t*>(p);
    p += al(4 * nnz);
    int32_t* ti = reinterpret_cast<int32_t*>(p);
    p += al(4 * int64_t(n));
    int32_t* dl = reinterpret_cast<int32_t*>(p);
    p += al(4 * int64_t(n));
    int32_t* fr = reinterpret_cast<int32_t*>(p);
    p += al(4 * (int64_t(max_degree) + 1));
    uint8_t* se = p;
    p += al(n);
    uint8_t* df = p;
    p += al(int64_t(n) + 4);
    int32_t* dc = reinterpret_cast<int32_t*>(p);
    cta_copy(o, off_g, 8 * (int64_t(n) + 1));
    cta_copy(nb, nbr_g, 4 * nnz);
    cta_copy(ti, tight, 4 * int64_t(n));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) se[i] = sel_g[i];
    for (int64_t i = threadIdx.x; i < int64_t(n) + 4; i += blockDim.x) df[i] = 0;
    if (threadIdx.x == 0) *dc = 0;
    __syncthreads();
    if (threadIdx.x >= 32) return;  // the other warps only helped stage
    off = o;
    nbr = nb;
    sel = se;
    tight = ti;
    dflag = df;
    dlist = dl;
    freed = fr;
    dcount = dc;
  }
  const int64_t swaps = warp_swap_loop(off, nbr, sel, tight, dflag, dlist, dcount, freed, n, lane);
  if (lane == 0) swaps_out[s] = swaps;
  if (smem) {
    __syncwarp();
    for (int64_t i = lane; i < n; i += 32) sel_g[i] = sel[i];
  }
}

// one_two_swap with a whole CTA per body (W warps): the two searches --
// the lowest swappable vertex in the dirty list, and the first swappable
// vertex at or after the frontier -- are evaluated by all W*32 threads
// (block-wide minimum; the frontier scan advances W*32 vertices per step),
// and warp 0 applies each swap exactly as k_mis_swap does.  The dirty list
// is compacted into a second buffer (entries are unique, so its order is
// irrelevant: only the minimum is used).  Same swaps, same order.
__host__ __device__ inline int64_t swap_cta_smem_bytes(int32_t n, int64_t nnz, int32_t max_degree) {
  return swap_smem_bytes(n, nnz, max_degree) + (4 * int64_t(n) + 15) / 16 * 16;
}

template <int W, bool SM>
__global__ void __launch_bounds__(32 * W)
    k_mis_swap_cta(const int64_t* __restrict__ off_g, const int32_t* __restrict__ nbr_g, int32_t n,
                   int32_t count, uint8_t* sel_all, int32_t* tight_all, uint8_t* dflag_all,
                   int32_t* dlist_all, int32_t* dlist2_all, int32_t* freed_all,
                   int32_t* dcount_all, int32_t max_degree, int64_t* swaps_out, int32_t smem,
                   const int32_t* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int32_t s_best, s_bu, s_bw, s_keep, s_nadd;
  const int s = blockIdx.x;
  if (s >= count) return;
  if (bad && bad[s]) return;  // not a maximal independent set: the host throws
  uint8_t* sel_g = sel_all + static_cast<int64_t>(s) * n;
  const int64_t* off = off_g;
  const int32_t* nbr = nbr_g;
  uint8_t* sel = sel_g;
  int32_t* tight = tight_all + static_cast<int64_t>(s) * n;
  uint8_t* dflag = dflag_all + static_cast<int64_t>(s) * (n + 4);
  // two dirty lists, swapped by `cur` (selects, not an indexed array: the
  // compiler then keeps their SMEM address space)
  int32_t* dla = dlist_all + static_cast<int64_t>(s) * n;
  int32_t* dlb = dlist2_all + static_cast<int64_t>(s) * n;
  int32_t* freed = freed_all + static_cast<int64_t>(s) * (max_degree + 1);
  int32_t* dcount = dcount_all + s;
  (void)smem;
  if constexpr (SM) {  // SMEM-resident state: the pointers below compile to LDS/STS
    auto al = [](int64_t b) { return (b + 15) / 16 * 16; };
    const int64_t nnz = off_g[n];
    unsigned char* p = sm;
    int64_t* o = reinterpret_cast<int64_t*>(p);
    p += al(8 * (int64_t(n) + 1));
    int32_t* nb = reinterpret_cast<int32_t*>(p);
    p += al(4 * nnz);
    int32_t* ti = reinterpret_cast<int32_t*>(p);
    p += al(4 * int64_t(n));
    int32_t* d0 = reinterpret_cast<int32_t*>(p);
    p += al(4 * int64_t(n));
    int32_t* fr = reinterpret_cast<int32_t*>(p);
    p += al(4 * (int64_t(max_degree) + 1));
    uint8_t* se = p;
    p += al(n);
    uint8_t* df = p;
    p += al(int64_t(n) + 4);
    int32_t* dc = reinterpret_cast<int32_t*>(p);
    p += 16;
    int32_t* d1 = reinterpret_cast<int32_t*>(p);
    cta_copy(o, off_g, 8 * (int64_t(n) + 1));
    cta_copy(nb, nbr_g, 4 * nnz);
    cta_copy(ti, tight, 4 * int64_t(n));
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) se[i] = sel_g[i];
    for (int64_t i = threadIdx.x; i < int64_t(n) + 4; i += blockDim.x) df[i] = 0;
    if (threadIdx.x == 0) *dc = 0;
    off = o;
    nbr = nb;
    sel = se;
    tight = ti;
    dflag = df;
    dla = d0;
    dlb = d1;
    freed = fr;
    dcount = dc;
  }
  __syncthreads();
  int cur = 0;
  int32_t frontier = 0;
  int64_t swaps = 0;
  for (;;) {
    // 1. lowest swappable vertex among the dirty ones (below the frontier)
    const int32_t nd = *reinterpret_cast<volatile int32_t*>(dcount);
    if (threadIdx.x == 0) {
      s_best = INT_MAX;
      s_keep = 0;
    }
    __syncthreads();
    int32_t mx = INT_MAX, mu = 0, mw = 0;
    for (int32_t k = threadIdx.x; k < nd; k += blockDim.x) {
      const int32_t x = (cur ? dlb : dla)[k];
      int32_t pu = 0, pw = 0;
      if (lane_swap_pair_fast(off, nbr, sel, tight, x, pu, pw)) {
        (cur ? dla : dlb)[atomicAdd(&s_keep, 1)] = x;  // re-checked after the next swap
        if (x < mx) {
          mx = x;
          mu = pu;
          mw = pw;
        }
      } else {
        dflag[x] = 0;
      }
    }
    if (mx != INT_MAX) atomicMin(&s_best, mx);
    __syncthreads();
    if (mx != INT_MAX && mx == s_best) {
      s_bu = mu;
      s_bw = mw;
    }
    if (threadIdx.x == 0) *dcount = s_keep;
    cur ^= 1;
    __syncthreads();
    if (s_best != INT_MAX) {
      cta_apply_swap(off, nbr, sel, tight, dflag, (cur ? dlb : dla), dcount, freed, s_best, s_bu, s_bw,
                     frontier, &s_nadd);
      ++swaps;
      continue;
    }
    // 2. first swappable vertex at or after the frontier.  The next one is
    // usually a few vertices on, so the window starts at two warps and
    // doubles up to the CTA (a step costs its slowest row search)
    if (threadIdx.x == 0) s_best = INT_MAX;
    __syncthreads();
    int32_t found = INT_MAX;
    for (int32_t base = frontier, win = 64; base < n; base += win, win = min(2 * win, static_cast<int32_t>(blockDim.x))) {
      const int32_t x = base + threadIdx.x;
      int32_t pu = 0, pw = 0;
      if (static_cast<int32_t>(threadIdx.x) < win && x < n && lane_swap_pair_fast(off, nbr, sel, tight, x, pu, pw)) {
        atomicMin(&s_best, x);
        mx = x;
        mu = pu;
        mw = pw;
      } else {
        mx = INT_MAX;
      }
      __syncthreads();
      found = s_best;
      if (found != INT_MAX) {
        if (mx == found) {
          s_bu = mu;
          s_bw = mw;
        }
        break;
      }
      __syncthreads();  // every thread has read s_best before the next step's atomicMin
    }
    __syncthreads();
    if (found == INT_MAX) break;
    frontier = found + 1;
    cta_apply_swap(off, nbr, sel, tight, dflag, (cur ? dlb : dla), dcount, freed, found, s_bu, s_bw, frontier,
                   &s_nadd);
    ++swaps;
  }
  if (threadIdx.x == 0) swaps_out[s] = swaps;
  if constexpr (SM)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sel_g[i] = sel[i];
}

// packed [count][W] <-> bytes [count][n]
__global__ void k_unpack(const uint64_t* __restrict__ packed, int64_t W, int32_t n, int32_t count,
                         uint8_t* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(count) * n;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / n, v = q % n;
    out[q] = (packed[s * W + (v >> 6)] >> (63 - (v & 63))) & 1;
  }
}

__global__ void k_pack_bytes(const uint8_t* __restrict__ in, int64_t W, int32_t n, int32_t count,
                             uint64_t* __restrict__ packed, int64_t* __restrict__ popc) {
  const int64_t total = static_cast<int64_t>(count) * W;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = q / W, w = q % W;
    uint64_t bits = 0;
    for (int i = 0; i < 64; ++i) {
      const int64_t v = w * 64 + i;
      if (v < n && in[s * n + v]) bits |= 1ull << (63 - i);
    }
    packed[q] = bits;
    if (popc && bits)
      atomicAdd(reinterpret_cast<unsigned long long*>(popc + s),
                static_cast<unsigned long long>(__popcll(bits)));
  }
}

int ls_grid(int64_t work) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 32)));
}

// build_gain_table for `count` bodies: light rows a thread each, rows of
// degree > kGainWarpDeg a warp each
void launch_gain(const mqo_graph* g, int32_t count, const uint8_t* side, int32_t* delta,
                 cudaStream_t st) {
  const int64_t cells = std::max<int64_t>(1, int64_t(count) * g->n);
  k_gain<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, g->n, count, side, delta);
  const int32_t heavy = g->h_deg_ge.size() > size_t(kGainWarpDeg) + 1 ? g->h_deg_ge[kGainWarpDeg + 1] : 0;
  if (heavy > 0)
    k_gain_heavy<<<ls_grid(int64_t(count) * heavy * 32), 256, 0, st>>>(g->d_off, g->d_nbr, g->d_order,
                                                                       heavy, g->n, count, side, delta);
  MQO_CUDA(cudaGetLastError());
}

}  // namespace

// -------------------------------------------------------------- host side
namespace mqo_b200 {

struct LsWork {
  uint8_t* bytes = nullptr;   // [count][n]
  int32_t* ints = nullptr;    // [count][n] delta / tight
  uint8_t* dflag = nullptr;   // [count][n+4]
  int32_t* dlist = nullptr;   // [count][n]
  int32_t* dlist2 = nullptr;  // [count][n] (compaction target of the CTA swap kernel)
  int32_t* freed = nullptr;   // [count][max_degree+1]
  int32_t* small = nullptr;   // [count] counters / flags
  int64_t* out64 = nullptr;   // [count]
  uint64_t* packed = nullptr; // [count][W]
};

// Runs local search op on `count` packed bodies already in device memory
// (`d_packed`, [count][W]); results written back in place.
//   op 0 one_flip_pass, 1 two_flip_pass, 2 one_two_flip (MaxCut: out64 =
//   gain), 3 one_two_swap (MIS: out64 = new size).
// one_flip_pass / two_flip_pass / one_two_flip (localsearch.cpp:139-190)
// for `count` bodies: 1-flip passes on one warp per body; 2-flip passes as
// host-driven sweeps of (grid candidate test, warp candidate scan) until a
// sweep flips nothing; one_two_flip alternates per body until a round gains
// nothing.  gains[s] = total gain.
void ensure_lo(mqo_graph* g, cudaStream_t st);

void maxcut_ls_host_driven(mqo_batch* b, int32_t op, int32_t count, uint8_t* side, int32_t* delta,
                           int64_t* d_out, cudaStream_t st) {
  mqo_graph* g = b->g;
  const int32_t n = g->n;
  const int64_t cells = std::max<int64_t>(1, int64_t(count) * n);
  const int blocks = (count + kLsWarps - 1) / kLsWarps;
  int32_t *d_live = nullptr, *d_live2 = nullptr, *d_und = nullptr;
  int64_t *d_g1 = nullptr, *d_g2 = nullptr;
  uint8_t* d_cand = nullptr;
  int32_t *d_cnt = nullptr, *d_list = nullptr, *d_len3 = nullptr;  // 1-flip closure (lazy)
  MQO_CUDA(cudaMallocAsync(&d_live, sizeof(int32_t) * count, st));
  MQO_CUDA(cudaMallocAsync(&d_live2, sizeof(int32_t) * count, st));
  MQO_CUDA(cudaMallocAsync(&d_und, sizeof(int32_t) * count, st));
  MQO_CUDA(cudaMallocAsync(&d_g1, sizeof(int64_t) * count, st));
  MQO_CUDA(cudaMallocAsync(&d_g2, sizeof(int64_t) * count, st));
  // marks of this sweep / of the next one (+64: the scan reads 16-byte
  // aligned windows past a body's end)
  MQO_CUDA(cudaMallocAsync(&d_cand, cells + 64, st));
  uint8_t* d_next = nullptr;
  if (g_scan_multi) MQO_CUDA(cudaMallocAsync(&d_next, cells + 64, st));
  int64_t* d_stats = nullptr;  // MQO_TRACE: 2-flip steps / commits per sweep
  if (trace_on()) {
    MQO_CUDA(cudaMallocAsync(&d_stats, 6 * sizeof(int64_t), st));
    MQO_CUDA(cudaMemsetAsync(d_stats, 0, 6 * sizeof(int64_t), st));
  }
  std::vector<int32_t> live(count, 1), live2(count);
  std::vector<int64_t> total(count, 0), g1(count, 0), g2(count, 0);
  auto two_flip = [&](const std::vector<int32_t>& who) {
    MQO_CUDA(cudaMemcpyAsync(d_live2, who.data(), sizeof(int32_t) * count, cudaMemcpyHostToDevice, st));
    MQO_CUDA(cudaMemsetAsync(d_g2, 0, sizeof(int64_t) * count, st));
    for (int sweep = 0;; ++sweep) {
      // the exact candidate test: every vertex in the first sweep, then only
      // those the last sweep's commits touched (its `next` marks)
      uint8_t* mask = nullptr;
      if (sweep > 0 && g_scan_multi) {
        std::swap(d_cand, d_next);
        mask = d_cand;  // tested in place: each cell reads only its own mark
      }
      k_two_cand<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, count, side,
                                                 delta, d_live2, d_cand, mask);
      const int32_t heavy = g->h_deg_ge.size() > size_t(kCandWarpDeg) + 1
                                ? g->h_deg_ge[kCandWarpDeg + 1] : 0;
      if (heavy > 0)
        k_two_cand_heavy<<<ls_grid(int64_t(count) * heavy * 32), 256, 0, st>>>(
            g->d_off, g->d_nbr, g->d_hmax, g->d_order, heavy, n, count, side, delta, d_live2,
            d_cand, mask);
      if (g_scan_multi) {
        MQO_CUDA(cudaMemsetAsync(d_next, 0, cells, st));
        // candidates per step = 32 warps x C (MQO_SCAN_C = 4 | 8 | 16)
        auto kern = g_scan_g == 8    ? (g_scan_c == 4 ? k_two_scan_multi<32, 4, 8>
                                                       : k_two_scan_multi<32, 8, 8>)
                    : g_scan_g == 16 ? k_two_scan_multi<32, 8, 16>
                    : g_scan_c == 4  ? k_two_scan_multi<32, 4, 32>
                    : g_scan_c == 16 ? k_two_scan_multi<32, 16, 32>
                                     : k_two_scan_multi<32, 8, 32>;
        kern<<<count, 32 * 32, 0, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, count, side, delta,
                                        d_cand, d_next, d_live2, d_g2, d_stats);
      }
      else if (g_scan_cta == 16)
        k_two_scan_cta<16><<<count, 32 * 16, 0, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, count,
                                                      side, delta, d_cand, d_live2, d_g2);
      else if (g_scan_cta == 32)
        k_two_scan_cta<32><<<count, 32 * 32, 0, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, count,
                                                      side, delta, d_cand, d_live2, d_g2);
      else if (g_scan_cta)
        k_two_scan_cta<8><<<count, 32 * 8, 0, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, count,
                                                    side, delta, d_cand, d_live2, d_g2);
      else
        k_two_scan<<<blocks, 32 * kLsWarps, 0, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, count, side,
                                                     delta, d_cand, d_live2, d_g2);
      MQO_CUDA(cudaGetLastError());
      MQO_CUDA(cudaMemcpyAsync(live2.data(), d_live2, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st));
      MQO_CUDA(cudaStreamSynchronize(st));
      bool any = false;
      for (int i = 0; i < count; ++i) any |= live2[i] != 0;
      if (d_stats) {
        int64_t sc[6] = {0, 0, 0, 0, 0, 0};
        MQO_CUDA(cudaMemcpy(sc, d_stats, sizeof(sc), cudaMemcpyDeviceToHost));
        MQO_CUDA(cudaMemset(d_stats, 0, sizeof(sc)));
        MQO_TRACE("two_flip sweep %d: %lld steps, %lld row commits (all bodies); Mcycles A %.2f "
                  "B %.2f C %.2f D %.2f", sweep, static_cast<long long>(sc[0]),
                  static_cast<long long>(sc[1]), sc[2] * 1e-6, sc[3] * 1e-6, sc[4] * 1e-6,
                  sc[5] * 1e-6);
      } else {
        MQO_TRACE("two_flip sweep %d", sweep);
      }
      if (!any) break;
    }
    MQO_CUDA(cudaMemcpyAsync(g2.data(), d_g2, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
    MQO_CUDA(cudaStreamSynchronize(st));
  };
  // one_flip_pass for the bodies in `who`: round-parallel passes (above)
  // until a pass flips nothing; delta is rebuilt after every pass
  // one CTA per body: when the body state fits SMEM, and the graph is small
  // or there are enough bodies to spread over the SMs (one large body runs
  // faster on the grid-wide rounds below)
  const bool flip_cta = one_flip_cta_fits(n, count);
  const bool flip_csr = flip_cta_smem_csr(n, 2 * g->m) <= kFlipCtaSmemMax;
  const int64_t flip_bytes = flip_csr ? flip_cta_smem_csr(n, 2 * g->m) : flip_cta_smem(n);
  auto one_flip = [&](const std::vector<int32_t>& who) {
    if (flip_cta) {  // small graphs: every pass of a body inside one CTA
      set_flip_cta_smem_attr();
      MQO_CUDA(cudaMemcpyAsync(d_live, who.data(), sizeof(int32_t) * count,
                               cudaMemcpyHostToDevice, st));
      (flip_csr ? k_one_flip_cta<true> : k_one_flip_cta<false>)<<<count, kFlipCtaThreads,
                                                                  static_cast<size_t>(flip_bytes), st>>>(
          g->d_off, g->d_nbr, n, side, delta, d_live, d_g1);
      MQO_CUDA(cudaGetLastError());
      MQO_CUDA(cudaMemcpyAsync(g1.data(), d_g1, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
      MQO_CUDA(cudaStreamSynchronize(st));
      MQO_TRACE("one_flip (CTA path)");
      return;
    }
    ensure_lo(g, st);
    if (!d_cnt) {  // closure state: counters, lists, [len | fa | fb] per body, kept
                   // with the batch (the engine's local-search calls reuse it)
      const size_t need = sizeof(int32_t) * (2 * cells + 3 * count);
      if (b->flip_bytes < need) {
        dfree(b, b->d_flip);
        dalloc(b, &b->d_flip, need);
        b->flip_bytes = need;
      }
      d_cnt = b->d_flip;
      d_list = d_cnt + cells;
      d_len3 = d_list + cells;
    }
    int32_t* d_len = d_len3;
    int32_t* d_fa = d_len3 + count;
    int32_t* d_fb = d_len3 + 2 * count;
    std::vector<int32_t> plive = who, und(count), lens(3 * count);
    std::vector<int64_t> pg(count);
    std::fill(g1.begin(), g1.end(), 0);
    for (int pass = 0;; ++pass) {
      bool any = false;
      for (int i = 0; i < count; ++i) any |= plive[i] != 0;
      if (!any) break;
      MQO_CUDA(cudaMemcpyAsync(d_live, plive.data(), sizeof(int32_t) * count,
                               cudaMemcpyHostToDevice, st));
      MQO_CUDA(cudaMemsetAsync(d_g1, 0, sizeof(int64_t) * count, st));
      // the seeds of P; a pass with many (a quarter of a body: the first
      // pass from a harvested state) runs the rounds over every vertex
      MQO_CUDA(cudaMemsetAsync(d_len3, 0, sizeof(int32_t) * 3 * count, st));
      k_flip_seed<<<ls_grid(cells), 256, 0, st>>>(n, count, delta, d_cand, d_cnt, d_list, d_len,
                                                  d_live);
      MQO_CUDA(cudaGetLastError());
      MQO_CUDA(cudaMemcpyAsync(lens.data(), d_len, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st));
      MQO_CUDA(cudaStreamSynchronize(st));
      bool listed = g_flip_closure;
      for (int i = 0; i < count; ++i) listed &= !plive[i] || int64_t(lens[i]) * 4 <= n;
      MQO_TRACE("one_flip pass %d: seeds of body 0 %d, %s", pass, lens[0], listed ? "closure" : "all vertices");
      if (listed) {  // the closure, four frontier steps per check
        for (int step = 0;; step += 4) {
          for (int r = 0; r < 4; ++r) {
            k_flip_front<<<1, 32, 0, st>>>(count, d_len, d_fa, d_fb);
            k_flip_close<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, g->d_lo, n, count,
                                                        side, d_cand, d_cnt, d_list, d_len, d_fa,
                                                        d_fb, d_live);
          }
          MQO_CUDA(cudaGetLastError());
          MQO_CUDA(cudaMemcpyAsync(lens.data(), d_len3, sizeof(int32_t) * 3 * count,
                                   cudaMemcpyDeviceToHost, st));
          MQO_CUDA(cudaStreamSynchronize(st));
          bool more = false;
          for (int i = 0; i < count; ++i) more |= lens[i] != lens[2 * count + i];  // len != fb
          if (!more) {
            MQO_TRACE("one_flip pass %d: closure of body 0 %d after %d steps", pass, lens[0], step + 4);
            break;
          }
        }
      } else {
        MQO_CUDA(cudaMemsetAsync(d_cand, 0, cells, st));  // every vertex undecided
      }
      int rounds = 0;
      for (;;) {  // four rounds per check; surplus rounds skip decided cells
        for (int r = 0; r < 4; ++r, ++rounds) {
          if (r == 3) MQO_CUDA(cudaMemsetAsync(d_und, 0, sizeof(int32_t) * count, st));
          k_flip_round<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, g->d_lo, n, count, side, delta,
                                                      d_cand, d_live, d_und);
        }
        MQO_CUDA(cudaGetLastError());
        MQO_CUDA(cudaMemcpyAsync(und.data(), d_und, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st));
        MQO_CUDA(cudaStreamSynchronize(st));
        bool left = false;
        for (int i = 0; i < count; ++i) left |= und[i] != 0;
        if (!left) break;
      }
      k_flip_commit<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, g->d_lo, n, count, side, delta, d_cand,
                                                   d_live, reinterpret_cast<unsigned long long*>(d_g1));
      k_flip_apply<<<ls_grid(cells), 256, 0, st>>>(n, count, side, d_cand, d_live);
      if (listed)  // every flip is listed: update the gains around them
        k_flip_update<<<ls_grid(int64_t(count) * 32 * 1024), 256, 0, st>>>(
            g->d_off, g->d_nbr, n, count, side, d_cand, delta, d_list, d_len, d_live);
      else
        launch_gain(g, count, side, delta, st);
      MQO_CUDA(cudaGetLastError());
      MQO_CUDA(cudaMemcpyAsync(pg.data(), d_g1, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
      MQO_CUDA(cudaStreamSynchronize(st));
      for (int i = 0; i < count; ++i) {
        if (!plive[i]) continue;
        g1[i] += pg[i];
        if (pg[i] == 0) plive[i] = 0;  // a pass without a flip ends one_flip_pass
      }
      MQO_TRACE("one_flip pass %d: %d rounds", pass, rounds);
    }
  };
  if (op == 0) {
    one_flip(live);
    total = g1;
  } else if (op == 1) {
    two_flip(live);
    total = g2;
  } else {
    for (int round = 0;; ++round) {
      bool any = false;
      for (int i = 0; i < count; ++i) any |= live[i] != 0;
      if (!any) break;
      one_flip(live);
      two_flip(live);
      for (int i = 0; i < count; ++i) {
        if (!live[i]) continue;
        const int64_t r = g1[i] + g2[i];
        total[i] += r;
        if (r == 0) live[i] = 0;  // localsearch.cpp:187-188
      }
      MQO_TRACE("one_two_flip round %d", round);
    }
  }
  MQO_CUDA(cudaMemcpyAsync(d_out, total.data(), sizeof(int64_t) * count, cudaMemcpyHostToDevice, st));
  MQO_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(d_live, st);
  cudaFreeAsync(d_live2, st);
  cudaFreeAsync(d_und, st);
  cudaFreeAsync(d_g1, st);
  cudaFreeAsync(d_g2, st);
  cudaFreeAsync(d_cand, st);
  if (d_next) cudaFreeAsync(d_next, st);
  if (d_stats) cudaFreeAsync(d_stats, st);

}

// Scratch of the (1,2)-swap kernels: dirty flags, the dirty list(s) and the
// freed-neighbour buffer per body.
void alloc_swap_lists(const mqo_graph* g, int32_t count, LsWork& w, cudaStream_t st,
                      bool second_list = false) {
  const int64_t n = g->n, cells = std::max<int64_t>(1, int64_t(count) * n);
  MQO_CUDA(cudaMallocAsync(&w.dflag, int64_t(count) * (n + 4), st));
  MQO_CUDA(cudaMemsetAsync(w.dflag, 0, int64_t(count) * (n + 4), st));
  MQO_CUDA(cudaMallocAsync(&w.dlist, sizeof(int32_t) * cells, st));
  if (second_list) MQO_CUDA(cudaMallocAsync(&w.dlist2, sizeof(int32_t) * cells, st));
  MQO_CUDA(cudaMallocAsync(&w.freed, sizeof(int32_t) * int64_t(count) * (g->max_degree + 1), st));
}

// k_mis_swap_cta (a CTA of 16 warps per body, CSR + state staged in SMEM
// when they fit) on bodies whose tightness is in w.ints; d_bad (may be
// null) marks bodies the input check rejected, which are skipped.
void launch_swap_cta(const mqo_graph* g, int32_t count, LsWork& w, int64_t* d_out,
                     cudaStream_t st, int32_t* d_bad) {
  alloc_swap_lists(g, count, w, st, true);
  const int64_t cbytes = swap_cta_smem_bytes(g->n, 2 * g->m, g->max_degree);
  static const bool swap_smem = [] {
    const char* e = std::getenv("MQO_SWAP_SMEM");
    return !(e && *e == '0');
  }();
  const bool csm = cbytes <= kSwapSmemMax - 1024 && g_swap_smem && swap_smem;
  auto kern = csm ? k_mis_swap_cta<16, true> : k_mis_swap_cta<16, false>;
  if (csm) {  // the SMEM opt-in, once per device
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    MQO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert(dev).second)
      MQO_CUDA(cudaFuncSetAttribute(k_mis_swap_cta<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSwapSmemMax - 1024)));
  }
  kern<<<count, 512, csm ? static_cast<size_t>(cbytes) : 0, st>>>(
      g->d_off, g->d_nbr, g->n, count, w.bytes, w.ints, w.dflag, w.dlist, w.dlist2, w.freed,
      w.small, g->max_degree, d_out, csm ? 1 : 0, d_bad);
  MQO_CUDA(cudaGetLastError());
}

// ---- single-launch local search for small bodies -------------------------
// A MaxCut call on small bodies used to be several launches (unpack, gain
// table, candidate tests, one scan launch per 2-flip sweep, pack) with a
// host round trip per sweep.  k_flip_small does the whole operation in ONE
// launch, one CTA per body, packed bodies in and out: unpack into SMEM,
// 1-flip passes as CTA decision rounds, 2-flip sweeps (rare moves) as the
// reference's sequential scan on one warp (a ballot finds the next row with
// a possible move among 32 vertices, the warp walks it), pack.  The CSR is
// staged in SMEM when it fits next to the state.
constexpr int64_t kSmallSmemMax = 226 * 1024;
constexpr int32_t kSmallMaxN = 16384;
constexpr int32_t kSmallTwoFlipMaxN = 4096;

__device__ __forceinline__ void small_unpack(const uint64_t* __restrict__ packed, int64_t W,
                                             int32_t n, uint8_t* dst) {
  for (int32_t v = threadIdx.x; v < n; v += blockDim.x)
    dst[v] = static_cast<uint8_t>((packed[v >> 6] >> (63 - (v & 63))) & 1u);
}
__device__ __forceinline__ void small_pack(const uint8_t* src, int64_t W, int32_t n,
                                           uint64_t* packed) {
  for (int64_t w = threadIdx.x; w < W; w += blockDim.x) {
    uint64_t word = 0;
    for (int b = 0; b < 64; ++b) {
      const int64_t v = w * 64 + b;
      if (v < n && src[v]) word |= 1ull << (63 - b);
    }
    packed[w] = word;
  }
}

// build_gain_table (localsearch.cpp:17-26), all threads
__device__ __forceinline__ void small_gains(const int64_t* off, const int32_t* nbr, int32_t n,
                                            const uint8_t* side, int32_t* delta) {
  for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
    const uint8_t sv = side[v];
    int32_t same = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) same += side[nbr[e]] == sv ? 1 : -1;
    delta[v] = same;
  }
}

// apply_flip (localsearch.cpp:28-33) by one warp
__device__ __forceinline__ void small_flip(const int64_t* off, const int32_t* nbr, uint8_t* side,
                                           int32_t* delta, int32_t v, int lane) {
  __syncwarp();
  if (lane == 0) {
    side[v] ^= 1;
    delta[v] = -delta[v];
  }
  __syncwarp();
  const uint8_t sv = side[v];
  for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
    const int32_t u = nbr[e];
    delta[u] += side[u] == sv ? 2 : -2;
  }
  __syncwarp();
}

// one_flip_pass (localsearch.cpp:139-157) for the single-launch kernel: the
// CTA decision rounds of cta_one_flip_pass, restricted per pass to the
// vertices that CAN flip.  P = the least set containing every v with
// d0[v] + 2 * |{u in P : u < v, u ~ v, side[u] != side[v]}| > 0 (seeds: the
// positive pass-start gains; each member raises its favourable upper
// neighbours' counters, a counter crossing zero admits its vertex exactly
// once).  By induction over the scan order every vertex the sequential pass
// flips is in P (its gain when reached is at most that bound), so the rest
// are decided "keep" before the rounds start and the rounds walk a compact
// list.  Late passes flip a handful of vertices, so P is small; the
// unrestricted rounds re-walked every undecided row (ncu r22: 30 rounds,
// 252k cycles at n = 1024, d = 16).
//
// Every phase is a chain of dependent SMEM loads per row, so a phase costs
// its longest row walk: each list item gets a group of G lanes (G = the
// largest power of two <= threads / items, <= 32) that stride its row and
// reduce with shuffles, so a short list still spreads over the CTA.  The
// gain table is built once and then updated from each pass's flips (a
// flipped row recomputed, its unflipped neighbours +-2), not rebuilt.
// SMEM (n <= 65535): d0, cnt [n] int32, lo, list [n] uint16, side, st [n]
// bytes.  Leaves d0 = the gain table of the final state.  Returns the gain
// on warp 0 (0 elsewhere).
__host__ __device__ inline int64_t small_state_bytes(int32_t n) { return (14 * int64_t(n) + 15) / 16 * 16; }

// lanes per item for `items` items over the CTA
__device__ __forceinline__ int group_lanes(int32_t items) {
  const int32_t per = items > 0 ? static_cast<int32_t>(blockDim.x) / items : 32;
  if (per >= 32) return 32;
  if (per <= 1) return 1;
  return 1 << (31 - __clz(per));
}

// sum over the G-lane group (G a power of two); every lane of the warp calls it
__device__ __forceinline__ int32_t group_sum(int32_t x, int G) {
  for (int o = 1; o < G; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ long long cta_one_flip_closure(const int64_t* off, const int32_t* nbr, int32_t n,
                                          uint8_t* sd, int32_t* d0, int32_t* cnt, uint16_t* lo,
                                          uint16_t* list, volatile uint8_t* st) {
  __shared__ int s_len;
  __shared__ long long s_part[32];
  const int32_t T = static_cast<int32_t>(blockDim.x);
  for (int32_t v = threadIdx.x; v < n; v += T) {  // lower rows are row prefixes
    int64_t a = off[v], b = off[v + 1];
    const int64_t e0 = a;
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (nbr[mid] < v) a = mid + 1; else b = mid;
    }
    lo[v] = static_cast<uint16_t>(a - e0);
    // build_gain_table (localsearch.cpp:17-26), once
    const uint8_t sv = sd[v];
    int32_t same = 0;
    const int32_t deg = static_cast<int32_t>(off[v + 1] - e0);
#pragma unroll 4
    for (int32_t k = 0; k < deg; ++k) same += sd[nbr[e0 + k]] == sv ? 1 : -1;
    d0[v] = same;
  }
  long long total = 0;
  for (;;) {
    if (threadIdx.x == 0) s_len = 0;
    __syncthreads();
    // the seeds of P; everything else "keep" until admitted
    for (int32_t v = threadIdx.x; v < n; v += T) {
      const int32_t d = d0[v];
      cnt[v] = d;
      if (d > 0) {
        st[v] = 0;
        list[atomicAdd(&s_len, 1)] = static_cast<uint16_t>(v);
      } else {
        st[v] = 1;
      }
    }
    // many seeds (a pass from a random state): P is most of the graph, and
    // its closure steps cost more than they save -- every vertex is listed
    __syncthreads();
    const bool all = int64_t(s_len) * 4 > n;
    if (all) {
      for (int32_t v = threadIdx.x; v < n; v += T) {
        list[v] = static_cast<uint16_t>(v);
        st[v] = 0;
      }
      __syncthreads();
      if (threadIdx.x == 0) s_len = n;
    }
    // the closure, one frontier per step
    for (int32_t a = all ? n : 0;;) {
      __syncthreads();
      const int32_t b = s_len;
      __syncthreads();  // every thread has b before anyone appends
      if (a == b) break;
      const int G = group_lanes(b - a);
      const int32_t gl = threadIdx.x & (G - 1);
      for (int32_t i = a + static_cast<int32_t>(threadIdx.x) / G; i < b; i += T / G) {
        const int32_t u = list[i];
        const uint8_t su = sd[u];
        const int64_t e1 = off[u + 1];
        for (int64_t e = off[u] + lo[u] + gl; e < e1; e += G) {
          const int32_t v = nbr[e];
          if (sd[v] == su) continue;
          const int32_t old = atomicAdd(&cnt[v], 2);
          if (old <= 0 && old > -2) {  // crossed zero: v joins P
            st[v] = 0;
            list[atomicAdd(&s_len, 1)] = static_cast<uint16_t>(v);
          }
        }
      }
      a = b;
    }
    const int32_t len = s_len;
    const int G = group_lanes(len);
    const int32_t gl = threadIdx.x & (G - 1);
    const int32_t ng = T / G;
    // warp-uniform trip counts (the group sums shuffle over whole warps);
    // a warp whose groups are all past the list skips the step
    const int32_t steps = (len + ng - 1) / ng;
    const int32_t wg0 = static_cast<int32_t>(threadIdx.x & ~31u) / G;  // the warp's first group
    // decision rounds (k_flip_round) over P
    for (;;) {
      int und = 0;
      for (int32_t t = 0; t < steps && t * ng + wg0 < len; ++t) {
        const int32_t i = t * ng + static_cast<int32_t>(threadIdx.x) / G;
        int32_t v = -1;
        if (i < len) {
          v = list[i];
          if (st[v]) v = -1;
        }
        int32_t add = 0, span = 0;  // span: up in the low 16 bits, -dn above
        uint8_t sv = 0;
        if (v >= 0) {
          sv = sd[v];
          const int64_t e0 = off[v];
          const int32_t L = lo[v];
#pragma unroll 4
          for (int32_t k = gl; k < L; k += G) {
            const int32_t u = nbr[e0 + k];
            const bool same = sd[u] == sv;
            const uint8_t su = st[u];
            if (su == 2)
              add += same ? -2 : 2;
            else if (su == 0)
              span += same ? (2 << 16) : 2;
          }
        }
        add = group_sum(add, G);
        span = group_sum(span, G);
        if (v >= 0 && gl == 0) {
          const int32_t base = d0[v] + add, dn = -(span >> 16), up = span & 0xffff;
          if (base + dn > 0)
            st[v] = 2;
          else if (base + up <= 0)
            st[v] = 1;
          else
            und = 1;
        }
      }
      if (!__syncthreads_or(und)) break;
    }
    // the pass's gain (k_flip_commit)
    long long g = 0;
    int flips = 0;
    for (int32_t t = 0; t < steps && t * ng + wg0 < len; ++t) {
      const int32_t i = t * ng + static_cast<int32_t>(threadIdx.x) / G;
      const int32_t v = i < len && st[list[i]] == 2 ? list[i] : -1;
      int32_t at = 0;
      if (v >= 0) {
        const uint8_t sv = sd[v];
        const int64_t e0 = off[v];
        const int32_t L = lo[v];
#pragma unroll 4
        for (int32_t k = gl; k < L; k += G) {
          const int32_t u = nbr[e0 + k];
          if (st[u] == 2) at += sd[u] == sv ? -2 : 2;
        }
      }
      at = group_sum(at, G);
      if (v >= 0 && gl == 0) {
        g += d0[v] + at;
        ++flips;
      }
    }
    for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = g;
    const bool any = __syncthreads_or(flips) != 0;
    if (threadIdx.x < 32) {  // the warp partials, summed on warp 0 only
      long long p = threadIdx.x < (T >> 5) ? s_part[threadIdx.x] : 0;
      for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
      total += p;
    }
    if (!any) break;  // a pass without a flip ends one_flip_pass
    for (int32_t i = threadIdx.x; i < len; i += T) {
      const int32_t v = list[i];
      if (st[v] == 2) sd[v] ^= 1;
    }
    __syncthreads();
    // the gain table of the new sides: flipped rows recomputed, their
    // unflipped neighbours +-2 (apply_flip, localsearch.cpp:28-33)
    for (int32_t t = 0; t < steps && t * ng + wg0 < len; ++t) {
      const int32_t i = t * ng + static_cast<int32_t>(threadIdx.x) / G;
      const int32_t v = i < len && st[list[i]] == 2 ? list[i] : -1;
      int32_t same = 0;
      if (v >= 0) {
        const uint8_t sv = sd[v];
        const int64_t e0 = off[v], e1 = off[v + 1];
        for (int64_t e = e0 + gl; e < e1; e += G) {
          const int32_t u = nbr[e];
          const bool eq = sd[u] == sv;
          same += eq ? 1 : -1;
          if (st[u] != 2) atomicAdd(&d0[u], eq ? 2 : -2);
        }
      }
      same = group_sum(same, G);
      if (v >= 0 && gl == 0) d0[v] = same;
    }
    __syncthreads();
  }
  return total;
}

// two_flip_pass (localsearch.cpp:159-181) of one body: every thread tests
// its vertices exactly (two_cand: a possible joint flip with a higher
// neighbour), then warp 0 visits the marked vertices in order, walks each
// row against the current state (continuing after each joint flip) and
// re-marks the later vertices whose test a flip can change
// (warp_mark_after_flip); sweeps repeat while one improves.  cand[n] bytes.
__device__ long long small_two_flip(const int64_t* off, const int32_t* nbr,
                                    const int32_t* __restrict__ hmax, int32_t n, uint8_t* side,
                                    int32_t* delta, uint8_t* cand) {
  const int lane = threadIdx.x & 31;
  __shared__ int s_improved;
  small_gains(off, nbr, n, side, delta);
  long long total = 0;
  for (;;) {
    __syncthreads();
    for (int32_t v = threadIdx.x; v < n; v += blockDim.x)
      cand[v] = two_cand(off, nbr, hmax, side, delta, v) ? 1 : 0;
    if (threadIdx.x == 0) s_improved = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
      volatile int32_t* vd = delta;
      volatile uint8_t* vs = side;
      volatile uint8_t* vc = cand;
      bool improved = false;
      for (int32_t c = 0; c < n; c += 32) {
        unsigned done = 0;
        for (;;) {
          const unsigned m = __ballot_sync(0xffffffffu, c + lane < n && vc[c + lane]) & ~done;
          if (!m) break;
          const int j = warp_first(m);
          const int32_t v = c + j;
          done = j == 31 ? ~0u : (2u << j) - 1u;
          const int64_t e1 = off[v + 1];
          for (int64_t e = off[v]; e < e1;) {
            const int64_t my = e + lane;
            bool hit = false;
            int32_t u = 0, joint = 0;
            if (my < e1) {
              u = nbr[my];
              if (u > v && vs[u] != vs[v]) {
                joint = vd[v] + vd[u] + 2;
                hit = joint > 0;
              }
            }
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (!hm) {
              e += 32;
              continue;
            }
            const int h = warp_first(hm);
            const int32_t uu = __shfl_sync(0xffffffffu, u, h);
            total += __shfl_sync(0xffffffffu, joint, h);
            small_flip(off, nbr, side, delta, v, lane);
            small_flip(off, nbr, side, delta, uu, lane);
            warp_mark_after_flip(off, nbr, cand, v, v, lane);
            warp_mark_after_flip(off, nbr, cand, uu, v, lane);
            improved = true;
            e += h + 1;
          }
        }
      }
      if (lane == 0 && improved) s_improved = 1;
    }
    __syncthreads();
    if (!s_improved) break;
  }
  __syncthreads();
  return total;
}

// OP: MQO_LS_ONE_FLIP / TWO_FLIP / ONE_TWO_FLIP; out[s] = the gain.  SMEM:
// d0 (the gain table), cnt, lo, list, sides, decision bytes
// (small_state_bytes), then the CSR when it fits.  1-flip passes run as CTA
// decision rounds over the vertices that can flip (cta_one_flip_closure),
// 2-flip sweeps on warp 0 (2-flip moves are rare next to 1-flip moves).
template <int OP, bool CSR>
__global__ void __launch_bounds__(kFlipCtaThreads, 1)
    k_flip_small(const int64_t* __restrict__ off_g, const int32_t* __restrict__ nbr_g,
                 const int32_t* __restrict__ hmax, int32_t n, int64_t W, uint64_t* packed,
                 int64_t* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int s = blockIdx.x;
  int32_t* d0 = reinterpret_cast<int32_t*>(sm);
  int32_t* cnt = d0 + n;
  uint16_t* lo = reinterpret_cast<uint16_t*>(cnt + n);
  uint16_t* list = lo + n;
  uint8_t* sd = reinterpret_cast<uint8_t*>(list + n);
  volatile uint8_t* st = sd + n;
  const int64_t* off = off_g;
  const int32_t* nbr = nbr_g;
  if constexpr (CSR) {
    int64_t* o = reinterpret_cast<int64_t*>(sm + small_state_bytes(n));
    int32_t* nb = reinterpret_cast<int32_t*>(sm + small_state_bytes(n) + (8 * (int64_t(n) + 1) + 15) / 16 * 16);
    const int64_t nnz = off_g[n];
    for (int64_t i = threadIdx.x; i <= n; i += blockDim.x) o[i] = off_g[i];
#pragma unroll 4
    for (int64_t i = threadIdx.x; i < nnz; i += blockDim.x) nb[i] = nbr_g[i];
    off = o;
    nbr = nb;
  }
  small_unpack(packed + s * W, W, n, sd);
  __syncthreads();
  long long total = 0;
  auto one_flip = [&] { return cta_one_flip_closure(off, nbr, n, sd, d0, cnt, lo, list, st); };
  if constexpr (OP == MQO_LS_ONE_FLIP) total = one_flip();
  uint8_t* cand = const_cast<uint8_t*>(st);  // the decision bytes double as 2-flip marks
  if constexpr (OP == MQO_LS_TWO_FLIP) total = small_two_flip(off, nbr, hmax, n, sd, d0, cand);
  if constexpr (OP == MQO_LS_ONE_TWO_FLIP) {  // localsearch.cpp:183-190
    for (;;) {
      const long long r = one_flip() + small_two_flip(off, nbr, hmax, n, sd, d0, cand);
      total += r;
      if (__syncthreads_or(r != 0) == 0) break;
    }
  }
  __syncthreads();
  small_pack(sd, W, n, packed + s * W);
  if (threadIdx.x == 0) out[s] = total;
}

inline int64_t small_csr_bytes(int32_t n, int64_t nnz) {
  return (8 * (int64_t(n) + 1) + 15) / 16 * 16 + 4 * nnz;
}

// d_bad (one_two_swap only, may be null, zeroed by the caller): when given,
// the input check of k_tight is left in d_bad[count] (bit 0 not independent, bit 1 not maximal)
// for the caller to raise after its copy-out, instead of a host round trip
// here; flagged bodies are left untouched.
// lower-neighbour count per row (binary search for the first entry >= v)
__global__ void k_lower_counts(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                               int32_t n, int32_t* __restrict__ lo) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t a = off[v], b = off[v + 1];
    const int64_t e0 = a;
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (nbr[mid] < v) a = mid + 1; else b = mid;
    }
    lo[v] = static_cast<int32_t>(a - e0);
  }
}

// lower-neighbour counts of the graph (k_lower_counts), built once
void ensure_lo(mqo_graph* g, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g->lazy_mu);
  if (g->d_lo) return;
  void* p = nullptr;
  const cudaStream_t ms = mem_stream(g->device);
  MQO_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * std::max(g->n, 1), ms));
  MQO_CUDA(cudaStreamSynchronize(ms));
  auto* lo = static_cast<int32_t*>(p);
  if (g->n) k_lower_counts<<<ls_grid(g->n), 256, 0, st>>>(g->d_off, g->d_nbr, g->n, lo);
  MQO_CUDA(cudaGetLastError());
  MQO_CUDA(cudaStreamSynchronize(st));
  g->d_lo = lo;
}

// hmax (k_hmax) of the graph, built once, complete before any stream uses it
void ensure_hmax(mqo_graph* g, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g->lazy_mu);
  if (g->d_hmax) return;
  int32_t* h = nullptr;
  {  // pool allocation on the graph's memory stream (freed there with the graph)
    const cudaStream_t ms = mem_stream(g->device);
    void* p = nullptr;
    MQO_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * std::max(g->n, 1), ms));
    MQO_CUDA(cudaStreamSynchronize(ms));
    h = static_cast<int32_t*>(p);
  }
  k_hmax<<<ls_grid(g->n), 256, 0, st>>>(g->d_off, g->d_nbr, g->n, h);
  const int32_t heavy = g->h_deg_ge.size() > size_t(kGainWarpDeg) + 1 ? g->h_deg_ge[kGainWarpDeg + 1] : 0;
  if (heavy > 0)
    k_hmax_heavy<<<ls_grid(int64_t(heavy) * 32), 256, 0, st>>>(g->d_off, g->d_nbr, g->d_order, heavy, h);
  MQO_CUDA(cudaGetLastError());
  MQO_CUDA(cudaStreamSynchronize(st));
  g->d_hmax = h;
}

// MQO_LS_SMALL=0 disables the single-launch small-body kernels (A/B runs)
const bool g_ls_small = [] {
  const char* e = std::getenv("MQO_LS_SMALL");
  return !(e && *e == '0');
}();

// The single-launch MaxCut kernels apply (n <= kSmallMaxN, state in SMEM);
// returns whether they were launched.  (one_two_swap keeps its CTA kernel:
// a swap is a sequential core on one warp either way, and the CTA searches
// are the faster part.)
bool local_search_small(mqo_batch* b, int32_t op, int32_t count, uint64_t* d_packed,
                        int64_t* d_out, cudaStream_t st, int32_t* /*d_bad*/) {
  mqo_graph* g = b->g;
  const int32_t n = g->n;
  if (!g_ls_small || n > kSmallMaxN || n == 0 || op == MQO_LS_ONE_TWO_SWAP) return false;
  // the 2-flip sweeps walk their moves on one warp: past a few thousand
  // vertices the multi-commit sweeps (k_two_scan_multi) win
  // (scripts/ls_small_probe.py: one_two_flip from random sides, n = 4096
  // 3.46 vs 3.48 ms, n = 16384 22.1 vs 9.7 ms)
  if (op != MQO_LS_ONE_FLIP && n > kSmallTwoFlipMaxN) return false;
  const int64_t state = small_state_bytes(n);
  if (state > kSmallSmemMax) return false;
  const bool csr = state + small_csr_bytes(n, 2 * g->m) <= kSmallSmemMax;
  const size_t smem = static_cast<size_t>(csr ? state + small_csr_bytes(n, 2 * g->m) : state);
  const int64_t W = body_words(n);
  if (op != MQO_LS_ONE_FLIP) ensure_hmax(g, st);
  auto launch = [&](auto kern) {
    static std::mutex mu;  // the SMEM opt-in, once per (kernel, device)
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    MQO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert({reinterpret_cast<const void*>(kern), dev}).second)
      MQO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmallSmemMax)));
    return kern;
  };
  void (*k)(const int64_t*, const int32_t*, const int32_t*, int32_t, int64_t, uint64_t*,
            int64_t*) = nullptr;
  if (op == MQO_LS_ONE_FLIP) k = csr ? launch(k_flip_small<0, true>) : launch(k_flip_small<0, false>);
  if (op == MQO_LS_TWO_FLIP) k = csr ? launch(k_flip_small<1, true>) : launch(k_flip_small<1, false>);
  if (op == MQO_LS_ONE_TWO_FLIP)
    k = csr ? launch(k_flip_small<2, true>) : launch(k_flip_small<2, false>);
  k<<<count, kFlipCtaThreads, smem, st>>>(g->d_off, g->d_nbr, g->d_hmax, n, W, d_packed, d_out);
  MQO_CUDA(cudaGetLastError());
  MQO_TRACE("local search op %d on %d bodies: single-launch kernel queued", op, count);
  return true;
}

void local_search_device(mqo_batch* b, int32_t op, int32_t count, uint64_t* d_packed,
                         int64_t* d_out, cudaStream_t st, int32_t* d_bad) {
  mqo_graph* g = b->g;
  const int32_t n = g->n;
  const int64_t W = body_words(n);
  if (count <= 0) return;
  MQO_TRACE("local search op %d on %d bodies", op, count);
  if (local_search_small(b, op, count, d_packed, d_out, st, d_bad)) return;
  LsWork w;
  const int64_t cells = std::max<int64_t>(1, int64_t(count) * n);
  if (op == 0 && one_flip_cta_fits(n, count)) {
    // one_flip_pass alone on the CTA path: the kernel builds its own gain
    // table, every body starts live and its pass gains are the result, so the
    // call is unpack -> k_one_flip_cta -> pack with no host round trip (the
    // caller's copy-out synchronises)
    const bool csr = flip_cta_smem_csr(n, 2 * g->m) <= kFlipCtaSmemMax;
    MQO_CUDA(cudaMallocAsync(&w.bytes, cells, st));
    MQO_CUDA(cudaMallocAsync(&w.ints, sizeof(int32_t) * cells, st));
    k_unpack<<<ls_grid(cells), 256, 0, st>>>(d_packed, W, n, count, w.bytes);
    set_flip_cta_smem_attr();
    (csr ? k_one_flip_cta<true> : k_one_flip_cta<false>)<<<
        count, kFlipCtaThreads,
        static_cast<size_t>(csr ? flip_cta_smem_csr(n, 2 * g->m) : flip_cta_smem(n)), st>>>(
        g->d_off, g->d_nbr, n, w.bytes, w.ints, nullptr, d_out);
    k_pack_bytes<<<ls_grid(int64_t(count) * W), 256, 0, st>>>(w.bytes, W, n, count, d_packed, nullptr);
    MQO_CUDA(cudaGetLastError());
    cudaFreeAsync(w.bytes, st);
    cudaFreeAsync(w.ints, st);
    MQO_TRACE("local search op 0 (CTA path) queued");
    return;
  }
  MQO_CUDA(cudaMallocAsync(&w.bytes, cells, st));
  MQO_CUDA(cudaMallocAsync(&w.ints, sizeof(int32_t) * cells, st));
  MQO_CUDA(cudaMallocAsync(&w.small, sizeof(int32_t) * count, st));
  MQO_CUDA(cudaMemsetAsync(w.small, 0, sizeof(int32_t) * count, st));
  MQO_CUDA(cudaMemsetAsync(d_out, 0, sizeof(int64_t) * count, st));
  k_unpack<<<ls_grid(cells), 256, 0, st>>>(d_packed, W, n, count, w.bytes);
  MQO_CUDA(cudaGetLastError());
  const int blocks = (count + kLsWarps - 1) / kLsWarps;
  if (op <= 2) {
    launch_gain(g, count, w.bytes, w.ints, st);
    MQO_CUDA(cudaGetLastError());
    if (trace_on()) {
      MQO_CUDA(cudaStreamSynchronize(st));
      MQO_TRACE("local search: bodies unpacked, gain tables built");
    }
    ensure_hmax(g, st);
    MQO_TRACE("local search: hmax ready");
    maxcut_ls_host_driven(b, op, count, w.bytes, w.ints, d_out, st);
  } else if (d_bad && g_swap_cta) {
    // the input check stays on the device: k_tight flags bad bodies in
    // d_bad (zeroed by the caller), which the swap kernel then leaves untouched
    k_tight<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, n, count, w.bytes, w.ints, d_bad);
    MQO_CUDA(cudaGetLastError());
    launch_swap_cta(g, count, w, d_out, st, d_bad);
    MQO_CUDA(cudaMemsetAsync(d_out, 0, sizeof(int64_t) * count, st));
  } else {
    k_tight<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, n, count, w.bytes, w.ints, w.small);
    MQO_CUDA(cudaGetLastError());
    std::vector<int32_t> flags(count);
    MQO_CUDA(cudaMemcpyAsync(flags.data(), w.small, sizeof(int32_t) * count,
                             cudaMemcpyDeviceToHost, st));
    MQO_CUDA(cudaStreamSynchronize(st));
    MQO_TRACE("one_two_swap: tightness checked");
    for (int i = 0; i < count; ++i) {
      if (flags[i] & 1) {
        cudaFreeAsync(w.bytes, st);
        cudaFreeAsync(w.ints, st);
        cudaFreeAsync(w.small, st);
        throw std::invalid_argument("one_two_swap: input not an independent set");
      }
      if (flags[i] & 2) {
        cudaFreeAsync(w.bytes, st);
        cudaFreeAsync(w.ints, st);
        cudaFreeAsync(w.small, st);
        throw std::invalid_argument("one_two_swap: input not maximal");
      }
    }
    MQO_CUDA(cudaMemsetAsync(w.small, 0, sizeof(int32_t) * count, st));
    cudaEvent_t ev[2] = {nullptr, nullptr};
    if (trace_on()) {
      cudaEventCreate(&ev[0]);
      cudaEventCreate(&ev[1]);
      cudaEventRecord(ev[0], st);
    }
    const int64_t sbytes = swap_smem_bytes(n, 2 * g->m, g->max_degree);
    const bool smem = sbytes <= kSwapSmemMax && g_swap_smem;
    if (g_swap_cta) {  // a CTA of 16 warps per body
      launch_swap_cta(g, count, w, d_out, st, nullptr);
    } else if (smem) {
      alloc_swap_lists(g, count, w, st);
      MQO_CUDA(cudaFuncSetAttribute(k_mis_swap, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSwapSmemMax)));
      k_mis_swap<<<count, 256, static_cast<size_t>(sbytes), st>>>(
          g->d_off, g->d_nbr, n, count, w.bytes, w.ints, w.dflag, w.dlist, w.freed, w.small,
          g->max_degree, d_out, 1);
    } else {
      alloc_swap_lists(g, count, w, st);
      k_mis_swap<<<blocks, 32 * kLsWarps, 0, st>>>(g->d_off, g->d_nbr, n, count, w.bytes, w.ints,
                                                   w.dflag, w.dlist, w.freed, w.small,
                                                   g->max_degree, d_out, 0);
    }
    MQO_CUDA(cudaGetLastError());
    if (trace_on()) {
      cudaEventRecord(ev[1], st);
      cudaEventSynchronize(ev[1]);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      MQO_TRACE("k_mis_swap: %.3f ms (%d bodies)", ms, count);
      cudaEventDestroy(ev[0]);
      cudaEventDestroy(ev[1]);
    }
    MQO_CUDA(cudaMemsetAsync(d_out, 0, sizeof(int64_t) * count, st));
  }
  k_pack_bytes<<<ls_grid(int64_t(count) * W), 256, 0, st>>>(w.bytes, W, n, count, d_packed,
                                                            op == 3 ? d_out : nullptr);
  MQO_CUDA(cudaGetLastError());
  cudaFreeAsync(w.bytes, st);
  cudaFreeAsync(w.ints, st);
  cudaFreeAsync(w.small, st);
  if (w.dflag) cudaFreeAsync(w.dflag, st);
  if (w.dlist) cudaFreeAsync(w.dlist, st);
  if (w.dlist2) cudaFreeAsync(w.dlist2, st);
  if (w.freed) cudaFreeAsync(w.freed, st);
  MQO_TRACE("local search op %d queued", op);
}

}  // namespace mqo_b200

extern "C" int mqo_local_search(mqo_batch* b, int32_t op, int32_t count, uint64_t* packed,
                                int64_t* out) {
  return guard([&] {
    if (!b || count < 0 || (count && (!packed || !out)))
      throw std::invalid_argument("mqo_local_search: bad arguments");
    if (op < 0 || op > 3) throw std::invalid_argument("mqo_local_search: unknown op");
    MQO_CUDA(cudaSetDevice(b->g->device));
    if (count == 0) return;
    const int64_t W = body_words(b->g->n);
    const int64_t words = W * count;
    // one device buffer [bodies | results | input flags] so the copy-out is a
    // single D2H; device and pinned staging persist with the batch, so a
    // small call is memcpy, H2D, the launch(es), D2H and one sync
    const int64_t total = words + count + (count + 1) / 2;
    const size_t bytes = sizeof(uint64_t) * total;
    cudaStream_t st = b->stream;
    if (b->ls_bytes < bytes) {
      dfree(b, b->d_ls);
      pinned_put(b->h_ls, b->ls_bytes);
      dalloc(b, &b->d_ls, bytes);
      b->h_ls = static_cast<uint64_t*>(pinned_get(bytes));
      b->ls_bytes = bytes;
    }
    uint64_t* d_packed = b->d_ls;
    uint64_t* h = b->h_ls;
    int64_t* d_out = reinterpret_cast<int64_t*>(d_packed + words);
    int32_t* d_bad = reinterpret_cast<int32_t*>(d_packed + words + count);
    std::memcpy(h, packed, sizeof(uint64_t) * words);
    MQO_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int32_t) * count, st));
    MQO_CUDA(cudaMemcpyAsync(d_packed, h, sizeof(uint64_t) * words, cudaMemcpyHostToDevice, st));
    MQO_TRACE("mqo_local_search: bodies uploaded");
    try {
      local_search_device(b, op, count, d_packed, d_out, st, op == 3 ? d_bad : nullptr);
    } catch (...) {
      cudaStreamSynchronize(st);
      throw;
    }
    MQO_CUDA(cudaMemcpyAsync(h, d_packed, bytes, cudaMemcpyDeviceToHost, st));
    MQO_CUDA(cudaStreamSynchronize(st));
    // one_two_swap's input check (localsearch.cpp:88-96), raised before the
    // caller's buffer is touched
    const int32_t* bad = reinterpret_cast<const int32_t*>(h + words + count);
    for (int32_t i = 0; i < count; ++i) {
      if (bad[i] & 1) throw std::invalid_argument("one_two_swap: input not an independent set");
      if (bad[i] & 2) throw std::invalid_argument("one_two_swap: input not maximal");
    }
    std::memcpy(packed, h, sizeof(uint64_t) * words);
    std::memcpy(out, h + words, sizeof(int64_t) * count);
    MQO_TRACE("mqo_local_search: done");
  });
}

// build_gain_table (kind 0) / build_tightness (kind 1) for `count` packed
// bodies: out [count][n] int32 (localsearch.cpp:9-26).
extern "C" int mqo_build_tables(mqo_batch* b, int32_t kind, int32_t count, const uint64_t* packed,
                                int32_t* out) {
  return guard([&] {
    if (!b || count < 0 || (count && (!packed || !out)))
      throw std::invalid_argument("mqo_build_tables: bad arguments");
    MQO_CUDA(cudaSetDevice(b->g->device));
    if (count == 0 || b->g->n == 0) return;
    mqo_graph* g = b->g;
    const int32_t n = g->n;
    const int64_t W = body_words(n), cells = int64_t(count) * n;
    cudaStream_t st = b->stream;
    uint64_t* d_packed = nullptr;
    uint8_t* d_bytes = nullptr;
    int32_t *d_out = nullptr, *d_flags = nullptr;
    MQO_CUDA(cudaMallocAsync(&d_packed, sizeof(uint64_t) * W * count, st));
    MQO_CUDA(cudaMallocAsync(&d_bytes, cells, st));
    MQO_CUDA(cudaMallocAsync(&d_out, sizeof(int32_t) * cells, st));
    MQO_CUDA(cudaMallocAsync(&d_flags, sizeof(int32_t) * count, st));
    MQO_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(int32_t) * count, st));
    MQO_CUDA(cudaMemcpyAsync(d_packed, packed, sizeof(uint64_t) * W * count, cudaMemcpyHostToDevice, st));
    k_unpack<<<ls_grid(cells), 256, 0, st>>>(d_packed, W, n, count, d_bytes);
    if (kind == 0)
      launch_gain(g, count, d_bytes, d_out, st);
    else
      k_tight<<<ls_grid(cells), 256, 0, st>>>(g->d_off, g->d_nbr, n, count, d_bytes, d_out, d_flags);
    MQO_CUDA(cudaGetLastError());
    MQO_CUDA(cudaMemcpyAsync(out, d_out, sizeof(int32_t) * cells, cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(d_packed, st);
    cudaFreeAsync(d_bytes, st);
    cudaFreeAsync(d_out, st);
    cudaFreeAsync(d_flags, st);
    MQO_CUDA(cudaStreamSynchronize(st));
  });
}
