// common.cuh -- shared internals of libmqo_b200.so: error plumbing for the C
// ABI (include/mqo_gpu.h), the graph / batch handle layouts, and the exact
// (no-FMA) fp64 helpers every kernel uses so results stay bit-identical to
// the reference's `-O3 -ffp-contract=off`-style scalar code.
#pragma once

#include <cuda_runtime.h>

#include <unistd.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "mqo_gpu.h"

namespace mqo_b200 {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
void set_error_line(int32_t line);

// graph_io.hpp:13-21: a parse failure with the offending 1-based line
// (a std::runtime_error in the reference; MQO_ERR_PARSE at the ABI).
struct ParseError : std::runtime_error {
  int32_t line;
  ParseError(int32_t l, const std::string& what)
      : std::runtime_error("line " + std::to_string(l) + ": " + what), line(l) {}
};

// MQO_TRACE=1: one stderr line per engine / trajectory stage (debugging).
bool trace_on();
double trace_clock();
#define MQO_TRACE(...)                                                          \
  do {                                                                         \
    if (::mqo_b200::trace_on()) {                                              \
      std::fprintf(stderr, "[mqo %d %.6f] ", (int)getpid(), ::mqo_b200::trace_clock()); \
      std::fprintf(stderr, __VA_ARGS__);                                       \
      std::fprintf(stderr, "\n");                                              \
      std::fflush(stderr);                                                     \
    }                                                                          \
  } while (0)

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// A failed collective (NCCL or a caller's mqo_comm callback) or a peer rank
// that failed: MQO_ERR_NCCL at the ABI.
struct CommError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Raised on the healthy ranks when a peer rank failed (the failed rank
// rethrows its own error).
struct PeerFailed : CommError {
  using CommError::CommError;
};

#define MQO_CUDA(expr)                                                           \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess)                                                       \
      throw ::mqo_b200::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// Runs `f`, mapping the reference's exception types onto the ABI codes.
template <typename F>
int guard(F&& f) {
  try {
    f();
    return MQO_OK;
  } catch (const ParseError& e) {
    set_error(e.what());
    set_error_line(e.line);
    return MQO_ERR_PARSE;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return MQO_ERR_INVALID;
  } catch (const std::logic_error& e) {
    set_error(e.what());
    return MQO_ERR_LOGIC;
  } catch (const CudaError& e) {
    set_error(e.what());
    return MQO_ERR_CUDA;
  } catch (const CommError& e) {
    set_error(e.what());
    return MQO_ERR_NCCL;
  } catch (const std::exception& e) {
    set_error(e.what());
    return MQO_ERR_OTHER;
  }
}

// ------------------------------------------------------ exact fp64 helpers
// The reference evaluates every expression as separately rounded IEEE
// operations (no contraction).  These intrinsics pin that on the device
// regardless of --fmad.
__device__ __forceinline__ double ex_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ex_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ex_mul(double a, double b) { return __dmul_rn(a, b); }

// clamp_to (pga.cpp:31-34): std::min(1.0, std::max(lo, t)) with the
// std::max/min tie rules spelled out (signed zeros, NaN behave identically).
__device__ __forceinline__ double clamp_box(double t, double lo) {
  const double a = lo < t ? t : lo;
  return a < 1.0 ? a : 1.0;
}

// ----------------------------------------------------------------- layout
// Chains per lane of the fused kernels: 4 (one 32-byte sector of X per
// lane per neighbour) for B >= 4, else 1.
inline int chains_per_lane(int B) { return B >= 4 ? 4 : 1; }

// Quads (lane work units) per row, padded so a row group is warp-aligned:
// a power of two <= 32, or a multiple of 32.
inline int quads_per_row(int B, int cpl) {
  int q = (B + cpl - 1) / cpl;
  if (q >= 32) return (q + 31) / 32 * 32;
  int p = 1;
  while (p < q) p <<= 1;
  return p;
}

// Per-chain trajectory control word (K2 state).
struct ChainCtl {
  int32_t active;
  int32_t iterations;
  int32_t reason;
  int32_t final_buf;
};

// Per-chain random stream: the full state of an mqo::Rng (rng.hpp:64-69),
// xoshiro words + the cached Box-Muller spare.  Layout == mqo_rng_state.
struct ChainRng {
  uint64_t s[4];
  double spare;
  int32_t has_spare;
  int32_t flags;  // bit 0: a rejection happened in the last parallel replay
};

// Packed solution bodies: vertex v is bit 63-(v&63) of word v>>6, so that
// comparing words as unsigned integers compares bodies lexicographically.
inline int64_t body_words(int32_t n) { return (static_cast<int64_t>(n) + 63) / 64; }

}  // namespace mqo_b200

// ------------------------------------------------------------- handles
struct mqo_batch;
namespace mqo_b200 {
// mem.cu: pinned host blocks from a process-wide cache (mapped, portable),
// and the per-device stream graph arrays are allocated / freed on
void* pinned_get(size_t bytes);
void pinned_put(void* p, size_t bytes);
cudaStream_t mem_stream(int device);
void keep_pool_memory(int device);
// Stream-ordered allocation of a batch buffer from the device's memory pool
// (freed with dfree on the batch stream).
template <typename T>
void dalloc(mqo_batch* b, T** p, size_t bytes);
void dfree(mqo_batch* b, void* p);
}  // namespace mqo_b200
struct mqo_graph {
  int device = 0;
  int32_t n = 0;
  int64_t m = 0;
  int32_t max_degree = 0;
  int64_t* d_off = nullptr;   // n+1
  int32_t* d_nbr = nullptr;   // 2m
  int32_t* d_order = nullptr; // rows by degree descending (stable by id)
  int32_t* d_cta = nullptr;   // slot layout of the SMEM trajectory path (lazy)
  int32_t* d_hmax = nullptr;  // max degree over higher neighbours (2-flip filter, lazy)
  int32_t* d_lo = nullptr;    // lower-neighbour count per row (1-flip rounds, lazy)
  int32_t* d_crow = nullptr;  // row of every 32nd CSR entry (edge-parallel cut, lazy)
  int64_t cta_words = 0;
  std::vector<int32_t> h_cta_rows, h_cta_base;  // per-slice rows / ELL base (host copy)
  // host copy of the CSR: filled at upload for host-only graphs, downloaded on
  // first use (mqo_b200::host_csr) for device graphs -- the upload itself
  // never touches the caller's neighbour array on the host
  std::vector<int64_t> h_off;
  std::vector<int32_t> h_nbr;
  bool h_csr = false;
  std::mutex host_mu;
  std::vector<int32_t> h_deg_ge;  // [max_degree + 2]: rows of degree >= d (heavy-row planning)
  std::mutex lazy_mu;  // guards the lazily built fields (d_cta, d_hmax): a graph may be
                       // shared by solves running on several host threads
};
namespace mqo_b200 {
// the host CSR of g (downloaded once for device graphs; thread-safe)
void host_csr(const mqo_graph* g);
// this host thread runs an engine rank that shares its GPU with another
// rank of the same process (mqo_solve_devices): no SMEM trajectory kernel
extern thread_local bool g_tls_no_cta_traj;
}  // namespace mqo_b200

struct mqo_batch {
  mqo_graph* g = nullptr;
  int32_t B = 0;    // chains
  int32_t cpl = 1;  // chains per lane
  int32_t Q = 1;    // quads (lane units) per row
  int32_t Bp = 0;   // padded chain stride = Q * cpl
  cudaStream_t stream = nullptr;
  double* d_x[2] = {nullptr, nullptr};  // vertex-major [n][Bp], double buffered
  double* d_v = nullptr;                // [n][Bp]
  double* d_aux = nullptr;              // [n][Bp] staging / gradient output (lazy)
  int cur = 0;                          // buffer holding the current x
  mqo_b200::ChainCtl* d_ctl = nullptr;  // [Bp]
  uint32_t* d_viol = nullptr;           // [3][Bp] MIS checker accumulators
  unsigned long long* d_chg = nullptr;  // [3][Bp] max |dx| accumulators (bits)
  int32_t* d_flag = nullptr;            // misc device flags [4]
  uint8_t* d_qmask = nullptr;           // [Q] active-chain mask per quad
  int32_t* h_flag = nullptr;            // pinned mirror [4]
  int coop_blocks = 0;                  // resident CTAs for the persistent kernel
  // solver state (solver.cu)
  mqo_b200::ChainRng* d_rng = nullptr;  // [Bp] per-chain streams
  uint64_t* d_pool = nullptr;           // [pool_cap][W] packed pool bodies
  int32_t pool_cap = 0, pool_size = 0;
  uint64_t* d_bodies = nullptr;         // [Bp][W] packed harvested bodies
  int64_t* d_scores = nullptr;          // [Bp]
  int32_t* d_valid = nullptr;           // [Bp]
  int32_t* d_pick = nullptr;            // [Bp] pool index drawn per chain
  uint8_t* d_state8 = nullptr;          // [n][Bp] harvest / local-search states
  uint32_t* d_sides = nullptr;          // [n][4*ceil(B/128)] MaxCut side bits, chain-minor
  int32_t* d_lastw = nullptr;           // [Bp][n] reset scratch
  int32_t* d_jdraw = nullptr;           // [Bp][n] reset draws j_i
  int32_t* d_counter = nullptr;         // [4] device counters
  uint64_t* d_ls = nullptr;             // mqo_local_search staging (device, grow-only)
  int32_t* d_flip = nullptr;            // 1-flip closure state [2][count * n] + 3 count (grow-only)
  size_t flip_bytes = 0;
  uint64_t* h_ls = nullptr;             // ... and its pinned host mirror
  size_t ls_bytes = 0;
};

namespace mqo_b200 {
template <typename T>
void dalloc(mqo_batch* b, T** p, size_t bytes) {
  void* q = nullptr;
  MQO_CUDA(cudaMallocAsync(&q, std::max<size_t>(bytes, 1), b->stream));
  *p = static_cast<T*>(q);
}
inline void dfree(mqo_batch* b, void* p) {
  if (p) cudaFreeAsync(p, b->stream);
}
}  // namespace mqo_b200
