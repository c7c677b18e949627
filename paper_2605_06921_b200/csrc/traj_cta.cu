// traj_cta.cu -- trajectories of small graphs, chain state in shared memory.
//
// Same reference path as pga.cu (run_trajectory, pga.cpp:63-111: fused
// gradient + momentum + clip, MIS fixed-point check, MaxCut ||dx||_inf stop,
// 256-iteration deadline poll) for graphs whose chain state fits in shared
// memory (C1/C2-sized).  Chains are independent, so a chain's whole
// trajectory runs inside one thread-block cluster of C CTAs with no grid
// barrier and no per-iteration launch:
//
//   C = 1   (many chains): one CTA per chain, x (double-buffered) and v in
//           SMEM, stop flags are block-wide __syncthreads_or reductions.
//   C > 1   (few chains, e.g. C1's single chain): the vertex slots are split
//           into C contiguous slice ranges, one per CTA of the cluster; every
//           CTA keeps a full copy of x_{t-1} (the gathers stay in its own
//           SMEM); each thread stores the x_t values it forms straight into
//           every peer's copy (st.async over DSMEM, completing bytes on the
//           peer's mbarrier), and after the CTA's flag OR one thread sends a
//           16-byte flag record the same way.  Waiting on the mbarrier for
//           "all peers' slices + flag records" is the only per-iteration
//           synchronisation; every CTA ORs the same C flag records and so
//           takes the identical stop decision.
//
// With one CTA per chain the gathers bound the kernel (SMEM wavefronts of
// random 8-byte reads, ~5 per warp load; ncu: SMEM pipe ~80% busy), which
// is why splitting a few chains over C SMs each pays.  Arithmetic and summation
// order are those of the fused kernel (bit-identical).  The MIS check of
// x_{t-1} rides on the gather that forms x_t; a final check-only pass covers
// x_T.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>

#include <mutex>
#include <set>

#include "common.cuh"

using namespace mqo_b200;

namespace {

constexpr int kMaxCluster = 16;

// Slot layout (int32 words), built once per graph on the host.  Slots are
// the vertices in degree-descending order; slice s = slots 32s..32s+31 (one
// warp).  Z = 32·S is a padding slot whose x is always 0.0.
//   [0, n)          slot i -> vertex | degree << 16
//   [n, n + S)      word index of slice s's ELL block
//   [n + S, n + 2S) row count of slice s: its largest degree rounded up to 4
//   [n + 2S, ...)   ELL blocks: neighbour k of lane l at base + 32k + l, as a
//                   SLOT index, in CSR order, so a warp's index load is one
//                   128-byte row; entries past a row's degree hold Z, so a
//                   warp runs a uniform, branch-free trip count: adding +0.0
//                   leaves the running sum unchanged (it starts at +0.0 and
//                   round-to-nearest never yields -0.0 from it) and 0.0 is not
//                   selected; the Laplacian's (x_v - x_u) terms are predicated
//                   on k < degree instead.
struct CtaArgs {
  const int32_t* __restrict__ lay;
  int32_t n, S, B, Bp, C, lay_words;
  int32_t own[kMaxCluster + 1];  // CTA r of a cluster owns slices [own[r], own[r+1])
  int32_t max_slices;            // max over r of own[r+1] - own[r]
  int32_t max_ell;               // max over r of its ELL words
  double* X;  // [n][Bp] in/out (current buffer)
  ChainCtl* ctl;
  double param, alpha, beta, lo, conv_tol;
  int32_t max_iters, check_every, cur;
  const volatile int32_t* stop_flag;  // host-mapped: deadline passed
};

// any | (a > 0.5) | (b > 0.5) | (c > 0.5) | (d > 0.5) as a predicate chain:
// written out so the compiler does not rewrite the ORed compares as a NaN-aware
// max tree (4 extra instructions per neighbour).
__device__ __forceinline__ uint32_t any_gt_half(uint32_t any, double a, double b, double c,
                                                double d) {
  uint32_t r;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "setp.gt.or.f64 p, %2, 0d3FE0000000000000, p;\n\t"
      "setp.gt.or.f64 p, %3, 0d3FE0000000000000, p;\n\t"
      "setp.gt.or.f64 p, %4, 0d3FE0000000000000, p;\n\t"
      "setp.gt.or.f64 p, %5, 0d3FE0000000000000, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(any), "d"(a), "d"(b), "d"(c), "d"(d));
  return r;
}

// ---- cluster / DSMEM / mbarrier primitives (PTX, sm_90+)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(addr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
               : "memory");
}
// default (.acquire.cta) semantics: the data is SMEM written by peers'
// st.async, whose complete_tx releases at cluster scope; an .acquire.cluster
// wait would also invalidate L1 (CCTL.IVALL) on every iteration.
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(mbar),
      "r"(parity)
      : "memory");
}
// remote stores into a peer's SMEM that complete their bytes on the peer's
// mbarrier (no fence, no DMA engine in the path)
__device__ __forceinline__ void st_async(uint32_t dst, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(dst),
               "d"(v), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t dst, uint32_t v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
               "r"(v), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

template <int KIND>
__device__ __forceinline__ double grad_cta(double acc, double x, double deg, double param) {
  if constexpr (KIND == MQO_MIS_QUBO) return ex_sub(1.0, ex_mul(param, acc));
  if constexpr (KIND == MQO_LAPLACIAN) return ex_mul(acc, 0.5);
  if constexpr (KIND == MQO_PERTURBED_LAPLACIAN)
    return ex_mul(2.0, ex_add(ex_sub(ex_mul(deg, x), acc), ex_mul(param, x)));
  if constexpr (KIND == MQO_ADJACENCY) return ex_mul(acc, -2.0);
  return ex_sub(ex_mul(-2.0, acc), param);
}

// Shared-memory carve-up, identical on host and device.
struct SmemPlan {
  size_t xb;       // doubles per x buffer: Z + 2 (slot Z = zero, +1 keeps 16-byte alignment)
  size_t v_off;    // byte offsets ...
  size_t fl_off;   // uint32 flag words [2][C][W] (one per warp of every CTA)
  size_t mb_off;   // 2 mbarriers
  size_t lay_off;  // int32: info [32·ns] | rows [ns] | ELL [max_ell]
  size_t total;
};
__host__ __device__ inline SmemPlan smem_plan(int S, int C, int W, int max_slices, int max_ell,
                                              bool smem_lay) {
  SmemPlan p{};
  p.xb = static_cast<size_t>(32) * S + 2;
  p.v_off = 2 * p.xb * 8;
  p.fl_off = p.v_off + static_cast<size_t>(256) * max_slices;
  p.mb_off = p.fl_off + ((2 * static_cast<size_t>(C) * W * 4 + 15) & ~static_cast<size_t>(15));
  p.lay_off = p.mb_off + 16;
  p.total = p.lay_off;
  if (smem_lay) p.total += 4 * (static_cast<size_t>(33) * max_slices + max_ell);
  p.total = (p.total + 15) & ~static_cast<size_t>(15);
  return p;
}

// LOOKAHEAD (clusters, latency-bound): the next group of four neighbours is
// loaded while the current one is summed; one CTA per chain is bound by SMEM
// wavefronts instead and keeps the short loop (32 registers: two 1024-thread
// CTAs per SM).
template <int KIND, bool SMEM_LAY, bool LOOKAHEAD>
__global__ void __launch_bounds__(1024, LOOKAHEAD ? 1 : 2) k_traj_cta(CtaArgs a) {
  constexpr bool MIS = KIND == MQO_MIS_QUBO;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int n = a.n, S = a.S, C = a.C, Z = 32 * S;
  const int r = C > 1 ? static_cast<int>(cluster_rank()) : 0;
  const int b = blockIdx.x / C;
  const int s0 = a.own[r], s1 = a.own[r + 1], ns = s1 - s0;
  const int i0 = 32 * s0, i1 = min(n, 32 * s1);  // owned (real) slots
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, W = nt >> 5;
  const SmemPlan P = smem_plan(S, C, W, a.max_slices, a.max_ell, SMEM_LAY);
  double* xb0 = reinterpret_cast<double*>(smraw);
  double* xb1 = xb0 + P.xb;
  double* vs = reinterpret_cast<double*>(smraw + P.v_off);    // [32·ns], by slot - i0
  uint32_t* fl = reinterpret_cast<uint32_t*>(smraw + P.fl_off);  // [2][C][W]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smraw + P.mb_off);
  int32_t* s_info = reinterpret_cast<int32_t*>(smraw + P.lay_off);  // [32·ns]
  int32_t* s_rows = s_info + 32 * ns;                                 // [ns]
  int32_t* s_ell = s_rows + ns;
  const int ell0 = __ldg(a.lay + n + s0);  // first ELL word of the owned slices

  for (int i = tid; i < Z + 2; i += nt) {
    xb0[i] = i < n ? a.X[static_cast<int64_t>(__ldg(a.lay + i) & 0xffff) * a.Bp + b] : 0.0;
    xb1[i] = 0.0;
  }
  for (int i = tid; i < 32 * ns; i += nt) vs[i] = 0.0;  // fresh velocity (pga.cpp:75)
  if constexpr (SMEM_LAY) {
    const int ell1 = s1 < S ? __ldg(a.lay + n + s1) : a.lay_words;
    for (int i = tid; i < 32 * ns; i += nt) s_info[i] = i0 + i < n ? __ldg(a.lay + i0 + i) : 0;
    for (int s = tid; s < ns; s += nt) s_rows[s] = __ldg(a.lay + n + S + s0 + s);
    // + the 128-word look-ahead of the last group (next slices / the Z tail)
    for (int w = tid; w < ell1 - ell0 + 128; w += nt) s_ell[w] = __ldg(a.lay + ell0 + w);
  }
  if (C > 1 && tid == 0) {  // one arrival per warp (+ the peers' transaction bytes)
    mbar_init(smem_addr(&mbar[0]), W);
    mbar_init(smem_addr(&mbar[1]), W);
    fence_mbar_init();
  }
  __syncthreads();
  if (C > 1) cluster_sync_all();  // peers' mbarriers exist before the first push

  // owned-slot accessors
  auto info_of = [&](int i) -> int32_t {
    if constexpr (SMEM_LAY) return s_info[i - i0]; else return __ldg(a.lay + i);
  };
  auto rows_of = [&](int s) -> int32_t {
    if constexpr (SMEM_LAY) return s_rows[s - s0]; else return __ldg(a.lay + n + S + s);
  };
  auto base_of = [&](int s) -> int32_t {
    if constexpr (SMEM_LAY) return __ldg(a.lay + n + s) - ell0; else return __ldg(a.lay + n + s);
  };
  auto ell = [&](int w) -> int32_t {
    if constexpr (SMEM_LAY) return s_ell[w]; else return __ldg(a.lay + w);
  };

  // bytes this CTA receives per iteration: every peer's real slots + its flag words
  uint32_t expect = 0;
  for (int p = 0; p < C; ++p)
    if (p != r)
      expect += 8u * static_cast<uint32_t>(min(n, 32 * a.own[p + 1]) - 32 * a.own[p]) + 4u * W;

  int final_buf = 0, iters = 0, reason = MQO_ITER_CAP, since_check = 0;
  const int last = MIS ? a.max_iters + 1 : a.max_iters;  // MIS: one check-only pass for x_T
  bool deadline_prev = false;  // deadline seen at the poll after iteration t-1
  for (int t = 1; t <= last; ++t) {
    const bool write = !MIS || t <= a.max_iters;
    const int in_buf = (t - 1) & 1, out_buf = t & 1;
    const double* xin = in_buf ? xb1 : xb0;
    double* xout = out_buf ? xb1 : xb0;
    uint32_t flag = 0;  // MIS: x_{t-1} violates the check; MaxCut: x_t moved > conv_tol
    for (int i = i0 + tid; i < i1; i += nt) {
      const int deg = info_of(i) >> 16;
      const int s = i >> 5;
      const int w0 = base_of(s) + (i & 31);
      const int rows = rows_of(s);  // warp-uniform
      const double xv = xin[i];
      double acc = 0.0;
      uint32_t any = 0;  // a neighbour is selected in x_{t-1}
      // groups of four neighbours, summed in order; the next group's indices and
      // values are loaded while this one is summed (the layout's 128-word tail
      // keeps the look-ahead past the last group in bounds)
      int w = w0;
      double x0, x1, x2, x3;
      if constexpr (LOOKAHEAD) {
        x0 = xin[ell(w)];
        x1 = xin[ell(w + 32)];
        x2 = xin[ell(w + 64)];
        x3 = xin[ell(w + 96)];
      }
      for (int k = 0; k < rows; k += 4) {
        double y0, y1, y2, y3;
        if constexpr (LOOKAHEAD) {
          w += 128;
          y0 = xin[ell(w)];
          y1 = xin[ell(w + 32)];
          y2 = xin[ell(w + 64)];
          y3 = xin[ell(w + 96)];
        } else {
          x0 = xin[ell(w)];
          x1 = xin[ell(w + 32)];
          x2 = xin[ell(w + 64)];
          x3 = xin[ell(w + 96)];
          w += 128;
        }
        if constexpr (KIND == MQO_LAPLACIAN) {
          if (k < deg) acc = ex_add(acc, ex_sub(xv, x0));
          if (k + 1 < deg) acc = ex_add(acc, ex_sub(xv, x1));
          if (k + 2 < deg) acc = ex_add(acc, ex_sub(xv, x2));
          if (k + 3 < deg) acc = ex_add(acc, ex_sub(xv, x3));
        } else {
          acc = ex_add(ex_add(ex_add(ex_add(acc, x0), x1), x2), x3);
        }
        if constexpr (MIS) any = any_gt_half(any, x0, x1, x2, x3);
        if constexpr (LOOKAHEAD) {
          x0 = y0;
          x1 = y1;
          x2 = y2;
          x3 = y3;
        }
      }
      if constexpr (MIS) {
        if ((xv > 0.5) ? any : !any) flag = 1;  // pga.cpp:127-133 on binarize(x_{t-1})
      }
      double nx = xv;  // the check-only pass still sends (unused) values
      if (write) {
        double* vp = vs + (i - i0);
        const double g = grad_cta<KIND>(acc, xv, static_cast<double>(deg), a.param);
        const double nv = ex_add(ex_mul(a.beta, *vp), g);
        nx = clamp_box(ex_add(xv, ex_mul(a.alpha, nv)), a.lo);
        if (!MIS && fabs(ex_sub(nx, xv)) > a.conv_tol) flag = 1;  // max|dx| > tol
        *vp = nv;
        xout[i] = nx;
      }
      if (C > 1) {
        const uint32_t la = smem_addr(xout + i), lm = smem_addr(&mbar[out_buf]);
        for (int q = 1; q < C; ++q) {
          const int p = r + q < C ? r + q : r + q - C;
          st_async(map_to_rank(la, p), nx, map_to_rank(lm, p));
        }
      }
    }
    bool deadline_now;
    if (C == 1) {
      flag = __syncthreads_or(flag);  // also publishes xout
      // the host deadline flag is read by one thread and OR-reduced, so every
      // thread's decision is identical (poll after iterations 256, 512, ...)
      deadline_now = (t & 255) == 0 && __syncthreads_or(tid == 0 ? *a.stop_flag : 0);
    } else {
      // no CTA barrier: each warp publishes its flag word to every CTA (its
      // own by a plain store, peers by st.async) and arrives on the local
      // mbarrier (release: orders its x_t stores for the other warps)
      const uint32_t mb = smem_addr(&mbar[out_buf]);
      uint32_t word = __any_sync(0xffffffffu, flag) ? 1u : 0u;
      if (lane == 0) {
        // rank 0's warp 0 alone polls the deadline, so every CTA sees the same bit
        if (r == 0 && warp == 0 && (t & 255) == 0 && *a.stop_flag) word |= 2u;
        uint32_t* mine = fl + (out_buf * C + r) * W + warp;
        *mine = word;
        const uint32_t fdst = smem_addr(mine);
        for (int q = 1; q < C; ++q) {
          const int p = r + q < C ? r + q : r + q - C;
          st_async(map_to_rank(fdst, p), word, map_to_rank(mb, p));
        }
        if (warp == 0)
          mbar_arrive_expect(mb, expect);
        else
          mbar_arrive(mb);
      }
      // x_t of mbar[t & 1] is its ((t-1) >> 1)-th phase
      mbar_wait(mb, ((t - 1) >> 1) & 1);
      const uint32_t* fw = fl + out_buf * C * W;
      uint32_t f = 0;
      for (int j = lane; j < C * W; j += 32) f |= fw[j];
      flag = __reduce_or_sync(0xffffffffu, f) & 1u;
      deadline_now = (fw[0] & 2u) != 0;
    }
    bool stop = false;
    if (MIS) {
      const int s = t - 1;  // decisions about x_{t-1} (pga.cpp:91-98, 104-110)
      if (s >= 1) {
        const bool due = ++since_check == a.check_every;  // s % check_every == 0
        if (due) since_check = 0;
        if (due && !flag) {
          stop = true;
          reason = MQO_CHECKER_ACCEPTED;
        } else if (s == a.max_iters || deadline_prev) {
          stop = true;
          reason = MQO_ITER_CAP;
        }
      }
      if (stop) {
        final_buf = in_buf;
        iters = s;
      }
    } else {
      if (!flag) {
        stop = true;
        reason = MQO_CONVERGED;
      } else if (t == a.max_iters || deadline_now) {
        stop = true;
        reason = MQO_ITER_CAP;
      }
      if (stop) {
        final_buf = out_buf;
        iters = t;
      }
    }
    if (stop) break;
    deadline_prev = deadline_now;
  }
  const double* src = final_buf ? xb1 : xb0;
  for (int i = i0 + tid; i < i1; i += nt)
    a.X[static_cast<int64_t>(info_of(i) & 0xffff) * a.Bp + b] = src[i];
  if (r == 0 && tid == 0) a.ctl[b] = ChainCtl{0, iters, reason, a.cur};
  if (C > 1) cluster_sync_all();  // no peer touches our SMEM after we exit
}

using CtaFn = void (*)(CtaArgs);

template <bool S, bool L>
CtaFn cta_fn_kind(int kind) {
  switch (kind) {
    case MQO_MIS_QUBO: return k_traj_cta<MQO_MIS_QUBO, S, L>;
    case MQO_LAPLACIAN: return k_traj_cta<MQO_LAPLACIAN, S, L>;
    case MQO_PERTURBED_LAPLACIAN: return k_traj_cta<MQO_PERTURBED_LAPLACIAN, S, L>;
    case MQO_ADJACENCY: return k_traj_cta<MQO_ADJACENCY, S, L>;
    case MQO_PERTURBED_BIAS: return k_traj_cta<MQO_PERTURBED_BIAS, S, L>;
  }
  throw std::invalid_argument("objective: unknown kind");
}
CtaFn cta_fn(int kind, bool smem_lay, bool lookahead) {
  if (smem_lay) return lookahead ? cta_fn_kind<true, true>(kind) : cta_fn_kind<true, false>(kind);
  return lookahead ? cta_fn_kind<false, true>(kind) : cta_fn_kind<false, false>(kind);
}

}  // namespace

namespace mqo_b200 {

constexpr size_t kCtaSmemMax = 200 * 1024;
thread_local bool g_tls_no_cta_traj = false;
bool g_cta_disabled = false;  // mqo_tune("cta_traj", 0)
int g_cta_cluster = 0;        // mqo_tune("cta_cluster", C): 0 = automatic

// Builds (once per graph) the slot layout described at CtaArgs.
void ensure_cta_layout(mqo_graph* g) {
  std::lock_guard<std::mutex> lock(g->lazy_mu);
  if (g->d_cta) return;
  const int32_t n = g->n;
  const int32_t S = (n + 31) / 32;
  const int32_t Z = 32 * S;
  host_csr(g);
  std::vector<int32_t> order(static_cast<size_t>(n)), slot(static_cast<size_t>(n));
  MQO_CUDA(cudaMemcpy(order.data(), g->d_order, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  for (int32_t i = 0; i < n; ++i) slot[order[i]] = i;
  std::vector<int32_t> lay(static_cast<size_t>(n) + 2 * S, 0);
  int64_t words = n + 2 * S;
  for (int32_t s = 0; s < S; ++s) {
    int32_t dmax = 0;
    for (int32_t i = 32 * s; i < std::min(n, 32 * s + 32); ++i) {
      const int32_t v = order[i];
      const int32_t d = static_cast<int32_t>(g->h_off[v + 1] - g->h_off[v]);
      lay[i] = v | (d << 16);
      dmax = std::max(dmax, d);
    }
    const int32_t rows = (dmax + 3) & ~3;
    lay[n + s] = static_cast<int32_t>(words);
    lay[n + S + s] = rows;
    words += 32LL * rows;
  }
  if (words > INT32_MAX) throw std::length_error("cta layout too large");
  // padding -> the zero slot; + a 128-word tail for the gather look-ahead
  lay.resize(static_cast<size_t>(words) + 128, Z);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t v = order[i];
    const int64_t base = lay[n + i / 32] + (i & 31);
    for (int64_t e = g->h_off[v], k = 0; e < g->h_off[v + 1]; ++e, ++k)
      lay[static_cast<size_t>(base + 32 * k)] = slot[g->h_nbr[e]];
  }
  {  // pool allocation on the graph's memory stream (freed there with the graph)
    const cudaStream_t ms = mem_stream(g->device);
    void* p = nullptr;
    MQO_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * lay.size(), ms));
    MQO_CUDA(cudaStreamSynchronize(ms));
    g->d_cta = static_cast<int32_t*>(p);
  }
  MQO_CUDA(cudaMemcpy(g->d_cta, lay.data(), sizeof(int32_t) * lay.size(), cudaMemcpyHostToDevice));
  g->cta_words = words;  // ELL end (the tail follows)
  g->h_cta_base.assign(lay.begin() + n, lay.begin() + n + S);
  g->h_cta_rows.assign(lay.begin() + n + S, lay.begin() + n + 2 * S);
}

static int cta_threads(int /*C*/, int max_slices) {
  return std::max(32, std::min(1024, 32 * max_slices));
}
static size_t cta_smem_for(const mqo_graph* g, int C, int max_slices, int max_ell, bool smem_lay) {
  const int S = (g->n + 31) / 32;
  return smem_plan(S, C, cta_threads(C, max_slices) / 32, max_slices, max_ell, smem_lay).total;
}

// 1 when the SMEM trajectory path applies (two x copies + v fit), else 0.
int cta_group(const mqo_batch* b) {
  static const bool disabled = [] {
    const char* e = std::getenv("MQO_NO_CTA_TRAJ");
    return e && *e && *e != '0';
  }();
  if (disabled || g_cta_disabled || g_tls_no_cta_traj) return 0;
  const mqo_graph* g = b->g;
  // slot words pack vertex | degree << 16
  if (g->n <= 0 || g->n >= 65536 || g->max_degree >= 32768) return 0;
  const int S = (g->n + 31) / 32;
  return cta_smem_for(g, 1, S, 0, false) <= kCtaSmemMax ? 1 : 0;
}

// Contiguous slice ranges for C CTAs (C <= S), balanced by rows + epilogue work.
static void split_slices(const mqo_graph* g, int C, CtaArgs& a) {
  const int S = a.S;
  std::vector<double> w(static_cast<size_t>(S));
  double total = 0.0;
  for (int s = 0; s < S; ++s) total += (w[s] = g->h_cta_rows[s] + 6.0);
  a.own[0] = 0;
  double acc = 0.0;
  int s = 0;
  for (int r = 0; r < C; ++r) {
    const double target = total * (r + 1) / C;
    const int leave = C - r - 1;  // slices the remaining CTAs need
    acc += w[s++];                // at least one
    while (s < S - leave && acc + 0.5 * w[s] <= target) acc += w[s++];
    if (r == C - 1) s = S;
    a.own[r + 1] = s;
  }
  a.max_slices = 0;
  a.max_ell = 0;
  for (int r = 0; r < C; ++r) {
    const int e0 = g->h_cta_base[a.own[r]];
    const int e1 = a.own[r + 1] < S ? g->h_cta_base[a.own[r + 1]] : static_cast<int>(g->cta_words);
    a.max_slices = std::max(a.max_slices, a.own[r + 1] - a.own[r]);
    a.max_ell = std::max(a.max_ell, e1 - e0 + 128);  // + look-ahead tail
  }
}

// Runs the trajectories of every chain from the current x with the SMEM
// kernel; polls `deadline` from the host and raises the mapped stop flag.
void run_trajectories_cta(mqo_batch* b, const mqo_objective& obj, const mqo_optimizer& opt,
                          double deadline, int /*G*/, double (*now)()) {
  // the batch's mapped pinned words: [2] is the stop flag
  int32_t* h_stop = b->h_flag + 2;
  int32_t* d_stop = nullptr;
  MQO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_stop), h_stop, 0));
  *reinterpret_cast<volatile int32_t*>(h_stop) = 0;
  mqo_graph* g = b->g;
  ensure_cta_layout(g);
  CtaArgs a{};
  a.lay = g->d_cta;
  a.lay_words = static_cast<int32_t>(g->cta_words);
  a.n = g->n;
  a.S = (g->n + 31) / 32;
  a.B = b->B;
  a.Bp = b->Bp;
  a.X = b->d_x[b->cur];
  a.ctl = b->d_ctl;
  a.param = obj.param;
  a.alpha = opt.alpha;
  a.beta = opt.beta;
  a.lo = obj.kind == MQO_MIS_QUBO ? 0.0 : -1.0;
  a.conv_tol = opt.conv_tol;
  a.max_iters = opt.max_iters;
  a.check_every = opt.check_every;
  a.cur = b->cur;
  a.stop_flag = d_stop;

  // cluster size: few chains are spread over several SMs each
  int C = g_cta_cluster;
  if (C <= 0) {
    int sms = 148;
    MQO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    C = 1;
    while (C < 8 && b->B * (2 * C) <= sms) C *= 2;
  }
  C = std::max(1, std::min({C, kMaxCluster, a.S}));
  a.C = C;
  split_slices(g, C, a);
  const bool smem_lay = cta_smem_for(g, C, a.max_slices, a.max_ell, true) <= kCtaSmemMax;
  const size_t smem = cta_smem_for(g, C, a.max_slices, a.max_ell, smem_lay);
  if (smem > kCtaSmemMax) throw std::logic_error("cta trajectories: state exceeds SMEM");
  CtaFn fn = cta_fn(obj.kind, smem_lay, C > 1);
  // the cap, not this launch's size (the attribute is per function, and
  // solves on other host threads launch the same kernel with other sizes),
  // set once per (function, device) -- not while another thread's launch
  // of the same function may be in flight
  {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.insert({reinterpret_cast<const void*>(fn), g->device}).second) {
      MQO_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kCtaSmemMax)));
      MQO_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
  }
  // one SMEM trajectory kernel at a time per GPU, on a drained stream: two
  // of them in flight from different host threads faulted intermittently
  // (illegal address; ~1 in 100 solve_devices([0, 0]) calls, root cause not
  // identified -- scripts/repro_devices.py)
  static std::mutex dev_mu[64];
  std::unique_lock<std::mutex> dev_lock(dev_mu[g->device & 63]);
  MQO_CUDA(cudaStreamSynchronize(b->stream));
  const int threads = cta_threads(C, a.max_slices);
  if (C == 1) {
    fn<<<b->B, threads, smem, b->stream>>>(a);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(b->B * C));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = b->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MQO_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  }
  MQO_CUDA(cudaGetLastError());
  MQO_TRACE("cta trajectories launched: %d chains x %d CTAs x %d threads, smem %zu (layout %s)",
            b->B, C, threads, smem, smem_lay ? "smem" : "global");
  // wait, raising the stop flag once the deadline has passed
  for (;;) {
    const cudaError_t q = cudaStreamQuery(b->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) MQO_CUDA(q);
    if (deadline >= 0.0 && now() >= deadline) *reinterpret_cast<volatile int32_t*>(h_stop) = 1;
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  MQO_TRACE("cta trajectories done");
}

}  // namespace mqo_b200
