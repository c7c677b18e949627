// pga.cu -- K1 `pga_step_fused` and K2 trajectory control: the hot path.
//
// Reference path replaced (relative to /root/reference/proj/core/):
//   Graph::adjacency_apply / laplacian_apply   graph.cpp:63-88   (the SpMV)
//   gradient epilogues                         objectives.cpp:101-134
//   step / run_trajectory loop body            pga.cpp:51-61, 79-88
//   MIS binarize + mis_fixed_point_check       pga.cpp:91-98, 113-135
//   MaxCut ||dx||_inf stop, deadline poll      pga.cpp:99-107
//
// One pass = one PGA iteration of every active chain.  Work unit = (row v,
// quad q): a lane owns CPL (4) consecutive chains of row v and gathers
// X[u][4q..4q+3] (one 32-byte sector) for every neighbour u of v, in CSR
// order, accumulating each chain sequentially -- the exact summation order
// of adjacency_apply, so every fp64 result is bit-identical.  Parallelism
// comes from rows x chains, never from splitting a row's sum.  The MIS
// fixed-point check of the previous iterate x_{t-1} is fused into the same
// gather (count of neighbours with x_u > 0.5), so it costs no extra bytes
// instead of the reference's second SpMV.  The MaxCut max|dx| is reduced
// per chain in the epilogue.
//
// Trajectories run as a cooperative persistent kernel: passes separated by
// grid.sync(); every CTA takes the (identical, redundant) per-chain stop
// decision after the barrier, CTA 0 records it.  Per-chain accumulators are
// triple-buffered by pass so no extra barrier is needed to reset them.
#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <ctime>

#include "common.cuh"

namespace cg = cooperative_groups;
using namespace mqo_b200;

namespace mqo_b200 {
extern bool g_cta_disabled;
extern int g_cta_cluster;
int cta_group(const mqo_batch* b);
void run_trajectories_cta(mqo_batch* b, const mqo_objective& obj, const mqo_optimizer& opt,
                          double deadline, int G, double (*now)());
double* aux_buffer(mqo_batch* b);
void upload_chain_major(mqo_batch* b, const double* host, double* dst);
void download_chain_major(mqo_batch* b, const double* src, double* host);
void launch_project(mqo_batch* b, double* x, int32_t problem);
}  // namespace mqo_b200

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

enum Mode : int { kStep = 0, kGrad = 1, kCheck = 2, kTraj = 3 };

struct PassArgs {
  const int64_t* __restrict__ off;
  const int32_t* __restrict__ nbr;
  const int32_t* __restrict__ order;
  int32_t n, B, Bp, Q;
  double* x[2];
  double* v;
  double* gout;
  double param, alpha, beta, lo;
  ChainCtl* ctl;
  uint32_t* viol;            // [3][Bp]
  unsigned long long* chg;   // [3][Bp]
  int32_t* flag;             // [0] active count, [1] non-binary flag
  int32_t base;              // buffer index holding x_0 (kTraj) / current x
  int32_t p_begin, p_end;    // passes [p_begin, p_end)
  int32_t T;                 // last iterate of the trajectory
  int32_t check_every;
  double conv_tol;
  int32_t is_mis;
  int32_t hot_rows;          // gathers of rows < hot_rows are kept in L2 (evict_last)
  int32_t q0, Qg;            // this launch's chain group: quads [q0, q0 + Qg) of Q
  uint8_t* qmask;            // [Q] active-chain mask per quad (per-launch path)
  int32_t cpl;
  // Heavy rows (see heavy_row): order[0, heavy) are staged through SMEM by
  // whole CTAs -- the first hblocks CTAs of every chain group -- and the
  // per-lane path walks rows [heavy, n) with the lblocks CTAs after them.
  int32_t heavy;             // rows of degree >= the heavy threshold (a prefix of order)
  int32_t hblocks, lblocks;  // CTAs per chain group for heavy / light rows (lblocks 0: rest)
  int32_t stage_doubles;     // SMEM staging capacity (doubles) of a heavy CTA
  int32_t stage_off;         // byte offset of the staging buffer in dynamic SMEM
  int32_t fuse_ctl;          // k_traj_pass: the last CTA of the pass runs k_traj_ctl's work
};

// Compile-time tuning of the fused kernels: neighbours in flight per lane,
// minimum resident CTAs per SM (register cap), cache-policy hints.
// MEM: 0 = two 128-bit ld.cg per lane, 1 = one 256-bit load with L2
// eviction-priority policies, 2 = one 256-bit load without policies.
template <int U_, int MINB_, int MEM_, bool PREFETCH_ = false>
struct Tune {
  static constexpr int U = U_;
  static constexpr int MINB = MINB_;
  static constexpr int MEM = MEM_;
  static constexpr bool PREFETCH = PREFETCH_;  // next batch's neighbour ids loaded early
  static constexpr bool HINT = MEM_ != 0;  // 256-bit path
  static constexpr bool POLICY = MEM_ == 1 || MEM_ == 3;
  static constexpr bool L2_64B = MEM_ == 3;  // neighbour gathers with the L2::64B fetch size
};
// Measured on B200 (scripts/tune_k1.py, profiles/r01_tune_k1.txt): 4
// neighbours in flight x 3 CTAs/SM for the MaxCut objectives, 3 x 4 CTAs/SM
// for MIS (its checker counters add registers).
using TuneDefault = Tune<4, 3, 1>;
using TuneMis = Tune<3, 4, 1>;
// Hub graphs (BA-like degree skew), MaxCut objectives: the next batch's
// neighbour ids loaded one batch early (C4 16 chains 0.278 -> 0.247 ms, 128
// chains 1.956 -> 1.941 ms; on ER graphs it costs registers for nothing:
// C3 x 256 0.221 -> 0.272 ms, so those keep TuneDefault), and with the
// prefetch hiding a round trip, 5 neighbours in flight beat 4 (C4 0.250 ->
// 0.245 / 0.965 -> 0.954 / 1.939 -> 1.922 ms at 16 / 64 / 128 chains; 4x4,
// 6x2, 6x3, 8x2 and 3x4 measured slower or spilling: smallb_probe variants).
using TuneHub = Tune<5, 3, 1, true>;
// The trajectory pass carries the stop-rule state too: at 5 in flight it
// spills (79 regs + 32 B stack) and runs slower than 4 (C4 per pass 0.262 /
// 0.986 / 1.975 ms at 4 vs 0.264 / 1.003 / 1.993 at 5).
using TuneHubTraj = Tune<4, 3, 1, true>;
// MIS with chain-tiled (L2-resident) gathers: the prefetch trims the L2
// round trips (C3 x 256 0.221 -> 0.214 ms, at the measured L2 read
// bandwidth); untiled ER graphs keep TuneMis (C5 16 chains 4.61 vs 4.91 ms).
using TuneMisTiled = Tune<3, 4, 1, true>;
template <int KIND>
using TuneFor = std::conditional_t<KIND == MQO_MIS_QUBO, TuneMis, TuneDefault>;

// Cache policies: gathers of hot rows are marked L2::evict_last, every
// streamed access (own row, velocity, stores) L2::evict_first, and nothing
// allocates in L1 (random gathers have no L1 reuse).  One 256-bit access
// per lane covers its 4 chains (one 32-byte sector).
enum Pol : int { kPolNormal = 0, kPolLast = 1, kPolFirst = 2, kPolNormal64 = 3, kPolLast64 = 4 };

template <int POL>
__device__ __forceinline__ void ld4(const double* p, double (&o)[4]) {
  if constexpr (POL == kPolLast)
    asm volatile("ld.global.L1::no_allocate.L2::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  else if constexpr (POL == kPolFirst)
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  else if constexpr (POL == kPolNormal64)
    asm volatile("ld.global.L1::no_allocate.L2::64B.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  else if constexpr (POL == kPolLast64)
    asm volatile("ld.global.L1::no_allocate.L2::evict_last.L2::64B.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}

template <bool POLICY>
__device__ __forceinline__ void st4(double* p, const double (&o)[4]) {
  if constexpr (POLICY)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(o[0]), "d"(o[1]), "d"(o[2]), "d"(o[3]) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(o[0]), "d"(o[1]), "d"(o[2]), "d"(o[3]) : "memory");
}

template <int CPL>
__device__ __forceinline__ void ldx(const double* p, double (&o)[CPL]) {
  if constexpr (CPL == 4) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    o[0] = a.x;
    o[1] = a.y;
    o[2] = b.x;
    o[3] = b.y;
  } else {
    o[0] = __ldcg(p);
  }
}

template <int CPL>
__device__ __forceinline__ void stx(double* p, const double (&o)[CPL], unsigned mask) {
  if constexpr (CPL == 4) {
    if (mask == 0xF) {
      __stcg(reinterpret_cast<double2*>(p), make_double2(o[0], o[1]));
      __stcg(reinterpret_cast<double2*>(p) + 1, make_double2(o[2], o[3]));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (mask & (1u << c)) __stcg(p + c, o[c]);
    }
  } else {
    if (mask & 1u) __stcg(p, o[0]);
  }
}

// Gradient epilogues, objectives.cpp:109-133, operation by operation.
template <int KIND>
__device__ __forceinline__ double grad_epi(double acc, double x, double deg, double param) {
  if constexpr (KIND == MQO_MIS_QUBO) return ex_sub(1.0, ex_mul(param, acc));
  if constexpr (KIND == MQO_LAPLACIAN) return ex_mul(acc, 0.5);
  if constexpr (KIND == MQO_PERTURBED_LAPLACIAN)
    return ex_mul(2.0, ex_add(ex_sub(ex_mul(deg, x), acc), ex_mul(param, x)));
  if constexpr (KIND == MQO_ADJACENCY) return ex_mul(acc, -2.0);
  return ex_sub(ex_mul(-2.0, acc), param);  // PerturbedBias
}

// Per-thread accumulators of one pass (this thread's fixed quad).
template <int CPL>
struct Acc {
  // bit c: chain c of the quad violates the MIS fixed-point check (MIS), or
  // moved by more than conv_tol this pass (MaxCut: max|dx| <= conv_tol
  // <=> no element exceeds it, NaN ignored exactly like std::max does)
  unsigned viol = 0;
  unsigned nonbin = 0;   // kCheck: a state not in {0,1}
};

// One (row, quad) work unit.
template <int KIND, int CPL, int MODE, bool CHECK, class TU>
__device__ __forceinline__ void row_unit(const PassArgs& a, const double* __restrict__ X,
                                         double* __restrict__ Xo, int32_t v, int32_t col,
                                         unsigned amask, bool write, Acc<CPL>& acc) {
  constexpr int U = CPL == 4 ? TU::U : 16;
  constexpr bool HINT = CPL == 4 && TU::HINT;
  constexpr int kFirst = TU::POLICY ? kPolFirst : kPolNormal;
  const int64_t e0 = __ldg(a.off + v), e1 = __ldg(a.off + v + 1);
  const int64_t rowbase = static_cast<int64_t>(v) * a.Bp + col;
  double xv[CPL];
  if constexpr (HINT)
    ld4<kFirst>(X + rowbase, xv);
  else
    ldx<CPL>(X + rowbase, xv);
  double s[CPL];
  unsigned nbsel = 0;  // bit c: some neighbour of v is selected (x_u > 0.5) in chain c
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    s[c] = 0.0;
  }
  // neighbour ids one batch ahead: the next batch's index loads are in
  // flight while this batch's gathers are (one round trip per batch instead
  // of two on rows longer than U)
  int32_t nx[U];
#pragma unroll
  for (int j = 0; j < U; ++j) nx[j] = (e0 + j < e1) ? __ldg(a.nbr + e0 + j) : -1;
  for (int64_t e = e0; e < e1; e += U) {
    int32_t us[U];
#pragma unroll
    for (int j = 0; j < U; ++j) us[j] = nx[j];
    if constexpr (TU::PREFETCH) {
#pragma unroll
      for (int j = 0; j < U; ++j) nx[j] = (e + U + j < e1) ? __ldg(a.nbr + e + U + j) : -1;
    }
    double val[U][CPL];
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (us[j] >= 0) {
        const double* src = X + static_cast<int64_t>(us[j]) * a.Bp + col;
        if constexpr (HINT) {
          if (TU::POLICY && us[j] < a.hot_rows)
            ld4<TU::L2_64B ? kPolLast64 : kPolLast>(src, val[j]);
          else
            ld4<TU::L2_64B ? kPolNormal64 : kPolNormal>(src, val[j]);
        } else {
          ldx<CPL>(src, val[j]);
        }
      }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (us[j] < 0) break;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        if constexpr (KIND == MQO_LAPLACIAN)
          s[c] = ex_add(s[c], ex_sub(xv[c], val[j][c]));  // graph.cpp:85
        else
          s[c] = ex_add(s[c], val[j][c]);               // graph.cpp:68
        if constexpr (CHECK) nbsel |= (val[j][c] > 0.5 ? 1u : 0u) << c;
      }
    }
    if constexpr (!TU::PREFETCH) {
#pragma unroll
      for (int j = 0; j < U; ++j) nx[j] = (e + U + j < e1) ? __ldg(a.nbr + e + U + j) : -1;
    }
  }
  if constexpr (CHECK) {
    // pga.cpp:125-133 on binarize(x) (pga.cpp:93): selected vertices must
    // have no selected neighbour, unselected ones at least one.
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const bool sel = xv[c] > 0.5;
      const bool any = (nbsel >> c) & 1u;  // count > 0 (pga.cpp:127-133)
      const bool bad = sel ? any : !any;
      if (bad && (amask & (1u << c))) acc.viol |= 1u << c;
      if constexpr (MODE == kCheck)
        if (xv[c] != 0.0 && xv[c] != 1.0 && (amask & (1u << c))) acc.nonbin = 1;
    }
  }
  if constexpr (MODE == kCheck) return;
  const double deg = static_cast<double>(e1 - e0);
  double g[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) g[c] = grad_epi<KIND>(s[c], xv[c], deg, a.param);
  if constexpr (MODE == kGrad) {
    stx<CPL>(a.gout + rowbase, g, amask);
    return;
  }
  if (!write) return;
  double vv[CPL], xn[CPL];
  if constexpr (HINT)
    ld4<kFirst>(a.v + rowbase, vv);
  else
    ldx<CPL>(a.v + rowbase, vv);
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    // pga.cpp:82-85: v = beta v + g ; next = clamp(x + alpha v)
    vv[c] = ex_add(ex_mul(a.beta, vv[c]), g[c]);
    xn[c] = clamp_box(ex_add(xv[c], ex_mul(a.alpha, vv[c])), a.lo);
    if constexpr (MODE == kTraj && !CHECK) {  // pga.cpp:86, 99-102
      const double d = fabs(ex_sub(xn[c], xv[c]));
      if (d > a.conv_tol && (amask & (1u << c))) acc.viol |= 1u << c;
    }
  }
  if constexpr (HINT) {
    if (amask == 0xF) {
      st4<TU::POLICY>(a.v + rowbase, vv);
      st4<TU::POLICY>(Xo + rowbase, xn);
      return;
    }
  }
  stx<CPL>(a.v + rowbase, vv, amask);
  stx<CPL>(Xo + rowbase, xn, amask);
}

// Walks this thread's (row, quad) units for one pass.  Thread -> quad is
// fixed for the whole launch so per-chain accumulators live in registers.
// CTA roles of a launch.  Fused chain groups: CTAs [g*S, (g+1)*S) sweep
// group g, S = hblocks + lblocks.  The block scheduler dispatches CTAs in
// index order, so the groups still run one after another (one L2-sized X
// slice live at a time, two at the seams) without a launch boundary -- and
// its tail -- between them; within a group the heavy-row CTAs (longest
// work) are dispatched first.
struct Role {
  bool heavy;
  int index, count;  // this CTA's index among the group's heavy / light CTAs, and their count
  int32_t qbase;     // first quad of the group
};
__device__ __forceinline__ Role cta_role(const PassArgs& a) {
  const int S = a.lblocks > 0 ? a.hblocks + a.lblocks : static_cast<int>(gridDim.x);
  const int grp = blockIdx.x / S, local = blockIdx.x % S;
  Role r;
  r.qbase = a.q0 + grp * a.Qg;
  r.heavy = local < a.hblocks;
  r.index = r.heavy ? local : local - a.hblocks;
  r.count = r.heavy ? a.hblocks : S - a.hblocks;
  return r;
}

template <int KIND, int CPL, int MODE, bool CHECK, class TU>
__device__ __forceinline__ void pass_rows(const PassArgs& a, const double* X, double* Xo,
                                          const uint8_t* qmask, bool write, Acc<CPL>& acc,
                                          int32_t& my_q, const Role& role) {
  const int lane = threadIdx.x & 31;
  const int vblock = role.index;
  const int vgrid = role.count;
  const int32_t qbase = role.qbase;
  const int gwarp = (vblock * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (vgrid * blockDim.x) >> 5;
  int32_t q, r0, rstep;
  if (a.Qg >= 32) {
    const int wpr = a.Qg >> 5;
    q = (gwarp % wpr) * 32 + lane;
    r0 = gwarp / wpr;
    rstep = nwarps / wpr;
  } else {
    const int rpw = 32 / a.Qg;
    q = lane & (a.Qg - 1);
    r0 = gwarp * rpw + lane / a.Qg;
    rstep = nwarps * rpw;
  }
  q += qbase;  // global quad
  my_q = q;
  const int32_t col = q * CPL;
  unsigned amask;
  if (qmask) {
    amask = qmask[q];
  } else {  // all real chains of the quad (padding chains skipped)
    const int real = a.B - col;
    amask = real >= CPL ? (1u << CPL) - 1u : (real > 0 ? (1u << real) - 1u : 0u);
  }
  if (!amask) return;
  for (int32_t r = a.heavy + r0; r < a.n; r += rstep)
    row_unit<KIND, CPL, MODE, CHECK, TU>(a, X, Xo, __ldg(a.order + r), col, amask, write, acc);
}

// ---------------------------------------------------------- heavy rows
// A lane-per-(row, quad) gather walks a row as one chain of dependent
// round trips (index load, then U neighbour loads): deg/U of them, ~1 us
// each -- 0.8 ms for the 3350-neighbour hub of BA(1e6,5), a floor under
// every pass however few chains run (measured: 0.82 ms/step at 4 chains,
// profiles/r11_smallb_c4.jsonl).  Rows of degree >= the heavy threshold
// are instead staged by a whole CTA: every thread issues cp.async copies
// of the row's neighbour values (coalesced per neighbour) into one SMEM
// half while one thread per chain sums the other half in CSR order -- the
// same fp64 additions in the same order, so results stay bit-identical --
// and the epilogue is the per-lane path's, one chain per thread.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kHeavyCols = 4;  // chains per thread in a heavy row (ncol <= 4 * kThreads)

// Stage neighbours [e, e + cnt) of the row: cnt x ncol doubles at dst.
__device__ __forceinline__ void heavy_issue(const PassArgs& a, const double* X, int64_t e,
                                            int cnt, int32_t col0, int ncol, bool pairs,
                                            double* dst) {
  if (pairs) {
    const int half = ncol >> 1, total = cnt * half;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int j = t / half, c2 = t - j * half;
      const int32_t u = __ldg(a.nbr + e + j);
      cp_async16(dst + j * ncol + 2 * c2, X + static_cast<int64_t>(u) * a.Bp + col0 + 2 * c2);
    }
  } else {
    const int total = cnt * ncol;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int j = t / ncol, c = t - j * ncol;
      const int32_t u = __ldg(a.nbr + e + j);
      cp_async8(dst + j * ncol + c, X + static_cast<int64_t>(u) * a.Bp + col0 + c);
    }
  }
  cp_async_commit();
}

template <int KIND, int CPL, int MODE, bool CHECK, class TU>
__device__ void heavy_row(const PassArgs& a, const double* X, double* Xo, int32_t v, int32_t col0,
                          int ncol, const uint8_t* qmask, bool write, uint32_t* viol_sink,
                          double* stage) {
  const int64_t e0 = __ldg(a.off + v), e1 = __ldg(a.off + v + 1);
  const int nb = max(1, (a.stage_doubles >> 1) / ncol);  // neighbours per SMEM half
  double* const half1 = stage + nb * ncol;
  const bool pairs = (ncol & 1) == 0 && (a.Bp & 1) == 0;
  const int64_t rowbase = static_cast<int64_t>(v) * a.Bp + col0;
  double s[kHeavyCols], xv[kHeavyCols];
  unsigned nbsel = 0;
#pragma unroll
  for (int k = 0; k < kHeavyCols; ++k) {
    s[k] = 0.0;
    const int c = threadIdx.x + k * blockDim.x;
    xv[k] = c < ncol ? __ldcg(X + rowbase + c) : 0.0;
  }
  if (e1 > e0) heavy_issue(a, X, e0, static_cast<int>(e1 - e0 < nb ? e1 - e0 : nb), col0, ncol, pairs,
                           stage);
  int k = 0;
  for (int64_t e = e0; e < e1; e += nb, ++k) {
    const int cnt = static_cast<int>(e1 - e < nb ? e1 - e : nb);
    if (e + nb < e1) {  // next chunk into the other half while this one is summed
      heavy_issue(a, X, e + nb, static_cast<int>(e1 - e - nb < nb ? e1 - e - nb : nb), col0, ncol, pairs,
                  (k & 1) ? stage : half1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* h = (k & 1) ? half1 : stage;
#pragma unroll
    for (int q = 0; q < kHeavyCols; ++q) {
      const int c = threadIdx.x + q * blockDim.x;
      if (c >= ncol) break;
      double acc = s[q];
      for (int j = 0; j < cnt; ++j) {
        const double val = h[j * ncol + c];
        if constexpr (KIND == MQO_LAPLACIAN)
          acc = ex_add(acc, ex_sub(xv[q], val));  // graph.cpp:85
        else
          acc = ex_add(acc, val);                 // graph.cpp:68
        if constexpr (CHECK) nbsel |= (val > 0.5 ? 1u : 0u) << q;
      }
      s[q] = acc;
    }
    __syncthreads();  // this half may be refilled by the next issue
  }
  const double deg = static_cast<double>(e1 - e0);
#pragma unroll
  for (int q = 0; q < kHeavyCols; ++q) {
    const int c = threadIdx.x + q * blockDim.x;
    if (c >= ncol) break;
    const int32_t b = col0 + c;
    const bool active = qmask ? ((qmask[b / CPL] >> (b % CPL)) & 1u) != 0 : b < a.B;
    if (!active) continue;
    if constexpr (CHECK) {  // pga.cpp:125-133 on binarize(x)
      const bool sel = xv[q] > 0.5;
      const bool any = (nbsel >> q) & 1u;
      if (sel ? any : !any) {
        if constexpr (MODE == kCheck)
          atomicOr(viol_sink + b, 1u);
        else
          viol_sink[b] = 1u;
      }
      if constexpr (MODE == kCheck)
        if (xv[q] != 0.0 && xv[q] != 1.0) atomicOr(reinterpret_cast<unsigned*>(a.flag + 1), 1u);
    }
    if constexpr (MODE == kCheck) continue;
    const double g = grad_epi<KIND>(s[q], xv[q], deg, a.param);
    if constexpr (MODE == kGrad) {
      __stcg(a.gout + rowbase + c, g);
      continue;
    }
    if (!write) continue;
    // pga.cpp:82-85: v = beta v + g ; next = clamp(x + alpha v)
    const double vv = ex_add(ex_mul(a.beta, __ldcg(a.v + rowbase + c)), g);
    const double xn = clamp_box(ex_add(xv[q], ex_mul(a.alpha, vv)), a.lo);
    if constexpr (MODE == kTraj && !CHECK)  // pga.cpp:86, 99-102
      if (fabs(ex_sub(xn, xv[q])) > a.conv_tol) viol_sink[b] = 1u;
    __stcg(a.v + rowbase + c, vv);
    __stcg(Xo + rowbase + c, xn);
  }
}

// The heavy-row CTAs of a group: rows role.index, role.index + count, ...
template <int KIND, int CPL, int MODE, bool CHECK, class TU>
__device__ __forceinline__ void heavy_rows(const PassArgs& a, const double* X, double* Xo,
                                           const uint8_t* qmask, bool write, uint32_t* viol_sink,
                                           const Role& role) {
  extern __shared__ __align__(16) unsigned char heavy_smem[];
  double* stage = reinterpret_cast<double*>(heavy_smem + a.stage_off);
  const int32_t col0 = role.qbase * CPL;
  const int ncol = min(a.Qg * CPL, a.B - col0);
  if (ncol <= 0) return;
  for (int32_t r = role.index; r < a.heavy; r += role.count)
    heavy_row<KIND, CPL, MODE, CHECK, TU>(a, X, Xo, __ldg(a.order + r), col0, ncol, qmask, write,
                                          viol_sink, stage);
}

// Folds thread accumulators into shared per-chain slots.
template <int CPL>
__device__ __forceinline__ void fold_to_smem(const Acc<CPL>& acc, int32_t q, uint32_t* s_viol) {
  if (!acc.viol) return;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (acc.viol & (1u << c)) atomicOr(s_viol + q * CPL + c, 1u);
}

// Single-pass kernels: step / gradient / fixed-point check.
template <int KIND, int CPL, int MODE, class TU>
__global__ void __launch_bounds__(kThreads, TU::MINB) k_pass(PassArgs a) {
  constexpr bool CHECK = MODE == kCheck;
  Acc<CPL> acc;
  int32_t q = 0;
  const double* X = a.x[a.base];
  double* Xo = a.x[a.base];  // kStep updates in place per unit: each unit
                             // reads its own row + neighbours of the input
  // kStep must not read rows another unit already updated, so it writes the
  // other buffer; the host flips `cur` afterwards.
  if constexpr (MODE == kStep) Xo = a.x[a.base ^ 1];
  const Role role = cta_role(a);
  if (role.heavy) {
    heavy_rows<KIND, CPL, MODE, CHECK, TU>(a, X, Xo, nullptr, true, a.viol, role);
    return;
  }
  pass_rows<KIND, CPL, MODE, CHECK, TU>(a, X, Xo, nullptr, true, acc, q, role);
  if constexpr (CHECK) {
    if (acc.viol) {
#pragma unroll
      for (int c = 0; c < CPL; ++c)
        if (acc.viol & (1u << c)) atomicOr(a.viol + q * CPL + c, 1u);
    }
    if (acc.nonbin) atomicOr(reinterpret_cast<unsigned*>(a.flag + 1), 1u);
  }
}

// Cooperative persistent trajectory kernel (K1 + K2).
template <int KIND, int CPL, class TU>
__global__ void __launch_bounds__(kThreads, TU::MINB) k_traj(PassArgs a) {
  constexpr bool MIS = KIND == MQO_MIS_QUBO;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned long long smem_u64[];
  unsigned long long* s_chg = smem_u64;                              // [Bp]
  uint32_t* s_viol = reinterpret_cast<uint32_t*>(s_chg + a.Bp);       // [Bp]
  uint8_t* s_active = reinterpret_cast<uint8_t*>(s_viol + a.Bp);      // [Bp]
  uint8_t* s_qmask = s_active + a.Bp;                                 // [Q]
  __shared__ int s_count;

  for (int b = threadIdx.x; b < a.Bp; b += blockDim.x)
    s_active[b] = (b < a.B && a.ctl[b].active) ? 1 : 0;
  __syncthreads();
  for (int q = threadIdx.x; q < a.Q; q += blockDim.x) {
    unsigned m = 0;
    for (int c = 0; c < CPL; ++c) m |= s_active[q * CPL + c] ? (1u << c) : 0u;
    s_qmask[q] = static_cast<uint8_t>(m);
  }

  for (int32_t p = a.p_begin; p < a.p_end; ++p) {
    const int slot = p % 3, next = (p + 1) % 3;
    if (blockIdx.x == 0)
      for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) {
        a.viol[next * a.Bp + b] = 0u;
        a.chg[next * a.Bp + b] = 0ull;
      }
    for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) {
      s_viol[b] = 0u;
      s_chg[b] = 0ull;
    }
    __syncthreads();

    const double* X = a.x[(a.base + p - 1) & 1];
    double* Xo = a.x[(a.base + p) & 1];
    const bool write = !MIS || p <= a.T;  // pass T+1 is check-only (MIS)
    Acc<CPL> acc;
    int32_t q = 0;
    pass_rows<KIND, CPL, kTraj, MIS, TU>(a, X, Xo, s_qmask, write, acc, q, cta_role(a));
    fold_to_smem<CPL>(acc, q, s_viol);
    __syncthreads();
    for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) {
      if (!s_active[b] || !s_viol[b]) continue;
      uint32_t* gv = a.viol + slot * a.Bp + b;
      if (*reinterpret_cast<volatile uint32_t*>(gv) == 0u) atomicOr(gv, 1u);
    }
    grid.sync();

    // K2: identical stop decisions in every CTA (pga.cpp:89-102).
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    int local = 0;
    for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) {
      if (!s_active[b]) continue;
      bool stop = false;
      ChainCtl c;
      if (MIS) {
        const int32_t t = p - 1;  // the iterate this pass checked
        if (t >= 1 && t % a.check_every == 0 && __ldcg(a.viol + slot * a.Bp + b) == 0u) {
          stop = true;
          c = ChainCtl{0, t, MQO_CHECKER_ACCEPTED, (a.base + t) & 1};
        }
      } else if (__ldcg(a.viol + slot * a.Bp + b) == 0u) {  // max|dx| <= conv_tol
        stop = true;
        c = ChainCtl{0, p, MQO_CONVERGED, (a.base + p) & 1};
      }
      if (stop) {
        s_active[b] = 0;
        if (blockIdx.x == 0) a.ctl[b] = c;
      } else {
        ++local;
      }
    }
    if (local) atomicAdd(&s_count, local);
    __syncthreads();
    for (int q2 = threadIdx.x; q2 < a.Q; q2 += blockDim.x) {
      unsigned m = 0;
      for (int c = 0; c < CPL; ++c) m |= s_active[q2 * CPL + c] ? (1u << c) : 0u;
      s_qmask[q2] = static_cast<uint8_t>(m);
    }
    const int count = s_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.flag[0] = count;
    __syncthreads();
    if (count == 0) break;
  }
}

// One trajectory pass as a plain launch, for large graphs where a pass is
// long enough that launch latency is irrelevant and the hardware block
// scheduler balances rows better than a static persistent split.  The stop
// decisions of pass p run in k_traj_ctl right after it (same stream).
__device__ void traj_ctl_cta(const PassArgs& a);

template <int KIND, int CPL, class TU>
__global__ void __launch_bounds__(kThreads, TU::MINB) k_traj_pass(PassArgs a) {
  constexpr bool MIS = KIND == MQO_MIS_QUBO;
  if (*reinterpret_cast<volatile int32_t*>(a.flag) == 0) return;  // every chain stopped
  extern __shared__ unsigned long long smem_u64[];
  unsigned long long* s_chg = smem_u64;
  uint32_t* s_viol = reinterpret_cast<uint32_t*>(s_chg + a.Bp);
  uint8_t* s_qmask = reinterpret_cast<uint8_t*>(s_viol + a.Bp);
  const int32_t p = a.p_begin;
  const int slot = p % 3;
  // the active-quad masks come from k_traj_ctl / k_qmask (one global read
  // per thread instead of a per-CTA rebuild from ChainCtl)
  (void)s_qmask;
  for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) s_viol[b] = 0u;
  (void)s_chg;
  __syncthreads();
  const double* X = a.x[(a.base + p - 1) & 1];
  double* Xo = a.x[(a.base + p) & 1];
  const bool write = !MIS || p <= a.T;
  Acc<CPL> acc;
  int32_t q = 0;
  const Role role = cta_role(a);
  if (role.heavy) {
    heavy_rows<KIND, CPL, kTraj, MIS, TU>(a, X, Xo, a.qmask, write, s_viol, role);
  } else {
    pass_rows<KIND, CPL, kTraj, MIS, TU>(a, X, Xo, a.qmask, write, acc, q, role);
    fold_to_smem<CPL>(acc, q, s_viol);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) {
    if (!s_viol[b]) continue;
    uint32_t* gv = a.viol + slot * a.Bp + b;
    if (*reinterpret_cast<volatile uint32_t*>(gv) == 0u) atomicOr(gv, 1u);
  }
  if (a.fuse_ctl) {
    // the pass's stop decisions by its last CTA (threadfence reduction):
    // one launch per pass instead of the pass + k_traj_ctl
    __shared__ unsigned s_ticket;
    __threadfence();  // every thread's accumulator atomics before the ticket
    __syncthreads();
    if (threadIdx.x == 0) {
      s_ticket = atomicAdd(reinterpret_cast<unsigned*>(a.flag + 3), 1u);
    }
    __syncthreads();
    if (s_ticket == gridDim.x - 1) {
      __threadfence();
      traj_ctl_cta(a);
      if (threadIdx.x == 0) a.flag[3] = 0;
    }
  }
}

// Active-chain mask per quad from ChainCtl (one CTA; after a __syncthreads
// that orders the ctl writes of the same CTA).
__device__ __forceinline__ void qmask_from_ctl(const ChainCtl* ctl, int32_t B, int32_t Q,
                                               int32_t cpl, uint8_t* qmask) {
  for (int q = threadIdx.x; q < Q; q += blockDim.x) {
    unsigned m = 0;
    for (int c = 0; c < cpl; ++c) {
      const int b = q * cpl + c;
      m |= (b < B && ctl[b].active) ? (1u << c) : 0u;
    }
    qmask[q] = static_cast<uint8_t>(m);
  }
}

__global__ void k_qmask(const ChainCtl* ctl, int32_t B, int32_t Q, int32_t cpl, uint8_t* qmask) {
  qmask_from_ctl(ctl, B, Q, cpl, qmask);
}

// K2 for the per-launch path: one CTA takes pass p's stop decisions
// (pga.cpp:89-102), clears the next accumulator slot, publishes the count.
__device__ void traj_ctl_cta(const PassArgs& a);
__global__ void k_traj_ctl(PassArgs a) {
  if (*reinterpret_cast<volatile int32_t*>(a.flag) == 0) return;
  traj_ctl_cta(a);
}
__device__ void traj_ctl_cta(const PassArgs& a) {
  __shared__ int s_count;
  const int32_t p = a.p_begin;
  const int slot = p % 3, next = (p + 1) % 3;
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  int local = 0;
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
    ChainCtl c = a.ctl[b];
    if (!c.active) continue;
    bool stop = false;
    if (a.is_mis) {
      const int32_t t = p - 1;
      if (t >= 1 && t % a.check_every == 0 &&
          *reinterpret_cast<const volatile uint32_t*>(a.viol + slot * a.Bp + b) == 0u) {
        stop = true;
        c = ChainCtl{0, t, MQO_CHECKER_ACCEPTED, (a.base + t) & 1};
      }
    } else if (*reinterpret_cast<const volatile uint32_t*>(a.viol + slot * a.Bp + b) == 0u) {  // max|dx| <= conv_tol
      stop = true;
      c = ChainCtl{0, p, MQO_CONVERGED, (a.base + p) & 1};
    }
    if (stop)
      a.ctl[b] = c;
    else
      ++local;
  }
  for (int b = threadIdx.x; b < a.Bp; b += blockDim.x) {
    a.viol[next * a.Bp + b] = 0u;
    a.chg[next * a.Bp + b] = 0ull;
  }
  if (local) atomicAdd(&s_count, local);
  __syncthreads();
  if (threadIdx.x == 0) a.flag[0] = s_count;
  qmask_from_ctl(a.ctl, a.B, a.Q, a.cpl, a.qmask);
}

// Chains still running at the end: IterCap at iterate T (pga.cpp:109-110).
__global__ void k_finalize(ChainCtl* ctl, int32_t B, int32_t T, int32_t base) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (ctl[b].active) ctl[b] = ChainCtl{0, T, MQO_ITER_CAP, (base + T) & 1};
}

__global__ void k_ctl_init(ChainCtl* ctl, int32_t B, int32_t Bp) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < Bp) ctl[b] = ChainCtl{b < B ? 1 : 0, 0, MQO_ITER_CAP, 0};
}

// Copies each chain's final iterate into buffer `dst` when it ended in the
// other one.
__global__ void k_gather_final(double* __restrict__ dst, const double* __restrict__ src,
                               const ChainCtl* __restrict__ ctl, int32_t dst_index,
                               int64_t count, int32_t Bp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(i % Bp);
    if (ctl[b].final_buf != dst_index) dst[i] = src[i];
  }
}

// ----------------------------------------------------------- dispatch

using PassFn = void (*)(PassArgs);

// K1 tuning variants (MQO_K1_VARIANT, default 0) -- kept selectable so the
// choice can be re-measured on new parts; 0 is the measured best.
int g_k1_variant = [] {
  const char* e = std::getenv("MQO_K1_VARIANT");
  return e ? std::atoi(e) : 0;
}();
// Fraction of the L2 given to evict_last gathers (hot_rows).  C4 (BA(1e6,5))
// per step / trajectory pass at 16 | 64 | 128 chains, MQO_HOT_FRAC sweep r32:
// 0.5 (round 1): 0.244 / 0.259 | 0.957 / 0.99 | 1.921 / 1.966 ms;
// 0.2: 0.239 / 0.253 | 0.938 / 0.966 | 1.893 / 1.939 ms (0.05 .. 0.9 measured;
// ER configs C3 / C5 flat).
double g_hot_frac = [] {
  const char* e = std::getenv("MQO_HOT_FRAC");
  return e ? std::atof(e) : 0.2;
}();
// CTAs per SM of the per-pass grids; 0 = automatic: 8 for a sweep over all
// chains, 4 per group for chain-tiled sweeps (profiles/r08_tune_grid.txt:
// ER(1e5) MIS x256 tiled: 0.2673 -> 0.2568 ms per trajectory pass; BA(1e6)
// x128 untiled: 8 is best).
int g_grid_per_sm = [] {
  const char* e = std::getenv("MQO_GRID_PER_SM");
  return e ? std::atoi(e) : 0;
}();
int k1_variant() { return g_k1_variant; }

template <int MODE, class TU>
PassFn pass_fn_tu(int kind, int cpl) {
#define MQO_K(K)                                                        \
  case K:                                                               \
    return cpl == 4 ? k_pass<K, 4, MODE, TU> : k_pass<K, 1, MODE, TU>;
  switch (kind) {
    MQO_K(MQO_MIS_QUBO)
    MQO_K(MQO_LAPLACIAN)
    MQO_K(MQO_PERTURBED_LAPLACIAN)
    MQO_K(MQO_ADJACENCY)
    MQO_K(MQO_PERTURBED_BIAS)
  }
#undef MQO_K
  throw std::invalid_argument("objective: unknown kind");
}

// A degree distribution with hubs: the maximum far above the mean (the
// same test as the persistent-trajectory split).
// (MQO_HUB_TUNE=0: TuneDefault everywhere, for A/B runs)
const bool g_hub_tune = [] {
  const char* e = std::getenv("MQO_HUB_TUNE");
  return !(e && *e == '0');
}();
bool hub_graph(const mqo_graph* g) {
  if (!g_hub_tune) return false;
  const double avg_deg = g->n ? 2.0 * static_cast<double>(g->m) / g->n : 0.0;
  return g->max_degree > 32.0 * avg_deg + 32.0;
}

template <int MODE>
PassFn pass_fn(int kind, int cpl, bool hubs = false, bool tiled = false) {
  if constexpr (MODE == kStep) {
    switch (k1_variant()) {
      case 1: return pass_fn_tu<MODE, Tune<8, 2, 0>>(kind, cpl);  // round-1 kernel
      case 2: return pass_fn_tu<MODE, Tune<6, 3, 2>>(kind, cpl);
      case 3: return pass_fn_tu<MODE, Tune<4, 4, 1>>(kind, cpl);
      case 4: return pass_fn_tu<MODE, Tune<4, 4, 2>>(kind, cpl);
      case 5: return pass_fn_tu<MODE, Tune<5, 3, 1>>(kind, cpl);
      case 6: return pass_fn_tu<MODE, Tune<4, 3, 1>>(kind, cpl);
      case 7: return pass_fn_tu<MODE, Tune<7, 3, 1>>(kind, cpl);
      case 8: return pass_fn_tu<MODE, Tune<3, 4, 1>>(kind, cpl);
      case 9: return pass_fn_tu<MODE, Tune<4, 3, 3>>(kind, cpl);   // L2::64B gathers
      case 10: return pass_fn_tu<MODE, Tune<3, 4, 3>>(kind, cpl);
      case 11: return pass_fn_tu<MODE, Tune<4, 3, 1, true>>(kind, cpl);  // index prefetch
      case 12: return pass_fn_tu<MODE, Tune<3, 4, 1, true>>(kind, cpl);
      case 13: return pass_fn_tu<MODE, Tune<5, 3, 1, true>>(kind, cpl);  // TuneHub
      case 14: return pass_fn_tu<MODE, Tune<6, 3, 1, true>>(kind, cpl);
      default: break;
    }
  }
  if constexpr (MODE == kStep)
    if (kind == MQO_MIS_QUBO && tiled) return pass_fn_tu<MODE, TuneMisTiled>(kind, cpl);
  if (kind == MQO_MIS_QUBO) return pass_fn_tu<MODE, TuneMis>(kind, cpl);
  if constexpr (MODE == kStep)
    if (hubs) return pass_fn_tu<MODE, TuneHub>(kind, cpl);
  return pass_fn_tu<MODE, TuneDefault>(kind, cpl);
}

PassFn traj_pass_fn(int kind, int cpl, bool hubs, bool tiled) {
#define MQO_K(K)                                                                             \
  case K:                                                                                    \
    if constexpr (K != MQO_MIS_QUBO)                                                         \
      if (hubs) return cpl == 4 ? k_traj_pass<K, 4, TuneHubTraj> : k_traj_pass<K, 1, TuneHubTraj>; \
    if constexpr (K == MQO_MIS_QUBO)                                                         \
      if (tiled) return cpl == 4 ? k_traj_pass<K, 4, TuneMisTiled> : k_traj_pass<K, 1, TuneMisTiled>; \
    return cpl == 4 ? k_traj_pass<K, 4, TuneFor<K>> : k_traj_pass<K, 1, TuneFor<K>>;
  switch (kind) {
    MQO_K(MQO_MIS_QUBO)
    MQO_K(MQO_LAPLACIAN)
    MQO_K(MQO_PERTURBED_LAPLACIAN)
    MQO_K(MQO_ADJACENCY)
    MQO_K(MQO_PERTURBED_BIAS)
  }
#undef MQO_K
  throw std::invalid_argument("objective: unknown kind");
}

PassFn traj_fn(int kind, int cpl) {
#define MQO_K(K) \
  case K:        \
    return cpl == 4 ? k_traj<K, 4, TuneFor<K>> : k_traj<K, 1, TuneFor<K>>;
  switch (kind) {
    MQO_K(MQO_MIS_QUBO)
    MQO_K(MQO_LAPLACIAN)
    MQO_K(MQO_PERTURBED_LAPLACIAN)
    MQO_K(MQO_ADJACENCY)
    MQO_K(MQO_PERTURBED_BIAS)
  }
#undef MQO_K
  throw std::invalid_argument("objective: unknown kind");
}

int sm_count(int device) {
  static int cached[64] = {0};
  if (!cached[device]) MQO_CUDA(cudaDeviceGetAttribute(&cached[device], cudaDevAttrMultiProcessorCount, device));
  return cached[device];
}

// Warps needed so every (row, quad) unit of a Qg-quad chain group has a thread.
int64_t warp_tasks(const mqo_batch* b, int Qg) {
  const int64_t n = b->g->n;
  if (Qg >= 32) return n * (Qg / 32);
  const int rpw = 32 / Qg;
  return (n + rpw - 1) / rpw;
}
int64_t warp_tasks(const mqo_batch* b) { return warp_tasks(b, b->Q); }

// A row spans wpr = Qg/32 warps; the thread -> quad map stays fixed only if
// the total warp count is a multiple of wpr.
int align_blocks(const mqo_batch* b, int64_t blocks, int Qg) {
  const int wpr = Qg >= 32 ? Qg / 32 : 1;
  if (wpr > kWarps) {
    const int per = wpr / kWarps;
    blocks = std::max<int64_t>(per, blocks / per * per);
  }
  return static_cast<int>(blocks);
}

int align_blocks(const mqo_batch* b, int64_t blocks) { return align_blocks(b, blocks, b->Q); }

// Grid of the per-pass kernels: g_grid_per_sm CTAs per SM (grid-stride
// over rows), never more than the work needs.
int pass_blocks(const mqo_batch* b, int Qg) {
  const int64_t need = (warp_tasks(b, Qg) + kWarps - 1) / kWarps;
  const int per_sm = g_grid_per_sm > 0 ? g_grid_per_sm : (Qg < b->Q ? 4 : 8);
  const int64_t cap = static_cast<int64_t>(sm_count(b->g->device)) * per_sm;
  return align_blocks(b, std::max<int64_t>(1, std::min(need, cap)), Qg);
}
int pass_blocks(const mqo_batch* b) { return pass_blocks(b, b->Q); }

// Chain tiling of the per-pass kernels.  A pass over all B chains gathers
// neighbour rows of n·8·B bytes at random; when that working set exceeds
// L2, almost every gather misses.  Sweeping the graph once per chain group
// shrinks the working set to n·8·Bg, so gathered row segments stay in L2
// between neighbours -- at the price of re-reading the CSR per group and of
// shorter row segments.  Measured (scripts/tune_k1.py --groups): ER(1e5,
// d=10) MIS, 256 chains: 0.324 -> 0.252 ms/step with 64-chain groups (51 MB
// slices); BA(1e6,5), 128 chains: no group size helps (a slice that fits L2
// leaves 8-16 chains per row, whose scattered 32-byte sectors run DRAM far
// below its streaming rate), so tiling applies only when a slice of >= 32
// chains fits in half the L2.
// g_group_quads: quads (4 chains) per group; 0 = automatic, -1 = off.
int g_group_quads = [] {
  const char* e = std::getenv("MQO_GROUP_QUADS");
  return e ? std::atoi(e) : 0;
}();
int group_quads(const mqo_batch* b) {
  const int Q = b->Q;
  if (g_group_quads < 0 || b->cpl != 4) return Q;
  int Qg = g_group_quads;
  if (Qg == 0) {
    static int l2[64] = {0};
    const int dev = b->g->device;
    if (!l2[dev]) MQO_CUDA(cudaDeviceGetAttribute(&l2[dev], cudaDevAttrL2CacheSize, dev));
    Qg = Q;
    while (Qg > 8 && static_cast<double>(b->g->n) * 32.0 * Qg > 0.5 * l2[dev]) Qg /= 2;
    if (static_cast<double>(b->g->n) * 32.0 * Qg > 0.5 * l2[dev]) return Q;  // no slice fits
  }
  // a group must tile Q: a power of two <= 32 dividing Q, or a multiple of 32 dividing Q
  Qg = std::max(1, std::min(Qg, Q));
  while (Q % Qg != 0 || (Qg < 32 && (Qg & (Qg - 1)) != 0) || (Qg > 32 && Qg % 32 != 0)) --Qg;
  return Qg;
}

void validate_objective(const mqo_objective& o) {  // objectives.cpp:27-38
  if (o.kind < 0 || o.kind > 4) throw std::invalid_argument("objective: unknown kind");
  if (o.kind == MQO_MIS_QUBO && !(o.param > 1.0))
    throw std::invalid_argument("mis-qubo: gamma must be > 1");
  if (o.kind == MQO_PERTURBED_LAPLACIAN && !(o.param > 0.0))
    throw std::invalid_argument("perturbed-laplacian: lambda must be > 0");
  if (o.kind == MQO_PERTURBED_BIAS && !(o.param > 0.0 && o.param < 2.0))
    throw std::invalid_argument("perturbed-bias: lambda must be in (0, 2)");
}

void validate_optimizer(const mqo_optimizer& c) {  // pga.cpp:9-18
  if (!(c.alpha > 0.0)) throw std::invalid_argument("optimizer: alpha must be > 0");
  if (c.beta < 0.0 || c.beta >= 1.0) throw std::invalid_argument("optimizer: beta must be in [0, 1)");
  if (c.max_iters < 1) throw std::invalid_argument("optimizer: max_iters must be >= 1");
  if (c.conv_tol < 0.0) throw std::invalid_argument("optimizer: conv_tol must be >= 0");
  if (c.check_every < 1) throw std::invalid_argument("optimizer: check_every must be >= 1");
}

// Rows whose gathers are marked L2::evict_last: a prefix of the vertex
// order (hubs come first in preferential-attachment labelings) sized to
// MQO_HOT_FRAC (default 0.2) of the L2.
int32_t hot_rows(const mqo_batch* b, int Qg) {
  const double frac = g_hot_frac;
  static int l2[64] = {0};
  const int dev = b->g->device;
  if (!l2[dev]) MQO_CUDA(cudaDeviceGetAttribute(&l2[dev], cudaDevAttrL2CacheSize, dev));
  const double rows = frac * l2[dev] / (8.0 * b->cpl * Qg);
  return static_cast<int32_t>(std::min<double>(b->g->n, std::max(0.0, rows)));
}
int32_t hot_rows(const mqo_batch* b) { return hot_rows(b, b->Q); }

PassArgs make_args(mqo_batch* b, const mqo_objective& obj) {
  PassArgs a{};
  const mqo_graph* g = b->g;
  a.off = g->d_off;
  a.nbr = g->d_nbr;
  a.order = g->d_order;
  a.n = g->n;
  a.B = b->B;
  a.Bp = b->Bp;
  a.Q = b->Q;
  a.q0 = 0;
  a.Qg = b->Q;
  a.x[0] = b->d_x[0];
  a.x[1] = b->d_x[1];
  a.v = b->d_v;
  a.param = obj.param;
  a.lo = obj.kind == MQO_MIS_QUBO ? 0.0 : -1.0;
  a.ctl = b->d_ctl;
  a.viol = b->d_viol;
  a.chg = b->d_chg;
  a.flag = b->d_flag;
  a.base = b->cur;
  a.is_mis = obj.kind == MQO_MIS_QUBO;
  a.hot_rows = hot_rows(b);
  a.cpl = b->cpl;
  a.qmask = b->d_qmask;
  return a;
}

// Heavy rows (heavy_row): the degree threshold of the SMEM-staged path.
// 0 = automatic: rows whose per-lane critical path -- deg/U dependent
// round trips of ~1 us -- would exceed half the pass's bandwidth time at
// the measured HBM rate, and at least 64; < 0 = off.  At 128 chains on
// BA(1e6,5) the threshold exceeds every degree (the bench kernel is
// unchanged); at 16 chains rows of degree >= ~570 are staged.
int g_heavy_deg = [] {
  const char* e = std::getenv("MQO_HEAVY_DEG");
  return e ? std::atoi(e) : 0;
}();
constexpr int kStageDoubles = 4096;  // 32 KB of SMEM staging per heavy CTA

struct HeavyPlan {
  int32_t heavy = 0, hblocks = 0;
  size_t smem = 0;  // dynamic SMEM bytes to add
};
HeavyPlan heavy_plan(const mqo_batch* b, int Qg, size_t base_smem) {
  HeavyPlan h;
  const mqo_graph* g = b->g;
  const int64_t ncol = std::min<int64_t>(int64_t(Qg) * b->cpl, b->B);
  if (g_heavy_deg < 0 || ncol > int64_t(kHeavyCols) * kThreads || g->h_deg_ge.empty()) return h;
  int64_t thr = g_heavy_deg;
  if (thr == 0) {
    const double nnz = 2.0 * static_cast<double>(g->m);
    const double bytes = 8.0 * (g->n + 1) + 4.0 * nnz + ncol * (8.0 * nnz + 32.0 * g->n);
    const double pass_us = bytes / 6.5e6;  // ~6.5 TB/s
    const int U = b->cpl == 4 ? 4 : 16;
    thr = std::max<int64_t>(64, static_cast<int64_t>(U * pass_us / 2.0));
  }
  if (thr > g->max_degree) return h;
  h.heavy = g->h_deg_ge[static_cast<size_t>(thr)];
  if (h.heavy <= 0) return h;
  h.hblocks = std::min<int32_t>(h.heavy, 2 * sm_count(g->device));
  h.smem = ((base_smem + 15) / 16) * 16 - base_smem + sizeof(double) * kStageDoubles;
  return h;
}

// One pass over every chain group: a single launch of Q/Qg groups x
// (hblocks heavy-row + `blocks` light-row) CTAs (MQO_FUSE_GROUPS=0: one
// launch per group, the earlier form).
bool g_fuse_groups = [] {
  const char* e = std::getenv("MQO_FUSE_GROUPS");
  return !(e && *e == '0');
}();
template <class F>
void launch_groups(const mqo_batch* b, PassArgs& a, int blocks, size_t smem, F fn) {
  const HeavyPlan hp = heavy_plan(b, a.Qg, smem);
  a.heavy = hp.heavy;
  a.hblocks = hp.hblocks;
  a.lblocks = blocks;
  a.stage_doubles = kStageDoubles;
  a.stage_off = static_cast<int32_t>((smem + 15) / 16 * 16);
  const size_t total_smem = smem + hp.smem;
  const int per_group = hp.hblocks + blocks;
  if (g_fuse_groups && a.Qg < b->Q) {
    a.q0 = 0;
    fn<<<per_group * (b->Q / a.Qg), kThreads, total_smem, b->stream>>>(a);
  } else {
    for (a.q0 = 0; a.q0 < b->Q; a.q0 += a.Qg) fn<<<per_group, kThreads, total_smem, b->stream>>>(a);
    a.q0 = 0;
  }
  a.heavy = a.hblocks = a.lblocks = 0;
}

// MQO_FUSE_CTL=0: k_traj_ctl as its own launch after every pass (A/B runs)
const bool g_fuse_ctl = [] {
  const char* e = std::getenv("MQO_FUSE_CTL");
  return !(e && *e == '0');
}();

// Problems up to this many (vertex, chain) cells run the persistent kernel.
int64_t g_persistent_cells = [] {
  const char* e = std::getenv("MQO_PERSISTENT_CELLS");
  return e ? std::atoll(e) : int64_t(1) << 22;
}();
int64_t persistent_cells() { return g_persistent_cells; }

double now_monotonic() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<double>(ts.tv_sec) + 1e-9 * static_cast<double>(ts.tv_nsec);
}

}  // namespace

namespace mqo_b200 {

// Enqueues one fused step on the batch stream (used by mqo_step and the
// engine); flips the current buffer.
void launch_step(mqo_batch* b, const mqo_objective& obj, const mqo_optimizer& opt) {
  PassArgs a = make_args(b, obj);
  a.alpha = opt.alpha;
  a.beta = opt.beta;
  if (b->g->n == 0) return;
  a.Qg = group_quads(b);
  PassFn fn = pass_fn<kStep>(obj.kind, b->cpl, hub_graph(b->g), g_hub_tune && a.Qg < b->Q);
  a.hot_rows = hot_rows(b, a.Qg);
  const int blocks = pass_blocks(b, a.Qg);
  launch_groups(b, a, blocks, 0, fn);
  MQO_CUDA(cudaGetLastError());
  b->cur ^= 1;
}

// Runs trajectories of every chain from the current x (already projected
// by the caller when required).  Returns with ctl[] filled and the final
// states gathered into buffer b->cur.
void run_trajectories(mqo_batch* b, const mqo_objective& obj, const mqo_optimizer& opt,
                      double deadline) {
  mqo_graph* g = b->g;
  const bool mis = obj.kind == MQO_MIS_QUBO;
  k_ctl_init<<<(b->Bp + 255) / 256, 256, 0, b->stream>>>(b->d_ctl, b->B, b->Bp);
  MQO_CUDA(cudaMemsetAsync(b->d_v, 0, sizeof(double) * int64_t(g->n) * b->Bp, b->stream));
  int32_t T = opt.max_iters;
  if (g->n == 0) {
    k_finalize<<<(b->B + 255) / 256, 256, 0, b->stream>>>(b->d_ctl, b->B, T, b->cur);
    return;
  }
  // Graphs whose per-chain state fits in SMEM: one CTA per chain, whole
  // trajectories without grid barriers (traj_cta.cu).
  if (const int G = cta_group(b)) {
    run_trajectories_cta(b, obj, opt, deadline, G, now_monotonic);
    return;
  }
  PassArgs a = make_args(b, obj);
  a.alpha = opt.alpha;
  a.beta = opt.beta;
  a.check_every = opt.check_every;
  a.conv_tol = opt.conv_tol;
  a.T = T;

  // Small problems: one cooperative persistent kernel per 256-pass chunk
  // (passes separated by grid.sync, launch-free).  Large problems: one
  // launch per pass + a one-CTA control kernel.
  // Persistent kernel: small problems always; up to 32M cells when the graph
  // is hub-light (its static row split stays balanced) and no chain tiling
  // applies (scripts/traj_paths.py: 5-15% fewer us per pass on ER(2e4..1e6)
  // for 4M-32M cells; BA(1e6) x 128 -- 128M cells, hubs -- is 25% slower
  // persistent).
  const int64_t cells = int64_t(g->n) * b->Bp;
  const double avg_deg = g->n ? 2.0 * static_cast<double>(g->m) / g->n : 0.0;
  // (the persistent kernel's static row split has no heavy-row CTAs: graphs
  // with rows the per-pass launches would stage take the per-pass path)
  const size_t base_smem = sizeof(unsigned long long) * b->Bp + sizeof(uint32_t) * b->Bp + b->Bp + b->Q;
  const bool persistent =
      heavy_plan(b, group_quads(b), base_smem).heavy == 0 &&
      (cells <= persistent_cells() ||
       (g_persistent_cells == (int64_t(1) << 22) && cells <= (int64_t(1) << 25) &&
        group_quads(b) == b->Q && g->max_degree <= 32.0 * avg_deg + 32.0));
  PassFn fn = persistent ? traj_fn(obj.kind, b->cpl)
                         : traj_pass_fn(obj.kind, b->cpl, hub_graph(g), g_hub_tune && group_quads(b) < b->Q);
  const size_t smem = base_smem;
  if (!persistent) {  // chain tiling (see group_quads)
    a.Qg = group_quads(b);
    a.hot_rows = hot_rows(b, a.Qg);
  }
  int blocks = pass_blocks(b, a.Qg);
  if (!persistent)
    k_qmask<<<1, 256, 0, b->stream>>>(b->d_ctl, b->B, b->Q, b->cpl, b->d_qmask);
  if (persistent) {
    int per_sm = 0;
    MQO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, reinterpret_cast<const void*>(fn), kThreads, smem));
    if (per_sm < 1) throw std::logic_error("trajectory kernel cannot be resident");
    const int64_t need = (warp_tasks(b) + kWarps - 1) / kWarps;
    blocks = align_blocks(
        b, std::max<int64_t>(1, std::min<int64_t>(need, int64_t(per_sm) * sm_count(g->device))));
  }
  b->h_flag[0] = b->B;
  MQO_CUDA(cudaMemcpyAsync(b->d_flag, b->h_flag, sizeof(int32_t), cudaMemcpyHostToDevice,
                           b->stream));

  int32_t last = mis ? T + 1 : T;  // MIS needs one check-only pass for x_T
  int32_t p = 1;
  while (p <= last) {
    // Chunks end on multiples of 256 so the deadline is polled where the
    // reference polls it ((iter & 255) == 0, pga.cpp:104-107).
    const int32_t chunk_end = std::min<int32_t>(last + 1, (p / 256 + 1) * 256 + 1);
    a.T = T;
    if (persistent) {
      MQO_CUDA(cudaMemsetAsync(b->d_viol, 0, sizeof(uint32_t) * 3 * b->Bp, b->stream));
      MQO_CUDA(cudaMemsetAsync(b->d_chg, 0, sizeof(unsigned long long) * 3 * b->Bp, b->stream));
      a.p_begin = p;
      a.p_end = chunk_end;
      void* args[] = {&a};
      MQO_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), blocks, kThreads,
                                           args, smem, b->stream));
    } else {
      if (p == 1) {
        MQO_CUDA(cudaMemsetAsync(b->d_flag + 3, 0, sizeof(int32_t), b->stream));  // fused-ctl tickets
        MQO_CUDA(cudaMemsetAsync(b->d_viol, 0, sizeof(uint32_t) * 3 * b->Bp, b->stream));
        MQO_CUDA(cudaMemsetAsync(b->d_chg, 0, sizeof(unsigned long long) * 3 * b->Bp, b->stream));
      }
      // one launch per pass (untiled, or the chain groups fused into one
      // grid): its last CTA takes the stop decisions
      a.fuse_ctl = g_fuse_ctl && (a.Qg == b->Q || g_fuse_groups) ? 1 : 0;
      for (int32_t q = p; q < chunk_end; ++q) {
        a.p_begin = q;
        a.p_end = q + 1;
        launch_groups(b, a, blocks, smem, fn);
        if (!a.fuse_ctl) k_traj_ctl<<<1, 256, 0, b->stream>>>(a);
      }
      a.fuse_ctl = 0;
      MQO_CUDA(cudaGetLastError());
    }
    MQO_CUDA(cudaMemcpyAsync(b->h_flag, b->d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost,
                             b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
    if (b->h_flag[0] == 0) break;
    const int32_t done = chunk_end - 1;  // passes completed
    if (deadline >= 0.0 && (done & 255) == 0 && done < T && now_monotonic() >= deadline) {
      T = done;  // IterCap at this iterate after (MIS) checking it
      last = mis ? T + 1 : T;
    }
    p = chunk_end;
  }
  k_finalize<<<(b->B + 255) / 256, 256, 0, b->stream>>>(b->d_ctl, b->B, T, b->cur);
  MQO_CUDA(cudaGetLastError());
  // Gather every chain's final iterate into one buffer.
  const int dst = (b->cur + T) & 1;
  const int64_t count = int64_t(g->n) * b->Bp;
  k_gather_final<<<std::min<int64_t>((count + 255) / 256, 148 * 32), 256, 0, b->stream>>>(
      b->d_x[dst], b->d_x[dst ^ 1], b->d_ctl, dst, count, b->Bp);
  MQO_CUDA(cudaGetLastError());
  b->cur = dst;
}

void read_outcomes(mqo_batch* b, int32_t* iterations, int32_t* reasons) {
  std::vector<ChainCtl> ctl(b->B);
  MQO_CUDA(cudaMemcpyAsync(ctl.data(), b->d_ctl, sizeof(ChainCtl) * b->B, cudaMemcpyDeviceToHost,
                           b->stream));
  MQO_CUDA(cudaStreamSynchronize(b->stream));
  for (int i = 0; i < b->B; ++i) {
    if (iterations) iterations[i] = ctl[i].iterations;
    if (reasons) reasons[i] = ctl[i].reason;
  }
}

}  // namespace mqo_b200

// Tuning knobs of the fused kernels (measurement scripts only):
//   "k1_variant"  K1 Tune<> instantiation (0 = default), "hot_frac"
//   fraction of L2 reserved (evict_last) for hot-row gathers, "heavy_deg"
//   degree threshold of the SMEM-staged heavy rows (0 auto, < 0 off).
extern "C" int mqo_tune(const char* key, double value) {
  return guard([&] {
    const std::string k = key ? key : "";
    if (k == "k1_variant")
      g_k1_variant = static_cast<int>(value);
    else if (k == "hot_frac")
      g_hot_frac = value;
    else if (k == "persistent_cells")
      g_persistent_cells = static_cast<int64_t>(value);
    else if (k == "fuse_groups")
      g_fuse_groups = value != 0.0;
    else if (k == "cta_traj")
      g_cta_disabled = value == 0.0;
    else if (k == "cta_cluster")
      g_cta_cluster = static_cast<int>(value);
    else if (k == "group_quads")
      g_group_quads = static_cast<int>(value);
    else if (k == "grid_per_sm")
      g_grid_per_sm = std::max(0, static_cast<int>(value));
    else if (k == "heavy_deg")
      g_heavy_deg = static_cast<int>(value);
    else
      throw std::invalid_argument("mqo_tune: unknown key");
  });
}

extern "C" int mqo_step(mqo_batch* b, const mqo_objective* obj, const mqo_optimizer* opt) {
  return guard([&] {
    if (!b || !obj || !opt) throw std::invalid_argument("mqo_step: null argument");
    validate_objective(*obj);
    MQO_CUDA(cudaSetDevice(b->g->device));
    launch_step(b, *obj, *opt);
  });
}

extern "C" int mqo_gradient(mqo_batch* b, const mqo_objective* obj, double* out) {
  return guard([&] {
    if (!b || !obj || !out) throw std::invalid_argument("mqo_gradient: null argument");
    validate_objective(*obj);
    MQO_CUDA(cudaSetDevice(b->g->device));
    if (b->g->n == 0) return;
    PassArgs a = make_args(b, *obj);
    // gradient output goes to the idle X buffer, then out through aux
    a.gout = b->d_x[b->cur ^ 1];
    pass_fn<kGrad>(obj->kind, b->cpl)<<<pass_blocks(b), kThreads, 0, b->stream>>>(a);
    MQO_CUDA(cudaGetLastError());
    download_chain_major(b, a.gout, out);
  });
}

extern "C" int mqo_run_trajectories(mqo_batch* b, const mqo_objective* obj,
                                    const mqo_optimizer* opt, double deadline_secs,
                                    int32_t* iterations, int32_t* reasons) {
  return guard([&] {
    if (!b || !obj || !opt) throw std::invalid_argument("mqo_run_trajectories: null argument");
    validate_optimizer(*opt);  // run_trajectory validates cfg (pga.cpp:65)
    if (obj->kind < 0 || obj->kind > 4) throw std::invalid_argument("objective: unknown kind");
    if (obj->kind == MQO_MIS_QUBO && !(obj->param > 1.0))
      throw std::invalid_argument("mis_fixed_point_check: gamma must be > 1");
    MQO_CUDA(cudaSetDevice(b->g->device));
    launch_project(b, b->d_x[b->cur], obj->kind == MQO_MIS_QUBO ? MQO_PROBLEM_MIS
                                                                 : MQO_PROBLEM_MAXCUT);
    run_trajectories(b, *obj, *opt, deadline_secs);
    read_outcomes(b, iterations, reasons);
  });
}

extern "C" int mqo_mis_fixed_point_check(mqo_batch* b, double gamma, double alpha,
                                         int32_t* fixed) {
  return guard([&] {
    if (!b || !fixed) throw std::invalid_argument("mqo_mis_fixed_point_check: null argument");
    if (!(gamma > 1.0)) throw std::invalid_argument("mis_fixed_point_check: gamma must be > 1");
    if (!(alpha > 0.0)) throw std::invalid_argument("mis_fixed_point_check: alpha must be > 0");
    MQO_CUDA(cudaSetDevice(b->g->device));
    MQO_CUDA(cudaMemsetAsync(b->d_viol, 0, sizeof(uint32_t) * b->Bp, b->stream));
    MQO_CUDA(cudaMemsetAsync(b->d_flag, 0, sizeof(int32_t) * 4, b->stream));
    if (b->g->n) {
      PassArgs a = make_args(b, mqo_objective{MQO_MIS_QUBO, gamma});
      pass_fn<kCheck>(MQO_MIS_QUBO, b->cpl)<<<pass_blocks(b), kThreads, 0, b->stream>>>(a);
      MQO_CUDA(cudaGetLastError());
    }
    std::vector<uint32_t> viol(b->Bp);
    MQO_CUDA(cudaMemcpyAsync(viol.data(), b->d_viol, sizeof(uint32_t) * b->Bp,
                             cudaMemcpyDeviceToHost, b->stream));
    MQO_CUDA(cudaMemcpyAsync(b->h_flag, b->d_flag, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost,
                             b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
    if (b->h_flag[1]) throw std::invalid_argument("mis_fixed_point_check: state not binary");
    for (int i = 0; i < b->B; ++i) fixed[i] = viol[i] ? 0 : 1;
  });
}
