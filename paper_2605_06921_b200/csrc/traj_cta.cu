// traj_cta.cu -- trajectories of small graphs, one CTA per chain group.
//
// Same reference path as pga.cu (run_trajectory, pga.cpp:63-111: fused
// gradient + momentum + clip, MIS fixed-point check, MaxCut ||dx||_inf stop,
// 256-iteration deadline poll) for graphs whose state fits in shared memory
// (C1/C2-sized: n x G x 24 B <= ~200 KB).  Chains are independent, so each
// CTA runs its G chains' whole trajectories with __syncthreads only -- no
// grid barrier, no per-iteration launch -- and x, v live in SMEM (the CSR
// is read through L1).  The MIS check of x_t is a second sweep over SMEM
// right after x_t is formed, in the reference's order.  Arithmetic and
// summation order are those of the fused kernel (bit-identical).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>

#include "common.cuh"

using namespace mqo_b200;

namespace {

struct CtaArgs {
  const int64_t* __restrict__ off;
  const int32_t* __restrict__ nbr;
  int32_t n, B, Bp, G;
  double* X;  // [n][Bp] in/out (current buffer)
  ChainCtl* ctl;
  double param, alpha, beta, lo, conv_tol;
  int32_t max_iters, check_every, cur;
  const volatile int32_t* stop_flag;  // host-mapped: deadline passed
};

template <int KIND>
__device__ __forceinline__ double grad_cta(double acc, double x, double deg, double param) {
  if constexpr (KIND == MQO_MIS_QUBO) return ex_sub(1.0, ex_mul(param, acc));
  if constexpr (KIND == MQO_LAPLACIAN) return ex_mul(acc, 0.5);
  if constexpr (KIND == MQO_PERTURBED_LAPLACIAN)
    return ex_mul(2.0, ex_add(ex_sub(ex_mul(deg, x), acc), ex_mul(param, x)));
  if constexpr (KIND == MQO_ADJACENCY) return ex_mul(acc, -2.0);
  return ex_sub(ex_mul(-2.0, acc), param);
}

template <int KIND>
__global__ void __launch_bounds__(512) k_traj_cta(CtaArgs a) {
  constexpr bool MIS = KIND == MQO_MIS_QUBO;
  extern __shared__ double sm[];
  const int G = a.G, cells = a.n * G;
  double* xs0 = sm;
  double* xs1 = sm + cells;
  double* vs = sm + 2 * cells;
  __shared__ unsigned long long s_chg[8];
  __shared__ int s_viol[8], s_active[8], s_final[8], s_iters[8], s_reason[8], s_any;
  const int b0 = blockIdx.x * G;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int my_c = tid % G;  // nt is a multiple of G: a thread keeps one chain

  for (int i = tid; i < cells; i += nt) {
    const int v = i / G, c = i % G;
    xs0[i] = a.X[static_cast<int64_t>(v) * a.Bp + b0 + c];
    vs[i] = 0.0;  // fresh velocity (pga.cpp:75)
  }
  if (tid < G) {
    s_active[tid] = (b0 + tid < a.B) ? 1 : 0;
    s_final[tid] = 0;
    s_iters[tid] = 0;
    s_reason[tid] = MQO_ITER_CAP;
  }
  __syncthreads();

  double* xin = xs0;
  double* xout = xs1;
  int out_buf = 1;
  for (int t = 1; t <= a.max_iters; ++t) {
    if (tid < G) {
      s_chg[tid] = 0ull;
      s_viol[tid] = 0;
    }
    __syncthreads();
    const bool active = s_active[my_c] != 0;
    double my_chg = 0.0;
    if (active) {
      for (int i = tid; i < cells; i += nt) {
        const int v = i / G;
        const int64_t e0 = __ldg(a.off + v), e1 = __ldg(a.off + v + 1);
        const double xv = xin[i];
        double acc = 0.0;
        for (int64_t e = e0; e < e1; ++e) {
          const double xu = xin[__ldg(a.nbr + e) * G + my_c];
          acc = KIND == MQO_LAPLACIAN ? ex_add(acc, ex_sub(xv, xu)) : ex_add(acc, xu);
        }
        const double g = grad_cta<KIND>(acc, xv, static_cast<double>(e1 - e0), a.param);
        const double nv = ex_add(ex_mul(a.beta, vs[i]), g);
        const double nx = clamp_box(ex_add(xv, ex_mul(a.alpha, nv)), a.lo);
        const double d = fabs(ex_sub(nx, xv));
        my_chg = my_chg < d ? d : my_chg;
        vs[i] = nv;
        xout[i] = nx;
      }
    }
    if (!MIS && active && my_chg > 0.0)
      atomicMax(&s_chg[my_c], static_cast<unsigned long long>(__double_as_longlong(my_chg)));
    __syncthreads();
    const bool check = MIS && (t % a.check_every == 0);
    if (check && active) {  // mis_fixed_point_check of binarize(x_t) (pga.cpp:91-98)
      bool bad = false;
      for (int i = tid; i < cells && !bad; i += nt) {
        const int v = i / G;
        int cnt = 0;
        for (int64_t e = __ldg(a.off + v); e < __ldg(a.off + v + 1); ++e)
          cnt += xout[__ldg(a.nbr + e) * G + my_c] > 0.5 ? 1 : 0;
        bad = xout[i] > 0.5 ? (cnt > 0) : (cnt < 1);
      }
      if (bad) atomicOr(&s_viol[my_c], 1);
    }
    __syncthreads();
    if (tid == 0) {
      bool poll = (t & 255) == 0 && *a.stop_flag;  // deadline, pga.cpp:104-107
      int any = 0;
      for (int c = 0; c < G; ++c) {
        if (!s_active[c]) continue;
        int reason = -1;
        if (MIS) {
          if (check && !s_viol[c]) reason = MQO_CHECKER_ACCEPTED;
        } else if (__longlong_as_double(static_cast<long long>(s_chg[c])) <= a.conv_tol) {
          reason = MQO_CONVERGED;
        }
        if (reason < 0 && (t == a.max_iters || poll)) reason = MQO_ITER_CAP;
        if (reason >= 0) {
          s_active[c] = 0;
          s_final[c] = out_buf;
          s_iters[c] = t;
          s_reason[c] = reason;
        } else {
          any = 1;
        }
      }
      s_any = any;
    }
    __syncthreads();
    if (!s_any) break;
    double* tmp = xin;
    xin = xout;
    xout = tmp;
    out_buf ^= 1;
  }
  // write every chain's final iterate back to the batch state
  for (int i = tid; i < cells; i += nt) {
    const int v = i / G, c = i % G;
    if (b0 + c >= a.B) continue;
    const double* src = s_final[c] ? xs1 : xs0;
    a.X[static_cast<int64_t>(v) * a.Bp + b0 + c] = src[i];
  }
  if (tid < G && b0 + tid < a.B)
    a.ctl[b0 + tid] = ChainCtl{0, s_iters[tid], s_reason[tid], a.cur};
}

using CtaFn = void (*)(CtaArgs);

CtaFn cta_fn(int kind) {
  switch (kind) {
    case MQO_MIS_QUBO: return k_traj_cta<MQO_MIS_QUBO>;
    case MQO_LAPLACIAN: return k_traj_cta<MQO_LAPLACIAN>;
    case MQO_PERTURBED_LAPLACIAN: return k_traj_cta<MQO_PERTURBED_LAPLACIAN>;
    case MQO_ADJACENCY: return k_traj_cta<MQO_ADJACENCY>;
    case MQO_PERTURBED_BIAS: return k_traj_cta<MQO_PERTURBED_BIAS>;
  }
  throw std::invalid_argument("objective: unknown kind");
}

}  // namespace

namespace mqo_b200 {

constexpr size_t kCtaSmemMax = 200 * 1024;
bool g_cta_disabled = false;  // mqo_tune("cta_traj", 0)

// Chains per CTA for the SMEM trajectory path (one: the most CTAs), or 0
// if a chain's state (x double-buffered + v, 24 B per vertex) does not fit.
int cta_group(const mqo_batch* b) {
  static const bool disabled = [] {
    const char* e = std::getenv("MQO_NO_CTA_TRAJ");
    return e && *e && *e != '0';
  }();
  if (disabled || g_cta_disabled) return 0;
  return static_cast<size_t>(b->g->n) * 24 <= kCtaSmemMax && b->g->n > 0 ? 1 : 0;
}

// Runs the trajectories of every chain from the current x with the SMEM
// kernel; polls `deadline` from the host and raises the mapped stop flag.
void run_trajectories_cta(mqo_batch* b, const mqo_objective& obj, const mqo_optimizer& opt,
                          double deadline, int G, double (*now)()) {
  // the batch's mapped pinned words: [2] is the stop flag
  int32_t* h_stop = b->h_flag + 2;
  int32_t* d_stop = nullptr;
  MQO_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_stop), h_stop, 0));
  *reinterpret_cast<volatile int32_t*>(h_stop) = 0;
  CtaArgs a{};
  a.off = b->g->d_off;
  a.nbr = b->g->d_nbr;
  a.n = b->g->n;
  a.B = b->B;
  a.Bp = b->Bp;
  a.G = G;
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
  const size_t smem = sizeof(double) * 3 * static_cast<size_t>(a.n) * G;
  CtaFn fn = cta_fn(obj.kind);
  MQO_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int blocks = (b->B + G - 1) / G;
  const int threads = std::max(G * 32, std::min(512, ((a.n * G + 31) / 32) * 32));
  fn<<<blocks, threads - threads % G, smem, b->stream>>>(a);
  MQO_CUDA(cudaGetLastError());
  MQO_TRACE("cta trajectories launched: %d CTAs x %d threads, smem %zu", blocks, threads, smem);
  // wait, raising the stop flag once the deadline has passed
  for (;;) {
    const cudaError_t q = cudaStreamQuery(b->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) MQO_CUDA(q);
    if (deadline >= 0.0 && now() >= deadline) *reinterpret_cast<volatile int32_t*>(h_stop) = 1;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  MQO_TRACE("cta trajectories done");
}

}  // namespace mqo_b200
