// traj_cta.cu -- trajectories of small graphs, one CTA per chain.
//
// Same reference path as pga.cu (run_trajectory, pga.cpp:63-111: fused
// gradient + momentum + clip, MIS fixed-point check, MaxCut ||dx||_inf stop,
// 256-iteration deadline poll) for graphs whose chain state -- and, when it
// fits, the CSR itself -- fits in shared memory (C1/C2-sized).  Chains are
// independent, so each CTA runs one chain's whole trajectory with no grid
// barrier and no per-iteration launch: x (double-buffered) and v live in
// SMEM, the stop flags are block-wide __syncthreads_or reductions, and every
// thread takes the (identical) stop decision itself.  The MIS check of x_t is
// a second SMEM sweep right after x_t is formed, in the reference's order.
// Arithmetic and summation order are those of the fused kernel
// (bit-identical).
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
  int32_t n, B, Bp;
  int64_t nnz;
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

// SMEM_CSR: offsets/neighbours copied to shared memory (int32) when they fit.
template <int KIND, bool SMEM_CSR>
__global__ void __launch_bounds__(512) k_traj_cta(CtaArgs a) {
  constexpr bool MIS = KIND == MQO_MIS_QUBO;
  extern __shared__ double sm[];
  const int n = a.n;
  double* xs0 = sm;
  double* xs1 = sm + n;
  double* vs = sm + 2 * n;
  int32_t* s_off = reinterpret_cast<int32_t*>(sm + 3 * n);  // [n+1]   (SMEM_CSR)
  int32_t* s_nbr = s_off + n + 1;                            // [nnz]   (SMEM_CSR)
  const int b = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;

  for (int v = tid; v < n; v += nt) {
    xs0[v] = a.X[static_cast<int64_t>(v) * a.Bp + b];
    vs[v] = 0.0;  // fresh velocity (pga.cpp:75)
  }
  if constexpr (SMEM_CSR) {
    for (int v = tid; v <= n; v += nt) s_off[v] = static_cast<int32_t>(a.off[v]);
    for (int64_t e = tid; e < a.nnz; e += nt) s_nbr[e] = a.nbr[e];
  }
  __syncthreads();
  auto row_begin = [&](int v) -> int32_t {
    if constexpr (SMEM_CSR) return s_off[v]; else return static_cast<int32_t>(__ldg(a.off + v));
  };
  auto nb = [&](int32_t e) -> int32_t {
    if constexpr (SMEM_CSR) return s_nbr[e]; else return __ldg(a.nbr + e);
  };

  double* xin = xs0;
  double* xout = xs1;
  int out_buf = 1, final_buf = 0, iters = 0, reason = MQO_ITER_CAP;
  for (int t = 1; t <= a.max_iters; ++t) {
    int exceed = 0;
    for (int v = tid; v < n; v += nt) {
      const int32_t e0 = row_begin(v), e1 = row_begin(v + 1);
      const double xv = xin[v];
      double acc = 0.0;
      int32_t e = e0;
      for (; e + 4 <= e1; e += 4) {  // four indices in flight, summed in order
        const int32_t u0 = nb(e), u1 = nb(e + 1), u2 = nb(e + 2), u3 = nb(e + 3);
        const double x0 = xin[u0], x1 = xin[u1], x2 = xin[u2], x3 = xin[u3];
        if constexpr (KIND == MQO_LAPLACIAN) {
          acc = ex_add(acc, ex_sub(xv, x0));
          acc = ex_add(acc, ex_sub(xv, x1));
          acc = ex_add(acc, ex_sub(xv, x2));
          acc = ex_add(acc, ex_sub(xv, x3));
        } else {
          acc = ex_add(ex_add(ex_add(ex_add(acc, x0), x1), x2), x3);
        }
      }
      for (; e < e1; ++e) {
        const double xu = xin[nb(e)];
        acc = KIND == MQO_LAPLACIAN ? ex_add(acc, ex_sub(xv, xu)) : ex_add(acc, xu);
      }
      const double g = grad_cta<KIND>(acc, xv, static_cast<double>(e1 - e0), a.param);
      const double nv = ex_add(ex_mul(a.beta, vs[v]), g);
      const double nx = clamp_box(ex_add(xv, ex_mul(a.alpha, nv)), a.lo);
      if (!MIS && fabs(ex_sub(nx, xv)) > a.conv_tol) exceed = 1;  // max|dx| > tol
      vs[v] = nv;
      xout[v] = nx;
    }
    exceed = __syncthreads_or(exceed);  // also publishes xout
    bool stop = false;
    if (MIS) {
      if (t % a.check_every == 0) {  // mis_fixed_point_check(binarize(x_t)), pga.cpp:91-98
        int bad = 0;
        for (int v = tid; v < n && !bad; v += nt) {
          const int32_t e1 = row_begin(v + 1);
          bool any = false;
          for (int32_t e = row_begin(v); e < e1 && !any; ++e) any = xout[nb(e)] > 0.5;
          bad = (xout[v] > 0.5) ? any : !any;
        }
        if (!__syncthreads_or(bad)) {
          stop = true;
          reason = MQO_CHECKER_ACCEPTED;
        }
      }
    } else if (!exceed) {
      stop = true;
      reason = MQO_CONVERGED;
    }
    // one thread reads the host flag; the block-wide OR keeps every thread's
    // decision identical
    const bool deadline_hit = (t & 255) == 0 && __syncthreads_or(tid == 0 ? *a.stop_flag : 0);
    if (!stop && (t == a.max_iters || deadline_hit)) {
      stop = true;  // iteration cap or deadline (pga.cpp:104-110)
      reason = MQO_ITER_CAP;
    }
    if (stop) {
      final_buf = out_buf;
      iters = t;
      break;
    }
    double* tmp = xin;
    xin = xout;
    xout = tmp;
    out_buf ^= 1;
  }
  const double* src = final_buf ? xs1 : xs0;
  for (int v = tid; v < n; v += nt) a.X[static_cast<int64_t>(v) * a.Bp + b] = src[v];
  if (tid == 0) a.ctl[b] = ChainCtl{0, iters, reason, a.cur};
}

using CtaFn = void (*)(CtaArgs);

template <bool S>
CtaFn cta_fn(int kind) {
  switch (kind) {
    case MQO_MIS_QUBO: return k_traj_cta<MQO_MIS_QUBO, S>;
    case MQO_LAPLACIAN: return k_traj_cta<MQO_LAPLACIAN, S>;
    case MQO_PERTURBED_LAPLACIAN: return k_traj_cta<MQO_PERTURBED_LAPLACIAN, S>;
    case MQO_ADJACENCY: return k_traj_cta<MQO_ADJACENCY, S>;
    case MQO_PERTURBED_BIAS: return k_traj_cta<MQO_PERTURBED_BIAS, S>;
  }
  throw std::invalid_argument("objective: unknown kind");
}

}  // namespace

namespace mqo_b200 {

constexpr size_t kCtaSmemMax = 200 * 1024;
bool g_cta_disabled = false;  // mqo_tune("cta_traj", 0)

size_t cta_state_bytes(const mqo_graph* g) { return static_cast<size_t>(g->n) * 24; }
size_t cta_csr_bytes(const mqo_graph* g) {
  return 4 * (static_cast<size_t>(g->n) + 1) + 4 * static_cast<size_t>(2 * g->m);
}

// 1 when the SMEM trajectory path applies (x double-buffered + v, 24 B per
// vertex, fits), else 0.
int cta_group(const mqo_batch* b) {
  static const bool disabled = [] {
    const char* e = std::getenv("MQO_NO_CTA_TRAJ");
    return e && *e && *e != '0';
  }();
  if (disabled || g_cta_disabled) return 0;
  return b->g->n > 0 && cta_state_bytes(b->g) <= kCtaSmemMax ? 1 : 0;
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
  CtaArgs a{};
  a.off = b->g->d_off;
  a.nbr = b->g->d_nbr;
  a.n = b->g->n;
  a.nnz = 2 * b->g->m;
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
  const bool smem_csr = cta_state_bytes(b->g) + cta_csr_bytes(b->g) <= kCtaSmemMax;
  const size_t smem = cta_state_bytes(b->g) + (smem_csr ? cta_csr_bytes(b->g) : 0);
  CtaFn fn = smem_csr ? cta_fn<true>(obj.kind) : cta_fn<false>(obj.kind);
  MQO_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int threads = std::max(32, std::min(512, ((a.n + 31) / 32) * 32));
  fn<<<b->B, threads, smem, b->stream>>>(a);
  MQO_CUDA(cudaGetLastError());
  MQO_TRACE("cta trajectories launched: %d CTAs x %d threads, smem %zu (csr %s)", b->B, threads,
            smem, smem_csr ? "smem" : "global");
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
