// batch.cu -- chain batches: device state of B independent trajectories of
// one graph (the reference keeps one RelaxedState / velocity vector per
// trajectory, objectives.hpp:45-48, pga.cpp:75).  Host buffers are
// chain-major [B][n] (the reference's vectors back to back); the device
// keeps X and V vertex-major [n][Bp] so a neighbour gather of all chains is
// one contiguous row.  Conversion is a tiled shared-memory transpose.
#include <algorithm>

#include "common.cuh"

using namespace mqo_b200;

namespace {

// chain-major [B][n] -> vertex-major [n][Bp]
__global__ void k_to_vertex_major(const double* __restrict__ src, double* __restrict__ dst,
                                  int32_t n, int32_t B, int32_t Bp) {
  __shared__ double tile[32][33];
  const int v0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int b = b0 + i, v = v0 + threadIdx.x;
    if (b < B && v < n) tile[i][threadIdx.x] = src[static_cast<int64_t>(b) * n + v];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int v = v0 + i, b = b0 + threadIdx.x;
    if (v < n && b < B) dst[static_cast<int64_t>(v) * Bp + b] = tile[threadIdx.x][i];
  }
}

// vertex-major [n][Bp] -> chain-major [B][n]
__global__ void k_to_chain_major(const double* __restrict__ src, double* __restrict__ dst,
                                 int32_t n, int32_t B, int32_t Bp) {
  __shared__ double tile[32][33];
  const int v0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int v = v0 + i, b = b0 + threadIdx.x;
    if (v < n && b < B) tile[i][threadIdx.x] = src[static_cast<int64_t>(v) * Bp + b];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int b = b0 + i, v = v0 + threadIdx.x;
    if (b < B && v < n) dst[static_cast<int64_t>(b) * n + v] = tile[threadIdx.x][i];
  }
}

__global__ void k_project(double* __restrict__ x, int64_t count, double lo) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = clamp_box(x[i], lo);
}

}  // namespace

namespace mqo_b200 {
double* aux_buffer(mqo_batch* b) {
  if (!b->d_aux)
    dalloc(b, &b->d_aux, sizeof(double) * std::max<int64_t>(1, int64_t(b->g->n) * b->Bp));
  return b->d_aux;
}

// Copy-in at the API: the host buffer is read completely before the call
// returns (for pinned memory cudaMemcpyAsync would otherwise still be
// reading it), so callers may reuse it at once.
void upload_chain_major(mqo_batch* b, const double* host, double* dst) {
  const mqo_graph* g = b->g;
  const int64_t count = static_cast<int64_t>(g->n) * b->B;
  if (b->Bp == 1) {  // one chain: vertex-major is chain-major, no staging
    MQO_CUDA(cudaMemcpyAsync(dst, host, sizeof(double) * count, cudaMemcpyHostToDevice, b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
    return;
  }
  double* staging = aux_buffer(b);
  MQO_CUDA(cudaMemcpyAsync(staging, host, sizeof(double) * count, cudaMemcpyHostToDevice,
                           b->stream));
  MQO_CUDA(cudaStreamSynchronize(b->stream));
  if (b->Bp != b->B)
    MQO_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * g->n * static_cast<int64_t>(b->Bp),
                             b->stream));
  if (g->n == 0 || b->B == 0) return;
  dim3 grid((g->n + 31) / 32, (b->B + 31) / 32), block(32, 8);
  k_to_vertex_major<<<grid, block, 0, b->stream>>>(staging, dst, g->n, b->B, b->Bp);
  MQO_CUDA(cudaGetLastError());
}

void download_chain_major(mqo_batch* b, const double* src, double* host) {
  const mqo_graph* g = b->g;
  const int64_t count = static_cast<int64_t>(g->n) * b->B;
  if (b->Bp == 1) {
    MQO_CUDA(cudaMemcpyAsync(host, src, sizeof(double) * count, cudaMemcpyDeviceToHost, b->stream));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
    return;
  }
  double* staging = aux_buffer(b);
  if (g->n && b->B) {
    dim3 grid((g->n + 31) / 32, (b->B + 31) / 32), block(32, 8);
    k_to_chain_major<<<grid, block, 0, b->stream>>>(src, staging, g->n, b->B, b->Bp);
    MQO_CUDA(cudaGetLastError());
  }
  MQO_CUDA(cudaMemcpyAsync(host, staging, sizeof(double) * count, cudaMemcpyDeviceToHost,
                           b->stream));
  MQO_CUDA(cudaStreamSynchronize(b->stream));
}

void free_solver_buffers(mqo_batch* b);

void launch_project(mqo_batch* b, double* x, int32_t problem) {
  const int64_t count = static_cast<int64_t>(b->g->n) * b->Bp;
  if (!count) return;
  const int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 16));
  k_project<<<blocks, 256, 0, b->stream>>>(x, count, problem == MQO_PROBLEM_MIS ? 0.0 : -1.0);
  MQO_CUDA(cudaGetLastError());
}
}  // namespace mqo_b200

namespace mqo_b200 {
// The per-round work (reset scratch, local-search workspaces) uses
// cudaMallocAsync; with the default pool's release threshold of 0 every
// stream synchronisation hands the memory back and the next round maps it
// again.  Keep it (MQO_POOL_RELEASE=1 restores the driver default).
void keep_pool_memory(int device) {
  static const bool release = [] {
    const char* e = std::getenv("MQO_POOL_RELEASE");
    return e && *e == '1';
  }();
  if (release) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
}
}  // namespace mqo_b200

extern "C" int mqo_batch_create(mqo_graph* g, int32_t chains, mqo_batch** out) {
  return guard([&] {
    if (!g || !out) throw std::invalid_argument("mqo_batch_create: null argument");
    if (chains < 1) throw std::invalid_argument("mqo_batch_create: chains must be >= 1");
    if (g->device < 0) throw std::invalid_argument("mqo_batch_create: host-only graph");
    auto* b = new mqo_batch;
    b->g = g;
    b->B = chains;
    b->cpl = chains_per_lane(chains);
    b->Q = quads_per_row(chains, b->cpl);
    b->Bp = b->Q * b->cpl;
    try {
      MQO_CUDA(cudaSetDevice(g->device));
      keep_pool_memory(g->device);
      MQO_CUDA(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
      // stream-ordered allocations from the device's pool, which keeps its
      // memory (keep_pool_memory): a solve's batch and scratch come back
      // without a driver mapping the next time (the engine creates a batch
      // per solve)
      const size_t state = sizeof(double) * std::max<int64_t>(1, int64_t(g->n) * b->Bp);
      dalloc(b, &b->d_x[0], state);
      dalloc(b, &b->d_x[1], state);
      dalloc(b, &b->d_v, state);
      MQO_CUDA(cudaMemsetAsync(b->d_x[0], 0, state, b->stream));
      MQO_CUDA(cudaMemsetAsync(b->d_x[1], 0, state, b->stream));
      MQO_CUDA(cudaMemsetAsync(b->d_v, 0, state, b->stream));
      dalloc(b, &b->d_ctl, sizeof(ChainCtl) * b->Bp);
      dalloc(b, &b->d_viol, sizeof(uint32_t) * 3 * b->Bp);
      dalloc(b, &b->d_chg, sizeof(unsigned long long) * 3 * b->Bp);
      dalloc(b, &b->d_flag, sizeof(int32_t) * 4);
      dalloc(b, &b->d_qmask, std::max(1, b->Q));
      b->h_flag = static_cast<int32_t*>(pinned_get(sizeof(int32_t) * 4));
      b->h_flag[2] = 0;
      MQO_CUDA(cudaStreamSynchronize(b->stream));
    } catch (...) {
      mqo_batch_free(b);
      throw;
    }
    *out = b;
  });
}

extern "C" int mqo_batch_free(mqo_batch* b) {
  return guard([&] {
    if (!b) return;
    cudaSetDevice(b->g->device);
    if (b->stream) {
      dfree(b, b->d_x[0]);
      dfree(b, b->d_x[1]);
      dfree(b, b->d_v);
      dfree(b, b->d_aux);
      dfree(b, b->d_ctl);
      dfree(b, b->d_viol);
      dfree(b, b->d_chg);
      dfree(b, b->d_flag);
      dfree(b, b->d_qmask);
      free_solver_buffers(b);
      dfree(b, b->d_ls);
      dfree(b, b->d_flip);
      cudaStreamSynchronize(b->stream);
    }
    pinned_put(b->h_ls, b->ls_bytes);
    pinned_put(b->h_flag, sizeof(int32_t) * 4);
    if (b->stream) cudaStreamDestroy(b->stream);
    delete b;
  });
}

extern "C" int mqo_batch_chains(const mqo_batch* b, int32_t* chains, int32_t* padded) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_batch_chains: null batch");
    if (chains) *chains = b->B;
    if (padded) *padded = b->Bp;
  });
}

extern "C" int mqo_batch_stream(const mqo_batch* b, void** stream) {
  return guard([&] {
    if (!b || !stream) throw std::invalid_argument("mqo_batch_stream: null argument");
    *stream = reinterpret_cast<void*>(b->stream);
  });
}

extern "C" int mqo_batch_sync(mqo_batch* b) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_batch_sync: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    MQO_CUDA(cudaStreamSynchronize(b->stream));
  });
}

extern "C" int mqo_batch_set_x(mqo_batch* b, const double* x) {
  return guard([&] {
    if (!b || !x) throw std::invalid_argument("mqo_batch_set_x: null argument");
    MQO_CUDA(cudaSetDevice(b->g->device));
    upload_chain_major(b, x, b->d_x[b->cur]);
  });
}

extern "C" int mqo_batch_get_x(mqo_batch* b, double* x) {
  return guard([&] {
    if (!b || !x) throw std::invalid_argument("mqo_batch_get_x: null argument");
    MQO_CUDA(cudaSetDevice(b->g->device));
    download_chain_major(b, b->d_x[b->cur], x);
  });
}

extern "C" int mqo_batch_set_v(mqo_batch* b, const double* v) {
  return guard([&] {
    if (!b || !v) throw std::invalid_argument("mqo_batch_set_v: null argument");
    MQO_CUDA(cudaSetDevice(b->g->device));
    upload_chain_major(b, v, b->d_v);
  });
}

extern "C" int mqo_batch_get_v(mqo_batch* b, double* v) {
  return guard([&] {
    if (!b || !v) throw std::invalid_argument("mqo_batch_get_v: null argument");
    MQO_CUDA(cudaSetDevice(b->g->device));
    download_chain_major(b, b->d_v, v);
  });
}

extern "C" int mqo_batch_zero_v(mqo_batch* b) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_batch_zero_v: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    MQO_CUDA(cudaMemsetAsync(b->d_v, 0, sizeof(double) * int64_t(b->g->n) * b->Bp, b->stream));
  });
}

extern "C" int mqo_project(mqo_batch* b, int32_t problem) {
  return guard([&] {
    if (!b) throw std::invalid_argument("mqo_project: null batch");
    MQO_CUDA(cudaSetDevice(b->g->device));
    launch_project(b, b->d_x[b->cur], problem);
  });
}
