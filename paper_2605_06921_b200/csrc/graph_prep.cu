// graph_prep.cu -- device pre-processing of a graph already in HBM
// (SURVEY §8f-3): strip_isolated (graph.cpp:180-198) and
// connected_components (graph.cpp:200-224).
//
// strip_isolated: removing degree-0 vertices leaves every prefix sum of the
// degrees unchanged, so the core CSR is a relabelling in place: core
// offsets[c] = offsets[core_to_orig[c]], core neighbours[e] =
// orig_to_core[neighbours[e]].  orig_to_core is monotone, so rows stay
// strictly ascending and the core equals the reference's from_edges
// rebuild.  One flag pass + one exclusive scan + two gathers.
//
// connected_components: the reference's DFS emits components in order of
// their smallest vertex, each sorted.  Here: union-find with CAS hooking of
// the larger root onto the smaller (parents only decrease, so the forest
// stays acyclic and a component's root is its smallest vertex), full path
// compression between rounds, until no edge joins two roots; components are
// then numbered by the rank of their root.
#include <cub/device/device_scan.cuh>

#include "common.cuh"

using namespace mqo_b200;

namespace {

inline int grid_for(int64_t work) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16)));
}

__global__ void k_degree_flags(const int64_t* __restrict__ off, int32_t n, int32_t* __restrict__ keep) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    keep[v] = off[v + 1] > off[v] ? 1 : 0;
}

// pos = exclusive scan of keep: kept v -> core index pos[v]; removed v is
// the (v - pos[v])-th removed vertex.
__global__ void k_strip_maps(const int64_t* __restrict__ off, const int32_t* __restrict__ pos,
                             int32_t n, int32_t* __restrict__ o2c, int32_t* __restrict__ c2o,
                             int32_t* __restrict__ removed, int64_t* __restrict__ core_off) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int32_t c = pos[v];
    if (off[v + 1] > off[v]) {
      o2c[v] = c;
      c2o[c] = v;
      core_off[c] = off[v];
    } else {
      o2c[v] = -1;
      removed[v - c] = v;
    }
  }
}

__global__ void k_remap(const int32_t* __restrict__ nbr, int64_t nnz, const int32_t* __restrict__ o2c,
                        int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = o2c[nbr[e]];
}

__device__ __forceinline__ int32_t root_of(const int32_t* p, int32_t x) {
  for (;;) {
    const int32_t y = *reinterpret_cast<const volatile int32_t*>(p + x);
    if (y == x) return x;
    x = y;
  }
}

__global__ void k_cc_init(int32_t n, int32_t* __restrict__ p) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) p[v] = v;
}

// Every edge (v < u) whose endpoints have different roots hooks the larger
// root onto the smaller with a CAS (a root that was hooked meanwhile makes
// the CAS fail; the edge is retried next round).
__global__ void k_cc_hook(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr, int32_t n,
                          int32_t* p, int32_t* changed) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    for (int64_t e = off[v + 1] - 1, e0 = off[v]; e >= e0; --e) {
      const int32_t u = nbr[e];
      if (u < v) break;  // each edge once, from its lower end
      const int32_t rv = root_of(p, v), ru = root_of(p, u);
      if (rv == ru) continue;
      const int32_t hi = max(rv, ru), lo = min(rv, ru);
      atomicCAS(p + hi, hi, lo);
      *changed = 1;
    }
  }
}

__global__ void k_cc_compress(int32_t n, int32_t* p) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    p[v] = root_of(p, v);
}

__global__ void k_root_flags(const int32_t* __restrict__ p, int32_t n, int32_t* __restrict__ is_root) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    is_root[v] = p[v] == v ? 1 : 0;
}

__global__ void k_cc_label(const int32_t* __restrict__ p, const int32_t* __restrict__ rank, int32_t n,
                           int32_t* __restrict__ comp) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    comp[v] = rank[p[v]];
}

// Device buffers freed on scope exit (stream-ordered).
struct DevBufs {
  cudaStream_t st;
  std::vector<void*> ptrs;
  template <class T>
  T* alloc(int64_t count) {
    void* p = nullptr;
    MQO_CUDA(cudaMallocAsync(&p, sizeof(T) * std::max<int64_t>(count, 1), st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~DevBufs() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
};

// exclusive scan of flags[n] into out[n]; returns the total
int32_t scan_flags(const int32_t* flags, int32_t* out, int32_t n, cudaStream_t st, DevBufs& bufs) {
  size_t bytes = 0;
  MQO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags, out, n, st));
  void* tmp = bufs.alloc<unsigned char>(static_cast<int64_t>(bytes));
  MQO_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, flags, out, n, st));
  int32_t last[2] = {0, 0};
  MQO_CUDA(cudaMemcpyAsync(&last[0], out + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  MQO_CUDA(cudaMemcpyAsync(&last[1], flags + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  MQO_CUDA(cudaStreamSynchronize(st));
  return last[0] + last[1];
}

void require_device_graph(const mqo_graph* g, const char* who) {
  if (!g) throw std::invalid_argument(std::string(who) + ": null graph");
  if (g->device < 0) throw std::invalid_argument(std::string(who) + ": host-only graph (device < 0)");
}

}  // namespace

extern "C" int mqo_graph_strip_isolated(const mqo_graph* g, mqo_graph** core, int32_t* core_to_orig,
                                        int32_t* orig_to_core, int32_t* removed, int32_t* n_core,
                                        int32_t* n_removed) {
  return guard([&] {
    require_device_graph(g, "mqo_graph_strip_isolated");
    if (!core || !n_core || !n_removed) throw std::invalid_argument("mqo_graph_strip_isolated: null out");
    const int32_t n = g->n;
    const int64_t nnz = 2 * g->m;
    MQO_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = nullptr;
    MQO_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    int32_t nc = 0;
    std::vector<int64_t> h_off(1, 0);
    std::vector<int32_t> h_nbr;
    {
      DevBufs bufs{st, {}};
      if (n > 0) {
        int32_t* keep = bufs.alloc<int32_t>(n);
        int32_t* pos = bufs.alloc<int32_t>(n);
        int32_t* o2c = bufs.alloc<int32_t>(n);
        int32_t* c2o = bufs.alloc<int32_t>(n);
        int32_t* rem = bufs.alloc<int32_t>(n);
        int64_t* coff = bufs.alloc<int64_t>(int64_t(n) + 1);
        int32_t* cnbr = bufs.alloc<int32_t>(nnz);
        k_degree_flags<<<grid_for(n), 256, 0, st>>>(g->d_off, n, keep);
        nc = scan_flags(keep, pos, n, st, bufs);
        k_strip_maps<<<grid_for(n), 256, 0, st>>>(g->d_off, pos, n, o2c, c2o, rem, coff);
        MQO_CUDA(cudaMemcpyAsync(coff + nc, g->d_off + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
        if (nnz) k_remap<<<grid_for(nnz), 256, 0, st>>>(g->d_nbr, nnz, o2c, cnbr);
        MQO_CUDA(cudaGetLastError());
        h_off.resize(static_cast<size_t>(nc) + 1);
        h_nbr.resize(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
        MQO_CUDA(cudaMemcpyAsync(h_off.data(), coff, sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost, st));
        if (nnz)
          MQO_CUDA(cudaMemcpyAsync(h_nbr.data(), cnbr, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, st));
        if (orig_to_core)
          MQO_CUDA(cudaMemcpyAsync(orig_to_core, o2c, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        if (core_to_orig && nc)
          MQO_CUDA(cudaMemcpyAsync(core_to_orig, c2o, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, st));
        if (removed && n > nc)
          MQO_CUDA(cudaMemcpyAsync(removed, rem, sizeof(int32_t) * (n - nc), cudaMemcpyDeviceToHost, st));
        MQO_CUDA(cudaStreamSynchronize(st));
      }
    }
    *n_core = nc;
    *n_removed = n - nc;
    MQO_TRACE("strip_isolated: %d -> %d vertices", n, nc);
    // the core handle (HBM CSR + host copy + degree order) through the standard path
    const int rc = mqo_graph_upload(nc, h_off.data(), h_nbr.data(), g->device, core);
    if (rc != MQO_OK) throw std::logic_error(mqo_last_error());
  });
}

extern "C" int mqo_graph_components(const mqo_graph* g, int32_t* comp, int32_t* count) {
  return guard([&] {
    require_device_graph(g, "mqo_graph_components");
    if (!comp || !count) throw std::invalid_argument("mqo_graph_components: null out");
    const int32_t n = g->n;
    *count = 0;
    if (n == 0) return;
    MQO_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = nullptr;
    MQO_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevBufs bufs{st, {}};
    int32_t* p = bufs.alloc<int32_t>(n);
    int32_t* flags = bufs.alloc<int32_t>(n);
    int32_t* rank = bufs.alloc<int32_t>(n);
    int32_t* d_changed = bufs.alloc<int32_t>(1);
    k_cc_init<<<grid_for(n), 256, 0, st>>>(n, p);
    int rounds = 0;
    for (;; ++rounds) {
      MQO_CUDA(cudaMemsetAsync(d_changed, 0, sizeof(int32_t), st));
      k_cc_hook<<<grid_for(n), 256, 0, st>>>(g->d_off, g->d_nbr, n, p, d_changed);
      k_cc_compress<<<grid_for(n), 256, 0, st>>>(n, p);
      MQO_CUDA(cudaGetLastError());
      int32_t changed = 0;
      MQO_CUDA(cudaMemcpyAsync(&changed, d_changed, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      MQO_CUDA(cudaStreamSynchronize(st));
      if (!changed) break;
    }
    k_root_flags<<<grid_for(n), 256, 0, st>>>(p, n, flags);
    *count = scan_flags(flags, rank, n, st, bufs);
    k_cc_label<<<grid_for(n), 256, 0, st>>>(p, rank, n, flags);
    MQO_CUDA(cudaGetLastError());
    MQO_CUDA(cudaMemcpyAsync(comp, flags, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    MQO_CUDA(cudaStreamSynchronize(st));
    MQO_TRACE("connected_components: %d components after %d hooking rounds", *count, rounds + 1);
  });
}
