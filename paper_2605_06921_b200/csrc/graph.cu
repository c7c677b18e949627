// graph.cu -- the CSR graph store in HBM (reference: Graph, graph.hpp:20-63;
// construction invariants graph.cpp:44-56).
//
// Device layout: int64 offsets[n+1], int32 neighbours[2m] exactly as the
// reference's CSR (rows strictly ascending -- the fused kernels accumulate
// in that order, which is what makes them bit-identical), plus an int32
// row order sorted by degree descending (stable by id) that the kernels
// walk so hub rows start first and rows of similar degree share a warp.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <thread>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace mqo_b200 {

static thread_local std::string g_last_error;
static thread_local int32_t g_last_error_line = 0;
void set_error(const std::string& msg) {
  g_last_error = msg;
  g_last_error_line = 0;
}
void set_error_line(int32_t line) { g_last_error_line = line; }
double trace_clock() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<double>(ts.tv_sec) + 1e-9 * static_cast<double>(ts.tv_nsec);
}
bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("MQO_TRACE");
    return e && *e && *e != '0';
  }();
  return on;
}

}  // namespace mqo_b200

using namespace mqo_b200;

namespace {
// Symmetry of an uploaded CSR (rows already checked sorted and in range):
// entry e = (v, u) needs v in row u.  One thread per entry; the row of e by
// binary search over the offsets; *bad = the smallest failing entry.
__global__ void k_check_symmetric(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                  int32_t n, int64_t nnz, unsigned long long* bad) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t lo = 0, hi = n - 1;  // row v: off[v] <= e < off[v + 1]
    while (lo < hi) {
      const int32_t mid = lo + (hi - lo + 1) / 2;
      if (off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const int32_t v = lo, u = nbr[e];
    int64_t a = off[u], b = off[u + 1];
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (nbr[mid] < v) a = mid + 1; else b = mid;
    }
    if (a == off[u + 1] || nbr[a] != v) atomicMin(bad, static_cast<unsigned long long>(e));
  }
}

// Graph::check_invariants (graph.cpp:44-56) + range checks of an uploaded
// CSR, a warp per row: *bad = the smallest (row << 32 | code) over the
// violations, code 0 = the row's offsets decrease (or leave [0, nnz]), else
// 1 + the entry's position in the row -- the order a sequential scan meets
// them; *maxdeg = the largest degree.
__global__ void k_check_rows(const int64_t* __restrict__ off, const int32_t* __restrict__ nbr,
                             int32_t n, int64_t nnz, unsigned long long* bad, int32_t* maxdeg) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  int32_t dmax = 0;
  for (int64_t v = w0; v < n; v += nw) {
    const int64_t b = off[v], e = off[v + 1];
    if (e < b || b < 0 || e > nnz) {
      if (lane == 0) atomicMin(bad, static_cast<unsigned long long>(v) << 32);
      continue;
    }
    dmax = max(dmax, static_cast<int32_t>(e - b));
    for (int64_t c = b; c < e; c += 32) {
      const int64_t i = c + lane;
      bool wrong = false;
      if (i < e) {
        const int32_t u = nbr[i];
        wrong = u < 0 || u >= n || u == v || (i > b && nbr[i - 1] >= u);
      }
      const unsigned m = __ballot_sync(0xffffffffu, wrong);
      if (m) {
        if (lane == 0)
          atomicMin(bad, (static_cast<unsigned long long>(v) << 32) |
                             static_cast<unsigned long long>(c + __ffs(m) - b));
        break;
      }
    }
  }
  for (int o = 16; o; o >>= 1) dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if (lane == 0 && dmax) atomicMax(maxdeg, dmax);
}

// sort keys of the degree-descending row order (stable radix sort by
// max_degree - degree) and the degree histogram
__global__ void k_order_keys(const int64_t* __restrict__ off, int32_t n, int32_t max_degree,
                             uint32_t* __restrict__ keys, int32_t* __restrict__ ids,
                             int32_t* __restrict__ hist) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t d = static_cast<int32_t>(off[v + 1] - off[v]);
    keys[v] = static_cast<uint32_t>(max_degree - d);
    ids[v] = static_cast<int32_t>(v);
    atomicAdd(hist + d, 1);
  }
}
}  // namespace

namespace mqo_b200 {
void host_csr(const mqo_graph* cg) {
  auto* g = const_cast<mqo_graph*>(cg);
  std::lock_guard<std::mutex> lock(g->host_mu);
  if (g->h_csr) return;
  int prev = 0;
  MQO_CUDA(cudaGetDevice(&prev));
  MQO_CUDA(cudaSetDevice(g->device));
  g->h_off.resize(static_cast<size_t>(g->n) + 1);
  g->h_nbr.resize(static_cast<size_t>(2 * g->m));
  const cudaError_t e1 =
      cudaMemcpy(g->h_off.data(), g->d_off, sizeof(int64_t) * (g->n + 1), cudaMemcpyDeviceToHost);
  const cudaError_t e2 = g->m ? cudaMemcpy(g->h_nbr.data(), g->d_nbr, sizeof(int32_t) * 2 * g->m,
                                           cudaMemcpyDeviceToHost)
                              : cudaSuccess;
  cudaSetDevice(prev);
  MQO_CUDA(e1);
  MQO_CUDA(e2);
  g->h_csr = true;
}
}  // namespace mqo_b200

extern "C" const char* mqo_last_error(void) { return g_last_error.c_str(); }
extern "C" int32_t mqo_last_error_line(void) { return g_last_error_line; }
extern "C" const char* mqo_version(void) { return "mqo_b200 0.1 sm_100a"; }

namespace {
// A device graph: the CSR goes to HBM as given and every check runs there
// (k_check_rows, then k_check_symmetric), the degree-descending row order is
// a stable radix sort on the device, and the host reads back a few words --
// the caller's neighbour array is never walked on the host (bench.py's e2e
// leg uploads the C4 graph every step: 32 ms with host checks, copies and a
// host counting sort).  Errors are the host path's, in the same order: the
// smallest failing (row, entry) is classified from the caller's row.
mqo_graph* upload_device(int32_t n, const int64_t* offsets, const int32_t* neighbors, int64_t nnz,
                         int32_t device) {
  auto* g = new mqo_graph;
  g->device = device;
  g->n = n;
  g->m = nnz / 2;
  void* scratch[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t ms = nullptr;
  unsigned long long* h_w = nullptr;  // pinned read-back words
  const size_t h_words = 4;
  auto cleanup = [&] {
    if (ms) {
      for (void* p : scratch)
        if (p) cudaFreeAsync(p, ms);
    }
    if (h_w) pinned_put(h_w, sizeof(unsigned long long) * h_words);
  };
  try {
    MQO_CUDA(cudaSetDevice(device));
    ms = mem_stream(device);
    void* p = nullptr;
    MQO_CUDA(cudaMallocAsync(&p, sizeof(int64_t) * (n + 1), ms));
    g->d_off = static_cast<int64_t*>(p);
    MQO_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * std::max<int64_t>(nnz, 1), ms));
    g->d_nbr = static_cast<int32_t*>(p);
    MQO_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * std::max<int32_t>(n, 1) + 16, ms));
    g->d_order = static_cast<int32_t*>(p);
    MQO_CUDA(cudaMemcpyAsync(g->d_off, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ms));
    if (nnz)
      MQO_CUDA(cudaMemcpyAsync(g->d_nbr, neighbors, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, ms));
    // flag words: [0] invariant key, [1] symmetry entry, [2] max degree
    MQO_CUDA(cudaMallocAsync(&scratch[0], sizeof(unsigned long long) * 4, ms));
    auto* d_w = static_cast<unsigned long long*>(scratch[0]);
    MQO_CUDA(cudaMemsetAsync(d_w, 0xff, sizeof(unsigned long long) * 2, ms));
    MQO_CUDA(cudaMemsetAsync(d_w + 2, 0, sizeof(unsigned long long) * 2, ms));
    const int grid = 148 * 16;
    if (n) k_check_rows<<<grid, 256, 0, ms>>>(g->d_off, g->d_nbr, n, nnz, d_w, reinterpret_cast<int32_t*>(d_w + 2));
    MQO_CUDA(cudaGetLastError());
    h_w = static_cast<unsigned long long*>(pinned_get(sizeof(unsigned long long) * h_words));
    MQO_CUDA(cudaMemcpyAsync(h_w, d_w, sizeof(unsigned long long) * 3, cudaMemcpyDeviceToHost, ms));
    MQO_CUDA(cudaStreamSynchronize(ms));
    if (h_w[0] != ~0ull) {  // the first violation in (row, entry) order
      const int64_t v = static_cast<int64_t>(h_w[0] >> 32);
      const int64_t code = static_cast<int64_t>(h_w[0] & 0xffffffffull);
      if (code == 0) throw std::logic_error("graph: offsets not monotone");
      const int64_t i = offsets[v] + code - 1;
      const int32_t u = neighbors[i];
      if (u < 0 || u >= n) throw std::invalid_argument("graph: vertex index out of range");
      if (u == v) throw std::logic_error("graph: self-loop");
      throw std::logic_error("graph: neighbor list not strictly ascending");
    }
    g->max_degree = static_cast<int32_t>(h_w[2] & 0xffffffffull);
    const int32_t D = g->max_degree;
    MQO_TRACE("graph upload: on the device, invariants checked");
    // symmetry, one thread per entry
    if (nnz)
      k_check_symmetric<<<static_cast<int>(std::min<int64_t>((nnz + 255) / 256, 148 * 64)), 256, 0, ms>>>(
          g->d_off, g->d_nbr, n, nnz, d_w + 1);
    // row order: stable radix sort of (D - degree, id), and the degree histogram
    MQO_CUDA(cudaMallocAsync(&scratch[1], sizeof(uint32_t) * 2 * std::max<int32_t>(n, 1), ms));
    MQO_CUDA(cudaMallocAsync(&scratch[2], sizeof(int32_t) * (std::max<int32_t>(n, 1) + D + 2), ms));
    auto* keys = static_cast<uint32_t*>(scratch[1]);
    auto* ids = static_cast<int32_t*>(scratch[2]);
    int32_t* hist = ids + std::max<int32_t>(n, 1);
    MQO_CUDA(cudaMemsetAsync(hist, 0, sizeof(int32_t) * (D + 2), ms));
    if (n) {
      k_order_keys<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, ms>>>(
          g->d_off, n, D, keys, ids, hist);
      int bits = 1;
      while (bits < 32 && (uint32_t(1) << bits) <= static_cast<uint32_t>(D)) ++bits;
      size_t tmp = 0;
      MQO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys + n, ids, g->d_order, n, 0,
                                               bits, ms));
      MQO_CUDA(cudaMallocAsync(&scratch[3], std::max<size_t>(tmp, 16), ms));
      MQO_CUDA(cub::DeviceRadixSort::SortPairs(scratch[3], tmp, keys, keys + n, ids, g->d_order, n,
                                               0, bits, ms));
    }
    MQO_CUDA(cudaGetLastError());
    g->h_deg_ge.assign(static_cast<size_t>(D) + 2, 0);
    MQO_CUDA(cudaMemcpyAsync(h_w, d_w + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ms));
    MQO_CUDA(cudaMemcpyAsync(g->h_deg_ge.data(), hist, sizeof(int32_t) * (D + 1),
                             cudaMemcpyDeviceToHost, ms));
    MQO_CUDA(cudaStreamSynchronize(ms));
    if (h_w[0] != ~0ull) throw std::logic_error("graph: adjacency not symmetric");
    for (int64_t d = D; d >= 0; --d) g->h_deg_ge[d] += g->h_deg_ge[d + 1];
    MQO_TRACE("graph upload: on the device, symmetry checked, rows ordered");
  } catch (...) {
    if (ms) cudaStreamSynchronize(ms);
    cleanup();
    mqo_graph_free(g);
    throw;
  }
  cleanup();
  return g;
}
}  // namespace

extern "C" int mqo_graph_upload(int32_t n, const int64_t* offsets, const int32_t* neighbors,
                                int32_t device, mqo_graph** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("mqo_graph_upload: null out");
    if (n < 0) throw std::invalid_argument("graph: negative vertex count");
    if (!offsets) throw std::invalid_argument("mqo_graph_upload: null offsets");
    if (offsets[0] != 0) throw std::logic_error("graph: offsets[0] != 0");
    const int64_t nnz = offsets[n];
    if (nnz < 0 || (nnz & 1)) throw std::logic_error("graph: degree sum != 2m");
    if (nnz > 0 && !neighbors) throw std::invalid_argument("mqo_graph_upload: null neighbors");
    if (device >= 0) {
      *out = upload_device(n, offsets, neighbors, nnz, device);
      return;
    }
    // Host-only graph: Graph::check_invariants (graph.cpp:44-56) + range
    // checks, then symmetry (u in N(v) <=> v in N(u)), which from_edges
    // guarantees and the local-search kernels rely on.  Rows are checked in
    // parallel chunks on host threads; the first violation in (row, entry)
    // order is reported, invariant violations before symmetry ones, as a
    // sequential scan would.
    struct Bad {
      int64_t at = INT64_MAX;  // global entry index (or row for "not monotone")
      int kind = 0;            // 1 not monotone, 2 range, 3 self-loop, 4 not ascending
    };
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int T = nnz > (int64_t(1) << 18) ? static_cast<int>(hw) : 1;
    std::vector<int32_t> cut(T + 1, n);
    cut[0] = 0;
    for (int t = 1; t < T; ++t) {  // chunk boundaries by entries
      const int64_t target = nnz / T * t;
      cut[t] = static_cast<int32_t>(std::upper_bound(offsets, offsets + n + 1, target) - offsets) - 1;
      cut[t] = std::max(cut[t], cut[t - 1]);
    }
    std::vector<Bad> inv(T), sym(T);
    std::vector<int32_t> dmax(T, 0);
    auto run = [&](auto&& body) {
      std::vector<std::thread> th;
      for (int t = 1; t < T; ++t) th.emplace_back(body, t);
      body(0);
      for (auto& x : th) x.join();
    };
    run([&](int t) {
      for (int32_t v = cut[t]; v < cut[t + 1]; ++v) {
        const int64_t b = offsets[v], e = offsets[v + 1];
        if (e < b) {
          inv[t] = {b, 1};
          return;
        }
        for (int64_t i = b; i < e; ++i) {
          const int32_t u = neighbors[i];
          const int kind = (u < 0 || u >= n) ? 2 : u == v ? 3 : (i > b && neighbors[i - 1] >= u) ? 4 : 0;
          if (kind) {
            inv[t] = {i, kind};
            return;
          }
        }
        dmax[t] = std::max<int32_t>(dmax[t], static_cast<int32_t>(e - b));
      }
    });
    for (const Bad& x : inv) {
      if (x.kind == 1) throw std::logic_error("graph: offsets not monotone");
      if (x.kind == 2) throw std::invalid_argument("graph: vertex index out of range");
      if (x.kind == 3) throw std::logic_error("graph: self-loop");
      if (x.kind == 4) throw std::logic_error("graph: neighbor list not strictly ascending");
    }
    const int32_t max_degree = *std::max_element(dmax.begin(), dmax.end());
    MQO_TRACE("graph upload: invariants checked (%d threads)", T);
    {  // symmetry on the host threads
      run([&](int t) {
        for (int32_t v = cut[t]; v < cut[t + 1]; ++v)
          for (int64_t i = offsets[v]; i < offsets[v + 1]; ++i) {
            const int32_t u = neighbors[i];
            if (!std::binary_search(neighbors + offsets[u], neighbors + offsets[u + 1], v)) {
              sym[t] = {i, 5};
              return;
            }
          }
      });
      for (const Bad& x : sym)
        if (x.kind) throw std::logic_error("graph: adjacency not symmetric");
      MQO_TRACE("graph upload: symmetry checked");
    }
    auto* g = new mqo_graph;
    g->device = device;
    g->n = n;
    g->m = nnz / 2;
    g->max_degree = max_degree;
    g->h_off.assign(offsets, offsets + n + 1);
    g->h_nbr.assign(neighbors, neighbors + nnz);

    MQO_TRACE("graph upload: host copies");
    g->h_deg_ge.assign(static_cast<size_t>(max_degree) + 2, 0);
    for (int32_t v = 0; v < n; ++v) ++g->h_deg_ge[static_cast<size_t>(offsets[v + 1] - offsets[v])];
    for (int64_t d = max_degree; d >= 0; --d) g->h_deg_ge[d] += g->h_deg_ge[d + 1];
    g->h_csr = true;  // host-only graph: CSR kept for host-side users, no HBM copy
    *out = g;
  });
}

extern "C" int mqo_graph_free(mqo_graph* g) {
  return guard([&] {
    if (!g) return;
    if (g->device >= 0) {  // the graph outlives its batches: no kernel still reads it
      cudaSetDevice(g->device);
      const cudaStream_t ms = mem_stream(g->device);
      for (void* p : {static_cast<void*>(g->d_off), static_cast<void*>(g->d_nbr),
                      static_cast<void*>(g->d_order), static_cast<void*>(g->d_cta),
                      static_cast<void*>(g->d_hmax), static_cast<void*>(g->d_lo),
                      static_cast<void*>(g->d_crow)})
        if (p) cudaFreeAsync(p, ms);
    }
    delete g;
  });
}

extern "C" int mqo_graph_row_order(const mqo_graph* g, int32_t* order) {
  return guard([&] {
    if (!g || !order) throw std::invalid_argument("mqo_graph_row_order: null argument");
    if (g->device < 0) throw std::invalid_argument("mqo_graph_row_order: host-only graph");
    MQO_CUDA(cudaSetDevice(g->device));
    if (g->n)
      MQO_CUDA(cudaMemcpy(order, g->d_order, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost));
  });
}

extern "C" int mqo_graph_info(const mqo_graph* g, int32_t* n, int64_t* m, int32_t* max_degree) {
  return guard([&] {
    if (!g) throw std::invalid_argument("mqo_graph_info: null graph");
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (max_degree) *max_degree = g->max_degree;
  });
}
