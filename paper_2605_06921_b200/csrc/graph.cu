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
}  // namespace

extern "C" const char* mqo_last_error(void) { return g_last_error.c_str(); }
extern "C" int32_t mqo_last_error_line(void) { return g_last_error_line; }
extern "C" const char* mqo_version(void) { return "mqo_b200 0.1 sm_100a"; }

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
    // Graph::check_invariants (graph.cpp:44-56) + range checks, then
    // symmetry (u in N(v) <=> v in N(u)), which from_edges guarantees and the
    // local-search kernels rely on.  Rows are checked in parallel chunks on
    // host threads; the first violation in (row, entry) order is reported,
    // invariant violations before symmetry ones, as a sequential scan would.
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
    if (device < 0) {  // host-only graph: symmetry on the host threads
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
    }  // device graphs: k_check_symmetric after the upload below
    auto* g = new mqo_graph;
    g->device = device;
    g->n = n;
    g->m = nnz / 2;
    g->max_degree = max_degree;
    g->h_off.assign(offsets, offsets + n + 1);
    g->h_nbr.assign(neighbors, neighbors + nnz);

    // Degree-descending row order (counting sort, stable in id).
    std::vector<int32_t> order(static_cast<size_t>(n));
    {
      std::vector<int64_t> count(static_cast<size_t>(max_degree) + 2, 0);
      for (int32_t v = 0; v < n; ++v) ++count[max_degree - (offsets[v + 1] - offsets[v])];
      int64_t acc = 0;
      for (auto& c : count) {
        const int64_t t = c;
        c = acc;
        acc += t;
      }
      for (int32_t v = 0; v < n; ++v)
        order[count[max_degree - (offsets[v + 1] - offsets[v])]++] = v;
    }
    MQO_TRACE("graph upload: host copies + row order");
    g->h_deg_ge.assign(static_cast<size_t>(max_degree) + 2, 0);
    for (int32_t v = 0; v < n; ++v) ++g->h_deg_ge[static_cast<size_t>(offsets[v + 1] - offsets[v])];
    for (int64_t d = max_degree; d >= 0; --d) g->h_deg_ge[d] += g->h_deg_ge[d + 1];
    if (device < 0) {  // host-only graph: CSR kept for host-side users, no HBM copy
      *out = g;
      return;
    }
    try {
      MQO_CUDA(cudaSetDevice(device));
      // stream-ordered pool allocations on the device's memory stream
      // (mem.cu): no page mapping per upload, no device-wide sync per free
      const cudaStream_t ms = mem_stream(device);
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
      if (n)
        MQO_CUDA(cudaMemcpyAsync(g->d_order, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, ms));
      // symmetry, one thread per entry on the device; the flag word rides
      // behind the order array
      unsigned long long* d_bad = reinterpret_cast<unsigned long long*>(
          reinterpret_cast<char*>(g->d_order) + (sizeof(int32_t) * std::max<int32_t>(n, 1) + 7) / 8 * 8);
      MQO_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), ms));
      if (nnz)
        k_check_symmetric<<<static_cast<int>(std::min<int64_t>((nnz + 255) / 256, 148 * 64)), 256, 0, ms>>>(
            g->d_off, g->d_nbr, n, nnz, d_bad);
      MQO_CUDA(cudaGetLastError());
      unsigned long long* h_bad = static_cast<unsigned long long*>(pinned_get(sizeof(unsigned long long)));
      const cudaError_t e1 = cudaMemcpyAsync(h_bad, d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ms);
      const cudaError_t e2 = cudaStreamSynchronize(ms);
      const unsigned long long bad = *h_bad;
      pinned_put(h_bad, sizeof(unsigned long long));
      MQO_CUDA(e1);
      MQO_CUDA(e2);
      if (bad != ~0ull) throw std::logic_error("graph: adjacency not symmetric");
      MQO_TRACE("graph upload: on the device, symmetry checked");
    } catch (...) {
      mqo_graph_free(g);
      throw;
    }
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
                      static_cast<void*>(g->d_hmax)})
        if (p) cudaFreeAsync(p, ms);
    }
    delete g;
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
