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
    // Graph::check_invariants (graph.cpp:44-56) + range checks.
    int32_t max_degree = 0;
    for (int32_t v = 0; v < n; ++v) {
      const int64_t b = offsets[v], e = offsets[v + 1];
      if (e < b) throw std::logic_error("graph: offsets not monotone");
      for (int64_t i = b; i < e; ++i) {
        const int32_t u = neighbors[i];
        if (u < 0 || u >= n) throw std::invalid_argument("graph: vertex index out of range");
        if (u == v) throw std::logic_error("graph: self-loop");
        if (i > b && neighbors[i - 1] >= u)
          throw std::logic_error("graph: neighbor list not strictly ascending");
      }
      max_degree = std::max<int32_t>(max_degree, static_cast<int32_t>(e - b));
    }
    // Symmetry (u in N(v) <=> v in N(u)), which from_edges guarantees and
    // the local-search kernels rely on, in O(m): rows are sorted, so the
    // lower entries of row u are exactly the v < u whose rows hold u, met in
    // ascending v when the rows are walked in order.
    {
      std::vector<int64_t> low(static_cast<size_t>(n), 0);  // lower entries of row u matched so far
      for (int32_t v = 0; v < n; ++v)
        for (int64_t i = offsets[v]; i < offsets[v + 1]; ++i) {
          const int32_t u = neighbors[i];
          if (u < v) continue;
          const int64_t at = offsets[u] + low[u];
          if (at >= offsets[u + 1] || neighbors[at] != v)
            throw std::logic_error("graph: adjacency not symmetric");
          ++low[u];
        }
      for (int32_t u = 0; u < n; ++u) {
        const int64_t b = offsets[u], e = offsets[u + 1];
        if (low[u] != (std::lower_bound(neighbors + b, neighbors + e, u) - (neighbors + b)))
          throw std::logic_error("graph: adjacency not symmetric");
      }
    }
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
    g->h_deg_ge.assign(static_cast<size_t>(max_degree) + 2, 0);
    for (int32_t v = 0; v < n; ++v) ++g->h_deg_ge[static_cast<size_t>(offsets[v + 1] - offsets[v])];
    for (int64_t d = max_degree; d >= 0; --d) g->h_deg_ge[d] += g->h_deg_ge[d + 1];
    if (device < 0) {  // host-only graph: CSR kept for host-side users, no HBM copy
      *out = g;
      return;
    }
    try {
      MQO_CUDA(cudaSetDevice(device));
      MQO_CUDA(cudaMalloc(&g->d_off, sizeof(int64_t) * (n + 1)));
      MQO_CUDA(cudaMalloc(&g->d_nbr, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
      MQO_CUDA(cudaMalloc(&g->d_order, sizeof(int32_t) * std::max<int32_t>(n, 1)));
      MQO_CUDA(cudaMemcpy(g->d_off, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
      if (nnz)
        MQO_CUDA(cudaMemcpy(g->d_nbr, neighbors, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
      if (n)
        MQO_CUDA(cudaMemcpy(g->d_order, order.data(), sizeof(int32_t) * n,
                            cudaMemcpyHostToDevice));
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
    if (g->device >= 0) cudaSetDevice(g->device);
    cudaFree(g->d_off);
    cudaFree(g->d_nbr);
    cudaFree(g->d_order);
    cudaFree(g->d_cta);
    cudaFree(g->d_hmax);
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
