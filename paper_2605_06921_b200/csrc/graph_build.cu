// graph_build.cu -- host-side graph construction behind the C ABI:
// Graph::from_edges (graph.cpp:8-42) and the seeded generators
// (graph.cpp:107-178).  Same algorithms and the same xoshiro draws as the
// reference, so a (spec, seed) pair yields the identical CSR; the result is
// uploaded to HBM by mqo_graph_upload.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "rng.cuh"

using namespace mqo_b200;

namespace {

// Canonical CSR from (u<v)-normalised packed keys: sort, unique, count,
// prefix sum, fill, per-row sort (graph.cpp:16-37).
void csr_from_keys(int32_t n, std::vector<uint64_t>& keys, std::vector<int64_t>& off,
                   std::vector<int32_t>& nbr) {
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  const int64_t m = static_cast<int64_t>(keys.size());
  off.assign(static_cast<size_t>(n) + 1, 0);
  for (uint64_t k : keys) {
    ++off[(k >> 32) + 1];
    ++off[(k & 0xffffffffu) + 1];
  }
  for (int32_t v = 0; v < n; ++v) off[v + 1] += off[v];
  nbr.resize(static_cast<size_t>(2 * m));
  std::vector<int64_t> cursor(off.begin(), off.end() - 1);
  // keys are sorted by (u, v).  First give every row its smaller
  // neighbours (for fixed v the keys with second == v arrive in ascending
  // u), then its larger ones (ascending v for fixed u): each row comes out
  // strictly ascending without the per-row sort of graph.cpp:35-37.
  for (uint64_t k : keys) {
    const int32_t u = static_cast<int32_t>(k >> 32), v = static_cast<int32_t>(k & 0xffffffffu);
    nbr[cursor[v]++] = u;
  }
  for (uint64_t k : keys) {
    const int32_t u = static_cast<int32_t>(k >> 32), v = static_cast<int32_t>(k & 0xffffffffu);
    nbr[cursor[u]++] = v;
  }
}

inline uint64_t key_of(int32_t u, int32_t v) {
  if (u > v) std::swap(u, v);
  return (static_cast<uint64_t>(static_cast<uint32_t>(u)) << 32) | static_cast<uint32_t>(v);
}

void build_from_edges(int32_t n, int64_t ne, const int32_t* eu, const int32_t* ev,
                      std::vector<int64_t>& off, std::vector<int32_t>& nbr) {
  if (n < 0) throw std::invalid_argument("graph: negative vertex count");
  std::vector<uint64_t> keys(static_cast<size_t>(ne));
  for (int64_t i = 0; i < ne; ++i) {
    const int32_t u = eu[i], v = ev[i];
    if (u < 0 || u >= n || v < 0 || v >= n)
      throw std::invalid_argument("graph: vertex index out of range");
    if (u == v) throw std::invalid_argument("graph: self-loop rejected");
    keys[i] = key_of(u, v);
  }
  csr_from_keys(n, keys, off, nbr);
}

void generate_er(int32_t n, double p, uint64_t seed, std::vector<int64_t>& off,
                 std::vector<int32_t>& nbr) {  // graph.cpp:107-116
  if (n < 0) throw std::invalid_argument("er: negative n");
  if (p < 0.0 || p > 1.0) throw std::invalid_argument("er: p outside [0,1]");
  Xoshiro r = xoshiro_seed(derive_seed(seed, 0x45521ULL));
  std::vector<uint64_t> keys;
  const double expect = 0.5 * static_cast<double>(n) * (n - 1.0) * p;
  keys.reserve(static_cast<size_t>(expect * 1.05 + 16));
  for (int32_t u = 0; u < n; ++u)
    for (int32_t v = u + 1; v < n; ++v)
      if (u01_of(xoshiro_next(r)) < p) keys.push_back(key_of(u, v));
  csr_from_keys(n, keys, off, nbr);
}

// O(m) Erdos-Renyi G(n, p) by geometric skipping over the canonical
// (u < v) pair order (Batagelj & Brandes 2005).  NOT the reference's draw
// sequence (which needs n(n-1)/2 draws: ~49 h at n = 1e7, SURVEY.md section
// 6); a distinct generator for the large configs whose edge list is fed to
// both sides.  Stream: Rng(derive_seed(seed, 0xE5F)).
void generate_er_fast(int32_t n, double p, uint64_t seed, std::vector<int64_t>& off,
                      std::vector<int32_t>& nbr) {
  if (n < 0) throw std::invalid_argument("er: negative n");
  if (p < 0.0 || p > 1.0) throw std::invalid_argument("er: p outside [0,1]");
  std::vector<uint64_t> keys;
  if (p > 0.0 && n > 1) {
    Xoshiro r = xoshiro_seed(derive_seed(seed, 0xE5FULL));
    const double expect = 0.5 * static_cast<double>(n) * (n - 1.0) * p;
    keys.reserve(static_cast<size_t>(expect * 1.01 + 1024));
    const double lq = std::log1p(-p);
    int64_t u = 0, v = 0;  // current pair (u, v) with v > u; start before (0, 1)
    for (;;) {
      double skip;
      if (p >= 1.0) {
        skip = 0.0;
      } else {
        double x = u01_of(xoshiro_next(r));
        skip = std::floor(std::log1p(-x) / lq);
      }
      // advance (u, v) by skip + 1 pairs in row-major (u < v) order
      int64_t adv = static_cast<int64_t>(skip) + 1;
      while (u < n && v + adv >= n) {
        adv -= (n - 1 - v);
        ++u;
        v = u;
      }
      if (u >= n - 1) break;
      v += adv;
      keys.push_back(key_of(static_cast<int32_t>(u), static_cast<int32_t>(v)));
    }
  }
  csr_from_keys(n, keys, off, nbr);
}

void generate_ba(int32_t n, int32_t m_attach, uint64_t seed, std::vector<int64_t>& off,
                 std::vector<int32_t>& nbr) {  // graph.cpp:118-146
  if (m_attach < 1) throw std::invalid_argument("ba: m_attach must be >= 1");
  if (m_attach >= n) throw std::invalid_argument("ba: m_attach must be < n");
  Xoshiro r = xoshiro_seed(derive_seed(seed, 0xBAULL));
  std::vector<uint64_t> keys;
  std::vector<int32_t> endpoints;
  keys.reserve(static_cast<size_t>(m_attach) * n);
  endpoints.reserve(static_cast<size_t>(2) * m_attach * n);
  for (int32_t v = 1; v <= m_attach; ++v) {
    keys.push_back(key_of(0, v));
    endpoints.push_back(0);
    endpoints.push_back(v);
  }
  std::vector<int32_t> targets;
  for (int32_t v = m_attach + 1; v < n; ++v) {
    targets.clear();
    while (static_cast<int32_t>(targets.size()) < m_attach) {
      const int32_t t = endpoints[xoshiro_index(r, endpoints.size())];
      if (std::find(targets.begin(), targets.end(), t) == targets.end()) targets.push_back(t);
    }
    for (int32_t t : targets) {
      keys.push_back(key_of(t, v));
      endpoints.push_back(t);
      endpoints.push_back(v);
    }
  }
  csr_from_keys(n, keys, off, nbr);
}

void generate_sbm(int32_t n, int32_t k, double p_in, double p_out, uint64_t seed,
                  std::vector<int64_t>& off, std::vector<int32_t>& nbr) {  // graph.cpp:148-165
  if (k < 1) throw std::invalid_argument("sbm: k must be >= 1");
  if (p_in < 0.0 || p_in > 1.0 || p_out < 0.0 || p_out > 1.0)
    throw std::invalid_argument("sbm: probabilities outside [0,1]");
  if (p_in <= p_out) throw std::invalid_argument("sbm: requires p_in > p_out");
  Xoshiro r = xoshiro_seed(derive_seed(seed, 0x5B3ULL));
  std::vector<uint64_t> keys;
  for (int32_t u = 0; u < n; ++u) {
    const int bu = static_cast<int>((static_cast<int64_t>(u) * k) / n);
    for (int32_t v = u + 1; v < n; ++v) {
      const int bv = static_cast<int>((static_cast<int64_t>(v) * k) / n);
      if (u01_of(xoshiro_next(r)) < (bu == bv ? p_in : p_out)) keys.push_back(key_of(u, v));
    }
  }
  csr_from_keys(n, keys, off, nbr);
}

}  // namespace

extern "C" int mqo_graph_from_edges(int32_t n, int64_t num_edges, const int32_t* eu,
                                    const int32_t* ev, int32_t device, mqo_graph** out) {
  std::vector<int64_t> off;
  std::vector<int32_t> nbr;
  const int rc = guard([&] {
    if (num_edges < 0 || (num_edges > 0 && (!eu || !ev)))
      throw std::invalid_argument("mqo_graph_from_edges: bad edge arrays");
    build_from_edges(n, num_edges, eu, ev, off, nbr);
  });
  if (rc) return rc;
  return mqo_graph_upload(n, off.data(), nbr.data(), device, out);
}

extern "C" int mqo_generate(const mqo_gen_spec* spec, int32_t device, mqo_graph** out) {
  std::vector<int64_t> off;
  std::vector<int32_t> nbr;
  int32_t n = 0;
  const int rc = guard([&] {
    if (!spec) throw std::invalid_argument("mqo_generate: null spec");
    n = spec->n;
    switch (spec->kind) {
      case MQO_GEN_ER: generate_er(spec->n, spec->p, spec->seed, off, nbr); break;
      case MQO_GEN_BA: generate_ba(spec->n, spec->m_attach, spec->seed, off, nbr); break;
      case MQO_GEN_ER_FAST: generate_er_fast(spec->n, spec->p, spec->seed, off, nbr); break;
      case MQO_GEN_SBM:
        generate_sbm(spec->n, spec->k, spec->p_in, spec->p_out, spec->seed, off, nbr);
        break;
      default: throw std::invalid_argument("mqo_generate: unknown generator kind");
    }
  });
  if (rc) return rc;
  return mqo_graph_upload(n, off.data(), nbr.data(), device, out);
}

extern "C" int mqo_graph_csr(const mqo_graph* g, int64_t* offsets, int32_t* neighbors) {
  return guard([&] {
    if (!g) throw std::invalid_argument("mqo_graph_csr: null graph");
    if (offsets) std::memcpy(offsets, g->h_off.data(), sizeof(int64_t) * g->h_off.size());
    if (neighbors) std::memcpy(neighbors, g->h_nbr.data(), sizeof(int32_t) * g->h_nbr.size());
  });
}

// ---------------------------------------------------------------- graph I/O
// Binary CSR cache ("MQOCSR01", n, m, offsets[n+1], neighbours[2m]) next to
// the reference's canonical text format ("n m" then m lines "u v", u < v;
// graph_io.cpp:74-92): large instances (C5: 8e7 edges) load in seconds.
extern "C" int mqo_graph_save(const mqo_graph* g, const char* path, int32_t format) {
  return guard([&] {
    if (!g || !path) throw std::invalid_argument("mqo_graph_save: null argument");
    FILE* f = std::fopen(path, format == 0 ? "wb" : "w");
    if (!f) throw std::runtime_error(std::string("cannot open output file: ") + path);
    bool ok = true;
    if (format == 0) {
      const char magic[8] = {'M', 'Q', 'O', 'C', 'S', 'R', '0', '1'};
      const int64_t n = g->n, m = g->m;
      ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(&n, 8, 1, f) == 1 &&
           std::fwrite(&m, 8, 1, f) == 1 &&
           std::fwrite(g->h_off.data(), 8, g->h_off.size(), f) == g->h_off.size() &&
           std::fwrite(g->h_nbr.data(), 4, g->h_nbr.size(), f) == g->h_nbr.size();
    } else {  // write_canonical, graph_io.cpp:89-92
      ok = std::fprintf(f, "%d %lld\n", g->n, static_cast<long long>(g->m)) > 0;
      for (int32_t v = 0; ok && v < g->n; ++v)
        for (int64_t e = g->h_off[v]; ok && e < g->h_off[v + 1]; ++e)
          if (v < g->h_nbr[e]) ok = std::fprintf(f, "%d %d\n", v, g->h_nbr[e]) > 0;
    }
    if (std::fclose(f) != 0 || !ok) throw std::runtime_error(std::string("write failed: ") + path);
  });
}

extern "C" int mqo_graph_load(const char* path, int32_t device, mqo_graph** out) {
  std::vector<int64_t> off;
  std::vector<int32_t> nbr;
  int32_t n = 0;
  const int rc = guard([&] {
    if (!path || !out) throw std::invalid_argument("mqo_graph_load: null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open graph file: ") + path);
    char magic[8] = {0};
    const size_t got = std::fread(magic, 1, 8, f);
    if (got == 8 && std::memcmp(magic, "MQOCSR01", 8) == 0) {
      int64_t n64 = 0, m = 0;
      if (std::fread(&n64, 8, 1, f) != 1 || std::fread(&m, 8, 1, f) != 1 || n64 < 0 || m < 0 ||
          n64 > INT32_MAX) {
        std::fclose(f);
        throw std::invalid_argument("graph file: bad binary header");
      }
      n = static_cast<int32_t>(n64);
      off.resize(static_cast<size_t>(n) + 1);
      nbr.resize(static_cast<size_t>(2 * m));
      const bool ok = std::fread(off.data(), 8, off.size(), f) == off.size() &&
                      std::fread(nbr.data(), 4, nbr.size(), f) == nbr.size();
      std::fclose(f);
      if (!ok) throw std::invalid_argument("graph file: truncated binary CSR");
      return;
    }
    // read_canonical (graph_io.cpp:74-87)
    std::rewind(f);
    long long nn = 0, mm = 0;
    if (std::fscanf(f, "%lld %lld", &nn, &mm) != 2) {
      std::fclose(f);
      throw std::invalid_argument("line 1: missing 'n m' header");
    }
    std::vector<int32_t> eu(static_cast<size_t>(mm)), ev(static_cast<size_t>(mm));
    for (long long i = 0; i < mm; ++i) {
      long long u = 0, v = 0;
      if (std::fscanf(f, "%lld %lld", &u, &v) != 2) {
        std::fclose(f);
        throw std::invalid_argument("line " + std::to_string(i + 2) + ": truncated edge list");
      }
      eu[i] = static_cast<int32_t>(u);
      ev[i] = static_cast<int32_t>(v);
    }
    std::fclose(f);
    n = static_cast<int32_t>(nn);
    build_from_edges(n, mm, eu.data(), ev.data(), off, nbr);
  });
  if (rc) return rc;
  return mqo_graph_upload(n, off.data(), nbr.data(), device, out);
}
