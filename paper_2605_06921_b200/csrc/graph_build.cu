// graph_build.cu -- host-side graph construction behind the C ABI:
// Graph::from_edges (graph.cpp:8-42) and the seeded generators
// (graph.cpp:107-178).  Same algorithms and the same xoshiro draws as the
// reference, so a (spec, seed) pair yields the identical CSR; the result is
// uploaded to HBM by mqo_graph_upload.
#include <algorithm>
#include <climits>
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

// O(m) stochastic block model: the reference's pair loop (graph.cpp:148-165)
// draws one Bernoulli per pair, O(n^2).  Blocks are contiguous (vertex v in
// block v*k/n), so row u's pairs (u, v > u) split into one p_in run -- the
// rest of u's block -- and one p_out run -- every later block.  Geometric
// skipping (Batagelj & Brandes 2005) over the concatenation of all p_in runs,
// and separately over all p_out runs, makes every pair an independent
// Bernoulli(p_in or p_out) draw, the reference's distribution, in O(n + m)
// expected work.  Not the reference's draw sequence; streams
// Rng(derive_seed(seed, 0x5B31)) (p_in) and (seed, 0x5B30) (p_out).
struct SkipRun {  // geometric skipping over a sequence of pair runs
  Xoshiro r;
  double lq;
  bool all, none;
  int64_t left = -1;  // pairs to skip before the next edge (-1: draw)
  explicit SkipRun(uint64_t seed, double p)
      : r(xoshiro_seed(seed)), lq(p < 1.0 ? std::log1p(-p) : 0.0), all(p >= 1.0), none(p <= 0.0) {}
  // calls emit(v) for every edge among the `len` pairs (u, first + i)
  template <class F>
  void run(int64_t first, int64_t len, F emit) {
    if (none || len <= 0) return;
    int64_t i = 0;
    for (;;) {
      if (left < 0) {
        left = all ? 0 : static_cast<int64_t>(std::floor(std::log1p(-u01_of(xoshiro_next(r))) / lq));
      }
      if (i + left >= len) {  // the skip runs past this run: carry the rest over
        left -= len - i;
        return;
      }
      i += left;
      emit(first + i);
      ++i;
      left = -1;
    }
  }
};

void generate_sbm_fast(int32_t n, int32_t k, double p_in, double p_out, uint64_t seed,
                       std::vector<int64_t>& off, std::vector<int32_t>& nbr) {
  if (k < 1) throw std::invalid_argument("sbm: k must be >= 1");
  if (p_in < 0.0 || p_in > 1.0 || p_out < 0.0 || p_out > 1.0)
    throw std::invalid_argument("sbm: probabilities outside [0,1]");
  if (p_in <= p_out) throw std::invalid_argument("sbm: requires p_in > p_out");
  std::vector<uint64_t> keys;
  SkipRun in(derive_seed(seed, 0x5B31ULL), p_in), out(derive_seed(seed, 0x5B30ULL), p_out);
  for (int32_t u = 0; u + 1 < n; ++u) {
    const int64_t bu = (static_cast<int64_t>(u) * k) / n;
    // first vertex of the next block: smallest v with v*k/n > bu
    const int64_t hi = std::min<int64_t>(n, ((bu + 1) * n + k - 1) / k);
    in.run(u + 1, hi - (u + 1), [&](int64_t v) { keys.push_back(key_of(u, static_cast<int32_t>(v))); });
    out.run(hi, n - hi, [&](int64_t v) { keys.push_back(key_of(u, static_cast<int32_t>(v))); });
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
      case MQO_GEN_SBM_FAST:
        generate_sbm_fast(spec->n, spec->k, spec->p_in, spec->p_out, spec->seed, off, nbr);
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
    host_csr(g);
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
    host_csr(g);
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

// ------------------------------------------------------- text formats
// graph_io.cpp:18-87, re-stated over an in-memory buffer: istream `>>`
// semantics for the tokens (whitespace-separated, an integer read stops at
// its first non-digit), the reference's ParseError messages and line numbers.
namespace {

thread_local std::string g_load_warnings;

struct Cursor {
  const char* p;
  const char* end;
  static bool ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }
  void skip_ws() { while (p < end && ws(*p)) ++p; }
  // operator>>(int64_t&): skip whitespace, optional sign, >= 1 digit; overflow fails
  bool read_i64(int64_t& out) {
    skip_ws();
    const char* q = p;
    bool neg = false;
    if (q < end && (*q == '+' || *q == '-')) neg = *q++ == '-';
    if (q >= end || *q < '0' || *q > '9') return false;
    unsigned long long v = 0;
    const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
    for (; q < end && *q >= '0' && *q <= '9'; ++q) {
      const unsigned d = static_cast<unsigned>(*q - '0');
      if (v > (lim - d) / 10) return false;
      v = v * 10 + d;
    }
    p = q;
    out = neg ? static_cast<int64_t>(0ull - v) : static_cast<int64_t>(v);
    return true;
  }
  bool read_i32(int32_t& out) {  // operator>>(int&): out-of-range fails
    int64_t v = 0;
    if (!read_i64(v) || v < INT32_MIN || v > INT32_MAX) return false;
    out = static_cast<int32_t>(v);
    return true;
  }
  std::string read_token() {
    skip_ws();
    const char* q = p;
    while (p < end && !ws(*p)) ++p;
    return std::string(q, p);
  }
};

// read_canonical (graph_io.cpp:74-87)
void parse_canonical(const char* text, size_t len, int32_t& n, std::vector<int64_t>& off,
                     std::vector<int32_t>& nbr) {
  Cursor c{text, text + len};
  int64_t m = 0;
  if (!c.read_i32(n) || !c.read_i64(m)) throw ParseError(1, "missing 'n m' header");
  // edges.reserve(static_cast<size_t>(m)) (graph_io.cpp:79) throws for m < 0
  if (m < 0) throw std::length_error("vector::reserve");
  std::vector<int32_t> eu, ev;
  if (m > 0) {
    eu.reserve(static_cast<size_t>(std::min<int64_t>(m, int64_t(1) << 32)));
    ev.reserve(eu.capacity());
  }
  for (int64_t i = 0; i < m; ++i) {
    int64_t u = 0, v = 0;
    if (!c.read_i64(u) || !c.read_i64(v))
      throw ParseError(static_cast<int32_t>(i + 2), "truncated edge list");
    eu.push_back(static_cast<int32_t>(u));  // static_cast<Vertex>, as the reference
    ev.push_back(static_cast<int32_t>(v));
  }
  build_from_edges(n, static_cast<int64_t>(eu.size()), eu.data(), ev.data(), off, nbr);
}

// parse_dimacs (graph_io.cpp:18-66)
void parse_dimacs(const char* text, size_t len, int32_t& n, std::vector<int64_t>& off,
                  std::vector<int32_t>& nbr, int64_t& declared_m) {
  const char* p = text;
  const char* end = text + len;
  int32_t lineno = 0;
  bool have_header = false;
  n = 0;
  declared_m = 0;
  std::vector<int32_t> eu, ev;
  while (p < end) {
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    if (!eol) eol = end;
    ++lineno;
    Cursor c{p, eol};
    p = eol < end ? eol + 1 : end;
    const std::string tag = c.read_token();
    if (tag.empty()) continue;  // blank line
    if (tag == "c") continue;
    if (tag == "p") {
      if (have_header) throw ParseError(lineno, "duplicate 'p' line");
      const std::string fmt = c.read_token();
      int64_t dm = 0;
      if (fmt.empty() || !c.read_i32(n) || !c.read_i64(dm))
        throw ParseError(lineno, "malformed 'p' line, expected 'p edge <n> <m>'");
      if (n < 0 || dm < 0) throw ParseError(lineno, "negative n or m");
      declared_m = dm;
      have_header = true;
      continue;
    }
    if (tag == "e") {
      if (!have_header) throw ParseError(lineno, "edge before 'p edge <n> <m>' header");
      int64_t u = 0, v = 0;
      if (!c.read_i64(u) || !c.read_i64(v)) throw ParseError(lineno, "malformed 'e' line");
      if (u < 1 || u > n || v < 1 || v > n) throw ParseError(lineno, "vertex index outside [1, n]");
      if (u == v) throw ParseError(lineno, "self-loop");
      eu.push_back(static_cast<int32_t>(u - 1));
      ev.push_back(static_cast<int32_t>(v - 1));
      continue;
    }
    throw ParseError(lineno, "unrecognized line tag '" + tag + "'");
  }
  if (!have_header) throw ParseError(lineno, "missing 'p edge <n> <m>' header");
  build_from_edges(n, static_cast<int64_t>(eu.size()), eu.data(), ev.data(), off, nbr);
  const int64_t parsed = static_cast<int64_t>(nbr.size() / 2);
  if (parsed != declared_m)
    g_load_warnings = "declared m=" + std::to_string(declared_m) + " but parsed m=" +
                      std::to_string(parsed) + " after deduplication";
}

bool looks_dimacs(const char* text, size_t len) {  // graph_io.cpp:97-98: peek()
  return len > 0 && (text[0] == 'c' || text[0] == 'p');
}

}  // namespace

extern "C" int mqo_graph_parse(const char* text, int64_t len, int32_t format, int32_t device,
                               int64_t* declared_edges, mqo_graph** out) {
  std::vector<int64_t> off;
  std::vector<int32_t> nbr;
  int32_t n = 0;
  g_load_warnings.clear();
  const int rc = guard([&] {
    if ((!text && len > 0) || len < 0 || !out) throw std::invalid_argument("mqo_graph_parse: bad arguments");
    if (format < 0 || format > 2) throw std::invalid_argument("mqo_graph_parse: unknown format");
    const bool dimacs = format == 2 || (format == 0 && looks_dimacs(text, static_cast<size_t>(len)));
    int64_t dm = 0;
    if (dimacs)
      parse_dimacs(text, static_cast<size_t>(len), n, off, nbr, dm);
    else
      parse_canonical(text, static_cast<size_t>(len), n, off, nbr);
    if (declared_edges) *declared_edges = dimacs ? dm : static_cast<int64_t>(nbr.size() / 2);
  });
  if (rc) return rc;
  return mqo_graph_upload(n, off.data(), nbr.data(), device, out);
}

extern "C" int64_t mqo_graph_load_warnings(char* buf, int64_t cap) {
  const int64_t len = static_cast<int64_t>(g_load_warnings.size());
  if (buf && cap > 0) {
    const int64_t k = std::min(len, cap - 1);
    std::memcpy(buf, g_load_warnings.data(), static_cast<size_t>(k));
    buf[k] = 0;
  }
  return len;
}

extern "C" int mqo_graph_load(const char* path, int32_t device, mqo_graph** out) {
  std::vector<int64_t> off;
  std::vector<int32_t> nbr;
  std::string text;
  int32_t n = 0;
  bool is_text = false;
  g_load_warnings.clear();
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
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::rewind(f);
    text.resize(size > 0 ? static_cast<size_t>(size) : 0);
    const bool ok = text.empty() || std::fread(&text[0], 1, text.size(), f) == text.size();
    std::fclose(f);
    if (!ok) throw std::runtime_error(std::string("cannot read graph file: ") + path);
    is_text = true;
  });
  if (rc) return rc;
  if (is_text)
    return mqo_graph_parse(text.data(), static_cast<int64_t>(text.size()), 0, device, nullptr, out);
  return mqo_graph_upload(n, off.data(), nbr.data(), device, out);
}
