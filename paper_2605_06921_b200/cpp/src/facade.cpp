// facade.cpp -- the reference's C++ API (mqo/graph.hpp, objectives.hpp,
// pga.hpp, solver.hpp, localsearch.hpp, presets.hpp) implemented over the C
// ABI of include/mqo_gpu.h.  Reference callers (its CLI, tests, benchmarks)
// recompile against these headers and link libmqo_core_b200.so instead of
// mqo::core; every matrix action, trajectory, reset, harvest, local search
// and the solver engine run on the B200.  Errors come back as the
// reference's exception types with its messages.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <limits>
#include <stdexcept>
#include <string>

#include "mqo/graph.hpp"
#include "mqo/graph_io.hpp"
#include "mqo/localsearch.hpp"
#include "mqo/objectives.hpp"
#include "mqo/pga.hpp"
#include "mqo/presets.hpp"
#include "mqo/solver.hpp"
#include "mqo_gpu.h"

namespace mqo {

namespace {

int g_device = [] {
  const char* e = std::getenv("MQO_DEVICE");
  return e ? std::atoi(e) : 0;
}();

void check(int rc) {
  if (rc == MQO_OK) return;
  const std::string msg = mqo_last_error();
  if (rc == MQO_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == MQO_ERR_LOGIC) throw std::logic_error(msg);
  if (rc == MQO_ERR_PARSE) {  // the ABI message already reads "line N: ..."
    const int line = mqo_last_error_line();
    const std::string prefix = "line " + std::to_string(line) + ": ";
    throw ParseError(line, msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
  }
  throw std::runtime_error(msg);
}

int32_t kind_of(const ObjectiveSpec& s) { return static_cast<int32_t>(s.index()); }

double param_of(const ObjectiveSpec& s) {
  if (const auto* q = std::get_if<MisQubo>(&s)) return q->gamma;
  if (const auto* p = std::get_if<PerturbedLaplacian>(&s)) return p->lambda;
  if (const auto* b = std::get_if<PerturbedBias>(&s)) return b->lambda;
  return 0.0;
}

mqo_objective obj_of(const ObjectiveSpec& s) { return mqo_objective{kind_of(s), param_of(s)}; }

mqo_optimizer opt_of(const OptimizerConfig& c) {
  return mqo_optimizer{c.alpha, c.beta, c.max_iters, c.conv_tol, c.check_every};
}

// RAII chain batch on a graph's device.
struct Batch {
  mqo_batch* b = nullptr;
  int chains = 0;
  Batch(const Graph& g, int chains_) : chains(chains_) {
    if (!g.handle()) throw std::invalid_argument("graph: not resident on a device");
    check(mqo_batch_create(g.handle(), chains_, &b));
  }
  ~Batch() { mqo_batch_free(b); }
  Batch(const Batch&) = delete;
  Batch& operator=(const Batch&) = delete;
};

// MQO_DEVICES: comma-separated device ids for the multi-GPU engine (empty
// or one id: the single-GPU path on the graph's device).
std::vector<int32_t> devices_from_env() {
  std::vector<int32_t> out;
  const char* e = std::getenv("MQO_DEVICES");
  if (!e) return out;
  std::string s(e), tok;
  for (size_t i = 0; i <= s.size(); ++i) {
    if (i == s.size() || s[i] == ',') {
      if (!tok.empty()) out.push_back(static_cast<int32_t>(std::stoi(tok)));
      tok.clear();
    } else if (s[i] != ' ') {
      tok += s[i];
    }
  }
  return out;
}

int64_t words(Vertex n) { return (static_cast<int64_t>(n) + 63) / 64; }

std::vector<uint64_t> pack(const std::vector<uint8_t>& bytes) {
  std::vector<uint64_t> p(words(static_cast<Vertex>(bytes.size())), 0);
  for (size_t v = 0; v < bytes.size(); ++v)
    if (bytes[v]) p[v >> 6] |= 1ull << (63 - (v & 63));
  return p;
}

std::vector<uint8_t> unpack(const uint64_t* p, Vertex n) {
  std::vector<uint8_t> out(n);
  for (Vertex v = 0; v < n; ++v) out[v] = (p[v >> 6] >> (63 - (v & 63))) & 1;
  return out;
}

std::vector<uint8_t> indicator(Vertex n, std::span<const Vertex> members) {
  std::vector<uint8_t> in(n, 0);
  for (Vertex v : members) in[v] = 1;
  return in;
}

std::vector<Vertex> members_of(const std::vector<uint8_t>& ind) {
  std::vector<Vertex> m;
  for (size_t v = 0; v < ind.size(); ++v)
    if (ind[v]) m.push_back(static_cast<Vertex>(v));
  return m;
}

// Gradient of one state through the fused kernel (mqo_gradient).
std::vector<double> device_gradient(int32_t kind, double param, const Graph& g,
                                    std::span<const double> x) {
  std::vector<double> out(g.n());
  if (g.n() == 0) return out;
  Batch b(g, 1);
  check(mqo_batch_set_x(b.b, x.data()));
  const mqo_objective o{kind, param};
  check(mqo_gradient(b.b, &o, out.data()));
  return out;
}

double mono_secs(std::chrono::steady_clock::time_point t) {
  // steady_clock is CLOCK_MONOTONIC on Linux, the clock the ABI polls.
  return std::chrono::duration<double>(t.time_since_epoch()).count();
}

}  // namespace

void set_device(int device) { g_device = device; }
int current_device() { return g_device; }

// ------------------------------------------------------------------ Graph
Graph Graph::adopt(mqo_graph* h) {
  Graph g;
  g.dev_ = std::shared_ptr<mqo_graph>(h, [](mqo_graph* p) { mqo_graph_free(p); });
  int32_t n = 0, dmax = 0;
  int64_t m = 0;
  check(mqo_graph_info(h, &n, &m, &dmax));
  g.n_ = n;
  g.m_ = m;
  g.max_degree_ = dmax;
  g.offsets_.assign(static_cast<size_t>(n) + 1, 0);
  g.neighbors_.assign(static_cast<size_t>(2 * m), 0);
  check(mqo_graph_csr(h, g.offsets_.data(), g.neighbors_.data()));
  return g;
}

Graph Graph::from_edges(Vertex n, std::vector<std::pair<Vertex, Vertex>> edges) {
  std::vector<int32_t> eu(edges.size()), ev(edges.size());
  for (size_t i = 0; i < edges.size(); ++i) {
    eu[i] = edges[i].first;
    ev[i] = edges[i].second;
  }
  mqo_graph* h = nullptr;
  check(mqo_graph_from_edges(n, static_cast<int64_t>(edges.size()), eu.data(), ev.data(),
                             g_device, &h));
  return adopt(h);
}

bool Graph::has_edge(Vertex u, Vertex v) const {
  const auto nb = neighbors(u);
  return std::binary_search(nb.begin(), nb.end(), v);
}

void Graph::adjacency_apply(std::span<const double> x, std::span<double> y) const {
  if (static_cast<Vertex>(x.size()) != n_ || static_cast<Vertex>(y.size()) != n_)
    throw std::invalid_argument("adjacency_apply: dimension mismatch");
  // grad f_A = -2 Ax; the scaling by -0.5 is exact in binary floating point
  const auto gr = device_gradient(MQO_ADJACENCY, 0.0, *this, x);
  for (Vertex v = 0; v < n_; ++v) y[v] = gr[v] * -0.5;
}

std::vector<double> Graph::adjacency_apply(std::span<const double> x) const {
  std::vector<double> y(n_);
  adjacency_apply(x, y);
  return y;
}

void Graph::laplacian_apply(std::span<const double> x, std::span<double> y) const {
  if (static_cast<Vertex>(x.size()) != n_ || static_cast<Vertex>(y.size()) != n_)
    throw std::invalid_argument("laplacian_apply: dimension mismatch");
  const auto gr = device_gradient(MQO_LAPLACIAN, 0.0, *this, x);  // (1/2) Lx, exact
  for (Vertex v = 0; v < n_; ++v) y[v] = gr[v] * 2.0;
}

std::vector<double> Graph::laplacian_apply(std::span<const double> x) const {
  std::vector<double> y(n_);
  laplacian_apply(x, y);
  return y;
}

std::vector<std::pair<Vertex, Vertex>> Graph::edges() const {
  std::vector<std::pair<Vertex, Vertex>> out;
  out.reserve(static_cast<size_t>(m_));
  for (Vertex v = 0; v < n_; ++v)
    for (Vertex u : neighbors(v))
      if (v < u) out.emplace_back(v, u);
  return out;
}

Graph generate(const GraphGenSpec& spec) {
  mqo_gen_spec s{};
  s.seed = spec.seed;
  if (const auto* er = std::get_if<ErSpec>(&spec.kind)) {
    s.kind = MQO_GEN_ER;
    s.n = er->n;
    s.p = er->p;
  } else if (const auto* ba = std::get_if<BaSpec>(&spec.kind)) {
    s.kind = MQO_GEN_BA;
    s.n = ba->n;
    s.m_attach = ba->m_attach;
  } else {
    const auto& sb = std::get<SbmSpec>(spec.kind);
    s.kind = MQO_GEN_SBM;
    s.n = sb.n;
    s.k = sb.k;
    s.p_in = sb.p_in;
    s.p_out = sb.p_out;
  }
  mqo_graph* h = nullptr;
  check(mqo_generate(&s, g_device, &h));
  return Graph::adopt(h);
}

StripResult strip_isolated(const Graph& g) {  // graph.cpp:180-198, on the device
  const size_t n = static_cast<size_t>(g.n());
  std::vector<int32_t> c2o(std::max<size_t>(n, 1)), o2c(std::max<size_t>(n, 1)),
      rem(std::max<size_t>(n, 1));
  int32_t nc = 0, nr = 0;
  mqo_graph* core = nullptr;
  check(mqo_graph_strip_isolated(g.handle(), &core, c2o.data(), o2c.data(), rem.data(), &nc, &nr));
  StripResult r;
  r.core = Graph::adopt(core);
  r.core_to_orig.assign(c2o.begin(), c2o.begin() + nc);
  r.orig_to_core.assign(o2c.begin(), o2c.begin() + static_cast<std::ptrdiff_t>(n));
  r.removed.assign(rem.begin(), rem.begin() + nr);
  return r;
}

std::vector<std::vector<Vertex>> connected_components(const Graph& g) {  // graph.cpp:200-224
  std::vector<int32_t> comp(std::max<size_t>(static_cast<size_t>(g.n()), 1));
  int32_t count = 0;
  check(mqo_graph_components(g.handle(), comp.data(), &count));
  std::vector<std::vector<Vertex>> comps(static_cast<size_t>(count));
  for (Vertex v = 0; v < g.n(); ++v) comps[static_cast<size_t>(comp[v])].push_back(v);
  return comps;
}

// ------------------------------------------------------------- objectives
Problem problem_of(const ObjectiveSpec& spec) {
  return std::holds_alternative<MisQubo>(spec) ? Problem::Mis : Problem::MaxCut;
}

BoxDomain domain_of(const ObjectiveSpec& spec) {
  return problem_of(spec) == Problem::Mis ? BoxDomain::Unit : BoxDomain::Symmetric;
}

const char* objective_name(const ObjectiveSpec& spec) {
  static const char* names[] = {"mis-qubo", "laplacian", "perturbed-laplacian", "adjacency",
                                "perturbed-bias"};
  return names[spec.index()];
}

void validate(const ObjectiveSpec& spec) {
  if (const auto* q = std::get_if<MisQubo>(&spec)) {
    if (!(q->gamma > 1.0)) throw std::invalid_argument("mis-qubo: gamma must be > 1");
  } else if (const auto* p = std::get_if<PerturbedLaplacian>(&spec)) {
    if (!(p->lambda > 0.0)) throw std::invalid_argument("perturbed-laplacian: lambda must be > 0");
  } else if (const auto* b = std::get_if<PerturbedBias>(&spec)) {
    if (!(b->lambda > 0.0 && b->lambda < 2.0))
      throw std::invalid_argument("perturbed-bias: lambda must be in (0, 2)");
  }
}

namespace {
void check_state(const ObjectiveSpec& spec, const Graph& g, const RelaxedState& s) {
  if (static_cast<Vertex>(s.x.size()) != g.n())
    throw std::invalid_argument("objective: state dimension mismatch");
  if (s.domain != domain_of(spec))
    throw std::invalid_argument("objective: state domain does not match objective");
}
}  // namespace

double value(const ObjectiveSpec& spec, const Graph& g, const RelaxedState& state) {
  // Test-only in the reference (never called by the solver); the quadratic
  // forms use the device SpMV, the O(n) reductions run in index order.
  check_state(spec, g, state);
  const auto& x = state.x;
  auto sum = [&] {
    double a = 0.0;
    for (double t : x) a += t;
    return a;
  };
  auto dot = [&](const std::vector<double>& y) {
    double a = 0.0;
    for (size_t i = 0; i < x.size(); ++i) a += x[i] * y[i];
    return a;
  };
  auto quad_lap = [&] {
    double acc = 0.0;
    for (Vertex v = 0; v < g.n(); ++v)
      for (Vertex u : g.neighbors(v))
        if (u > v) {
          const double d = x[v] - x[u];
          acc += d * d;
        }
    return acc;
  };
  if (const auto* q = std::get_if<MisQubo>(&spec))
    return sum() - 0.5 * q->gamma * dot(g.adjacency_apply(x));
  if (std::holds_alternative<Laplacian>(spec)) return 0.25 * quad_lap();
  if (const auto* p = std::get_if<PerturbedLaplacian>(&spec)) {
    double xx = 0.0;
    for (double t : x) xx += t * t;
    return quad_lap() + p->lambda * xx;
  }
  if (std::holds_alternative<Adjacency>(spec)) return -dot(g.adjacency_apply(x));
  const auto& b = std::get<PerturbedBias>(spec);
  return -b.lambda * sum() - dot(g.adjacency_apply(x));
}

void gradient(const ObjectiveSpec& spec, const Graph& g, const RelaxedState& state,
              std::span<double> out) {
  check_state(spec, g, state);
  if (out.size() != state.x.size()) throw std::invalid_argument("gradient: output dimension mismatch");
  const auto gr = device_gradient(kind_of(spec), param_of(spec), g, state.x);
  std::copy(gr.begin(), gr.end(), out.begin());
}

std::vector<double> gradient(const ObjectiveSpec& spec, const Graph& g, const RelaxedState& state) {
  std::vector<double> out(state.x.size());
  gradient(spec, g, state, out);
  return out;
}

Solution extract_solution(Problem problem, const Graph& g, const RelaxedState& state) {
  if (static_cast<Vertex>(state.x.size()) != g.n())
    throw std::invalid_argument("extract_solution: dimension mismatch");
  Solution sol;
  const int32_t p = problem == Problem::Mis ? MQO_PROBLEM_MIS : MQO_PROBLEM_MAXCUT;
  std::vector<uint64_t> packed(std::max<int64_t>(1, words(g.n())));
  if (g.n() > 0) {
    Batch b(g, 1);
    check(mqo_batch_set_x(b.b, state.x.data()));
    check(mqo_extract(b.b, p, &sol.score, nullptr, packed.data()));
  }
  const auto bytes = unpack(packed.data(), g.n());
  if (problem == Problem::Mis)
    sol.body = IndependentSet{members_of(bytes)};
  else
    sol.body = CutPartition{bytes};
  return sol;
}

int64_t cut_value(const Graph& g, std::span<const uint8_t> side) {
  if (static_cast<Vertex>(side.size()) != g.n())
    throw std::invalid_argument("cut_value: dimension mismatch");
  if (g.n() == 0) return 0;
  std::vector<double> x(g.n());
  for (Vertex v = 0; v < g.n(); ++v) x[v] = side[v] ? 1.0 : -1.0;
  Batch b(g, 1);
  check(mqo_batch_set_x(b.b, x.data()));
  int64_t score = 0;
  check(mqo_extract(b.b, MQO_PROBLEM_MAXCUT, &score, nullptr, nullptr));
  return score;
}

bool is_independent(const Graph& g, std::span<const Vertex> members) {
  if (g.n() == 0) return true;
  std::vector<double> x(g.n(), 0.0);
  for (Vertex v : members) x[v] = 1.0;
  Batch b(g, 1);
  check(mqo_batch_set_x(b.b, x.data()));
  int32_t ind = 0;
  check(mqo_extract(b.b, MQO_PROBLEM_MIS, nullptr, &ind, nullptr));
  return ind != 0;
}

int64_t score_solution(const Graph& g, const Solution& solution) {
  if (const auto* is = std::get_if<IndependentSet>(&solution.body))
    return static_cast<int64_t>(is->members.size());
  return cut_value(g, std::get<CutPartition>(solution.body).side);
}

// -------------------------------------------------------------------- PGA
void validate(const OptimizerConfig& c) {
  if (!(c.alpha > 0.0)) throw std::invalid_argument("optimizer: alpha must be > 0");
  if (c.beta < 0.0 || c.beta >= 1.0) throw std::invalid_argument("optimizer: beta must be in [0, 1)");
  if (c.max_iters < 1) throw std::invalid_argument("optimizer: max_iters must be >= 1");
  if (c.conv_tol < 0.0) throw std::invalid_argument("optimizer: conv_tol must be >= 0");
  if (c.check_every < 1) throw std::invalid_argument("optimizer: check_every must be >= 1");
}

const char* stop_reason_name(StopReason r) {
  switch (r) {
    case StopReason::Converged: return "converged";
    case StopReason::CheckerAccepted: return "checker-accepted";
    case StopReason::IterCap: return "iter-cap";
  }
  return "?";
}

void project(RelaxedState& state) {
  // elementwise clamp; a trivial host loop (pga.cpp:47-49) -- the device
  // path projects inside run_trajectory
  const double lo = state.domain == BoxDomain::Unit ? 0.0 : -1.0;
  for (double& t : state.x) {
    const double a = lo < t ? t : lo;
    t = a < 1.0 ? a : 1.0;
  }
}

void step(const ObjectiveSpec& spec, const Graph& g, RelaxedState& state,
          std::vector<double>& velocity, const OptimizerConfig& cfg) {
  velocity.resize(state.x.size(), 0.0);
  check_state(spec, g, state);
  if (g.n() == 0) return;
  Batch b(g, 1);
  check(mqo_batch_set_x(b.b, state.x.data()));
  check(mqo_batch_set_v(b.b, velocity.data()));
  const mqo_objective o = obj_of(spec);
  const mqo_optimizer op = opt_of(cfg);
  check(mqo_step(b.b, &o, &op));
  check(mqo_batch_get_x(b.b, state.x.data()));
  check(mqo_batch_get_v(b.b, velocity.data()));
}

std::vector<TrajectoryOutcome> run_trajectories(const ObjectiveSpec& spec, const Graph& g,
                                                std::vector<RelaxedState> inits,
                                                const OptimizerConfig& cfg,
                                                std::optional<Deadline> deadline) {
  validate(cfg);
  const int B = static_cast<int>(inits.size());
  std::vector<TrajectoryOutcome> out(B);
  if (B == 0) return out;
  const Vertex n = g.n();
  std::vector<double> x(static_cast<size_t>(B) * n);
  for (int c = 0; c < B; ++c) {
    if (static_cast<Vertex>(inits[c].x.size()) != n)
      throw std::invalid_argument("objective: state dimension mismatch");
    std::copy(inits[c].x.begin(), inits[c].x.end(), x.begin() + static_cast<size_t>(c) * n);
  }
  std::vector<int32_t> it(B), rs(B);
  if (n > 0) {
    Batch b(g, B);
    check(mqo_batch_set_x(b.b, x.data()));
    const mqo_objective o = obj_of(spec);
    const mqo_optimizer op = opt_of(cfg);
    check(mqo_run_trajectories(b.b, &o, &op, deadline ? mono_secs(*deadline) : -1.0, it.data(),
                               rs.data()));
    check(mqo_batch_get_x(b.b, x.data()));
  }
  for (int c = 0; c < B; ++c) {
    out[c].state.domain = inits[c].domain;
    out[c].state.x.assign(x.begin() + static_cast<size_t>(c) * n,
                          x.begin() + static_cast<size_t>(c + 1) * n);
    out[c].iterations = it[c];
    out[c].reason = static_cast<StopReason>(rs[c]);
  }
  return out;
}

TrajectoryOutcome run_trajectory(const ObjectiveSpec& spec, const Graph& g, RelaxedState init,
                                 const OptimizerConfig& cfg, std::optional<Deadline> deadline) {
  std::vector<RelaxedState> v;
  v.push_back(std::move(init));
  return std::move(run_trajectories(spec, g, std::move(v), cfg, deadline)[0]);
}

bool mis_fixed_point_check(const Graph& g, std::span<const double> x, double gamma, double alpha) {
  if (static_cast<Vertex>(x.size()) != g.n())
    throw std::invalid_argument("mis_fixed_point_check: dimension mismatch");
  if (g.n() == 0) return true;
  Batch b(g, 1);
  check(mqo_batch_set_x(b.b, x.data()));
  int32_t fixed = 0;
  check(mqo_mis_fixed_point_check(b.b, gamma, alpha, &fixed));
  return fixed != 0;
}

bool maxcut_binary_fixed_point_check(const ObjectiveSpec& spec, const Graph& g,
                                     std::span<const double> x) {
  if (problem_of(spec) != Problem::MaxCut)
    throw std::invalid_argument("maxcut_binary_fixed_point_check: MaxCut objectives only");
  if (static_cast<Vertex>(x.size()) != g.n())
    throw std::invalid_argument("maxcut_binary_fixed_point_check: dimension mismatch");
  for (double t : x)
    if (t != 1.0 && t != -1.0)
      throw std::invalid_argument("maxcut_binary_fixed_point_check: state not in {-1,1}^n");
  const auto gr = device_gradient(kind_of(spec), param_of(spec), g, x);
  for (Vertex v = 0; v < g.n(); ++v)
    if (x[v] * gr[v] < 0.0) return false;
  return true;
}

// ----------------------------------------------------------------- solver
void validate(const SolverConfig& c) {
  validate(c.objective);
  validate(c.optimizer);
  if (c.reset_fraction < 0.0 || c.reset_fraction >= 1.0)
    throw std::invalid_argument("solver: reset_fraction must be in [0, 1)");
  if (c.reset_rounds < 0) throw std::invalid_argument("solver: reset_rounds must be >= 0");
  if (c.init_noise < 0.0) throw std::invalid_argument("solver: init_noise must be >= 0");
  if (!(c.time_budget_secs > 0.0)) throw std::invalid_argument("solver: time_budget_secs must be > 0");
  if (c.pool.batch < 1 || c.pool.keep < 1)
    throw std::invalid_argument("solver: pool batch and keep must be >= 1");
  if (c.max_outer_loops && *c.max_outer_loops < 1)
    throw std::invalid_argument("solver: max_outer_loops must be >= 1");
}

RelaxedState init_state(Problem problem, const Graph& g, double sigma, Rng& rng) {
  RelaxedState s;
  s.domain = problem == Problem::Mis ? BoxDomain::Unit : BoxDomain::Symmetric;
  s.x.resize(g.n());
  const Rng::State st = rng.state();
  mqo_rng_state r{{st.s[0], st.s[1], st.s[2], st.s[3]}, st.spare, st.has_spare ? 1 : 0, 0};
  const int32_t pr = problem == Problem::Mis ? MQO_PROBLEM_MIS : MQO_PROBLEM_MAXCUT;
  if (g.n() == 0 || g.max_degree() < 1) {
    // the reference's argument errors (solver.cpp:31-33), no draws
    check(mqo_init_state_host(g.handle(), pr, sigma, &r, s.x.data()));
  } else {  // K3 on the device: one chain, bit-identical to Rng::normal
    Batch b(g, 1);
    check(mqo_batch_set_streams(b.b, &r));
    check(mqo_init_states(b.b, pr, sigma));
    check(mqo_batch_get_x(b.b, s.x.data()));
    check(mqo_batch_get_streams(b.b, &r));
  }
  rng.set_state({{r.s[0], r.s[1], r.s[2], r.s[3]}, r.spare, r.has_spare != 0});
  return s;
}

std::vector<Vertex> global_reset(RelaxedState& state, double rho, Rng& rng) {
  if (rho < 0.0 || rho >= 1.0) throw std::invalid_argument("global_reset: rho must be in [0, 1)");
  const auto n = static_cast<Vertex>(state.x.size());
  std::vector<Vertex> chosen;
  if (n == 0) return chosen;
  // the draws need no graph: a one-edge placeholder graph of n vertices
  const Graph g = n >= 2 ? Graph::from_edges(n, {{0, 1}}) : Graph::from_edges(n, {});
  Batch b(g, 1);
  std::vector<double> ones(n, 1.0);
  check(mqo_batch_set_x(b.b, ones.data()));
  const Rng::State st = rng.state();
  mqo_rng_state r{{st.s[0], st.s[1], st.s[2], st.s[3]}, st.spare, st.has_spare ? 1 : 0, 0};
  check(mqo_batch_set_streams(b.b, &r));
  check(mqo_global_reset(b.b, rho));
  check(mqo_batch_get_streams(b.b, &r));
  check(mqo_batch_get_x(b.b, ones.data()));
  rng.set_state({{r.s[0], r.s[1], r.s[2], r.s[3]}, r.spare, r.has_spare != 0});
  for (Vertex v = 0; v < n; ++v)
    if (ones[v] == 0.0) {
      chosen.push_back(v);
      state.x[v] = 0.0;
    }
  return chosen;
}

namespace {

RunReport run_engine(const Graph& g, const SolverConfig& cfg) {
  validate(cfg);
  mqo_solver_config c{};
  c.objective = kind_of(cfg.objective);
  c.param = param_of(cfg.objective);
  c.alpha = cfg.optimizer.alpha;
  c.beta = cfg.optimizer.beta;
  c.max_iters = cfg.optimizer.max_iters;
  c.conv_tol = cfg.optimizer.conv_tol;
  c.check_every = cfg.optimizer.check_every;
  c.reset_fraction = cfg.reset_fraction;
  c.reset_rounds = cfg.reset_rounds;
  c.init_noise = cfg.init_noise;
  c.time_budget_secs = cfg.time_budget_secs;
  c.seed = cfg.seed;
  c.local_search = cfg.local_search ? 1 : 0;
  c.pool_batch = cfg.pool.batch;
  c.pool_keep = cfg.pool.keep;
  c.has_init_constant = cfg.init_constant.has_value();
  c.init_constant = cfg.init_constant.value_or(0.0);
  c.has_stop_at_score = cfg.stop_at_score.has_value();
  c.stop_at_score = cfg.stop_at_score.value_or(0);
  c.has_max_outer_loops = cfg.max_outer_loops.has_value();
  c.max_outer_loops = cfg.max_outer_loops.value_or(0);
  c.init_mode = cfg.init_on_device ? MQO_INIT_DEVICE : MQO_INIT_EXACT;
  if (g.n() == 0) throw std::invalid_argument("solver: empty graph");
  mqo_run_report r{};
  std::vector<uint8_t> body(g.n());
  // MQO_DEVICES="0,1,...,7": shard the B chains over those GPUs of this
  // process (mqo_solve_devices, NCCL over NVLink); the report is the same
  // as the single-GPU run (Mode P).
  std::vector<int32_t> devs = devices_from_env();
  if (static_cast<int>(devs.size()) > c.pool_batch) devs.resize(c.pool_batch);  // >= 1 chain per rank
  if (devs.size() > 1)
    check(mqo_solve_devices(g.handle(), &c, devs.data(), static_cast<int32_t>(devs.size()),
                            MQO_SOLVE_POOLED, &r, body.data(), nullptr));
  else
    check(mqo_solve_pooled(g.handle(), &c, nullptr, &r, body.data()));
  RunReport rep;
  rep.config = cfg;
  rep.found_solution = r.found_solution != 0;
  rep.best.score = r.score;
  if (problem_of(cfg.objective) == Problem::Mis)
    rep.best.body = IndependentSet{members_of(body)};
  else
    rep.best.body = CutPartition{body};
  rep.phases = PhaseGains{r.after_gradient, r.after_reset_loop, r.after_local_search};
  rep.outer_loops = r.outer_loops;
  rep.trajectories = r.trajectories;
  rep.resets_accepted = r.resets_accepted;
  rep.resets_rejected = r.resets_rejected;
  rep.total_iterations = r.total_iterations;
  rep.last_trajectory_stop = static_cast<StopReason>(r.last_trajectory_stop);
  rep.elapsed_secs = r.elapsed_secs;
  if (r.warnings & MQO_WARN_EDGELESS)
    rep.warnings.push_back("graph has no edges; returning the trivial solution");
  if (r.warnings & MQO_WARN_RESET_NOOP)
    rep.warnings.push_back("floor(rho * n) = 0: global resets are no-ops");
  if (r.warnings & MQO_WARN_NO_SOLUTION)
    rep.warnings.push_back("budget exhausted before the first trajectory finished");
  return rep;
}

}  // namespace

RunReport solve_mis(const Graph& g, const SolverConfig& cfg) {
  if (problem_of(cfg.objective) != Problem::Mis)
    throw std::invalid_argument("solve_mis: objective must be the MIS QUBO");
  if (cfg.pool.batch != 1 || cfg.pool.keep != 1)
    throw std::invalid_argument("solve_mis: sequential solver requires batch = keep = 1");
  return run_engine(g, cfg);
}

RunReport solve_maxcut(const Graph& g, const SolverConfig& cfg) {
  if (problem_of(cfg.objective) != Problem::MaxCut)
    throw std::invalid_argument("solve_maxcut: objective must be a MaxCut formulation");
  if (cfg.pool.batch != 1 || cfg.pool.keep != 1)
    throw std::invalid_argument("solve_maxcut: sequential solver requires batch = keep = 1");
  return run_engine(g, cfg);
}

RunReport solve_pooled(const Graph& g, const SolverConfig& cfg) { return run_engine(g, cfg); }

// ---------------------------------------------------------- local search
namespace {
std::vector<int32_t> device_table(const Graph& g, int kind, const std::vector<uint8_t>& bytes) {
  std::vector<int32_t> out(g.n(), 0);
  if (g.n() == 0) return out;
  Batch b(g, 1);
  const auto p = pack(bytes);
  check(mqo_build_tables(b.b, kind, 1, p.data(), out.data()));
  return out;
}

int64_t device_ls(const Graph& g, int op, std::vector<uint8_t>& bytes) {
  if (g.n() == 0) return op == MQO_LS_ONE_TWO_SWAP ? 0 : 0;
  Batch b(g, 1);
  auto p = pack(bytes);
  int64_t out = 0;
  check(mqo_local_search(b.b, op, 1, p.data(), &out));
  bytes = unpack(p.data(), g.n());
  return out;
}
}  // namespace

TightnessTable build_tightness(const Graph& g, std::span<const Vertex> members) {
  return TightnessTable{device_table(g, 1, indicator(g.n(), members))};
}

GainTable build_gain_table(const Graph& g, std::span<const uint8_t> side) {
  const auto t = device_table(g, 0, std::vector<uint8_t>(side.begin(), side.end()));
  return GainTable{std::vector<int64_t>(t.begin(), t.end())};
}

void apply_flip(const Graph& g, std::vector<uint8_t>& side, GainTable& gains, Vertex v) {
  // O(d(v)) bookkeeping on caller-owned host tables (localsearch.cpp:28-33)
  side[v] ^= 1;
  gains.delta[v] = -gains.delta[v];
  for (Vertex u : g.neighbors(v)) gains.delta[u] += side[u] == side[v] ? 2 : -2;
}

std::vector<Vertex> greedy_maximalize(const Graph& g, std::vector<Vertex> members) {
  if (!is_independent(g, members))
    throw std::invalid_argument("greedy_maximalize: input not independent");
  if (g.n() == 0) return members;
  std::vector<double> x(g.n(), 0.0);
  for (Vertex v : members) x[v] = 1.0;
  Batch b(g, 1);
  check(mqo_batch_set_x(b.b, x.data()));
  std::vector<uint64_t> packed(words(g.n()));
  int32_t valid = 0;
  int64_t score = 0;
  check(mqo_harvest(b.b, MQO_PROBLEM_MIS, &score, &valid, packed.data()));
  return members_of(unpack(packed.data(), g.n()));
}

std::vector<Vertex> one_two_swap(const Graph& g, std::vector<Vertex> members) {
  auto ind = indicator(g.n(), members);
  device_ls(g, MQO_LS_ONE_TWO_SWAP, ind);
  return members_of(ind);
}

int64_t one_flip_pass(const Graph& g, std::vector<uint8_t>& side) {
  if (static_cast<Vertex>(side.size()) != g.n())
    throw std::invalid_argument("one_flip_pass: dimension mismatch");
  return device_ls(g, MQO_LS_ONE_FLIP, side);
}

int64_t two_flip_pass(const Graph& g, std::vector<uint8_t>& side) {
  if (static_cast<Vertex>(side.size()) != g.n())
    throw std::invalid_argument("two_flip_pass: dimension mismatch");
  return device_ls(g, MQO_LS_TWO_FLIP, side);
}

int64_t one_two_flip(const Graph& g, std::vector<uint8_t>& side) {
  return device_ls(g, MQO_LS_ONE_TWO_FLIP, side);
}

// ---------------------------------------------------------------- presets
Preset preset_for(Problem problem, Vertex n, double mean_degree) {
  // Appendix-G rows (presets.cpp:17-38), nearest in (log n, log d) space.
  struct Row {
    double n, d;
    Preset p;
  };
  static const Row mis[] = {{1000, 100, {0.80, 0.30, 0.70, 60}},   {1000, 300, {0.80, 0.45, 0.70, 60}},
                            {1000, 500, {0.80, 0.45, 0.60, 60}},   {3000, 100, {0.80, 0.30, 0.60, 60}},
                            {3000, 300, {0.80, 0.45, 0.60, 60}},   {3000, 1000, {0.80, 0.45, 0.50, 60}},
                            {10000, 5000, {0.80, 0.75, 0.50, 60}}, {20000, 10000, {0.80, 0.75, 0.50, 60}},
                            {30000, 15000, {0.80, 0.75, 0.50, 60}}};
  static const Row cut[] = {{100, 50, {0.0025, 0.90, 0.80, 90}},    {1000, 100, {0.0025, 0.80, 0.80, 90}},
                            {1000, 500, {0.0025, 0.80, 0.80, 90}},  {1000, 800, {0.0025, 0.80, 0.80, 90}},
                            {30000, 15000, {5e-5, 0.80, 0.80, 90}}, {30000, 24000, {5e-5, 0.80, 0.80, 90}},
                            {40000, 20000, {5e-5, 0.80, 0.80, 90}}, {40000, 32000, {5e-5, 0.80, 0.80, 90}}};
  const Row* rows = problem == Problem::Mis ? mis : cut;
  const int count = problem == Problem::Mis ? 9 : 8;
  const double ln = std::log(std::max(1.0, static_cast<double>(n)));
  const double ld = std::log(std::max(1.0, mean_degree));
  double best = std::numeric_limits<double>::infinity();
  Preset out = rows[0].p;
  for (int i = 0; i < count; ++i) {
    const double dn = ln - std::log(rows[i].n), dd = ld - std::log(rows[i].d);
    if (dn * dn + dd * dd < best) {
      best = dn * dn + dd * dd;
      out = rows[i].p;
    }
  }
  return out;
}

// --------------------------------------------------------------- graph_io
namespace {

std::vector<std::string> load_warnings() {
  std::vector<std::string> out;
  const int64_t k = mqo_graph_load_warnings(nullptr, 0);
  if (k <= 0) return out;
  std::string buf(static_cast<size_t>(k) + 1, '\0');
  mqo_graph_load_warnings(buf.data(), k + 1);
  buf.resize(static_cast<size_t>(k));
  std::istringstream in(buf);
  for (std::string w; std::getline(in, w);) out.push_back(w);
  return out;
}

Graph parse_text(const std::string& text, int32_t format, int64_t* declared) {
  mqo_graph* h = nullptr;
  check(mqo_graph_parse(text.data(), static_cast<int64_t>(text.size()), format, g_device,
                        declared, &h));
  return Graph::adopt(h);
}

}  // namespace

DimacsResult parse_dimacs_text(const std::string& text) {
  DimacsResult r;
  r.graph = parse_text(text, 2, &r.declared_edges);
  r.parsed_edges = r.graph.m();
  r.warnings = load_warnings();
  return r;
}

DimacsResult parse_dimacs(std::istream& in) {
  return parse_dimacs_text(std::string(std::istreambuf_iterator<char>(in), {}));
}

Graph read_canonical(std::istream& in) {
  return parse_text(std::string(std::istreambuf_iterator<char>(in), {}), 1, nullptr);
}

void write_canonical(const Graph& g, std::ostream& out) {
  out << g.n() << ' ' << g.m() << '\n';
  for (const auto& [u, v] : g.edges()) out << u << ' ' << v << '\n';
}

Graph load_graph_file(const std::string& path, std::vector<std::string>* warnings) {
  mqo_graph* h = nullptr;
  const int rc = mqo_graph_load(path.c_str(), g_device, &h);
  check(rc);
  if (warnings) {
    const auto w = load_warnings();
    warnings->insert(warnings->end(), w.begin(), w.end());
  }
  return Graph::adopt(h);
}

void write_graph_file(const Graph& g, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open output file: " + path);
  write_canonical(g, out);
}

}  // namespace mqo
