// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the reference mQO core (compiled unmodified from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libref.so) behind the C interface of oracle/mqo_oracle.h, so
// the tests can run the reference itself side by side with the plain-C
// restatement and with the CUDA path.  Every function forwards to the
// reference API named in its comment; exceptions become status codes.
#include <algorithm>
#include <cstring>
#include <sstream>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "mqo/graph.hpp"
#include "mqo/graph_io.hpp"
#include "mqo/localsearch.hpp"
#include "mqo/objectives.hpp"
#include "mqo/pga.hpp"
#include "mqo/presets.hpp"
#include "mqo/rng.hpp"
#include "mqo/solver.hpp"

extern "C" {
#include "mqo_oracle.h"
}

using namespace mqo;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_INVALID;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ORC_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_OTHER;
  }
}

ObjectiveSpec spec_of(int32_t kind, double param) {
  switch (kind) {
    case ORC_MIS_QUBO: return MisQubo{param};
    case ORC_LAPLACIAN: return Laplacian{};
    case ORC_PERTURBED_LAPLACIAN: return PerturbedLaplacian{param};
    case ORC_ADJACENCY: return Adjacency{};
    case ORC_PERTURBED_BIAS: return PerturbedBias{param};
  }
  throw std::invalid_argument("objective: unknown kind");
}

BoxDomain domain_of_kind(int32_t kind) {
  return kind == ORC_MIS_QUBO ? BoxDomain::Unit : BoxDomain::Symmetric;
}

const Graph& G(void* g) { return *static_cast<Graph*>(g); }
Rng& R(void* r) { return *static_cast<Rng*>(r); }

std::vector<Vertex> members_of(const Graph& g, const uint8_t* ind) {
  std::vector<Vertex> m;
  for (Vertex v = 0; v < g.n(); ++v)
    if (ind[v]) m.push_back(v);
  return m;
}

void write_indicator(const Graph& g, const std::vector<Vertex>& m, uint8_t* ind) {
  std::memset(ind, 0, static_cast<size_t>(g.n()));
  for (Vertex v : m) ind[v] = 1;
}

template <typename F>
int flip_call(void* g, uint8_t* side, int64_t* gain, F&& f) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] {
    std::vector<uint8_t> s(side, side + n);
    *gain = f(G(g), s);
    std::memcpy(side, s.data(), n);
  });
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
const char* orc_impl_name(void) { return "reference"; }

void* orc_rng_new(uint64_t seed) { return new Rng(seed); }
void orc_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t orc_rng_next_u64(void* r) { return R(r).next_u64(); }
double orc_rng_uniform01(void* r) { return R(r).uniform01(); }
uint64_t orc_rng_uniform_index(void* r, uint64_t n) { return R(r).uniform_index(n); }
double orc_rng_normal(void* r, double mean, double sd) { return R(r).normal(mean, sd); }
uint64_t orc_derive_seed(uint64_t master, uint64_t stream) {
  return derive_seed(master, stream);
}

int orc_graph_from_edges(int32_t n, int64_t ne, const int32_t* eu, const int32_t* ev,
                         void** out) {
  return guard([&] {
    std::vector<std::pair<Vertex, Vertex>> edges(static_cast<size_t>(ne));
    for (int64_t i = 0; i < ne; ++i) edges[i] = {eu[i], ev[i]};
    *out = new Graph(Graph::from_edges(n, std::move(edges)));
  });
}

int orc_generate_er(int32_t n, double p, uint64_t seed, void** out) {
  return guard([&] { *out = new Graph(generate({ErSpec{n, p}, seed})); });
}
int orc_generate_ba(int32_t n, int32_t m_attach, uint64_t seed, void** out) {
  return guard([&] { *out = new Graph(generate({BaSpec{n, m_attach}, seed})); });
}
int orc_generate_sbm(int32_t n, int32_t k, double p_in, double p_out, uint64_t seed,
                     void** out) {
  return guard([&] { *out = new Graph(generate({SbmSpec{n, k, p_in, p_out}, seed})); });
}

void orc_graph_free(void* g) { delete static_cast<Graph*>(g); }

int orc_strip_isolated(void* g, void** core, int32_t* core_to_orig, int32_t* orig_to_core,
                       int32_t* removed, int32_t* n_core, int32_t* n_removed) {
  return guard([&] {
    StripResult r = strip_isolated(G(g));
    std::copy(r.core_to_orig.begin(), r.core_to_orig.end(), core_to_orig);
    std::copy(r.orig_to_core.begin(), r.orig_to_core.end(), orig_to_core);
    std::copy(r.removed.begin(), r.removed.end(), removed);
    *n_core = static_cast<int32_t>(r.core_to_orig.size());
    *n_removed = static_cast<int32_t>(r.removed.size());
    *core = new Graph(std::move(r.core));
  });
}

int orc_components(void* g, int32_t* comp, int32_t* count) {
  return guard([&] {
    const auto comps = connected_components(G(g));
    for (size_t c = 0; c < comps.size(); ++c)
      for (Vertex v : comps[c]) comp[v] = static_cast<int32_t>(c);
    *count = static_cast<int32_t>(comps.size());
  });
}

void orc_graph_info(void* g, int32_t* n, int64_t* m, int32_t* max_degree) {
  *n = G(g).n();
  *m = G(g).m();
  *max_degree = G(g).max_degree();
}

void orc_graph_csr(void* gp, int64_t* offsets, int32_t* nbrs) {
  const Graph& g = G(gp);
  int64_t pos = 0;
  offsets[0] = 0;
  for (Vertex v = 0; v < g.n(); ++v) {
    for (Vertex u : g.neighbors(v)) nbrs[pos++] = u;
    offsets[v + 1] = pos;
  }
}

int orc_adjacency_apply(void* g, const double* x, double* y) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] { G(g).adjacency_apply({x, n}, {y, n}); });
}
int orc_laplacian_apply(void* g, const double* x, double* y) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] { G(g).laplacian_apply({x, n}, {y, n}); });
}

int orc_validate_objective(int32_t kind, double param) {
  return guard([&] { validate(spec_of(kind, param)); });
}

int orc_gradient(void* g, int32_t kind, double param, const double* x, double* out) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] {
    RelaxedState s{std::vector<double>(x, x + n), domain_of_kind(kind)};
    gradient(spec_of(kind, param), G(g), s, std::span<double>(out, n));
  });
}

int orc_value(void* g, int32_t kind, double param, const double* x, double* out) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] {
    RelaxedState s{std::vector<double>(x, x + n), domain_of_kind(kind)};
    *out = value(spec_of(kind, param), G(g), s);
  });
}

int orc_extract_solution(void* gp, int32_t problem, const double* x, uint8_t* body,
                         int64_t* score) {
  const Graph& g = G(gp);
  const size_t n = static_cast<size_t>(g.n());
  return guard([&] {
    RelaxedState s{std::vector<double>(x, x + n),
                   problem == ORC_PROBLEM_MIS ? BoxDomain::Unit : BoxDomain::Symmetric};
    const Solution sol =
        extract_solution(problem == ORC_PROBLEM_MIS ? Problem::Mis : Problem::MaxCut, g, s);
    *score = sol.score;
    if (const auto* is = std::get_if<IndependentSet>(&sol.body))
      write_indicator(g, is->members, body);
    else
      std::memcpy(body, std::get<CutPartition>(sol.body).side.data(), n);
  });
}

int64_t orc_cut_value(void* g, const uint8_t* side) {
  return cut_value(G(g), {side, static_cast<size_t>(G(g).n())});
}

int orc_is_independent(void* g, const uint8_t* ind) {
  const auto m = members_of(G(g), ind);
  return is_independent(G(g), m) ? 1 : 0;
}

int orc_validate_optimizer(double alpha, double beta, int32_t max_iters, double conv_tol,
                           int32_t check_every) {
  return guard([&] {
    OptimizerConfig c{alpha, beta, max_iters, conv_tol, check_every};
    validate(c);
  });
}

void orc_project(double* x, int32_t n, int32_t problem) {
  RelaxedState s{std::vector<double>(x, x + n),
                 problem == ORC_PROBLEM_MIS ? BoxDomain::Unit : BoxDomain::Symmetric};
  project(s);
  std::memcpy(x, s.x.data(), static_cast<size_t>(n) * sizeof(double));
}

int orc_step(void* g, int32_t kind, double param, double* x, double* v, double alpha,
             double beta) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] {
    RelaxedState s{std::vector<double>(x, x + n), domain_of_kind(kind)};
    std::vector<double> vel(v, v + n);
    OptimizerConfig c;
    c.alpha = alpha;
    c.beta = beta;
    step(spec_of(kind, param), G(g), s, vel, c);
    std::memcpy(x, s.x.data(), n * sizeof(double));
    std::memcpy(v, vel.data(), n * sizeof(double));
  });
}

int orc_run_trajectory(void* g, int32_t kind, double param, double* x, double alpha,
                       double beta, int32_t max_iters, double conv_tol,
                       int32_t check_every, int32_t* iterations, int32_t* reason) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] {
    OptimizerConfig c{alpha, beta, max_iters, conv_tol, check_every};
    RelaxedState s{std::vector<double>(x, x + n), domain_of_kind(kind)};
    const TrajectoryOutcome out = run_trajectory(spec_of(kind, param), G(g), std::move(s), c);
    std::memcpy(x, out.state.x.data(), n * sizeof(double));
    *iterations = out.iterations;
    *reason = static_cast<int32_t>(out.reason);
  });
}

int orc_mis_fixed_point_check(void* g, const double* x, double gamma, double alpha,
                              int32_t* fixed) {
  const size_t n = static_cast<size_t>(G(g).n());
  return guard([&] { *fixed = mis_fixed_point_check(G(g), {x, n}, gamma, alpha) ? 1 : 0; });
}

int orc_init_state(void* g, int32_t problem, double sigma, void* rng, double* x) {
  return guard([&] {
    const RelaxedState s = init_state(
        problem == ORC_PROBLEM_MIS ? Problem::Mis : Problem::MaxCut, G(g), sigma, R(rng));
    std::memcpy(x, s.x.data(), s.x.size() * sizeof(double));
  });
}

int orc_global_reset(double* x, int32_t n, double rho, void* rng, int32_t* chosen,
                     int32_t* k) {
  return guard([&] {
    RelaxedState s{std::vector<double>(x, x + n), BoxDomain::Unit};
    const auto c = global_reset(s, rho, R(rng));
    std::memcpy(x, s.x.data(), static_cast<size_t>(n) * sizeof(double));
    if (chosen) std::memcpy(chosen, c.data(), c.size() * sizeof(int32_t));
    if (k) *k = static_cast<int32_t>(c.size());
  });
}

int orc_build_tightness(void* g, const uint8_t* ind, int32_t* tight) {
  return guard([&] {
    const auto t = build_tightness(G(g), members_of(G(g), ind));
    std::memcpy(tight, t.selected_neighbors.data(), t.selected_neighbors.size() * 4);
  });
}

int orc_build_gain_table(void* g, const uint8_t* side, int64_t* delta) {
  return guard([&] {
    const auto t = build_gain_table(G(g), {side, static_cast<size_t>(G(g).n())});
    std::memcpy(delta, t.delta.data(), t.delta.size() * 8);
  });
}

int orc_greedy_maximalize(void* g, uint8_t* ind, int32_t* size) {
  return guard([&] {
    const auto m = greedy_maximalize(G(g), members_of(G(g), ind));
    write_indicator(G(g), m, ind);
    *size = static_cast<int32_t>(m.size());
  });
}

int orc_one_two_swap(void* g, uint8_t* ind, int32_t* size) {
  return guard([&] {
    const auto m = one_two_swap(G(g), members_of(G(g), ind));
    write_indicator(G(g), m, ind);
    *size = static_cast<int32_t>(m.size());
  });
}

int orc_one_flip_pass(void* g, uint8_t* side, int64_t* gain) {
  return flip_call(g, side, gain, [](const Graph& gr, std::vector<uint8_t>& s) {
    return one_flip_pass(gr, s);
  });
}
int orc_two_flip_pass(void* g, uint8_t* side, int64_t* gain) {
  return flip_call(g, side, gain, [](const Graph& gr, std::vector<uint8_t>& s) {
    return two_flip_pass(gr, s);
  });
}
int orc_one_two_flip(void* g, uint8_t* side, int64_t* gain) {
  return flip_call(g, side, gain, [](const Graph& gr, std::vector<uint8_t>& s) {
    return one_two_flip(gr, s);
  });
}

int orc_solve_pooled(void* gp, const orc_solver_cfg* c, orc_report* rep, uint8_t* best_body) {
  const Graph& g = G(gp);
  return guard([&] {
    SolverConfig cfg;
    cfg.objective = spec_of(c->objective, c->param);
    cfg.optimizer = OptimizerConfig{c->alpha, c->beta, c->max_iters, c->conv_tol,
                                    c->check_every};
    cfg.reset_fraction = c->reset_fraction;
    cfg.reset_rounds = c->reset_rounds;
    cfg.init_noise = c->init_noise;
    cfg.time_budget_secs = c->time_budget_secs;
    cfg.seed = c->seed;
    cfg.local_search = c->local_search != 0;
    cfg.pool = {c->pool_batch, c->pool_keep};
    if (c->has_init_constant) cfg.init_constant = c->init_constant;
    if (c->has_stop_at_score) cfg.stop_at_score = c->stop_at_score;
    if (c->has_max_outer_loops) cfg.max_outer_loops = c->max_outer_loops;
    const RunReport r = solve_pooled(g, cfg);
    std::memset(rep, 0, sizeof *rep);
    rep->score = r.best.score;
    rep->found_solution = r.found_solution ? 1 : 0;
    rep->after_gradient = r.phases.after_gradient;
    rep->after_reset_loop = r.phases.after_reset_loop;
    rep->after_local_search = r.phases.after_local_search;
    rep->outer_loops = r.outer_loops;
    rep->trajectories = r.trajectories;
    rep->resets_accepted = r.resets_accepted;
    rep->resets_rejected = r.resets_rejected;
    rep->total_iterations = r.total_iterations;
    rep->last_trajectory_stop = static_cast<int32_t>(r.last_trajectory_stop);
    rep->elapsed_secs = r.elapsed_secs;
    rep->n_warnings = static_cast<int32_t>(r.warnings.size());
    if (best_body) {
      if (const auto* is = std::get_if<IndependentSet>(&r.best.body))
        write_indicator(g, is->members, best_body);
      else
        std::memcpy(best_body, std::get<CutPartition>(r.best.body).side.data(),
                    static_cast<size_t>(g.n()));
    }
  });
}

int orc_preset_for(int32_t problem, int32_t n, double mean_degree, double* alpha,
                   double* momentum, double* rho, int32_t* reset_rounds) {
  const Preset p =
      preset_for(problem == ORC_PROBLEM_MIS ? Problem::Mis : Problem::MaxCut, n, mean_degree);
  *alpha = p.alpha;
  *momentum = p.momentum;
  *rho = p.rho;
  *reset_rounds = p.reset_rounds;
  return ORC_OK;
}

}  // extern "C"

// ---- graph text formats (reference-only probe; used by
// tests/golden/make_graph_io_golden.py to freeze the reference's behaviour)
// fmt 1 = read_canonical (graph_io.cpp:74-87), 2 = parse_dimacs_text
// (18-71), 0 = load_graph_file's sniffing (94-106) applied to the text.
// Returns 0 ok, 1 ParseError, 2 invalid_argument, 3 other; on success the
// CSR goes to off/nbr (caller-sized n+1 / 2m; pass NULL first to size).
extern "C" int ref_parse_graph(const char* text, int64_t len, int32_t fmt, int32_t* n,
                               int64_t* m, int64_t* declared, int64_t* off, int32_t* nbr,
                               char* msg, int64_t cap, int32_t* line) {
  auto put = [&](const std::string& s) {
    if (msg && cap > 0) {
      const size_t k = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(msg, s.data(), k);
      msg[k] = 0;
    }
  };
  *line = 0;
  try {
    std::string t(text, static_cast<size_t>(len));
    Graph g;
    std::vector<std::string> warnings;
    *declared = -1;
    const bool dimacs = fmt == 2 || (fmt == 0 && !t.empty() && (t[0] == 'c' || t[0] == 'p'));
    if (dimacs) {
      DimacsResult r = parse_dimacs_text(t);
      *declared = r.declared_edges;
      warnings = r.warnings;
      g = std::move(r.graph);
    } else {
      std::istringstream in(t);
      g = read_canonical(in);
    }
    *n = g.n();
    *m = g.m();
    if (off) {
      for (Vertex v = 0; v <= g.n(); ++v) off[v] = v == 0 ? 0 : off[v - 1] + g.degree(v - 1);
      int64_t k = 0;
      for (Vertex v = 0; v < g.n(); ++v)
        for (Vertex u : g.neighbors(v)) nbr[k++] = u;
    }
    std::string w;
    for (size_t i = 0; i < warnings.size(); ++i) w += (i ? "\n" : "") + warnings[i];
    put(w);
    return 0;
  } catch (const ParseError& e) {
    put(e.what());
    *line = e.line();
    return 1;
  } catch (const std::invalid_argument& e) {
    put(e.what());
    return 2;
  } catch (const std::exception& e) {
    put(e.what());
    return 3;
  }
}

// ---- the reference CLI (tools/src/cli_common.cpp, cmd_basic.cpp,
// cmd_sweep.cpp), for RunRecord parity of paper_2605_06921_b200/cli.py.
// `args`: '\n'-separated key=value lines naming SolveOptions fields
// (cli_common.hpp:33-48; "cmd" = solve | sweep, plus param / values / seeds
// / jobs / jsonl for sweep).  The command writes its record to `out`
// (SolveOptions::out_file / the sweep's jsonl path) exactly as the
// reference binary would print it.  Returns the command's exit code, or -1
// with the message in orc_last_error() when it throws.
#include "cli_common.hpp"

extern "C" int orc_cli_run(const char* args) {
  using namespace mqo::cli;
  try {
    SolveOptions opt;
    std::string cmd = "solve", param, values, seeds = "", jsonl;
    int jobs = 1;
    std::istringstream in(args ? args : "");
    std::string line;
    while (std::getline(in, line)) {
      const auto eq = line.find('=');
      if (eq == std::string::npos) continue;
      const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
      if (k == "cmd") cmd = v;
      else if (k == "problem") opt.problem = v;
      else if (k == "graph") opt.graph_file = v;
      else if (k == "gen") opt.gen_spec = v;
      else if (k == "objective") opt.objective = v;
      else if (k == "preset") opt.preset = v;
      else if (k == "report") opt.report = v;
      else if (k == "out") opt.out_file = v;
      else if (k == "budget_secs") opt.budget_secs = std::stod(v);
      else if (k == "seed") opt.seed = std::stoull(v);
      else if (k == "alpha") opt.alpha = std::stod(v);
      else if (k == "momentum") opt.momentum = std::stod(v);
      else if (k == "rho") opt.rho = std::stod(v);
      else if (k == "lambda") opt.lambda = std::stod(v);
      else if (k == "gamma") opt.gamma = std::stod(v);
      else if (k == "sigma") opt.sigma = std::stod(v);
      else if (k == "conv_tol") opt.conv_tol = std::stod(v);
      else if (k == "tgs") opt.tgs = std::stoi(v);
      else if (k == "max_iters") opt.max_iters = std::stoi(v);
      else if (k == "check_every") opt.check_every = std::stoi(v);
      else if (k == "pool_b") opt.pool_b = std::stoi(v);
      else if (k == "pool_k") opt.pool_k = std::stoi(v);
      else if (k == "max_outer") opt.max_outer = std::stoi(v);
      else if (k == "init_constant") opt.init_constant = std::stod(v);
      else if (k == "stop_at_score") opt.stop_at_score = std::stoll(v);
      else if (k == "no_local_search") opt.no_local_search = v == "1";
      else if (k == "param") param = v;
      else if (k == "values") values = v;
      else if (k == "seeds") seeds = v;
      else if (k == "jobs") jobs = std::stoi(v);
      else if (k == "jsonl") jsonl = v;
      else throw std::invalid_argument("orc_cli_run: unknown key " + k);
    }
    if (cmd == "solve") return cmd_solve(opt);
    if (cmd == "sweep") return cmd_sweep(opt, param, values, seeds, jobs, jsonl);
    throw std::invalid_argument("orc_cli_run: unknown cmd " + cmd);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
