// facade_tests.cpp -- the reference's unit-test cases
// (/root/reference/proj/tests/test_{graph,objectives,pga,localsearch,solver}.cpp),
// re-hosted as plain checks (doctest is not available) and compiled
// against the drop-in headers cpp/include/mqo/*.hpp + libmqo_core_b200.so.
// A reference caller needs no source change: these are its calls.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mqo/graph.hpp"
#include "mqo/graph_io.hpp"
#include "mqo/localsearch.hpp"
#include "mqo/objectives.hpp"
#include "mqo/pga.hpp"
#include "mqo/presets.hpp"
#include "mqo/solver.hpp"

using namespace mqo;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                   \
  do {                                             \
    bool caught = false;                           \
    try {                                          \
      (void)(expr);                                \
    } catch (const T&) {                           \
      caught = true;                               \
    } catch (...) {                                \
    }                                              \
    CHECK(caught);                                 \
  } while (0)

namespace {
Graph path(Vertex n) {
  std::vector<std::pair<Vertex, Vertex>> e;
  for (Vertex v = 0; v + 1 < n; ++v) e.emplace_back(v, v + 1);
  return Graph::from_edges(n, e);
}
Graph cycle(Vertex n) {
  std::vector<std::pair<Vertex, Vertex>> e;
  for (Vertex v = 0; v < n; ++v) e.emplace_back(v, (v + 1) % n);
  return Graph::from_edges(n, e);
}
Graph complete(Vertex n) {
  std::vector<std::pair<Vertex, Vertex>> e;
  for (Vertex u = 0; u < n; ++u)
    for (Vertex v = u + 1; v < n; ++v) e.emplace_back(u, v);
  return Graph::from_edges(n, e);
}
Graph star(Vertex leaves) {
  std::vector<std::pair<Vertex, Vertex>> e;
  for (Vertex v = 1; v <= leaves; ++v) e.emplace_back(0, v);
  return Graph::from_edges(leaves + 1, e);
}
Graph petersen() {
  std::vector<std::pair<Vertex, Vertex>> e;
  for (Vertex v = 0; v < 5; ++v) {
    e.emplace_back(v, (v + 1) % 5);
    e.emplace_back(v, v + 5);
    e.emplace_back(v + 5, 5 + (v + 2) % 5);
  }
  return Graph::from_edges(10, e);
}
Graph er(Vertex n, double p, uint64_t seed) { return generate({ErSpec{n, p}, seed}); }

SolverConfig mis_config(uint64_t seed, double budget = 2.0) {
  SolverConfig c;
  c.objective = MisQubo{2.0};
  c.optimizer.alpha = 0.8;
  c.optimizer.beta = 0.3;
  c.reset_fraction = 0.5;
  c.reset_rounds = 20;
  c.time_budget_secs = budget;
  c.seed = seed;
  return c;
}
SolverConfig maxcut_config(uint64_t seed, double budget = 2.0) {
  SolverConfig c;
  c.objective = PerturbedBias{0.001};
  c.optimizer.alpha = 0.0025;
  c.optimizer.beta = 0.8;
  c.reset_fraction = 0.8;
  c.reset_rounds = 20;
  c.time_budget_secs = budget;
  c.seed = seed;
  return c;
}
bool same_report(const RunReport& a, const RunReport& b) {
  return a.best.score == b.best.score && a.best.body == b.best.body &&
         a.outer_loops == b.outer_loops && a.trajectories == b.trajectories &&
         a.resets_accepted == b.resets_accepted && a.resets_rejected == b.resets_rejected &&
         a.total_iterations == b.total_iterations &&
         a.phases.after_gradient == b.phases.after_gradient &&
         a.phases.after_reset_loop == b.phases.after_reset_loop &&
         a.phases.after_local_search == b.phases.after_local_search;
}
}  // namespace

static void test_graph() {
  const Graph k3 = complete(3);
  CHECK(k3.n() == 3 && k3.m() == 3 && k3.max_degree() == 2);
  const Graph g = Graph::from_edges(4, {{1, 0}, {0, 1}, {2, 3}, {3, 2}, {1, 3}});
  CHECK(g.m() == 3 && g.has_edge(1, 3) && !g.has_edge(0, 2));
  CHECK_THROWS_AS(Graph::from_edges(3, {{1, 1}}), std::invalid_argument);
  CHECK_THROWS_AS(Graph::from_edges(3, {{0, 3}}), std::invalid_argument);
  // test_graph.cpp:71-76
  CHECK(k3.adjacency_apply(std::vector<double>{1, -1, -1}) == (std::vector<double>{-2, 0, 0}));
  CHECK(k3.laplacian_apply(std::vector<double>{1, -1, -1}) == (std::vector<double>{4, -2, -2}));
  const Graph e = er(30, 0.3, 5);
  for (double c : {0.3, -0.7})
    for (double y : e.laplacian_apply(std::vector<double>(30, c))) CHECK(y == 0.0);
  const Graph ba = generate({BaSpec{2000, 3}, 9});
  CHECK(ba.m() == 3 + 3 * (2000 - 4));
  const auto sr = strip_isolated(Graph::from_edges(5, {{0, 2}}));
  CHECK(sr.core.n() == 2 && sr.removed == (std::vector<Vertex>{1, 3, 4}));
  CHECK(connected_components(path(4)).size() == 1);
}

// test_graph.cpp:132-189
static void test_graph_io() {
  {
    const auto r = parse_dimacs_text("c a comment\np edge 3 3\ne 1 2\ne 2 3\ne 1 3\n");
    CHECK(r.graph.n() == 3 && r.graph.m() == 3 && r.warnings.empty());
  }
  {
    const auto r = parse_dimacs_text("p edge 3 2\ne 1 2\ne 2 1\n");
    CHECK(r.graph.n() == 3 && r.graph.m() == 1);
    CHECK(r.warnings.size() == 1 && r.warnings[0].find("declared m=2") != std::string::npos);
  }
  {
    bool ok = false;
    try {
      parse_dimacs_text("e 1 2\n");
    } catch (const ParseError& e) {
      ok = std::string(e.what()) == "line 1: edge before 'p edge <n> <m>' header" && e.line() == 1;
    }
    CHECK(ok);
    int line = 0;
    try {
      parse_dimacs_text("p edge 3 2\ne 1 2\ne 1 9\n");
    } catch (const ParseError& e) {
      line = e.line();
    }
    CHECK(line == 3);
    CHECK_THROWS_AS(parse_dimacs_text("p edge 3 1\ne 1 1\n"), ParseError);
    CHECK_THROWS_AS(parse_dimacs_text("p edge 3 1\nq 1 2\n"), ParseError);
    CHECK_THROWS_AS(parse_dimacs_text("p edge 3 1\ne one two\n"), ParseError);
  }
  {
    const Graph g = er(37, 0.2, 21);
    std::stringstream buffer;
    write_canonical(g, buffer);
    const Graph back = read_canonical(buffer);
    CHECK(back.n() == g.n() && back.edges() == g.edges());
  }
  {
    const Graph g = er(12, 0.3, 31);
    const std::string canon = "/tmp/mqo_b200_test_canonical.g";
    write_graph_file(g, canon);
    CHECK(load_graph_file(canon).edges() == g.edges());
    const std::string dimacs = "/tmp/mqo_b200_test_dimacs.g";
    {
      std::ofstream out(dimacs);
      out << "c tiny triangle\np edge 3 3\ne 1 2\ne 2 3\ne 1 3\n";
    }
    std::vector<std::string> warnings;
    const Graph k3 = load_graph_file(dimacs, &warnings);
    CHECK(k3.n() == 3 && k3.m() == 3 && warnings.empty());
  }
}

static void test_objectives() {
  const Graph k3 = complete(3);
  CHECK(gradient(MisQubo{2.0}, k3, {{1, 0, 0}, BoxDomain::Unit}) == (std::vector<double>{1, -1, -1}));
  CHECK(gradient(PerturbedBias{0.25}, k3, {{0, 0, 0}, BoxDomain::Symmetric}) ==
        (std::vector<double>{-0.25, -0.25, -0.25}));
  CHECK_THROWS_AS(validate(ObjectiveSpec{MisQubo{1.0}}), std::invalid_argument);
  CHECK_THROWS_AS(gradient(MisQubo{2.0}, k3, {{1, 0, 0}, BoxDomain::Symmetric}),
                  std::invalid_argument);
  const auto s = extract_solution(Problem::Mis, k3, {{0.5, 0.5, 0.5}, BoxDomain::Unit});
  CHECK(s.score == 0 && std::get<IndependentSet>(s.body).members.empty());
  const auto c = extract_solution(Problem::MaxCut, k3, {{0.5, -0.5, 0.0}, BoxDomain::Symmetric});
  CHECK(c.score == 2 && std::get<CutPartition>(c.body).side == (std::vector<uint8_t>{1, 0, 0}));
  CHECK(cut_value(cycle(4), std::vector<uint8_t>{0, 1, 0, 1}) == 4);
  CHECK(is_independent(cycle(5), std::vector<Vertex>{0, 2}));
  CHECK(!is_independent(cycle(5), std::vector<Vertex>{0, 1}));
  // binary identities (test_objectives.cpp:160-175)
  const Graph g = er(10, 0.5, 3);
  Rng rng(1);
  for (int t = 0; t < 20; ++t) {
    std::vector<uint8_t> side(10);
    std::vector<double> x(10);
    for (int v = 0; v < 10; ++v) {
      side[v] = rng.next_u64() & 1;
      x[v] = side[v] ? 1.0 : -1.0;
    }
    const double cut = static_cast<double>(cut_value(g, side));
    CHECK(value(Laplacian{}, g, {x, BoxDomain::Symmetric}) == cut);
    CHECK(value(Adjacency{}, g, {x, BoxDomain::Symmetric}) == 4 * cut - 2.0 * g.m());
  }
}

static void test_pga() {
  const Graph k3 = complete(3);
  RelaxedState unit{{1.3, -0.2, 0.5}, BoxDomain::Unit};
  project(unit);
  CHECK(unit.x == (std::vector<double>{1.0, 0.0, 0.5}));
  OptimizerConfig cfg;
  cfg.alpha = 0.1;
  RelaxedState x{{1.0, 0.0, 0.0}, BoxDomain::Unit};
  std::vector<double> vel;
  step(MisQubo{2.0}, k3, x, vel, cfg);
  CHECK(x.x == (std::vector<double>{1.0, 0.0, 0.0}));
  OptimizerConfig c8;
  c8.alpha = 0.8;
  auto out = run_trajectory(MisQubo{2.0}, k3, {{0.9, 0.1, 0.1}, BoxDomain::Unit}, c8);
  CHECK(out.reason == StopReason::CheckerAccepted && out.state.x == (std::vector<double>{1, 0, 0}));
  OptimizerConfig c1;
  c1.alpha = 0.1;
  out = run_trajectory(PerturbedBias{0.001}, k3, {{0.6, -0.5, -0.4}, BoxDomain::Symmetric}, c1);
  CHECK(out.reason == StopReason::Converged && out.state.x == (std::vector<double>{1, -1, -1}));
  CHECK(extract_solution(Problem::MaxCut, k3, out.state).score == 2);
  OptimizerConfig cap;
  cap.alpha = 1e-9;
  cap.max_iters = 12;
  out = run_trajectory(MisQubo{2.0}, k3, {{0.4, 0.4, 0.4}, BoxDomain::Unit}, cap);
  CHECK(out.reason == StopReason::IterCap && out.iterations == 12);
  // bit-determinism (test_pga.cpp:121-135)
  const Graph g = er(30, 0.2, 79);
  OptimizerConfig cd;
  cd.alpha = 0.0025;
  cd.beta = 0.8;
  RelaxedState init{std::vector<double>(30), BoxDomain::Symmetric};
  Rng r5(5);
  for (auto& v : init.x) v = (r5.next_u64() & 1 ? 1.0 : -1.0) * 0.5;
  const auto a = run_trajectory(PerturbedBias{0.001}, g, init, cd);
  const auto b = run_trajectory(PerturbedBias{0.001}, g, init, cd);
  CHECK(a.iterations == b.iterations && a.state.x == b.state.x);
  CHECK(mis_fixed_point_check(k3, std::vector<double>{1, 0, 0}, 2.0, 0.8));
  CHECK(!mis_fixed_point_check(path(3), std::vector<double>{1, 0, 0}, 2.0, 0.8));
  CHECK(mis_fixed_point_check(cycle(5), std::vector<double>{1, 0, 1, 0, 0}, 2.0, 0.8));
  CHECK_THROWS_AS(mis_fixed_point_check(k3, std::vector<double>{0.5, 0, 0}, 2.0, 0.8),
                  std::invalid_argument);
  CHECK(maxcut_binary_fixed_point_check(Adjacency{}, k3, std::vector<double>{1, -1, -1}));
  CHECK_THROWS_AS(maxcut_binary_fixed_point_check(MisQubo{2.0}, k3, std::vector<double>{1, -1, -1}),
                  std::invalid_argument);
}

static void test_localsearch() {
  CHECK(greedy_maximalize(cycle(5), {0}) == (std::vector<Vertex>{0, 2}));
  CHECK_THROWS_AS(greedy_maximalize(complete(3), {0, 1}), std::invalid_argument);
  CHECK(one_two_swap(cycle(5), {0, 2}) == (std::vector<Vertex>{0, 2}));
  CHECK(one_two_swap(star(4), {0}) == (std::vector<Vertex>{1, 2, 3, 4}));
  CHECK(one_two_swap(path(5), {1, 3}) == (std::vector<Vertex>{1, 3}));
  CHECK_THROWS_AS(one_two_swap(complete(3), {0, 1}), std::invalid_argument);
  CHECK_THROWS_AS(one_two_swap(path(3), {0}), std::invalid_argument);
  std::vector<uint8_t> side{0, 0, 0};
  CHECK(one_flip_pass(complete(3), side) == 2 && cut_value(complete(3), side) == 2);
  std::vector<uint8_t> c4{0, 1, 0, 1};
  CHECK(one_flip_pass(cycle(4), c4) == 0 && c4 == (std::vector<uint8_t>{0, 1, 0, 1}));
  std::vector<uint8_t> p3{0, 1, 0};
  CHECK(two_flip_pass(path(3), p3) == 0);
  // gain-table bookkeeping (test_localsearch.cpp:107-135)
  Rng rng(109);
  for (int t = 0; t < 5; ++t) {
    const Graph g = er(18, 0.3, derive_seed(109, t));
    std::vector<uint8_t> s(18);
    for (auto& q : s) q = rng.next_u64() & 1;
    GainTable gains = build_gain_table(g, s);
    for (int k = 0; k < 40; ++k) apply_flip(g, s, gains, static_cast<Vertex>(rng.uniform_index(18)));
    CHECK(gains.delta == build_gain_table(g, s).delta);
  }
  const auto tt = build_tightness(cycle(5), std::vector<Vertex>{0, 2});
  CHECK(tt.selected_neighbors == (std::vector<int32_t>{0, 2, 0, 1, 1}));
  // swaps never shrink, end irreparable-by-construction (test_localsearch.cpp:61-75)
  for (int t = 0; t < 10; ++t) {
    const Graph g = er(24, rng.uniform(0.08, 0.35), derive_seed(103, t));
    const auto start = greedy_maximalize(g, {});
    const auto improved = one_two_swap(g, start);
    CHECK(improved.size() >= start.size() && is_independent(g, improved));
  }
}

static void test_solver() {
  // init_state (test_solver.cpp:55-81)
  Rng r1(1);
  const auto s = init_state(Problem::Mis, star(3), 0.0, r1);
  CHECK(s.x[0] == 0.0 && std::abs(s.x[1] - (1.0 - 1.0 / 3.0)) < 1e-15);
  Rng r2(1);
  for (double v : init_state(Problem::MaxCut, cycle(4), 0.0, r2).x) CHECK(v == -1.0);
  Rng a9(9), b9(9);
  const Graph g40 = er(40, 0.2, 3);
  CHECK(init_state(Problem::Mis, g40, 0.15, a9).x == init_state(Problem::Mis, g40, 0.15, b9).x);
  CHECK_THROWS_AS(init_state(Problem::Mis, Graph::from_edges(4, {}), 0.1, r1), std::invalid_argument);
  // init_state through the facade == the reference's Rng consumption
  Rng ref(derive_seed(5, 1)), dev(derive_seed(5, 1));
  const auto xi = init_state(Problem::Mis, g40, 0.15, dev);
  for (int v = 0; v < 40; ++v) {
    const double ratio = 1.0 - static_cast<double>(g40.degree(v)) / g40.max_degree();
    double base = ratio + ref.normal(0.0, 0.15);
    base = std::min(1.0, std::max(0.0, base));
    CHECK(xi.x[v] == base);
  }
  CHECK(ref.next_u64() == dev.next_u64());
  // global_reset (test_solver.cpp:83-118)
  RelaxedState st{std::vector<double>(10, 1.0), BoxDomain::Unit};
  Rng r5(5);
  const auto chosen = global_reset(st, 0.5, r5);
  int zeroed = 0;
  for (double v : st.x) zeroed += v == 0.0;
  CHECK(chosen.size() == 5 && zeroed == 5);
  // the same draws as a host partial Fisher-Yates on the reference Rng
  Rng h5(5);
  std::vector<Vertex> order(10);
  for (int v = 0; v < 10; ++v) order[v] = v;
  for (int i = 0; i < 5; ++i) std::swap(order[i], order[i + h5.uniform_index(10 - i)]);
  std::vector<Vertex> expect(order.begin(), order.begin() + 5);
  std::sort(expect.begin(), expect.end());
  CHECK(chosen == expect);
  CHECK(r5.next_u64() == h5.next_u64());
  // small optima + guards (test_solver.cpp:120-165)
  CHECK(solve_mis(cycle(5), mis_config(3, 1.0)).best.score == 2);
  SolverConfig pc = mis_config(4, 5.0);
  pc.stop_at_score = 4;
  CHECK(solve_mis(petersen(), pc).best.score == 4);
  CHECK(solve_maxcut(complete(3), maxcut_config(5, 1.0)).best.score == 2);
  CHECK(solve_maxcut(cycle(5), maxcut_config(6, 1.0)).best.score == 4);
  CHECK_THROWS_AS(solve_mis(cycle(5), maxcut_config(1)), std::invalid_argument);
  SolverConfig bad = mis_config(1);
  bad.reset_fraction = 1.0;
  CHECK_THROWS_AS(solve_mis(cycle(5), bad), std::invalid_argument);
  const RunReport edgeless = solve_mis(Graph::from_edges(6, {}), mis_config(1, 0.5));
  CHECK(edgeless.best.score == 6 && !edgeless.warnings.empty());
  SolverConfig tiny = mis_config(1);
  tiny.time_budget_secs = 1e-9;
  const RunReport none = solve_mis(er(30, 0.2, 311), tiny);
  CHECK(!none.found_solution && none.best.score == 0 && !none.warnings.empty());
  // reproducibility and B=K=1 pooled == sequential (test_solver.cpp:192-214)
  const Graph g50 = er(50, 0.15, 313);
  SolverConfig rc = mis_config(23, 60.0);
  rc.max_outer_loops = 2;
  rc.reset_rounds = 8;
  CHECK(same_report(solve_mis(g50, rc), solve_mis(g50, rc)));
  CHECK(same_report(solve_mis(g50, rc), solve_pooled(g50, rc)));
  // reports are internally consistent (test_solver.cpp:167-181)
  const Graph g60 = er(60, 0.1, 307);
  SolverConfig cc = mis_config(17, 1.5);
  cc.reset_rounds = 10;
  const RunReport r = solve_mis(g60, cc);
  CHECK(r.phases.after_gradient <= r.phases.after_reset_loop);
  CHECK(r.phases.after_reset_loop <= r.phases.after_local_search);
  CHECK(r.best.score == r.phases.after_local_search);
  CHECK(r.best.score == score_solution(g60, r.best) && r.found_solution && r.outer_loops >= 1);
  // a pool dominates the singleton run (test_solver.cpp:234-245)
  const Graph g200 = er(200, 0.1, 331);
  SolverConfig single = maxcut_config(41, 120.0);
  single.max_outer_loops = 1;
  single.reset_rounds = 10;
  SolverConfig pooled = single;
  pooled.pool = {8, 4};
  CHECK(solve_pooled(g200, pooled).best.score >= solve_pooled(g200, single).best.score);
  // presets
  const Preset p = preset_for(Problem::MaxCut, 1000000, 10.0);
  CHECK(p.alpha == 0.0025 && p.momentum == 0.8 && p.rho == 0.8 && p.reset_rounds == 90);
}

int main() {
  const std::vector<std::pair<const char*, std::function<void()>>> suites = {
      {"graph", test_graph},         {"graph_io", test_graph_io},
      {"objectives", test_objectives}, {"pga", test_pga},
      {"localsearch", test_localsearch}, {"solver", test_solver}};
  for (const auto& [name, fn] : suites) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "suite %s threw: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
