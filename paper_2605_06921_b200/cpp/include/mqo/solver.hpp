#pragma once
// Drop-in for the reference's mqo/solver.hpp (solver.hpp:11-80).  The
// engine runs on the B200 backend; `SolverConfig` gains one optional knob
// (init_on_device) whose default keeps reference bit-parity.
#include <optional>
#include <string>

#include "mqo/pga.hpp"
#include "mqo/rng.hpp"

namespace mqo {

struct PoolConfig {
  int batch = 1;
  int keep = 1;
};

struct SolverConfig {
  ObjectiveSpec objective = MisQubo{};
  OptimizerConfig optimizer;
  double reset_fraction = 0.5;
  int reset_rounds = 60;
  double init_noise = 0.15;
  double time_budget_secs = 10.0;
  uint64_t seed = 1;
  bool local_search = true;
  PoolConfig pool;
  std::optional<double> init_constant;
  std::optional<int64_t> stop_at_score;
  std::optional<int> max_outer_loops;
  bool init_on_device = false;  // B200: CUDA-libm Box-Muller (not bit-exact)
};
void validate(const SolverConfig& cfg);

struct PhaseGains {
  int64_t after_gradient = 0;
  int64_t after_reset_loop = 0;
  int64_t after_local_search = 0;
};

struct RunReport {
  Solution best;
  bool found_solution = false;
  PhaseGains phases;
  int outer_loops = 0;
  int trajectories = 0;
  int64_t resets_accepted = 0;
  int64_t resets_rejected = 0;
  int64_t total_iterations = 0;
  StopReason last_trajectory_stop = StopReason::IterCap;
  double elapsed_secs = 0.0;
  std::vector<std::string> warnings;
  SolverConfig config;
};

RelaxedState init_state(Problem problem, const Graph& g, double sigma, Rng& rng);
std::vector<Vertex> global_reset(RelaxedState& state, double rho, Rng& rng);

RunReport solve_mis(const Graph& g, const SolverConfig& cfg);
RunReport solve_maxcut(const Graph& g, const SolverConfig& cfg);
RunReport solve_pooled(const Graph& g, const SolverConfig& cfg);

}  // namespace mqo
