/*
 * mqo_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * C interface shared by the two CPU checkers of the B200 mQO path:
 *   liboracle.so      plain-C restatement of the reference algorithm
 *                     (oracle/mqo_oracle.c, compiled by oracle/Makefile);
 *   _ref/libref.so    the reference core itself, compiled from
 *                     /root/reference/proj/core/src/ (.cpp) behind
 *                     oracle/ref_shim.cpp (same symbols, same meaning).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.  Nothing in the product
 * package (paper_2605_06921_b200/) links or calls them.
 *
 * Conventions: graphs and RNGs are opaque handles; bodies are uint8[n]
 * (MIS: membership indicator, MaxCut: side); every int-returning entry
 * point returns 0 on success, 1 for std::invalid_argument, 2 for
 * std::logic_error, 3 for anything else, with orc_last_error() holding the
 * message.
 */
#ifndef MQO_ORACLE_H
#define MQO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_LOGIC = 2, ORC_OTHER = 3 };

/* objective kinds, in the order of the reference ObjectiveSpec variant
 * (objectives.hpp:34-35) */
enum {
  ORC_MIS_QUBO = 0,
  ORC_LAPLACIAN = 1,
  ORC_PERTURBED_LAPLACIAN = 2,
  ORC_ADJACENCY = 3,
  ORC_PERTURBED_BIAS = 4
};
enum { ORC_PROBLEM_MIS = 0, ORC_PROBLEM_MAXCUT = 1 };
/* StopReason order of pga.hpp:23 */
enum { ORC_CONVERGED = 0, ORC_CHECKER_ACCEPTED = 1, ORC_ITER_CAP = 2 };

typedef struct {
  int32_t objective;
  double param; /* gamma (MIS) or lambda (perturbed objectives) */
  double alpha, beta;
  int32_t max_iters;
  double conv_tol;
  int32_t check_every;
  double reset_fraction;
  int32_t reset_rounds;
  double init_noise;
  double time_budget_secs;
  uint64_t seed;
  int32_t local_search;
  int32_t pool_batch, pool_keep;
  int32_t has_init_constant;
  double init_constant;
  int32_t has_stop_at_score;
  int64_t stop_at_score;
  int32_t has_max_outer_loops;
  int32_t max_outer_loops;
} orc_solver_cfg;

typedef struct {
  int64_t score;
  int32_t found_solution;
  int64_t after_gradient, after_reset_loop, after_local_search;
  int32_t outer_loops, trajectories;
  int64_t resets_accepted, resets_rejected, total_iterations;
  int32_t last_trajectory_stop;
  double elapsed_secs;
  int32_t n_warnings;
} orc_report;

const char* orc_last_error(void);
const char* orc_impl_name(void); /* "oracle-c" or "reference" */

/* --- RNG (rng.hpp) --- */
void* orc_rng_new(uint64_t seed);
void orc_rng_free(void* rng);
uint64_t orc_rng_next_u64(void* rng);
double orc_rng_uniform01(void* rng);
uint64_t orc_rng_uniform_index(void* rng, uint64_t n);
double orc_rng_normal(void* rng, double mean, double stddev);
uint64_t orc_derive_seed(uint64_t master, uint64_t stream);

/* --- Graph (graph.hpp) --- */
int orc_graph_from_edges(int32_t n, int64_t ne, const int32_t* eu, const int32_t* ev,
                         void** out);
/* oracle-c only (test helper): wrap an already canonical CSR */
int orc_graph_from_csr(int32_t n, const int64_t* off, const int32_t* nbr, void** out);
int orc_generate_er(int32_t n, double p, uint64_t seed, void** out);
int orc_generate_ba(int32_t n, int32_t m_attach, uint64_t seed, void** out);
int orc_generate_sbm(int32_t n, int32_t k, double p_in, double p_out, uint64_t seed,
                     void** out);
void orc_graph_free(void* g);
void orc_graph_info(void* g, int32_t* n, int64_t* m, int32_t* max_degree);
void orc_graph_csr(void* g, int64_t* offsets, int32_t* nbrs);
/* strip_isolated / connected_components (graph.cpp:180-224); arrays sized n */
int orc_strip_isolated(void* g, void** core, int32_t* core_to_orig, int32_t* orig_to_core,
                       int32_t* removed, int32_t* n_core, int32_t* n_removed);
int orc_components(void* g, int32_t* comp, int32_t* count);
int orc_adjacency_apply(void* g, const double* x, double* y);
int orc_laplacian_apply(void* g, const double* x, double* y);

/* --- Objectives (objectives.hpp) --- */
int orc_validate_objective(int32_t kind, double param);
int orc_gradient(void* g, int32_t kind, double param, const double* x, double* out);
int orc_value(void* g, int32_t kind, double param, const double* x, double* out);
/* returns score; body[n] out */
int orc_extract_solution(void* g, int32_t problem, const double* x, uint8_t* body,
                         int64_t* score);
int64_t orc_cut_value(void* g, const uint8_t* side);
int orc_is_independent(void* g, const uint8_t* indicator);

/* --- PGA (pga.hpp) --- */
int orc_validate_optimizer(double alpha, double beta, int32_t max_iters, double conv_tol,
                           int32_t check_every);
void orc_project(double* x, int32_t n, int32_t problem);
/* one step in place; v has length n (zero-initialised by the caller for a
 * fresh velocity) */
int orc_step(void* g, int32_t kind, double param, double* x, double* v, double alpha,
             double beta);
int orc_run_trajectory(void* g, int32_t kind, double param, double* x, double alpha,
                       double beta, int32_t max_iters, double conv_tol,
                       int32_t check_every, int32_t* iterations, int32_t* reason);
int orc_mis_fixed_point_check(void* g, const double* x, double gamma, double alpha,
                              int32_t* fixed);

/* --- Solver pieces (solver.hpp) --- */
int orc_init_state(void* g, int32_t problem, double sigma, void* rng, double* x);
/* zeroes floor(rho n) coordinates; chosen[] (sorted) gets the vertices;
 * *k gets their count */
int orc_global_reset(double* x, int32_t n, double rho, void* rng, int32_t* chosen,
                     int32_t* k);

/* --- Local search (localsearch.hpp) --- */
int orc_build_tightness(void* g, const uint8_t* indicator, int32_t* tight);
int orc_build_gain_table(void* g, const uint8_t* side, int64_t* delta);
/* indicator in/out; *size out */
int orc_greedy_maximalize(void* g, uint8_t* indicator, int32_t* size);
int orc_one_two_swap(void* g, uint8_t* indicator, int32_t* size);
int orc_one_flip_pass(void* g, uint8_t* side, int64_t* gain);
int orc_two_flip_pass(void* g, uint8_t* side, int64_t* gain);
int orc_one_two_flip(void* g, uint8_t* side, int64_t* gain);

/* --- Engine (solver.cpp run_engine) --- */
int orc_solve_pooled(void* g, const orc_solver_cfg* cfg, orc_report* report,
                     uint8_t* best_body);
/* reference only: the CLI solve / sweep commands (see ref_shim.cpp) */
int orc_cli_run(const char* args);
int orc_preset_for(int32_t problem, int32_t n, double mean_degree, double* alpha,
                   double* momentum, double* rho, int32_t* reset_rounds);

#ifdef __cplusplus
}
#endif

#endif
