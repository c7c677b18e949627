/*
 * mqo_gpu.h -- the C ABI of the B200-native mQO inner loop
 * (libmqo_b200.so, built from paper_2605_06921_b200/csrc).
 *
 * This is the drop-in boundary under the reference's C++ API
 * (/root/reference/proj/core/include/mqo/).  Plain pointers, sizes and POD
 * structs only: no torch or C++ types, no exceptions cross it.  Every entry
 * point returns MQO_OK (0) or an error code, with mqo_last_error() holding a
 * thread-local message; MQO_ERR_INVALID / MQO_ERR_LOGIC correspond to the
 * reference's std::invalid_argument / std::logic_error (and carry the same
 * messages), so a C++ facade can rethrow them unchanged.
 *
 * Each declaration cites the reference interface it replaces (file:line,
 * relative to /root/reference/proj/core/).  Layouts: a "batch" holds B
 * chains (independent trajectories) of one graph on one device.  Host
 * state buffers are chain-major, B rows of n doubles -- chain b is exactly
 * the reference's std::vector<double> RelaxedState::x (objectives.hpp:45-48).
 * On the device the batch is stored vertex-major (X[v][B_pad]) so that a
 * neighbour gather of all chains is one coalesced row read.
 */
#ifndef MQO_GPU_H
#define MQO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status --------------------------------------------------------- */
enum {
  MQO_OK = 0,
  MQO_ERR_INVALID = 1, /* std::invalid_argument in the reference */
  MQO_ERR_LOGIC = 2,   /* std::logic_error in the reference */
  MQO_ERR_CUDA = 3,
  MQO_ERR_NCCL = 4,
  MQO_ERR_OTHER = 5,
  MQO_ERR_PARSE = 6 /* mqo::ParseError (graph_io.hpp:13-21), a std::runtime_error */
};

/* Thread-local message of the last failing call on this thread. */
const char* mqo_last_error(void);
/* 1-based line of the last MQO_ERR_PARSE on this thread (ParseError::line,
 * graph_io.hpp:17), else 0. */
int32_t mqo_last_error_line(void);
/* Library identification, e.g. "mqo_b200 0.1 sm_100a". */
const char* mqo_version(void);

/* ---- enums mirroring the reference ------------------------------------ */
/* ObjectiveSpec alternatives, objectives.hpp:22-35 (variant index order). */
enum {
  MQO_MIS_QUBO = 0,
  MQO_LAPLACIAN = 1,
  MQO_PERTURBED_LAPLACIAN = 2,
  MQO_ADJACENCY = 3,
  MQO_PERTURBED_BIAS = 4
};
/* Problem, objectives.hpp:12. */
enum { MQO_PROBLEM_MIS = 0, MQO_PROBLEM_MAXCUT = 1 };
/* StopReason, pga.hpp:23. */
enum { MQO_CONVERGED = 0, MQO_CHECKER_ACCEPTED = 1, MQO_ITER_CAP = 2 };

/* ObjectiveSpec (objectives.hpp:22-35): kind + gamma/lambda. */
typedef struct {
  int32_t kind;
  double param; /* MisQubo::gamma, PerturbedLaplacian/PerturbedBias::lambda */
} mqo_objective;

/* OptimizerConfig (pga.hpp:13-19). */
typedef struct {
  double alpha;
  double beta;
  int32_t max_iters;
  double conv_tol;
  int32_t check_every;
} mqo_optimizer;

/* ---- graph store (graph.hpp:20-63) ------------------------------------
 * Uploads an immutable CSR (int64 offsets[n+1], int32 neighbours[2m], rows
 * strictly ascending, no self loops, symmetric) to `device`.  The
 * invariants of Graph::check_invariants (graph.cpp:44-56) and symmetry are
 * verified -- on the device for device graphs, on host threads for
 * host-only ones -- and the first violation in (row, entry) order returns
 * MQO_ERR_LOGIC / MQO_ERR_INVALID with the reference's message.

 * device < 0 keeps a host-only graph (CSR readable, no batches).
 * Replaces: Graph storage + Graph::from_edges's output (graph.cpp:8-42). */
typedef struct mqo_graph mqo_graph;
int mqo_graph_upload(int32_t n, const int64_t* offsets, const int32_t* neighbors,
                     int32_t device, mqo_graph** out);
int mqo_graph_free(mqo_graph* g);
int mqo_graph_info(const mqo_graph* g, int32_t* n, int64_t* m, int32_t* max_degree);
/* Copies the canonical CSR back (offsets[n+1], neighbors[2m]). */
int mqo_graph_csr(const mqo_graph* g, int64_t* offsets, int32_t* neighbors);
/* The kernels' row schedule of a device graph: vertices by degree
 * descending, ties by id (order[n]).  Diagnostic; no reference
 * counterpart. */
int mqo_graph_row_order(const mqo_graph* g, int32_t* order);

/* Graph::from_edges (graph.hpp:26, graph.cpp:8-42): edges in any order and
 * orientation, duplicates collapsed, self loops rejected
 * (MQO_ERR_INVALID, reference messages); canonical CSR uploaded. */
int mqo_graph_from_edges(int32_t n, int64_t num_edges, const int32_t* eu, const int32_t* ev,
                         int32_t device, mqo_graph** out);

/* GraphGenSpec (graph.hpp:67-91) and generate() (graph.cpp:169-178):
 * bit-identical graphs to the reference for the same (spec, seed). */
/* MQO_GEN_ER_FAST: O(m) G(n,p) by geometric skipping -- a different draw
 * sequence from the reference's O(n^2) ER (graph.cpp:107-116, infeasible at
 * n = 1e7); used for the large configs, with the edge list then fed to both
 * sides. */
/* MQO_GEN_SBM_FAST: O(m) stochastic block model (geometric skipping over
 * the p_in and p_out pair runs of each row; the reference's distribution,
 * not its O(n^2) draw sequence, graph.cpp:148-165). */
enum { MQO_GEN_ER = 0, MQO_GEN_BA = 1, MQO_GEN_SBM = 2, MQO_GEN_ER_FAST = 3, MQO_GEN_SBM_FAST = 4 };
typedef struct {
  int32_t kind;
  int32_t n;
  double p;         /* ErSpec::p */
  int32_t m_attach; /* BaSpec::m_attach */
  int32_t k;        /* SbmSpec::k */
  double p_in, p_out;
  uint64_t seed;
} mqo_gen_spec;
int mqo_generate(const mqo_gen_spec* spec, int32_t device, mqo_graph** out);

/* Graph files (graph_io.cpp:74-106): format 0 = binary CSR cache
 * ("MQOCSR01" n m offsets neighbours), 1 = the reference's canonical text
 * ("n m" + one "u v" line per edge, u < v).  mqo_graph_load sniffs the
 * format -- binary magic, DIMACS by a leading 'c' or 'p' (graph_io.cpp:98),
 * else canonical -- and uploads to `device` (< 0: host-only); text errors
 * are MQO_ERR_PARSE with the reference's "line N: ..." message.
 * Replaces: Graph load_graph_file(path, warnings*) (graph_io.hpp:45),
 * void write_graph_file(g, path) (46). */
int mqo_graph_save(const mqo_graph* g, const char* path, int32_t format);
int mqo_graph_load(const char* path, int32_t device, mqo_graph** out);
/* Parse an in-memory graph text: format 0 = sniff (as mqo_graph_load),
 * 1 = canonical (read_canonical, graph_io.hpp:41), 2 = DIMACS edge format
 * (parse_dimacs, graph_io.hpp:35; *declared_edges = the 'p' line's m, may
 * be NULL).  Replaces: DimacsResult parse_dimacs(istream&) /
 * parse_dimacs_text(const string&) (graph_io.hpp:35-36), Graph
 * read_canonical(istream&) (41). */
int mqo_graph_parse(const char* text, int64_t len, int32_t format, int32_t device,
                    int64_t* declared_edges, mqo_graph** out);
/* Warnings of the last mqo_graph_load / mqo_graph_parse on this thread
 * (DimacsResult::warnings, e.g. "declared m=2 but parsed m=1 after
 * deduplication"), '\n'-separated; returns the full length, copies at most
 * cap-1 bytes + NUL into buf (buf may be NULL when cap == 0). */
int64_t mqo_graph_load_warnings(char* buf, int64_t cap);

/* Device pre-processing on a graph in HBM.
 * strip_isolated (graph.hpp:95-104, graph.cpp:180-198): *core = the graph
 * without its degree-0 vertices (same device); caller-sized arrays of n:
 * core_to_orig (first *n_core used), orig_to_core (-1 for removed vertices),
 * removed (ascending, first *n_removed used); any array may be NULL.
 * Replaces: StripResult strip_isolated(const Graph&). */
int mqo_graph_strip_isolated(const mqo_graph* g, mqo_graph** core, int32_t* core_to_orig,
                             int32_t* orig_to_core, int32_t* removed, int32_t* n_core,
                             int32_t* n_removed);
/* connected_components (graph.hpp:106, graph.cpp:200-224): comp[v] = index
 * of v's component, components numbered in the reference's output order
 * (by smallest vertex); *count = number of components.  The reference's
 * sorted member lists are the stable grouping of v by comp[v].
 * Replaces: std::vector<std::vector<Vertex>> connected_components(const Graph&). */
int mqo_graph_components(const mqo_graph* g, int32_t* comp, int32_t* count);

/* ---- chain batch -------------------------------------------------------
 * A batch of `chains` relaxed states (RelaxedState, objectives.hpp:45-48)
 * plus velocities, the per-chain xoshiro streams and control words, on the
 * graph's device, with its own CUDA stream. */
typedef struct mqo_batch mqo_batch;
int mqo_batch_create(mqo_graph* g, int32_t chains, mqo_batch** out);
int mqo_batch_free(mqo_batch* b);
int mqo_batch_chains(const mqo_batch* b, int32_t* chains, int32_t* padded);
/* The cudaStream_t the batch launches on (for event timing by callers). */
int mqo_batch_stream(const mqo_batch* b, void** stream);
/* Blocks until all work queued on the batch stream has finished. */
int mqo_batch_sync(mqo_batch* b);

/* Host <-> device state copies.  x / v are chain-major [chains][n]
 * doubles (chain b = the reference's std::vector<double>). */
int mqo_batch_set_x(mqo_batch* b, const double* x);
int mqo_batch_get_x(mqo_batch* b, double* x);
int mqo_batch_set_v(mqo_batch* b, const double* v);
int mqo_batch_get_v(mqo_batch* b, double* v);
/* Zeroes every velocity (the fresh `velocity` of run_trajectory,
 * pga.cpp:75). */
int mqo_batch_zero_v(mqo_batch* b);

/* project() on every chain (pga.cpp:47-49, clamp pga.cpp:31-34). */
int mqo_project(mqo_batch* b, int32_t problem);

/* gradient() of every chain at its current x, written chain-major to the
 * host buffer `out` [chains][n] (objectives.cpp:101-134; the dominant SpMV
 * is Graph::adjacency_apply / laplacian_apply, graph.cpp:63-88). */
int mqo_gradient(mqo_batch* b, const mqo_objective* obj, double* out);

/* step() on every chain, in place on the device state: v = beta v + grad,
 * x = clamp(x + alpha v) (pga.cpp:51-61).  Asynchronous on the batch
 * stream; bit-identical to the reference for every chain. */
int mqo_step(mqo_batch* b, const mqo_objective* obj, const mqo_optimizer* opt);

/* run_trajectory() on every chain from its current x (pga.cpp:63-111):
 * projects, zeroes the velocity, iterates the fused step with the MIS
 * fixed-point checker (pga.cpp:91-98,113-135) or the MaxCut ||dx||_inf stop
 * (pga.cpp:99-102) until each chain stops.  `deadline_secs` is an absolute
 * CLOCK_MONOTONIC time (<0: none) polled every 256 iterations like
 * pga.cpp:104-107.  On return the device x of chain b is its
 * TrajectoryOutcome::state; iterations[b] / reasons[b] (host arrays, may be
 * NULL) receive TrajectoryOutcome::iterations / reason. */
int mqo_run_trajectories(mqo_batch* b, const mqo_objective* obj, const mqo_optimizer* opt,
                         double deadline_secs, int32_t* iterations, int32_t* reasons);

/* mis_fixed_point_check() on every chain's current (binary) x
 * (pga.cpp:113-135).  fixed[b] in {0,1}.  Returns MQO_ERR_INVALID with the
 * reference message when a state is not binary or gamma/alpha are out of
 * range. */
int mqo_mis_fixed_point_check(mqo_batch* b, double gamma, double alpha, int32_t* fixed);

/* Tuning knobs of the fused kernels, for measurement scripts:
 * "k1_variant" (K1 instantiation, 0 = default) and "hot_frac" (fraction of
 * L2 kept for gathers of hot rows).  Not needed for normal use. */
int mqo_tune(const char* key, double value);

/* ---- per-chain random streams (rng.hpp:13-86) ---------------------------
 * The complete state of an mqo::Rng: xoshiro256** words plus the cached
 * Box-Muller spare.  Chain b of a batch owns one stream. */
typedef struct {
  uint64_t s[4];
  double spare;
  int32_t has_spare;
  int32_t flags; /* internal */
} mqo_rng_state;
/* Chain b <- Rng(derive_seed(master_seed, first_stream + b)); the solver
 * uses first_stream = 1 (solver.cpp:234-236). */
int mqo_batch_seed_streams(mqo_batch* b, uint64_t master_seed, uint64_t first_stream);
int mqo_batch_get_streams(mqo_batch* b, mqo_rng_state* out);
int mqo_batch_set_streams(mqo_batch* b, const mqo_rng_state* in);

/* ---- K3 init_state (solver.cpp:30-46) ----------------------------------
 * x_b = Pi(d_base + N(0, sigma^2)) drawn from chain b's stream in vertex
 * order (Box-Muller, rng.hpp:49-62), replayed segment-parallel on the
 * device.  sigma == 0 draws nothing.  Box-Muller's log / sincos are device
 * replays of the host glibc 2.39 routines the reference calls (__log_fma,
 * __sincos_fma; csrc/glibc_math.cuh): bit-identical to init_state. */
int mqo_init_states(mqo_batch* b, int32_t problem, double sigma);
/* The init_constant path (solver.cpp:283-287): x = Pi(c 1), no draws. */
int mqo_init_constant(mqo_batch* b, int32_t problem, double c);

/* ---- K4 conditional reset -----------------------------------------------
 * global_reset (solver.cpp:48-63) on every chain's current x: zeroes the
 * floor(rho n) coordinates a partial Fisher-Yates over chain b's stream
 * picks -- bit-identical draws and chosen sets, resolved in parallel. */
int mqo_global_reset(mqo_batch* b, double rho);
/* The device copy of the TopK pool: `count` packed bodies of
 * ceil(n/64) words each (bit 63-(v%64) of word v/64 = vertex v). */
int mqo_set_pool(mqo_batch* b, int32_t count, const uint64_t* packed);
/* One reset round start (solver.cpp:301-303): chain b draws
 * pool.at(uniform_index(pool.size())), encodes it (encode_solution,
 * solver.cpp:147-160) and applies global_reset.  picks[b] (may be NULL)
 * receives the drawn pool index. */
int mqo_reset_from_pool(mqo_batch* b, int32_t problem, double rho, int32_t* picks);

/* ---- K5/K6 harvest (solver.cpp:166-175) ---------------------------------
 * extract_solution (objectives.cpp:143-161) of every chain's current x;
 * MIS: is_independent (173-180) -> valid[b] = 0 when dependent (the
 * reference discards it), else greedy_maximalize (localsearch.cpp:35-56);
 * MaxCut: cut_value (163-171).  scores[b], valid[b] and the packed bodies
 * [chains][ceil(n/64)] (each may be NULL) are written to host memory. */
int mqo_harvest(mqo_batch* b, int32_t problem, int64_t* scores, int32_t* valid,
                uint64_t* packed);

/* extract_solution (objectives.cpp:143-161) without repair: MIS members are
 * x > 0.5 (score |I|; independent[b] = is_independent, 173-180), MaxCut
 * sides x > 0 (score cut_value, 163-171).  Any output may be NULL. */
int mqo_extract(mqo_batch* b, int32_t problem, int64_t* scores, int32_t* independent,
                uint64_t* packed);

/* build_gain_table (kind 0, localsearch.cpp:17-26) or build_tightness
 * (kind 1, 9-15) for `count` packed bodies; out = int32 [count][n]. */
int mqo_build_tables(mqo_batch* b, int32_t kind, int32_t count, const uint64_t* packed,
                     int32_t* out);

/* ---- K7/K8 local search (localsearch.hpp:28-48) ---------------------------
 * Runs `op` on `count` packed bodies (host, [count][ceil(n/64)], updated in
 * place) on the batch's device (a CTA per body, or grid-wide rounds for one
 * large body), with the reference's exact index-ordered first-improvement
 * commits:
 *   MQO_LS_ONE_FLIP     one_flip_pass  (localsearch.cpp:139-157), out = gain
 *   MQO_LS_TWO_FLIP     two_flip_pass  (159-181),                 out = gain
 *   MQO_LS_ONE_TWO_FLIP one_two_flip   (183-190),                 out = gain
 *   MQO_LS_ONE_TWO_SWAP one_two_swap   (88-137),                  out = |I|
 * one_two_swap rejects a non-maximal or dependent input with
 * MQO_ERR_INVALID and the reference's message (the first offending body in
 * order); `packed` and `out` are then left untouched. */
enum { MQO_LS_ONE_FLIP = 0, MQO_LS_TWO_FLIP = 1, MQO_LS_ONE_TWO_FLIP = 2, MQO_LS_ONE_TWO_SWAP = 3 };
int mqo_local_search(mqo_batch* b, int32_t op, int32_t count, uint64_t* packed, int64_t* out);

/* ---- the solver engine (solver.hpp:11-80, run_engine solver.cpp:192-372) -- */
/* init_state noise source.  Both values select the device kernel K3,
 * which is bit-identical to the reference (glibc log / sincos replayed on
 * the device); the field is kept for ABI compatibility with round-1
 * callers (EXACT used to run Box-Muller on host threads). */
enum { MQO_INIT_EXACT = 0, MQO_INIT_DEVICE = 1 };
/* RunReport::warnings (solver.cpp:222,230,362), as bits in emission order. */
enum { MQO_WARN_EDGELESS = 1, MQO_WARN_RESET_NOOP = 2, MQO_WARN_NO_SOLUTION = 4 };

/* SolverConfig (solver.hpp:17-36) + device placement. */
typedef struct {
  int32_t objective; /* MQO_MIS_QUBO ... MQO_PERTURBED_BIAS */
  double param;      /* gamma / lambda */
  double alpha, beta;
  int32_t max_iters;
  double conv_tol;
  int32_t check_every;
  double reset_fraction; /* rho */
  int32_t reset_rounds;  /* T_gs */
  double init_noise;     /* sigma */
  double time_budget_secs;
  uint64_t seed;
  int32_t local_search;
  int32_t pool_batch, pool_keep; /* B, K */
  int32_t has_init_constant;
  double init_constant;
  int32_t has_stop_at_score;
  int64_t stop_at_score;
  int32_t has_max_outer_loops;
  int32_t max_outer_loops;
  int32_t init_mode; /* ignored: init is always the bit-exact device K3 */
} mqo_solver_config;

/* RunReport (solver.hpp:42-61); the best body goes to a separate buffer. */
typedef struct {
  int64_t score;
  int32_t found_solution;
  int64_t after_gradient, after_reset_loop, after_local_search;
  int32_t outer_loops, trajectories;
  int64_t resets_accepted, resets_rejected, total_iterations;
  int32_t last_trajectory_stop;
  double elapsed_secs;
  int32_t n_warnings;
  int32_t warnings; /* MQO_WARN_* bits */
} mqo_run_report;

/* Optional communicator for sharding the B chains over ranks (one process
 * per GPU).  allgather: every rank contributes `bytes` from `send`; `recv`
 * receives world * bytes in rank order.  allreduce_max_u64 (in place,
 * element-wise max over ranks) and broadcast (`bytes` of `buf` from rank
 * `root` to all) are used by mqo_solve_replicas; either may be NULL, and is
 * then emulated with allgather.  Return 0 on success. */
typedef struct {
  void* ctx;
  int32_t rank, world;
  int (*allgather)(void* ctx, const void* send, void* recv, size_t bytes);
  int (*allreduce_max_u64)(void* ctx, uint64_t* data, size_t count);
  int (*broadcast)(void* ctx, void* buf, size_t bytes, int32_t root);
} mqo_comm;

/* Native communicators, replacing the caller
 * callbacks above for GPU runs.  NCCL is loaded at first use (dlopen of
 * libnccl.so.2); its failures and a failed peer rank are MQO_ERR_NCCL with
 * the message in mqo_last_error() (and, for a failed collective inside a
 * callback, mqo_comm_last_error()).  Communicators are freed with
 * mqo_comm_free.
 *   mqo_nccl_unique_id     rank 0 creates the id; ship it to the other ranks
 *                          out of band (torch.distributed, MPI, a file)
 *   mqo_comm_nccl_create   one process per GPU: this process's rank
 *   mqo_comm_create_devices  one process driving `ndev` distinct GPUs
 *                          (ncclCommInitAll); out[ndev]
 *   mqo_comm_create_local  `world` ranks that are host threads of this
 *                          process, exchanging through host memory (ranks
 *                          sharing one GPU, where NCCL refuses); out[world]
 * Replaces: the reference's in-process parallel_for over chains
 * (solver.cpp:78-106), whose results are thread-count independent
 * (tests/test_solver.cpp:221-233). */
#define MQO_NCCL_ID_BYTES 128
int mqo_nccl_unique_id(uint8_t* id /* [MQO_NCCL_ID_BYTES] */);
int mqo_comm_nccl_create(int32_t rank, int32_t world, const uint8_t* id, int32_t device,
                         mqo_comm** out);
int mqo_comm_create_devices(int32_t ndev, const int32_t* devices, mqo_comm** out);
int mqo_comm_create_local(int32_t world, mqo_comm** out);
int mqo_comm_free(mqo_comm* c);
/* Message of the last failed native collective on this thread ("" if none). */
const char* mqo_comm_last_error(void);

/* solve_pooled (solver.hpp:80): runs the engine on `g`'s device.
 * best_body (may be NULL) receives the best solution as uint8[n]
 * (MIS indicator / MaxCut side).  With comm != NULL rank r owns chains
 * [r*ceil(B/world), ...) and every rank returns the identical report.
 * solve_mis / solve_maxcut are solve_pooled with the reference's guards. */
int mqo_solve_pooled(mqo_graph* g, const mqo_solver_config* cfg, const mqo_comm* comm,
                     mqo_run_report* report, uint8_t* best_body);

/* "Mode R": every rank runs an independent pooled
 * solver over its chain shard [r*ceil(B/world), ...) -- chain b keeps stream
 * derive_seed(seed, b+1) -- with no exchange while solving; then ONE
 * allreduce-max over the packed key (score << 16 | 0xFFFF - rank) selects
 * the best rank (ties: lowest rank) and its body is broadcast.  The report
 * is the winner's with trajectories / iterations / resets summed and phase
 * maxima taken over ranks; rank_scores (may be NULL) receives every rank's
 * best score.  Cheaper than mqo_solve_pooled's per-round merge, but not
 * equal to the single-GPU B-chain run (each rank keeps its own pool).
 * With comm == NULL it is mqo_solve_pooled. */
int mqo_solve_replicas(mqo_graph* g, const mqo_solver_config* cfg, const mqo_comm* comm,
                       mqo_run_report* report, uint8_t* best_body, int64_t* rank_scores);

/* One process, several GPUs: solve_pooled (mode MQO_SOLVE_POOLED, "Mode P":
 * the report equals the single-GPU B-chain run) or the replica solve (mode
 * MQO_SOLVE_REPLICAS, "Mode R") of `g` over `devices[ndev]`, one host thread
 * per GPU.  Rank r runs on devices[r] with its own copy of the graph
 * (uploaded from g's host CSR unless devices[r] is g's device) and chains
 * [r*ceil(B/ndev), ...).  Distinct devices exchange over NCCL
 * (ncclCommInitAll); repeated devices fall back to the in-process exchange
 * (tests on one GPU).  rank_scores (may be NULL, MQO_SOLVE_REPLICAS only)
 * receives every rank's best score.  A failure on any rank fails the call
 * on every rank (the first rank's error is returned). */
enum { MQO_SOLVE_POOLED = 0, MQO_SOLVE_REPLICAS = 1 };
int mqo_solve_devices(mqo_graph* g, const mqo_solver_config* cfg, const int32_t* devices,
                      int32_t ndev, int32_t mode, mqo_run_report* report, uint8_t* best_body,
                      int64_t* rank_scores);

/* init_state on the host for one stream with this process's libm, for
 * host-only graphs (device < 0): x[n] out, *st advanced like Rng.  Graphs in
 * HBM use mqo_init_states (the facade's init_state does). */
int mqo_init_state_host(const mqo_graph* g, int32_t problem, double sigma, mqo_rng_state* st,
                        double* x);

#ifdef __cplusplus
}
#endif

#endif /* MQO_GPU_H */
