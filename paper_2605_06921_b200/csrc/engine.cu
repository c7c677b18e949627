// engine.cu -- the mQO solver engine (reference: run_engine,
// solver.cpp:192-372; solve_pooled / solve_mis / solve_maxcut 376-392) as
// native host orchestration of the device kernels:
//
//   Phase 1  fresh trajectories      init (K3) -> K1/K2 -> harvest (K5/K6)
//   Phase 2  T_gs reset rounds        pick+encode+global_reset (K4) -> K1/K2 -> K5
//   Phase 3  local search over pool   K7/K8
//   final polish of the incumbent
//
// Merges run in global chain order on the host (TopKPool semantics of
// solver.cpp:108-145, 252-275) over packed bodies; only candidates that can
// enter the pool cross PCIe.  With a communicator the B chains are sharded
// over ranks (chain b keeps stream derive_seed(seed, b+1)), every merge
// all-gathers the per-chain records and the needed bodies, and every rank
// replays the identical merge -- results do not depend on the rank count.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <exception>
#include <thread>

#include "common.cuh"
#include "rng.cuh"

using namespace mqo_b200;

namespace mqo_b200 {
void init_states_device(mqo_batch* b, int32_t problem, double sigma);
void init_states_constant(mqo_batch* b, int32_t problem, double c);
void reset_from_pool(mqo_batch* b, int32_t problem, double rho);
void harvest_device(mqo_batch* b, int32_t problem);
void run_trajectories(mqo_batch* b, const mqo_objective& obj, const mqo_optimizer& opt,
                      double deadline);
void read_outcomes(mqo_batch* b, int32_t* iterations, int32_t* reasons);
void launch_project(mqo_batch* b, double* x, int32_t problem);
void upload_chain_major(mqo_batch* b, const double* host, double* dst);
void local_search_device(mqo_batch* b, int32_t op, int32_t count, uint64_t* d_packed,
                         int64_t* d_out, cudaStream_t st, int32_t* d_bad = nullptr);

// init_state (solver.cpp:30-46) on the host with this process's libm, for
// host-only graphs (mqo_init_state_host).  The engine and device graphs use
// K3 (init_states_device).  Consumes `st` exactly like Rng.
void host_init_state(const int64_t* off, int32_t n, int32_t dmax, int32_t problem, double sigma,
                     mqo_rng_state& st, double* x) {
  Xoshiro r{{st.s[0], st.s[1], st.s[2], st.s[3]}};
  const double dm = static_cast<double>(dmax);
  for (int32_t v = 0; v < n; ++v) {
    const double ratio = 1.0 - static_cast<double>(off[v + 1] - off[v]) / dm;
    double base = problem == MQO_PROBLEM_MIS ? ratio : 2.0 * ratio - 1.0;
    if (sigma > 0.0) {  // Rng::normal(0, sigma), rng.hpp:49-62
      double nv;
      if (st.has_spare) {
        st.has_spare = 0;
        nv = 0.0 + sigma * st.spare;
      } else {
        double u1 = u01_of(xoshiro_next(r));
        const double u2 = u01_of(xoshiro_next(r));
        while (u1 <= 0.0) u1 = u01_of(xoshiro_next(r));
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.141592653589793 * u2;
        st.spare = rad * std::sin(theta);
        st.has_spare = 1;
        nv = 0.0 + sigma * rad * std::cos(theta);
      }
      base += nv;
    }
    const double lo = problem == MQO_PROBLEM_MIS ? 0.0 : -1.0;
    const double a = lo < base ? base : lo;
    x[v] = a < 1.0 ? a : 1.0;
  }
  for (int w = 0; w < 4; ++w) st.s[w] = r.s[w];
}

}  // namespace mqo_b200

namespace {

using Clock = std::chrono::steady_clock;

double mono_now() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<double>(ts.tv_sec) + 1e-9 * static_cast<double>(ts.tv_nsec);
}

struct Entry {
  int64_t score = 0;
  std::vector<uint64_t> body;  // packed, W words
};

// body_less (solver.cpp:107-112) on packed bodies.  MaxCut: the side
// vectors compare lexicographically == the packed words compare as
// unsigned integers.  MIS: pool comparisons only ever involve equal scores
// (= equal sizes); then the member list with the lower first differing
// vertex is smaller, i.e. the larger packed word.
bool body_less(int problem, const std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
  for (size_t w = 0; w < a.size(); ++w)
    if (a[w] != b[w]) return problem == MQO_PROBLEM_MAXCUT ? a[w] < b[w] : a[w] > b[w];
  return false;
}

struct TopKPool {  // solver.cpp:121-145
  int k;
  int problem;
  std::vector<Entry> e;
  bool before(const Entry& a, const Entry& b) const {
    if (a.score != b.score) return a.score > b.score;
    return body_less(problem, a.body, b.body);
  }
  bool offer(const Entry& s) {  // returns true if the pool changed
    auto pos = std::lower_bound(e.begin(), e.end(), s,
                                [&](const Entry& x, const Entry& y) { return before(x, y); });
    if (pos != e.end() && pos->score == s.score && pos->body == s.body) return false;
    const size_t idx = static_cast<size_t>(pos - e.begin());
    e.insert(pos, s);
    if (static_cast<int>(e.size()) > k) e.resize(k);
    return idx < e.size();
  }
};

void validate(const mqo_solver_config& c) {  // solver.cpp:14-28
  if (c.objective < 0 || c.objective > 4) throw std::invalid_argument("objective: unknown kind");
  if (c.objective == MQO_MIS_QUBO && !(c.param > 1.0))
    throw std::invalid_argument("mis-qubo: gamma must be > 1");
  if (c.objective == MQO_PERTURBED_LAPLACIAN && !(c.param > 0.0))
    throw std::invalid_argument("perturbed-laplacian: lambda must be > 0");
  if (c.objective == MQO_PERTURBED_BIAS && !(c.param > 0.0 && c.param < 2.0))
    throw std::invalid_argument("perturbed-bias: lambda must be in (0, 2)");
  if (!(c.alpha > 0.0)) throw std::invalid_argument("optimizer: alpha must be > 0");
  if (c.beta < 0.0 || c.beta >= 1.0) throw std::invalid_argument("optimizer: beta must be in [0, 1)");
  if (c.max_iters < 1) throw std::invalid_argument("optimizer: max_iters must be >= 1");
  if (c.conv_tol < 0.0) throw std::invalid_argument("optimizer: conv_tol must be >= 0");
  if (c.check_every < 1) throw std::invalid_argument("optimizer: check_every must be >= 1");
  if (c.reset_fraction < 0.0 || c.reset_fraction >= 1.0)
    throw std::invalid_argument("solver: reset_fraction must be in [0, 1)");
  if (c.reset_rounds < 0) throw std::invalid_argument("solver: reset_rounds must be >= 0");
  if (c.init_noise < 0.0) throw std::invalid_argument("solver: init_noise must be >= 0");
  if (!(c.time_budget_secs > 0.0)) throw std::invalid_argument("solver: time_budget_secs must be > 0");
  if (c.pool_batch < 1 || c.pool_keep < 1)
    throw std::invalid_argument("solver: pool batch and keep must be >= 1");
  if (c.has_max_outer_loops && c.max_outer_loops < 1)
    throw std::invalid_argument("solver: max_outer_loops must be >= 1");
}

// Message of the last failed collective on this thread (set by the native
// communicators in comm.cu; empty for caller-supplied callbacks).
std::string comm_error_text() {
  const char* m = mqo_comm_last_error();
  return m && *m ? std::string(m) : std::string("callback returned an error");
}

// Communicator wrapper (single process when comm == nullptr).
struct Comm {
  const mqo_comm* c;
  int rank() const { return c ? c->rank : 0; }
  int world() const { return c ? c->world : 1; }
  void allgather(const void* send, void* recv, size_t bytes) const {
    if (!c) {
      std::memcpy(recv, send, bytes);
      return;
    }
    if (c->allgather(c->ctx, send, recv, bytes) != 0)
      throw CommError("mqo_comm.allgather failed: " + comm_error_text());
  }
  void allreduce_max(uint64_t* data, size_t count) const {
    if (world() == 1) return;
    if (c->allreduce_max_u64) {
      if (c->allreduce_max_u64(c->ctx, data, count) != 0)
        throw CommError("mqo_comm.allreduce_max_u64 failed: " + comm_error_text());
      return;
    }
    std::vector<uint64_t> all(count * world());
    allgather(data, all.data(), count * sizeof(uint64_t));
    for (int r = 0; r < world(); ++r)
      for (size_t i = 0; i < count; ++i) data[i] = std::max(data[i], all[r * count + i]);
  }
  void broadcast(void* buf, size_t bytes, int root) const {
    if (world() == 1) return;
    if (c->broadcast) {
      if (c->broadcast(c->ctx, buf, bytes, root) != 0)
        throw CommError("mqo_comm.broadcast failed: " + comm_error_text());
      return;
    }
    std::vector<uint8_t> all(bytes * world());
    allgather(buf, all.data(), bytes);
    std::memcpy(buf, all.data() + bytes * root, bytes);
  }
};

struct Engine {
  mqo_graph* g;
  mqo_solver_config cfg;
  Comm comm;
  int problem;
  int32_t n;
  int64_t W;
  int B_global, B_local, first_chain;
  int chain_offset = 0;  // single-process engines: first global chain (Mode R shards)
  int rank_id = -1;      // Mode R: the outer rank of this shard engine
  uint64_t* stage = nullptr;  // pinned staging for local-search bodies
  size_t stage_words = 0;
  ~Engine() { pinned_put(stage, sizeof(uint64_t) * stage_words); }
  mqo_batch* batch = nullptr;
  TopKPool pool;
  Entry best;
  bool have_best = false;
  bool pool_dirty = true;
  mqo_run_report rep{};
  int64_t best_of_gradient = 0, best_of_resets = 0, best_of_ls = 0;
  double t0 = 0.0, deadline = 0.0;
  // per-merge gathered records (global chain order)
  std::vector<int64_t> g_scores;
  std::vector<int32_t> g_valid, g_iters, g_stops;

  // Failure handling across ranks.  Local device work of a rank runs
  // through local(): an exception is parked in `pending` instead of leaving
  // the engine, the rank skips further local work but still joins the next
  // collective with an error flag, and every rank then throws at the same
  // point -- a failure on one rank can never leave its peers blocked in a
  // collective.  Single-process engines rethrow immediately.
  std::exception_ptr pending;
  const int fault_rank = [] {
    const char* e = std::getenv("MQO_FAULT_RANK");
    return e && *e ? std::atoi(e) : -1;
  }();
  template <typename F>
  void local(F&& f) {
    if (pending) return;
    try {
      f();
    } catch (...) {
      if (comm.world() == 1) throw;
      pending = std::current_exception();
    }
  }
  void raise_if(bool any_failed) {
    if (!any_failed) return;
    if (pending) std::rethrow_exception(pending);
    throw PeerFailed("mqo: a peer rank failed; the collective solve was aborted on every rank");
  }

  // Deadline decisions are collective: any rank past the deadline stops
  // every rank at the same point, so the ranks' merge sequences never
  // diverge (each decision is one tiny all-gather, which also carries the
  // error flag).
  bool past_deadline() {
    const uint8_t mine = (mono_now() >= deadline ? 1 : 0) | (pending ? 2 : 0);
    if (comm.world() == 1) return mine != 0;
    std::vector<uint8_t> all(comm.world());
    comm.allgather(&mine, all.data(), 1);
    bool past = false, failed = false;
    for (uint8_t a : all) {
      past |= (a & 1) != 0;
      failed |= (a & 2) != 0;
    }
    raise_if(failed);
    return past;
  }
  bool target_hit() const {
    return have_best && cfg.has_stop_at_score && best.score >= cfg.stop_at_score;
  }

  // Phase-1 init (solver.cpp:283-289): init_constant or init_state, both
  // on the device; the Box-Muller noise replays the reference's glibc
  // log / sincos bit for bit (glibc_math.cuh), so there is no host path.
  void init_phase() {
    if (cfg.has_init_constant) {
      init_states_constant(batch, problem, cfg.init_constant);
      return;
    }
    init_states_device(batch, problem, cfg.init_noise);
  }

  void trajectories() {
    const mqo_objective obj{cfg.objective, cfg.param};
    const mqo_optimizer opt{cfg.alpha, cfg.beta, cfg.max_iters, cfg.conv_tol, cfg.check_every};
    launch_project(batch, batch->d_x[batch->cur], problem);
    run_trajectories(batch, obj, opt, deadline);
  }

  // Gathers this phase's per-chain records in global chain order and the
  // bodies of the candidates that can touch the pool, then merges
  // (solver.cpp:252-275).
  void harvest_and_merge(bool count_resets) {
    std::vector<int32_t> iters(B_local), stops(B_local), dep(B_local);
    std::vector<int64_t> scores(B_local);
    local([&] {
      harvest_device(batch, problem);
      read_outcomes(batch, iters.data(), stops.data());
      MQO_CUDA(cudaMemcpyAsync(scores.data(), batch->d_scores, sizeof(int64_t) * B_local,
                               cudaMemcpyDeviceToHost, batch->stream));
      MQO_CUDA(cudaMemcpyAsync(dep.data(), batch->d_valid, sizeof(int32_t) * B_local,
                               cudaMemcpyDeviceToHost, batch->stream));
      MQO_CUDA(cudaStreamSynchronize(batch->stream));
    });
    // record = {score, valid, iters, stop} for every local chain, padded,
    // after one header word carrying this rank's error flag
    const int world = comm.world();
    const int per = (B_global + world - 1) / world;
    const size_t stride = static_cast<size_t>(per) * 4 + 1;
    std::vector<int64_t> rec(stride, 0), all(rec.size() * world);
    rec[0] = pending ? 1 : 0;
    for (int i = 0; i < B_local && !pending; ++i) {
      rec[1 + 4 * i] = scores[i];
      rec[1 + 4 * i + 1] = problem == MQO_PROBLEM_MIS ? (dep[i] ? 0 : 1) : 1;
      rec[1 + 4 * i + 2] = iters[i];
      rec[1 + 4 * i + 3] = stops[i];
    }
    comm.allgather(rec.data(), all.data(), rec.size() * sizeof(int64_t));
    bool failed = false;
    for (int r = 0; r < world; ++r) failed |= all[r * stride] != 0;
    raise_if(failed);
    g_scores.assign(B_global, 0);
    g_valid.assign(B_global, 0);
    g_iters.assign(B_global, 0);
    g_stops.assign(B_global, 0);
    for (int r = 0; r < world; ++r)
      for (int i = 0; i < per; ++i) {
        const int b = r * per + i;
        if (b >= B_global) break;
        const int64_t* q = all.data() + static_cast<size_t>(r) * stride + 1 + static_cast<size_t>(i) * 4;
        g_scores[b] = q[0];
        g_valid[b] = static_cast<int32_t>(q[1]);
        g_iters[b] = static_cast<int32_t>(q[2]);
        g_stops[b] = static_cast<int32_t>(q[3]);
      }
    // candidates that can change the pool or the incumbent: score >= the
    // pool's current worst when it is full (the worst only rises during a
    // merge, so this start-of-merge threshold is conservative)
    const bool full = static_cast<int>(pool.e.size()) >= pool.k;
    const int64_t thr = full ? pool.e.back().score : INT64_MIN;
    auto needed = [&](int b) { return g_valid[b] && (g_scores[b] >= thr || !have_best); };
    std::vector<std::vector<uint64_t>> bodies(B_global);
    // local bodies
    std::vector<int> mine;
    for (int i = 0; i < B_local; ++i)
      if (needed(first_chain + i)) mine.push_back(i);
    std::vector<uint64_t> local(static_cast<size_t>(mine.size()) * W);
    for (size_t k = 0; k < mine.size(); ++k)
      MQO_CUDA(cudaMemcpyAsync(local.data() + k * W, batch->d_bodies + static_cast<int64_t>(mine[k]) * W,
                               sizeof(uint64_t) * W, cudaMemcpyDeviceToHost, batch->stream));
    MQO_CUDA(cudaStreamSynchronize(batch->stream));
    if (world == 1) {
      for (size_t k = 0; k < mine.size(); ++k)
        bodies[mine[k]].assign(local.begin() + k * W, local.begin() + (k + 1) * W);
    } else {
      // every rank knows every rank's needed set from the gathered records
      std::vector<int> cnt(world, 0);
      int maxc = 0;
      for (int b = 0; b < B_global; ++b)
        if (needed(b)) maxc = std::max(maxc, ++cnt[b / per]);
      std::vector<uint64_t> send(static_cast<size_t>(std::max(maxc, 1)) * W, 0),
          recv(send.size() * world);
      std::copy(local.begin(), local.end(), send.begin());
      comm.allgather(send.data(), recv.data(), send.size() * sizeof(uint64_t));
      for (int r = 0; r < world; ++r) {
        int k = 0;
        for (int i = 0; i < per; ++i) {
          const int b = r * per + i;
          if (b >= B_global || !needed(b)) continue;
          const uint64_t* src = recv.data() + (static_cast<size_t>(r) * send.size()) + k * W;
          bodies[b].assign(src, src + W);
          ++k;
        }
      }
    }
    for (int b = 0; b < B_global; ++b) {
      rep.total_iterations += g_iters[b];
      rep.last_trajectory_stop = g_stops[b];
      ++rep.trajectories;
      if (!g_valid[b]) continue;
      const int64_t sc = g_scores[b];
      if (count_resets)
        best_of_resets = std::max(best_of_resets, sc);
      else
        best_of_gradient = std::max(best_of_gradient, sc);
      const bool better = !have_best || sc > best.score;
      if (!needed(b)) {  // cannot enter a full pool: offer is a no-op
        if (count_resets) ++rep.resets_rejected;
        continue;
      }
      Entry e{sc, std::move(bodies[b])};
      if (pool.offer(e)) pool_dirty = true;
      if (better) {
        best = std::move(e);
        have_best = true;
        if (count_resets) ++rep.resets_accepted;
      } else if (count_resets) {
        ++rep.resets_rejected;
      }
    }
  }

  void upload_pool() {
    if (!pool_dirty) return;
    std::vector<uint64_t> packed(pool.e.size() * W);
    for (size_t i = 0; i < pool.e.size(); ++i)
      std::copy(pool.e[i].body.begin(), pool.e[i].body.end(), packed.begin() + i * W);
    if (mqo_set_pool(batch, static_cast<int32_t>(pool.e.size()), packed.data()) != MQO_OK)
      throw CudaError(mqo_last_error());
    pool_dirty = false;
  }

  // Polishes `members` bodies with one_two_swap / one_two_flip on the
  // device (solver.cpp:318-327); scores updated like the reference.
  void polish(std::vector<Entry>& members) {
    if (members.empty()) return;
    const int count = static_cast<int>(members.size());
    uint64_t* d_packed = nullptr;
    int64_t* d_out = nullptr;
    cudaStream_t st = batch->stream;
    MQO_TRACE("polish: %d bodies", count);
    // one pinned staging buffer: [count][W] bodies + [count] outputs
    const size_t words = static_cast<size_t>(count) * W;
    if (stage_words < words + count) {
      pinned_put(stage, sizeof(uint64_t) * stage_words);
      stage = static_cast<uint64_t*>(pinned_get(sizeof(uint64_t) * (words + count)));
      stage_words = words + count;
    }
    for (int i = 0; i < count; ++i) std::copy(members[i].body.begin(), members[i].body.end(), stage + i * W);
    MQO_CUDA(cudaMallocAsync(&d_packed, sizeof(uint64_t) * (words + count), st));
    d_out = reinterpret_cast<int64_t*>(d_packed + words);
    MQO_CUDA(cudaMemcpyAsync(d_packed, stage, sizeof(uint64_t) * words, cudaMemcpyHostToDevice, st));
    const int op = problem == MQO_PROBLEM_MIS ? MQO_LS_ONE_TWO_SWAP : MQO_LS_ONE_TWO_FLIP;
    local_search_device(batch, op, count, d_packed, d_out, st);
    MQO_CUDA(cudaMemcpyAsync(stage, d_packed, sizeof(uint64_t) * (words + count),
                             cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(d_packed, st);
    MQO_CUDA(cudaStreamSynchronize(st));
    MQO_TRACE("polish: %d bodies done", count);
    const int64_t* out = reinterpret_cast<const int64_t*>(stage + words);
    for (int i = 0; i < count; ++i) {
      std::copy(stage + i * W, stage + (i + 1) * W, members[i].body.begin());
      members[i].score = problem == MQO_PROBLEM_MIS ? out[i] : members[i].score + out[i];
    }
  }

  // Phase-3 polish with the pool members dealt round-robin over the ranks,
  // results all-gathered back (identical on every rank).
  void polish_sharded(std::vector<Entry>& members) {
    const int world = comm.world(), rank = comm.rank();
    if (world == 1) return polish(members);
    const int count = static_cast<int>(members.size());
    std::vector<Entry> mine;
    for (int i = rank; i < count; i += world) mine.push_back(members[i]);
    local([&] { polish(mine); });
    const int per = (count + world - 1) / world;
    const size_t rec = 1 + static_cast<size_t>(W);  // score + body words
    const size_t stride = 1 + static_cast<size_t>(per) * rec;  // error flag + records
    std::vector<uint64_t> send(stride, 0), recv(send.size() * world);
    send[0] = pending ? 1 : 0;
    for (size_t k = 0; k < mine.size() && !pending; ++k) {
      send[1 + k * rec] = static_cast<uint64_t>(mine[k].score);
      std::copy(mine[k].body.begin(), mine[k].body.end(), send.begin() + 1 + k * rec + 1);
    }
    comm.allgather(send.data(), recv.data(), send.size() * sizeof(uint64_t));
    bool failed = false;
    for (int r = 0; r < world; ++r) failed |= recv[r * stride] != 0;
    raise_if(failed);
    for (int i = 0; i < count; ++i) {
      const int r = i % world, k = i / world;
      const uint64_t* src = recv.data() + static_cast<size_t>(r) * stride + 1 + static_cast<size_t>(k) * rec;
      members[i].score = static_cast<int64_t>(src[0]);
      members[i].body.assign(src + 1, src + rec);
    }
  }

  void run() {
    validate(cfg);
    problem = cfg.objective == MQO_MIS_QUBO ? MQO_PROBLEM_MIS : MQO_PROBLEM_MAXCUT;
    t0 = mono_now();
    deadline = t0 + cfg.time_budget_secs;
    rep = mqo_run_report{};
    rep.last_trajectory_stop = MQO_ITER_CAP;
    n = g->n;
    if (n == 0) throw std::invalid_argument("solver: empty graph");
    W = body_words(n);
    pool.k = cfg.pool_keep;
    pool.problem = problem;
    if (g->m == 0) {  // solver.cpp:221-226, trivial_solution 176-189
      rep.warnings |= MQO_WARN_EDGELESS;
      best.body.assign(W, 0);
      if (problem == MQO_PROBLEM_MIS) {
        for (int32_t v = 0; v < n; ++v) best.body[v >> 6] |= 1ull << (63 - (v & 63));
        best.score = n;
      }
      best_of_gradient = best.score;
      have_best = true;
      return finish();
    }
    if (cfg.reset_rounds > 0 && static_cast<int32_t>(std::floor(cfg.reset_fraction * n)) == 0)
      rep.warnings |= MQO_WARN_RESET_NOOP;

    B_global = cfg.pool_batch;
    const int world = comm.world(), rank = comm.rank();
    const int per = (B_global + world - 1) / world;
    first_chain = std::min(B_global, rank * per);
    B_local = std::max(0, std::min(B_global, first_chain + per) - first_chain);
    if (B_local < 1) throw std::invalid_argument("solver: more ranks than chains");
    try {
      local([&] {
        if (mqo_batch_create(g, B_local, &batch) != MQO_OK) throw CudaError(mqo_last_error());
        if (mqo_batch_seed_streams(batch, cfg.seed,
                                   1 + static_cast<uint64_t>(first_chain + chain_offset)) != MQO_OK)
          throw CudaError(mqo_last_error());
      });
      loop();
    } catch (...) {
      if (batch) mqo_batch_free(batch);
      batch = nullptr;
      throw;
    }
    mqo_batch_free(batch);
    batch = nullptr;
    finish();
  }

  void loop() {
    const mqo_objective obj{cfg.objective, cfg.param};
    (void)obj;
    while (!past_deadline() && !target_hit()) {
      if (cfg.has_max_outer_loops && rep.outer_loops >= cfg.max_outer_loops) break;
      // Phase 1 (solver.cpp:280-296)
      MQO_TRACE("outer %d: init", rep.outer_loops);
      local([&] {
        init_phase();
        MQO_TRACE("outer %d: trajectories", rep.outer_loops);
        trajectories();
      });
      MQO_TRACE("outer %d: harvest", rep.outer_loops);
      harvest_and_merge(false);
      // Phase 2 (298-312)
      for (int round = 0; round < cfg.reset_rounds; ++round) {
        if (past_deadline() || target_hit() || pool.e.empty()) break;
        MQO_TRACE("round %d: reset", round);
        local([&] {
          if (fault_rank == (rank_id >= 0 ? rank_id : comm.rank()))  // MQO_FAULT_RANK (tests)
            throw std::runtime_error("injected fault on rank " + std::to_string(fault_rank));
          upload_pool();
          reset_from_pool(batch, problem, cfg.reset_fraction);
          MQO_TRACE("round %d: trajectories", round);
          trajectories();
        });
        MQO_TRACE("round %d: harvest", round);
        harvest_and_merge(true);
      }
      // Phase 3 (314-339)
      if (cfg.local_search && !pool.e.empty() && !past_deadline() && !target_hit()) {
        std::vector<Entry> polished = pool.e;
        MQO_TRACE("outer %d: local search", rep.outer_loops);
        polish_sharded(polished);
        for (auto& s : polished) {
          best_of_ls = std::max(best_of_ls, s.score);
          const bool better = !have_best || s.score > best.score;
          if (pool.offer(s)) pool_dirty = true;
          if (better) {
            best = s;
            have_best = true;
          }
        }
      }
      ++rep.outer_loops;
    }
    // final polish (344-359)
    MQO_TRACE("final polish");
    if (cfg.local_search && have_best) {
      std::vector<Entry> p{best};
      polish(p);
      best_of_ls = std::max(best_of_ls, p[0].score);
      if (pool.offer(p[0])) pool_dirty = true;
      if (p[0].score > best.score) best = p[0];
    }
    if (!have_best) {  // 361-370
      rep.warnings |= MQO_WARN_NO_SOLUTION;
      best.body.assign(W, 0);
      best.score = 0;
    }
  }

  void finish() {  // 209-219
    rep.found_solution = have_best ? 1 : 0;
    rep.score = best.score;
    rep.after_gradient = best_of_gradient;
    rep.after_reset_loop = std::max(best_of_gradient, best_of_resets);
    rep.after_local_search = std::max(rep.after_reset_loop, best_of_ls);
    rep.elapsed_secs = mono_now() - t0;
    rep.n_warnings = __builtin_popcount(static_cast<unsigned>(rep.warnings));
  }
};

}  // namespace

namespace {

void solve_pooled_impl(mqo_graph* g, const mqo_solver_config* cfg, const mqo_comm* comm,
                       mqo_run_report* report, uint8_t* best_body) {
    if (!g || !cfg || !report) throw std::invalid_argument("mqo_solve_pooled: null argument");
    if (g->device >= 0) MQO_CUDA(cudaSetDevice(g->device));
    Engine e;
    e.g = g;
    e.cfg = *cfg;
    e.comm = Comm{comm};
    e.run();
    *report = e.rep;
    if (best_body) {
      for (int32_t v = 0; v < g->n; ++v)
        best_body[v] = e.best.body.empty() ? 0 : (e.best.body[v >> 6] >> (63 - (v & 63))) & 1;
    }
}

void solve_replicas_impl(mqo_graph* g, const mqo_solver_config* cfg, const mqo_comm* comm,
                         mqo_run_report* report, uint8_t* best_body, int64_t* rank_scores) {
    if (!g || !cfg || !report) throw std::invalid_argument("mqo_solve_replicas: null argument");
    if (g->device >= 0) MQO_CUDA(cudaSetDevice(g->device));
    const Comm cm{comm};
    const int world = cm.world(), rank = cm.rank();
    validate(*cfg);
    const int per = (cfg->pool_batch + world - 1) / world;
    const int first = std::min(cfg->pool_batch, rank * per);
    const int local = std::max(0, std::min(cfg->pool_batch, first + per) - first);
    if (local < 1) throw std::invalid_argument("solver: more ranks than chains");
    Engine e;  // an independent single-process solver over this rank's shard
    e.g = g;
    e.cfg = *cfg;
    e.cfg.pool_batch = local;
    e.comm = Comm{nullptr};
    e.chain_offset = first;
    e.rank_id = rank;
    // a local failure still joins the all-reduce (error word), so no peer
    // is left waiting; then every rank throws
    std::exception_ptr failure;
    try {
      e.run();
    } catch (...) {
      if (world == 1) throw;
      failure = std::current_exception();
    }
    // the one exchange: argmax over ranks (a single tiny all-reduce)
    const int64_t sc = !failure && e.rep.found_solution ? e.best.score : -1;
    uint64_t key[2] = {(static_cast<uint64_t>(sc + 1) << 16) | static_cast<uint64_t>(0xFFFF - rank),
                       failure ? 1ull : 0ull};
    cm.allreduce_max(key, 2);
    if (key[1]) {
      if (failure) std::rethrow_exception(failure);
      throw PeerFailed("mqo: a peer rank failed; the replica solve was aborted on every rank");
    }
    const int winner = 0xFFFF - static_cast<int>(key[0] & 0xFFFF);
    // counters: the winner's report, sums / maxima over ranks
    mqo_run_report mine = e.rep;
    std::vector<mqo_run_report> all(world);
    cm.allgather(&mine, all.data(), sizeof(mqo_run_report));
    mqo_run_report r = all[winner];
    r.outer_loops = r.trajectories = 0;
    r.resets_accepted = r.resets_rejected = r.total_iterations = 0;
    r.elapsed_secs = 0.0;
    r.warnings = 0;
    for (const auto& a : all) {
      r.trajectories += a.trajectories;
      r.resets_accepted += a.resets_accepted;
      r.resets_rejected += a.resets_rejected;
      r.total_iterations += a.total_iterations;
      r.outer_loops = std::max(r.outer_loops, a.outer_loops);
      r.after_gradient = std::max(r.after_gradient, a.after_gradient);
      r.after_reset_loop = std::max(r.after_reset_loop, a.after_reset_loop);
      r.after_local_search = std::max(r.after_local_search, a.after_local_search);
      r.elapsed_secs = std::max(r.elapsed_secs, a.elapsed_secs);
      r.warnings |= a.warnings;
    }
    r.n_warnings = __builtin_popcount(static_cast<unsigned>(r.warnings));
    if (rank_scores)
      for (int q = 0; q < world; ++q) rank_scores[q] = all[q].found_solution ? all[q].score : -1;
    std::vector<uint64_t> body(e.W > 0 ? e.W : 1, 0);
    if (rank == winner && !e.best.body.empty()) std::copy(e.best.body.begin(), e.best.body.end(), body.begin());
    cm.broadcast(body.data(), sizeof(uint64_t) * body.size(), winner);
    *report = r;
    if (best_body)
      for (int32_t v = 0; v < g->n; ++v) best_body[v] = (body[v >> 6] >> (63 - (v & 63))) & 1;
}

}  // namespace

extern "C" int mqo_solve_pooled(mqo_graph* g, const mqo_solver_config* cfg, const mqo_comm* comm,
                                mqo_run_report* report, uint8_t* best_body) {
  return guard([&] { solve_pooled_impl(g, cfg, comm, report, best_body); });
}

extern "C" int mqo_solve_replicas(mqo_graph* g, const mqo_solver_config* cfg, const mqo_comm* comm,
                                  mqo_run_report* report, uint8_t* best_body,
                                  int64_t* rank_scores) {
  return guard([&] { solve_replicas_impl(g, cfg, comm, report, best_body, rank_scores); });
}

extern "C" int mqo_solve_devices(mqo_graph* g, const mqo_solver_config* cfg, const int32_t* devices,
                                 int32_t ndev, int32_t mode, mqo_run_report* report,
                                 uint8_t* best_body, int64_t* rank_scores) {
  return guard([&] {
    if (!g || !cfg || !report || !devices || ndev < 1)
      throw std::invalid_argument("mqo_solve_devices: bad argument");
    if (mode != MQO_SOLVE_POOLED && mode != MQO_SOLVE_REPLICAS)
      throw std::invalid_argument("mqo_solve_devices: unknown mode");
    validate(*cfg);
    if (ndev > cfg->pool_batch) throw std::invalid_argument("solver: more ranks than chains");
    if (ndev == 1 && devices[0] == g->device) {
      if (mode == MQO_SOLVE_POOLED) return solve_pooled_impl(g, cfg, nullptr, report, best_body);
      return solve_replicas_impl(g, cfg, nullptr, report, best_body, rank_scores);
    }
    bool distinct = true;
    for (int i = 0; i < ndev; ++i)
      for (int j = 0; j < i; ++j) distinct &= devices[i] != devices[j];
    // per-rank graphs: g itself on its own device, else a copy of its CSR
    std::vector<mqo_graph*> graphs(ndev, nullptr), owned;
    std::vector<mqo_comm*> comms(ndev, nullptr);
    auto cleanup = [&] {
      for (mqo_comm* c : comms)
        if (c) mqo_comm_free(c);
      for (mqo_graph* q : owned) mqo_graph_free(q);
    };
    try {
      for (int r = 0; r < ndev; ++r) {
        if (devices[r] == g->device) {
          graphs[r] = g;
          continue;
        }
        for (int q = 0; q < r && !graphs[r]; ++q)
          if (devices[q] == devices[r]) graphs[r] = graphs[q];
        if (graphs[r]) continue;
        mqo_graph* copy = nullptr;
        host_csr(g);
        if (mqo_graph_upload(g->n, g->h_off.data(), g->h_nbr.data(), devices[r], &copy) != MQO_OK)
          throw CudaError(mqo_last_error());
        owned.push_back(copy);
        graphs[r] = copy;
      }
      const int rc = distinct ? mqo_comm_create_devices(ndev, devices, comms.data())
                              : mqo_comm_create_local(ndev, comms.data());
      if (rc != MQO_OK) throw CommError(mqo_last_error());
      std::vector<std::exception_ptr> errors(ndev);
      std::vector<mqo_run_report> reports(ndev);
      std::vector<std::thread> threads;
      for (int r = 0; r < ndev; ++r)
        threads.emplace_back([&, r] {
          try {
            MQO_CUDA(cudaSetDevice(devices[r]));
            // ranks sharing a GPU: the SMEM/cluster trajectory kernel is left
            // out (an intermittent fault with another rank's work in flight,
            // DESIGN.md section 8); the per-pass kernels give the same report
            static const bool allow = [] {  // MQO_SHARED_CTA=1: keep it (stress runs)
              const char* e = std::getenv("MQO_SHARED_CTA");
              return e && *e == '1';
            }();
            g_tls_no_cta_traj = !distinct && !allow;
            if (mode == MQO_SOLVE_POOLED)
              solve_pooled_impl(graphs[r], cfg, comms[r], &reports[r], r == 0 ? best_body : nullptr);
            else
              solve_replicas_impl(graphs[r], cfg, comms[r], &reports[r],
                                  r == 0 ? best_body : nullptr, r == 0 ? rank_scores : nullptr);
          } catch (...) {
            errors[r] = std::current_exception();
          }
        });
      for (auto& t : threads) t.join();
      // the failing rank's own error, not a peer's "a peer rank failed"
      std::exception_ptr first;
      for (auto& e : errors) {
        if (!e) continue;
        try {
          std::rethrow_exception(e);
        } catch (const PeerFailed&) {
          if (!first) first = e;
        } catch (...) {
          std::rethrow_exception(e);
        }
      }
      if (first) std::rethrow_exception(first);
      *report = reports[0];
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    if (g->device >= 0) MQO_CUDA(cudaSetDevice(g->device));
  });
}

extern "C" int mqo_init_state_host(const mqo_graph* g, int32_t problem, double sigma,
                                   mqo_rng_state* st, double* x) {
  return guard([&] {
    if (!g || !st || !x) throw std::invalid_argument("mqo_init_state_host: null argument");
    if (g->n == 0) throw std::invalid_argument("init_state: empty graph");
    if (g->max_degree < 1)
      throw std::invalid_argument("init_state: edgeless graph (strip isolated vertices upstream)");
    host_csr(g);
    host_init_state(g->h_off.data(), g->n, g->max_degree, problem, sigma, *st, x);
  });
}
