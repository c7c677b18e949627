// Per-call latency of single-vector C-ABI calls (the reference's one-vector
// shape) without any Python in the loop.
//   g++ -O2 -std=c++17 -Iinclude scripts/abi_latency.cpp -Lpaper_2605_06921_b200 -lmqo_b200 \
//       -Wl,-rpath,$PWD/paper_2605_06921_b200 -o /tmp/abi_latency && /tmp/abi_latency 1024
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "mqo_gpu.h"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 1024;
  mqo_gen_spec spec{};
  spec.kind = MQO_GEN_ER;
  spec.n = n;
  spec.p = 16.0 / n;
  spec.seed = 1;
  mqo_graph* g = nullptr;
  if (mqo_generate(&spec, 0, &g)) return std::printf("%s\n", mqo_last_error()), 1;
  mqo_batch* b = nullptr;
  if (mqo_batch_create(g, 1, &b)) return std::printf("%s\n", mqo_last_error()), 1;
  std::vector<double> x(n, 0.5), y(n);
  mqo_batch_set_x(b, x.data());
  mqo_objective obj{MQO_ADJACENCY, 0.0};
  for (int i = 0; i < 100; ++i) mqo_gradient(b, &obj, y.data());
  const int reps = 2000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) mqo_gradient(b, &obj, y.data());
  const double us =
      std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
  std::printf("n=%d mqo_gradient B=1: %.2f us/call (y[0]=%g)\n", n, us, y[0]);
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) mqo_batch_set_x(b, x.data());
  std::printf("n=%d mqo_batch_set_x B=1: %.2f us/call\n", n,
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps);
  mqo_batch_free(b);
  mqo_graph_free(g);
  return 0;
}
