// mem.cu -- allocation helpers that keep driver calls off the solve path.
//
// * Pinned host blocks (mapped, portable) come from a process-wide cache:
//   cudaHostAlloc / cudaFreeHost cost milliseconds and cudaFreeHost
//   synchronises the device, and the engine needs a few small pinned
//   buffers per solve (batch control words, local-search staging).
// * Graph arrays are allocated stream-ordered from the device's memory pool
//   on a per-device stream (mqo_graph_upload / free): cudaMalloc /
//   cudaFree map and unmap pages and cudaFree synchronises the device.
#include <map>
#include <mutex>

#include "common.cuh"

namespace mqo_b200 {

namespace {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;  // size -> block
}  // namespace

void* pinned_get(size_t bytes) {
  bytes = std::max<size_t>(64, (bytes + 63) / 64 * 64);
  {
    std::lock_guard<std::mutex> lock(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= 4 * bytes) {
      void* p = it->second;
      g_pin_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  MQO_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  return p;
}

void pinned_put(void* p, size_t bytes) {
  if (!p) return;
  bytes = std::max<size_t>(64, (bytes + 63) / 64 * 64);
  std::lock_guard<std::mutex> lock(g_pin_mu);
  g_pin_free.emplace(bytes, p);
}

cudaStream_t mem_stream(int device) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {nullptr};
  std::lock_guard<std::mutex> lock(mu);
  if (!streams[device]) {
    keep_pool_memory(device);
    MQO_CUDA(cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking));
  }
  return streams[device];
}

}  // namespace mqo_b200
