// comm.cu -- native communicators for sharding the engine's B chains over
// GPUs (the reference's only parallelism is the
// parallel_for over chains, solver.cpp:78-106, whose result-independence
// contract is tests/test_solver.cpp:221-233).
//
//   * NCCL over NVLink / NVSwitch: one rank per GPU, either one process per
//     GPU (mqo_comm_nccl_create with a unique id shipped out of band) or all
//     GPUs of one process (mqo_comm_create_devices -> ncclCommInitAll, one
//     host thread per GPU).  The engine's collectives are tiny (per-chain
//     records, a few packed bodies, one argmax key), so they are staged
//     through pinned host memory into a per-rank device buffer and run on the
//     rank's own stream: ncclAllGather / ncclAllReduce(max) / ncclBroadcast.
//   * An in-process exchange (mqo_comm_create_local) for ranks that are host
//     threads sharing one device -- NCCL refuses two ranks on one GPU; used
//     by the single-GPU tests of the multi-rank engine.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: torch's bundled
// copy when torch is already loaded, else the system one), so the library
// itself has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "common.cuh"

using namespace mqo_b200;

namespace {

thread_local std::string g_comm_error;

int comm_fail(const std::string& msg) {
  g_comm_error = msg;
  return MQO_ERR_NCCL;
}

// ------------------------------------------------------------ NCCL loader
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      api.error = std::string("NCCL not available: ") + dlerror();
      return;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + s;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.error.empty()) throw CommError(api.error);
  return api;
}

#define MQO_NCCL(expr)                                                             \
  do {                                                                             \
    ncclResult_t _r = (expr);                                                      \
    if (_r != ncclSuccess)                                                         \
      throw CommError(std::string(#expr) + ": " + nccl().GetErrorString(_r));      \
  } while (0)

// ------------------------------------------------------------- NCCL ranks
struct NcclRank {
  ncclComm_t comm = nullptr;
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  uint8_t* dbuf = nullptr;  // device staging
  size_t dcap = 0;
  uint8_t* hbuf = nullptr;  // pinned staging
  size_t hcap = 0;
  ~NcclRank() {
    if (comm) nccl().CommDestroy(comm);
    if (dbuf) cudaFree(dbuf);
    if (hbuf) cudaFreeHost(hbuf);
    if (stream) cudaStreamDestroy(stream);
  }
  void reserve(size_t bytes) {
    if (dcap < bytes) {
      if (dbuf) MQO_CUDA(cudaFree(dbuf));
      dbuf = nullptr;
      MQO_CUDA(cudaMalloc(&dbuf, bytes));
      dcap = bytes;
    }
    if (hcap < bytes) {
      if (hbuf) MQO_CUDA(cudaFreeHost(hbuf));
      hbuf = nullptr;
      MQO_CUDA(cudaMallocHost(&hbuf, bytes));
      hcap = bytes;
    }
  }
};

template <typename F>
int comm_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return comm_fail(e.what());
  }
}

// recv[world * bytes] <- every rank's send[bytes], in rank order
int nccl_allgather(void* ctx, const void* send, void* recv, size_t bytes) {
  return comm_guard([&] {
    auto* r = static_cast<NcclRank*>(ctx);
    MQO_CUDA(cudaSetDevice(r->device));
    const size_t total = bytes * static_cast<size_t>(r->world);
    r->reserve(bytes + total);
    uint8_t* dsend = r->dbuf;
    uint8_t* drecv = r->dbuf + bytes;
    std::memcpy(r->hbuf, send, bytes);
    MQO_CUDA(cudaMemcpyAsync(dsend, r->hbuf, bytes, cudaMemcpyHostToDevice, r->stream));
    MQO_NCCL(nccl().AllGather(dsend, drecv, bytes, ncclUint8, r->comm, r->stream));
    MQO_CUDA(cudaMemcpyAsync(r->hbuf, drecv, total, cudaMemcpyDeviceToHost, r->stream));
    MQO_CUDA(cudaStreamSynchronize(r->stream));
    std::memcpy(recv, r->hbuf, total);
  });
}

// element-wise max over ranks, in place
int nccl_allreduce_max(void* ctx, uint64_t* data, size_t count) {
  return comm_guard([&] {
    auto* r = static_cast<NcclRank*>(ctx);
    MQO_CUDA(cudaSetDevice(r->device));
    const size_t bytes = count * sizeof(uint64_t);
    r->reserve(bytes);
    std::memcpy(r->hbuf, data, bytes);
    MQO_CUDA(cudaMemcpyAsync(r->dbuf, r->hbuf, bytes, cudaMemcpyHostToDevice, r->stream));
    MQO_NCCL(nccl().AllReduce(r->dbuf, r->dbuf, count, ncclUint64, ncclMax, r->comm, r->stream));
    MQO_CUDA(cudaMemcpyAsync(r->hbuf, r->dbuf, bytes, cudaMemcpyDeviceToHost, r->stream));
    MQO_CUDA(cudaStreamSynchronize(r->stream));
    std::memcpy(data, r->hbuf, bytes);
  });
}

int nccl_broadcast(void* ctx, void* buf, size_t bytes, int32_t root) {
  return comm_guard([&] {
    auto* r = static_cast<NcclRank*>(ctx);
    MQO_CUDA(cudaSetDevice(r->device));
    r->reserve(bytes);
    std::memcpy(r->hbuf, buf, bytes);
    MQO_CUDA(cudaMemcpyAsync(r->dbuf, r->hbuf, bytes, cudaMemcpyHostToDevice, r->stream));
    MQO_NCCL(nccl().Broadcast(r->dbuf, r->dbuf, bytes, ncclUint8, root, r->comm, r->stream));
    MQO_CUDA(cudaMemcpyAsync(r->hbuf, r->dbuf, bytes, cudaMemcpyDeviceToHost, r->stream));
    MQO_CUDA(cudaStreamSynchronize(r->stream));
    std::memcpy(buf, r->hbuf, bytes);
  });
}

// ---------------------------------------------------- in-process ranks
// Host threads of one process exchanging through shared memory: a
// generation barrier around each all-gather (write own slot, barrier, read,
// and a leading barrier so no rank overwrites the buffer while a peer still
// reads the previous collective).
struct LocalHub {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<uint8_t> buf;
  void barrier() {
    std::unique_lock<std::mutex> lock(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return gen != g; });
    }
  }
};

struct LocalRank {
  std::shared_ptr<LocalHub> hub;
  int rank = 0;
};

int local_allgather(void* ctx, const void* send, void* recv, size_t bytes) {
  return comm_guard([&] {
    auto* r = static_cast<LocalRank*>(ctx);
    LocalHub& h = *r->hub;
    const size_t total = bytes * static_cast<size_t>(h.world);
    h.barrier();
    {
      std::lock_guard<std::mutex> lock(h.mu);
      if (h.buf.size() < total) h.buf.resize(total);
      std::memcpy(h.buf.data() + bytes * static_cast<size_t>(r->rank), send, bytes);
    }
    h.barrier();
    std::memcpy(recv, h.buf.data(), total);
  });
}

// the mqo_comm handed out owns its rank state through `ctx`
struct OwnedComm {
  mqo_comm c{};
  std::unique_ptr<NcclRank> nccl_rank;
  std::unique_ptr<LocalRank> local_rank;
};

mqo_comm* wrap_nccl(std::unique_ptr<NcclRank> r) {
  auto* o = new OwnedComm;
  o->c.ctx = r.get();
  o->c.rank = r->rank;
  o->c.world = r->world;
  o->c.allgather = nccl_allgather;
  o->c.allreduce_max_u64 = nccl_allreduce_max;
  o->c.broadcast = nccl_broadcast;
  o->nccl_rank = std::move(r);
  return &o->c;
}

}  // namespace

extern "C" const char* mqo_comm_last_error(void) { return g_comm_error.c_str(); }

extern "C" int mqo_nccl_unique_id(uint8_t* id) {
  return guard([&] {
    if (!id) throw std::invalid_argument("mqo_nccl_unique_id: null id");
    ncclUniqueId u;
    MQO_NCCL(nccl().GetUniqueId(&u));
    static_assert(sizeof(u.internal) == MQO_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, u.internal, MQO_NCCL_ID_BYTES);
  });
}

extern "C" int mqo_comm_nccl_create(int32_t rank, int32_t world, const uint8_t* id, int32_t device,
                                    mqo_comm** out) {
  return guard([&] {
    if (!id || !out) throw std::invalid_argument("mqo_comm_nccl_create: null argument");
    if (world < 1 || rank < 0 || rank >= world)
      throw std::invalid_argument("mqo_comm_nccl_create: rank out of range");
    ncclUniqueId u;
    std::memcpy(u.internal, id, MQO_NCCL_ID_BYTES);
    auto r = std::make_unique<NcclRank>();
    r->device = device;
    r->rank = rank;
    r->world = world;
    MQO_CUDA(cudaSetDevice(device));
    MQO_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    MQO_NCCL(nccl().CommInitRank(&r->comm, world, u, rank));
    *out = wrap_nccl(std::move(r));
  });
}

extern "C" int mqo_comm_create_devices(int32_t ndev, const int32_t* devices, mqo_comm** out) {
  return guard([&] {
    if (ndev < 1 || !devices || !out) throw std::invalid_argument("mqo_comm_create_devices: bad argument");
    for (int i = 0; i < ndev; ++i)
      for (int j = 0; j < i; ++j)
        if (devices[i] == devices[j])
          throw std::invalid_argument("mqo_comm_create_devices: NCCL needs distinct devices "
                                      "(use mqo_comm_create_local for ranks sharing a GPU)");
    std::vector<ncclComm_t> comms(ndev);
    MQO_NCCL(nccl().CommInitAll(comms.data(), ndev, devices));
    for (int i = 0; i < ndev; ++i) {
      auto r = std::make_unique<NcclRank>();
      r->comm = comms[i];
      r->device = devices[i];
      r->rank = i;
      r->world = ndev;
      MQO_CUDA(cudaSetDevice(devices[i]));
      MQO_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
      out[i] = wrap_nccl(std::move(r));
    }
  });
}

extern "C" int mqo_comm_create_local(int32_t world, mqo_comm** out) {
  return guard([&] {
    if (world < 1 || !out) throw std::invalid_argument("mqo_comm_create_local: bad argument");
    auto hub = std::make_shared<LocalHub>();
    hub->world = world;
    for (int i = 0; i < world; ++i) {
      auto* o = new OwnedComm;
      o->local_rank = std::make_unique<LocalRank>();
      o->local_rank->hub = hub;
      o->local_rank->rank = i;
      o->c.ctx = o->local_rank.get();
      o->c.rank = i;
      o->c.world = world;
      o->c.allgather = local_allgather;  // max / broadcast are derived from it
      out[i] = &o->c;
    }
  });
}

extern "C" int mqo_comm_free(mqo_comm* c) {
  return guard([&] {
    if (!c) return;
    delete reinterpret_cast<OwnedComm*>(c);  // c is the first member of OwnedComm
  });
}
