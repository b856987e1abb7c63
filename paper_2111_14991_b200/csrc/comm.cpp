// Transports of candidate-axis sharding (gtc_comm.hpp, include/gridtune_cuda.h
// "candidate-axis sharding").  The reference has no multi-device path; the
// exchange it needs is the one SURVEY.md §8(e) derives from
// strategies.hpp:404-418 (global mean variance -> lambda) and
// portfolio.hpp:32-61 (argmax over the union of the shards).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/gridtune_cuda.h"
#include "gtc_comm.hpp"

extern "C" void gtc_internal_set_error(const char* msg);

namespace {

int comm_fail(int code, const std::string& msg) {
  gtc_internal_set_error(msg.c_str());
  return code;
}

#define COMM_CUDA(call)                                                                              \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return comm_fail(GTC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---- NCCL, opened at run time --------------------------------------------------
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // an already loaded libnccl (e.g. torch's) is found by its soname first
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) {
      const char* e = dlerror();
      a.error = std::string("NCCL unavailable: ") + (e ? e : "libnccl.so.2 not found");
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(a.handle, name));
      if (!fn && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.AllGather, "ncclAllGather");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.CommCount, "ncclCommCount");
    sym(a.CommUserRank, "ncclCommUserRank");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const NcclApi& a = nccl();
  return comm_fail(GTC_ERR_CUDA, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error"));
}

struct NcclComm final : gtc_comm {
  ncclComm_t comm = nullptr;
  bool owned = false;
  ~NcclComm() override {
    if (owned && comm) nccl().CommDestroy(comm);
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) override {
    const ncclResult_t r = nccl().AllGather(send, recv, bytes, ncclUint8, comm, stream);
    return r == ncclSuccess ? GTC_OK : nccl_fail(r, "ncclAllGather");
  }
  const char* kind() const override { return "nccl"; }
};

// ---- in-process group: peer copies ordered by CUDA events ------------------------
// Every member thread calls allgather once per exchange (like an NCCL rank):
// it records "ready" after its send buffer, meets the others at a host
// barrier, pulls every member's buffer with peer copies after that member's
// "ready", records "done", meets them again and makes its stream wait for
// every member's "done" -- so no member overwrites its send buffer (next
// iteration) before every copy of it has landed.  Only enqueues; the host
// threads run ahead of the devices like NCCL's.
struct LocalShared {
  explicit LocalShared(int n) : n(n), send(n, nullptr), device(n, 0), ready(n, nullptr), done(n, nullptr) {}
  ~LocalShared() {
    for (cudaEvent_t e : ready)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : done)
      if (e) cudaEventDestroy(e);
  }
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  bool broken = false;
  std::vector<const void*> send;
  std::vector<int> device;
  std::vector<cudaEvent_t> ready, done;

  // false when a member left the group or the wait timed out
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const unsigned long long g = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != g || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
  void abandon() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

struct LocalComm final : gtc_comm {
  std::shared_ptr<LocalShared> sh;
  ~LocalComm() override {
    if (sh) sh->abandon();
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) override {
    LocalShared& s = *sh;
    int dev = 0;
    COMM_CUDA(cudaGetDevice(&dev));
    if (!s.ready[rank]) {
      COMM_CUDA(cudaEventCreateWithFlags(&s.ready[rank], cudaEventDisableTiming));
      COMM_CUDA(cudaEventCreateWithFlags(&s.done[rank], cudaEventDisableTiming));
    }
    s.send[rank] = send;
    s.device[rank] = dev;
    COMM_CUDA(cudaEventRecord(s.ready[rank], stream));
    if (!s.barrier()) return comm_fail(GTC_ERR_CUDA, "local shard group: a member left or timed out");
    unsigned char* out = static_cast<unsigned char*>(recv);
    for (int i = 0; i < s.n; ++i) {
      COMM_CUDA(cudaStreamWaitEvent(stream, s.ready[i], 0));
      if (s.device[i] == dev)
        COMM_CUDA(cudaMemcpyAsync(out + (size_t)i * bytes, s.send[i], bytes, cudaMemcpyDeviceToDevice, stream));
      else
        COMM_CUDA(cudaMemcpyPeerAsync(out + (size_t)i * bytes, dev, s.send[i], s.device[i], bytes, stream));
    }
    COMM_CUDA(cudaEventRecord(s.done[rank], stream));
    if (!s.barrier()) return comm_fail(GTC_ERR_CUDA, "local shard group: a member left or timed out");
    for (int i = 0; i < s.n; ++i)
      if (i != rank) COMM_CUDA(cudaStreamWaitEvent(stream, s.done[i], 0));
    return GTC_OK;
  }
  const char* kind() const override { return "local"; }
};

}  // namespace

extern "C" int gtc_comm_nccl_id(uint8_t* id_out) {
  if (!id_out) return comm_fail(GTC_ERR_INVALID, "null argument");
  const NcclApi& a = nccl();
  if (!a.error.empty()) return comm_fail(GTC_ERR_CUDA, a.error);
  ncclUniqueId id;
  const ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == GTC_NCCL_ID_BYTES, "NCCL unique id size");
  std::memcpy(id_out, &id, sizeof id);
  return GTC_OK;
}

extern "C" int gtc_comm_create_nccl(const uint8_t* id, int32_t rank, int32_t nranks, int32_t device,
                                    gtc_comm** out) {
  if (!id || !out) return comm_fail(GTC_ERR_INVALID, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return comm_fail(GTC_ERR_INVALID, "bad rank / nranks");
  const NcclApi& a = nccl();
  if (!a.error.empty()) return comm_fail(GTC_ERR_CUDA, a.error);
  COMM_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  auto c = std::make_unique<NcclComm>();
  const ncclResult_t r = a.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  c->owned = true;
  c->rank = rank;
  c->nranks = nranks;
  *out = c.release();
  return GTC_OK;
}

extern "C" int gtc_comm_wrap_nccl(void* nccl_comm, gtc_comm** out) {
  if (!nccl_comm || !out) return comm_fail(GTC_ERR_INVALID, "null argument");
  const NcclApi& a = nccl();
  if (!a.error.empty()) return comm_fail(GTC_ERR_CUDA, a.error);
  auto c = std::make_unique<NcclComm>();
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  ncclResult_t r = a.CommUserRank(c->comm, &c->rank);
  if (r == ncclSuccess) r = a.CommCount(c->comm, &c->nranks);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommUserRank/ncclCommCount");
  *out = c.release();
  return GTC_OK;
}

extern "C" int gtc_comm_create_local(int32_t nranks, gtc_comm** out) {
  if (!out || nranks < 1) return comm_fail(GTC_ERR_INVALID, "bad arguments");
  auto sh = std::make_shared<LocalShared>(nranks);
  for (int i = 0; i < nranks; ++i) {
    auto* c = new LocalComm();
    c->sh = sh;
    c->rank = i;
    c->nranks = nranks;
    out[i] = c;
  }
  return GTC_OK;
}

extern "C" int gtc_comm_destroy(gtc_comm* c) {
  delete c;
  return GTC_OK;
}

extern "C" int32_t gtc_comm_rank(const gtc_comm* c) { return c ? c->rank : -1; }
extern "C" int32_t gtc_comm_size(const gtc_comm* c) { return c ? c->nranks : -1; }
