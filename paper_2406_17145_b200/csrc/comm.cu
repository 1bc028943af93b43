// NCCL transport for the stage executor: stage-edge P2P pieces and the per-iteration
// DP all-reduce, driven from the C-ABI so the per-rank iteration (kernels + transfers)
// can be captured into one CUDA graph.  NCCL is resolved at run time from the already
// loaded libnccl.so.2 (the one PyTorch ships) — no link-time dependency.
#include <dlfcn.h>

#include <cstring>

#include <mutex>
#include <string>

#include "common.cuh"

namespace gpp {
namespace {

typedef struct { char internal[128]; } UniqueId;  // == ncclUniqueId
typedef void* Comm;                                 // == ncclComm_t
enum { NCCL_UINT8 = 1, NCCL_FLOAT32 = 7, NCCL_SUM = 0 };

struct Nccl {
  int (*getUniqueId)(UniqueId*) = nullptr;
  int (*commInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*commDestroy)(Comm) = nullptr;
  int (*send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  const char* (*getErrorString)(int) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.getUniqueId = reinterpret_cast<int (*)(UniqueId*)>(dlsym(h, "ncclGetUniqueId"));
    n.commInitRank = reinterpret_cast<int (*)(Comm*, int, UniqueId, int)>(dlsym(h, "ncclCommInitRank"));
    n.commDestroy = reinterpret_cast<int (*)(Comm)>(dlsym(h, "ncclCommDestroy"));
    n.send = reinterpret_cast<int (*)(const void*, size_t, int, int, Comm, cudaStream_t)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<int (*)(void*, size_t, int, int, Comm, cudaStream_t)>(dlsym(h, "ncclRecv"));
    n.allReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, Comm, cudaStream_t)>(
        dlsym(h, "ncclAllReduce"));
    n.allGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, Comm, cudaStream_t)>(
        dlsym(h, "ncclAllGather"));
    n.groupStart = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupStart"));
    n.groupEnd = reinterpret_cast<int (*)()>(dlsym(h, "ncclGroupEnd"));
    n.getErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.send && n.recv && n.allReduce &&
           n.groupStart && n.groupEnd;
  });
  return n;
}

int nccl_status(int r, const char* what) {
  if (r == 0) return GPP_OK;
  set_error(std::string(what) + ": " + (nccl().getErrorString ? nccl().getErrorString(r) : "nccl error"));
  return GPP_ERR_CUDA;
}

}  // namespace
}  // namespace gpp

using namespace gpp;

extern "C" {

int gpp_nccl_available(void) { return nccl().ok ? 1 : 0; }

int gpp_nccl_unique_id(void* out128) {
  GPP_ARG_CHECK(out128, "null pointer");
  if (!nccl().ok) { set_error("libnccl.so.2 not loadable"); return GPP_ERR_UNSUPPORTED; }
  return nccl_status(nccl().getUniqueId(static_cast<UniqueId*>(out128)), "ncclGetUniqueId");
}

// Initialise n communicators in one NCCL group (no cross-communicator deadlock):
// comm i has nranks[i] members, this process is rank ranks[i], id = ids + 128*i.
int gpp_comm_init_group(int n, const void* ids, const int* nranks, const int* ranks, void** comms) {
  GPP_ARG_CHECK(n >= 0 && (n == 0 || (ids && nranks && ranks && comms)), "bad argument");
  if (!nccl().ok) { set_error("libnccl.so.2 not loadable"); return GPP_ERR_UNSUPPORTED; }
  int rc = nccl_status(nccl().groupStart(), "ncclGroupStart");
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    UniqueId id;
    memcpy(&id, static_cast<const char*>(ids) + 128 * i, 128);
    rc = nccl_status(nccl().commInitRank(reinterpret_cast<Comm*>(&comms[i]), nranks[i], id, ranks[i]),
                     "ncclCommInitRank");
    if (rc) { nccl().groupEnd(); return rc; }
  }
  return nccl_status(nccl().groupEnd(), "ncclGroupEnd(init)");
}

int gpp_comm_destroy(void* comm) {
  if (!comm) return GPP_OK;
  return nccl_status(nccl().commDestroy(comm), "ncclCommDestroy");
}

int gpp_send(void* comm, const void* buf, int64_t bytes, int peer, void* stream) {
  GPP_ARG_CHECK(comm && buf && bytes >= 0, "bad argument");
  return nccl_status(nccl().send(buf, static_cast<size_t>(bytes), NCCL_UINT8, peer, comm,
                                 static_cast<cudaStream_t>(stream)), "ncclSend");
}

int gpp_recv(void* comm, void* buf, int64_t bytes, int peer, void* stream) {
  GPP_ARG_CHECK(comm && buf && bytes >= 0, "bad argument");
  return nccl_status(nccl().recv(buf, static_cast<size_t>(bytes), NCCL_UINT8, peer, comm,
                                 static_cast<cudaStream_t>(stream)), "ncclRecv");
}

int gpp_allreduce_f32(void* comm, void* buf, int64_t count, void* stream) {
  GPP_ARG_CHECK(comm && buf && count >= 0, "bad argument");
  return nccl_status(nccl().allReduce(buf, buf, static_cast<size_t>(count), NCCL_FLOAT32, NCCL_SUM, comm,
                                      static_cast<cudaStream_t>(stream)), "ncclAllReduce");
}

int gpp_allgather(void* comm, const void* send, void* recv, int64_t bytes_per_rank, void* stream) {
  GPP_ARG_CHECK(comm && send && recv && bytes_per_rank >= 0, "bad argument");
  if (!nccl().allGather) { set_error("ncclAllGather unavailable"); return GPP_ERR_UNSUPPORTED; }
  return nccl_status(nccl().allGather(send, recv, static_cast<size_t>(bytes_per_rank), NCCL_UINT8, comm,
                                      static_cast<cudaStream_t>(stream)), "ncclAllGather");
}

int gpp_group_start(void) { return nccl_status(nccl().groupStart(), "ncclGroupStart"); }
int gpp_group_end(void) { return nccl_status(nccl().groupEnd(), "ncclGroupEnd"); }

}  // extern "C"
