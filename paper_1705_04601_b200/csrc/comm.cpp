// NCCL communicator of a multi-GPU job: one process per GPU,
// bootstrapped through the caller's process group (torch.distributed carries
// the 128-byte NCCL unique id), then used for the job's only collectives:
// the sum of the per-rank checks (||S||_F^2, ||y||^2, flops) and of the
// distributed result vectors (each rank's S rows are disjoint, so a sum
// all-reduce of the N-vectors assembles y = S w on every rank), and the max of
// the per-rank step times.  The data path itself has no exchange: every shard
// recomputes its halo Q / R^.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2 -- the copy torch
// already loaded if any), so the library itself has no link-time dependency
// on it; a missing NCCL is H2SP_ENCCL, never a fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "h2sp_internal.h"

using namespace h2sp;

namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef struct ncclComm *ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat64 = 8;  // ncclFloat64
constexpr int kNcclSum = 0, kNcclMax = 2;

struct Nccl {
  bool tried = false, ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl &nccl() {
  static Nccl n;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (n.tried) return n;
  n.tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    n.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return n;
  }
  n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(dlsym(h, "ncclAllReduce"));
  n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
  n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce && n.GetErrorString;
  if (!n.ok) n.err = "libnccl.so.2 lacks an expected symbol";
  return n;
}

h2sp_status nccl_fail(const char *what, ncclResult_t r) {
  return fail(H2SP_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

struct h2sp_comm_s {
  ncclComm_t comm;
  int rank, world, device;
};

extern "C" {

h2sp_status h2sp_comm_unique_id(void *id) {
  if (!id) return fail(H2SP_EINVAL, "NULL id buffer");
  Nccl &n = nccl();
  if (!n.ok) return fail(H2SP_ENCCL, n.err);
  ncclUniqueId u;
  if (ncclResult_t r = n.GetUniqueId(&u)) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(id, &u, sizeof(u));
  return H2SP_OK;
}

h2sp_status h2sp_comm_init(const void *id, int rank, int world, h2sp_comm *out) {
  if (!id || !out) return fail(H2SP_EINVAL, "NULL id or output");
  if (world < 1 || rank < 0 || rank >= world) return fail(H2SP_EINVAL, "rank outside [0, world)");
  *out = nullptr;
  Nccl &n = nccl();
  if (!n.ok) return fail(H2SP_ENCCL, n.err);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(H2SP_ECUDA, "no CUDA device");
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  if (ncclResult_t r = n.CommInitRank(&c, world, u, rank)) return nccl_fail("ncclCommInitRank", r);
  *out = new h2sp_comm_s{c, rank, world, dev};
  return H2SP_OK;
}

h2sp_status h2sp_comm_allreduce(h2sp_comm comm, double *buf, int64_t n, int op, void *stream) {
  if (!comm || (!buf && n)) return fail(H2SP_EINVAL, "NULL communicator or buffer");
  if (op != H2SP_SUM && op != H2SP_MAX) return fail(H2SP_EINVAL, "op must be H2SP_SUM or H2SP_MAX");
  if (n == 0) return H2SP_OK;
  Nccl &nc = nccl();
  if (ncclResult_t r = nc.AllReduce(buf, buf, size_t(n), kNcclFloat64, op == H2SP_SUM ? kNcclSum : kNcclMax,
                                    comm->comm, (cudaStream_t)stream))
    return nccl_fail("ncclAllReduce", r);
  return H2SP_OK;
}

h2sp_status h2sp_comm_info(h2sp_comm comm, int *rank, int *world) {
  if (!comm) return fail(H2SP_EINVAL, "NULL communicator");
  if (rank) *rank = comm->rank;
  if (world) *world = comm->world;
  return H2SP_OK;
}

void h2sp_comm_destroy(h2sp_comm comm) {
  if (!comm) return;
  if (nccl().ok) nccl().CommDestroy(comm->comm);
  delete comm;
}

}  // extern "C"
