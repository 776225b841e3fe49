// comm.cpp -- see comm.h.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace hmat {

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  std::string error;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) {
      a.error = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.handle, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.handle, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(a.handle, "ncclAllReduce"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.handle, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.handle, "ncclGetErrorString"));
    a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(a.handle, "ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(a.handle, "ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.handle, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.handle, "ncclGroupEnd"));
    a.CommGetAsyncError = reinterpret_cast<decltype(a.CommGetAsyncError)>(dlsym(a.handle, "ncclCommGetAsyncError"));
    a.CommCount = reinterpret_cast<decltype(a.CommCount)>(dlsym(a.handle, "ncclCommCount"));
    a.CommUserRank = reinterpret_cast<decltype(a.CommUserRank)>(dlsym(a.handle, "ncclCommUserRank"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.CommDestroy || !a.GetErrorString || !a.Send ||
        !a.Recv || !a.GroupStart || !a.GroupEnd || !a.CommGetAsyncError || !a.CommCount || !a.CommUserRank)
      a.error = "libnccl is missing a required symbol";
  });
  return a;
}

std::string nccl_err(const char* what, ncclResult_t r) {
  return std::string(what) + ": " + api().GetErrorString(r);
}

}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
};

std::string comm_unique_id(void* out128) {
  NcclApi& a = api();
  if (!a.error.empty()) return a.error;
  ncclUniqueId id;
  ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_err("ncclGetUniqueId", r);
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return "";
}

std::string comm_create(const void* id128, int nranks, int rank, Comm** out) {
  NcclApi& a = api();
  if (!a.error.empty()) return a.error;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  Comm* c = new Comm;
  ncclResult_t r = a.CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_err("ncclCommInitRank", r);
  }
  *out = c;
  return "";
}

std::string comm_allreduce_sum(Comm* c, double* buf, size_t count, cudaStream_t stream) {
  if (count == 0) return "";
  ncclResult_t r = api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, stream);
  if (r != ncclSuccess) return nccl_err("ncclAllReduce", r);
  return "";
}

std::string comm_swap_round(Comm* c, const double* buf, double* tmp, size_t count, int partner, cudaStream_t stream) {
  NcclApi& a = api();
  ncclResult_t r = a.GroupStart();
  if (r != ncclSuccess) return nccl_err("ncclGroupStart", r);
  ncclResult_t rs = a.Send(buf, count, ncclFloat64, partner, c->comm, stream);
  ncclResult_t rr = a.Recv(tmp, count, ncclFloat64, partner, c->comm, stream);
  r = a.GroupEnd();
  if (rs != ncclSuccess) return nccl_err("ncclSend", rs);
  if (rr != ncclSuccess) return nccl_err("ncclRecv", rr);
  if (r != ncclSuccess) return nccl_err("ncclGroupEnd", r);
  return "";
}

std::string comm_tree_allreduce_sum(Comm* c, double* buf, double* tmp, size_t count, int nranks, int rank,
                                    cudaStream_t stream) {
  if (count == 0) return "";
  for (int bit = 1; bit < nranks; bit <<= 1) {
    std::string m = comm_swap_round(c, buf, tmp, count, rank ^ bit, stream);
    if (!m.empty()) return m;
    cudaError_t e = launch_add_inplace(buf, tmp, count, stream);
    if (e != cudaSuccess) return std::string("add_inplace: ") + cudaGetErrorString(e);
  }
  return "";
}

std::string comm_async_error(Comm* c) {
  if (!c || !c->comm) return "";
  ncclResult_t st = ncclSuccess;
  ncclResult_t r = api().CommGetAsyncError(c->comm, &st);
  if (r != ncclSuccess) return nccl_err("ncclCommGetAsyncError", r);
  if (st != ncclSuccess && st != ncclInProgress) return nccl_err("NCCL asynchronous error", st);
  return "";
}

std::string comm_info(Comm* c, int* nranks, int* rank) {
  NcclApi& a = api();
  ncclResult_t r = a.CommCount(c->comm, nranks);
  if (r != ncclSuccess) return nccl_err("ncclCommCount", r);
  r = a.CommUserRank(c->comm, rank);
  if (r != ncclSuccess) return nccl_err("ncclCommUserRank", r);
  return "";
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm) api().CommDestroy(c->comm);
  delete c;
}

}  // namespace hmat
