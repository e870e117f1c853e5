// nccl_dl.cu -- dlopen'ed NCCL (prefers the copy torch already loaded into the process).
#include "nccl_dl.h"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

namespace ipr {
namespace {

struct Api {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

Api &api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { a.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return; }
    a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
    a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
    a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
    a.errStr = (decltype(a.errStr))dlsym(h, "ncclGetErrorString");
    a.ok = a.getUniqueId && a.commInitRank && a.allGather && a.commDestroy && a.errStr;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

}  // namespace

bool NcclComm::unique_id(void *out128, std::string *err) {
  Api &a = api();
  if (!a.ok) { *err = a.why; return false; }
  ncclUniqueId id;
  ncclResult_t r = a.getUniqueId(&id);
  if (r != ncclSuccess) { *err = a.errStr(r); return false; }
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  memcpy(out128, &id, 128);
  return true;
}

bool NcclComm::init(int world, int rank, const void *uid128, std::string *err) {
  Api &a = api();
  if (!a.ok) { *err = a.why; return false; }
  ncclUniqueId id;
  memcpy(&id, uid128, 128);
  ncclComm_t c = nullptr;
  ncclResult_t r = a.commInitRank(&c, world, id, rank);
  if (r != ncclSuccess) { *err = std::string("ncclCommInitRank: ") + a.errStr(r); return false; }
  comm_ = c;
  return true;
}

bool NcclComm::allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) {
  Api &a = api();
  if (!comm_) { err_ = "communicator not initialised"; return false; }
  ncclResult_t r = a.allGather(send, recv, bytes, ncclInt8, (ncclComm_t)comm_, s);
  if (r != ncclSuccess) { err_ = a.errStr(r); return false; }
  return true;
}

void NcclComm::destroy() {
  if (comm_) { api().commDestroy((ncclComm_t)comm_); comm_ = nullptr; }
}

}  // namespace ipr
