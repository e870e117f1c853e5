// nccl_dl.cu -- the transports of nccl_dl.h: dlopen'ed NCCL (prefers the copy torch already loaded
// into the process) and the in-process local group used to run the sharded path on one device.
#include "nccl_dl.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

namespace ipr {
namespace {

struct Api {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommSplit) commSplit = nullptr;
  decltype(&ncclCommCount) commCount = nullptr;
  decltype(&ncclCommUserRank) commUserRank = nullptr;
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
    a.send = (decltype(a.send))dlsym(h, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
    a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
    a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
    a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
    a.commSplit = (decltype(a.commSplit))dlsym(h, "ncclCommSplit");          // NCCL >= 2.18 (2-D grids only)
    a.commCount = (decltype(a.commCount))dlsym(h, "ncclCommCount");
    a.commUserRank = (decltype(a.commUserRank))dlsym(h, "ncclCommUserRank");
    a.errStr = (decltype(a.errStr))dlsym(h, "ncclGetErrorString");
    a.ok = a.getUniqueId && a.commInitRank && a.allGather && a.send && a.recv && a.groupStart && a.groupEnd &&
           a.commDestroy && a.errStr;
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
  world_ = world; rank_ = rank;
  return true;
}

bool NcclComm::allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) {
  Api &a = api();
  if (!comm_) { err_ = "communicator not initialised"; return false; }
  ncclResult_t r = a.allGather(send, recv, bytes, ncclInt8, (ncclComm_t)comm_, s);
  if (r != ncclSuccess) { err_ = a.errStr(r); return false; }
  return true;
}

bool NcclComm::alltoall(const void *send, void *recv, size_t bytes, cudaStream_t s) {
  Api &a = api();
  if (!comm_) { err_ = "communicator not initialised"; return false; }
  ncclResult_t r = a.groupStart();
  for (int h = 0; h < world_ && r == ncclSuccess; ++h) {
    r = a.send((const char *)send + h * bytes, bytes, ncclInt8, h, (ncclComm_t)comm_, s);
    if (r == ncclSuccess) r = a.recv((char *)recv + h * bytes, bytes, ncclInt8, h, (ncclComm_t)comm_, s);
  }
  const ncclResult_t e = a.groupEnd();
  if (r == ncclSuccess) r = e;
  if (r != ncclSuccess) { err_ = a.errStr(r); return false; }
  return true;
}

Transport *NcclComm::split(int color, int key, std::string *err) {
  Api &a = api();
  if (!comm_) { *err = "communicator not initialised"; return nullptr; }
  if (!a.commSplit || !a.commCount || !a.commUserRank) { *err = "this NCCL has no ncclCommSplit"; return nullptr; }
  ncclComm_t sub = nullptr;
  ncclResult_t r = a.commSplit((ncclComm_t)comm_, color, key, &sub, nullptr);
  if (r != ncclSuccess) { *err = std::string("ncclCommSplit: ") + a.errStr(r); return nullptr; }
  NcclComm *t = new NcclComm();
  t->comm_ = sub;
  a.commCount(sub, &t->world_);
  a.commUserRank(sub, &t->rank_);
  return t;
}

NcclComm::~NcclComm() {
  if (comm_) { api().commDestroy((ncclComm_t)comm_); comm_ = nullptr; }
}

// ---------------------------------------------------------------------------------------
// Local group: world ranks in one process on one device.  An exchange is
//   1. rank r publishes its buffers and records `ready` on its stream; host barrier;
//   2. rank r's stream waits for every peer's `ready`, copies what it needs from the peers' buffers,
//      records `done`; host barrier;
//   3. rank r's stream waits for every peer's `done` (no rank overwrites a buffer a peer still reads).
// Each event is re-recorded only after the barrier that follows every wait on it.
// ---------------------------------------------------------------------------------------
struct LocalGroup {
  int world = 0;
  std::vector<int> color, key;            // split() exchange area
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  struct Slot { const void *send = nullptr; void *recv = nullptr; cudaEvent_t ready = nullptr, done = nullptr; };
  std::vector<Slot> slot;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++arrived == world) { arrived = 0; ++generation; cv.notify_all(); return; }
    cv.wait(lk, [&] { return generation != gen; });
  }
};

namespace {
// A rank of a local group, or of a sub-group of it (split): `members` are the group's world ranks in
// sub-rank order.  Every collective still passes the WORLD barrier: in the SPMD engine every rank
// reaches each (sub-)collective at the same program point, and copies come from members only.
class LocalRank : public Transport {
 public:
  LocalRank(LocalGroup *g, int rank) : g_(g), rank_(rank) {
    for (int r = 0; r < g->world; ++r) members_.push_back(r);
    sub_ = rank;
  }
  LocalRank(LocalGroup *g, int rank, std::vector<int> members, int sub)
      : g_(g), rank_(rank), members_(std::move(members)), sub_(sub) {}
  Transport *split(int color, int key, std::string *err) override {
    g_->color[rank_] = color; g_->key[rank_] = key;
    g_->barrier();
    std::vector<std::pair<int, int>> mk;   // (key, world rank) of my color
    for (int r = 0; r < g_->world; ++r)
      if (g_->color[r] == color && std::find(members_.begin(), members_.end(), r) != members_.end())
        mk.push_back({g_->key[r], r});
    std::sort(mk.begin(), mk.end());
    g_->barrier();                          // everyone has read color / key before the next split
    std::vector<int> m;
    int sub = -1;
    for (size_t i = 0; i < mk.size(); ++i) { m.push_back(mk[i].second); if (mk[i].second == rank_) sub = (int)i; }
    if (sub < 0) { *err = "local split: rank not in its own color"; return nullptr; }
    return new LocalRank(g_, rank_, m, sub);
  }
  bool allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override {
    return exchange(send, recv, bytes, s, false);
  }
  bool alltoall(const void *send, void *recv, size_t bytes, cudaStream_t s) override {
    return exchange(send, recv, bytes, s, true);
  }
  const char *last_error() const override { return err_.c_str(); }

 private:
  bool ck(cudaError_t e) {
    if (e == cudaSuccess) return true;
    err_ = cudaGetErrorString(e);
    return false;
  }
  bool exchange(const void *send, void *recv, size_t bytes, cudaStream_t s, bool a2a) {
    LocalGroup::Slot &me = g_->slot[rank_];
    me.send = send; me.recv = recv;
    bool ok = ck(cudaEventRecord(me.ready, s));
    g_->barrier();
    for (int h = 0; h < (int)members_.size() && ok; ++h) {
      const int wr = members_[h];
      const LocalGroup::Slot &peer = g_->slot[wr];
      const char *src = a2a ? (const char *)peer.send + sub_ * bytes : (const char *)peer.send;
      char *dst = (char *)recv + h * bytes;
      if (wr != rank_) ok = ck(cudaStreamWaitEvent(s, peer.ready, 0));
      if (ok && src != dst) ok = ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (ok) ok = ck(cudaEventRecord(me.done, s));
    g_->barrier();
    for (int h = 0; h < (int)members_.size() && ok; ++h)
      if (members_[h] != rank_) ok = ck(cudaStreamWaitEvent(s, g_->slot[members_[h]].done, 0));
    return ok;
  }
  LocalGroup *g_;
  int rank_;                 // world rank
  std::vector<int> members_;
  int sub_;                  // rank within members_
  std::string err_;
};
}  // namespace

LocalGroup *local_group_create(int world, std::string *err) {
  if (world < 1 || world > 64) { *err = "local group: world must be in [1, 64]"; return nullptr; }
  LocalGroup *g = new LocalGroup();
  g->world = world;
  g->slot.resize(world);
  g->color.assign(world, 0);
  g->key.assign(world, 0);
  for (auto &sl : g->slot) {
    if (cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess) {
      *err = std::string("local group: cudaEventCreate: ") + cudaGetErrorString(cudaGetLastError());
      local_group_destroy(g);
      return nullptr;
    }
  }
  return g;
}

void local_group_destroy(LocalGroup *g) {
  if (!g) return;
  for (auto &sl : g->slot) {
    if (sl.ready) cudaEventDestroy(sl.ready);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  delete g;
}

Transport *local_transport(LocalGroup *g, int rank, std::string *err) {
  if (!g || rank < 0 || rank >= g->world) { *err = "local group: bad rank"; return nullptr; }
  return new LocalRank(g, rank);
}

int local_group_world(const LocalGroup *g) { return g ? g->world : 0; }

}  // namespace ipr
