// nccl_dl.h -- the rank-to-rank data exchange of the column-panel decomposition (the
// "data exchange" of PAPER.md:138-141 [Sec. 3.2]) behind one small interface:
//   * NcclComm: NCCL loaded at run time with dlopen (no link-time dependency; world == 1 never touches
//     it) -- one process per GPU over NVLink / NVSwitch, the production transport;
//   * a local group: `world` ranks in ONE process on ONE device, each with its own context, stream and
//     host thread; the exchange is stream-ordered device copies fenced by CUDA events and host barriers
//     (no kernel ever waits on another rank).  It exists so the sharded engine path (panel layouts,
//     partial gathers, the tri form's mirror exchange) runs -- and is compared bit for bit with
//     world = 1 -- on a one-GPU box (ipr_testing.h).
// Both transports are collective: every rank calls the same operations in the same order.
#pragma once
#include <cstddef>
#include <string>
#include <cuda_runtime.h>

namespace ipr {

class Transport {
 public:
  virtual ~Transport() = default;
  // recv[r * bytes .. (r + 1) * bytes) = rank r's send (in place when send == recv + rank * bytes)
  virtual bool allgather(const void *send, void *recv, size_t bytes_per_rank, cudaStream_t s) = 0;
  // recv[r * bytes ..) = rank r's send[rank * bytes ..) (send and recv distinct)
  virtual bool alltoall(const void *send, void *recv, size_t bytes_per_peer, cudaStream_t s) = 0;
  virtual const char *last_error() const = 0;
  // collective over this transport's ranks: the sub-transport of the ranks with the same color, ordered
  // by key (2-D grids: a grid row / a grid column); nullptr + *err on failure.  Owned by the caller.
  virtual Transport *split(int color, int key, std::string *err) = 0;
};

class NcclComm : public Transport {
 public:
  static bool unique_id(void *out128, std::string *err);
  bool init(int world, int rank, const void *uid128, std::string *err);
  bool allgather(const void *send, void *recv, size_t bytes_per_rank, cudaStream_t s) override;
  bool alltoall(const void *send, void *recv, size_t bytes_per_peer, cudaStream_t s) override;
  const char *last_error() const override { return err_.c_str(); }
  Transport *split(int color, int key, std::string *err) override;
  ~NcclComm() override;

 private:
  void *comm_ = nullptr;
  int world_ = 1, rank_ = 0;
  std::string err_;
};

struct LocalGroup;
LocalGroup *local_group_create(int world, std::string *err);
void local_group_destroy(LocalGroup *g);
// the transport of one rank of a local group (owned by the caller); nullptr + *err on failure
Transport *local_transport(LocalGroup *g, int rank, std::string *err);
int local_group_world(const LocalGroup *g);

}  // namespace ipr
