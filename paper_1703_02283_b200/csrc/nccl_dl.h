// nccl_dl.h -- NCCL loaded at run time with dlopen (no link-time dependency; world == 1 never
// touches NCCL).  Used for the column-panel all-gathers of SURVEY 8(e) over NVLink/NVSwitch.
#pragma once
#include <cstddef>
#include <string>
#include <cuda_runtime.h>

namespace ipr {

class NcclComm {
 public:
  static bool unique_id(void *out128, std::string *err);
  bool init(int world, int rank, const void *uid128, std::string *err);
  bool allgather(const void *send, void *recv, size_t bytes_per_rank, cudaStream_t s);
  void destroy();
  const char *last_error() const { return err_.c_str(); }
  bool active() const { return comm_ != nullptr; }

 private:
  void *comm_ = nullptr;
  std::string err_;
};

}  // namespace ipr
