// Tensor-parallel collectives for the head-sharded path (config 5, a module
// store larger than one GPU's HBM; heads, MLP columns and the vocabulary split over the
// ranks, one all-reduce after each row-parallel GEMM).  Two implementations behind one
// interface, both on the model's stream:
//   NcclCollective   one process per GPU, NCCL over NVLink/NVSwitch (libnccl is opened
//                    at run time, so the library loads on hosts without it)
//   LocalCollective  every rank a thread of one process on one device (tests: the real
//                    sharded forward on a single GPU); deterministic rank-order sums
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace pcb::coll {

class Collective {
 public:
  virtual ~Collective() = default;
  int rank = 0, size = 1;
  // in-place sum of n floats across ranks
  virtual void all_reduce_sum(float* buf, size_t n, cudaStream_t s) = 0;
  // recv[r * n + i] = send_r[i]
  virtual void all_gather(const float* send, float* recv, size_t n, cudaStream_t s) = 0;
};

// ---- NCCL ----
constexpr int kNcclIdBytes = 128;
void nccl_unique_id(uint8_t out[kNcclIdBytes]);
std::shared_ptr<Collective> make_nccl(const uint8_t id[kNcclIdBytes], int rank, int size, int device);

// ---- one process, ranks as threads on one device ----
class LocalGroup {
 public:
  explicit LocalGroup(int size);
  ~LocalGroup();
  int size() const { return size_; }
  // host barrier of all ranks; throws after a timeout (a rank failed)
  void barrier();
  float* slot(int r, size_t n);  // device staging slot of rank r (>= n floats)
  cudaEvent_t event(int r, int which);

 private:
  int size_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t generation_ = 0;
  std::vector<float*> slots_;
  std::vector<size_t> caps_;
  std::vector<cudaEvent_t> events_;
};
std::shared_ptr<Collective> make_local(std::shared_ptr<LocalGroup> g, int rank);

}  // namespace pcb::coll
