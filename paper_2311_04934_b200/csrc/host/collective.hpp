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

// ---- peer memory: one process per rank, buffers shared through CUDA IPC ----
// Each rank owns one device region [flags][2 slots of cap floats]; every rank maps every
// peer's region (cudaIpcOpenMemHandle: NVLink/NVSwitch loads between GPUs, or plain device
// memory when several ranks share one GPU).  A collective is one-shot: publish into this
// rank's slot (generation parity), release the generation flag at system scope, then every
// rank reads all slots in rank order (deterministic sums) once every peer's flag has it.
constexpr int kIpcHandleBytes = 64;
class PeerRegion {
 public:
  PeerRegion(int rank, int size, int device, size_t cap_floats);
  ~PeerRegion();
  PeerRegion(const PeerRegion&) = delete;
  PeerRegion& operator=(const PeerRegion&) = delete;
  void handle(uint8_t out[kIpcHandleBytes]) const;                    // this rank's IPC handle
  void open(const uint8_t* handles /* [size][kIpcHandleBytes] */);    // map every peer
  int rank, size, device;
  size_t cap;                 // floats per slot
  char* local = nullptr;      // this rank's region
  std::vector<char*> peers;   // every rank's region (local for r == rank)
  char** d_peers = nullptr;   // the same table on the device
};
std::shared_ptr<Collective> make_peer(std::shared_ptr<PeerRegion> region);

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
