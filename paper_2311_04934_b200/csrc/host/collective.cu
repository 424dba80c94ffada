#include "collective.hpp"

#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <string>

#include "errors.hpp"

namespace pcb::coll {

#define CKC(x)                                                                                                     \
  do {                                                                                                             \
    cudaError_t e_ = (x);                                                                                          \
    if (e_ != cudaSuccess) throw Error(ErrorCode::CudaError, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// NCCL, resolved with dlopen (types mirror nccl.h: ncclUniqueId is 128 bytes,
// ncclFloat32 = 7, ncclSum = 0, ncclSuccess = 0).
// ---------------------------------------------------------------------------
namespace {
struct NcclId {
  char internal[kNcclIdBytes];
};
using ncclComm_t = void*;
struct NcclApi {
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
constexpr int kFloat32 = 7, kSum = 0;

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) throw Error(ErrorCode::CudaError, "libnccl not found: the head-sharded path needs NCCL");
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p) throw Error(ErrorCode::CudaError, std::string("NCCL symbol missing: ") + s);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void ck_nccl(int r, const char* what) {
  if (r != 0) throw Error(ErrorCode::CudaError, std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclCollective : public Collective {
 public:
  NcclCollective(const uint8_t id[kNcclIdBytes], int r, int n, int device) {
    rank = r;
    size = n;
    CKC(cudaSetDevice(device));
    NcclId nid;
    std::memcpy(nid.internal, id, kNcclIdBytes);
    ck_nccl(nccl().CommInitRank(&comm_, n, nid, r), "ncclCommInitRank");
  }
  ~NcclCollective() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void all_reduce_sum(float* buf, size_t n, cudaStream_t s) override {
    ck_nccl(nccl().AllReduce(buf, buf, n, kFloat32, kSum, comm_, s), "ncclAllReduce");
  }
  void all_gather(const float* send, float* recv, size_t n, cudaStream_t s) override {
    ck_nccl(nccl().AllGather(send, recv, n, kFloat32, comm_, s), "ncclAllGather");
  }

 private:
  ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------------------
// Ranks as threads on one device.  all_reduce: every rank stages its buffer in its
// slot, all ranks meet, each sums the slots in rank order into its own buffer, all
// ranks meet again before a slot may be reused.
// ---------------------------------------------------------------------------
__global__ void k_sum_slots(float* const* slots, int size, float* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float acc = slots[0][i];
    for (int r = 1; r < size; ++r) acc = __fadd_rn(acc, slots[r][i]);
    out[i] = acc;
  }
}

class LocalCollective : public Collective {
 public:
  LocalCollective(std::shared_ptr<LocalGroup> g, int r) : g_(std::move(g)) {
    rank = r;
    size = g_->size();
    CKC(cudaMalloc(&d_slots_, sizeof(float*) * size));
  }
  ~LocalCollective() override {
    if (d_slots_) cudaFree(d_slots_);
  }
  void all_reduce_sum(float* buf, size_t n, cudaStream_t s) override {
    stage(buf, n, s);
    std::vector<float*> ptrs(size);
    for (int r = 0; r < size; ++r) ptrs[r] = g_->slot(r, n);
    CKC(cudaMemcpyAsync(d_slots_, ptrs.data(), sizeof(float*) * size, cudaMemcpyHostToDevice, s));
    k_sum_slots<<<148, 256, 0, s>>>(d_slots_, size, buf, n);
    CKC(cudaGetLastError());
    finish(s);
  }
  void all_gather(const float* send, float* recv, size_t n, cudaStream_t s) override {
    stage(send, n, s);
    for (int r = 0; r < size; ++r)
      CKC(cudaMemcpyAsync(recv + static_cast<size_t>(r) * n, g_->slot(r, n), n * 4, cudaMemcpyDeviceToDevice, s));
    finish(s);
  }

 private:
  void stage(const float* src, size_t n, cudaStream_t s) {
    g_->barrier();  // every rank has sized its slot for this collective
    CKC(cudaMemcpyAsync(g_->slot(rank, n), src, n * 4, cudaMemcpyDeviceToDevice, s));
    CKC(cudaEventRecord(g_->event(rank, 0), s));
    g_->barrier();
    for (int r = 0; r < size; ++r) CKC(cudaStreamWaitEvent(s, g_->event(r, 0), 0));
  }
  void finish(cudaStream_t s) {
    CKC(cudaEventRecord(g_->event(rank, 1), s));
    g_->barrier();
    for (int r = 0; r < size; ++r) CKC(cudaStreamWaitEvent(s, g_->event(r, 1), 0));  // slots free again
  }
  std::shared_ptr<LocalGroup> g_;
  float** d_slots_ = nullptr;
};
}  // namespace

void nccl_unique_id(uint8_t out[kNcclIdBytes]) {
  NcclId id;
  ck_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, kNcclIdBytes);
}

std::shared_ptr<Collective> make_nccl(const uint8_t id[kNcclIdBytes], int rank, int size, int device) {
  return std::make_shared<NcclCollective>(id, rank, size, device);
}

LocalGroup::LocalGroup(int size) : size_(size), slots_(size, nullptr), caps_(size, 0), events_(2 * size, nullptr) {
  for (auto& e : events_) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}
LocalGroup::~LocalGroup() {
  for (float* p : slots_)
    if (p) cudaFree(p);
  for (auto& e : events_)
    if (e) cudaEventDestroy(e);
}
void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  const uint64_t gen = generation_;
  if (++arrived_ == size_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
    return;
  }
  if (!cv_.wait_for(lk, std::chrono::seconds(120), [&] { return generation_ != gen; }))
    throw Error(ErrorCode::Internal, "tensor-parallel group: a rank did not reach the collective");
}
float* LocalGroup::slot(int r, size_t n) {
  std::lock_guard<std::mutex> lk(mu_);
  if (caps_[r] < n) {
    if (slots_[r]) {
      CKC(cudaDeviceSynchronize());
      cudaFree(slots_[r]);
    }
    CKC(cudaMalloc(&slots_[r], n * 4));
    caps_[r] = n;
  }
  return slots_[r];
}
cudaEvent_t LocalGroup::event(int r, int which) { return events_[which * size_ + r]; }

std::shared_ptr<Collective> make_local(std::shared_ptr<LocalGroup> g, int rank) {
  return std::make_shared<LocalCollective>(std::move(g), rank);
}

}  // namespace pcb::coll
