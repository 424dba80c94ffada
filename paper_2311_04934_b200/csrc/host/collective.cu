#include "collective.hpp"

#include <dlfcn.h>

#include <algorithm>
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

// ---------------------------------------------------------------------------
// Peer memory (CUDA IPC).  Region layout: 256 B of flags (the first u64 = the last
// published generation), then slots [2][cap] fp32.
// ---------------------------------------------------------------------------
constexpr size_t kFlagBytes = 256;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// every thread of the grid has finished its stores of this rank's slot (stream order: this
// single-thread kernel runs after the copy); make them visible system-wide, then publish
__global__ void k_peer_signal(char* local, unsigned long long gen) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(reinterpret_cast<unsigned long long*>(local)), "l"(gen)
               : "memory");
}

__device__ void peer_wait_all(char* const* peers, int size, unsigned long long gen) {
  if (threadIdx.x < size) {
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(peers[threadIdx.x]);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(f) < gen) {
      __nanosleep(256);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60ull * 1000000000ull) {  // a rank stopped participating: fail, do not hang
        printf("[pcb] peer collective: rank %d never published generation %llu\n", threadIdx.x, gen);
        __trap();
      }
    }
  }
  __syncthreads();
}

// out[i] = sum over ranks (rank order) of slot_r[i]
__global__ void k_peer_reduce(char* const* peers, int size, int parity, size_t cap, unsigned long long gen, float* out,
                              size_t n) {
  peer_wait_all(peers, size, gen);
  const size_t off = kFlagBytes + static_cast<size_t>(parity) * cap * 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float acc = reinterpret_cast<const float*>(peers[0] + off)[i];
    for (int r = 1; r < size; ++r) acc = __fadd_rn(acc, reinterpret_cast<const float*>(peers[r] + off)[i]);
    out[i] = acc;
  }
}

// recv[r * n + i] = slot_r[i]
__global__ void k_peer_gather(char* const* peers, int size, int parity, size_t cap, unsigned long long gen, float* recv,
                              size_t n) {
  peer_wait_all(peers, size, gen);
  const size_t off = kFlagBytes + static_cast<size_t>(parity) * cap * 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n * size; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / n, j = i - r * n;
    recv[i] = reinterpret_cast<const float*>(peers[r] + off)[j];
  }
}

class PeerCollective : public Collective {
 public:
  explicit PeerCollective(std::shared_ptr<PeerRegion> reg) : reg_(std::move(reg)) {
    rank = reg_->rank;
    size = reg_->size;
  }
  void all_reduce_sum(float* buf, size_t n, cudaStream_t s) override {
    const unsigned long long gen = publish(buf, n, s);
    k_peer_reduce<<<grid(n), 256, 0, s>>>(reg_->d_peers, size, static_cast<int>(gen & 1), reg_->cap, gen, buf, n);
    CKC(cudaGetLastError());
  }
  void all_gather(const float* send, float* recv, size_t n, cudaStream_t s) override {
    const unsigned long long gen = publish(send, n, s);
    k_peer_gather<<<grid(n * size), 256, 0, s>>>(reg_->d_peers, size, static_cast<int>(gen & 1), reg_->cap, gen, recv,
                                                 n);
    CKC(cudaGetLastError());
  }

 private:
  static unsigned grid(size_t n) { return static_cast<unsigned>(std::min<size_t>(592, (n + 255) / 256 + 1)); }
  // Slot gen & 1 is free: every peer finished reading it (collective gen - 2) before it
  // published gen - 1, and this rank's previous collective waited for every gen - 1.
  unsigned long long publish(const float* src, size_t n, cudaStream_t s) {
    if (n > reg_->cap) throw Error(ErrorCode::ShapeMismatch, "peer collective: message exceeds the shared slot");
    const unsigned long long gen = ++gen_;
    CKC(cudaMemcpyAsync(reg_->local + kFlagBytes + (gen & 1) * reg_->cap * 4, src, n * 4, cudaMemcpyDeviceToDevice, s));
    k_peer_signal<<<1, 1, 0, s>>>(reg_->local, gen);
    CKC(cudaGetLastError());
    return gen;
  }
  std::shared_ptr<PeerRegion> reg_;
  unsigned long long gen_ = 0;
};

void nccl_unique_id(uint8_t out[kNcclIdBytes]) {
  NcclId id;
  ck_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, kNcclIdBytes);
}

std::shared_ptr<Collective> make_nccl(const uint8_t id[kNcclIdBytes], int rank, int size, int device) {
  return std::make_shared<NcclCollective>(id, rank, size, device);
}

PeerRegion::PeerRegion(int r, int n, int dev, size_t cap_floats) : rank(r), size(n), device(dev), cap(cap_floats) {
  if (n < 1 || r < 0 || r >= n) throw Error(ErrorCode::InvalidConfig, "peer region: bad rank / size");
  CKC(cudaSetDevice(dev));
  CKC(cudaMalloc(&local, kFlagBytes + 2 * cap * 4));
  CKC(cudaMemset(local, 0, kFlagBytes));
  peers.assign(n, nullptr);
  peers[r] = local;
}
PeerRegion::~PeerRegion() {
  cudaSetDevice(device);
  for (int r = 0; r < size; ++r)
    if (peers[r] && peers[r] != local) cudaIpcCloseMemHandle(peers[r]);
  if (d_peers) cudaFree(d_peers);
  if (local) cudaFree(local);
}
void PeerRegion::handle(uint8_t out[kIpcHandleBytes]) const {
  cudaIpcMemHandle_t h;
  CKC(cudaIpcGetMemHandle(&h, local));
  static_assert(sizeof(h) == kIpcHandleBytes, "IPC handle size");
  std::memcpy(out, &h, kIpcHandleBytes);
}
void PeerRegion::open(const uint8_t* handles) {
  CKC(cudaSetDevice(device));
  for (int r = 0; r < size; ++r) {
    if (r == rank || peers[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + static_cast<size_t>(r) * kIpcHandleBytes, kIpcHandleBytes);
    void* p = nullptr;
    CKC(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    peers[r] = static_cast<char*>(p);
  }
  CKC(cudaMalloc(&d_peers, sizeof(char*) * size));
  CKC(cudaMemcpy(d_peers, peers.data(), sizeof(char*) * size, cudaMemcpyHostToDevice));
}
std::shared_ptr<Collective> make_peer(std::shared_ptr<PeerRegion> region) {
  if (!region->d_peers) throw Error(ErrorCode::InvalidConfig, "peer region not opened");
  return std::make_shared<PeerCollective>(std::move(region));
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
