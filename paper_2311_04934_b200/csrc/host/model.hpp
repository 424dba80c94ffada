// Device model: config, weights in HBM, KV blocks and the forward orchestration
// of the hot path.  API shape mirrors the reference's pc::model (model.hpp:12-139)
// — ModelConfig JSON/hash, Model::forward / forward_masked / generate,
// weight_checksum — while every op runs as an sm_100a kernel (kernels.cuh).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "errors.hpp"

namespace pcb::coll {
class Collective;
}

namespace pcb::model {

enum class PosEncoding { Rope, Alibi, AbsTable };

struct ModelConfig {
  int n_layers = 4;
  int n_heads = 8;
  int head_dim = 32;
  int hidden = 256;
  int vocab_size = 512;
  PosEncoding pos_encoding = PosEncoding::Rope;
  int64_t max_position = 8192;
  int bytes_per_element = 2;  // store accounting (reference semantics)
  uint64_t seed = 42;

  static ModelConfig from_json(const std::string& text);  // reference model.cpp:59-80
  std::string to_json() const;                            // canonical (model.cpp:82-94)
  uint64_t hash() const;                                  // FNV-1a of to_json()
};

uint64_t fnv1a64(const void* data, size_t len);
uint64_t splitmix64(uint64_t x);

enum DType : int { F32 = 0, BF16 = 1 };

// KV rows for every layer, layout [L][2][cap][hidden] in one allocation (device,
// or pinned host for the slow tier).  K is stored post-RoPE, V raw; position
// IDs ride along on the host (reference KVState, model.hpp:34-44).
struct KVBlock {
  int dtype = BF16, n_layers = 0, hidden = 0;
  int64_t rows = 0, cap = 0;
  void* data = nullptr;
  bool host = false;
  bool view = false;  // non-owning window into another allocation
  std::vector<int64_t> positions;

  KVBlock() = default;
  KVBlock(const KVBlock&) = delete;
  KVBlock& operator=(const KVBlock&) = delete;
  ~KVBlock();

  size_t elem() const { return dtype == F32 ? 4 : 2; }
  size_t row_bytes() const { return static_cast<size_t>(hidden) * elem(); }
  size_t plane_bytes() const { return static_cast<size_t>(cap) * row_bytes(); }
  size_t bytes() const { return plane_bytes() * 2 * n_layers; }
  char* plane(int l, int which) const { return static_cast<char*>(data) + (static_cast<size_t>(l) * 2 + which) * plane_bytes(); }
  char* k(int l) const { return plane(l, 0); }
  char* v(int l) const { return plane(l, 1); }
};
using KVPtr = std::shared_ptr<KVBlock>;

struct ForwardOutput {
  std::vector<float> logits;  // [seq][vocab] host
  int64_t seq = 0;
  int vocab = 0;
  KVPtr new_kv;
  const float* row(int64_t i) const { return logits.data() + i * vocab; }
};

struct Weights;
struct Workspace;

class Model {
 public:
  // Tensor parallel (head-sharded) when tp_size > 1: this rank holds
  // heads [r H/T, (r+1) H/T) of Wq/Wk/Wv and its KV, the matching input columns of Wo,
  // MLP columns [r 4d/T, ...) of W1 and input columns of W2, and vocab rows
  // [r V/T, ...) of the unembedding; `comm` all-reduces after Wo and W2 and gathers
  // the vocab shards of the logits.
  Model(const ModelConfig& config, int dtype, int device, int tp_rank = 0, int tp_size = 1,
        std::shared_ptr<coll::Collective> comm = nullptr);
  ~Model();
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;

  const ModelConfig& config() const { return cfg_; }
  int dtype() const { return dtype_; }
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  int tp_rank() const { return tp_rank_; }
  int tp_size() const { return tp_size_; }
  int kv_width() const { return dl_; }  // hidden columns of K/V this rank stores

  KVPtr alloc_kv(int64_t cap, bool host = false) const;

  // ---- hot-path core ----
  // Runs n tokens over `kv` whose first kv.rows rows are the past (P).  The n
  // new K/V rows are written in place at rows [P, P+n) (kv.cap >= P+n), so an
  // assembled request cache needs no copy.  Computes logits for the last
  // `logit_rows` rows into device memory (0 = none: module precompute skips the
  // unembed).  mask ([n][n], P == 0) or block ids ([n], -1 = sees all earlier
  // rows) select exact masked attention (reference forward_masked / oracle).
  void run(const int32_t* tokens, const int64_t* positions, int64_t n, KVBlock& kv, const uint8_t* mask,
           const int32_t* block_ids, int64_t logit_rows);
  // Batched forward (B requests, micro-batched suffix prefill): each item's n tokens
  // run over its own cache (all caches of one call share a capacity); logits of the
  // last row of every item land in device_logits() rows [0, B).
  struct BatchItem {
    const int32_t* tokens;
    const int64_t* positions;
    int64_t n;
    KVBlock* kv;
  };
  void run_batch(const std::vector<BatchItem>& items, bool last_row_logits);
  // The next run()/run_batch() waits for events[l] before layer l's attention (past K/V
  // rows still streaming in, e.g. the pinned-host tier); consumed by that call.
  void set_layer_events(const cudaEvent_t* events, int n) { layer_events_.assign(events, events + n); }
  // Zero-copy cached prefix (engine serve): until cleared, a single-request forward treats
  // the request cache's rows [0, sum of the blocks' rows) as these blocks' rows, read in
  // place by the chain's attention phase (those cache rows are never filled).  Only valid
  // while fused_attention_ok() holds for every forward of the request; run() throws otherwise.
  void set_kv_prefix(const std::vector<const KVBlock*>& blocks);
  void clear_kv_prefix() { kv_prefix_.clear(); kv_prefix_rows_ = 0; kv_prefix_batch_.clear(); }
  // the same for run_batch: request b's cache rows [0, its blocks' rows) are its blocks
  // (batched attention kernel, per-request segment tables); needs batched_zero_copy_ok()
  void set_kv_prefix_batch(const std::vector<std::vector<const KVBlock*>>& per_request);
  bool batched_zero_copy_ok() const;
  bool fused_attention_ok(int64_t n) const;  // n-token single-request forwards use the chain attention phase
  const float* device_logits() const;  // [logit_rows][vocab] after run()
  int32_t* device_argmax() const;      // scratch int32 slots
  void argmax_last(int64_t logit_rows);  // device argmax of each logits row -> device_argmax()

  // ---- reference-shaped API (model.hpp:59-91) ----
  ForwardOutput forward(const std::vector<int>& tokens, const std::vector<int64_t>& positions,
                        const KVBlock* past = nullptr);
  ForwardOutput forward_masked(const std::vector<int>& tokens, const std::vector<int64_t>& positions,
                               const std::vector<uint8_t>& mask);
  std::vector<int> generate(KVBlock& kv, int last_token, int64_t last_position, int n_steps);
  uint64_t weight_checksum(const std::string& tensor_name) const;

  // Copies rows [0, src.rows) of `src` into `dst` rows [dst_row, ...) (D2D or H2D).
  void copy_rows(const KVBlock& src, KVBlock& dst, int64_t dst_row) const;
  KVPtr to_host(const KVBlock& src) const;  // pinned host copy (slow tier)

  // ---- live per-kernel-class timing (CUDA events on the model stream) ----
  enum ProfCat { PROF_GEMM = 0, PROF_ATTN = 1, PROF_ASM = 2, PROF_OTHER = 3, PROF_N = 4 };
  void set_profiling(bool on);
  void prof_begin();
  void prof_end(int cat, double alg_bytes, double alg_flops);
  std::string profile_json();  // syncs, returns per-class {ms, launches, bytes, flops}, resets

  mutable std::atomic<long> forward_tokens{0};
  bool force_simt = false;       // testing: route bf16 GEMM/attention through SIMT kernels
  bool force_simt_gemm = false;  // testing: SIMT GEMM only
  bool force_simt_attn = false;  // testing: SIMT attention only
  int attn_pair = 1;             // paired-tile prefill attention: 0 off, 1 when it fills the GPU, 2 always
  bool use_chain = true;         // few-token GEMM/LN segments as one persistent chain kernel (PCB_CHAIN=0: off)
  bool ln_fold = true;           // chain: LayerNorm folded into the neighbouring GEMMs (PCB_LN_FOLD=0: off)
  int chain_group = 9;           // chain: layers per launch when the attention is a chain phase (1: per layer)
  bool chain_attn = true;        // chain: a single request's attention as the chain's first phase (PCB_CHAIN_ATTN=0: off)
  bool zero_copy = true;         // serve: cached modules read in place by the attention, no assembly copy (PCB_ZERO_COPY=0: off)
  int64_t launches = 0;          // kernels launched by run() (bench evidence)

 private:
  void validate(const int32_t* tokens, const int64_t* positions, int64_t n, const KVBlock& kv) const;
  void gemm(const void* A, const void* W, int64_t M, int N, int K, const void* epi, bool packed);
  void run_impl(const BatchItem* items, int B, const uint8_t* mask, const int32_t* block_ids, int64_t logit_rows,
                bool per_segment_logits);
  void chain(const void* steps, int n_steps);  // kern::ChainStep[n_steps]

  ModelConfig cfg_;
  int dtype_, device_;
  int tp_rank_ = 0, tp_size_ = 1;
  int dl_ = 0, fl_ = 0, vl_ = 0;  // local attention width, MLP width, vocab rows
  std::shared_ptr<coll::Collective> comm_;
  std::vector<cudaEvent_t> layer_events_;
  const int32_t* device_token_ = nullptr;  // generate(): this step's token is already on the device
  std::vector<const KVBlock*> kv_prefix_;
  std::vector<std::vector<const KVBlock*>> kv_prefix_batch_;
  int64_t kv_prefix_rows_ = 0;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<Weights> w_;
  std::unique_ptr<Workspace> ws_;
  struct Prof;
  std::unique_ptr<Prof> prof_;
};

int argmax_lowest(const float* logits, int n);

}  // namespace pcb::model
