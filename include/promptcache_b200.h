/*
 * promptcache_b200 — C ABI of the B200-native Prompt Cache hot path.
 *
 * The reference (arXiv 2311.04934 artifact, /root/reference/proj) exposes its
 * hot path as the C++ API in namespace pc::* and has no FFI of its own.  Each
 * entry point below replaces the reference interface cited beside it; a caller
 * binding this header (ctypes / cgo / JNI) gets the reference's behaviour with
 * every numeric op executed by sm_100a kernels.  No C++ types cross the ABI:
 * handles are opaque, arrays are plain pointers + sizes, strings are UTF-8.
 *
 * Errors: every int-returning call returns PCB_OK (0) or (pc::ErrorCode ordinal
 * + 1) — the exception the reference would have thrown (errors.hpp:8-30); the
 * message is in pcb_last_error() (thread-local).  char* results are malloc'd
 * (free with pcb_free) and NULL on error.  There is NO CPU fallback: without a
 * CUDA device, pcb_model_create fails with PCB_ERR_CUDA.
 */
#ifndef PROMPTCACHE_B200_H
#define PROMPTCACHE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PCB_OK = 0,
  PCB_ERR_SYNTAX = 1, PCB_ERR_MISSING_SCHEMA_ATTR, PCB_ERR_UNKNOWN_ROLE, PCB_ERR_TOKENIZER,
  PCB_ERR_FREE_TEXT_OVERFLOW, PCB_ERR_ARG_TOO_LONG, PCB_ERR_INVALID_CONFIG, PCB_ERR_POSITION_OUT_OF_RANGE,
  PCB_ERR_SHAPE_MISMATCH, PCB_ERR_UNKNOWN_MODULE, PCB_ERR_CAPACITY_EXCEEDED, PCB_ERR_IO,
  PCB_ERR_VERSION_MISMATCH, PCB_ERR_CONFIG_HASH_MISMATCH, PCB_ERR_VALIDATION_FAILED, PCB_ERR_POSITION_OVERLAP,
  PCB_ERR_UNKNOWN_CALL, PCB_ERR_RECURSION, PCB_ERR_DUPLICATE_NAME, PCB_ERR_INVALID_PROGRAM, PCB_ERR_INTERNAL,
  PCB_ERR_CUDA /* device failure (no reference equivalent) */
};
enum { PCB_DTYPE_F32 = 0, PCB_DTYPE_BF16 = 1 };
enum { PCB_TIER_FAST = 0, PCB_TIER_SLOW = 1 };

typedef struct pcb_schema pcb_schema;     /* SchemaDoc (+ llama2 chat expansion) + LayoutPlan */
typedef struct pcb_prompt pcb_prompt;     /* PromptDoc */
typedef struct pcb_model pcb_model;       /* pc::model::Model on one device */
typedef struct pcb_kv pcb_kv;             /* pc::model::KVState, device resident */
typedef struct pcb_store pcb_store;       /* pc::cache::ModuleStore */
typedef struct pcb_response pcb_response; /* pc::engine::ServeResponse */
typedef struct pcb_group pcb_group;       /* tensor-parallel ranks as threads of one process (tests) */
typedef struct pcb_peer pcb_peer;         /* this rank's CUDA-IPC region of a peer-memory TP group */

const char* pcb_last_error(void);
int pcb_last_error_code(void);
void pcb_free(void* p);
const char* pcb_version(void);

/* ---- PML (reference pml.hpp:142-155) and layout (layout.hpp:88-94) ---- */
int pcb_schema_parse(const char* pml, int expand_chat, pcb_schema** out); /* parse_schema + expand_chat_tags(llama2) + plan_layout */
int pcb_schema_from_ast(const char* ast_json, pcb_schema** out);          /* in-memory SchemaDoc (JSON interchange) + plan_layout */
void pcb_schema_destroy(pcb_schema* s);
char* pcb_schema_to_ast(const pcb_schema* s);
char* pcb_schema_serialize(const pcb_schema* s);                          /* pml::serialize(SchemaDoc) */
char* pcb_schema_plan_json(const pcb_schema* s);                          /* LayoutPlan, every field */
int pcb_prompt_parse(const char* pml, pcb_prompt** out);                  /* pml::parse_prompt */
int pcb_prompt_from_ast(const char* ast_json, pcb_prompt** out);
void pcb_prompt_destroy(pcb_prompt* p);
char* pcb_prompt_to_ast(const pcb_prompt* p);
char* pcb_prompt_serialize(const pcb_prompt* p);                          /* pml::serialize(PromptDoc) */
char* pcb_validate(const pcb_prompt* p, const pcb_schema* s);             /* ValidationReport::to_json */
char* pcb_resolve(const pcb_prompt* p, const pcb_schema* s);              /* layout::resolve_prompt, JSON */

/* ---- model config (model.cpp:59-96) ---- */
char* pcb_config_canonical(const char* config_json);                     /* ModelConfig::to_json */
int pcb_config_hash(const char* config_json, uint64_t* out);             /* ModelConfig::hash */
int64_t pcb_per_token_bytes(const char* config_json);                    /* cache::per_token_bytes (cache.cpp:36-38) */

/* ---- model (model.hpp:59-91) ---- */
int pcb_model_create(const char* config_json, int dtype, int device, pcb_model** out);
/* Head-sharded (tensor-parallel) model, SURVEY §8e config 5 -- no reference counterpart
 * (the reference is single-process): rank tp_rank of tp_size holds n_heads/tp_size heads of
 * every layer and of the module store, 4*hidden/tp_size MLP columns and vocab_size/tp_size
 * unembedding rows; collectives run over NCCL (nccl_id from pcb_nccl_unique_id on one rank,
 * shared out of band) or, for single-GPU tests, a pcb_group of threads.  Every rank then
 * calls the same pcb_store_* / pcb_serve sequence in lockstep. */
int pcb_nccl_unique_id(uint8_t* out_128_bytes);
int pcb_group_create(int size, pcb_group** out);
void pcb_group_destroy(pcb_group* g);
int pcb_model_create_tp(const char* config_json, int dtype, int device, int tp_rank, int tp_size,
                        const uint8_t* nccl_id, pcb_group* group, pcb_model** out);
/* Peer-memory transport (one process per rank; no NCCL): each rank creates its region
 * (cap_floats >= the largest collective: n_tokens * hidden for the all-reduces, n_tokens *
 * vocab/tp for the logits gather) and receives its 64-byte CUDA IPC handle; after every
 * rank has exchanged handles out of band (handles [tp_size][64] in rank order),
 * pcb_peer_open maps the peers and pcb_model_create_tp_peer builds the rank's model.
 * Collectives are one-shot kernels over the mapped slots (NVLink loads between GPUs). */
int pcb_peer_create(int tp_rank, int tp_size, int device, int64_t cap_floats, uint8_t* handle_out_64, pcb_peer** out);
int pcb_peer_open(pcb_peer* p, const uint8_t* handles);
void pcb_peer_destroy(pcb_peer* p);
int pcb_model_create_tp_peer(const char* config_json, int dtype, pcb_peer* peer, pcb_model** out);
void pcb_model_destroy(pcb_model* m);
/* Options (value 0/1 unless noted): "profile" (per-kernel-class CUDA-event timing),
 * "force_simt" / "force_simt_gemm" / "force_simt_attn" (testing: SIMT kernels only),
 * "chain" (few-token forwards as persistent chain kernels), "ln_fold" (LayerNorm folded into
 * the chain's GEMMs), "chain_attn" (a single request's attention as a chain phase),
 * "chain_group" (layers per chain launch when the attention is a chain phase, default 9;
 * 1 = one launch per layer), "zero_copy" (serve / serve_batch read cached modules in place
 * instead of the concat_kv copy), "attn_pair" (paired-tile prefill attention: 0 off, 1 when
 * it fills the GPU (default), 2 whenever it applies).
 * Returns PCB_ERR_INVALID_CONFIG for an unknown key. */
int pcb_model_set_option(pcb_model* m, const char* key, int64_t value);
int pcb_model_weight_checksum(pcb_model* m, const char* tensor, uint64_t* out);
/* Model::forward / forward_masked: logits_out [n][vocab] (host, may be NULL);
 * past may be NULL; mask [n][n] (NULL = causal); new_kv may be NULL. */
int pcb_model_forward(pcb_model* m, const int32_t* tokens, const int64_t* positions, int64_t n, const pcb_kv* past,
                      const uint8_t* mask, float* logits_out, pcb_kv** new_kv);
/* Model::generate: kv grows by n_steps rows; out[n_steps] */
int pcb_model_generate(pcb_model* m, pcb_kv* kv, int32_t last_token, int64_t last_position, int32_t n_steps,
                       int32_t* out);
int64_t pcb_model_forward_tokens(const pcb_model* m);
int64_t pcb_model_launches(const pcb_model* m);   /* kernels launched by this model so far */
/* with option "profile"=1: per kernel class {gemm, attention, assembly, other} CUDA-event
 * milliseconds, launch counts and algorithmic bytes / flops since the last call (resets) */
char* pcb_model_profile_json(pcb_model* m);
/* device timer on the model's stream: stop=0 records the start event; stop=1 records the end event,
 * waits for it and returns the elapsed device milliseconds */
int pcb_model_timer(pcb_model* m, int stop, double* ms_out);
int pcb_model_sync(pcb_model* m);

/* ---- KV blocks (model.hpp:34-44) ---- */
int64_t pcb_kv_rows(const pcb_kv* kv);
int pcb_kv_positions(const pcb_kv* kv, int64_t* out);
int pcb_kv_read(const pcb_kv* kv, int layer, int which /*0=K,1=V*/, float* out /*[rows][hidden]*/);
int pcb_kv_upload(pcb_model* m, const float* k, const float* v /*[L][rows][hidden]*/, const int64_t* positions,
                  int64_t rows, pcb_kv** out);
int pcb_kv_concat(pcb_model* m, const pcb_kv* const* kvs, int n, pcb_kv** out); /* engine::concat_kv (engine.cpp:174-185) */
void pcb_kv_destroy(pcb_kv* kv);

/* ---- module store (cache.hpp:46-108) ---- */
int pcb_store_create(pcb_model* m, pcb_store** out);
void pcb_store_destroy(pcb_store* s);
int pcb_store_set_capacity(pcb_store* s, int tier, int64_t bytes);
int pcb_store_encode_module(pcb_store* s, const pcb_schema* sc, const char* module, int tier); /* encode_module + insert */
int pcb_store_encode_schema(pcb_store* s, const pcb_schema* sc, int tier, int* count);        /* encode_schema */
int pcb_store_encode_scaffold(pcb_store* s, const pcb_schema* sc, const char* members_json, int tier);
/* Installs precomputed rows as module `module` of the schema (the reference's insert of an
 * encode_module result, cache.cpp:288-301 + cache.hpp:58; SURVEY §8b pcb_store_put_kv): kv must
 * hold exactly the module's own rows at its schema positions (PCB_ERR_SHAPE_MISMATCH
 * otherwise); the block is shared with the store, not copied (slow tier: pinned host copy). */
int pcb_store_put_kv(pcb_store* s, const pcb_schema* sc, const char* module, const pcb_kv* kv, int tier);
int pcb_store_lookup(pcb_store* s, const char* schema, const char* name, pcb_kv** out);       /* *out NULL on miss */
int64_t pcb_store_size(const pcb_store* s);
char* pcb_store_stats_json(const pcb_store* s);
int pcb_store_save(const pcb_store* s, const char* path);                                    /* PCST v1 */
int pcb_store_load(pcb_store* s, const char* path);

/* ---- engine (engine.hpp:50-62) ---- */
int pcb_serve(pcb_store* s, const pcb_schema* sc, const pcb_prompt* p, int max_new_tokens, int use_cache,
              int use_scaffolds, pcb_response** out);
// Micro-batched first-token serving (config 4: many requests, differing module
// combinations): micro_batch requests share one assembly launch and one suffix
// prefill.  Replaces a loop of engine::serve (reference engine.cpp:187-258) with
// max_new_tokens = 1; out[i] receives one response handle per prompt.
int pcb_serve_batch(pcb_store* s, const pcb_schema* sc, const pcb_prompt* const* prompts, int n, int micro_batch,
                    pcb_response** out);
int pcb_oracle_serve(pcb_model* m, const pcb_schema* sc, const pcb_prompt* p, int max_new_tokens,
                     pcb_response** out);
char* pcb_response_json(const pcb_response* r);                       /* ServeResponse::to_json (+device timings) */
int pcb_response_tokens(const pcb_response* r, int32_t* out, int cap); /* returns count */
int pcb_response_first_logits(const pcb_response* r, float* out, int cap);
void pcb_response_destroy(pcb_response* r);

#ifdef __cplusplus
}
#endif
#endif
