/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 *
 * Plain-C restatement of the reference's numeric hot path
 * (/root/reference/proj/core/src/model.cpp and engine.cpp:174-185), fp32
 * storage with fp64 accumulation exactly as the reference does.  Pinned against
 * the compiled reference (oracle/_ref) by tests/test_oracle.py.
 */
#ifndef PC_ORACLE_H
#define PC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n_layers, n_heads, head_dim, hidden, vocab_size;
  int pos_encoding; /* 0 rope, 1 alibi, 2 abs_table (model.hpp:12) */
  int64_t max_position;
  uint64_t seed;
} pco_config;

typedef struct pco_model pco_model;

uint64_t pco_fnv1a64(const void* data, uint64_t len);
uint64_t pco_splitmix64(uint64_t x);
/* fill_uniform (model.cpp:122-127) */
void pco_fill_uniform(float* out, uint64_t count, const char* name, uint64_t seed, float scale);

pco_model* pco_model_create(const pco_config* cfg);
void pco_model_destroy(pco_model* m);
/* Model::weight_checksum (model.cpp:248-267) */
int pco_weight_checksum(const pco_model* m, const char* name, uint64_t* out);

/* Model::run (model.cpp:304-443).  past_k/past_v: [n_layers][P][hidden] or NULL
 * when P == 0; mask: [n][n] or NULL.  logits_out: [n][vocab] (may be NULL);
 * new_k/new_v: [n_layers][n][hidden] (may be NULL).  Returns 0 or an error code. */
int pco_forward(const pco_model* m, const int32_t* tokens, const int64_t* pos, int64_t n,
                const float* past_k, const float* past_v, const int64_t* past_pos, int64_t P,
                const uint8_t* mask, float* logits_out, float* new_k, float* new_v);

/* argmax_lowest (model.cpp:457-462) */
int pco_argmax_lowest(const float* logits, int n);

#ifdef __cplusplus
}
#endif
#endif
