/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 * See pc_oracle.h.  Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj/core/src). */
#include "pc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* model.cpp:16-33 */
uint64_t pco_fnv1a64(const void* data, uint64_t len) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 14695981039346656037ULL;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

uint64_t pco_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* Pcg32 (model.hpp:127-139) */
typedef struct { uint64_t state; } pcg32;
static uint32_t pcg_next(pcg32* g) {
  uint64_t old = g->state;
  g->state = old * 6364136223846793005ULL + 1442695040888963407ULL;
  uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = (uint32_t)(old >> 59u);
  return (xs >> rot) | (xs << ((-rot) & 31u));
}
static void pcg_init(pcg32* g, uint64_t seed) {
  g->state = seed + 1442695040888963407ULL;
  (void)pcg_next(g);
}

/* fill_uniform (model.cpp:122-127): symmetric(scale) = (2*uniform-1)*scale in fp32 */
void pco_fill_uniform(float* out, uint64_t count, const char* name, uint64_t seed, float scale) {
  pcg32 g;
  pcg_init(&g, pco_splitmix64(pco_fnv1a64(name, strlen(name)) ^ pco_splitmix64(seed)));
  for (uint64_t i = 0; i < count; ++i) {
    volatile float u = (float)(pcg_next(&g) >> 8) * (1.0f / 16777216.0f);
    volatile float t = 2.0f * u - 1.0f;
    out[i] = t * scale;
  }
}

typedef struct {
  float *wq, *wk, *wv, *wo, *w1, *w2;
} pco_layer;

struct pco_model {
  pco_config c;
  float *embed, *unembed;
  pco_layer* layers;
  double *rope_cos, *rope_sin;
  float* alibi;
  float* abs_table;
};

static float* falloc(uint64_t n) { return (float*)malloc(n * sizeof(float)); }

/* Model::Model (model.cpp:183-246); LN gamma = 1, beta = 0 so they are implicit. */
pco_model* pco_model_create(const pco_config* cfg) {
  const pco_config* c = cfg;
  if (c->hidden != c->n_heads * c->head_dim || c->head_dim % 2) return NULL;
  pco_model* m = (pco_model*)calloc(1, sizeof(pco_model));
  m->c = *cfg;
  const int d = c->hidden;
  const float ws = 1.0f / sqrtf((float)d);
  m->embed = falloc((uint64_t)c->vocab_size * d);
  m->unembed = falloc((uint64_t)c->vocab_size * d);
  pco_fill_uniform(m->embed, (uint64_t)c->vocab_size * d, "embed", c->seed, 0.1f);
  pco_fill_uniform(m->unembed, (uint64_t)c->vocab_size * d, "unembed", c->seed, ws);
  m->layers = (pco_layer*)calloc(c->n_layers, sizeof(pco_layer));
  char name[64];
  for (int l = 0; l < c->n_layers; ++l) {
    pco_layer* L = &m->layers[l];
    float** slots[6] = {&L->wq, &L->wk, &L->wv, &L->wo, &L->w1, &L->w2};
    const char* nm[6] = {"wq", "wk", "wv", "wo", "w1", "w2"};
    for (int t = 0; t < 6; ++t) {
      uint64_t cnt = (t >= 4) ? (uint64_t)4 * d * d : (uint64_t)d * d;
      float sc = (t == 5) ? 1.0f / sqrtf((float)(4 * d)) : ws;
      *slots[t] = falloc(cnt);
      snprintf(name, sizeof name, "layer%d.%s", l, nm[t]);
      pco_fill_uniform(*slots[t], cnt, name, c->seed, sc);
    }
  }
  if (c->pos_encoding == 0) { /* model.cpp:220-230 */
    int half = c->head_dim / 2;
    m->rope_cos = (double*)malloc(sizeof(double) * c->max_position * half);
    m->rope_sin = (double*)malloc(sizeof(double) * c->max_position * half);
    for (int64_t p = 0; p < c->max_position; ++p)
      for (int i = 0; i < half; ++i) {
        double theta = pow(10000.0, -2.0 * i / c->head_dim);
        m->rope_cos[p * half + i] = cos(p * theta);
        m->rope_sin[p * half + i] = sin(p * theta);
      }
  }
  if (c->pos_encoding == 1) { /* model.cpp:231-236 */
    m->alibi = falloc(c->n_heads);
    for (int h = 0; h < c->n_heads; ++h) m->alibi[h] = (float)pow(2.0, -8.0 * (h + 1) / c->n_heads);
  }
  if (c->pos_encoding == 2) { /* model.cpp:237-245 */
    m->abs_table = falloc((uint64_t)c->max_position * d);
    for (int64_t p = 0; p < c->max_position; ++p)
      for (int i = 0; i < d / 2; ++i) {
        double theta = p / pow(10000.0, 2.0 * i / d);
        m->abs_table[p * d + 2 * i] = (float)sin(theta);
        m->abs_table[p * d + 2 * i + 1] = (float)cos(theta);
      }
  }
  return m;
}

void pco_model_destroy(pco_model* m) {
  if (!m) return;
  free(m->embed);
  free(m->unembed);
  for (int l = 0; l < m->c.n_layers; ++l) {
    pco_layer* L = &m->layers[l];
    free(L->wq); free(L->wk); free(L->wv); free(L->wo); free(L->w1); free(L->w2);
  }
  free(m->layers);
  free(m->rope_cos); free(m->rope_sin); free(m->alibi); free(m->abs_table);
  free(m);
}

/* Model::weight_checksum (model.cpp:248-267) */
int pco_weight_checksum(const pco_model* m, const char* name, uint64_t* out) {
  const int d = m->c.hidden;
  if (!strcmp(name, "embed")) { *out = pco_fnv1a64(m->embed, 4ull * m->c.vocab_size * d); return 0; }
  if (!strcmp(name, "unembed")) { *out = pco_fnv1a64(m->unembed, 4ull * m->c.vocab_size * d); return 0; }
  char buf[64];
  const char* nm[6] = {"wq", "wk", "wv", "wo", "w1", "w2"};
  for (int l = 0; l < m->c.n_layers; ++l)
    for (int t = 0; t < 6; ++t) {
      snprintf(buf, sizeof buf, "layer%d.%s", l, nm[t]);
      if (!strcmp(buf, name)) {
        const pco_layer* L = &m->layers[l];
        const float* p[6] = {L->wq, L->wk, L->wv, L->wo, L->w1, L->w2};
        uint64_t cnt = (t >= 4) ? 4ull * d * d : (uint64_t)d * d;
        *out = pco_fnv1a64(p[t], cnt * 4);
        return 0;
      }
    }
  return 21; /* Internal */
}

/* dotf (model.cpp:136-147): 4 fp64 lanes, fixed combine order */
static float dotf(const float* a, const float* b, int n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    s0 += (double)a[i] * (double)b[i];
    s1 += (double)a[i + 1] * (double)b[i + 1];
    s2 += (double)a[i + 2] * (double)b[i + 2];
    s3 += (double)a[i + 3] * (double)b[i + 3];
  }
  for (; i < n; ++i) s0 += (double)a[i] * (double)b[i];
  return (float)((s0 + s1) + (s2 + s3));
}

/* linear (model.cpp:149-154): out[i][o] = dot(x[i], w[o]) */
static void linear(const float* x, const float* w, float* out, int64_t n, int in, int outdim) {
  for (int64_t i = 0; i < n; ++i)
    for (int o = 0; o < outdim; ++o) out[i * outdim + o] = dotf(x + i * in, w + (int64_t)o * in, in);
}

/* layer_norm (model.cpp:156-174) with gamma = 1, beta = 0 */
static void layer_norm(const float* x, float* out, int64_t n, int d) {
  for (int64_t i = 0; i < n; ++i) {
    const float* row = x + i * d;
    double mean = 0.0;
    for (int j = 0; j < d; ++j) mean += row[j];
    mean /= d;
    double var = 0.0;
    for (int j = 0; j < d; ++j) {
      double c = row[j] - mean;
      var += c * c;
    }
    var /= d;
    double inv = 1.0 / sqrt(var + 1e-5);
    for (int j = 0; j < d; ++j) out[i * d + j] = (float)((row[j] - mean) * inv) * 1.0f + 0.0f;
  }
}

/* gelu (model.cpp:176-179) */
static float gelu(float x) {
  double t = 0.7978845608028654 * (x + 0.044715 * x * x * x);
  return (float)(0.5 * x * (1.0 + tanh(t)));
}

/* rope_rotate_with_table (model.cpp:273-282) */
static void rope(const pco_model* m, float* v, int64_t p) {
  int half = m->c.head_dim / 2;
  const double* cs = m->rope_cos + p * half;
  const double* sn = m->rope_sin + p * half;
  for (int i = 0; i < half; ++i) {
    double a = v[2 * i], b = v[2 * i + 1];
    v[2 * i] = (float)(a * cs[i] - b * sn[i]);
    v[2 * i + 1] = (float)(a * sn[i] + b * cs[i]);
  }
}

/* Model::run (model.cpp:304-443) */
int pco_forward(const pco_model* m, const int32_t* tokens, const int64_t* pos, int64_t n,
                const float* past_k, const float* past_v, const int64_t* past_pos, int64_t P,
                const uint8_t* mask, float* logits_out, float* new_k, float* new_v) {
  const pco_config* c = &m->c;
  const int d = c->hidden, hd = c->head_dim, H = c->n_heads;
  for (int64_t i = 0; i < n; ++i) {
    if (pos[i] < 0 || pos[i] >= c->max_position) return 8;  /* PositionOutOfRange */
    if (tokens[i] < 0 || tokens[i] >= c->vocab_size) return 9; /* ShapeMismatch */
  }
  const int64_t total = P + n;
  const float inv_sqrt = 1.0f / sqrtf((float)hd);
  float* h = falloc(n * d);
  float* norm = falloc(n * d);
  float* q = falloc(n * d);
  float* kn = falloc(n * d);
  float* vn = falloc(n * d);
  float* attn = falloc(n * d);
  float* proj = falloc(n * d);
  float* mid = falloc(n * 4 * d);
  float* kbuf = falloc(total * d);
  float* vbuf = falloc(total * d);
  int64_t* posbuf = (int64_t*)malloc(sizeof(int64_t) * total);
  float* scores = falloc(total);
  double* acc = (double*)malloc(sizeof(double) * hd);
  for (int64_t j = 0; j < P; ++j) posbuf[j] = past_pos ? past_pos[j] : j;
  for (int64_t i = 0; i < n; ++i) posbuf[P + i] = pos[i];

  for (int64_t i = 0; i < n; ++i) { /* embed (354-362) */
    memcpy(h + i * d, m->embed + (int64_t)tokens[i] * d, d * sizeof(float));
    if (c->pos_encoding == 2)
      for (int j = 0; j < d; ++j) h[i * d + j] += m->abs_table[pos[i] * d + j];
  }
  for (int l = 0; l < c->n_layers; ++l) {
    const pco_layer* L = &m->layers[l];
    layer_norm(h, norm, n, d);
    linear(norm, L->wq, q, n, d, d);
    linear(norm, L->wk, kn, n, d, d);
    linear(norm, L->wv, vn, n, d, d);
    if (c->pos_encoding == 0)
      for (int64_t i = 0; i < n; ++i)
        for (int hh = 0; hh < H; ++hh) {
          rope(m, q + i * d + hh * hd, pos[i]);
          rope(m, kn + i * d + hh * hd, pos[i]);
        }
    if (P > 0) {
      memcpy(kbuf, past_k + (int64_t)l * P * d, P * d * sizeof(float));
      memcpy(vbuf, past_v + (int64_t)l * P * d, P * d * sizeof(float));
    }
    memcpy(kbuf + P * d, kn, n * d * sizeof(float));
    memcpy(vbuf + P * d, vn, n * d * sizeof(float));
    if (new_k) memcpy(new_k + (int64_t)l * n * d, kn, n * d * sizeof(float));
    if (new_v) memcpy(new_v + (int64_t)l * n * d, vn, n * d * sizeof(float));

    for (int64_t i = 0; i < n; ++i)
      for (int hh = 0; hh < H; ++hh) { /* attention (401-427) */
        const float* qv = q + i * d + hh * hd;
        const int64_t limit = mask ? n - 1 : P + i;
        double maxs = -1e30;
        for (int64_t j = 0; j <= limit; ++j) {
          if (mask && !mask[i * n + j]) continue;
          float s = dotf(qv, kbuf + j * d + hh * hd, hd) * inv_sqrt;
          if (c->pos_encoding == 1) s += m->alibi[hh] * (float)(posbuf[j] - posbuf[P + i]);
          scores[j] = s;
          if (s > maxs) maxs = s;
        }
        double denom = 0.0;
        for (int x = 0; x < hd; ++x) acc[x] = 0.0;
        for (int64_t j = 0; j <= limit; ++j) {
          if (mask && !mask[i * n + j]) continue;
          double w = exp((double)scores[j] - maxs);
          denom += w;
          const float* vv = vbuf + j * d + hh * hd;
          for (int x = 0; x < hd; ++x) acc[x] += w * vv[x];
        }
        for (int x = 0; x < hd; ++x) attn[i * d + hh * hd + x] = (float)(acc[x] / denom);
      }
    linear(attn, L->wo, proj, n, d, d);
    for (int64_t i = 0; i < n * d; ++i) h[i] += proj[i];
    layer_norm(h, norm, n, d);
    linear(norm, L->w1, mid, n, d, 4 * d);
    for (int64_t i = 0; i < n * 4 * d; ++i) mid[i] = gelu(mid[i]);
    linear(mid, L->w2, proj, n, 4 * d, d);
    for (int64_t i = 0; i < n * d; ++i) h[i] += proj[i];
  }
  layer_norm(h, norm, n, d);
  if (logits_out) linear(norm, m->unembed, logits_out, n, d, c->vocab_size);
  free(h); free(norm); free(q); free(kn); free(vn); free(attn); free(proj); free(mid);
  free(kbuf); free(vbuf); free(posbuf); free(scores); free(acc);
  return 0;
}

/* argmax_lowest (model.cpp:457-462) */
int pco_argmax_lowest(const float* logits, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (logits[i] > logits[best]) best = i;
  return best;
}
