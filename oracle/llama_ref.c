/* CPU oracle of the chunked-prefill compute side — see llama_ref.h.
 * TEST INFRASTRUCTURE ONLY. Standard Llama-3 block (RMSNorm, RoPE theta,
 * GQA causal attention, SwiGLU), fp32 math, bf16 rounding at the points the
 * GPU rounds. Parity with the reference: unpinned (the reference has no model). */
#include "llama_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------ generator */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint16_t ref_bf16_from_float(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu)) return (uint16_t)((x >> 16) | 0x40u);
  x += 0x7FFFu + ((x >> 16) & 1u); /* round to nearest even */
  return (uint16_t)(x >> 16);
}

float ref_bf16_to_float(uint16_t b) {
  uint32_t x = (uint32_t)b << 16;
  float f;
  memcpy(&f, &x, 4);
  return f;
}

static float round_bf16(float f) { return ref_bf16_to_float(ref_bf16_from_float(f)); }

uint16_t ref_weight_bits(unsigned long long seed, uint32_t tensor_id, uint64_t logical_index, float scale) {
  const uint64_t h = mix64(seed ^ mix64(((uint64_t)tensor_id << 40) ^ logical_index));
  const float u = (float)(int32_t)(h >> 40) * (1.0f / 8388608.0f) - 1.0f;
  return ref_bf16_from_float(u * scale);
}

void ref_weight_matrix_bits(unsigned long long seed, uint32_t tid, long long rows, long long cols, float scale,
                            uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (long long r = 0; r < rows; ++r)
    for (long long k = 0; k < cols; ++k)
      out[r * cols + k] = ref_weight_bits(seed, tid, (uint64_t)(r * cols + k), scale);
}

void ref_weight_row_bits(unsigned long long seed, uint32_t tid, long long row, long long cols, float scale,
                         uint16_t* out) {
  for (long long k = 0; k < cols; ++k) out[k] = ref_weight_bits(seed, tid, (uint64_t)(row * cols + k), scale);
}

void ref_round_bf16(float* x, long long n) {
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < n; ++i) x[i] = round_bf16(x[i]);
}

enum { W_Q = 0, W_K = 1, W_V = 2, W_O = 3, W_GATE = 4, W_UP = 5, W_DOWN = 6 };
#define TID_EMBED (1u << 20)
#define TID_LMHEAD ((1u << 20) + 1u)

/* ------------------------------------------------------------ model */
typedef struct layer_w {
  float *wq, *wk, *wv, *wo, *wg, *wu, *wd; /* row-major [out][in] */
} layer_w;

struct ref_model {
  ref_config c;
  long long max_tokens;
  int G, qd, kvd;
  float s_h, s_o, s_f;
  float* kv;     /* [L][2][nkv][max_tokens][hd] */
  float* rope;   /* [max_tokens][hd/2][2] */
  layer_w* cached;
  int n_cached;
  /* current chunk */
  long long start;
  int len;
  float* h;      /* [len][H] */
};

static float* gen_matrix(const ref_model* m, uint32_t tid, int rows, int cols, float scale) {
  float* w = (float*)malloc((size_t)rows * cols * sizeof(float));
  if (!w) return NULL;
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int k = 0; k < cols; ++k)
      w[(size_t)r * cols + k] = ref_bf16_to_float(ref_weight_bits(m->c.seed, tid, (uint64_t)r * cols + k, scale));
  return w;
}

static int gen_layer(const ref_model* m, int l, layer_w* lw) {
  const int H = m->c.hidden, F = m->c.ffn;
  lw->wq = gen_matrix(m, 16u * l + W_Q, m->qd, H, m->s_h);
  lw->wk = gen_matrix(m, 16u * l + W_K, m->kvd, H, m->s_h);
  lw->wv = gen_matrix(m, 16u * l + W_V, m->kvd, H, m->s_h);
  lw->wo = gen_matrix(m, 16u * l + W_O, H, m->qd, m->s_o);
  lw->wg = gen_matrix(m, 16u * l + W_GATE, F, H, m->s_h);
  lw->wu = gen_matrix(m, 16u * l + W_UP, F, H, m->s_h);
  lw->wd = gen_matrix(m, 16u * l + W_DOWN, H, F, m->s_f);
  return (lw->wq && lw->wk && lw->wv && lw->wo && lw->wg && lw->wu && lw->wd) ? 0 : -1;
}

static void free_layer(layer_w* lw) {
  free(lw->wq);
  free(lw->wk);
  free(lw->wv);
  free(lw->wo);
  free(lw->wg);
  free(lw->wu);
  free(lw->wd);
  memset(lw, 0, sizeof *lw);
}

ref_model* ref_create(const ref_config* cfg, long long max_tokens, long long cache_weight_bytes) {
  ref_model* m = (ref_model*)calloc(1, sizeof *m);
  if (!m) return NULL;
  m->c = *cfg;
#ifdef _OPENMP
  if (cfg->threads > 0) omp_set_num_threads(cfg->threads);
#endif
  m->max_tokens = max_tokens;
  m->G = cfg->n_heads / cfg->n_kv_heads;
  m->qd = cfg->n_heads * cfg->head_dim;
  m->kvd = cfg->n_kv_heads * cfg->head_dim;
  m->s_h = 1.0f / sqrtf((float)cfg->hidden);
  m->s_o = 1.0f / sqrtf((float)(cfg->n_heads * cfg->head_dim));
  m->s_f = 1.0f / sqrtf((float)cfg->ffn);
  const size_t kv_elems = (size_t)cfg->n_layers * 2 * cfg->n_kv_heads * (size_t)max_tokens * cfg->head_dim;
  m->kv = (float*)calloc(kv_elems, sizeof(float));
  const int half = cfg->head_dim / 2;
  m->rope = (float*)malloc((size_t)max_tokens * half * 2 * sizeof(float));
  if (!m->kv || !m->rope) {
    ref_destroy(m);
    return NULL;
  }
  for (long long p = 0; p < max_tokens; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = pow((double)cfg->rope_theta, -2.0 * i / cfg->head_dim);
      const double a = (double)p * inv;
      m->rope[(p * half + i) * 2] = (float)cos(a);
      m->rope[(p * half + i) * 2 + 1] = (float)sin(a);
    }
  const long long per_layer =
      4LL * ((long long)m->qd * cfg->hidden + 2LL * m->kvd * cfg->hidden + (long long)cfg->hidden * m->qd +
             3LL * cfg->ffn * cfg->hidden);
  if (cache_weight_bytes >= per_layer * cfg->n_layers) {
    m->cached = (layer_w*)calloc((size_t)cfg->n_layers, sizeof(layer_w));
    for (int l = 0; l < cfg->n_layers; ++l)
      if (gen_layer(m, l, &m->cached[l])) {
        ref_destroy(m);
        return NULL;
      }
    m->n_cached = cfg->n_layers;
  }
  return m;
}

void ref_destroy(ref_model* m) {
  if (!m) return;
  for (int l = 0; l < m->n_cached; ++l) free_layer(&m->cached[l]);
  free(m->cached);
  free(m->kv);
  free(m->rope);
  free(m->h);
  free(m);
}

float* ref_kv(ref_model* m) { return m->kv; }
long long ref_max_tokens(const ref_model* m) { return m->max_tokens; }

static float* kv_at(ref_model* m, int layer, int kv, int head, long long pos) {
  return m->kv + ((((size_t)layer * 2 + kv) * m->c.n_kv_heads + head) * (size_t)m->max_tokens + pos) * m->c.head_dim;
}

/* ------------------------------------------------------------ math */
/* out[t][n] = sum_k x[t][k] * w[n][k] */
static void matmul(const float* x, const float* w, float* out, int T, int N, int K) {
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) {
    const float* wr = w + (size_t)n * K;
    for (int t = 0; t < T; ++t) {
      const float* xr = x + (size_t)t * K;
      float acc = 0.f;
      for (int k = 0; k < K; ++k) acc += xr[k] * wr[k];
      out[(size_t)t * N + n] = acc;
    }
  }
}

static void rmsnorm_bf16(const float* h, float* y, int T, int H, float eps) {
  for (int t = 0; t < T; ++t) {
    double ss = 0.0;
    for (int i = 0; i < H; ++i) ss += (double)h[(size_t)t * H + i] * h[(size_t)t * H + i];
    const float r = 1.0f / sqrtf((float)(ss / H) + eps);
    for (int i = 0; i < H; ++i) y[(size_t)t * H + i] = round_bf16(h[(size_t)t * H + i] * r); /* gamma = 1 */
  }
}

static void rope_rows(const ref_model* m, float* x, int T, int heads, long long pos0) {
  const int hd = m->c.head_dim, half = hd / 2;
  for (int t = 0; t < T; ++t)
    for (int h = 0; h < heads; ++h) {
      float* v = x + ((size_t)t * heads + h) * hd;
      const float* cs = m->rope + (size_t)(pos0 + t) * half * 2;
      for (int i = 0; i < half; ++i) {
        const float a = v[i], b = v[i + half], c = cs[2 * i], s = cs[2 * i + 1];
        v[i] = a * c - b * s;
        v[i + half] = b * c + a * s;
      }
    }
}

/* attention of T queries (positions pos0..) over cached keys [0, pos0 + t] */
static void attention(ref_model* m, int layer, const float* q, float* out, int T, long long pos0) {
  const int hd = m->c.head_dim, nq = m->c.n_heads;
  const float scale = 1.0f / sqrtf((float)hd);
#pragma omp parallel
  {
    float* sc = (float*)malloc((size_t)(pos0 + T) * sizeof(float));
#pragma omp for collapse(2) schedule(dynamic, 4)
    for (int t = 0; t < T; ++t)
      for (int h = 0; h < nq; ++h) {
        const long long p = pos0 + t;
        const int g = h / m->G;
        const float* qv = q + ((size_t)t * nq + h) * hd;
        float mx = -INFINITY;
        for (long long j = 0; j <= p; ++j) {
          const float* kv = kv_at(m, layer, 0, g, j);
          float s = 0.f;
          for (int d = 0; d < hd; ++d) s += qv[d] * kv[d];
          s *= scale;
          sc[j] = s;
          if (s > mx) mx = s;
        }
        double den = 0.0;
        for (long long j = 0; j <= p; ++j) {
          sc[j] = expf(sc[j] - mx);
          den += sc[j];
        }
        float* o = out + ((size_t)t * nq + h) * hd;
        for (int d = 0; d < hd; ++d) o[d] = 0.f;
        for (long long j = 0; j <= p; ++j) {
          const float* vv = kv_at(m, layer, 1, g, j);
          const float w = (float)(sc[j] / den);
          for (int d = 0; d < hd; ++d) o[d] += w * vv[d];
        }
        for (int d = 0; d < hd; ++d) o[d] = round_bf16(o[d]);
      }
    free(sc);
  }
}

int ref_begin_chunk(ref_model* m, const int32_t* tokens, long long start, int len) {
  if (start < 0 || start + len > m->max_tokens || len < 1) return -1;
  const int H = m->c.hidden;
  free(m->h);
  m->h = (float*)malloc((size_t)len * H * sizeof(float));
  if (!m->h) return -2;
  m->start = start;
  m->len = len;
#pragma omp parallel for schedule(static)
  for (int t = 0; t < len; ++t)
    for (int i = 0; i < H; ++i)
      m->h[(size_t)t * H + i] = ref_bf16_to_float(ref_weight_bits(m->c.seed, TID_EMBED, (uint64_t)tokens[t] * H + i, 1.0f));
  return 0;
}

/* One block over the current chunk. q_only: compute q from the hidden state
 * but take K/V from the cache (first-token step over a complete cache). */
static int block(ref_model* m, int l, int q_only) {
  const int T = m->len, H = m->c.hidden, F = m->c.ffn, hd = m->c.head_dim;
  const int nq = m->c.n_heads, nkv = m->c.n_kv_heads;
  layer_w tmp = {0};
  layer_w* w = l < m->n_cached ? &m->cached[l] : &tmp;
  if (w == &tmp && gen_layer(m, l, &tmp)) return -2;
  float* xn = (float*)malloc((size_t)T * H * sizeof(float));
  float* q = (float*)malloc((size_t)T * m->qd * sizeof(float));
  float* kk = (float*)malloc((size_t)T * m->kvd * sizeof(float));
  float* vv = (float*)malloc((size_t)T * m->kvd * sizeof(float));
  float* at = (float*)malloc((size_t)T * m->qd * sizeof(float));
  float* o = (float*)malloc((size_t)T * (H > F ? H : F) * sizeof(float));
  float* g = (float*)malloc((size_t)T * F * sizeof(float));
  float* u = (float*)malloc((size_t)T * F * sizeof(float));
  rmsnorm_bf16(m->h, xn, T, H, m->c.rms_eps);
  matmul(xn, w->wq, q, T, m->qd, H);
  rope_rows(m, q, T, nq, m->start);
  for (size_t i = 0; i < (size_t)T * m->qd; ++i) q[i] = round_bf16(q[i]);
  if (!q_only) {
    matmul(xn, w->wk, kk, T, m->kvd, H);
    matmul(xn, w->wv, vv, T, m->kvd, H);
    rope_rows(m, kk, T, nkv, m->start);
    for (int t = 0; t < T; ++t)
      for (int hh = 0; hh < nkv; ++hh)
        for (int d = 0; d < hd; ++d) {
          kv_at(m, l, 0, hh, m->start + t)[d] = round_bf16(kk[((size_t)t * nkv + hh) * hd + d]);
          kv_at(m, l, 1, hh, m->start + t)[d] = round_bf16(vv[((size_t)t * nkv + hh) * hd + d]);
        }
  }
  attention(m, l, q, at, T, m->start);
  matmul(at, w->wo, o, T, H, m->qd);
  for (size_t i = 0; i < (size_t)T * H; ++i) m->h[i] += o[i];
  rmsnorm_bf16(m->h, xn, T, H, m->c.rms_eps);
  matmul(xn, w->wg, g, T, F, H);
  matmul(xn, w->wu, u, T, F, H);
  for (size_t i = 0; i < (size_t)T * F; ++i) {
    const float a = g[i];
    g[i] = round_bf16(a / (1.0f + expf(-a)) * u[i]);
  }
  matmul(g, w->wd, o, T, H, F);
  for (size_t i = 0; i < (size_t)T * H; ++i) m->h[i] += o[i];
  free(xn);
  free(q);
  free(kk);
  free(vv);
  free(at);
  free(o);
  free(g);
  free(u);
  if (w == &tmp) free_layer(&tmp);
  return 0;
}

int ref_run_layers(ref_model* m, int layer_begin, int layer_end) {
  if (!m->h) return -1;
  for (int l = layer_begin; l < layer_end; ++l) {
    const int st = block(m, l, 0);
    if (st) return st;
  }
  return 0;
}

int ref_final_logits(ref_model* m, int row, float* logits) {
  if (!m->h || row < 0 || row >= m->len) return -1;
  const int H = m->c.hidden;
  float* xn = (float*)malloc((size_t)H * sizeof(float));
  rmsnorm_bf16(m->h + (size_t)row * H, xn, 1, H, m->c.rms_eps);
#pragma omp parallel for schedule(static)
  for (int n = 0; n < m->c.vocab; ++n) {
    float acc = 0.f;
    for (int k = 0; k < H; ++k)
      acc += xn[k] * ref_bf16_to_float(ref_weight_bits(m->c.seed, TID_LMHEAD, (uint64_t)n * H + k, m->s_h));
    logits[n] = acc;
  }
  free(xn);
  return 0;
}

int ref_last_token_logits(ref_model* m, int32_t token, long long T, float* logits) {
  int st = ref_begin_chunk(m, &token, T - 1, 1);
  for (int l = 0; st == 0 && l < m->c.n_layers; ++l) st = block(m, l, 1);
  return st ? st : ref_final_logits(m, 0, logits);
}

int ref_load_chunk(ref_model* m, const uint16_t* tier, long long start, int len) {
  const int hd = m->c.head_dim, nkv = m->c.n_kv_heads;
  if (start < 0 || start + len > m->max_tokens) return -1;
  size_t i = 0;
  for (int l = 0; l < m->c.n_layers; ++l)
    for (int kv = 0; kv < 2; ++kv)
      for (int h = 0; h < nkv; ++h)
        for (int t = 0; t < len; ++t) {
          float* dst = kv_at(m, l, kv, h, start + t);
          for (int d = 0; d < hd; ++d) dst[d] = ref_bf16_to_float(tier[i++]);
        }
  return 0;
}
