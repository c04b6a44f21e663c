/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (see gpt_oracle.h for the contract and anchoring).
 *
 * fp32 storage, fp32 FMA dot products (8-lane partial sums), double for row statistics and
 * loss sums. OpenMP over rows/heads. Every routine is the textbook definition of the op; the
 * function comments cite the paper section / reference convention they follow.
 */
#include "gpt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_TENSORS_PER_LAYER 16

typedef float v8f __attribute__((vector_size(32), aligned(4), may_alias));

/* ------------------------------------------------------------------ counters / hashes */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

float orc_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate */
    u &= 0xffff0000u;
  } else {
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
  }
  memcpy(&x, &u, 4);
  return x;
}

float orc_init_value(uint64_t seed, int tensor_id, int64_t idx, float stddev) {
  uint64_t key = mix64(seed ^ ((uint64_t)(uint32_t)tensor_id << 48));
  int64_t s = 0;
  for (int i = 0; i < 4; ++i) s += (int64_t)(mix64(key + (uint64_t)idx * 4u + (uint64_t)i) >> 40);
  int32_t c = (int32_t)(s - ((int64_t)2 << 24));
  float scale = (float)((double)stddev * sqrt(3.0) / 16777216.0);
  return (float)c * scale;
}

int orc_dropout_keep(uint64_t seed, int step, int layer, int site, int64_t elem, float p) {
  /* one 64-bit hash per 4 consecutive elements; element e uses bits [16*(e%4), 16*(e%4)+16) */
  if (p <= 0.f) return 1;
  uint64_t key = mix64(seed ^ 0xD6E8FEB86659FD93ULL ^ ((uint64_t)(uint32_t)step << 40) ^
                       ((uint64_t)(uint32_t)(layer & 0xFFFF) << 16) ^ (uint64_t)(uint32_t)site);
  uint64_t h = mix64(key + ((uint64_t)elem >> 2));
  uint32_t r = (uint32_t)(h >> (16 * (elem & 3))) & 0xFFFFu;
  uint32_t thr = (uint32_t)((double)p * 65536.0);
  return r >= thr;
}

void orc_gen_tokens(uint64_t seed, int64_t n, int vocab, int32_t* out) {
  /* std::mt19937_64 restated (Matsumoto & Nishimura 2004 parameters). */
  uint64_t mt[312];
  int mti;
  mt[0] = seed;
  for (mti = 1; mti < 312; ++mti)
    mt[mti] = 6364136223846793005ULL * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  mti = 312;
  for (int64_t i = 0; i < n; ++i) {
    if (mti >= 312) {
      for (int k = 0; k < 312; ++k) {
        uint64_t x = (mt[k] & 0xFFFFFFFF80000000ULL) | (mt[(k + 1) % 312] & 0x7FFFFFFFULL);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        mt[k] = mt[(k + 156) % 312] ^ xa;
      }
      mti = 0;
    }
    uint64_t y = mt[mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    out[i] = (int32_t)(y % (uint64_t)vocab);
  }
}

/* ------------------------------------------------------------------ parameter layout */
int orc_num_tensors(const orc_model* m) { return 2 + ORC_TENSORS_PER_LAYER * m->num_layers + 2; }

int orc_tensor_info(const orc_model* m, int id, int64_t* offset, int64_t* rows, int64_t* cols) {
  const int64_t d = m->hidden_size, V = m->vocab_size, s = m->seq_length;
  int64_t off = 0;
  for (int t = 0; t <= id; ++t) {
    int64_t r = 0, c = 1;
    if (t == 0) { r = V; c = d; }
    else if (t == 1) { r = s; c = d; }
    else if (t >= 2 + ORC_TENSORS_PER_LAYER * m->num_layers) { r = d; c = 1; }
    else {
      switch ((t - 2) % ORC_TENSORS_PER_LAYER) {
        case 0: case 1: case 5: case 6: case 7: case 11: r = d; break;
        case 2: r = 3 * d; c = d; break;
        case 3: r = 3 * d; break;
        case 4: r = d; c = d; break;
        case 8: r = 4 * d; c = d; break;
        case 9: r = 4 * d; break;
        case 10: r = d; c = 4 * d; break;
        default: r = 0; c = 0; break;
      }
    }
    if (t == id) {
      if (offset) *offset = off;
      if (rows) *rows = r;
      if (cols) *cols = c;
      return 0;
    }
    off += r * c;
  }
  return -1;
}

int64_t orc_param_numel(const orc_model* m) {
  int64_t off, r, c;
  int last = orc_num_tensors(m) - 1;
  orc_tensor_info(m, last, &off, &r, &c);
  return off + r * c;
}

/* Init std per tensor: 0.02 for embeddings/QKV/fc1, 0.02/sqrt(2L) for the output
 * projections feeding the residual (Megatron scaled init); LN gamma = 1, others 0. */
float orc_init_std(const orc_model* m, int id) {
  if (id == 0 || id == 1) return 0.02f;
  if (id >= 2 + ORC_TENSORS_PER_LAYER * m->num_layers) return 0.f;
  switch ((id - 2) % ORC_TENSORS_PER_LAYER) {
    case 2: case 8: return 0.02f;
    case 4: case 10: return (float)(0.02 / sqrt(2.0 * m->num_layers));
    default: return 0.f;
  }
}

float orc_init_const(const orc_model* m, int id) {
  if (id >= 2 + ORC_TENSORS_PER_LAYER * m->num_layers) return (id - 2 - ORC_TENSORS_PER_LAYER * m->num_layers) == 0 ? 1.f : 0.f;
  if (id < 2) return 0.f;
  int j = (id - 2) % ORC_TENSORS_PER_LAYER;
  return (j == 0 || j == 6) ? 1.f : 0.f;
}

void orc_init_params(const orc_model* m, uint64_t seed, float* params) {
  int nt = orc_num_tensors(m);
  for (int id = 0; id < nt; ++id) {
    int64_t off, r, c;
    orc_tensor_info(m, id, &off, &r, &c);
    float sd = orc_init_std(m, id), cv = orc_init_const(m, id);
    int64_t n = r * c;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) params[off + i] = sd > 0.f ? orc_init_value(seed, id, i, sd) : cv;
  }
}

/* ------------------------------------------------------------------ dense algebra */
static inline float dot8(const float* a, const float* b, int64_t K) {
  v8f acc = {0, 0, 0, 0, 0, 0, 0, 0};
  int64_t k = 0;
  for (; k + 8 <= K; k += 8) acc += *(const v8f*)(a + k) * *(const v8f*)(b + k);
  float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  for (; k < K; ++k) s += a[k] * b[k];
  return s;
}

/* C[M,N] (+)= A[M,K] . B[N,K]^T, row-major with leading dims. 4x4 register blocks of 8-lane
 * partial sums; OpenMP over 64x64 output blocks. */
static void gemm_nt(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                    int64_t ldb, float* C, int64_t ldc, int accumulate) {
  const int64_t BI = 64, BJ = 64;
  int64_t nbi = (M + BI - 1) / BI, nbj = (N + BJ - 1) / BJ;
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int64_t bi = 0; bi < nbi; ++bi) {
    for (int64_t bj = 0; bj < nbj; ++bj) {
      int64_t i0 = bi * BI, i1 = i0 + BI < M ? i0 + BI : M;
      int64_t j0 = bj * BJ, j1 = j0 + BJ < N ? j0 + BJ : N;
      int64_t i = i0;
      for (; i + 4 <= i1; i += 4) {
        int64_t j = j0;
        for (; j + 4 <= j1; j += 4) {
          v8f acc[4][4];
          for (int x = 0; x < 4; ++x)
            for (int y = 0; y < 4; ++y) acc[x][y] = (v8f){0, 0, 0, 0, 0, 0, 0, 0};
          int64_t k = 0;
          for (; k + 8 <= K; k += 8) {
            v8f a0 = *(const v8f*)(A + (i + 0) * lda + k), a1 = *(const v8f*)(A + (i + 1) * lda + k);
            v8f a2 = *(const v8f*)(A + (i + 2) * lda + k), a3 = *(const v8f*)(A + (i + 3) * lda + k);
            for (int y = 0; y < 4; ++y) {
              v8f b = *(const v8f*)(B + (j + y) * ldb + k);
              acc[0][y] += a0 * b;
              acc[1][y] += a1 * b;
              acc[2][y] += a2 * b;
              acc[3][y] += a3 * b;
            }
          }
          for (int x = 0; x < 4; ++x)
            for (int y = 0; y < 4; ++y) {
              v8f v = acc[x][y];
              float s = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
              for (int64_t kk = k; kk < K; ++kk) s += A[(i + x) * lda + kk] * B[(j + y) * ldb + kk];
              float* c = C + (i + x) * ldc + j + y;
              *c = accumulate ? *c + s : s;
            }
        }
        for (; j < j1; ++j)
          for (int x = 0; x < 4; ++x) {
            float s = dot8(A + (i + x) * lda, B + j * ldb, K);
            float* c = C + (i + x) * ldc + j;
            *c = accumulate ? *c + s : s;
          }
      }
      for (; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) {
          float s = dot8(A + i * lda, B + j * ldb, K);
          float* c = C + i * ldc + j;
          *c = accumulate ? *c + s : s;
        }
    }
  }
}

static float* transpose(const float* X, int64_t R, int64_t Cc) {
  float* T = (float*)malloc(sizeof(float) * R * Cc);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < Cc; ++c)
    for (int64_t r = 0; r < R; ++r) T[c * R + r] = X[r * Cc + c];
  return T;
}

/* Linear forward (Megatron ColumnParallel/RowParallel semantics):
 * Y[T,N] = X[T,K] W[N,K]^T + b. */
static void linear_fwd(int64_t T, int64_t N, int64_t K, const float* X, const float* W,
                       const float* b, float* Y) {
  gemm_nt(T, N, K, X, K, W, K, Y, N, 0);
  if (b) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t)
      for (int64_t n = 0; n < N; ++n) Y[t * N + n] += b[n];
  }
}

/* dX[T,K] = dY W ; dW[N,K] += dY^T X ; db[N] += colsum(dY). */
static void linear_bwd(int64_t T, int64_t N, int64_t K, const float* X, const float* W,
                       const float* dY, float* dX, float* dW, float* db) {
  if (dX) {
    float* Wt = transpose(W, N, K);
    gemm_nt(T, K, N, dY, N, Wt, N, dX, K, 0);
    free(Wt);
  }
  float* dYt = transpose(dY, T, N);
  float* Xt = transpose(X, T, K);
  gemm_nt(N, K, T, dYt, T, Xt, T, dW, K, 1);
  if (db) {
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
      double s = 0;
      for (int64_t t = 0; t < T; ++t) s += dYt[n * T + t];
      db[n] += (float)s;
    }
  }
  free(dYt);
  free(Xt);
}

/* LayerNorm eps 1e-5 (Megatron default). */
#define LN_EPS 1e-5f
static void ln_fwd(int64_t T, int64_t d, const float* x, const float* g, const float* b, float* y,
                   float* mean, float* rstd) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const float* xr = x + t * d;
    double s = 0, ss = 0;
    for (int64_t i = 0; i < d; ++i) s += xr[i];
    double mu = s / d;
    for (int64_t i = 0; i < d; ++i) ss += (xr[i] - mu) * (xr[i] - mu);
    float rs = (float)(1.0 / sqrt(ss / d + LN_EPS));
    mean[t] = (float)mu;
    rstd[t] = rs;
    for (int64_t i = 0; i < d; ++i) y[t * d + i] = ((xr[i] - (float)mu) * rs) * g[i] + b[i];
  }
}

static void ln_bwd(int64_t T, int64_t d, const float* x, const float* g, const float* mean,
                   const float* rstd, const float* dy, float* dx_accum, float* dg, float* db) {
  double* dgs = (double*)calloc((size_t)d, sizeof(double));
  double* dbs = (double*)calloc((size_t)d, sizeof(double));
#pragma omp parallel
  {
    double* dgl = (double*)calloc((size_t)d, sizeof(double));
    double* dbl = (double*)calloc((size_t)d, sizeof(double));
#pragma omp for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      const float *xr = x + t * d, *dyr = dy + t * d;
      float mu = mean[t], rs = rstd[t];
      double s1 = 0, s2 = 0;
      for (int64_t i = 0; i < d; ++i) {
        float xh = (xr[i] - mu) * rs;
        float gy = dyr[i] * g[i];
        s1 += gy;
        s2 += gy * xh;
        dgl[i] += dyr[i] * xh;
        dbl[i] += dyr[i];
      }
      float m1 = (float)(s1 / d), m2 = (float)(s2 / d);
      for (int64_t i = 0; i < d; ++i) {
        float xh = (xr[i] - mu) * rs;
        dx_accum[t * d + i] += rs * (dyr[i] * g[i] - m1 - xh * m2);
      }
    }
#pragma omp critical
    for (int64_t i = 0; i < d; ++i) {
      dgs[i] += dgl[i];
      dbs[i] += dbl[i];
    }
    free(dgl);
    free(dbl);
  }
  for (int64_t i = 0; i < d; ++i) {
    dg[i] += (float)dgs[i];
    db[i] += (float)dbs[i];
  }
  free(dgs);
  free(dbs);
}

static inline float gelu_t(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
static inline float gelu_t_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float t = tanhf(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

static void round_bf16(float* x, int64_t n, int on) {
  if (!on) return;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) x[i] = orc_bf16(x[i]);
}

/* Causal multi-head attention forward on qkv[T, 3d] laid out (q heads | k heads | v heads),
 * each head hd contiguous (TP splits whole heads). Stores probabilities P for
 * the backward pass. */
static void attn_fwd(int nseq, int s, int heads, int hd, const float* qkv, float* o, float* P) {
  const int64_t d = (int64_t)heads * hd, ld = 3 * d;
  const float scale = 1.f / sqrtf((float)hd);
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < nseq; ++b)
    for (int h = 0; h < heads; ++h) {
      float* Pbh = P + ((int64_t)b * heads + h) * s * s;
      for (int i = 0; i < s; ++i) {
        const float* q = qkv + ((int64_t)b * s + i) * ld + (int64_t)h * hd;
        float* pr = Pbh + (int64_t)i * s;
        float mx = -INFINITY;
        for (int j = 0; j <= i; ++j) {
          const float* k = qkv + ((int64_t)b * s + j) * ld + d + (int64_t)h * hd;
          pr[j] = dot8(q, k, hd) * scale;
          if (pr[j] > mx) mx = pr[j];
        }
        double sum = 0;
        for (int j = 0; j <= i; ++j) {
          pr[j] = expf(pr[j] - mx);
          sum += pr[j];
        }
        float inv = (float)(1.0 / sum);
        for (int j = 0; j <= i; ++j) pr[j] *= inv;
        for (int j = i + 1; j < s; ++j) pr[j] = 0.f;
        float* orow = o + ((int64_t)b * s + i) * d + (int64_t)h * hd;
        for (int c = 0; c < hd; ++c) orow[c] = 0.f;
        for (int j = 0; j <= i; ++j) {
          const float* v = qkv + ((int64_t)b * s + j) * ld + 2 * d + (int64_t)h * hd;
          float pj = pr[j];
          for (int c = 0; c < hd; ++c) orow[c] += pj * v[c];
        }
      }
    }
}

static void attn_bwd(int nseq, int s, int heads, int hd, const float* qkv, const float* o,
                     const float* P, const float* dO, float* dqkv) {
  const int64_t d = (int64_t)heads * hd, ld = 3 * d;
  const float scale = 1.f / sqrtf((float)hd);
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
  for (int b = 0; b < nseq; ++b)
    for (int h = 0; h < heads; ++h) {
      const float* Pbh = P + ((int64_t)b * heads + h) * s * s;
      float* dS = (float*)malloc(sizeof(float) * s);
      for (int i = 0; i < s; ++i) {
        const float* dorow = dO + ((int64_t)b * s + i) * d + (int64_t)h * hd;
        const float* orow = o + ((int64_t)b * s + i) * d + (int64_t)h * hd;
        float Di = dot8(dorow, orow, hd);
        const float* pr = Pbh + (int64_t)i * s;
        for (int j = 0; j <= i; ++j) {
          const float* v = qkv + ((int64_t)b * s + j) * ld + 2 * d + (int64_t)h * hd;
          float dp = dot8(dorow, v, hd);
          dS[j] = pr[j] * (dp - Di);
        }
        float* dq = dqkv + ((int64_t)b * s + i) * ld + (int64_t)h * hd;
        const float* q = qkv + ((int64_t)b * s + i) * ld + (int64_t)h * hd;
        for (int j = 0; j <= i; ++j) {
          const float* k = qkv + ((int64_t)b * s + j) * ld + d + (int64_t)h * hd;
          float* dk = dqkv + ((int64_t)b * s + j) * ld + d + (int64_t)h * hd;
          float* dv = dqkv + ((int64_t)b * s + j) * ld + 2 * d + (int64_t)h * hd;
          float ds = dS[j] * scale, pj = pr[j];
          for (int c = 0; c < hd; ++c) {
            dq[c] += ds * k[c];
            dk[c] += ds * q[c];
            dv[c] += pj * dorow[c];
          }
        }
      }
      free(dS);
    }
}

/* ------------------------------------------------------------------ model */
typedef struct {
  const orc_model* m;
  const orc_opts* o;
  const float* p; /* parameters (possibly bf16-rounded copy) */
  int64_t T;
  int nseq;
  int64_t sample0;
  int step;
  /* per-layer saved activations */
  float **h_in, **a, **mu1, **rs1, **qkv, **att, **P, **h_mid, **m2, **mu2, **rs2, **u, **g;
  float *h_out, *hf, *muf, *rsf, *logits;
} fwd_state;

static const float* T_(const fwd_state* st, int id) {
  int64_t off;
  orc_tensor_info(st->m, id, &off, NULL, NULL);
  return st->p + off;
}

static void dropout_apply(const fwd_state* st, int layer, int site, float* x, int64_t d) {
  float p = st->o->dropout;
  if (p <= 0.f) return;
  float sc = (float)(1.0 / (1.0 - (double)p));
  int64_t base = st->sample0 * (int64_t)st->m->seq_length * d;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < st->T * d; ++i)
    x[i] = orc_dropout_keep(st->o->seed, st->step, layer, site, base + i, p) ? x[i] * sc : 0.f;
}

static void forward(fwd_state* st, const int32_t* tokens) {
  const orc_model* m = st->m;
  const int L = m->num_layers, s = m->seq_length, heads = m->num_heads;
  const int64_t d = m->hidden_size, V = m->vocab_size, T = st->T;
  const int hd = (int)(d / heads);
  const int em = st->o->bf16_emulate;
  float* h = (float*)malloc(sizeof(float) * T * d);
  const float *wte = T_(st, 0), *wpe = T_(st, 1);
  for (int b = 0; b < st->nseq; ++b)
    for (int i = 0; i < s; ++i) {
      int tok = tokens[(int64_t)b * (s + 1) + i];
      for (int64_t c = 0; c < d; ++c) h[((int64_t)b * s + i) * d + c] = wte[tok * d + c] + wpe[i * d + c];
    }
  dropout_apply(st, 0xFFFF, 2, h, d);
  round_bf16(h, T * d, em);
  for (int l = 0; l < L; ++l) {
    const int base = 2 + ORC_TENSORS_PER_LAYER * l;
    st->h_in[l] = h;
    st->a[l] = (float*)malloc(sizeof(float) * T * d);
    st->mu1[l] = (float*)malloc(sizeof(float) * T);
    st->rs1[l] = (float*)malloc(sizeof(float) * T);
    ln_fwd(T, d, h, T_(st, base + 0), T_(st, base + 1), st->a[l], st->mu1[l], st->rs1[l]);
    round_bf16(st->a[l], T * d, em);
    st->qkv[l] = (float*)malloc(sizeof(float) * T * 3 * d);
    linear_fwd(T, 3 * d, d, st->a[l], T_(st, base + 2), T_(st, base + 3), st->qkv[l]);
    round_bf16(st->qkv[l], T * 3 * d, em);
    st->att[l] = (float*)malloc(sizeof(float) * T * d);
    st->P[l] = (float*)malloc(sizeof(float) * (int64_t)st->nseq * heads * s * s);
    attn_fwd(st->nseq, s, heads, hd, st->qkv[l], st->att[l], st->P[l]);
    round_bf16(st->att[l], T * d, em);
    float* y = (float*)malloc(sizeof(float) * T * d);
    linear_fwd(T, d, d, st->att[l], T_(st, base + 4), NULL, y);
    round_bf16(y, T * d, em);
    const float* bo = T_(st, base + 5);
    for (int64_t t = 0; t < T; ++t)
      for (int64_t c = 0; c < d; ++c) y[t * d + c] += bo[c];
    dropout_apply(st, l, 0, y, d);
    float* hm = (float*)malloc(sizeof(float) * T * d);
    for (int64_t i = 0; i < T * d; ++i) hm[i] = h[i] + y[i];
    round_bf16(hm, T * d, em);
    st->h_mid[l] = hm;
    st->m2[l] = (float*)malloc(sizeof(float) * T * d);
    st->mu2[l] = (float*)malloc(sizeof(float) * T);
    st->rs2[l] = (float*)malloc(sizeof(float) * T);
    ln_fwd(T, d, hm, T_(st, base + 6), T_(st, base + 7), st->m2[l], st->mu2[l], st->rs2[l]);
    round_bf16(st->m2[l], T * d, em);
    st->u[l] = (float*)malloc(sizeof(float) * T * 4 * d);
    linear_fwd(T, 4 * d, d, st->m2[l], T_(st, base + 8), T_(st, base + 9), st->u[l]);
    round_bf16(st->u[l], T * 4 * d, em);
    st->g[l] = (float*)malloc(sizeof(float) * T * 4 * d);
    for (int64_t i = 0; i < T * 4 * d; ++i) st->g[l][i] = gelu_t(st->u[l][i]);
    round_bf16(st->g[l], T * 4 * d, em);
    linear_fwd(T, d, 4 * d, st->g[l], T_(st, base + 10), NULL, y);
    round_bf16(y, T * d, em);
    const float* b2 = T_(st, base + 11);
    for (int64_t t = 0; t < T; ++t)
      for (int64_t c = 0; c < d; ++c) y[t * d + c] += b2[c];
    dropout_apply(st, l, 1, y, d);
    float* hn = (float*)malloc(sizeof(float) * T * d);
    for (int64_t i = 0; i < T * d; ++i) hn[i] = hm[i] + y[i];
    round_bf16(hn, T * d, em);
    free(y);
    h = hn;
  }
  st->h_out = h;
  const int fid = 2 + ORC_TENSORS_PER_LAYER * L;
  st->hf = (float*)malloc(sizeof(float) * T * d);
  st->muf = (float*)malloc(sizeof(float) * T);
  st->rsf = (float*)malloc(sizeof(float) * T);
  ln_fwd(T, d, h, T_(st, fid), T_(st, fid + 1), st->hf, st->muf, st->rsf);
  round_bf16(st->hf, T * d, em);
  st->logits = (float*)malloc(sizeof(float) * T * V);
  gemm_nt(T, V, d, st->hf, d, wte, d, st->logits, V, 0);
  round_bf16(st->logits, T * V, em);
}

/* Softmax cross-entropy per token; writes dlogits = scale*(softmax - onehot) in place when
 * dscale != 0. Returns sum CE. */
static double cross_entropy(int64_t T, int64_t V, float* logits, const int32_t* tokens, int nseq,
                            int s, double dscale, float* tok_loss) {
  double total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    int b = (int)(t / s), i = (int)(t % s);
    int label = tokens[(int64_t)b * (s + 1) + i + 1];
    float* row = logits + t * V;
    float mx = -INFINITY;
    for (int64_t v = 0; v < V; ++v) mx = row[v] > mx ? row[v] : mx;
    double se = 0;
    for (int64_t v = 0; v < V; ++v) se += exp((double)row[v] - mx);
    double lse = mx + log(se);
    double li = lse - row[label];
    total += li;
    if (tok_loss) tok_loss[t] = (float)li;
    if (dscale != 0) {
      for (int64_t v = 0; v < V; ++v) row[v] = (float)(dscale * exp((double)row[v] - lse));
      row[label] -= (float)dscale;
    }
  }
  (void)nseq;
  return total;
}

static void free_state(fwd_state* st) {
  const int L = st->m->num_layers;
  free(st->h_in[0]);
  for (int l = 0; l < L; ++l) {
    free(st->a[l]); free(st->mu1[l]); free(st->rs1[l]); free(st->qkv[l]); free(st->att[l]);
    free(st->P[l]); free(st->h_mid[l]); free(st->m2[l]); free(st->mu2[l]); free(st->rs2[l]);
    free(st->u[l]); free(st->g[l]);
    if (l + 1 < L) free(st->h_in[l + 1]);
  }
  free(st->h_out);
  free(st->hf); free(st->muf); free(st->rsf); free(st->logits);
  free(st->h_in); free(st->a); free(st->mu1); free(st->rs1); free(st->qkv); free(st->att);
  free(st->P); free(st->h_mid); free(st->m2); free(st->mu2); free(st->rs2); free(st->u); free(st->g);
}

static float* params_view(const orc_model* m, const orc_opts* o, const float* params) {
  if (!o->bf16_emulate) return NULL;
  int64_t n = orc_param_numel(m);
  float* c = (float*)malloc(sizeof(float) * n);
  for (int64_t i = 0; i < n; ++i) c[i] = orc_bf16(params[i]);
  return c;
}

static void init_state(fwd_state* st, const orc_model* m, const orc_opts* o, const float* p,
                       int nseq, int64_t sample0, int step) {
  memset(st, 0, sizeof(*st));
  st->m = m; st->o = o; st->p = p;
  st->nseq = nseq; st->T = (int64_t)nseq * m->seq_length; st->sample0 = sample0; st->step = step;
  size_t L = (size_t)m->num_layers;
  float*** arrs[] = {&st->h_in, &st->a, &st->mu1, &st->rs1, &st->qkv, &st->att, &st->P,
                     &st->h_mid, &st->m2, &st->mu2, &st->rs2, &st->u, &st->g};
  for (size_t i = 0; i < sizeof(arrs) / sizeof(arrs[0]); ++i) *arrs[i] = (float**)calloc(L, sizeof(float*));
}

double orc_forward(const orc_model* m, const orc_opts* o, const float* params,
                   const int32_t* tokens, int nseq, int64_t sample0, int step, float* tok_loss) {
  float* pv = params_view(m, o, params);
  fwd_state st;
  init_state(&st, m, o, pv ? pv : params, nseq, sample0, step);
  forward(&st, tokens);
  double loss = cross_entropy(st.T, m->vocab_size, st.logits, tokens, nseq, m->seq_length, 0, tok_loss);
  free_state(&st);
  free(pv);
  return loss;
}

double orc_fwd_bwd(const orc_model* m, const orc_opts* o, const float* params,
                   const int32_t* tokens, int nseq, int64_t sample0, int step, double loss_scale,
                   float* grads, float* act_out) {
  float* pv = params_view(m, o, params);
  fwd_state st;
  init_state(&st, m, o, pv ? pv : params, nseq, sample0, step);
  forward(&st, tokens);
  const int L = m->num_layers, s = m->seq_length, heads = m->num_heads;
  const int64_t d = m->hidden_size, V = m->vocab_size, T = st.T;
  const int hd = (int)(d / heads);
  if (act_out) memcpy(act_out, st.hf, sizeof(float) * T * d);
  double loss = cross_entropy(T, V, st.logits, tokens, nseq, s, loss_scale, NULL);
  float* G = grads;
#define GR(id) (G + ({ int64_t _o; orc_tensor_info(m, (id), &_o, NULL, NULL); _o; }))
  /* LM head (tied): dhf = dlogits . wte ; dwte += dlogits^T . hf */
  float* dhf = (float*)malloc(sizeof(float) * T * d);
  linear_bwd(T, V, d, st.hf, T_(&st, 0), st.logits, dhf, GR(0), NULL);
  const int fid = 2 + ORC_TENSORS_PER_LAYER * L;
  float* dh = (float*)calloc((size_t)(T * d), sizeof(float));
  ln_bwd(T, d, st.h_out, T_(&st, fid), st.muf, st.rsf, dhf, dh, GR(fid), GR(fid + 1));
  free(dhf);
  float* dy = (float*)malloc(sizeof(float) * T * d);
  float* tmp = (float*)malloc(sizeof(float) * T * 4 * d);
  for (int l = L - 1; l >= 0; --l) {
    const int base = 2 + ORC_TENSORS_PER_LAYER * l;
    /* MLP branch: dy = dropout'(dh) */
    memcpy(dy, dh, sizeof(float) * T * d);
    dropout_apply(&st, l, 1, dy, d);
    float* dg = tmp;
    linear_bwd(T, d, 4 * d, st.g[l], T_(&st, base + 10), dy, dg, GR(base + 10), GR(base + 11));
    for (int64_t i = 0; i < T * 4 * d; ++i) dg[i] *= gelu_t_grad(st.u[l][i]);
    float* dm = (float*)malloc(sizeof(float) * T * d);
    linear_bwd(T, 4 * d, d, st.m2[l], T_(&st, base + 8), dg, dm, GR(base + 8), GR(base + 9));
    ln_bwd(T, d, st.h_mid[l], T_(&st, base + 6), st.mu2[l], st.rs2[l], dm, dh, GR(base + 6), GR(base + 7));
    /* attention branch */
    memcpy(dy, dh, sizeof(float) * T * d);
    dropout_apply(&st, l, 0, dy, d);
    float* datt = dm;
    linear_bwd(T, d, d, st.att[l], T_(&st, base + 4), dy, datt, GR(base + 4), GR(base + 5));
    float* dqkv = (float*)calloc((size_t)(T * 3 * d), sizeof(float));
    attn_bwd(st.nseq, s, heads, hd, st.qkv[l], st.att[l], st.P[l], datt, dqkv);
    float* da = datt;
    linear_bwd(T, 3 * d, d, st.a[l], T_(&st, base + 2), dqkv, da, GR(base + 2), GR(base + 3));
    ln_bwd(T, d, st.h_in[l], T_(&st, base + 0), st.mu1[l], st.rs1[l], da, dh, GR(base + 0), GR(base + 1));
    free(dqkv);
    free(dm);
  }
  /* embeddings */
  memcpy(dy, dh, sizeof(float) * T * d);
  dropout_apply(&st, 0xFFFF, 2, dy, d);
  float *dwte = GR(0), *dwpe = GR(1);
  for (int b = 0; b < nseq; ++b)
    for (int i = 0; i < s; ++i) {
      int tok = tokens[(int64_t)b * (s + 1) + i];
      const float* r = dy + ((int64_t)b * s + i) * d;
      for (int64_t c = 0; c < d; ++c) {
        dwte[tok * d + c] += r[c];
        dwpe[i * d + c] += r[c];
      }
    }
#undef GR
  free(dy);
  free(tmp);
  free(dh);
  free_state(&st);
  free(pv);
  return loss;
}

void orc_adam(int64_t n, float* p, const float* g, float* mom, float* var, int step,
              const orc_opts* o) {
  const double bc1 = 1.0 - pow((double)o->beta1, step), bc2 = 1.0 - pow((double)o->beta2, step);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float gi = g[i];
    mom[i] = o->beta1 * mom[i] + (1.f - o->beta1) * gi;
    var[i] = o->beta2 * var[i] + (1.f - o->beta2) * gi * gi;
    float mh = (float)(mom[i] / bc1), vh = (float)(var[i] / bc2);
    p[i] -= o->lr * (mh / (sqrtf(vh) + o->eps) + o->weight_decay * p[i]);
  }
}

/* Bounded CPU-baseline sample: one decoder layer fwd+bwd on nseq sequences. */
double orc_time_layer(const orc_model* m0, int nseq, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  orc_model m = *m0;
  m.num_layers = 1;
  orc_opts o;
  memset(&o, 0, sizeof(o));
  const int64_t d = m.hidden_size, T = (int64_t)nseq * m.seq_length;
  const int heads = m.num_heads, s = m.seq_length, hd = (int)(d / heads);
  int64_t np = orc_param_numel(&m);
  float* params = (float*)malloc(sizeof(float) * np);
  float* grads = (float*)calloc((size_t)np, sizeof(float));
  orc_init_params(&m, 1, params);
  fwd_state st;
  init_state(&st, &m, &o, params, nseq, 0, 1);
  float* x = (float*)malloc(sizeof(float) * T * d);
  for (int64_t i = 0; i < T * d; ++i) x[i] = orc_init_value(7, 99, i, 1.0f);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  /* forward of one layer (same code path as forward(), inlined for a single layer) */
  const int base = 2;
  float* a = (float*)malloc(sizeof(float) * T * d);
  float *mu1 = (float*)malloc(sizeof(float) * T), *rs1 = (float*)malloc(sizeof(float) * T);
  ln_fwd(T, d, x, T_(&st, base), T_(&st, base + 1), a, mu1, rs1);
  float* qkv = (float*)malloc(sizeof(float) * T * 3 * d);
  linear_fwd(T, 3 * d, d, a, T_(&st, base + 2), T_(&st, base + 3), qkv);
  float* att = (float*)malloc(sizeof(float) * T * d);
  float* P = (float*)malloc(sizeof(float) * (int64_t)nseq * heads * s * s);
  attn_fwd(nseq, s, heads, hd, qkv, att, P);
  float* y = (float*)malloc(sizeof(float) * T * d);
  linear_fwd(T, d, d, att, T_(&st, base + 4), T_(&st, base + 5), y);
  float* hm = (float*)malloc(sizeof(float) * T * d);
  for (int64_t i = 0; i < T * d; ++i) hm[i] = x[i] + y[i];
  float* m2 = (float*)malloc(sizeof(float) * T * d);
  float *mu2 = (float*)malloc(sizeof(float) * T), *rs2 = (float*)malloc(sizeof(float) * T);
  ln_fwd(T, d, hm, T_(&st, base + 6), T_(&st, base + 7), m2, mu2, rs2);
  float* u = (float*)malloc(sizeof(float) * T * 4 * d);
  linear_fwd(T, 4 * d, d, m2, T_(&st, base + 8), T_(&st, base + 9), u);
  float* g = (float*)malloc(sizeof(float) * T * 4 * d);
  for (int64_t i = 0; i < T * 4 * d; ++i) g[i] = gelu_t(u[i]);
  linear_fwd(T, d, 4 * d, g, T_(&st, base + 10), T_(&st, base + 11), y);
  /* backward with dy = 1e-3 */
  float* dh = (float*)malloc(sizeof(float) * T * d);
  for (int64_t i = 0; i < T * d; ++i) dh[i] = 1e-3f;
  float* dg = (float*)malloc(sizeof(float) * T * 4 * d);
  int64_t off[16];
  for (int j = 0; j < 12; ++j) orc_tensor_info(&m, base + j, &off[j], NULL, NULL);
  linear_bwd(T, d, 4 * d, g, T_(&st, base + 10), dh, dg, grads + off[10], grads + off[11]);
  for (int64_t i = 0; i < T * 4 * d; ++i) dg[i] *= gelu_t_grad(u[i]);
  float* dm = (float*)malloc(sizeof(float) * T * d);
  linear_bwd(T, 4 * d, d, m2, T_(&st, base + 8), dg, dm, grads + off[8], grads + off[9]);
  ln_bwd(T, d, hm, T_(&st, base + 6), mu2, rs2, dm, dh, grads + off[6], grads + off[7]);
  linear_bwd(T, d, d, att, T_(&st, base + 4), dh, dm, grads + off[4], grads + off[5]);
  float* dqkv = (float*)calloc((size_t)(T * 3 * d), sizeof(float));
  attn_bwd(nseq, s, heads, hd, qkv, att, P, dm, dqkv);
  linear_bwd(T, 3 * d, d, a, T_(&st, base + 2), dqkv, dm, grads + off[2], grads + off[3]);
  ln_bwd(T, d, x, T_(&st, base), mu1, rs1, dm, dh, grads + off[0], grads + off[1]);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(a); free(mu1); free(rs1); free(qkv); free(att); free(P); free(y); free(hm); free(m2);
  free(mu2); free(rs2); free(u); free(g); free(dh); free(dg); free(dm); free(dqkv); free(x);
  free(params); free(grads);
  free(st.h_in); free(st.a); free(st.mu1); free(st.rs1); free(st.qkv); free(st.att); free(st.P);
  free(st.h_mid); free(st.m2); free(st.mu2); free(st.rs2); free(st.u); free(st.g);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
