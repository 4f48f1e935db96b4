/*
 * mst_oracle.c — CPU restatement of the reference's mini-sequence path.
 * TEST INFRASTRUCTURE ONLY (see mst_oracle.h for the contract and the
 * file:line map into /root/reference).
 */
#include "mst_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_SHAPE 1
#define ORC_ERR_CONFIG 4
#define ORC_ERR_DATA 5

static int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }

/* ================================================================ rng
 * rng.hpp:8-72: splitmix64 seeding, FNV-1a name hashing, xoshiro256++,
 * 53-bit uniform, modulo uniform_below, Box-Muller without caching. */
uint64_t orc_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t orc_fnv1a64(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ull;
  }
  return h;
}

void orc_rng_init(orc_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  r->root_seed = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = orc_splitmix64(&sm);
}

void orc_rng_fork(const orc_rng* r, const char* name, orc_rng* out) { orc_rng_init(out, r->root_seed ^ orc_fnv1a64(name)); }

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

uint64_t orc_rng_next_u64(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}

double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

uint64_t orc_rng_uniform_below(orc_rng* r, uint64_t n) { return orc_rng_next_u64(r) % n; }

double orc_rng_gaussian(orc_rng* r) {
  double u1 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586477 * u2);
}

float orc_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return x; /* inf / nan */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

void orc_fill_gaussian_bf16(orc_rng* r, float* out, int64_t n, double std) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_round_bf16((float)(std * orc_rng_gaussian(r)));
}

void orc_fill_labels(orc_rng* r, int32_t* out, int64_t n, int64_t vocab, double p_ignore) {
  for (int64_t i = 0; i < n; ++i) {
    const double u = orc_rng_uniform(r);
    const int32_t lab = (int32_t)orc_rng_uniform_below(r, (uint64_t)vocab);
    out[i] = u < p_ignore ? -100 : lab;
  }
}

/* ================================================================ counters
 * memtrack.hpp:19-35 conventions: matmul 2NKP flops, NK+KP+NP hbm,
 * "weights." operands add to weight reads; silu fwd 4 flops/elem hbm 2e;
 * silu bwd 4/3e; elementwise 1/3e; CE fwd 5 per logit, e + 2 rows;
 * CE bwd 5 per logit, 2e + 2 rows; copies 0 flops, 2e. */
static orc_counters g_ctr;
void orc_counters_reset(void) { memset(&g_ctr, 0, sizeof(g_ctr)); }
void orc_counters_get(orc_counters* out) { *out = g_ctr; }
static void count_matmul(int64_t n, int64_t k, int64_t p, uint64_t weight_elems) {
  const uint64_t f = 2ull * (uint64_t)n * (uint64_t)k * (uint64_t)p;
  g_ctr.flops += f;
  g_ctr.matmul_flops += f;
  g_ctr.hbm_elements += (uint64_t)(n * k + k * p + n * p);
  g_ctr.weight_read_elements += weight_elems;
}
static void count_op(uint64_t flops, uint64_t hbm) {
  g_ctr.flops += flops;
  g_ctr.hbm_elements += hbm;
}

/* ================================================================ memory
 * Live/peak bytes per label class, replayed like MemReport::replay_peak
 * (memtrack.hpp:97-110).  f64 tensors (8 bytes per element). */
static uint64_t g_live[ORC_MEM_NCLASS], g_peak_cls[ORC_MEM_NCLASS], g_live_total, g_peak_total;
void orc_mem_reset(void) {
  memset(g_live, 0, sizeof(g_live));
  memset(g_peak_cls, 0, sizeof(g_peak_cls));
  g_live_total = g_peak_total = 0;
}
static double* talloc(int64_t elems, int cls) {
  const uint64_t b = (uint64_t)elems * 8u;
  g_live[cls] += b;
  g_live_total += b;
  if (g_live[cls] > g_peak_cls[cls]) g_peak_cls[cls] = g_live[cls];
  if (g_live_total > g_peak_total) g_peak_total = g_live_total;
  return (double*)calloc((size_t)(elems > 0 ? elems : 1), sizeof(double));
}
static void tfree(double* p, int64_t elems, int cls) {
  const uint64_t b = (uint64_t)elems * 8u;
  g_live[cls] -= b;
  g_live_total -= b;
  free(p);
}
uint64_t orc_mem_peak(void) { return g_peak_total; }
uint64_t orc_mem_peak_class(int cls) { return (cls >= 0 && cls < ORC_MEM_NCLASS) ? g_peak_cls[cls] : 0; }
uint64_t orc_mem_live(void) { return g_live_total; }

/* ================================================================ chunk plan
 * SPEC.md:286-294.  Balanced rule: exactly min(M,N)
 * contiguous chunks, the first N mod M of size ceil(N/M). */
int orc_make_chunk_plan(int64_t n, int64_t m, int64_t* bounds, int64_t* count) {
  if (n <= 0) return ORC_ERR_DATA;
  if (m <= 0) return ORC_ERR_CONFIG;
  const int64_t c = i64min(n, m), q = n / c, r = n % c;
  bounds[0] = 0;
  for (int64_t i = 0; i < c; ++i) bounds[i + 1] = bounds[i] + q + (i < r ? 1 : 0);
  *count = c;
  return ORC_OK;
}

/* ================================================================ f64 math
 * matmul: SPEC.md:34-42 — C[i,j] = sum_k A[i,k] B[k,j] accumulated
 * sequentially in ascending k (i-k-j order keeps that per element). */
void orc_matmul_f64(const double* a, const double* b, double* c, int64_t n, int64_t k, int64_t p) {
  for (int64_t i = 0; i < n; ++i) {
    double* ci = c + i * p;
    for (int64_t j = 0; j < p; ++j) ci[j] = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) {
      const double av = a[i * k + kk];
      const double* bk = b + kk * p;
      for (int64_t j = 0; j < p; ++j) ci[j] += av * bk[j];
    }
  }
}

/* C[n,p] = A^T B with A stored [k,n] (used for X^T dG etc.). */
static void matmul_tn(const double* a, const double* b, double* c, int64_t n, int64_t k, int64_t p) {
  for (int64_t i = 0; i < n; ++i) {
    double* ci = c + i * p;
    for (int64_t j = 0; j < p; ++j) ci[j] = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) {
      const double av = a[kk * n + i];
      const double* bk = b + kk * p;
      for (int64_t j = 0; j < p; ++j) ci[j] += av * bk[j];
    }
  }
}

/* C[n,p] = A B^T with B stored [p,k]: B is transposed into a temporary and
 * the i-k-j product is used, so each element still accumulates in ascending
 * k (bitwise identical to the dot-product form). */
static void matmul_nt(const double* a, const double* b, double* c, int64_t n, int64_t k, int64_t p) {
  double* bt = (double*)malloc(sizeof(double) * (size_t)(k * p));
  for (int64_t j = 0; j < p; ++j)
    for (int64_t kk = 0; kk < k; ++kk) bt[kk * p + j] = b[j * k + kk];
  orc_matmul_f64(a, bt, c, n, k, p);
  free(bt);
}

static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }
/* SPEC.md:43-51 */
double orc_silu_f64(double x) { return x * sigm(x); }
/* upstream * (s + x s (1 - s)) */
double orc_silu_backward_f64(double x, double upstream) {
  const double s = sigm(x);
  return upstream * (s + x * s * (1.0 - s));
}
static double rb(double x, int round) { return round ? (double)orc_round_bf16((float)x) : x; }

/* ---------------------------------------------------------------- MLP
 * One MLP block over rows [0,n) of X (a chunk, or all rows = standard). */
static void mlp_fwd_rows(const double* X, const double* Wg, const double* Wu, const double* Wd, int64_t n, int64_t H,
                         int64_t I, double* O, int round) {
  double* G = talloc(n * I, ORC_MEM_INTER_MLP);
  double* U = talloc(n * I, ORC_MEM_INTER_MLP);
  double* h = talloc(n * I, ORC_MEM_INTER_MLP);
  orc_matmul_f64(X, Wg, G, n, H, I);
  count_matmul(n, H, I, (uint64_t)(H * I));
  orc_matmul_f64(X, Wu, U, n, H, I);
  count_matmul(n, H, I, (uint64_t)(H * I));
  for (int64_t e = 0; e < n * I; ++e) h[e] = rb(G[e] * sigm(G[e]) * U[e], round);
  count_op(4ull * n * I, 2ull * n * I); /* silu */
  count_op(1ull * n * I, 3ull * n * I); /* hadamard */
  orc_matmul_f64(h, Wd, O, n, I, H);
  count_matmul(n, I, H, (uint64_t)(I * H));
  for (int64_t e = 0; e < n * H; ++e) O[e] = rb(O[e], round);
  tfree(h, n * I, ORC_MEM_INTER_MLP);
  tfree(U, n * I, ORC_MEM_INTER_MLP);
  tfree(G, n * I, ORC_MEM_INTER_MLP);
}

/* Backward of one MLP block over n rows (recomputes G, U, h — the saved
 * set of SPEC.md:197 plus U, App. A-5).  Chunk weight grads go to cWg/cWu/cWd. */
static void mlp_bwd_rows(const double* dO, const double* X, const double* Wg, const double* Wu, const double* Wd,
                         int64_t n, int64_t H, int64_t I, double* dX, double* cWg, double* cWu, double* cWd,
                         int round) {
  double* G = talloc(n * I, ORC_MEM_INTER_MLP);
  double* U = talloc(n * I, ORC_MEM_INTER_MLP);
  double* h = talloc(n * I, ORC_MEM_INTER_MLP);
  double* dh = talloc(n * I, ORC_MEM_INTER_MLP);
  double* dG = talloc(n * I, ORC_MEM_INTER_MLP);
  double* dU = talloc(n * I, ORC_MEM_INTER_MLP);
  double* t = talloc(n * H, ORC_MEM_ACT);
  orc_matmul_f64(X, Wg, G, n, H, I);
  count_matmul(n, H, I, (uint64_t)(H * I));
  orc_matmul_f64(X, Wu, U, n, H, I);
  count_matmul(n, H, I, (uint64_t)(H * I));
  matmul_nt(dO, Wd, dh, n, H, I); /* dh = dO W_d^T */
  count_matmul(n, H, I, (uint64_t)(I * H));
  for (int64_t e = 0; e < n * I; ++e) {
    const double s = sigm(G[e]), act = G[e] * s;
    h[e] = rb(act * U[e], round);
    dG[e] = rb(dh[e] * U[e] * (s * (1.0 + G[e] * (1.0 - s))), round);
    dU[e] = rb(dh[e] * act, round);
  }
  count_op(4ull * n * I, 3ull * n * I);
  count_op(2ull * n * I, 6ull * n * I);
  matmul_tn(h, dO, cWd, I, n, H); /* dW_down = h^T dO */
  count_matmul(I, n, H, 0);
  matmul_nt(dG, Wg, dX, n, I, H); /* dX = dG W_g^T + dU W_u^T */
  count_matmul(n, I, H, (uint64_t)(H * I));
  matmul_nt(dU, Wu, t, n, I, H);
  count_matmul(n, I, H, (uint64_t)(H * I));
  for (int64_t e = 0; e < n * H; ++e) dX[e] = rb(dX[e] + t[e], round);
  count_op(1ull * n * H, 3ull * n * H);
  matmul_tn(X, dG, cWg, H, n, I); /* dW_gate = X^T dG, dW_up = X^T dU (App. A-3) */
  count_matmul(H, n, I, 0);
  matmul_tn(X, dU, cWu, H, n, I);
  count_matmul(H, n, I, 0);
  tfree(t, n * H, ORC_MEM_ACT);
  tfree(dU, n * I, ORC_MEM_INTER_MLP);
  tfree(dG, n * I, ORC_MEM_INTER_MLP);
  tfree(dh, n * I, ORC_MEM_INTER_MLP);
  tfree(h, n * I, ORC_MEM_INTER_MLP);
  tfree(U, n * I, ORC_MEM_INTER_MLP);
  tfree(G, n * I, ORC_MEM_INTER_MLP);
}

/* blocks-std mlp_forward */
int orc_mlp_forward_f64(const double* X, const double* Wg, const double* Wu, const double* Wd, int64_t N, int64_t H,
                        int64_t I, double* O, int round_bf16) {
  if (N <= 0 || H <= 0 || I <= 0) return ORC_ERR_SHAPE;
  mlp_fwd_rows(X, Wg, Wu, Wd, N, H, I, O, round_bf16);
  return ORC_OK;
}

/* blocks-std mlp_backward */
int orc_mlp_backward_f64(const double* dO, const double* X, const double* Wg, const double* Wu, const double* Wd,
                         int64_t N, int64_t H, int64_t I, double* dX, double* dWg, double* dWu, double* dWd,
                         int round_bf16) {
  if (N <= 0 || H <= 0 || I <= 0) return ORC_ERR_SHAPE;
  mlp_bwd_rows(dO, X, Wg, Wu, Wd, N, H, I, dX, dWg, dWu, dWd, round_bf16);
  return ORC_OK;
}

/* miniseq_mlp_forward, SPEC.md:295-303 / Alg. 1 */
int orc_miniseq_mlp_forward_f64(const double* X, const double* Wg, const double* Wu, const double* Wd, int64_t N,
                                int64_t H, int64_t I, int64_t M, double* O, int round_bf16) {
  if (H <= 0 || I <= 0) return ORC_ERR_SHAPE;
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(i64min(N > 0 ? N : 1, M > 0 ? M : 1) + 1));
  int64_t c;
  int st = orc_make_chunk_plan(N, M, b, &c);
  if (st) {
    free(b);
    return st;
  }
  for (int64_t i = 0; i < c; ++i) {
    const int64_t r0 = b[i], n = b[i + 1] - b[i];
    count_op(0, 2ull * n * H); /* slice_rows copy */
    mlp_fwd_rows(X + r0 * H, Wg, Wu, Wd, n, H, I, O + r0 * H, round_bf16);
    count_op(0, 2ull * n * H); /* concat_rows copy */
  }
  free(b);
  return ORC_OK;
}

static void acc_or_assign(double* dst, const double* src, int64_t n, int first) {
  if (first)
    memcpy(dst, src, sizeof(double) * (size_t)n);
  else
    for (int64_t e = 0; e < n; ++e) dst[e] += src[e];
}

/* miniseq_mlp_backward, SPEC.md:304-312 / Alg. 3: ascending chunks, dW
 * accumulated sequentially (first chunk assigns, so M=1 is bitwise std). */
int orc_miniseq_mlp_backward_f64(const double* dO, const double* X, const double* Wg, const double* Wu,
                                 const double* Wd, int64_t N, int64_t H, int64_t I, int64_t M, double* dX,
                                 double* dWg, double* dWu, double* dWd, int round_bf16) {
  if (H <= 0 || I <= 0) return ORC_ERR_SHAPE;
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(i64min(N > 0 ? N : 1, M > 0 ? M : 1) + 1));
  int64_t c;
  int st = orc_make_chunk_plan(N, M, b, &c);
  if (st) {
    free(b);
    return st;
  }
  double* cWg = talloc(H * I, ORC_MEM_GRAD);
  double* cWu = talloc(H * I, ORC_MEM_GRAD);
  double* cWd = talloc(I * H, ORC_MEM_GRAD);
  for (int64_t i = 0; i < c; ++i) {
    const int64_t r0 = b[i], n = b[i + 1] - b[i];
    mlp_bwd_rows(dO + r0 * H, X + r0 * H, Wg, Wu, Wd, n, H, I, dX + r0 * H, cWg, cWu, cWd, round_bf16);
    acc_or_assign(dWg, cWg, H * I, i == 0);
    acc_or_assign(dWu, cWu, H * I, i == 0);
    acc_or_assign(dWd, cWd, I * H, i == 0);
  }
  tfree(cWd, I * H, ORC_MEM_GRAD);
  tfree(cWu, H * I, ORC_MEM_GRAD);
  tfree(cWg, H * I, ORC_MEM_GRAD);
  free(b);
  return ORC_OK;
}

/* ---------------------------------------------------------------- LM-Head
 * Per-chunk forward: logits, lse, loss-sum and valid count. */
static void head_fwd_rows(const double* X, const int32_t* L, const double* Wout, int64_t n, int64_t H, int64_t V,
                          double* lse, double* sum_out, double* valid_out) {
  double* Z = talloc(n * V, ORC_MEM_INTER_HEAD);
  orc_matmul_f64(X, Wout, Z, n, H, V);
  count_matmul(n, H, V, (uint64_t)(H * V));
  count_op(5ull * n * V, (uint64_t)(n * V + 2 * n));
  double s = 0.0, cnt = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const double* z = Z + r * V;
    double mx = -INFINITY;
    for (int64_t v = 0; v < V; ++v) mx = z[v] > mx ? z[v] : mx;
    double se = 0.0;
    for (int64_t v = 0; v < V; ++v) se += exp(z[v] - mx);
    lse[r] = mx + log(se);
    const int32_t lab = L[r];
    if (lab >= 0 && lab < V) {
      s += lse[r] - z[lab];
      cnt += 1.0;
    }
  }
  *sum_out = s;
  *valid_out = cnt;
  tfree(Z, n * V, ORC_MEM_INTER_HEAD);
}

/* Per-chunk backward: dl = (exp(z - lse) - onehot) * scale.
 * round == 2 additionally replays the GPU single-pass head's rounding
 * (tuning dl_rowscale=0): the softmax numerator
 * exp(z - m_tile) relative to its 256-column vocabulary tile's maximum is
 * stored in bf16 first; the label column is computed from the fp32 logit.
 * round == 3 replays the row-scaled head (the GPU default): numerators
 * 2^(z log2e - R) stored in bf16 with R = 0 while every tile maximum lies
 * within +-64 (log2 units; else the tile maximum, then rescaled to the row
 * reference R*), label column (p_label - 1) 2^(lse2 - R*), per-row factor
 * f = scale 2^(R* - lse2); dX = bf16(f * (e' W_out^T)), dW_out += bf16(f X)^T e'. */
#define ORC_CE_REF_WINDOW 64.0
static void head_bwd_rows_rowscale(const double* X, const int32_t* L, const double* Wout, int64_t n, int64_t H,
                                   int64_t V, const double* lse, double scale, double* dX, double* cWout, double* Z) {
  const double log2e = 1.4426950408889634;
  double* f = (double*)malloc(sizeof(double) * (size_t)n);
  double* Xs = (double*)malloc(sizeof(double) * (size_t)(n * H));
  for (int64_t r = 0; r < n; ++r) {
    double* z = Z + r * V;
    const int32_t lab = L[r];
    const int valid = lab >= 0 && lab < V;
    const double zlab = valid ? z[lab] : 0.0;
    const double l2 = lse[r] * log2e;
    int special = 0;
    for (int64_t t0 = 0; t0 < V; t0 += 256) {
      const int64_t t1 = t0 + 256 < V ? t0 + 256 : V;
      double mt = -INFINITY;
      for (int64_t v = t0; v < t1; ++v) mt = z[v] * log2e > mt ? z[v] * log2e : mt;
      if (fabs(mt) > ORC_CE_REF_WINDOW) special = 1;
    }
    const double rs = (!special || fabs(l2) <= ORC_CE_REF_WINDOW) ? 0.0 : rint(l2);
    for (int64_t t0 = 0; t0 < V; t0 += 256) {
      const int64_t t1 = t0 + 256 < V ? t0 + 256 : V;
      double mt = -INFINITY;
      for (int64_t v = t0; v < t1; ++v) mt = z[v] * log2e > mt ? z[v] * log2e : mt;
      const double ref = fabs(mt) <= ORC_CE_REF_WINDOW ? 0.0 : mt;
      for (int64_t v = t0; v < t1; ++v) {
        double e = rb(exp2(z[v] * log2e - ref), 1);
        if (ref != rs) e = rb(e * exp2(ref - rs), 1);
        z[v] = e;
      }
    }
    if (valid) z[lab] = rb((exp(zlab - lse[r]) - 1.0) * exp2(l2 - rs), 1);
    f[r] = valid ? scale * exp2(rs - l2) : 0.0;
    for (int64_t k = 0; k < H; ++k) Xs[r * H + k] = rb(X[r * H + k] * f[r], 1);
  }
  count_op(5ull * n * V, (uint64_t)(2 * n * V + 2 * n));
  matmul_nt(Z, Wout, dX, n, V, H); /* dX = f * (e' W_out^T) */
  count_matmul(n, V, H, (uint64_t)(H * V));
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = 0; k < H; ++k) dX[r * H + k] = rb(dX[r * H + k] * f[r], 1);
  matmul_tn(Xs, Z, cWout, H, n, V); /* dW_out = (f X)^T e' */
  count_matmul(H, n, V, 0);
  free(Xs);
  free(f);
}

static void head_bwd_rows(const double* X, const int32_t* L, const double* Wout, int64_t n, int64_t H, int64_t V,
                          const double* lse, double scale, double* dX, double* cWout, int round) {
  double* Z = talloc(n * V, ORC_MEM_INTER_HEAD);
  orc_matmul_f64(X, Wout, Z, n, H, V);
  count_matmul(n, H, V, (uint64_t)(H * V));
  if (round == 3) {
    head_bwd_rows_rowscale(X, L, Wout, n, H, V, lse, scale, dX, cWout, Z);
    tfree(Z, n * V, ORC_MEM_INTER_HEAD);
    return;
  }
  for (int64_t r = 0; r < n; ++r) {
    double* z = Z + r * V;
    const int32_t lab = L[r];
    const int valid = lab >= 0 && lab < V;
    for (int64_t t0 = 0; t0 < V; t0 += 256) {
      const int64_t t1 = t0 + 256 < V ? t0 + 256 : V;
      double mt = -INFINITY;
      for (int64_t v = t0; v < t1; ++v) mt = z[v] > mt ? z[v] : mt;
      for (int64_t v = t0; v < t1; ++v) {
        double p;
        if (round == 2 && v != lab)
          p = rb(exp(z[v] - mt), 1) * exp(mt - lse[r]);
        else
          p = exp(z[v] - lse[r]);
        z[v] = valid ? rb((p - (v == lab ? 1.0 : 0.0)) * scale, round) : 0.0;
      }
    }
  }
  count_op(5ull * n * V, (uint64_t)(2 * n * V + 2 * n));
  matmul_nt(Z, Wout, dX, n, V, H); /* dX = dl W_out^T */
  count_matmul(n, V, H, (uint64_t)(H * V));
  for (int64_t e = 0; e < n * H; ++e) dX[e] = rb(dX[e], round);
  matmul_tn(X, Z, cWout, H, n, V); /* dW_out = X^T dl */
  count_matmul(H, n, V, 0);
  tfree(Z, n * V, ORC_MEM_INTER_HEAD);
}

static int64_t count_valid(const int32_t* L, int64_t n, int64_t V) {
  int64_t c = 0;
  for (int64_t r = 0; r < n; ++r) c += (L[r] >= 0 && L[r] < V);
  return c;
}

/* blocks-std lmhead_forward: mean CE over non-ignored rows; all ignored -> error */
int orc_lmhead_forward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H, int64_t V,
                           double* loss, double* lse) {
  if (N <= 0 || H <= 0 || V <= 0) return ORC_ERR_SHAPE;
  double s, cnt;
  head_fwd_rows(X, L, Wout, N, H, V, lse, &s, &cnt);
  if (cnt == 0.0) return ORC_ERR_DATA;
  *loss = s / cnt;
  return ORC_OK;
}

/* blocks-std lmhead_backward: dl = (softmax - onehot) * grad_loss / n_valid */
int orc_lmhead_backward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H, int64_t V,
                            double grad_loss, double* dX, double* dWout, int round_bf16) {
  if (N <= 0 || H <= 0 || V <= 0) return ORC_ERR_SHAPE;
  const int64_t nv = count_valid(L, N, V);
  if (nv == 0) return ORC_ERR_DATA;
  double* lse = (double*)malloc(sizeof(double) * (size_t)N);
  double s, cnt;
  head_fwd_rows(X, L, Wout, N, H, V, lse, &s, &cnt);
  head_bwd_rows(X, L, Wout, N, H, V, lse, grad_loss / (double)nv, dX, dWout, round_bf16);
  free(lse);
  return ORC_OK;
}

/* miniseq_lmhead_forward, SPEC.md:313-321 / Alg. 2 */
int orc_miniseq_lmhead_forward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H,
                                   int64_t V, int64_t M, int mode, double* loss, double* lse, double* chunk_sum,
                                   double* chunk_valid) {
  if (H <= 0 || V <= 0) return ORC_ERR_SHAPE;
  if (mode != 0 && mode != 1) return ORC_ERR_CONFIG;
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(i64min(N > 0 ? N : 1, M > 0 ? M : 1) + 1));
  int64_t c;
  int st = orc_make_chunk_plan(N, M, b, &c);
  if (st) {
    free(b);
    return st;
  }
  double tot = 0.0, tv = 0.0, pm = 0.0;
  for (int64_t i = 0; i < c; ++i) {
    const int64_t r0 = b[i], n = b[i + 1] - b[i];
    double s, cnt;
    head_fwd_rows(X + r0 * H, L + r0, Wout, n, H, V, lse + r0, &s, &cnt);
    if (chunk_sum) chunk_sum[i] = s;
    if (chunk_valid) chunk_valid[i] = cnt;
    tot = i == 0 ? s : tot + s;
    tv += cnt;
    if (cnt > 0) pm += s / cnt; /* degenerate chunk contributes 0 in paper-mean */
  }
  free(b);
  if (tv == 0.0) return ORC_ERR_DATA;
  *loss = mode == 0 ? tot / tv : pm / (double)c;
  return ORC_OK;
}

/* miniseq_lmhead_backward, SPEC.md:322-330 / Alg. 4 (logits recomputed per chunk). */
int orc_miniseq_lmhead_backward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H,
                                    int64_t V, int64_t M, int mode, double grad_loss, double* dX, double* dWout,
                                    int round_bf16) {
  if (H <= 0 || V <= 0) return ORC_ERR_SHAPE;
  if (mode != 0 && mode != 1) return ORC_ERR_CONFIG;
  int64_t* b = (int64_t*)malloc(sizeof(int64_t) * (size_t)(i64min(N > 0 ? N : 1, M > 0 ? M : 1) + 1));
  int64_t c;
  int st = orc_make_chunk_plan(N, M, b, &c);
  if (st) {
    free(b);
    return st;
  }
  const int64_t nv = count_valid(L, N, V);
  if (nv == 0) {
    free(b);
    return ORC_ERR_DATA;
  }
  double* lse = (double*)malloc(sizeof(double) * (size_t)N);
  double* cW = talloc(H * V, ORC_MEM_GRAD);
  for (int64_t i = 0; i < c; ++i) {
    const int64_t r0 = b[i], n = b[i + 1] - b[i];
    double s, cnt;
    head_fwd_rows(X + r0 * H, L + r0, Wout, n, H, V, lse + r0, &s, &cnt); /* saved lse of the forward */
    const double scale = mode == 0 ? grad_loss / (double)nv : (cnt > 0 ? grad_loss / ((double)c * cnt) : 0.0);
    head_bwd_rows(X + r0 * H, L + r0, Wout, n, H, V, lse + r0, scale, dX + r0 * H, cW, round_bf16);
    acc_or_assign(dWout, cW, H * V, i == 0);
  }
  tfree(cW, H * V, ORC_MEM_GRAD);
  free(lse);
  free(b);
  return ORC_OK;
}

/* ================================================================ f32 block
 * CPU baseline.  Same algorithm, f32, sequential-K matmuls blocked for
 * cache reuse (4 output rows x 128 columns per block; per-element k order
 * unchanged), OpenMP over row blocks. */
#define IB 16
#define JB 64

/* C[n,p] (+)= A B.  Blocks of IB rows x JB columns; each block runs k in
 * ascending order, so per-element accumulation order is the SPEC's. */
static void mm_nn_f32(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int64_t n,
                      int64_t k, int64_t p, int accumulate, int nth) {
  (void)nth;
  const int64_t nib = (n + IB - 1) / IB, njb = (p + JB - 1) / JB;
#pragma omp parallel for collapse(2) schedule(dynamic, 4) num_threads(nth) if (nth > 1)
  for (int64_t bi = 0; bi < nib; ++bi)
    for (int64_t bj = 0; bj < njb; ++bj) {
      const int64_t i0 = bi * IB, j0 = bj * JB;
      const int64_t ib = i64min(IB, n - i0), jb = i64min(JB, p - j0);
      float acc[IB][JB];
      for (int64_t r = 0; r < IB; ++r)
        for (int64_t j = 0; j < JB; ++j) acc[r][j] = (accumulate && r < ib && j < jb) ? C[(i0 + r) * ldc + j0 + j] : 0.f;
      if (jb == JB) {
        for (int64_t kk = 0; kk < k; ++kk) {
          const float* b = B + kk * ldb + j0;
          for (int64_t r = 0; r < ib; ++r) {
            const float a = A[(i0 + r) * lda + kk];
#pragma omp simd
            for (int64_t j = 0; j < JB; ++j) acc[r][j] += a * b[j];
          }
        }
      } else {
        for (int64_t kk = 0; kk < k; ++kk) {
          const float* b = B + kk * ldb + j0;
          for (int64_t r = 0; r < ib; ++r) {
            const float a = A[(i0 + r) * lda + kk];
            for (int64_t j = 0; j < jb; ++j) acc[r][j] += a * b[j];
          }
        }
      }
      for (int64_t r = 0; r < ib; ++r) memcpy(C + (i0 + r) * ldc + j0, acc[r], sizeof(float) * (size_t)jb);
    }
}

/* C[n,p] (+)= A^T B, A stored [k,n] (lda), B [k,p]. */
static void mm_tn_f32(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int64_t n,
                      int64_t k, int64_t p, int accumulate, int nth) {
  (void)nth;
  const int64_t nib = (n + IB - 1) / IB, njb = (p + JB - 1) / JB;
#pragma omp parallel for collapse(2) schedule(dynamic, 4) num_threads(nth) if (nth > 1)
  for (int64_t bi = 0; bi < nib; ++bi)
    for (int64_t bj = 0; bj < njb; ++bj) {
      const int64_t i0 = bi * IB, j0 = bj * JB;
      const int64_t ib = i64min(IB, n - i0), jb = i64min(JB, p - j0);
      float acc[IB][JB];
      for (int64_t r = 0; r < IB; ++r)
        for (int64_t j = 0; j < JB; ++j) acc[r][j] = (accumulate && r < ib && j < jb) ? C[(i0 + r) * ldc + j0 + j] : 0.f;
      for (int64_t kk = 0; kk < k; ++kk) {
        const float* b = B + kk * ldb + j0;
        const float* a = A + kk * lda + i0;
        for (int64_t r = 0; r < ib; ++r) {
          const float av = a[r];
          if (jb == JB) {
#pragma omp simd
            for (int64_t j = 0; j < JB; ++j) acc[r][j] += av * b[j];
          } else {
            for (int64_t j = 0; j < jb; ++j) acc[r][j] += av * b[j];
          }
        }
      }
      for (int64_t r = 0; r < ib; ++r) memcpy(C + (i0 + r) * ldc + j0, acc[r], sizeof(float) * (size_t)jb);
    }
}

void orc_transpose_f32(const float* a, float* at, int64_t rows, int64_t cols, int nth) {
  (void)nth;
#pragma omp parallel for schedule(static) num_threads(nth) if (nth > 1)
  for (int64_t r0 = 0; r0 < rows; r0 += 64)
    for (int64_t c0 = 0; c0 < cols; c0 += 64)
      for (int64_t r = r0; r < i64min(rows, r0 + 64); ++r)
        for (int64_t c = c0; c < i64min(cols, c0 + 64); ++c) at[c * rows + r] = a[r * cols + c];
}

static float sigf(float x) { return 1.0f / (1.0f + expf(-x)); }

int orc_block_step_f32(orc_block_f32* B, int nth) {
  const int64_t N = B->N, H = B->H, I = B->I, V = B->V;
  if (N <= 0 || H <= 0 || I <= 0 || V <= 0) return ORC_ERR_SHAPE;
  int64_t cm = i64min(N, B->M_mlp), chh = i64min(N, B->M_head);
  int64_t *bm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cm + 1)), *bh = (int64_t*)malloc(sizeof(int64_t) * (size_t)(chh + 1));
  int st = orc_make_chunk_plan(N, B->M_mlp, bm, &cm);
  if (!st) st = orc_make_chunk_plan(N, B->M_head, bh, &chh);
  if (st) {
    free(bm);
    free(bh);
    return st;
  }
  int64_t nmax = 0;
  for (int64_t i = 0; i < cm; ++i) nmax = bm[i + 1] - bm[i] > nmax ? bm[i + 1] - bm[i] : nmax;
  int64_t nhmax = 0;
  for (int64_t i = 0; i < chh; ++i) nhmax = bh[i + 1] - bh[i] > nhmax ? bh[i + 1] - bh[i] : nhmax;
  float* O = (float*)malloc(sizeof(float) * (size_t)(N * H));
  float* dO = (float*)malloc(sizeof(float) * (size_t)(N * H));
  float* lse = (float*)malloc(sizeof(float) * (size_t)N);
  float* G = (float*)malloc(sizeof(float) * (size_t)(nmax * I));
  float* U = (float*)malloc(sizeof(float) * (size_t)(nmax * I));
  float* hh = (float*)malloc(sizeof(float) * (size_t)(nmax * I));
  float* dh = (float*)malloc(sizeof(float) * (size_t)(nmax * I));
  float* Z = (float*)malloc(sizeof(float) * (size_t)(nhmax * V));
  /* MLP forward (Alg. 1) */
  for (int64_t c = 0; c < cm; ++c) {
    const int64_t r0 = bm[c], n = bm[c + 1] - bm[c];
    const float* Xc = B->X + r0 * H;
    mm_nn_f32(Xc, H, B->Wg, I, G, I, n, H, I, 0, nth);
    mm_nn_f32(Xc, H, B->Wu, I, U, I, n, H, I, 0, nth);
    for (int64_t e = 0; e < n * I; ++e) hh[e] = G[e] * sigf(G[e]) * U[e];
    mm_nn_f32(hh, I, B->Wd, H, O + r0 * H, H, n, I, H, 0, nth);
  }
  /* LM-Head forward (Alg. 2, token-weighted) */
  double lsum = 0.0;
  int64_t nvalid = 0;
  for (int64_t c = 0; c < chh; ++c) {
    const int64_t r0 = bh[c], n = bh[c + 1] - bh[c];
    mm_nn_f32(O + r0 * H, H, B->Wout, V, Z, V, n, H, V, 0, nth);
    for (int64_t r = 0; r < n; ++r) {
      const float* z = Z + r * V;
      float mx = -INFINITY;
      for (int64_t v = 0; v < V; ++v) mx = z[v] > mx ? z[v] : mx;
      double se = 0.0;
      for (int64_t v = 0; v < V; ++v) se += expf(z[v] - mx);
      lse[r0 + r] = mx + (float)log(se);
      const int32_t lab = B->L[r0 + r];
      if (lab >= 0 && lab < V) {
        lsum += lse[r0 + r] - z[lab];
        nvalid++;
      }
    }
  }
  B->loss = nvalid ? lsum / (double)nvalid : NAN;
  const float scale = nvalid ? 1.0f / (float)nvalid : 0.0f;
  /* LM-Head backward (Alg. 4): recompute logits, dlogits, dO, dW_out */
  for (int64_t c = 0; c < chh; ++c) {
    const int64_t r0 = bh[c], n = bh[c + 1] - bh[c];
    mm_nn_f32(O + r0 * H, H, B->Wout, V, Z, V, n, H, V, 0, nth);
    for (int64_t r = 0; r < n; ++r) {
      float* z = Z + r * V;
      const int32_t lab = B->L[r0 + r];
      const int valid = lab >= 0 && lab < V;
      for (int64_t v = 0; v < V; ++v) z[v] = valid ? (expf(z[v] - lse[r0 + r]) - (v == lab ? 1.f : 0.f)) * scale : 0.f;
    }
    mm_nn_f32(Z, V, B->WoutT, H, dO + r0 * H, H, n, V, H, 0, nth);
    mm_tn_f32(O + r0 * H, H, Z, V, B->dWout, V, H, n, V, c > 0, nth);
  }
  /* MLP backward (Alg. 3) */
  for (int64_t c = 0; c < cm; ++c) {
    const int64_t r0 = bm[c], n = bm[c + 1] - bm[c];
    const float* Xc = B->X + r0 * H;
    const float* dOc = dO + r0 * H;
    mm_nn_f32(Xc, H, B->Wg, I, G, I, n, H, I, 0, nth);
    mm_nn_f32(Xc, H, B->Wu, I, U, I, n, H, I, 0, nth);
    mm_nn_f32(dOc, H, B->WdT, I, dh, I, n, H, I, 0, nth);
    for (int64_t e = 0; e < n * I; ++e) {
      const float s = sigf(G[e]), act = G[e] * s;
      hh[e] = act * U[e];
      const float dg = dh[e] * U[e] * (s * (1.f + G[e] * (1.f - s)));
      U[e] = dh[e] * act; /* dU */
      G[e] = dg;          /* dG */
    }
    mm_tn_f32(hh, I, dOc, H, B->dWd, H, I, n, H, c > 0, nth);
    mm_nn_f32(G, I, B->WgT, H, B->dX + r0 * H, H, n, I, H, 0, nth);
    mm_nn_f32(U, I, B->WuT, H, B->dX + r0 * H, H, n, I, H, 1, nth);
    mm_tn_f32(Xc, H, G, I, B->dWg, I, H, n, I, c > 0, nth);
    mm_tn_f32(Xc, H, U, I, B->dWu, I, H, n, I, c > 0, nth);
  }
  free(O);
  free(dO);
  free(lse);
  free(G);
  free(U);
  free(hh);
  free(dh);
  free(Z);
  free(bm);
  free(bh);
  return ORC_OK;
}
