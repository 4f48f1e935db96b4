/*
 * mst_oracle.h — CPU restatement of the reference's mini-sequence path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or the timed CPU baseline — never as part of the
 * product path (libmst.so has no dependency on it).
 *
 * Restates, function by function (citations into /root/reference):
 *   rng            proj/include/minitrain/rng.hpp:8-72
 *   matmul         SPEC.md:34-42, SPEC.md:96 (sequential K accumulation)
 *   silu(_bwd)
 *   counters       proj/include/minitrain/memtrack.hpp:19-35, 163-175
 *   blocks-std     SPEC.md:197-232 (MLP / LM-Head, standard = unchunked)
 *   miniseq        SPEC.md:286-361, Alg. 1-4
 *
 * Parity pinning: the Rng is checked bit-for-bit against the reference's own
 * rng.hpp compiled from /root/reference (oracle/ref_build.sh ->
 * tests/golden/rng_golden.json); the math is checked against every SPEC
 * known-answer example (tests/test_oracle.py).  The reference ships no
 * miniseq implementation, so beyond those KATs the restatement is
 * "parity pinned to SPEC examples".
 */
#ifndef MST_ORACLE_H_
#define MST_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- rng */
typedef struct orc_rng {
  uint64_t root_seed;
  uint64_t s[4];
} orc_rng;

uint64_t orc_splitmix64(uint64_t* state);
uint64_t orc_fnv1a64(const char* s);
void orc_rng_init(orc_rng* r, uint64_t seed);
void orc_rng_fork(const orc_rng* r, const char* name, orc_rng* out);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
uint64_t orc_rng_uniform_below(orc_rng* r, uint64_t n);
double orc_rng_gaussian(orc_rng* r);
/* Fill helpers: out[i] = bf16(std * gaussian()) as float; labels uniform in
 * [0,V) with probability p_ignore of -100 (draws: uniform then below). */
void orc_fill_gaussian_bf16(orc_rng* r, float* out, int64_t n, double std);
void orc_fill_labels(orc_rng* r, int32_t* out, int64_t n, int64_t vocab, double p_ignore);
float orc_round_bf16(float x);

/* ---------------------------------------------------------------- counters */
typedef struct orc_counters {
  uint64_t flops, matmul_flops, hbm_elements, weight_read_elements;
} orc_counters;
void orc_counters_reset(void);
void orc_counters_get(orc_counters* out);

/* Memory tracker (memtrack.hpp:138-228 semantics, label classes only). */
enum { ORC_MEM_ACT = 0, ORC_MEM_INTER_MLP = 1, ORC_MEM_INTER_HEAD = 2, ORC_MEM_GRAD = 3, ORC_MEM_NCLASS = 4 };
void orc_mem_reset(void);
/* peak of total live bytes, and peak per class (replayed, memtrack.hpp:97-110) */
uint64_t orc_mem_peak(void);
uint64_t orc_mem_peak_class(int cls);
uint64_t orc_mem_live(void);

/* ---------------------------------------------------------------- chunk plan */
int orc_make_chunk_plan(int64_t n, int64_t m, int64_t* bounds, int64_t* count);

/* ---------------------------------------------------------------- f64 ops
 * All matrices row-major.  round_bf16 != 0 rounds to bf16 exactly where the
 * GPU stores bf16 (h, O, dlogits, dX of the head, dG, dU, dX of the MLP).
 * Return 0 on success or an mst_status-compatible error code. */
void orc_matmul_f64(const double* a, const double* b, double* c, int64_t n, int64_t k, int64_t p);
double orc_silu_f64(double x);
double orc_silu_backward_f64(double x, double upstream);

int orc_mlp_forward_f64(const double* X, const double* Wg, const double* Wu, const double* Wd, int64_t N, int64_t H,
                        int64_t I, double* O, int round_bf16);
int orc_mlp_backward_f64(const double* dO, const double* X, const double* Wg, const double* Wu, const double* Wd,
                         int64_t N, int64_t H, int64_t I, double* dX, double* dWg, double* dWu, double* dWd,
                         int round_bf16);
int orc_lmhead_forward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H, int64_t V,
                           double* loss, double* lse);
int orc_lmhead_backward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H, int64_t V,
                            double grad_loss, double* dX, double* dWout, int round_bf16);

int orc_miniseq_mlp_forward_f64(const double* X, const double* Wg, const double* Wu, const double* Wd, int64_t N,
                                int64_t H, int64_t I, int64_t M, double* O, int round_bf16);
int orc_miniseq_mlp_backward_f64(const double* dO, const double* X, const double* Wg, const double* Wu,
                                 const double* Wd, int64_t N, int64_t H, int64_t I, int64_t M, double* dX,
                                 double* dWg, double* dWu, double* dWd, int round_bf16);
/* mode 0 token-weighted, 1 paper-mean.  chunk_sum/chunk_valid: [num chunks] or NULL. */
int orc_miniseq_lmhead_forward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H,
                                   int64_t V, int64_t M, int mode, double* loss, double* lse, double* chunk_sum,
                                   double* chunk_valid);
int orc_miniseq_lmhead_backward_f64(const double* X, const int32_t* L, const double* Wout, int64_t N, int64_t H,
                                    int64_t V, int64_t M, int mode, double grad_loss, double* dX, double* dWout,
                                    int round_bf16);

/* ---------------------------------------------------------------- f32 block
 * The CPU baseline: one MLP -> LM-Head block fwd+bwd in f32 with the same
 * sequential-K matmuls, parallelised over output rows with OpenMP when
 * nthreads > 1 (SPEC.md:99 allows distinct tensors on distinct threads; the
 * per-element accumulation order is unchanged, so results are bitwise equal
 * to nthreads == 1).  Weights are passed with their transposes (a CPU layout
 * choice made once, outside the step).  Returns 0 or an error code. */
typedef struct orc_block_f32 {
  int64_t N, H, I, V, M_mlp, M_head;
  const float *X, *Wg, *Wu, *Wd, *Wout;     /* SPEC orientation */
  const float *WgT, *WuT, *WdT, *WoutT;     /* transposes */
  const int32_t* L;
  float *dX, *dWg, *dWu, *dWd, *dWout;      /* outputs */
  double loss;
} orc_block_f32;
int orc_block_step_f32(orc_block_f32* b, int nthreads);
void orc_transpose_f32(const float* a, float* at, int64_t rows, int64_t cols, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
