/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU oracle for the ColTrast late-interaction (MaxSim) hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * this library.  The product path (paper_2505_04846_b200/) never imports, links or calls it, and this
 * file shares no code, header, table or constant with the CUDA path.
 *
 * Arithmetic is IEEE float64 unless a function states otherwise.  Compile with -O2
 * -ffp-contract=off (no FMA contraction: NORM below is specified operation by operation).
 *
 * Functions and the passage each follows (PAPER.md = /root/reference/PAPER.md line numbers,
 * SPEC.md = /root/reference/SPEC.md line numbers; DESIGN.md "Readings" lists every gap reading):
 *
 *   oracle_norm_rows      NORM: per-row L2 normalisation on entry ("MaxSim uses cosine per token pair
 *                         (rows normalized on entry to the store)"; cosine
 *                         §2.2).  The exact fp32 recipe is DESIGN.md reading R1 (SURVEY §8(c) NORM).
 *                         pinned: tests/test_oracle_pins.py::test_norm_* (exact-rational reference,
 *                         power-of-two scale invariance, exactly-representable unit rows).
 *   oracle_maxsim         S(q,d) = sum_i max_j <q_i, d_j> (§2.2 "maximizing pairwise
 *                         similarity between query and text token embeddings"; Fig.3B;
 *                         SPEC.md:259-267 [OP] maxsim).  Length masking: readings R2/R3.
 *                         pinned: P1 brute force, P2 permutations, P3 single-token closed form,
 *                         P4 = len_q, P5 bound/monotone, P6 SPEC example, P10 masking adversary.
 *   oracle_maxsim_matrix  the same, for every (query, doc) pair (OpenMP over pairs only).
 *   oracle_topk           exact top-k: all scores, stable order (score desc, id asc), first min(k,n),
 *                         padded (-inf, -1) (§2.3 "identify the nearest neighbors";
 *                         SPEC.md:193-201 [OP] search; reading R6/R7).  pinned: P9.
 *   oracle_infonce        L = mean_i [ logsumexp_j (S_ij / tau) - S_{i,pos_i} / tau ]  (PAPER.md:252
 *                         "L_LI is maxsim loss"; SPEC.md:339-347 [OP] li_loss; tau reading R9).
 *                         pinned: P7 closed forms, P8 torch cross_entropy float64.
 *   oracle_maxsim_infonce_grad  NEXT N1: dL_LI/dx by the chain rule through argmax + normalisation
 *                         (PAPER.md:247-252 training; SPEC.md:357-365 grad_check).
 *                         pinned: central finite differences in float64 (<= 1e-4 relative).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- bf16 <-> fp32 (bit level) */

static float o_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* IEEE round-to-nearest-even of a finite float32 to bfloat16. */
static uint16_t o_f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

/* ---------------------------------------------------------------- NORM (reading R1)
 * For one row x[0..d) (fp32; bf16 inputs are widened exactly first):
 *   1. acc = 0.0f; for k ascending: acc = fmaf(x_k, x_k, acc)      (one rounding per step)
 *   2. acc == 0  -> error (SPEC ZeroVector)
 *   3. inv = 1.0f / sqrtf(acc)                                      (two correctly rounded ops)
 *   4. y_k = RNE_bf16(x_k * inv)                                     (fp32 RN multiply, then RNE)
 * in_dtype: 0 = float32 rows, 1 = bfloat16 rows (uint16 bit patterns).
 * assume_normalized != 0: skip steps 1-3 and store RNE_bf16(x_k) (reading R12).
 * Returns -1 on success, else the index of the first zero row (2) or non-finite row.
 * status_out (may be NULL): 0 ok, 1 zero row, 2 non-finite entry.
 */
int64_t oracle_norm_rows(const void* x, int32_t in_dtype, int64_t n_rows, int32_t d,
                         int32_t assume_normalized, uint16_t* y, int32_t* status_out) {
  if (status_out) *status_out = 0;
  for (int64_t r = 0; r < n_rows; ++r) {
    float row[4096];
    if (d > 4096) return r;
    for (int32_t k = 0; k < d; ++k) {
      if (in_dtype == 0) row[k] = ((const float*)x)[r * d + k];
      else row[k] = o_bf16_to_f32(((const uint16_t*)x)[r * d + k]);
      if (!isfinite(row[k])) {
        if (status_out) *status_out = 2;
        return r;
      }
    }
    if (assume_normalized) {
      for (int32_t k = 0; k < d; ++k) y[r * d + k] = o_f32_to_bf16_rne(row[k]);
      continue;
    }
    float acc = 0.0f;
    for (int32_t k = 0; k < d; ++k) acc = fmaf(row[k], row[k], acc);
    if (acc == 0.0f) {
      if (status_out) *status_out = 1;
      return r;
    }
    float s = sqrtf(acc);
    float inv = 1.0f / s;
    for (int32_t k = 0; k < d; ++k) {
      float p = row[k] * inv;
      y[r * d + k] = o_f32_to_bf16_rne(p);
    }
  }
  return -1;
}

/* ---------------------------------------------------------------- MaxSim
 * q:   len_q rows of dim d (bf16 bit patterns, already NORM'd), row-major
 * doc: len_d rows of dim d
 * Query rows i >= len_q and doc rows j >= len_d are simply not visited (readings R2, R3): the max
 * runs over the chunk's real tokens only, the sum over the query's real tokens only.  No length
 * normalisation (R4).  Every bf16 value widens exactly to float64.
 */
double oracle_maxsim(const uint16_t* q, int32_t len_q, const uint16_t* doc, int32_t len_d,
                     int32_t d) {
  double s = 0.0;
  for (int32_t i = 0; i < len_q; ++i) {
    double m = -INFINITY;
    for (int32_t j = 0; j < len_d; ++j) {
      double dot = 0.0;
      for (int32_t k = 0; k < d; ++k)
        dot += (double)o_bf16_to_f32(q[(int64_t)i * d + k]) *
               (double)o_bf16_to_f32(doc[(int64_t)j * d + k]);
      if (dot > m) m = dot;
    }
    s += m;
  }
  return s;
}

/* All pairs.  q_tokens: [n_q][q_stride_rows][d]; d_tokens: [n_d][d_stride_rows][d];
 * out: [n_q][n_d] float64.  OpenMP over pairs only (no blocking or reordering of the arithmetic).
 * n_threads <= 0: OpenMP default. */
void oracle_maxsim_matrix(const uint16_t* q_tokens, const int32_t* q_lens, int64_t n_q,
                          int32_t q_stride_rows, const uint16_t* d_tokens, const int32_t* d_lens,
                          int64_t n_d, int32_t d_stride_rows, int32_t d, double* out,
                          int32_t n_threads) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#else
  (void)n_threads;
#endif
  int64_t total = n_q * n_d;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < total; ++t) {
    int64_t i = t / n_d, j = t % n_d;
    out[t] = oracle_maxsim(q_tokens + i * (int64_t)q_stride_rows * d, q_lens[i],
                           d_tokens + j * (int64_t)d_stride_rows * d, d_lens[j], d);
  }
}

int32_t oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------- exact top-k
 * Sort all n candidates by score descending, ties by ascending id, keep the
 * first min(k, n), pad the rest with (-inf, -1) (reading R7).
 */
typedef struct {
  double score;
  int64_t id;
} o_hit;

static int o_hit_cmp(const void* a, const void* b) {
  const o_hit* x = (const o_hit*)a;
  const o_hit* y = (const o_hit*)b;
  if (x->score > y->score) return -1;
  if (x->score < y->score) return 1;
  if (x->id < y->id) return -1;
  if (x->id > y->id) return 1;
  return 0;
}

void oracle_topk(const double* scores, const int64_t* ids, int64_t n, int32_t k,
                 double* out_scores, int64_t* out_ids) {
  o_hit* h = (o_hit*)malloc(sizeof(o_hit) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    h[i].score = scores[i];
    h[i].id = ids[i];
  }
  qsort(h, (size_t)n, sizeof(o_hit), o_hit_cmp);
  for (int32_t r = 0; r < k; ++r) {
    if (r < n) {
      out_scores[r] = h[r].score;
      out_ids[r] = h[r].id;
    } else {
      out_scores[r] = -INFINITY;
      out_ids[r] = -1;
    }
  }
  free(h);
}

/* ---------------------------------------------------------------- InfoNCE over MaxSim scores
 * ("L_LI is maxsim loss" citing ColBERT; SPEC.md:339-347 li_loss: "softmax
 * cross-entropy over in-batch passages using maxsim scores ... loss = mean_i -log softmax(s_i)[i]")
 * S: [B][M] float64, pos: [B] (positive column per row), tau > 0 (reading R9; tau = 1 is SPEC's li_loss).
 *   z_ij = S_ij / tau
 *   l_i  = logsumexp_j z_ij - z_{i,pos_i}        (logsumexp max-shifted, float64)
 *   L    = (1/B) sum_i l_i
 */
double oracle_infonce(const double* S, int32_t B, int32_t M, const int32_t* pos, double tau) {
  double total = 0.0;
  for (int32_t i = 0; i < B; ++i) {
    double mx = -INFINITY;
    for (int32_t j = 0; j < M; ++j) {
      double z = S[(int64_t)i * M + j] / tau;
      if (z > mx) mx = z;
    }
    double sum = 0.0;
    for (int32_t j = 0; j < M; ++j) sum += exp(S[(int64_t)i * M + j] / tau - mx);
    double lse = mx + log(sum);
    total += lse - S[(int64_t)i * M + pos[i]] / tau;
  }
  return total / (double)B;
}

/* ---------------------------------------------------------------- NEXT N1: gradient of L_LI
 * Backward of L = mean_i [logsumexp_j(S_ij/tau) - S_{i,pos_i}/tau], S_ij = MaxSim(Q_i, D_j), through
 * the argmax of every max and through the row normalisation (chain rule; the paper gives no formula:
 * the ColTrast objective is trained by backpropagation; SPEC.md:357-365 grad_check):
 *   G_ij            = (softmax_j(S_i/tau)_j - [j == pos_i]) / (B * tau)
 *   a(i,t,j)        = argmax_{u < len_j} <qn_{i,t}, dn_{j,u}>        (lowest u on exact ties)
 *   dL/dqn_{i,t}    = sum_j G_ij dn_{j,a(i,t,j)}
 *   dL/ddn_{j,u}    = sum_i sum_{t : a(i,t,j) = u} G_ij qn_{i,t}
 *   dL/dx (row)     = (g - yn (yn . g)) / ||x||      with yn = x / ||x||
 * x_q: [B][q_stride][d] float64 raw query rows, x_d: [M][d_stride][d] raw doc rows (only real rows used).
 * exact_norm = 1: qn/dn = x/||x|| in float64 (differentiable: the finite-difference pin);
 * exact_norm = 0: qn/dn = the library's NORM (bf16 rounded; the GPU's operands) -- the argmax and the
 *                 dot products use those values, the Jacobian uses yn = x/||x|| in float64.
 * Outputs: loss (return value), grad_q/grad_d same shapes as x_q/x_d (padding rows 0),
 * amax_out (may be NULL): [B][M][q_stride] int32 argmax indices, gap_out (may be NULL): the gap
 * between the best and second-best dot for each (i, t, j) (near-ties decide argmax ambiguously),
 * amax2_out (may be NULL): the second-best index.
 */
static double o_dot(const double* a, const double* b, int32_t d) {
  double s = 0.0;
  for (int32_t k = 0; k < d; ++k) s += a[k] * b[k];
  return s;
}

static void o_prepare_rows(const double* x, int64_t n_items, int32_t stride, const int32_t* lens,
                           int32_t d, int32_t exact_norm, double* out) {
  for (int64_t i = 0; i < n_items; ++i)
    for (int32_t r = 0; r < stride; ++r) {
      const double* row = x + (i * stride + r) * d;
      double* o = out + (i * stride + r) * d;
      if (r >= lens[i]) {
        for (int32_t k = 0; k < d; ++k) o[k] = 0.0;
        continue;
      }
      if (exact_norm) {
        double n = sqrt(o_dot(row, row, d));
        for (int32_t k = 0; k < d; ++k) o[k] = row[k] / n;
      } else {
        float f[4096];
        uint16_t y[4096];
        for (int32_t k = 0; k < d; ++k) f[k] = (float)row[k];
        oracle_norm_rows(f, 0, 1, d, 0, y, NULL);
        for (int32_t k = 0; k < d; ++k) o[k] = (double)o_bf16_to_f32(y[k]);
      }
    }
}

double oracle_maxsim_infonce_grad(const double* x_q, const int32_t* q_lens, int32_t B, int32_t q_stride,
                                  const double* x_d, const int32_t* d_lens, int32_t M, int32_t d_stride,
                                  int32_t d, const int32_t* pos, double tau, int32_t exact_norm,
                                  double* grad_q, double* grad_d, int32_t* amax_out, double* gap_out,
                                  int32_t* amax2_out) {
  double* qn = (double*)malloc(sizeof(double) * (size_t)B * q_stride * d);
  double* dn = (double*)malloc(sizeof(double) * (size_t)M * d_stride * d);
  double* S = (double*)malloc(sizeof(double) * (size_t)B * M);
  int32_t* a = (int32_t*)calloc((size_t)B * M * q_stride, sizeof(int32_t));
  double* gq = (double*)calloc((size_t)B * q_stride * d, sizeof(double));
  double* gd = (double*)calloc((size_t)M * d_stride * d, sizeof(double));
  o_prepare_rows(x_q, B, q_stride, q_lens, d, exact_norm, qn);
  o_prepare_rows(x_d, M, d_stride, d_lens, d, exact_norm, dn);
  /* forward: S and the argmax of every max */
  for (int32_t i = 0; i < B; ++i)
    for (int32_t j = 0; j < M; ++j) {
      double s = 0.0;
      for (int32_t t = 0; t < q_lens[i]; ++t) {
        double best = -INFINITY, second = -INFINITY;
        int32_t arg = 0, arg2 = 0;
        for (int32_t u = 0; u < d_lens[j]; ++u) {
          double v = o_dot(qn + ((int64_t)i * q_stride + t) * d, dn + ((int64_t)j * d_stride + u) * d, d);
          if (v > best) { second = best; arg2 = arg; best = v; arg = u; }
          else if (v > second) { second = v; arg2 = u; }
        }
        if (amax2_out) amax2_out[((int64_t)i * M + j) * q_stride + t] = arg2;
        s += best;
        a[((int64_t)i * M + j) * q_stride + t] = arg;
        if (gap_out) gap_out[((int64_t)i * M + j) * q_stride + t] = best - second;
      }
      S[(int64_t)i * M + j] = s;
    }
  double loss = oracle_infonce(S, B, M, pos, tau);
  /* G = dL/dS */
  for (int32_t i = 0; i < B; ++i) {
    double mx = -INFINITY, sum = 0.0;
    for (int32_t j = 0; j < M; ++j) mx = fmax(mx, S[(int64_t)i * M + j] / tau);
    for (int32_t j = 0; j < M; ++j) sum += exp(S[(int64_t)i * M + j] / tau - mx);
    for (int32_t j = 0; j < M; ++j) {
      double G = (exp(S[(int64_t)i * M + j] / tau - mx) / sum - (j == pos[i] ? 1.0 : 0.0)) / (B * tau);
      for (int32_t t = 0; t < q_lens[i]; ++t) {
        int32_t u = a[((int64_t)i * M + j) * q_stride + t];
        double* g1 = gq + ((int64_t)i * q_stride + t) * d;
        double* g2 = gd + ((int64_t)j * d_stride + u) * d;
        const double* qv = qn + ((int64_t)i * q_stride + t) * d;
        const double* dv = dn + ((int64_t)j * d_stride + u) * d;
        for (int32_t k = 0; k < d; ++k) {
          g1[k] += G * dv[k];
          g2[k] += G * qv[k];
        }
      }
    }
  }
  /* through the normalisation: dx = (g - y (y.g)) / ||x|| */
  for (int pass = 0; pass < 2; ++pass) {
    const double* x = pass ? x_d : x_q;
    const int32_t* lens = pass ? d_lens : q_lens;
    int64_t n = pass ? M : B;
    int32_t stride = pass ? d_stride : q_stride;
    double* g = pass ? gd : gq;
    double* out = pass ? grad_d : grad_q;
    for (int64_t i = 0; i < n; ++i)
      for (int32_t r = 0; r < stride; ++r) {
        const double* row = x + (i * stride + r) * d;
        double* gr = g + (i * stride + r) * d;
        double* o = out + (i * stride + r) * d;
        if (r >= lens[i]) {
          for (int32_t k = 0; k < d; ++k) o[k] = 0.0;
          continue;
        }
        double nrm = sqrt(o_dot(row, row, d));
        double yg = 0.0;
        for (int32_t k = 0; k < d; ++k) yg += row[k] / nrm * gr[k];
        for (int32_t k = 0; k < d; ++k) o[k] = (gr[k] - row[k] / nrm * yg) / nrm;
      }
  }
  if (amax_out) memcpy(amax_out, a, sizeof(int32_t) * (size_t)B * M * q_stride);
  free(qn); free(dn); free(S); free(a); free(gq); free(gd);
  return loss;
}
