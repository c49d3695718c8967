/* attn_oracle.c -- plain fp64 masked softmax attention.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this.  It shares no code with the CUDA path.
 *
 * What it computes (section 2.1; section 2.4):
 *   for q-head h (kv head g = h / (Hq/Hkv), reading R13) and row i:
 *     J_i = { j <= i }                                              dense layer
 *     J_i = { j <= i : j < si  or  i-j < sl  or  i >= N-last }       triangle layer
 *           (= M - M^middle with the 0-based reading R1)
 *     s_ij = scale * sum_c q[h,i,c] k[g,j,c]          (fp64 from bf16-decoded inputs)
 *     m_i  = max_{j in J_i} s_ij,  l_i = sum_{j in J_i} exp(s_ij - m_i)
 *     o[h,i,:] = sum_{j in J_i} exp(s_ij - m_i) v[g,j,:] / l_i,  lse = m_i + ln l_i
 * Two passes per row (max, then exp-sum and weighted V), the literal predicate
 * evaluated for every (i, j), no blocking.  Masked entries are never formed
 * (c = +inf, reading R3).  OpenMP over (head, row).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

static int admitted(int64_t i, int64_t j, int64_t n, int64_t si, int64_t sl, int64_t last,
                    int dense) {
  if (j > i) return 0;                      /* causal: i >= j                     */
  if (dense) return 1;                      /* layer < tri_start: M  */
  int middle = (i < n - last) && (j >= si) && (i - j >= sl); /* M^middle P:L163-172 */
  return !middle;                           /* M - M^middle          */
}

/* q: [hq][n][d], k,v: [hkv][n][d] as bf16 bit patterns, contiguous.
 * rows: nrows row indices (NULL = all n rows).  out_o: [hq][nrows][d], out_lse: [hq][nrows]
 * (either may be NULL).  Returns the number of threads used, or -1 on bad arguments. */
int oracle_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t n,
                     int hq, int hkv, int d, int64_t si, int64_t sl, int64_t last, int dense,
                     double scale, const int64_t *rows, int64_t nrows, double *out_o,
                     double *out_lse, int threads) {
  if (!q || !k || !v || n < 1 || hq < 1 || hkv < 1 || hq % hkv || d < 1) return -1;
  if (!rows) nrows = n;
  int g = hq / hkv;
  int used = 1;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
  used = omp_get_max_threads();
#endif
  int64_t total = (int64_t)hq * nrows;
#pragma omp parallel
  {
    double *qd = (double *)malloc(sizeof(double) * d);
    double *acc = (double *)malloc(sizeof(double) * d);
    double *srow = (double *)malloc(sizeof(double) * n);
#pragma omp for schedule(dynamic, 16)
    for (int64_t t = 0; t < total; ++t) {
      int h = (int)(t / nrows);
      int64_t ri = t % nrows;
      int64_t i = rows ? rows[ri] : ri;
      int kvh = h / g;
      const uint16_t *qr = q + ((int64_t)h * n + i) * d;
      for (int c = 0; c < d; ++c) qd[c] = bf16_to_double(qr[c]);
      /* pass 1: scores and max */
      double m = -INFINITY;
      for (int64_t j = 0; j <= i; ++j) {
        if (!admitted(i, j, n, si, sl, last, dense)) continue;
        const uint16_t *kr = k + ((int64_t)kvh * n + j) * d;
        double s = 0.0;
        for (int c = 0; c < d; ++c) s += qd[c] * bf16_to_double(kr[c]);
        s *= scale;
        srow[j] = s;
        if (s > m) m = s;
      }
      /* pass 2: exp-sum and weighted V */
      double l = 0.0;
      for (int c = 0; c < d; ++c) acc[c] = 0.0;
      for (int64_t j = 0; j <= i; ++j) {
        if (!admitted(i, j, n, si, sl, last, dense)) continue;
        double p = exp(srow[j] - m);
        l += p;
        const uint16_t *vr = v + ((int64_t)kvh * n + j) * d;
        for (int c = 0; c < d; ++c) acc[c] += p * bf16_to_double(vr[c]);
      }
      if (out_o) {
        double *o = out_o + ((int64_t)h * nrows + ri) * d;
        for (int c = 0; c < d; ++c) o[c] = acc[c] / l;
      }
      if (out_lse) out_lse[(int64_t)h * nrows + ri] = m + log(l);
    }
    free(qd);
    free(acc);
    free(srow);
  }
  return used;
}

/* Number of admitted (i, j) pairs per head, by enumerating the predicate. */
int64_t oracle_pair_count(int64_t n, int64_t si, int64_t sl, int64_t last, int dense) {
  int64_t tot = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j <= i; ++j) tot += admitted(i, j, n, si, sl, last, dense);
  return tot;
}
