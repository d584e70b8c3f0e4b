/* CPU oracle for the KPM hot path -- TEST INFRASTRUCTURE ONLY (see header).
 *
 * Compiled with -ffp-contract=off so every multiply and add rounds separately,
 * as in the reference's compiled kernel (no FMA in _spmv*.so, SURVEY.md
 * Appendix A) and in numpy's einsum column reduction (kpm.py:108).
 */
#include "kpm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* graph.py:69-81: rows get both directions of every canonical pair (a loop
 * once), each row's columns sorted ascending (lexsort((cv, ru))), row_ptr
 * by counting + cumsum.  Duplicate pairs (raw generator output) collapse to
 * one entry, as np.unique does on the canonical keys before the build. */
int64_t orc_csr_from_edges(int64_t n, const int64_t *u, const int64_t *v,
                           int64_t m, int flags, int64_t *row_ptr,
                           int64_t *col_idx) {
  /* Counting scatter, then per-row sort + unique: the result (sorted unique
   * neighbours per row) does not depend on the scatter order, so the passes
   * run on OpenMP threads (atomic counters) and stay deterministic. */
  const int keep_loops = flags & 1;
  int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt) return -1;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(|| : bad)
  for (int64_t e = 0; e < m; ++e) {
    int64_t a = u[e], b = v[e];
    if (a < 0 || b < 0 || a >= n || b >= n) { bad = 1; continue; }
    if (a == b) {
      if (keep_loops) {
#pragma omp atomic
        cnt[a + 1]++;
      }
      continue;
    }
#pragma omp atomic
    cnt[a + 1]++;
#pragma omp atomic
    cnt[b + 1]++;
  }
  if (bad) { free(cnt); return -1; }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t *pos = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
  memcpy(pos, cnt, ((size_t)n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int64_t a = u[e], b = v[e], p;
    if (a == b) {
      if (keep_loops) {
#pragma omp atomic capture
        p = pos[a]++;
        col_idx[p] = a;
      }
      continue;
    }
#pragma omp atomic capture
    p = pos[a]++;
    col_idx[p] = b;
#pragma omp atomic capture
    p = pos[b]++;
    col_idx[p] = a;
  }
  free(pos);
  /* sort + unique per row; each thread compacts a contiguous block of rows
   * in place (row_ptr[i+1] holds the row's unique count for now), then the
   * blocks are moved left in order */
  int nt = 1;
#pragma omp parallel
  {
#pragma omp single
    nt = omp_get_num_threads();
  }
  int64_t *blk_lo = (int64_t *)malloc(sizeof(int64_t) * (nt + 1));
  int64_t *blk_w = (int64_t *)malloc(sizeof(int64_t) * (nt + 1));
  for (int t = 0; t <= nt; ++t) blk_lo[t] = n * t / nt;
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    int64_t w = cnt[blk_lo[t]];
    for (int64_t i = blk_lo[t]; i < blk_lo[t + 1]; ++i) {
      int64_t s = cnt[i], e = cnt[i + 1];
      qsort(col_idx + s, (size_t)(e - s), sizeof(int64_t), cmp_i64);
      const int64_t w0 = w;
      for (int64_t jj = s; jj < e; ++jj) {
        if (jj > s && col_idx[jj] == col_idx[jj - 1]) continue;
        col_idx[w++] = col_idx[jj];
      }
      row_ptr[i + 1] = w - w0;
    }
    blk_w[t] = w - cnt[blk_lo[t]];
  }
  int64_t w = 0;
  row_ptr[0] = 0;
  for (int t = 0; t < nt; ++t) {
    const int64_t src = cnt[blk_lo[t]];
    if (blk_w[t] && src != w)
      memmove(col_idx + w, col_idx + src, sizeof(int64_t) * (size_t)blk_w[t]);
    for (int64_t i = blk_lo[t]; i < blk_lo[t + 1]; ++i) row_ptr[i + 1] += row_ptr[i];
    w += blk_w[t];
  }
  free(blk_lo);
  free(blk_w);
  free(cnt);
  return w;
}

/* graph.py:47-54 (deg = sum of unit weights, a loop counted once) and
 * operators.py:108-109: dinv = 1/sqrt(max(deg,1e-300)) if deg > 0 else 0. */
void orc_dinv(int64_t n, const int64_t *row_ptr, double *dinv) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double deg = (double)(row_ptr[i + 1] - row_ptr[i]);
    dinv[i] = deg > 0 ? 1.0 / sqrt(deg) : 0.0;
  }
}

/* operators.py:110: norm_w = w * dinv[rows] * dinv[cols], w = 1.0. */
void orc_normadj_values(int64_t n, const int64_t *row_ptr,
                        const int64_t *col_idx, const double *dinv,
                        double *data) {
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t jj = row_ptr[i]; jj < row_ptr[i + 1]; ++jj)
      data[jj] = (1.0 * dinv[i]) * dinv[col_idx[jj]];
}

/* _spmv.pyx:11-22 _row and :25-39 csr_matvec. */
void orc_csr_matvec(int64_t n_rows, const int64_t *indptr,
                    const int64_t *indices, const double *data,
                    const double *x, int64_t k, double *out, int threads) {
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int64_t i = 0; i < n_rows; ++i) {
    double *o = out + i * k;
    for (int64_t c = 0; c < k; ++c) o[c] = 0.0;
    for (int64_t jj = indptr[i]; jj < indptr[i + 1]; ++jj) {
      const double w = data[jj];
      const double *xr = x + indices[jj] * k;
      for (int64_t c = 0; c < k; ++c) o[c] += w * xr[c];
    }
  }
}

/* operators.py:142-148 ScaledOperator.apply: y = A x; y -= shift*x;
 * y /= scale (each only when the parameter is not the identity). */
static void scaled_apply(int64_t n, const int64_t *indptr,
                         const int64_t *indices, const double *data,
                         double shift, double scale, const double *x,
                         int64_t k, double *y, int threads) {
  orc_csr_matvec(n, indptr, indices, data, x, k, y, threads);
  if (shift != 0.0) {
    for (int64_t e = 0; e < n * k; ++e) y[e] -= shift * x[e];
  }
  if (scale != 1.0) {
    for (int64_t e = 0; e < n * k; ++e) y[e] /= scale;
  }
}

typedef void (*collect_fn)(int m, const double *t, void *ctx);

/* kpm.py:73-89 _recurrence: T0 = copy(z); T1 = H T0; T_m = 2 H T_{m-1} -
 * T_{m-2} computed as (apply; *= 2.0; -= prev), three rotating buffers. */
static void recurrence(int64_t n, const int64_t *indptr,
                       const int64_t *indices, const double *data,
                       double shift, double scale, const double *z, int64_t k,
                       int m_max, collect_fn collect, void *ctx, int threads) {
  size_t sz = (size_t)n * (size_t)k;
  double *t_prev = (double *)malloc(sz * sizeof(double) + 8);
  double *t_cur = (double *)malloc(sz * sizeof(double) + 8);
  double *scratch = (double *)malloc(sz * sizeof(double) + 8);
  memcpy(t_prev, z, sz * sizeof(double));
  collect(0, t_prev, ctx);
  if (m_max > 0) {
    scaled_apply(n, indptr, indices, data, shift, scale, t_prev, k, t_cur,
                 threads);
    collect(1, t_cur, ctx);
    for (int m = 2; m <= m_max; ++m) {
      double *t_next = scratch;
      scaled_apply(n, indptr, indices, data, shift, scale, t_cur, k, t_next,
                   threads);
      for (size_t e = 0; e < sz; ++e) {
        t_next[e] *= 2.0;
        t_next[e] -= t_prev[e];
      }
      collect(m, t_next, ctx);
      scratch = t_prev;
      t_prev = t_cur;
      t_cur = t_next;
    }
  }
  free(t_prev);
  free(t_cur);
  free(scratch);
}

struct dos_ctx {
  const double *z;
  int64_t n, k;
  double *contrib;
};

/* kpm.py:107-108 contrib[m] = einsum('ij,ij->j', z, t_m): numpy walks rows in
 * order and accumulates each column with a separately rounded multiply and
 * add (checked bit-for-bit against numpy 2.3 by tests/test_oracle.py). */
static void dos_collect(int m, const double *t, void *vctx) {
  struct dos_ctx *c = (struct dos_ctx *)vctx;
  double *row = c->contrib + (int64_t)m * c->k;
  for (int64_t j = 0; j < c->k; ++j) row[j] = 0.0;
  for (int64_t i = 0; i < c->n; ++i) {
    const double *zr = c->z + i * c->k, *tr = t + i * c->k;
    for (int64_t j = 0; j < c->k; ++j) row[j] += zr[j] * tr[j];
  }
}

void orc_dos_contrib(int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *data, double shift, double scale,
                     const double *z, int64_t k, int m_max, double *contrib,
                     int threads) {
  struct dos_ctx c = {z, n, k, contrib};
  recurrence(n, indptr, indices, data, shift, scale, z, k, m_max, dos_collect,
             &c, threads);
}

struct ldos_ctx {
  const double *z;
  int64_t n, k;
  double *num;
};

/* kpm.py:135-136 num[m] = einsum('ij,ij->i', z, t_m).  numpy reduces a row
 * with SIMD partial sums; the oracle sums columns in order, so the two agree
 * to rounding (~1e-16 relative), not bitwise. */
static void ldos_collect(int m, const double *t, void *vctx) {
  struct ldos_ctx *c = (struct ldos_ctx *)vctx;
  double *row = c->num + (int64_t)m * c->n;
  for (int64_t i = 0; i < c->n; ++i) {
    const double *zr = c->z + i * c->k, *tr = t + i * c->k;
    double s = 0.0;
    for (int64_t j = 0; j < c->k; ++j) s += zr[j] * tr[j];
    row[i] = s;
  }
}

void orc_ldos_num(int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *data, double shift, double scale,
                  const double *z, int64_t k, int m_max, double *num,
                  int threads) {
  struct ldos_ctx c = {z, n, k, num};
  recurrence(n, indptr, indices, data, shift, scale, z, k, m_max,
             ldos_collect, &c, threads);
}

struct blk_ctx {
  int want;
  size_t sz;
  double *out;
};

static void blk_collect(int m, const double *t, void *vctx) {
  struct blk_ctx *c = (struct blk_ctx *)vctx;
  if (m == c->want) memcpy(c->out, t, c->sz * sizeof(double));
}

void orc_recurrence_block(int64_t n, const int64_t *indptr,
                          const int64_t *indices, const double *data,
                          double shift, double scale, const double *z,
                          int64_t k, int steps, double *t_out, int threads) {
  struct blk_ctx c = {steps, (size_t)n * (size_t)k, t_out};
  recurrence(n, indptr, indices, data, shift, scale, z, k, steps, blk_collect,
             &c, threads);
}

/* ---- R-MAT harness generator (Philox4x32-10, Salmon et al. SC'11) ---- */
static inline void philox4x32_10(uint32_t ctr[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)M0 * ctr[0];
    uint64_t p1 = (uint64_t)M1 * ctr[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ ctr[1] ^ k0, n2 = hi0 ^ ctr[3] ^ k1;
    ctr[0] = n0;
    ctr[1] = lo1;
    ctr[2] = n2;
    ctr[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

void orc_rmat_edges(int scale, uint64_t seed, uint32_t ta, uint32_t tab,
                    uint32_t tabc, int64_t e0, int64_t count, int64_t *u,
                    int64_t *v, int threads) {
  (void)threads;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int64_t t = 0; t < count; ++t) {
    uint64_t e = (uint64_t)(e0 + t);
    int64_t a = 0, b = 0;
    uint32_t w[4];
    for (int l = 0; l < scale; ++l) {
      if ((l & 3) == 0) {
        w[0] = (uint32_t)e;
        w[1] = (uint32_t)(e >> 32);
        w[2] = (uint32_t)(l >> 2);
        w[3] = 0u;
        philox4x32_10(w, k0, k1);
      }
      uint32_t r = w[l & 3];
      int bu = r >= tab;                  /* quadrants c, d: lower half */
      int bv = (r >= ta && r < tab) || r >= tabc; /* quadrants b, d */
      a = (a << 1) | bu;
      b = (b << 1) | bv;
    }
    u[t] = a;
    v[t] = b;
  }
}
