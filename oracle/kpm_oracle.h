/* CPU oracle for the KPM hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference (netdos 0.1.0) algorithm for the
 * Chebyshev-moment path, used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the CHECKER.  Nothing in the shipped
 * package (paper_1905_09758_b200/) may link, import or call it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/netdos/).  Parity is pinned by tests/test_oracle.py
 * against fixtures produced by the reference itself (tests/golden/).
 */
#ifndef KPM_ORACLE_H
#define KPM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* graph.py:69-81 _csr_from_canonical, preceded by the canonicalise / drop
 * self-loop / dedup step the harness applies to raw generator output
 * (graph.py:130-160 semantics for an unweighted edge list without loops).
 * Writes row_ptr[n+1]; returns nnz, or -1 on a bad id.  col_idx must hold
 * 2*m entries (upper bound).  flags: 1 = keep self-loops (stored once). */
int64_t orc_csr_from_edges(int64_t n, const int64_t *u, const int64_t *v,
                           int64_t m, int flags, int64_t *row_ptr,
                           int64_t *col_idx);

/* graph.py:47-54 degrees + operators.py:108-110 d^-1/2 (isolated -> 0). */
void orc_dinv(int64_t n, const int64_t *row_ptr, double *dinv);

/* operators.py:110 norm_w = (w*dinv[r])*dinv[c] with w = 1.0. */
void orc_normadj_values(int64_t n, const int64_t *row_ptr,
                        const int64_t *col_idx, const double *dinv,
                        double *data);

/* _kernels/_spmv.pyx:11-39 csr_matvec: out[i,c] = sum_jj data[jj]*x[j,c] in
 * stored order, separate multiply and add roundings, OpenMP static rows. */
void orc_csr_matvec(int64_t n_rows, const int64_t *indptr,
                    const int64_t *indices, const double *data,
                    const double *x, int64_t k, double *out, int threads);

/* kpm.py:73-117 dos_moments' recurrence + per-probe collect (einsum
 * 'ij,ij->j', kpm.py:108).  operators.py:142-148 ScaledOperator.apply
 * epilogue (shift, scale) applied with separate roundings.
 * contrib is (m_max+1) x k row-major. */
void orc_dos_contrib(int64_t n, const int64_t *indptr, const int64_t *indices,
                     const double *data, double shift, double scale,
                     const double *z, int64_t k, int m_max, double *contrib,
                     int threads);

/* kpm.py:120-152 pdos_moments' collect (einsum 'ij,ij->i', kpm.py:136):
 * num is (m_max+1) x n row-major. */
void orc_ldos_num(int64_t n, const int64_t *indptr, const int64_t *indices,
                  const double *data, double shift, double scale,
                  const double *z, int64_t k, int m_max, double *num,
                  int threads);

/* kpm.py:76-89: the T_m block after `steps` recurrence steps (T_0 = z).
 * Used for the bit-exact T_k comparison with the CUDA path. */
void orc_recurrence_block(int64_t n, const int64_t *indptr,
                          const int64_t *indices, const double *data,
                          double shift, double scale, const double *z,
                          int64_t k, int steps, double *t_out, int threads);

/* R-MAT harness generator (no reference counterpart: SURVEY.md §9.2).
 * Edge e, level l: uniform = Philox4x32-10(key=(seed_lo,seed_hi),
 * ctr=(e_lo,e_hi,l/4,0)).word[l%4]; quadrant by thresholds ta<tb<tc on the
 * uint32 uniform.  Writes edges [e0, e0+count). */
void orc_rmat_edges(int scale, uint64_t seed, uint32_t ta, uint32_t tab,
                    uint32_t tabc, int64_t e0, int64_t count, int64_t *u,
                    int64_t *v, int threads);

#ifdef __cplusplus
}
#endif
#endif
