/* libkpm -- B200-native KPM Chebyshev-moment engine: the C-ABI drop-in
 * boundary for the hot path of netdos 0.1.0 (arXiv 1905.09758).
 *
 * Plain C types only (no torch, no CUDA types in signatures).  One context
 * drives one GPU; multi-GPU runs use one process per GPU (probe sharding,
 * SURVEY.md §8e) and combine per-probe results on the host side.
 *
 * Pointer arguments documented "host-or-device" are classified with
 * cudaPointerGetAttributes: device pointers are used in place (no copy),
 * host pointers are staged through the context's stream.
 *
 * Every entry point returns KPM_OK (0) or a negative KPM_E* status; the
 * message is available from kpm_last_error() (thread-local).  Python maps
 * KPM_EINVAL -> ValueError, KPM_ENONFINITE -> RecurrenceBlowupError,
 * KPM_EZEROMASS -> ValueError("zero probe mass at node k...") (the
 * reference's exception types and messages, errors.py:1-33, kpm.py:111-147).
 *
 * Citations: paths relative to /root/reference/pkg/src/netdos/.
 */
#ifndef LIBKPM_H
#define LIBKPM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KPM_ABI_VERSION 1

enum {
  KPM_OK = 0,
  KPM_EINVAL = -1,      /* bad argument                                   */
  KPM_ENONFINITE = -2,  /* recurrence overflowed (kpm.py:111-114)          */
  KPM_ENOMEM = -3,      /* device allocation failed                        */
  KPM_ECUDA = -4,       /* CUDA runtime error                              */
  KPM_EZEROMASS = -5,   /* zero probe mass at a node (kpm.py:145-147)      */
  KPM_ENODEV = -6       /* no usable sm_100 device                         */
};

/* recurrence modes (kpm_run_create) */
enum {
  KPM_MODE_DOS_DOUBLING = 0, /* global moments, ceil(M/2) steps, T_2k = 2T_k^2-I */
  KPM_MODE_DOS_DIRECT = 1,   /* global moments, M steps, z^T T_m z (kpm.py:108) */
  KPM_MODE_LDOS = 2          /* per-node moments, M steps (kpm.py:136)        */
};

/* flags for kpm_run_create */
enum {
  KPM_LDOS_RAW = 1 /* pdos normalized=False: num * trace_scale (kpm.py:150) */
};

typedef struct kpm_ctx kpm_ctx;
typedef struct kpm_graph kpm_graph;
typedef struct kpm_run kpm_run;

/* ------------------------------------------------------------ context --- */
int kpm_abi_version(void);
const char *kpm_last_error(void);
int kpm_device_count(int *count);
/* Bind a context (and its own non-blocking stream) to CUDA device `device`. */
int kpm_init(int device, kpm_ctx **out);
void kpm_finalize(kpm_ctx *ctx);
/* The context's cudaStream_t, for event timing by the caller. */
void *kpm_ctx_stream(kpm_ctx *ctx);
int kpm_ctx_synchronize(kpm_ctx *ctx);
/* device memory owned by the caller through the library */
int kpm_device_alloc(kpm_ctx *ctx, int64_t bytes, void **out);
int kpm_device_free(kpm_ctx *ctx, void *ptr);
/* stream-ordered copy; kind 0 = H2D, 1 = D2H, 2 = D2D; host buffers should
 * be pinned (kpm_host_alloc) for async transfers. */
int kpm_memcpy(kpm_ctx *ctx, void *dst, const void *src, int64_t bytes, int kind);
int kpm_host_alloc(int64_t bytes, void **out);
/* free / total device memory of the context's GPU (probe batch sizing) */
int kpm_mem_info(kpm_ctx *ctx, int64_t *free_bytes, int64_t *total_bytes);
int kpm_host_free(void *ptr);
/* Touch every page of a caller-owned (pageable) host result buffer with
 * `threads` host threads (<= 0: up to 16), after advising transparent huge
 * pages, so a following D2H copy does not pay the first-touch page faults on
 * one thread.  The buffer's contents are overwritten.  Host-only; meant to
 * run while queued kernels execute (C2: 808 MB of per-node moments). */
int kpm_host_prefault(void *ptr, int64_t bytes, int threads);

/* ------------------------------------------------------------- graphs --- */
/* Device graph loader (K1-K3).  Replaces graph.py:69-81 _csr_from_canonical
 * (+ the canonicalise/self-loop/dedup step of build_csr, graph.py:130-160)
 * followed by graph.py:47-54 degrees and the normalized-adjacency branch of
 * build_operator, operators.py:105-113.  Input: m edges (u[e], v[e]),
 * int64, host-or-device.  Self-loops are dropped unless keep_loops != 0 (then
 * stored once at (i,i)); duplicates are merged (unit weights).  Output: int64
 * row_ptr, int32 col_idx sorted per row, fp64 dinv = deg>0 ? 1/sqrt(deg) : 0
 * bit-identical to the reference; H's values are never stored. */
int kpm_graph_from_edges(kpm_ctx *ctx, int64_t n, const int64_t *u,
                         const int64_t *v, int64_t m, int keep_loops,
                         kpm_graph **out);

/* Explicit CSR (any operator kind): replaces SymmetricCSROperator
 * (operators.py:50-65) wrapped by rescale_operator / ScaledOperator.apply
 * (operators.py:124-176): y = (A x - shift*x) / scale with separate
 * roundings.  values == NULL selects the implicit normalized adjacency
 * h_ij = dinv_i*dinv_j computed from the degree of each row (the
 * reference's kind="normalized-adjacency" operator), in which case shift and
 * scale must be 0 and 1.  indptr/indices int64, host-or-device. */
int kpm_graph_from_csr(kpm_ctx *ctx, int64_t n, const int64_t *indptr,
                       const int64_t *indices, int64_t nnz,
                       const double *values, double shift, double scale,
                       kpm_graph **out);

/* Copy a graph to another context (another GPU over NVLink/NVSwitch peer
 * copies, or a second context on the same GPU): probe columns / LDOS shards
 * of one dos_moments / pdos_moments call then run on every GPU of the process
 * (the reference's `threads` knob, kpm.py:92-93, mapped to devices). */
int kpm_graph_replicate(kpm_graph *src, kpm_ctx *ctx, kpm_graph **out);

/* Same with int32 column indices (the device layout: no widening copy; a
 * host CSR of 2e9 nonzeros is 8 GB instead of 16 GB). */
int kpm_graph_from_csr32(kpm_ctx *ctx, int64_t n, const int64_t *indptr,
                         const int32_t *indices, int64_t nnz, const double *values,
                         double shift, double scale, kpm_graph **out);

int kpm_graph_info(kpm_graph *g, int64_t *n, int64_t *nnz, int64_t *max_degree);
/* Build, ahead of the first run, whatever a run of k probe columns on this
 * graph needs beside its own buffers -- for large implicit graphs the
 * gather-ordered twin of the CSR (vertices renumbered by degree, each row's
 * neighbours hottest-first; see kpm_run_create) -- so that a caller sizing
 * probe batches from free memory sees it.  *twin = 1 when such runs step on
 * the twin (their row sums then follow the twin's neighbour order, not the
 * reference's; KPM_REORDER=0 disables, =1 forces). */
int kpm_graph_prepare(kpm_graph *g, int64_t k, int32_t *twin);
/* Copy the device CSR back (any pointer may be NULL): bit-exactness checks. */
int kpm_graph_export(kpm_graph *g, int64_t *row_ptr, int32_t *col_idx,
                     double *dinv);
void kpm_graph_free(kpm_graph *g);

/* ---------------------------------------------------- native SpMM (L0) --- */
/* Drop-in for the reference's only FFI, _kernels/_spmv.pyx:25-39
 * csr_matvec(indptr, indices, data, x, out, threads): out[i,c] =
 * sum_jj data[jj]*x[indices[jj],c] in stored order, separate multiply/add
 * roundings (bit-identical to the Cython kernel).  x is n_x_rows x k
 * row-major, out is n_rows x k row-major; all host-or-device. */
int kpm_csr_matvec(kpm_ctx *ctx, int64_t n_rows, const int64_t *indptr,
                   const int64_t *indices, const double *data, int64_t nnz,
                   const double *x, int64_t n_x_rows, int64_t k, double *out);

/* ----------------------------------------------------------- probes --- */
/* make_probes(kind=RADEMACHER) on the device (probes.py:52-54,86-89):
 * column j = 1 - 2*bit, the bit stream of numpy's Philox4x64-10 seeded by
 * SeedSequence(seed).spawn(nz)[j] -- the host passes each column's 128-bit
 * Philox key (keys[2j], keys[2j+1]); output is bit-identical to numpy.
 * z (device) is n x ldz row-major; columns [col0, col0+ncols). */
int kpm_probes_rademacher(kpm_ctx *ctx, int64_t n, int64_t ncols,
                          const uint64_t *keys, double *z, int64_t ldz,
                          int64_t col0);

/* -------------------------------------------------- motif projection --- */
/* The probe-deflation loop of filter_probes (motifs.py:400-403): for each
 * sparse vector u (vec_ptr/vec_idx/vec_val, CSR over vectors) in order,
 * coeff = u . Z[idx,:]; Z[idx,:] -= outer(u, coeff).  Vectors are grouped
 * (group_ptr over vectors) so that groups have pairwise disjoint support and
 * run in parallel; vectors within a group run in list order.  z is n x ldz
 * (host-or-device, updated in place), k columns. */
int kpm_filter_probes(kpm_ctx *ctx, int64_t n, int64_t k, double *z,
                      int64_t ldz, int64_t n_groups, const int64_t *group_ptr,
                      const int64_t *vec_ptr, const int64_t *vec_idx,
                      const double *vec_val);

/* --------------------------------------------------------- recurrence --- */
/* A moment run over one probe batch: dos_moments (kpm.py:92-117) or
 * pdos_moments (kpm.py:120-152).  The run owns two n x ld fp64 recurrence
 * blocks (three for DIRECT/LDOS: the probes stay resident).
 * Neighbour order: a row's sum adds its neighbours in the CSR's stored order
 * (_spmv.pyx:11-39), so T_k is bit-identical to the reference -- except for
 * large implicit graphs (one gathered column tile of T_k >= 32x the L2), which
 * step on the gather-ordered twin (kpm_graph_prepare): another fixed order,
 * same tolerances on every result, rows of every input/output still in the
 * caller's numbering.  Environment KPM_REORDER=0 always keeps the CSR's order,
 * =1 forces the twin where one can be built. */
int kpm_run_create(kpm_graph *g, int64_t k, int32_t mode, int32_t m_max,
                   int32_t flags, kpm_run **out);
/* probes: n x k row-major with row stride ldz (host-or-device) */
int kpm_run_set_probes(kpm_run *r, const double *z, int64_t ldz);
/* device-generated Rademacher probes (see kpm_probes_rademacher) */
int kpm_run_set_rademacher(kpm_run *r, const uint64_t *keys);
/* Advance by up to `steps` SpMM recurrence steps (asynchronous on the
 * context stream); *remaining receives the steps still to go (may be NULL).
 * Each step is one fused kernel (SpMM + three-term update + moment
 * reduction) plus one deterministic finalize kernel. */
int kpm_run_advance(kpm_run *r, int32_t steps, int32_t *remaining);
int kpm_run_total_steps(kpm_run *r);
/* Kernel timing for the roofline: when enabled, kpm_run_advance brackets
 * every fused step kernel with CUDA events on the context stream;
 * kpm_run_kernel_time synchronises and returns the summed milliseconds and
 * the launch count since the last reset. */
int kpm_run_set_timing(kpm_run *r, int enable);
int kpm_run_kernel_time(kpm_run *r, double *ms, int32_t *launches);
/* Global modes: contrib (m_max+1) x k, contrib[m][j] = z_j^T T_m z_j
 * (kpm.py:107-108).  LDOS: values n x (m_max+1) = (num/den).T (kpm.py:148),
 * or num*trace_scale with KPM_LDOS_RAW.  `out` host-or-device.  Returns
 * KPM_ENONFINITE if any moment overflowed, KPM_EZEROMASS (node index in
 * *bad_node, may be NULL) for a zero probe mass in normalized LDOS. */
int kpm_run_result(kpm_run *r, double *out, double trace_scale,
                   int64_t *bad_node);
/* LDOS runs: out may be NULL -- the values are finished in place and stay in
 * the run's own n x (m_max+1) device buffer, returned by kpm_run_ldos_values
 * (valid until kpm_run_free), e.g. for kpm_ldos_histogram without a copy. */
int kpm_run_ldos_values(kpm_run *r, const double **values);
/* LDOS probe batches / GPU shards: dst's raw per-node sums and probe masses
 * += src's (src may live on another GPU: peer copy).  Both runs must have run
 * all their steps and not yet been finished by kpm_run_result; the zero-mass
 * check and the normalisation then apply to the combined sums. */
int kpm_run_accumulate(kpm_run *dst, kpm_run *src);
/* Free the recurrence blocks of a completed run, keeping its results (the
 * (m_max+1) x k contributions or the n x (m_max+1) LDOS sums). */
int kpm_run_trim(kpm_run *r);
/* Device pointer of the current T_k block and its row stride (tests); for a
 * run on the twin a copy in the caller's row order (valid until the next call). */
int kpm_run_block(kpm_run *r, const double **t_k, int64_t *ld, int32_t *k_index);
void kpm_run_free(kpm_run *r);

/* One-shot conveniences over kpm_run_*: z host-or-device n x k (ldz = k). */
int kpm_dos_contrib(kpm_graph *g, const double *z, int64_t k, int32_t m_max,
                    int32_t doubling, double *contrib);
int kpm_ldos(kpm_graph *g, const double *z, int64_t k, int32_t m_max,
             int32_t flags, double trace_scale, double *values,
             int64_t *bad_node);

/* ------------------------------------------------------ motif scan --- */
/* Device motif detection (motifs.py:189-311 semantics, unit weights): for
 * every row two 64-bit label sums over N(i) (open twins) and N(i)+{i}
 * (closed twins) are radix-sorted with the row ids; each sorted position is
 * verified exactly against its run head.  Host outputs, n entries each:
 * *_rows sorted rows, *_head position of the run head, *_ok 1 = equal to the
 * head (0 for excluded rows: self-loops; closed: isolated); chain_hub[x] /
 * chain_mid[x]: hub and middle node of the pendant path x - b - hub, or -1. */
int kpm_motif_scan(kpm_graph *g, int64_t *open_rows, int8_t *open_ok,
                   int64_t *open_head, int64_t *closed_rows, int8_t *closed_ok,
                   int64_t *closed_head, int64_t *chain_hub, int64_t *chain_mid);

/* ------------------------------------------------ row partitions (§8e) --- */
/* Graphs too large to replicate: rank q of R holds rows [part_lo[q],
 * part_lo[q+1]) of the CSR (column ids stay global) and the matching row
 * block of every recurrence vector.  Gathers of rows owned by another rank
 * read the owner's block directly -- peer memory over NVLink/NVSwitch
 * (CUDA IPC handles, kpm_ipc_*) or, for R partitions on one device, plain
 * device memory -- so there is no separate halo copy: the "halo exchange" is
 * the fused kernel's own peer loads.  Ranks must synchronise between steps. */
int kpm_graph_from_csr_part(kpm_ctx *ctx, int64_t n_global, int64_t row_lo,
                            int64_t n_local, const int64_t *indptr,
                            const int64_t *indices, int64_t nnz,
                            const double *values, double shift, double scale,
                            kpm_graph **out);
/* R-MAT rows [row_lo, row_hi) of the full draw stream (kpm_graph_rmat). */
int kpm_graph_rmat_part(kpm_ctx *ctx, int scale, int64_t n_edges, uint64_t seed,
                        uint32_t ta, uint32_t tab, uint32_t tabc, int64_t row_lo,
                        int64_t row_hi, kpm_graph **out);
int kpm_graph_part_info(kpm_graph *g, int64_t *row0, int64_t *n_global);
/* install d^-1/2 of ALL n_global rows (each rank computes its own rows'
 * part from its degrees, kpm_graph_export; ranks all-gather them) */
int kpm_graph_set_dinv(kpm_graph *g, const double *dinv_global);
/* the run's own a/b recurrence blocks (for kpm_ipc_get_handle / peers) */
int kpm_run_blocks(kpm_run *r, void **a, void **b);
/* part_lo[nparts+1] global row bounds; peer_a/peer_b[q] = partition q's
 * blocks as addressable from this device.  Global-moment results become raw
 * per-partition sums (summed across ranks, then the doubling transform, on
 * the host); LDOS rows are each rank's own. */
int kpm_run_set_partition(kpm_run *r, int nparts, const int64_t *part_lo, int me,
                          const void *const *peer_a, const void *const *peer_b);
/* CUDA IPC: 64-byte handle of a device allocation / open a peer's handle */
int kpm_ipc_get_handle(const void *dptr, void *handle);
int kpm_ipc_open_handle(kpm_ctx *ctx, const void *handle, void **dptr);
int kpm_ipc_close(void *dptr);

/* ------------------------------------------------- harness generators --- */
/* R-MAT edge draws [e0, e0+count) on the device (no reference counterpart,
 * SURVEY.md §9.2): Philox4x32-10(key=seed, ctr=(e, level/4)), quadrant by
 * uint32 thresholds ta < tab < tabc; u, v int64 device buffers.  Bit-
 * identical to oracle/kpm_oracle.c orc_rmat_edges. */
int kpm_rmat_edges(kpm_ctx *ctx, int scale, uint64_t seed, uint32_t ta,
                   uint32_t tab, uint32_t tabc, int64_t e0, int64_t count,
                   int64_t *u, int64_t *v);
/* Host-side (no GPU): the reference's preferential_attachment(n, m, seed)
 * (testkit.py:175-198) draw-for-draw.  pcg = numpy PCG64 state of
 * default_rng(seed): {state_hi, state_lo, inc_hi, inc_lo, has_uint32,
 * uinteger}.  u/v receive the m(m+1)/2 + (n-m-1)m canonical edges in the
 * reference's order. */
int kpm_gen_preferential_attachment(int64_t n, int64_t m, const uint64_t *pcg,
                                    int64_t *u, int64_t *v);
/* Fused R-MAT -> graph: draws n_edges edges as above and feeds them straight
 * into the device loader (== kpm_rmat_edges + kpm_graph_from_edges with
 * keep_loops = 0, without materialising u/v). */
int kpm_graph_rmat(kpm_ctx *ctx, int scale, int64_t n_edges, uint64_t seed,
                   uint32_t ta, uint32_t tab, uint32_t tabc, kpm_graph **out);

/* --------------------------------------------- graph file ingest (§8f) --- */
/* Replaces the line loops of _parse_edgelist / _parse_matrix_market
 * (fileio.py:28-47, :76-95) and the id compaction of parse_graph_file
 * (fileio.py:121-126).  The text (host or device pointer) is tokenised on the
 * device, one thread per line: blank lines and lines starting with '%' (and
 * '#' when KPM_PARSE_HASH_COMMENTS) are skipped; 2 or 3 whitespace-separated
 * tokens; the first two are integers, stored minus `base`.
 * Outputs are device arrays of n_lines entries (free with kpm_device_free):
 * u, v and status (0 skipped, 2/3 token count, -1 malformed, -2 the host
 * parser must decide: over-long or '_' integer tokens).  *unusual != 0 when
 * the text holds bytes the device tokenizer does not model (non-ASCII,
 * 0x1c-0x1f, NUL/DEL, bare '\r'); the caller then parses on the host. */
#define KPM_PARSE_HASH_COMMENTS 1
int kpm_parse_edges(kpm_ctx *ctx, const char *text, int64_t len, int64_t base,
                    int flags, int64_t *n_lines, int64_t **u, int64_t **v,
                    int8_t **status, int32_t *unusual);
/* Compacts the kept lines (status 2/3) of kpm_parse_edges into m edges
 * (device eu, ev; free with kpm_device_free).  compact_ids != 0: ids are
 * mapped onto 0..n-1 by rank among the sorted unique ids, returned in
 * *ids (device, n entries) -- np.unique + lookup, fileio.py:122-125;
 * otherwise n = n_declared and *ids = NULL.  info[5]: [0] bit 0: some line
 * had a weight token, bit 1: some line has status -2, [1] self-loop present, [2] a same-direction repeated edge
 * (build_csr would sum weights), [3] first line (0-based) with status -1 or
 * INT32_MAX, [4] an id outside [0, n). */
int kpm_edges_finalize(kpm_ctx *ctx, int64_t n_lines, int64_t *u, int64_t *v,
                       const int8_t *status, int compact_ids, int64_t n_declared,
                       int64_t *m, int64_t *n, int64_t **eu, int64_t **ev,
                       int64_t **ids, int32_t *info);

/* ------------------------------------------ per-node histograms (§8f) --- */
/* histogram_from_moments for per-node moments (density.py:63-108, the
 * `coef @ table` product): masses[i][b] = sum_m (values[i][m]*damping[m]) *
 * table[m][b]; norm[i] = values[i][0]*damping[0] (NULL damping = 1).
 * values n x ld (ld >= m_max+1, e.g. the LDOS result left in HBM by
 * kpm_run_result), table (m_max+1) x bins (cheb_bin_masses), masses n x bins:
 * all host-or-device; norm (n) may be NULL.  *min_mass = min over all masses
 * (NaN if any is NaN, as ndarray.min) for the negativity check. */
int kpm_ldos_histogram(kpm_ctx *ctx, const double *values, int64_t n, int64_t ld,
                       int32_t m_max, const double *damping, const double *table,
                       int32_t bins, double *masses, double *norm, double *min_mass);

/* ------------------------------------------------ Lanczos (§8f row 4) --- */
/* lanczos_factorize (lanczos.py:46-91) for k start vectors at once on the
 * operator of g (explicit values or the implicit normalized adjacency, with
 * its shift/scale: ScaledOperator.apply semantics).  z: n x ldz row-major
 * (host-or-device), column c the start vector; z_norm[c] = ||z_c|| computed
 * by the caller (q_0 = z / z_norm, as the reference).  Runs min(steps, n)
 * iterations with two classical Gram-Schmidt passes against the whole basis.
 * Host outputs: alphas k x S, betas k x (S-1) (S = min(steps, n)),
 * taken[c] = iterations run, exhausted[c] = 1 on a vanishing residual
 * (beta <= 1e-12 max(hnorm, 1e-300)), status[c] = 0 ok, 1 non-finite alpha,
 * 2 non-finite residual (taken[c] is then the reference's `iterations`).
 * basis (optional, host-or-device): k x S x n, vector-major. */
int kpm_lanczos(kpm_graph *g, const double *z, int64_t ldz, int64_t k, int32_t steps,
                const double *z_norm, double *alphas, double *betas, int32_t *taken,
                int32_t *exhausted, int32_t *status, double *basis);

#ifdef __cplusplus
}
#endif
#endif
