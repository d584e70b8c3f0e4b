// The fused KPM recurrence step and the run API.
//
// One launch per recurrence step computes, for every row i and probe column c,
//     acc      = sum_{jj in row i, stored order} h_ij * X[j, c]
//     T_{k+1}  = 2*acc - T_{k-1}            (T_1 = acc)
// with h_ij = dinv_i * dinv_j formed on the fly (H is never stored), every
// multiply and add separately rounded (__dmul_rn/__dadd_rn, no FMA), i.e.
// exactly the arithmetic of the reference's _spmv.pyx:11-22 _row followed by
// kpm.py:86-87 (`t_next *= 2.0; t_next -= t_prev`).  The T blocks are
// therefore BIT-IDENTICAL to the reference's _recurrence (kpm.py:73-89).
// In the same pass the kernel reduces the moment contributions:
//   DOUBLING  per probe <T_{k+1},T_k> and <T_{k+1},T_{k+1}>, giving
//             mu_{2k+1} = 2<T_{k+1},T_k> - mu_1 and mu_{2k+2} = 2<T_{k+1},T_{k+1}> - mu_0
//             (T_{2k} = 2 T_k^2 - I), ceil(M/2) steps for M moments;
//   DIRECT    per probe z^T T_{k+1} (kpm.py:107-108 einsum 'ij,ij->j');
//   LDOS      per node sum_c z_ic T_{k+1,ic} (kpm.py:135-136 'ij,ij->i'),
//             written straight into the (n, M+1) result as num/den.
// Global sums are deterministic: rows are grouped into load-balanced chunks
// that depend only on the graph (kpm_graph.cu), each warp of a CTA owns a
// fixed row subsequence, warps combine in fixed order into one partial per
// chunk, and a finalize kernel sums chunks in fixed order.
//
// Layout: X/T blocks are n x ld fp64 row-major (the reference's C-contiguous
// n x nz probe block, rows padded to ld = multiple of the lane vector width);
// one warp owns one row, lane l owns columns [l*C, l*C+C) of each 32*C-wide
// column tile, so every gathered neighbour row is one coalesced 8*ld-byte
// read; neighbour ids / weights are loaded 32 at a time by the lanes and
// broadcast with shuffles, and U gathers are kept in flight per warp.
#include <cmath>
#include <cstdlib>

#include "kpm_internal.cuh"

namespace kpm {

enum { MODE_DBL = 0, MODE_DIRECT = 1, MODE_LDOS = 2 };
constexpr int kMaxParts = KPM_MAX_PARTS;

struct StepParams {
  const int64_t *row_ptr;
  const int32_t *col;
  const double *dinv;
  const double *vals;      // explicit operator values (or nullptr)
  double shift, scale;     // explicit epilogue
  const double *X;         // T_k, gather source (read-only in this launch)
  const double *Xprev;     // T_{k-1} own rows (may alias Y)
  double *Y;               // T_{k+1}
  const double *Z;         // probes (DIRECT / LDOS)
  const double *den;       // LDOS normaliser
  double *ldos;            // LDOS result, n x (M+1)
  int ldos_col;            // moment index written this step
  int ldos_stride;         // M+1
  int ldos_raw;            // KPM_LDOS_RAW
  int64_t ld;
  const int32_t *chunk_start;
  const int32_t *chunk_order;
  double *partial;         // n_chunks x 2 x ld
  int32_t *flag;
  // heavy (hub) rows: column-sliced tasks at the head of the work queue
  const int32_t *heavy_rows;
  int32_t n_heavy;
  int64_t n_heavy_tasks;
  int64_t heavy_threshold;
  int32_t n_chunks;
  unsigned long long *queue;  // work-queue counter (zeroed before each launch)
  int stream;              // stream light chunks (single tile) across rows
  // row partitions (kMaxParts): this launch works local rows of partition
  // `me`; a gathered row j lives in the block of its owner (peer memory on
  // another GPU, or another block on this one) -- see kpm_run_set_partition
  int nparts;
  int64_t row0;            // global id of local row 0 (dinv is global)
  int64_t part_lo[kMaxParts + 1];
  const double *xparts[kMaxParts];
  int raw;                 // finalize writes raw sums (partitions combine on host)
  double *hpart;           // n_heavy x 2 x ld (global modes)
  double hot_dinv;         // gathered rows with dinv_j <= hot_dinv are "hot" (L2 policy)
  int bulk;                // TMA bulk-copy gathers (light_bulk): 0 off, 1 C=4, 2 all
  double *hldos;           // n_heavy x n_slices (LDOS)
  int64_t col0, tw;        // column tile of this launch: [col0, col0 + tw) (default 0, ld)
  int tile;                // run the 4-column layout as 64-column gather4 tiles
  int g4;                  // TMA gather4 light path: 0 off, 1 for C <= 2, 2 all layouts
  int lean;                // per-lane async gathers for C <= 2 (light_lean)
  int ntiles;              // gather4: light items per chunk = 64-column tiles of one launch
  int fuse_tiles;          // run all 64-column tiles of a step as one launch
  int hot_rows;            // gather-ordered twin: gathered ids < hot_rows are hot (L2 policy)
  const int32_t *perm;     // gather-ordered twin: perm[row] = the caller's row id (else NULL)
  // gather-ordered twin: d^-1/2 of ids >= dstep_h from the degree-step table
  // (kpm_graph::dstep_id / dstep_val, staged in shared memory) instead of an
  // 8-byte gather per nonzero; dstep_h = INT32_MAX: no table
  const int32_t *dstep_id;
  const double *dstep_val;
  int dstep_h;
  int64_t hub_off;         // dynamic smem (doubles) of warp 0's hub ring (kpm_step_kernel)
  unsigned long long *trace;  // KPM_TRACE: per work item (start ns, end ns, smid<<32|warp)
};

// row id in the caller's numbering (per-node outputs of a run on the twin)
__device__ __forceinline__ size_t out_row(const StepParams &p, int64_t row) {
  return p.perm ? (size_t)p.perm[row] : (size_t)row;
}

// KPM_TRACE diagnostics: one record per work item of one traced launch
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_item(const StepParams &p, unsigned long long item,
                                           unsigned long long t0) {
  if (p.trace && (threadIdx.x & 31) == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    p.trace[3 * item] = t0;
    p.trace[3 * item + 1] = gtimer();
    p.trace[3 * item + 2] = ((unsigned long long)smid << 32) | (threadIdx.x >> 5);
  }
}

// Address of gathered row j (global id) in the current T_k block.
__device__ __forceinline__ const double *gather_row(const StepParams &p, uint32_t j) {
  if (p.nparts <= 1) return p.X + (size_t)j * (uint32_t)p.ld;
  int o = 0;
#pragma unroll
  for (int q = 1; q < kMaxParts; ++q) o += (q < p.nparts && (int64_t)j >= p.part_lo[q]);
  return p.xparts[o] + (size_t)(j - (uint32_t)p.part_lo[o]) * (uint32_t)p.ld;
}

// Hub rows (degree >= heavy_threshold) are cut into kSlice-column slices and
// one warp owns one (row, slice) task.  Its serial chain -- every (row, column)
// sum is added in CSR order, bit-exact with the reference's _row -- is as long
// as the hub's degree, so the task is a deep software pipeline: lane
// (nb = lane/4, cg = lane%4) copies column cg of neighbour nb of each
// 8-neighbour wave into its own shared-memory slot with cp.async (LDGSTS),
// together with the wave's col ids (2*kHubDepth waves ahead) and dinv_j / the
// stored value (kHubDepth waves ahead).  A lane only reads back what it copied
// itself, so one per-thread cp.async group per wave is the whole
// synchronisation, and 8*kHubDepth neighbours stay in flight per warp (the
// former register-gather version waited one memory latency per 32 neighbours
// and set the launch length on R-MAT: the 406k-degree hub of C3 took the whole
// 52.7 ms step at P = 32, profiles/r01_trace_report.json).  Products h_ij*X[j,c] are
// formed in parallel and added in neighbour order through shuffles.
constexpr int kSlice = 4;
constexpr int kTileW = 64;  // column tile of the 4-column layouts' gather4 passes
constexpr int kHubDepth = 16;
// per-warp hub ring: rows [kHubDepth][32] + dinv_j [kHubDepth][8] doubles,
// col ids [2*kHubDepth][8] int32
constexpr int kHubRingDoubles = kHubDepth * 32 + kHubDepth * 8 + kHubDepth * 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async_8(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_4(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
// streamed operands (read once per step): L2 evict_first
__device__ __forceinline__ void cp_async_4_first(uint32_t dst, const void *src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int MODE, bool EXPL, bool FIRST>
__device__ __forceinline__ void heavy_task(const StepParams &p, int64_t t, double *hub) {
  const int lane = threadIdx.x & 31;
  const int nb = lane >> 2, cg = lane & 3;
  const int64_t ld = p.ld;
  const int nsl = (int)((p.tw + kSlice - 1) / kSlice);  // slices of this launch's column tile
  const int h = (int)(t / nsl), sl = (int)(t % nsl);
  const int i = p.heavy_rows[h];
  const int64_t beg = p.row_ptr[i], end = p.row_ptr[i + 1];
  const int64_t d = end - beg;
  double di = 0.0;
  if constexpr (!EXPL) di = p.dinv[p.row0 + i];
  const int64_t c = p.col0 + (int64_t)sl * kSlice + cg;
  const bool active = (int64_t)sl * kSlice + cg < p.tw;
  const uint32_t rows_sa = smem_u32(hub);                     // [D][32] doubles
  const uint32_t w_sa = rows_sa + kHubDepth * 32 * 8;         // [D][8] doubles
  const uint32_t col_sa = w_sa + kHubDepth * 8 * 8;           // [2D][8] int32
  const int64_t nw = (d + 7) >> 3;
  auto col_slot = [&](int64_t w) {
    return col_sa + (uint32_t)(((w % (2 * kHubDepth)) * 8 + nb) * 4);
  };
  // col id of neighbour nb of wave w (lane nb*4 copies it)
  auto issue_col = [&](int64_t w) {
    const int64_t e = beg + w * 8 + nb;
    if (cg == 0 && e < end) cp_async_4(col_slot(w), p.col + e);
  };
  // column c of neighbour nb of wave w, and its weight (col ids landed)
  auto issue_row = [&](int64_t w) {
    if (w >= nw) return;  // warp-uniform
    const int64_t e = beg + w * 8 + nb;
    int j = 0;
    if (cg == 0 && e < end) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(j) : "r"(col_slot(w)));
    j = __shfl_sync(0xffffffffu, j, lane & ~3);
    if (e < end) {
      const uint32_t slot = (uint32_t)(w % kHubDepth);
      if (active) cp_async_8(rows_sa + (slot * 32 + lane) * 8, gather_row(p, (uint32_t)j) + c);
      if (cg == 0) {
        if constexpr (EXPL) cp_async_8(w_sa + (slot * 8 + nb) * 8, p.vals + e);
        else cp_async_8(w_sa + (slot * 8 + nb) * 8, p.dinv + j);
      }
    }
  };
  for (int w = 0; w < 2 * kHubDepth; ++w) issue_col(w);
  cp_async_commit();
  cp_async_wait<0>();
  for (int w = 0; w < kHubDepth; ++w) {
    issue_row(w);
    cp_async_commit();
  }
  double acc = 0.0;
  for (int64_t w = 0; w < nw; ++w) {
    cp_async_wait<kHubDepth - 1>();  // wave w's rows / weights and col(w + D) landed
    const uint32_t slot = (uint32_t)(w % kHubDepth);
    double x = 0.0, wv = 0.0;
    if (active) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(rows_sa + (slot * 32 + lane) * 8));
    if (cg == 0) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wv) : "r"(w_sa + (slot * 8 + nb) * 8));
    wv = __shfl_sync(0xffffffffu, wv, lane & ~3);
    double hh;
    if constexpr (EXPL) hh = wv;
    else hh = __dmul_rn(di, wv);  // (1*dinv_i)*dinv_j, operators.py:110
    const double prod = __dmul_rn(hh, x);
    const int64_t cnt = d - w * 8;
    if (cnt >= 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, u * 4 + cg));
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double v = __shfl_sync(0xffffffffu, prod, u * 4 + cg);
        if (u < cnt) acc = __dadd_rn(acc, v);
      }
    }
    issue_row(w + kHubDepth);
    issue_col(w + 2 * kHubDepth);
    cp_async_commit();
  }
  cp_async_wait<0>();
  // epilogue on lanes 0..3 (lane cg holds the sum of column c)
  double part = 0.0;
  if (nb == 0 && active) {
    const size_t off = (size_t)i * ld + c;
    double y = acc, xo = 0.0;
    if constexpr (EXPL || MODE == MODE_DBL) xo = __ldg(p.X + off);
    if constexpr (EXPL) {
      if (p.shift != 0.0) y = __dsub_rn(y, __dmul_rn(p.shift, xo));
      if (p.scale != 1.0) y = __ddiv_rn(y, p.scale);
    }
    if constexpr (!FIRST) y = __dsub_rn(__dmul_rn(2.0, y), p.Xprev[off]);
    p.Y[off] = y;
    double *hp = p.hpart + (size_t)h * 2 * ld + c;
    if constexpr (MODE == MODE_DBL) {
      hp[0] = __dmul_rn(y, xo);
      hp[ld] = __dmul_rn(y, y);
    } else if constexpr (MODE == MODE_DIRECT) {
      hp[0] = __dmul_rn(__ldg(p.Z + off), y);
    } else {
      part = __dmul_rn(__ldg(p.Z + off), y);
    }
  }
  if constexpr (MODE == MODE_LDOS) {
    // slice sum over its columns in order (lanes 0..3)
    double tot = __shfl_sync(0xffffffffu, part, 0);
#pragma unroll
    for (int g2 = 1; g2 < kSlice; ++g2) tot = __dadd_rn(tot, __shfl_sync(0xffffffffu, part, g2));
    if (lane == 0) p.hldos[(size_t)h * nsl + sl] = tot;
  }
}

template <int C>
__device__ __forceinline__ void ld_vec(const double *p, double (&v)[C]) {
  if constexpr (C == 1) {
    v[0] = __ldg(p);
  } else if constexpr (C == 2) {
    double2 t = __ldg(reinterpret_cast<const double2 *>(p));
    v[0] = t.x; v[1] = t.y;
  } else {
    double2 t0 = __ldg(reinterpret_cast<const double2 *>(p));
    double2 t1 = __ldg(reinterpret_cast<const double2 *>(p + 2));
    v[0] = t0.x; v[1] = t0.y; v[2] = t1.x; v[3] = t1.y;
  }
}

// L2 eviction policies for gathered rows (the bulk path's hot rows)
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// plain (coherent) load: Xprev may alias Y
template <int C>
__device__ __forceinline__ void ld_vec_rw(const double *p, double (&v)[C]) {
  if constexpr (C == 1) {
    v[0] = *p;
  } else if constexpr (C == 2) {
    double2 t = *reinterpret_cast<const double2 *>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
    double2 t0 = *reinterpret_cast<const double2 *>(p);
    double2 t1 = *reinterpret_cast<const double2 *>(p + 2);
    v[0] = t0.x; v[1] = t0.y; v[2] = t1.x; v[3] = t1.y;
  }
}

template <int C>
__device__ __forceinline__ void st_vec(double *p, const double (&v)[C]) {
  if constexpr (C == 1) {
    *p = v[0];
  } else if constexpr (C == 2) {
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
  } else {
    *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2 *>(p + 2) = make_double2(v[2], v[3]);
  }
}

// T_{k+1} rows are written once and next read a whole step later: evict_first
template <int C>
__device__ __forceinline__ void st_vec_first(double *p, const double (&v)[C], uint64_t pol) {
  if constexpr (C == 1) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v[0]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v[0]),
                 "d"(v[1]), "l"(pol)
                 : "memory");
    if constexpr (C == 4)
      asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p + 2), "d"(v[2]),
                   "d"(v[3]), "l"(pol)
                   : "memory");
  }
}

__device__ __forceinline__ double warp_sum_fixed(double x) {
  // fixed butterfly: same tree for every call -> deterministic
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// One light row chunk, worked by one warp: rows in order, one row at a time
// (lane l owns columns [l*C, l*C+C) of each 32*C-wide tile), per-warp moment
// accumulators in shared memory, written to the chunk's own partial slot.
template <int C, int MODE, bool EXPL, bool FIRST, bool INIT, int U>
__device__ __forceinline__ void light_chunk(const StepParams &p, int chunk, double *my) {
  const int lane = threadIdx.x & 31;
  const int64_t ld = p.ld;
  const int ntiles = (int)((ld + 32 * C - 1) / (32 * C));
  if constexpr (MODE != MODE_LDOS) {
    for (int64_t e = lane; e < 2 * ld; e += 32) my[e] = 0.0;
    __syncwarp();
  }
  const int r0 = p.chunk_start[chunk], r1 = p.chunk_start[chunk + 1];
  int64_t beg = 0, end = 0;
  if constexpr (!INIT) {
    if (r0 < r1) end = p.row_ptr[r0];
  }
  for (int i = r0; i < r1; ++i) {
    const size_t rowoff = (size_t)i * ld;
    double di = 0.0;
    if constexpr (!INIT) {
      beg = end;
      end = p.row_ptr[i + 1];
      if (p.n_heavy > 0 && end - beg >= p.heavy_threshold) continue;  // hub task
      if constexpr (!EXPL) di = p.dinv[p.row0 + i];
    }
    double lsum = 0.0;  // LDOS lane partial
    for (int t = 0; t < ntiles; ++t) {
      const int64_t c0 = ((int64_t)t * 32 + lane) * C;
      const bool active = c0 < ld;
      double y[C], xo[C], pv[C], zv[C];
      // own-row operands first: independent of the neighbour walk
      if (active) {
        if constexpr (INIT || EXPL || MODE == MODE_DBL) ld_vec<C>(p.X + rowoff + c0, xo);
        if constexpr (!INIT && !FIRST) ld_vec_rw<C>(p.Xprev + rowoff + c0, pv);
        if constexpr (!INIT && MODE != MODE_DBL) ld_vec<C>(p.Z + rowoff + c0, zv);
      }
      double acc[C];
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0.0;
      if constexpr (!INIT) {
        for (int64_t base = beg; base < end; base += 32) {
          const int cnt = (int)min((int64_t)32, end - base);
          int jl = 0;
          double hl = 0.0;
          if (lane < cnt) {
            jl = p.col[base + lane];
            if constexpr (EXPL) {
              hl = p.vals[base + lane];
            } else {
              const double dj = __ldg(p.dinv + jl);
              hl = __dmul_rn(di, dj);
            }
          }
          for (int q = 0; q < cnt; q += U) {
            double v[U][C];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int j = __shfl_sync(0xffffffffu, jl, (q + u) & 31);
#pragma unroll
              for (int c = 0; c < C; ++c) v[u][c] = 0.0;
              if (q + u < cnt && active) ld_vec<C>(gather_row(p, (uint32_t)j) + c0, v[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const double h = __shfl_sync(0xffffffffu, hl, (q + u) & 31);
              if (q + u < cnt) {
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(h, v[u][c]));
              }
            }
          }
        }
      }
      if (!active) continue;
      if constexpr (INIT) {
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = zv[c] = xo[c];  // T_0 = z
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = acc[c];
        if constexpr (EXPL) {
          // operators.py:144-147: y -= shift*x; y /= scale (separate roundings)
          if (p.shift != 0.0) {
#pragma unroll
            for (int c = 0; c < C; ++c) y[c] = __dsub_rn(y[c], __dmul_rn(p.shift, xo[c]));
          }
          if (p.scale != 1.0) {
#pragma unroll
            for (int c = 0; c < C; ++c) y[c] = __ddiv_rn(y[c], p.scale);
          }
        }
        if constexpr (!FIRST) {
#pragma unroll
          for (int c = 0; c < C; ++c) y[c] = __dsub_rn(__dmul_rn(2.0, y[c]), pv[c]);
        }
        st_vec<C>(p.Y + rowoff + c0, y);
      }
      if constexpr (MODE == MODE_DBL) {
        double *s1 = my + c0, *s2 = my + ld + c0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if constexpr (INIT) {
            s1[c] = __dadd_rn(s1[c], __dmul_rn(y[c], y[c]));
          } else {
            s1[c] = __dadd_rn(s1[c], __dmul_rn(y[c], xo[c]));
            s2[c] = __dadd_rn(s2[c], __dmul_rn(y[c], y[c]));
          }
        }
      } else if constexpr (MODE == MODE_DIRECT) {
        double *s1 = my + c0;
#pragma unroll
        for (int c = 0; c < C; ++c) s1[c] = __dadd_rn(s1[c], __dmul_rn(zv[c], y[c]));
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) lsum = __dadd_rn(lsum, __dmul_rn(zv[c], y[c]));
      }
    }
    if constexpr (MODE == MODE_LDOS) {
      const double num = warp_sum_fixed(lsum);
      if (lane == 0) {
        if (!isfinite(num)) atomicOr(p.flag, 1);
        if constexpr (INIT) {
          // kpm.py:144-147: den = einsum(z, z) (same reduction as num[0])
          double *den = const_cast<double *>(p.den);
          den[out_row(p, i)] = num;  // zero mass is checked on the final den (kpm_run_result)
        }
        p.ldos[out_row(p, i) * p.ldos_stride + p.ldos_col] = num;  // raw num[m, i]
      }
    }
  }
  if constexpr (MODE != MODE_LDOS) {
    __syncwarp();
    const int nred = (MODE == MODE_DBL && !INIT) ? 2 : 1;
    double *out = p.partial + (size_t)chunk * 2 * ld;
    for (int64_t e = lane; e < nred * ld; e += 32) out[e] = my[e];
    __syncwarp();
  }
}

// Row epilogue shared by the streamed path: y = acc (+ explicit shift/scale),
// T_{k+1} = 2y - T_{k-1}, store, and fold the moment products of this row.
template <int C, int MODE, bool EXPL, bool FIRST>
__device__ __forceinline__ void stream_finish_row(const StepParams &p, int row, bool active,
                                                  int64_t c0, const double (&acc)[C],
                                                  const double (&xo)[C], const double (&pv)[C],
                                                  const double (&zv)[C], double *my) {
  const int lane = threadIdx.x & 31;
  const int64_t ld = p.ld;
  double lsum = 0.0;
  if (active) {
    double y[C];
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = acc[c];
    if constexpr (EXPL) {
      if (p.shift != 0.0) {
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = __dsub_rn(y[c], __dmul_rn(p.shift, xo[c]));
      }
      if (p.scale != 1.0) {
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = __ddiv_rn(y[c], p.scale);
      }
    }
    if constexpr (!FIRST) {
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = __dsub_rn(__dmul_rn(2.0, y[c]), pv[c]);
    }
    st_vec<C>(p.Y + (size_t)row * ld + c0, y);
    if constexpr (MODE == MODE_DBL) {
      double *s1 = my + c0, *s2 = my + ld + c0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        s1[c] = __dadd_rn(s1[c], __dmul_rn(y[c], xo[c]));
        s2[c] = __dadd_rn(s2[c], __dmul_rn(y[c], y[c]));
      }
    } else if constexpr (MODE == MODE_DIRECT) {
      double *s1 = my + c0;
#pragma unroll
      for (int c = 0; c < C; ++c) s1[c] = __dadd_rn(s1[c], __dmul_rn(zv[c], y[c]));
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) lsum = __dadd_rn(lsum, __dmul_rn(zv[c], y[c]));
    }
  }
  if constexpr (MODE == MODE_LDOS) {
    const double num = warp_sum_fixed(lsum);
    if (lane == 0) {
      if (!isfinite(num)) atomicOr(p.flag, 1);
      p.ldos[out_row(p, row) * p.ldos_stride + p.ldos_col] = num;
    }
  }
}

#ifndef KPM_FAST_MINC
#define KPM_FAST_MINC 1  // smallest column layout that uses the full-wave fast path
#endif
// Light chunk as ONE stream of nonzeros (single column tile, ld <= 32*C):
// neighbour ids / weights are fetched 32 at a time across row boundaries and
// U gathers stay in flight continuously, so short rows no longer serialise on
// their own load latencies; a row is finished the moment its last neighbour
// is added (same per-row sequential order => still bit-exact).  The next
// row's own operands (T_k, T_{k-1}, z) are prefetched one row ahead.  Hub rows
// are singleton chunks and never appear here.
template <int C, int MODE, bool EXPL, bool FIRST, int U>
__device__ __forceinline__ void light_stream(const StepParams &p, int chunk, double *my) {
  const int lane = threadIdx.x & 31;
  const int64_t ld = p.ld;
  const int64_t c0 = (int64_t)lane * C;
  const bool active = c0 < ld;
  const bool full_lanes = ld == 32 * C;  // every lane owns C real columns
  const int r0 = p.chunk_start[chunk], r1 = p.chunk_start[chunk + 1];
  if constexpr (MODE != MODE_LDOS) {
    for (int64_t e = lane; e < 2 * ld; e += 32) my[e] = 0.0;
    __syncwarp();
  }
  // a singleton chunk holding a hub row: its hub tasks write the row
  if (r1 - r0 == 1 && p.n_heavy > 0 &&
      p.row_ptr[r1] - p.row_ptr[r0] >= p.heavy_threshold) {
    if constexpr (MODE != MODE_LDOS) {
      double *out = p.partial + (size_t)chunk * 2 * ld;
      for (int64_t e = lane; e < 2 * ld; e += 32) out[e] = 0.0;
    }
    return;
  }
  // lane window over the chunk's rows: row_ptr[wb+lane] and dinv[wb+lane]
  int wb = r0;
  int64_t wrp = p.row_ptr[min(r0 + lane, r1)];
  double wdi = 0.0;
  if constexpr (!EXPL) wdi = (r0 + lane < r1) ? p.dinv[p.row0 + r0 + lane] : 0.0;
  auto refill = [&](int base) {
    wb = base;
    wrp = p.row_ptr[min(base + lane, r1)];
    if constexpr (!EXPL) wdi = (base + lane < r1) ? p.dinv[p.row0 + base + lane] : 0.0;
  };
  // row_ptr[r] for wb <= r <= wb+31 (r <= r1)
  auto rp = [&](int r) { return __shfl_sync(0xffffffffu, wrp, r - wb); };

  const int64_t K0 = __shfl_sync(0xffffffffu, wrp, 0);
  const int64_t K1 = p.row_ptr[r1];
  int row = r0;
  if (row + 1 - wb > 31) refill(row);
  int64_t rend = rp(row + 1);
  double di = 0.0;
  if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
  // own operands of the current row
  double xo[C], pv[C], zv[C];
  auto own = [&](int r, double (&a)[C], double (&b)[C], double (&cz)[C]) {
#pragma unroll
    for (int c = 0; c < C; ++c) a[c] = b[c] = cz[c] = 0.0;
    if (r < r1 && active) {
      const size_t off = (size_t)r * ld + c0;
      if constexpr (EXPL || MODE == MODE_DBL) ld_vec<C>(p.X + off, a);
      if constexpr (!FIRST) ld_vec_rw<C>(p.Xprev + off, b);
      if constexpr (MODE != MODE_DBL) ld_vec<C>(p.Z + off, cz);
    }
  };
  own(row, xo, pv, zv);
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;

  // finish every row whose nonzeros are exhausted at position kk
  auto advance = [&](int64_t kk) {
    while (row < r1 && kk == rend) {
      stream_finish_row<C, MODE, EXPL, FIRST>(p, row, active, c0, acc, xo, pv, zv, my);
      ++row;
      if (row >= r1) break;
      if (row + 1 - wb > 31) refill(row);
      rend = rp(row + 1);
      if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0.0;
      own(row, xo, pv, zv);
    }
  };
  advance(K0);  // leading empty rows

  for (int64_t kb = K0; kb < K1; kb += 32) {
    const int cnt = (int)min((int64_t)32, K1 - kb);
    int jl = 0;
    double wl = 0.0;  // dinv_j (implicit) or the stored value (explicit)
    if (lane < cnt) {
      jl = p.col[kb + lane];
      if constexpr (EXPL) wl = p.vals[kb + lane];
      else wl = __ldg(p.dinv + jl);
    }
    for (int q = 0; q < cnt; q += U) {
      double v[U][C];
      if (C >= KPM_FAST_MINC && full_lanes && q + U <= cnt && kb + q + U <= rend) {
        // fast path: a full wave inside the current row -- no predicates,
        // no per-neighbour row-end checks
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = __shfl_sync(0xffffffffu, jl, q + u);
          ld_vec<C>(gather_row(p, (uint32_t)j) + c0, v[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double w = __shfl_sync(0xffffffffu, wl, q + u);
          double h;
          if constexpr (EXPL) h = w;
          else h = __dmul_rn(di, w);
#pragma unroll
          for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(h, v[u][c]));
        }
        advance(kb + q + U);
        continue;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = __shfl_sync(0xffffffffu, jl, (q + u) & 31);
#pragma unroll
        for (int c = 0; c < C; ++c) v[u][c] = 0.0;
        if (q + u < cnt && active)
          ld_vec<C>(gather_row(p, (uint32_t)j) + c0, v[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double w = __shfl_sync(0xffffffffu, wl, (q + u) & 31);
        if (q + u < cnt) {
          double h;
          if constexpr (EXPL) h = w;
          else h = __dmul_rn(di, w);  // (1*dinv_i)*dinv_j, operators.py:110
#pragma unroll
          for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(h, v[u][c]));
          advance(kb + q + u + 1);
        }
      }
    }
  }
  advance(K1);  // trailing empty rows
  if constexpr (MODE != MODE_LDOS) {
    __syncwarp();
    const int nred = MODE == MODE_DBL ? 2 : 1;
    double *out = p.partial + (size_t)chunk * 2 * ld;
    for (int64_t e = lane; e < nred * ld; e += 32) out[e] = my[e];
    __syncwarp();
  }
}

// ------------------------------------------------ bulk-copy gathers (C = 4)
// The same streamed light chunk for the 4-column layout (one column tile,
// ld <= 128), with the neighbour rows moved by the TMA engine instead of
// register loads: every gathered row (8*ld <= 1 KB) is one cp.async.bulk
// global->shared copy completing on its own mbarrier, so the bytes in flight
// per warp no longer cost registers.  A warp owns a ring of kBulkSlots row
// slots; nonzeros are issued in waves of kBulkWave (lane L of the issuing
// half-warp copies one row into slot L; one mbarrier per wave collects the
// copies' bytes), kBulkSlots / kBulkWave waves are in flight, and the
// consumer waits once per wave and adds the rows IN CSR ORDER from shared memory
// (same products, same sequential sums => still bit-identical).  Neighbour ids
// are loaded two batches ahead and their dinv_j one batch ahead, so neither
// dependent load sits on the critical path.  Optional L2 policies: rows of
// vertices with dinv_j <= hot_dinv (high degree, re-gathered many times per
// step) are copied with evict_last, the rest with evict_first.
#ifndef KPM_BULK_WAVE
#define KPM_BULK_WAVE 8
#endif
constexpr int kBulkWave = KPM_BULK_WAVE;
#ifndef KPM_BULK_SLOTS
#define KPM_BULK_SLOTS 8
#endif
#ifndef KPM_BULK_SLOTS2
#define KPM_BULK_SLOTS2 16
#endif
#ifndef KPM_BULK_SLOTS1
#define KPM_BULK_SLOTS1 32
#endif
// ring slots per warp for the 4-, 2- and 1-column layouts (rows of <= 1 KB,
// 512 B, 256 B): about 8 KB of gathers in flight per warp in each case
template <int C>
struct BulkShape {
  static constexpr int slots = C == 4 ? KPM_BULK_SLOTS : (C == 2 ? KPM_BULK_SLOTS2 : KPM_BULK_SLOTS1);
  static_assert(slots % kBulkWave == 0 && slots <= 32, "ring shape");
};

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bulk_gather(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar, int pol_kind, uint64_t pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  if (pol_kind) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// Row epilogue of the bulk path: as stream_finish_row, with the moment
// products folded into per-lane registers (the lane owns fixed columns).
template <int C, int MODE, bool EXPL, bool FIRST, bool SFIRST = false>
__device__ __forceinline__ void bulk_finish_row(const StepParams &p, int row, bool active,
                                                int64_t c0, const double (&acc)[C],
                                                const double (&xo)[C], const double (&pv)[C],
                                                const double (&zv)[C], double (&s1)[C],
                                                double (&s2)[C], uint64_t pol_first = 0) {
  const int lane = threadIdx.x & 31;
  double lsum = 0.0;
  if (active) {
    double y[C];
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = acc[c];
    if constexpr (EXPL) {
      if (p.shift != 0.0) {
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = __dsub_rn(y[c], __dmul_rn(p.shift, xo[c]));
      }
      if (p.scale != 1.0) {
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = __ddiv_rn(y[c], p.scale);
      }
    }
    if constexpr (!FIRST) {
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = __dsub_rn(__dmul_rn(2.0, y[c]), pv[c]);
    }
    if constexpr (SFIRST) st_vec_first<C>(p.Y + (size_t)row * p.ld + c0, y, pol_first);
    else st_vec<C>(p.Y + (size_t)row * p.ld + c0, y);
    if constexpr (MODE == MODE_DBL) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        s1[c] = __dadd_rn(s1[c], __dmul_rn(y[c], xo[c]));
        s2[c] = __dadd_rn(s2[c], __dmul_rn(y[c], y[c]));
      }
    } else if constexpr (MODE == MODE_DIRECT) {
#pragma unroll
      for (int c = 0; c < C; ++c) s1[c] = __dadd_rn(s1[c], __dmul_rn(zv[c], y[c]));
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) lsum = __dadd_rn(lsum, __dmul_rn(zv[c], y[c]));
    }
  }
  if constexpr (MODE == MODE_LDOS) {
    const double num = warp_sum_fixed(lsum);
    if (lane == 0) {
      if (!isfinite(num)) atomicOr(p.flag, 1);
      p.ldos[out_row(p, row) * p.ldos_stride + p.ldos_col] = num;
    }
  }
}

// per-warp data region of the bulk kernel: the gather ring + weights, or the
// hub ring when hub tasks exist (whichever is larger); the mbarriers follow
__host__ __device__ inline size_t bulk_data_doubles(int slots, int64_t ld, bool hubs) {
  const size_t ring = (size_t)slots * ld + slots;
  return hubs && ring < (size_t)kHubRingDoubles ? (size_t)kHubRingDoubles : ring;
}

struct BulkRing {
  double *slot;     // slots x ld doubles
  double *wv;       // slots: dinv_j (implicit) or the stored value
  uint64_t *bar;    // one mbarrier per wave group (slots / kBulkWave)
  uint32_t phase;   // bit g: parity of group g's next completion (warp-uniform)
};

template <int C, int MODE, bool EXPL, bool FIRST>
__device__ __forceinline__ void light_bulk(const StepParams &p, int chunk, BulkRing &ring) {
  constexpr int kBulkSlots = BulkShape<C>::slots;
  const int lane = threadIdx.x & 31;
  const int64_t ld = p.ld;
  const int64_t c0 = (int64_t)lane * C;
  const bool active = c0 < ld;
  const uint32_t rbytes = (uint32_t)(ld * sizeof(double));
  const int r0 = p.chunk_start[chunk], r1 = p.chunk_start[chunk + 1];
  double s1[C], s2[C];
#pragma unroll
  for (int c = 0; c < C; ++c) s1[c] = s2[c] = 0.0;
  if (r1 - r0 == 1 && p.n_heavy > 0 &&
      p.row_ptr[r1] - p.row_ptr[r0] >= p.heavy_threshold) {
    if constexpr (MODE != MODE_LDOS) {
      double *out = p.partial + (size_t)chunk * 2 * ld;
      for (int64_t e = lane; e < 2 * ld; e += 32) out[e] = 0.0;
    }
    return;
  }
  int wb = r0;
  int64_t wrp = p.row_ptr[min(r0 + lane, r1)];
  double wdi = 0.0;
  if constexpr (!EXPL) wdi = (r0 + lane < r1) ? p.dinv[p.row0 + r0 + lane] : 0.0;
  auto refill = [&](int base) {
    wb = base;
    wrp = p.row_ptr[min(base + lane, r1)];
    if constexpr (!EXPL) wdi = (base + lane < r1) ? p.dinv[p.row0 + base + lane] : 0.0;
  };
  auto rp = [&](int r) { return __shfl_sync(0xffffffffu, wrp, r - wb); };
  const int64_t K0 = __shfl_sync(0xffffffffu, wrp, 0);
  const int64_t K1 = p.row_ptr[r1];
  int row = r0;
  if (row + 1 - wb > 31) refill(row);
  int64_t rend = rp(row + 1);
  double di = 0.0;
  if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
  double xo[C], pv[C], zv[C];
  auto own = [&](int r) {
#pragma unroll
    for (int c = 0; c < C; ++c) xo[c] = pv[c] = zv[c] = 0.0;
    if (r < r1 && active) {
      const size_t off = (size_t)r * ld + c0;
      if constexpr (EXPL || MODE == MODE_DBL) ld_vec<C>(p.X + off, xo);
      if constexpr (!FIRST) ld_vec_rw<C>(p.Xprev + off, pv);
      if constexpr (MODE != MODE_DBL) ld_vec<C>(p.Z + off, zv);
    }
  };
  own(row);
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  auto advance = [&](int64_t kk) {
    while (row < r1 && kk == rend) {
      bulk_finish_row<C, MODE, EXPL, FIRST>(p, row, active, c0, acc, xo, pv, zv, s1, s2);
      ++row;
      if (row >= r1) break;
      if (row + 1 - wb > 31) refill(row);
      rend = rp(row + 1);
      if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0.0;
      own(row);
    }
  };
  advance(K0);

  // neighbour ids two batches ahead, dinv_j / values one batch ahead
  const int64_t nnz = K1 - K0;
  auto ld_col = [&](int64_t b) -> int {
    const int64_t e = K0 + b * 32 + lane;
    return e < K1 ? p.col[e] : 0;
  };
  auto ld_w = [&](int64_t b, int j) -> double {
    const int64_t e = K0 + b * 32 + lane;
    if (e >= K1) return 0.0;
    if constexpr (EXPL) return p.vals[e];
    else return __ldg(p.dinv + j);
  };
  int jc = ld_col(0), jn = ld_col(1), jnn = 0;
  double wc = ld_w(0, jc), wn = 0.0;
  int64_t cur_b = 0;  // batch held in (jc, wc)
  // L2 policy (profiles/r02_ncu_summary.md section 3): cold rows evict_first, hot
  // rows no hint (evict_last on TMA copies does not hold lines); hot = id below
  // hot_rows on the gather-ordered twin, else a degree threshold
  const bool hints = p.hot_dinv > 0.0 || p.hot_rows > 0;
  const uint64_t pol_first = hints ? l2_policy_first() : 0;
  auto issue = [&](int64_t w) {  // wave w -> slots (w % nw) * kBulkWave + k
    const int64_t e0 = w * kBulkWave;
    if (e0 >= nnz) return;
    const int64_t b = e0 >> 5;
    if (b != cur_b) {  // advance the batch registers (b == cur_b + 1)
      jc = jn;
      jn = jnn;
      wc = wn;
      cur_b = b;
      jnn = ld_col(b + 2);
      wn = ld_w(b + 1, jn);
    } else if (b == 0 && w == 0) {
      jnn = ld_col(2);
      wn = ld_w(1, jn);
    }
    const int src_lane = (int)(e0 & 31) + (lane & (kBulkWave - 1));
    const int j = __shfl_sync(0xffffffffu, jc, src_lane);
    const double wv = __shfl_sync(0xffffffffu, wc, src_lane);
    const int g = (int)(w % (kBulkSlots / kBulkWave));
    const int base = g * kBulkWave;
    const int k = lane - base;
    if (k >= 0 && k < kBulkWave) {
      // every lane of the group arrives (count kBulkWave); lanes with a
      // nonzero also add their copy's bytes to the wave's transaction count
      if (e0 + k < nnz) {
        const int L = base + k;
        ring.wv[L] = wv;
        bool hot = false;
        if (p.hot_rows > 0) hot = j < p.hot_rows;
        else if constexpr (!EXPL) hot = wv <= p.hot_dinv;
        bulk_gather(ring.slot + (size_t)L * ld,
                    p.nparts <= 1 ? p.X + (size_t)(uint32_t)j * (uint32_t)ld : gather_row(p, (uint32_t)j),
                    rbytes, ring.bar + g, (hints && !hot) ? 1 : 0, pol_first);
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(ring.bar + g))
                     : "memory");
      }
    }
  };
  constexpr int kWaves = kBulkSlots / kBulkWave;
  const int64_t nwaves = (nnz + kBulkWave - 1) / kBulkWave;
  // inactive lanes (c0 >= ld) read column 0 of the slot; their sums are unused
  const uint32_t slot_sa = smem_u32(ring.slot) + (uint32_t)(active ? c0 : 0) * 8u;
  const uint32_t wv_sa = smem_u32(ring.wv);
#pragma unroll
  for (int w = 0; w < kWaves; ++w) issue(w);
  __syncwarp();
  for (int64_t w = 0; w < nwaves; ++w) {
    const int g = (int)(w % kWaves);
    const int base = g * kBulkWave;
    const int cnt = (int)min((int64_t)kBulkWave, nnz - w * kBulkWave);
    mbar_wait(ring.bar + g, (ring.phase >> g) & 1u);  // the whole wave landed
    ring.phase ^= 1u << g;
    const int64_t e0 = K0 + w * kBulkWave;
    // one neighbour: 32 B of the slot per lane + its weight (shared loads by
    // 32-bit shared-window address, no generic->shared conversion per use)
    auto add_one = [&](int L) {
      double v[C];
      const uint32_t a = slot_sa + (uint32_t)L * rbytes;
      if constexpr (C == 1) {
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v[0]) : "r"(a));
      } else {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a));
        if constexpr (C == 4)
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + 16));
      }
      double wv;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wv) : "r"(wv_sa + 8u * (uint32_t)L));
      double h;
      if constexpr (EXPL) h = wv;
      else h = __dmul_rn(di, wv);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(h, v[c]));
    };
    if (cnt == kBulkWave && e0 + kBulkWave <= rend) {
      // fast path: a full wave inside the current row, no row-end checks
#pragma unroll
      for (int k = 0; k < kBulkWave; ++k) add_one(base + k);
      advance(e0 + kBulkWave);
    } else {
      for (int k = 0; k < cnt; ++k) {
        add_one(base + k);
        advance(e0 + k + 1);
      }
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(w + kWaves);
    __syncwarp();
  }
  advance(K1);
  if constexpr (MODE != MODE_LDOS) {
    if (active) {
      double *out = p.partial + (size_t)chunk * 2 * ld + c0;
      st_vec<C>(out, s1);
      if constexpr (MODE == MODE_DBL) st_vec<C>(out + ld, s2);
    }
  }
}

#ifndef KPM_BULK_THREADS
#define KPM_BULK_THREADS 256
#endif
#ifndef KPM_BULK_MINB
#define KPM_BULK_MINB 2
#endif
#ifndef KPM_BULK_MINB2
#define KPM_BULK_MINB2 3
#endif
#ifndef KPM_BULK_MINB1
#define KPM_BULK_MINB1 2
#endif
template <int C>
struct BulkTune {
  static constexpr int minb = C == 4 ? KPM_BULK_MINB : (C == 2 ? KPM_BULK_MINB2 : KPM_BULK_MINB1);
};
template <int C, int MODE, bool EXPL, bool FIRST>
__global__ void __launch_bounds__(KPM_BULK_THREADS, BulkTune<C>::minb)
kpm_step_bulk_kernel(const StepParams p) {
  constexpr int kBulkSlots = BulkShape<C>::slots;
  extern __shared__ __align__(16) double sbulk[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t ld = p.ld;
  // per warp: [kBulkSlots*ld ring][kBulkSlots values] (or the hub ring) [kBulkSlots bars]
  const size_t data = bulk_data_doubles(kBulkSlots, ld, p.n_heavy_tasks > 0);
  double *base = sbulk + (size_t)warp * (data + kBulkSlots);
  BulkRing ring;
  ring.slot = base;
  ring.wv = ring.slot + (size_t)kBulkSlots * ld;
  ring.bar = reinterpret_cast<uint64_t *>(base + data);
  ring.phase = 0;
  if (lane < kBulkSlots / kBulkWave) mbar_init(ring.bar + lane, kBulkWave);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int64_t total = p.n_heavy_tasks + p.n_chunks;
  for (;;) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(p.queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if ((int64_t)item >= total) break;
    const unsigned long long t0 = p.trace ? gtimer() : 0;
    if ((int64_t)item < p.n_heavy_tasks) {
      heavy_task<MODE, EXPL, FIRST>(p, (int64_t)item, base);
    } else {
      const int chunk = p.chunk_order[(int64_t)item - p.n_heavy_tasks];
      light_bulk<C, MODE, EXPL, FIRST>(p, chunk, ring);
    }
    trace_item(p, item, t0);
  }
}

// ------------------------------------- per-lane async gathers (C <= 2)
// Small probe blocks (P <= 64: one or two columns per lane, one column tile).
// Here a neighbour row is only 256-512 B, so the bulk path's per-copy cost (a
// uniform-register waterfall of ~9 instructions per cp.async.bulk) dominated:
// ~34 warp instructions per nonzero at P = 32, issue-bound (ncu,
// profiles/r01_ncu_summary.md).  This path moves every neighbour row with ONE
// cp.async (LDGSTS) per warp -- lane l copies its own C columns into its own
// slot -- so a lane reads back only what it copied.  Per wave of 8 nonzeros:
// the wave's col ids (lanes 0..7, 2*D waves ahead) and dinv_j / stored values
// (lanes 0..7, D waves ahead) ride in the same per-thread cp.async groups; the
// consumer waits for the group of D waves ago, __syncwarp()s (the weights were
// copied by other lanes) and adds the 8 rows IN CSR ORDER (bit-identical sums).
// The rows' own operands (T_k, T_{k-1}, z) come through an R-row prefetch ring
// completed on one mbarrier per slot (cp.async.mbarrier.arrive.noinc), so short
// and empty rows no longer wait one memory latency each.
template <int C, int MODE, bool EXPL, bool FIRST>
struct Lean {
  static constexpr int D = 4 / C;  // waves of 8 gathered rows in flight (8 KB)
  static constexpr int R = 8 / C;  // own-row prefetch depth
  static constexpr int NOP = ((EXPL || MODE == MODE_DBL) ? 1 : 0) + (FIRST ? 0 : 1) +
                             (MODE != MODE_DBL ? 1 : 0);
  static constexpr int W = 32 * C;  // doubles of one row tile
  static constexpr int rows_d = D * 8 * W;
  static constexpr int wv_d = D * 8;
  static constexpr int col_d = D * 8;  // [2D][8] int32
  static constexpr int own_d = R * (NOP > 0 ? NOP : 1) * W;
  static constexpr int bar_d = R;
  static constexpr int data_d = rows_d + wv_d + col_d + own_d + bar_d;
  static constexpr int warp_d = data_d > kHubRingDoubles ? data_d : kHubRingDoubles;
  static_assert(rows_d >= kHubRingDoubles, "hub ring must not reach the mbarriers");
};

template <int C>
__device__ __forceinline__ void cp_async_cols(uint32_t dst, const double *src) {
  if constexpr (C == 1) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  } else {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    if constexpr (C == 4)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(src + 2)
                   : "memory");
  }
}
template <int C>
__device__ __forceinline__ void cp_async_cols_hint(uint32_t dst, const double *src, uint64_t pol) {
  if constexpr (C == 1) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(dst),
                 "l"(src), "l"(pol)
                 : "memory");
  } else {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                 "l"(src), "l"(pol)
                 : "memory");
    if constexpr (C == 4)
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst + 16),
                   "l"(src + 2), "l"(pol)
                   : "memory");
  }
}
template <int C>
__device__ __forceinline__ void lds_cols(uint32_t a, double (&v)[C]) {
  if constexpr (C == 1) {
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v[0]) : "r"(a));
  } else {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a));
    if constexpr (C == 4)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + 16));
  }
}

template <int C, int MODE, bool EXPL, bool FIRST>
__device__ __forceinline__ void light_lean(const StepParams &p, int chunk, double *base,
                                           uint32_t &ophase) {
  using L = Lean<C, MODE, EXPL, FIRST>;
  constexpr int D = L::D, R = L::R, W = L::W, NOP = L::NOP;
  const int lane = threadIdx.x & 31;
  const int64_t ld = p.ld;
  const int64_t c0 = (int64_t)lane * C;
  const bool active = c0 < ld;
  const int r0 = p.chunk_start[chunk], r1 = p.chunk_start[chunk + 1];
  double s1[C], s2[C];
#pragma unroll
  for (int c = 0; c < C; ++c) s1[c] = s2[c] = 0.0;
  if (r1 - r0 == 1 && p.n_heavy > 0 &&
      p.row_ptr[r1] - p.row_ptr[r0] >= p.heavy_threshold) {
    if constexpr (MODE != MODE_LDOS) {
      double *out = p.partial + (size_t)chunk * 2 * ld;
      for (int64_t e = lane; e < 2 * ld; e += 32) out[e] = 0.0;
    }
    return;
  }
  const uint32_t rows_sa = smem_u32(base);
  const uint32_t wv_sa = rows_sa + L::rows_d * 8;
  const uint32_t col_sa = wv_sa + L::wv_d * 8;
  const uint32_t own_sa = col_sa + L::col_d * 8;
  uint64_t *obar = reinterpret_cast<uint64_t *>(base + L::rows_d + L::wv_d + L::col_d + L::own_d);

  int wb = r0;
  int64_t wrp = p.row_ptr[min(r0 + lane, r1)];
  double wdi = 0.0;
  if constexpr (!EXPL) wdi = (r0 + lane < r1) ? p.dinv[p.row0 + r0 + lane] : 0.0;
  auto refill = [&](int b) {
    wb = b;
    wrp = p.row_ptr[min(b + lane, r1)];
    if constexpr (!EXPL) wdi = (b + lane < r1) ? p.dinv[p.row0 + b + lane] : 0.0;
  };
  auto rp = [&](int r) { return __shfl_sync(0xffffffffu, wrp, r - wb); };
  const int64_t K0 = __shfl_sync(0xffffffffu, wrp, 0);
  const int64_t K1 = p.row_ptr[r1];
  const int64_t nnz = K1 - K0;
  const int64_t nw = (nnz + 7) >> 3;

  // own operands of row r -> ring slot (r - r0) % R
  auto issue_own = [&](int r) {
    if (r >= r1) return;  // warp-uniform
    const int sl = (r - r0) & (R - 1);
    if (active) {
      const size_t off = (size_t)r * ld + c0;
      const uint32_t dst = own_sa + (uint32_t)(sl * NOP * W + lane * C) * 8;
      int q = 0;
      if constexpr (EXPL || MODE == MODE_DBL) cp_async_cols<C>(dst + (q++) * W * 8, p.X + off);
      if constexpr (!FIRST) cp_async_cols<C>(dst + (q++) * W * 8, p.Xprev + off);
      if constexpr (MODE != MODE_DBL) cp_async_cols<C>(dst + (q++) * W * 8, p.Z + off);
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(obar + sl))
                 : "memory");
  };
  auto col_slot = [&](int64_t w) { return col_sa + (uint32_t)((w % (2 * D)) * 32); };
  auto issue_col = [&](int64_t w) {
    const int64_t e = w * 8 + lane;
    if (lane < 8 && e < nnz) cp_async_4(col_slot(w) + lane * 4, p.col + K0 + e);
  };
  auto issue_rows = [&](int64_t w) {
    if (w >= nw) return;  // warp-uniform
    const uint32_t sl = (uint32_t)(w % D);
    const int cnt = (int)min((int64_t)8, nnz - w * 8);
    int j[8];
    const uint32_t ca = col_slot(w);
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(j[0]), "=r"(j[1]), "=r"(j[2]), "=r"(j[3]) : "r"(ca));
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(j[4]), "=r"(j[5]), "=r"(j[6]), "=r"(j[7]) : "r"(ca + 16));
    const uint32_t dst = rows_sa + (uint32_t)(sl * 8 * W + lane * C) * 8;
    if (active) {
      if (p.nparts <= 1) {  // hoisted: the partition lookup costs ~25 instructions per row
        const double *xc = p.X + c0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < cnt) cp_async_cols<C>(dst + (uint32_t)(k * W) * 8, xc + (size_t)(uint32_t)j[k] * (uint32_t)ld);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < cnt) cp_async_cols<C>(dst + (uint32_t)(k * W) * 8, gather_row(p, (uint32_t)j[k]) + c0);
      }
    }
    if (lane < cnt) {
      const uint32_t wd = wv_sa + (sl * 8 + lane) * 8;
      if constexpr (EXPL) {
        cp_async_8(wd, p.vals + K0 + w * 8 + lane);
      } else {
        int jl;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(jl) : "r"(ca + lane * 4));
        cp_async_8(wd, p.dinv + jl);
      }
    }
  };

  // col ids of the first 2D waves, then the own rows and the first D waves
#pragma unroll
  for (int w = 0; w < 2 * D; ++w) issue_col(w);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) issue_own(r0 + r);
#pragma unroll
  for (int w = 0; w < D; ++w) {
    issue_rows(w);
    cp_async_commit();
  }

  int row = r0;
  if (row + 1 - wb > 31) refill(row);
  int64_t rend = rp(row + 1) - K0;  // nonzero positions relative to K0
  double di = 0.0;
  if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  auto finish = [&](int r) {
    const int sl = (r - r0) & (R - 1);
    mbar_wait(obar + sl, (ophase >> sl) & 1u);
    ophase ^= 1u << sl;
    double xo[C], pv[C], zv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) xo[c] = pv[c] = zv[c] = 0.0;
    if (active) {
      const uint32_t a = own_sa + (uint32_t)(sl * NOP * W + lane * C) * 8;
      int q = 0;
      if constexpr (EXPL || MODE == MODE_DBL) lds_cols<C>(a + (q++) * W * 8, xo);
      if constexpr (!FIRST) lds_cols<C>(a + (q++) * W * 8, pv);
      if constexpr (MODE != MODE_DBL) lds_cols<C>(a + (q++) * W * 8, zv);
    }
    bulk_finish_row<C, MODE, EXPL, FIRST>(p, r, active, c0, acc, xo, pv, zv, s1, s2);
    issue_own(r + R);
  };
  auto advance = [&](int64_t kk) {
    while (row < r1 && kk == rend) {
      finish(row);
      ++row;
      if (row >= r1) break;
      if (row + 1 - wb > 31) refill(row);
      rend = rp(row + 1) - K0;
      if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0.0;
    }
  };
  advance(0);  // leading empty rows

  const uint32_t my_rows = rows_sa + (uint32_t)(lane * C) * 8;
  for (int64_t w = 0; w < nw; ++w) {
    cp_async_wait<D - 1>();  // wave w's rows + weights, col ids of wave w + D
    __syncwarp();
    const uint32_t sl = (uint32_t)(w % D);
    const int64_t e0 = w * 8;
    const int cnt = (int)min((int64_t)8, nnz - e0);
    auto add_one = [&](int k) {
      double v[C];
      lds_cols<C>(my_rows + (uint32_t)((sl * 8 + k) * W) * 8, v);
      double wv;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wv) : "r"(wv_sa + (sl * 8 + k) * 8));
      double h;
      if constexpr (EXPL) h = wv;
      else h = __dmul_rn(di, wv);  // (1*dinv_i)*dinv_j, operators.py:110
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(h, v[c]));
    };
    if (cnt == 8 && e0 + 8 <= rend) {
#pragma unroll
      for (int k = 0; k < 8; ++k) add_one(k);
      advance(e0 + 8);
    } else {
      for (int k = 0; k < cnt; ++k) {
        add_one(k);
        advance(e0 + k + 1);
      }
    }
    __syncwarp();  // every lane is done with the wave's weights
    issue_rows(w + D);
    issue_col(w + 2 * D);
    cp_async_commit();
  }
  advance(nnz);
  cp_async_wait<0>();
  if constexpr (MODE != MODE_LDOS) {
    if (active) {
      double *out = p.partial + (size_t)chunk * 2 * ld + c0;
      st_vec<C>(out, s1);
      if constexpr (MODE == MODE_DBL) st_vec<C>(out + ld, s2);
    }
  }
}

#ifndef KPM_LEAN_MINB
#define KPM_LEAN_MINB 2
#endif
template <int C, int MODE, bool EXPL, bool FIRST>
__global__ void __launch_bounds__(256, KPM_LEAN_MINB) kpm_step_lean_kernel(const StepParams p) {
  using L = Lean<C, MODE, EXPL, FIRST>;
  extern __shared__ __align__(16) double slean[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double *base = slean + (size_t)warp * L::warp_d;
  uint64_t *obar = reinterpret_cast<uint64_t *>(base + L::rows_d + L::wv_d + L::col_d + L::own_d);
  if (lane < L::R) mbar_init(obar + lane, 32);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t ophase = 0;
  const int64_t total = p.n_heavy_tasks + p.n_chunks;
  for (;;) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(p.queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if ((int64_t)item >= total) break;
    const unsigned long long t0 = p.trace ? gtimer() : 0;
    if ((int64_t)item < p.n_heavy_tasks) {
      heavy_task<MODE, EXPL, FIRST>(p, (int64_t)item, base);
    } else {
      const int chunk = p.chunk_order[(int64_t)item - p.n_heavy_tasks];
      light_lean<C, MODE, EXPL, FIRST>(p, chunk, base, ophase);
    }
    trace_item(p, item, t0);
  }
}

// ------------------------------------------------ TMA gather4 light path
// The gathered neighbour rows are moved by the tensor engine's row gather:
// ONE cp.async.bulk.tensor...tile::gather4 (SASS UTMALDG.2D.GATHER4) copies
// four whole rows of the T_k block (tensor map n x ld fp64, box ld x 1) into
// the warp's ring, issued by lane 0 -- no per-lane copies, no uniform-register
// waterfall per row.  A wave is WAVE neighbours (WAVE/4 gather4 ops) completing
// on one mbarrier: lane 0 arrives with expect_tx for the rows, lanes 0..WAVE-1
// copy dinv_j / the stored value and the col ids of the wave 2D ahead with
// cp.async and arrive through cp.async.mbarrier.arrive.noinc, so a completed
// wave also has the col ids of the wave its slot is refilled with.  The
// consumer adds the rows IN CSR ORDER from shared memory (bit-identical sums);
// own operands come through the light_lean prefetch ring.
// Tuning (B200 sweeps, profiles/r01_ncu_summary.md): one wave in flight per
// warp.  Session 2: 24 warps per SM with 4 KB of rows per warp beat 16 warps
// with 8 KB in two 8-row waves (P=32 26.1 -> 23.5 ms, P=64 38.5 -> 32.3 ms on
// C3).  Session 3: the per-wave bookkeeping (issue, barrier, row-end checks:
// ~140 of the ~210 instructions per 8-row wave) costs power under the B200's
// power cap, so for P=64 one 16-row wave per warp at 16 warps per SM wins in
// the steady state (C3 P=128 as two 64-column tiles 73.1 -> 69.2 ms), and for
// P=32 one 32-row wave at 16 warps per SM (C3 24.9 -> 23.2 ms, C5 neutral).
#ifndef KPM_G4_WAVE1
#define KPM_G4_WAVE1 32
#endif
#ifndef KPM_G4_D1
#define KPM_G4_D1 1
#endif
#ifndef KPM_G4_MINB1
#define KPM_G4_MINB1 2
#endif
#ifndef KPM_G4_WAVE2
#define KPM_G4_WAVE2 16
#endif
#ifndef KPM_G4_D2
#define KPM_G4_D2 1
#endif
#ifndef KPM_G4_MINB2
#define KPM_G4_MINB2 2
#endif
#ifndef KPM_G4_OWN
#define KPM_G4_OWN 4
#endif
#ifndef KPM_G4_THREADS
#define KPM_G4_THREADS 256
#endif
template <int C>
struct G4Tune {  // neighbours per wave, waves in flight, resident 256-thread CTAs
  static constexpr int wave = C == 1 ? KPM_G4_WAVE1 : (C == 2 ? KPM_G4_WAVE2 : 4);
  static constexpr int d = C == 1 ? KPM_G4_D1 : (C == 2 ? KPM_G4_D2 : 1);
  static constexpr int minb = C == 1 ? KPM_G4_MINB1 : (C == 2 ? KPM_G4_MINB2 : 3);
};
template <int C, int MODE, bool EXPL, bool FIRST>
struct G4 {
  static constexpr int WAVE = G4Tune<C>::wave;  // neighbours per wave
  static constexpr int D = G4Tune<C>::d;        // waves in flight
  static constexpr int R = C == 4 ? 2 : KPM_G4_OWN / C;  // own-row prefetch depth
  static constexpr int NOP = Lean<C, MODE, EXPL, FIRST>::NOP;
  static constexpr int W = 32 * C;
  static constexpr int slot_d = ((WAVE * W * 8 + 127) / 128) * 128 / 8;  // one wave's rows
  static constexpr int rows_d = D * slot_d;
  static constexpr int wv_d = 2 * D * WAVE;   // [D][WAVE] doubles used (sized for 2D)
  static constexpr int col_d = 2 * D * WAVE;  // [2D][WAVE] int32 used (sized for 4D)
  static constexpr int own_d = R * (NOP > 0 ? NOP : 1) * W;
  static constexpr int bar_d = D + R;
  static constexpr int data_d = rows_d + wv_d + col_d + own_d;
  static constexpr int warp_d = ((data_d > kHubRingDoubles ? data_d : kHubRingDoubles) + bar_d + 15) / 16 * 16;
  static_assert(D >= 1 && R >= 1 && (R & (R - 1)) == 0, "gather4 ring shape");
};

// One elected lane of a converged warp (lane 0): unlike `lane == 0`, ptxas
// knows a single thread runs the guarded TMA issue, so the uniform-register
// operands need no waterfall loop.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tma_gather4_hint(uint32_t dst, const CUtensorMap *tm, int x,
                                                 int j0, int j1, int j2, int j3, uint32_t bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(tm), "r"(x), "r"(j0), "r"(j1), "r"(j2), "r"(j3), "r"(bar), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *tm, int x, int j0,
                                            int j1, int j2, int j3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(tm), "r"(x), "r"(j0), "r"(j1), "r"(j2), "r"(j3), "r"(bar)
      : "memory");
}

template <int C, int MODE, bool EXPL, bool FIRST>
__device__ __forceinline__ void light_g4(const StepParams &p, const CUtensorMap *tm, int chunk,
                                         const int64_t col0, const int64_t tw, double *base,
                                         uint32_t &ophase, uint32_t &wphase,
                                         const uint32_t dtab_sa) {
  using L = G4<C, MODE, EXPL, FIRST>;
  constexpr int D = L::D, R = L::R, W = L::W, NOP = L::NOP, WAVE = L::WAVE;
  const int lane = threadIdx.x & 31;
  const int64_t ld = p.ld;
  // this launch's column tile [col0, col0 + tw): lane l owns columns col0 + [lC, lC + C)
  const int64_t c0 = col0 + (int64_t)lane * C;
  const bool active = (int64_t)lane * C < tw;
  const int r0 = p.chunk_start[chunk], r1 = p.chunk_start[chunk + 1];
  double s1[C], s2[C];
#pragma unroll
  for (int c = 0; c < C; ++c) s1[c] = s2[c] = 0.0;
  if (r1 - r0 == 1 && p.n_heavy > 0 &&
      p.row_ptr[r1] - p.row_ptr[r0] >= p.heavy_threshold) {
    if constexpr (MODE != MODE_LDOS) {
      double *out = p.partial + (size_t)chunk * 2 * ld;
      for (int64_t e = lane; e < 2 * ld; e += 32) out[e] = 0.0;
    }
    return;
  }
  // L2 policy (tools/exp/l2policy.cu, profiles/r02_ncu_summary.md): on this
  // part evict_last does not hold TMA-copied lines, the stream access-policy
  // window does not apply to TMA reads, but evict_first on everything that is
  // touched once per step does protect the rest.  On the gather-ordered twin
  // (hot_rows > 0: ids are degree ranks, rows list their hottest neighbours
  // first) a gather4 group whose four ids are all >= hot_rows is cold: cold
  // groups, the own rows of T_{k-1} / z, the col ids and the T_{k+1} stores
  // carry evict_first, groups with a hot row no hint.  One code path: the
  // stream operands always carry a policy, evict_normal when nothing is
  // protected (the caller's CSR order).
  uint64_t pol_first;
  if (p.hot_rows > 0) pol_first = l2_policy_first();
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_first));
  const uint32_t rows_sa = smem_u32(base);
  const uint32_t wv_sa = rows_sa + L::rows_d * 8;
  const uint32_t col_sa = wv_sa + L::wv_d * 8;
  const uint32_t own_sa = col_sa + L::col_d * 8;
  uint64_t *wbar = reinterpret_cast<uint64_t *>(base + L::warp_d - L::bar_d);
  uint64_t *obar = wbar + D;
  const uint32_t rbytes = (uint32_t)tw * 8u;  // one gathered row segment in shared memory

  int wb = r0;
  int64_t wrp = p.row_ptr[min(r0 + lane, r1)];
  double wdi = 0.0;
  if constexpr (!EXPL) wdi = (r0 + lane < r1) ? p.dinv[p.row0 + r0 + lane] : 0.0;
  auto refill = [&](int b) {
    wb = b;
    wrp = p.row_ptr[min(b + lane, r1)];
    if constexpr (!EXPL) wdi = (b + lane < r1) ? p.dinv[p.row0 + b + lane] : 0.0;
  };
  auto rp = [&](int r) { return __shfl_sync(0xffffffffu, wrp, r - wb); };
  const int64_t K0 = __shfl_sync(0xffffffffu, wrp, 0);
  const int64_t K1 = p.row_ptr[r1];
  const int nnz = (int)(K1 - K0);  // a light chunk holds < 2^31 nonzeros
  const int nw = (nnz + WAVE - 1) / WAVE;

  auto issue_own = [&](int r) {
    if (r >= r1) return;  // warp-uniform
    const int sl = (r - r0) & (R - 1);
    if (active) {
      const size_t off = (size_t)r * ld + c0;
      const uint32_t dst = own_sa + (uint32_t)(sl * NOP * W + lane * C) * 8;
      int q = 0;
      // the own row of T_k is also gathered by its neighbours: no hint
      if constexpr (EXPL || MODE == MODE_DBL) cp_async_cols<C>(dst + (q++) * W * 8, p.X + off);
      if constexpr (!FIRST) cp_async_cols_hint<C>(dst + (q++) * W * 8, p.Xprev + off, pol_first);
      if constexpr (MODE != MODE_DBL) cp_async_cols_hint<C>(dst + (q++) * W * 8, p.Z + off, pol_first);
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(obar + sl))
                 : "memory");
  };
  auto col_slot = [&](int w) { return col_sa + (uint32_t)((w % (2 * D)) * WAVE * 4); };
  auto issue_col = [&](int w) {
    const int e = w * WAVE + lane;
    if (lane < WAVE && e < nnz) cp_async_4_first(col_slot(w) + lane * 4, p.col + K0 + e, pol_first);
  };
  // wave w: rows by gather4 (lane 0), weights by lanes < cnt; the caller then
  // lets lanes < WAVE arrive (noinc) after also issuing col(w + D)
  auto issue_wave = [&](int w) {
    const uint32_t sl = (uint32_t)(w % D);
    const int cnt = min(WAVE, nnz - w * WAVE);
    const uint32_t ca = col_slot(w);
    const uint32_t bar = smem_u32(wbar + sl);
    // this lane's neighbour id (weights below); one ballot gives the elected
    // lane every group's "all four ids cold" test (ids past a chunk's last
    // nonzero vote hot: their group just goes unhinted)
    int jl = 0;
    if (lane < cnt) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(jl) : "r"(ca + lane * 4));
    const uint32_t cold_mask =
        __ballot_sync(0xffffffffu, p.hot_rows > 0 && lane < cnt && jl >= p.hot_rows);
    if (elect_one()) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the warp's reads of the slot
      int j[WAVE];
#pragma unroll
      for (int q = 0; q < WAVE / 4; ++q)
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(j[4 * q]), "=r"(j[4 * q + 1]), "=r"(j[4 * q + 2]), "=r"(j[4 * q + 3])
                     : "r"(ca + 16 * q));
      if (cnt < WAVE) {  // the chunk's last wave
#pragma unroll
        for (int k = 1; k < WAVE; ++k)
          if (k >= cnt) j[k] = j[0];  // a valid row; its bytes land unused
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)WAVE * rbytes)
                   : "memory");
      const uint32_t dst = rows_sa + sl * (uint32_t)(L::slot_d * 8);
      // gather-ordered twin: rows are sorted hottest-first, so whole groups
      // are cold (all four ids >= hot_rows) without any reordering
#pragma unroll
      for (int q = 0; q < WAVE / 4; ++q) {
        const bool cold = ((cold_mask >> (4 * q)) & 0xFu) == 0xFu;
        if (cold)
          tma_gather4_hint(dst + 4 * q * rbytes, tm, (int)col0, j[4 * q], j[4 * q + 1],
                           j[4 * q + 2], j[4 * q + 3], bar, pol_first);
        else
          tma_gather4(dst + 4 * q * rbytes, tm, (int)col0, j[4 * q], j[4 * q + 1],
                      j[4 * q + 2], j[4 * q + 3], bar);
      }
    }
    if (lane < cnt) {
      const uint32_t wd = wv_sa + (sl * WAVE + lane) * 8;
      if constexpr (EXPL) {
        cp_async_8(wd, p.vals + K0 + w * WAVE + lane);
      } else {
        if (jl >= p.dstep_h) {
          // twin: ids are degree ranks, so dinv is a step function of the id;
          // largest e with dstep_id[e] <= jl (dstep_id[0] = dstep_h), then the
          // same double the array holds
          uint32_t e = 0;
#pragma unroll
          for (int s = kDinvSteps / 2; s > 0; s >>= 1) {
            int t;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(t) : "r"(dtab_sa + (e + s) * 4));
            if (t <= jl) e += s;
          }
          double dv;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(dv) : "r"(dtab_sa + kDinvSteps * 4 + e * 8));
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(wd), "d"(dv) : "memory");
        } else {
          cp_async_8(wd, p.dinv + jl);
        }
      }
    }
  };
  auto arrive_wave = [&](int w) {
    if (lane < WAVE)
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                       smem_u32(wbar + (uint32_t)(w % D)))
                   : "memory");
  };

#pragma unroll
  for (int w = 0; w < 2 * D; ++w) issue_col(w);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) issue_own(r0 + r);
#pragma unroll
  for (int w = 0; w < D; ++w) {
    if (w < nw) {
      issue_wave(w);
      arrive_wave(w);
    }
  }

  int row = r0;
  if (row + 1 - wb > 31) refill(row);
  int64_t rend = rp(row + 1) - K0;
  double di = 0.0;
  if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  auto finish = [&](int r) {
    const int sl = (r - r0) & (R - 1);
    mbar_wait(obar + sl, (ophase >> sl) & 1u);
    ophase ^= 1u << sl;
    double xo[C], pv[C], zv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) xo[c] = pv[c] = zv[c] = 0.0;
    if (active) {
      const uint32_t a = own_sa + (uint32_t)(sl * NOP * W + lane * C) * 8;
      int q = 0;
      if constexpr (EXPL || MODE == MODE_DBL) lds_cols<C>(a + (q++) * W * 8, xo);
      if constexpr (!FIRST) lds_cols<C>(a + (q++) * W * 8, pv);
      if constexpr (MODE != MODE_DBL) lds_cols<C>(a + (q++) * W * 8, zv);
    }
    bulk_finish_row<C, MODE, EXPL, FIRST, true>(p, r, active, c0, acc, xo, pv, zv, s1, s2,
                                                pol_first);
    issue_own(r + R);
  };
  auto advance = [&](int64_t kk) {
    while (row < r1 && kk == rend) {
      finish(row);
      ++row;
      if (row >= r1) break;
      if (row + 1 - wb > 31) refill(row);
      rend = rp(row + 1) - K0;
      if constexpr (!EXPL) di = __shfl_sync(0xffffffffu, wdi, row - wb);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0.0;
    }
  };
  advance(0);

  const uint32_t my_col = (uint32_t)(active ? lane * C : 0) * 8u;
  for (int w = 0; w < nw; ++w) {
    const uint32_t sl = (uint32_t)(w % D);
    mbar_wait(wbar + sl, (wphase >> sl) & 1u);
    wphase ^= 1u << sl;
    if (p.dstep_h != 0x7fffffff) __syncwarp();  // table weights were plain shared stores
    const int e0 = w * WAVE;
    const int cnt = min(WAVE, nnz - e0);
    const uint32_t slot = rows_sa + sl * (uint32_t)(L::slot_d * 8) + my_col;
    const uint32_t wslot = wv_sa + sl * WAVE * 8;
    auto add_h = [&](int k, double h) {
      double v[C];
      lds_cols<C>(slot + k * rbytes, v);
#pragma unroll
      for (int c = 0; c < C; ++c)
        acc[c] = __dadd_rn(acc[c], __dmul_rn(h, v[c]));
    };
    auto add_one = [&](int k) {
      double wv;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wv) : "r"(wslot + k * 8));
      if constexpr (EXPL) add_h(k, wv);
      else add_h(k, __dmul_rn(di, wv));  // (1*dinv_i)*dinv_j, operators.py:110
    };
    if (cnt == WAVE && e0 + WAVE <= rend) {
      // the whole wave belongs to one row: each h_ij = dinv_i * dinv_j is
      // formed once (lane k for neighbour k, the same rounding) and broadcast
      // in pairs, instead of once per lane and neighbour
      if constexpr (!EXPL) {
        if (lane < WAVE) {
          double wk;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wk) : "r"(wslot + lane * 8));
          wk = __dmul_rn(di, wk);  // (1*dinv_i)*dinv_j, operators.py:110
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(wslot + lane * 8), "d"(wk) : "memory");
        }
        __syncwarp();
      }
#pragma unroll
      for (int k = 0; k < WAVE; k += 2) {
        double h0, h1;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(h0), "=d"(h1) : "r"(wslot + k * 8));
        add_h(k, h0);
        add_h(k + 1, h1);
      }
      advance(e0 + WAVE);
    } else {
      // row by row: the current row's nonzeros inside this wave without a
      // row-end test per nonzero (advance() left rend > e0 + k)
      int k = 0;
      while (k < cnt) {
        const int kend = max(k + 1, (int)min((int64_t)cnt, rend - e0));
        for (; k < kend; ++k) add_one(k);
        advance(e0 + k);
      }
    }
    __syncwarp();  // the whole warp is done with the slot and its weights
    if (w + D < nw) {
      issue_wave(w + D);
      issue_col(w + 2 * D);
      arrive_wave(w + D);
    }
  }
  advance(nnz);
  if constexpr (MODE != MODE_LDOS) {
    if (active) {
      double *out = p.partial + (size_t)chunk * 2 * ld + c0;
      st_vec<C>(out, s1);
      if constexpr (MODE == MODE_DBL) st_vec<C>(out + ld, s2);
    }
  }
}

template <int C, int MODE, bool EXPL, bool FIRST>
__global__ void __launch_bounds__(KPM_G4_THREADS, G4Tune<C>::minb)
kpm_step_g4_kernel(const StepParams p, const __grid_constant__ CUtensorMap tm) {
  using L = G4<C, MODE, EXPL, FIRST>;
  extern __shared__ __align__(128) double sg4[];
  // degree-step table of the twin: [kDinvSteps] int32 first ids, then the doubles
  __shared__ __align__(8) unsigned char s_dtab[kDinvSteps * 12];
  if (p.dstep_h != 0x7fffffff) {
    int32_t *did = reinterpret_cast<int32_t *>(s_dtab);
    double *dval = reinterpret_cast<double *>(s_dtab + kDinvSteps * 4);
    for (int e = threadIdx.x; e < kDinvSteps; e += blockDim.x) {
      did[e] = p.dstep_id[e];
      dval[e] = p.dstep_val[e];
    }
    __syncthreads();
  }
  const uint32_t dtab_sa = smem_u32(s_dtab);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double *base = sg4 + (size_t)warp * L::warp_d;
  uint64_t *wbar = reinterpret_cast<uint64_t *>(base + L::warp_d - L::bar_d);
  if (lane < L::D) mbar_init(wbar + lane, 1 + L::WAVE);
  else if (lane < L::D + L::R) mbar_init(wbar + lane, 32);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  uint32_t ophase = 0, wphase = 0;
  // light items: ntiles column tiles x n_chunks (tile-major); ntiles > 1 only
  // for the fused 64-column tiles of a 4-column layout (ld % 64 == 0)
  const int64_t total = p.n_heavy_tasks + (int64_t)p.ntiles * p.n_chunks;
  for (;;) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(p.queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if ((int64_t)item >= total) break;
    const unsigned long long t0 = p.trace ? gtimer() : 0;
    if ((int64_t)item < p.n_heavy_tasks) {
      heavy_task<MODE, EXPL, FIRST>(p, (int64_t)item, base);
    } else {
      const int64_t li = (int64_t)item - p.n_heavy_tasks;
      const int64_t t = li / p.n_chunks;
      const int chunk = p.chunk_order[li - t * p.n_chunks];
      // constant tile widths give the consumer immediate shared-memory offsets
      if (C == 2 && p.ntiles > 1)
        light_g4<C, MODE, EXPL, FIRST>(p, &tm, chunk, p.col0 + t * kTileW, kTileW, base,
                                            ophase, wphase, dtab_sa);
      else if (p.tw == 32 * C)
        light_g4<C, MODE, EXPL, FIRST>(p, &tm, chunk, p.col0, 32 * C, base, ophase, wphase,
                                       dtab_sa);
      else
        light_g4<C, MODE, EXPL, FIRST>(p, &tm, chunk, p.col0, p.tw, base, ophase, wphase,
                                       dtab_sa);
    }
    trace_item(p, item, t0);
  }
}

// Persistent fused step kernel.  Work items: [0, n_heavy_tasks) hub-row
// slices in degree-descending order, then the light row chunks.  Warps grab
// items from one atomic counter (dynamic load balance, hubs first); every item
// writes its own partial slot, so the reduction order is fixed by the graph
// alone -- independent of the schedule, the launch shape and the probe count.
// Occupancy / memory-level-parallelism per lane layout (tuned on B200 with
// tools/step_timer.py): resident 256-thread CTAs per SM and gathers in flight.
#ifndef KPM_MINB4
#define KPM_MINB4 3
#endif
#ifndef KPM_MINB2
#define KPM_MINB2 4
#endif
#ifndef KPM_MINB1
#define KPM_MINB1 3
#endif
#ifndef KPM_U4
#define KPM_U4 4
#endif
#ifndef KPM_U2
#define KPM_U2 4
#endif
#ifndef KPM_U1
#define KPM_U1 4
#endif
#ifndef KPM_STREAM_MAXC
#define KPM_STREAM_MAXC 2  // stream light chunks for the 1- and 2-column layouts
#endif
template <int C>
struct Tune {
  static constexpr int minb = C == 4 ? KPM_MINB4 : (C == 2 ? KPM_MINB2 : KPM_MINB1);
  static constexpr int u = C == 4 ? KPM_U4 : (C == 2 ? KPM_U2 : KPM_U1);
};

template <int C, int MODE, bool EXPL, bool FIRST, bool INIT, int U>
__global__ void __launch_bounds__(256, Tune<C>::minb)
kpm_step_kernel(const StepParams p) {
  extern __shared__ double sacc[];  // [W][2][ld] per-warp accumulators
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double *my = sacc + (size_t)warp * 2 * p.ld;
  const int64_t n_heavy_tasks = INIT ? 0 : p.n_heavy_tasks;
  const int64_t total = n_heavy_tasks + p.n_chunks;
  for (;;) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(p.queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if ((int64_t)item >= total) break;
    const unsigned long long t0 = p.trace ? gtimer() : 0;
    if constexpr (!INIT) {
      if ((int64_t)item < n_heavy_tasks) {
        heavy_task<MODE, EXPL, FIRST>(p, (int64_t)item, sacc + p.hub_off + (size_t)warp * kHubRingDoubles);
        trace_item(p, item, t0);
        continue;
      }
    }
    const int chunk = p.chunk_order[(int64_t)item - n_heavy_tasks];
    if constexpr (!INIT) {
      if constexpr (C <= KPM_STREAM_MAXC) {
        if (p.stream && p.ld <= 32 * C) {
          light_stream<C, MODE, EXPL, FIRST, U>(p, chunk, my);
          trace_item(p, item, t0);
          continue;
        }
      }
    }
    light_chunk<C, MODE, EXPL, FIRST, INIT, U>(p, chunk, my);
    trace_item(p, item, t0);
  }
}

// Level 1 of the deterministic reduction: consecutive groups of kGroup chunk
// partials summed in chunk order.
constexpr int kGroup = 32;

__global__ void reduce_groups_kernel(const double *__restrict__ partial, int n_chunks,
                                     int64_t ld, int64_t k, int nred,
                                     double *__restrict__ gpart) {
  const int64_t n_groups = (n_chunks + kGroup - 1) / kGroup;
  const int64_t per = nred * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_groups * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / per, e = t % per;
    const int red = (int)(e / k);
    const int64_t c = e % k;
    const int ch1 = (int)min((int64_t)n_chunks, (g + 1) * kGroup);
    double s = 0.0;
    for (int ch = (int)(g * kGroup); ch < ch1; ++ch)
      s = __dadd_rn(s, partial[(size_t)ch * 2 * ld + red * ld + c]);
    gpart[(size_t)g * 2 * ld + red * ld + c] = s;
  }
}

// Level 2: groups (then hub rows) in fixed order -> contrib rows.
//   which = 0: INIT       contrib[0] = S1
//   which = 1: DIRECT     contrib[m] = S1
//   which = 2: DBL step s contrib[2s-1] = 2 S1 - mu_1 (s==1: S1),
//                         contrib[2s]   = 2 S2 - mu_0     (if 2s <= M)
__global__ void finalize_kernel(const double *__restrict__ gpart, int n_groups,
                                const double *__restrict__ hpart, int n_heavy, int64_t ld,
                                int64_t k, int which, int m, int m_max, int raw,
                                double *__restrict__ contrib) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int nred = which == 2 ? 2 : 1;
  if (gw >= nred * k) return;
  const int red = (int)(gw / k);
  const int64_t c = gw % k;
  double s = 0.0;
  for (int g = lane; g < n_groups; g += 32)
    s = __dadd_rn(s, gpart[(size_t)g * 2 * ld + red * ld + c]);
  s = warp_sum_fixed(s);
  if (n_heavy > 0) {  // hub rows after the chunks, in hub-list order
    double sh = 0.0;
    for (int hh = lane; hh < n_heavy; hh += 32)
      sh = __dadd_rn(sh, hpart[(size_t)hh * 2 * ld + red * ld + c]);
    s = __dadd_rn(s, warp_sum_fixed(sh));
  }
  if (lane != 0) return;
  if (which == 0) {
    contrib[c] = s;
  } else if (which == 1) {
    contrib[(size_t)m * ld + c] = s;
  } else {
    if (red == 0) {
      const int row = 2 * m - 1;
      if (row <= m_max)
        contrib[(size_t)row * ld + c] =
            (m == 1 || raw) ? s : __dsub_rn(__dmul_rn(2.0, s), contrib[ld + c]);
    } else {
      const int row = 2 * m;
      if (row <= m_max)
        contrib[(size_t)row * ld + c] = raw ? s : __dsub_rn(__dmul_rn(2.0, s), contrib[c]);
    }
  }
}

// LDOS hub rows: sum the per-slice partials in slice order.
__global__ void ldos_heavy_kernel(const double *__restrict__ hldos, const int32_t *rows,
                                  int n_heavy, int nsl, double *ldos, int64_t stride,
                                  int col, int32_t *flag, const int32_t *perm) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_heavy) return;
  double s = hldos[(size_t)h * nsl];
  for (int q = 1; q < nsl; ++q) s = __dadd_rn(s, hldos[(size_t)h * nsl + q]);
  if (!isfinite(s)) atomicOr(flag, 1);
  ldos[(size_t)(perm ? perm[rows[h]] : rows[h]) * stride + col] = s;
}

// ---------------------------------------------------------------- dispatch
template <typename K>
static int resident_blocks(K kern, size_t smem) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 256, smem) != cudaSuccess ||
      nb < 1) {
    cudaGetLastError();
    nb = 1;
  }
  return nb;
}

template <int C, int MODE>
static cudaError_t launch_bulk(const kpm_run *r, const StepParams &p, bool expl, bool first,
                               cudaStream_t st) {
  constexpr int kBulkSlots = BulkShape<C>::slots;
  void (*kern)(StepParams);
  if (expl && first) kern = kpm_step_bulk_kernel<C, MODE, true, true>;
  else if (expl) kern = kpm_step_bulk_kernel<C, MODE, true, false>;
  else if (first) kern = kpm_step_bulk_kernel<C, MODE, false, true>;
  else kern = kpm_step_bulk_kernel<C, MODE, false, false>;
  const int threads = KPM_BULK_THREADS;
  const size_t per_warp = bulk_data_doubles(kBulkSlots, p.ld, p.n_heavy_tasks > 0) + kBulkSlots;
  const size_t smem = (size_t)(threads / 32) * per_warp * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t items = p.n_chunks + p.n_heavy_tasks;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess ||
      nb < 1) {
    cudaGetLastError();
    nb = 1;
  }
  int64_t grid = (int64_t)r->g->ctx->sm_count * nb;
  const int64_t need = (items + threads / 32 - 1) / (threads / 32);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  e = cudaMemsetAsync(p.queue, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, threads, smem, st>>>(p);
  return cudaGetLastError();
}

template <int C, int MODE, bool EXPL, bool FIRST>
static cudaError_t launch_lean_k(const kpm_run *r, const StepParams &p, cudaStream_t st) {
  void (*kern)(StepParams) = kpm_step_lean_kernel<C, MODE, EXPL, FIRST>;
  const int threads = 256;
  const size_t smem = (size_t)(threads / 32) * Lean<C, MODE, EXPL, FIRST>::warp_d * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t items = p.n_chunks + p.n_heavy_tasks;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess ||
      nb < 1) {
    cudaGetLastError();
    nb = 1;
  }
  int64_t grid = (int64_t)r->g->ctx->sm_count * nb;
  const int64_t need = (items + threads / 32 - 1) / (threads / 32);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  e = cudaMemsetAsync(p.queue, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, threads, smem, st>>>(p);
  return cudaGetLastError();
}

template <int C, int MODE, bool EXPL, bool FIRST>
static cudaError_t launch_g4_k(const kpm_run *r, const StepParams &p, const CUtensorMap &tm,
                               cudaStream_t st) {
  void (*kern)(StepParams, CUtensorMap) = kpm_step_g4_kernel<C, MODE, EXPL, FIRST>;
  const int threads = KPM_G4_THREADS;  // warps are independent; CTA size sets smem granularity
  const size_t smem = (size_t)(threads / 32) * G4<C, MODE, EXPL, FIRST>::warp_d * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t items = (int64_t)p.ntiles * p.n_chunks + p.n_heavy_tasks;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess ||
      nb < 1) {
    cudaGetLastError();
    nb = 1;
  }
  int64_t grid = (int64_t)r->g->ctx->sm_count * nb;
  const int64_t need = (items + threads / 32 - 1) / (threads / 32);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  e = cudaMemsetAsync(p.queue, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, threads, smem, st>>>(p, tm);
  return cudaGetLastError();
}

template <int C, int MODE>
static cudaError_t launch_g4(const kpm_run *r, const StepParams &p, bool expl, bool first,
                             const CUtensorMap &tm, cudaStream_t st) {
  if (expl && first) return launch_g4_k<C, MODE, true, true>(r, p, tm, st);
  if (expl) return launch_g4_k<C, MODE, true, false>(r, p, tm, st);
  if (first) return launch_g4_k<C, MODE, false, true>(r, p, tm, st);
  return launch_g4_k<C, MODE, false, false>(r, p, tm, st);
}

template <int C, int MODE>
static cudaError_t launch_lean(const kpm_run *r, const StepParams &p, bool expl, bool first,
                               cudaStream_t st) {
  if (expl && first) return launch_lean_k<C, MODE, true, true>(r, p, st);
  if (expl) return launch_lean_k<C, MODE, true, false>(r, p, st);
  if (first) return launch_lean_k<C, MODE, false, true>(r, p, st);
  return launch_lean_k<C, MODE, false, false>(r, p, st);
}

template <int C, int MODE, bool INIT>
static cudaError_t launch_c(const kpm_run *r, const StepParams &p, bool expl, bool first,
                            cudaStream_t st) {
  if constexpr (!INIT) {
    const int blk = p.X == r->a ? 0 : (p.X == r->b ? 1 : -1);
    // the 4-column layout of the global modes as 64-column gather4 passes over
    // the same row-major blocks: smaller gathered segments keep twice the rows
    // in L2 and run 24 warps per SM (C3: 2 x 32.2 ms vs 70.0 ms per step);
    // every column's sums are unchanged, so the results are bitwise the same
    if (C == 4 && MODE != MODE_LDOS && p.tile && p.g4 && r->tm_tile_ok && p.nparts <= 1 &&
        blk >= 0) {
      if (p.fuse_tiles && p.ld % kTileW == 0) {
        // one launch over every tile: hub slices span the full width, light
        // items are (tile, chunk) pairs, so the second tile's chunks fill the
        // first tile's tail
        StepParams q = p;
        q.ntiles = (int)(p.ld / kTileW);
        return launch_g4<2, MODE>(r, q, expl, first, r->tm[blk][1], st);
      }
      for (int64_t t0 = 0; t0 < p.ld; t0 += 64) {
        StepParams q = p;
        q.col0 = t0;
        q.tw = p.ld - t0 < 64 ? p.ld - t0 : 64;
        q.n_heavy_tasks = (int64_t)p.n_heavy * ((q.tw + kSlice - 1) / kSlice);
        cudaError_t e = launch_g4<2, MODE>(r, q, expl, first, r->tm[blk][q.tw == 64 ? 1 : 2], st);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
    // TMA gather4 for one column tile (tensor maps of both blocks encoded)
    if (p.ld <= 32 * C && p.g4 >= (C == 4 ? 2 : 1) && r->tm_ok && p.nparts <= 1 && blk >= 0)
      return launch_g4<C, MODE>(r, p, expl, first, r->tm[blk][0], st);
  }
  if constexpr (!INIT && C <= 2) {
    // per-lane async gathers for one column tile of 1 or 2 columns per lane
    if (p.ld <= 32 * C && p.lean) return launch_lean<C, MODE>(r, p, expl, first, st);
  }
  if constexpr (!INIT) {
    // bulk-copy gathers for a single column tile; KPM_BULK: 0 off, 1 the
    // 4-column layout only, 2 every layout (default)
    // (bulk copies move multiples of 16 B: rows of an even number of doubles;
    // row-partitioned runs gather peer GPUs' blocks with plain loads -- the
    // bulk path is only exercised single-device here)
    if (p.ld <= 32 * C && (p.ld & 1) == 0 && p.nparts <= 1 &&
        (C == 4 ? p.bulk >= 1 : p.bulk >= 2))
      return launch_bulk<C, MODE>(r, p, expl, first, st);
  }
  constexpr int U = Tune<C>::u;
  const int threads = 256;
  size_t smem = (MODE == MODE_LDOS) ? 0 : (size_t)(threads / 32) * 2 * p.ld * sizeof(double);
  StepParams q = p;  // + one hub ring per warp after the accumulators
  q.hub_off = (int64_t)(smem / sizeof(double));
  if (!INIT && p.n_heavy_tasks > 0) smem += (size_t)(threads / 32) * kHubRingDoubles * sizeof(double);
  void (*kern)(StepParams);
  if (INIT) kern = kpm_step_kernel<C, MODE, false, true, true, U>;
  else if (expl && first) kern = kpm_step_kernel<C, MODE, true, true, false, U>;
  else if (expl) kern = kpm_step_kernel<C, MODE, true, false, false, U>;
  else if (first) kern = kpm_step_kernel<C, MODE, false, true, false, U>;
  else kern = kpm_step_kernel<C, MODE, false, false, false, U>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int64_t items = p.n_chunks + (INIT ? 0 : p.n_heavy_tasks);
  int64_t grid = (int64_t)r->g->ctx->sm_count * resident_blocks(kern, smem);
  const int64_t need = (items + 7) / 8;  // 8 warps per CTA
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  cudaError_t e = cudaMemsetAsync(p.queue, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, threads, smem, st>>>(q);
  return cudaGetLastError();
}

template <int MODE, bool INIT>
static cudaError_t launch_mode(const kpm_run *r, const StepParams &p, bool expl, bool first,
                               cudaStream_t st) {
  switch (r->cpl) {
    case 1: return launch_c<1, MODE, INIT>(r, p, expl, first, st);
    case 2: return launch_c<2, MODE, INIT>(r, p, expl, first, st);
    default: return launch_c<4, MODE, INIT>(r, p, expl, first, st);
  }
}

static cudaError_t launch_step(const kpm_run *r, const StepParams &p, bool init,
                               bool first, cudaStream_t st) {
  const bool expl = r->g->values != nullptr;
  if (r->g->n_chunks == 0) return cudaSuccess;
  switch (r->mode) {
    case KPM_MODE_DOS_DOUBLING:
      return init ? launch_mode<MODE_DBL, true>(r, p, expl, first, st)
                  : launch_mode<MODE_DBL, false>(r, p, expl, first, st);
    case KPM_MODE_DOS_DIRECT:
      return init ? launch_mode<MODE_DIRECT, true>(r, p, expl, first, st)
                  : launch_mode<MODE_DIRECT, false>(r, p, expl, first, st);
    default:
      return init ? launch_mode<MODE_LDOS, true>(r, p, expl, first, st)
                  : launch_mode<MODE_LDOS, false>(r, p, expl, first, st);
  }
}

static StepParams base_params(const kpm_run *r) {
  StepParams p{};
  const kpm_graph *g = r->g;
  p.row_ptr = g->row_ptr;
  p.col = g->col_idx;
  p.dinv = g->dinv_all ? g->dinv_all : g->dinv;
  p.row0 = g->row0;
  p.nparts = r->nparts > 1 ? r->nparts : 1;
  for (int q = 0; q <= kMaxParts; ++q) p.part_lo[q] = q <= r->nparts ? r->part_lo[q] : 0;
  p.vals = g->values;
  p.shift = g->shift;
  p.scale = g->scale;
  p.Z = r->z;
  p.den = r->den;
  p.ldos = r->ldos;
  p.ldos_stride = r->m_max + 1;
  p.ldos_raw = (r->flags & KPM_LDOS_RAW) != 0;
  p.ld = r->ld;
  p.chunk_start = g->chunk_start;
  p.chunk_order = g->chunk_order;
  p.n_chunks = g->n_chunks;
  p.partial = r->partial;
  p.flag = r->flag;
  p.queue = r->queue;
  p.heavy_rows = g->heavy_rows;
  p.n_heavy = g->n_heavy;
  p.heavy_threshold = g->heavy_threshold;
  const int64_t nsl = (r->ld + kSlice - 1) / kSlice;
  p.n_heavy_tasks = g->n_heavy * nsl;
  p.hpart = r->hpart;
  p.hldos = r->hldos;
  p.stream = 1;
  if (const char *e = getenv("KPM_STREAM")) p.stream = atoi(e);
  p.col0 = 0;
  p.tw = r->ld;
  p.tile = 1;  // 4-column layouts (DOS modes) as 64-column gather4 passes (KPM_TILE=0: off)
  if (const char *e = getenv("KPM_TILE")) p.tile = atoi(e);
  p.g4 = 1;  // TMA gather4 light path for the 1- and 2-column layouts (KPM_G4=2: also 4)
  if (const char *e = getenv("KPM_G4")) p.g4 = atoi(e);
  p.lean = 1;  // per-lane async gathers for the 1- and 2-column layouts (KPM_LEAN=0: off)
  if (const char *e = getenv("KPM_LEAN")) p.lean = atoi(e);
  p.ntiles = 1;
  p.fuse_tiles = 1;  // 64-column tiles of one step in one launch (KPM_FUSE_TILES=0: per tile)
  if (const char *e = getenv("KPM_FUSE_TILES")) p.fuse_tiles = atoi(e);
  p.bulk = 2;  // bulk-copy gathers in every layout (KPM_BULK=1: 4-column only, 0: none)
  if (const char *e = getenv("KPM_BULK")) p.bulk = atoi(e);
  // hot rows (L2 evict_last in the bulk path): the highest-degree rows whose
  // T_k rows fill at most kHotBytes of L2, by power-of-two degree class;
  // KPM_HOT_DEGREE=<d> overrides (0 disables)
  p.hot_dinv = -1.0;
  {
    double kHotBytes = 64.0 * 1024 * 1024;
    if (const char *e = getenv("KPM_HOT_MB")) kHotBytes = atof(e) * 1024 * 1024;
    const double budget = kHotBytes / (8.0 * (double)r->ld);
    double rows = 0.0, hot_deg = 0.0;
    for (int b = kDegBuckets - 1; b >= 0; --b) {
      rows += (double)g->deg_hist[b];
      if (rows > budget) break;
      hot_deg = deg_bucket_lo(b);
    }
    if (const char *e = getenv("KPM_HOT_DEGREE")) hot_deg = atof(e);
    if (hot_deg > 0) p.hot_dinv = 1.0 / sqrt(hot_deg);
  }
  // gather-ordered twin: the hottest rows (lowest new ids) stay unhinted, every
  // other gather is evict_first (profiles/r02_ncu_summary.md: flat between 100k and 400k rows)
  p.perm = g->perm;
  p.dstep_id = g->dstep_id;
  p.dstep_val = g->dstep_val;
  p.dstep_h = 0x7fffffff;
  if (g->dstep_id && g->dstep_val) {
    p.dstep_h = g->dstep_h;
    if (const char *e = getenv("KPM_DINV_TABLE")) {
      if (atoi(e) == 0) p.dstep_h = 0x7fffffff;
    }
  }
  p.hot_rows = 0;
  if (g->perm) {
    p.hot_rows = 250000;
    if (const char *e = getenv("KPM_HOT_ROWS")) p.hot_rows = atoi(e);
    if (p.hot_rows > g->n) p.hot_rows = (int)g->n;
  }
  return p;
}

static cudaError_t launch_finalize(const kpm_run *r, int which, int m, cudaStream_t st) {
  const int nred = which == 2 ? 2 : 1;
  if (r->g->n_chunks == 0) return cudaSuccess;
  const int n_groups = (r->g->n_chunks + kGroup - 1) / kGroup;
  const int64_t work = (int64_t)n_groups * nred * r->k;
  int64_t b1 = (work + 255) / 256;
  if (b1 > 148 * 16) b1 = 148 * 16;
  reduce_groups_kernel<<<(unsigned)b1, 256, 0, st>>>(r->partial, r->g->n_chunks, r->ld, r->k,
                                                      nred, r->gpart);
  const int64_t warps = nred * r->k;
  const int64_t blocks = (warps * 32 + 255) / 256;
  const int nh = which == 0 ? 0 : r->g->n_heavy;
  finalize_kernel<<<(unsigned)blocks, 256, 0, st>>>(r->gpart, n_groups, r->hpart, nh, r->ld,
                                                     r->k, which, m, r->m_max,
                                                     r->partitioned ? 1 : 0, r->contrib);
  return cudaGetLastError();
}

// ----------------------------------------------------------- probes (K0)
// numpy Philox4x64-10 (Random123 constants) for make_probes(RADEMACHER).
__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
}

// Element i of a column is bit 31 of the i-th 32-bit half-word of the
// column's Philox stream (numpy: integers(0, 2) -> Lemire on next_uint32,
// low half first; counter incremented before each 4-word block).
// Rows [row0, row0+n) of the columns (global row i -> local row i - row0).
__global__ void rademacher_kernel(int64_t n, int64_t ncols, const uint64_t *__restrict__ keys,
                                  double *__restrict__ z, int64_t ldz, int64_t col0,
                                  int64_t row0, const int32_t *__restrict__ iperm = nullptr) {
  const int64_t b0 = row0 / 8, nblk = (row0 + n + 7) / 8 - b0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nblk * ncols;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = b0 + t / ncols, j = t % ncols;
    uint64_t c[4] = {(uint64_t)b + 1, 0, 0, 0};
    philox4x64_10(c, keys[2 * j], keys[2 * j + 1]);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t i = b * 8 + q - row0;
      if (i >= 0 && i < n) {
        const uint32_t half = (q & 1) ? (uint32_t)(c[q >> 1] >> 32) : (uint32_t)c[q >> 1];
        const int64_t io = iperm ? (int64_t)iperm[i] : i;  // row of a run on the twin
        z[io * ldz + col0 + j] = (half >> 31) ? -1.0 : 1.0;
      }
    }
  }
}

// rows of a block between the caller's order and the twin's: out[r] = in[perm[r]]
// (gather) or out[perm[r]] = in[r] (scatter), ld doubles per row
__global__ void permute_rows_kernel(const double *__restrict__ in, double *__restrict__ out,
                                    const int32_t *__restrict__ perm, int64_t n, int64_t ld,
                                    int scatter) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * ld;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ld, c = t - r * ld;
    const int64_t o = perm[r];
    if (scatter) out[o * ld + c] = in[t];
    else out[t] = in[o * ld + c];
  }
}

// kpm.py:145-147: the first node with zero probe mass (den == 0)
__global__ void first_zero_kernel(const double *__restrict__ den, int64_t n, int32_t *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (den[i] == 0.0) atomicMin(flag, (int32_t)i);
}

// dst += src (raw per-node sums of two probe batches / GPU shards)
__global__ void add_inplace_kernel(double *__restrict__ dst, const double *__restrict__ src,
                                   int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __dadd_rn(dst[i], src[i]);
}

__global__ void or_flag_kernel(int32_t *dst, const int32_t *src) { dst[0] |= src[0]; }
__global__ void set_i32_kernel(int32_t *dst, int32_t v) { dst[0] = v; }

// kpm.py:148-150: values = (num / den).T, or num * trace_scale (raw); the
// num array is already node-major (n, M+1).
__global__ void ldos_finish(double *__restrict__ v, const double *__restrict__ den,
                            int64_t n, int64_t stride, int raw, double ts) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * stride;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[t];
    v[t] = raw ? __dmul_rn(x, ts) : __ddiv_rn(x, den[t / stride]);
  }
}

__global__ void zero_pad_cols(double *z, int64_t n, int64_t k, int64_t ld) {
  const int64_t w = ld - k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * w;
       t += (int64_t)gridDim.x * blockDim.x)
    z[(t / w) * ld + k + t % w] = 0.0;
}

static int grid_of(int64_t work) {
  int64_t b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

// ------------------------------------------- standalone SpMM (L0 drop-in)
// _spmv.pyx:11-22: out[i,c] = 0; out[i,c] += data[jj]*x[j,c] in stored order.
__global__ void csr_matvec_kernel(int64_t n_rows, const int64_t *__restrict__ indptr,
                                  const int64_t *__restrict__ indices,
                                  const double *__restrict__ data,
                                  const double *__restrict__ x, int64_t k,
                                  double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nw) {
    const int64_t beg = indptr[i], end = indptr[i + 1];
    for (int64_t c0 = 0; c0 < k; c0 += 32) {
      const int64_t c = c0 + lane;
      double acc = 0.0;
      for (int64_t base = beg; base < end; base += 32) {
        const int cnt = (int)min((int64_t)32, end - base);
        int64_t jl = 0;
        double wl = 0.0;
        if (lane < cnt) {
          jl = indices[base + lane];
          wl = data[base + lane];
        }
        for (int q = 0; q < cnt; ++q) {
          const int64_t j = __shfl_sync(0xffffffffu, jl, q);
          const double w = __shfl_sync(0xffffffffu, wl, q);
          if (c < k) acc = __dadd_rn(acc, __dmul_rn(w, x[j * k + c]));
        }
      }
      if (c < k) out[i * k + c] = acc;
    }
  }
}

// ------------------------------------------ motif projection (K7)
// motifs.py:400-403 per vector, groups of disjoint support in parallel.
__global__ void filter_kernel(double *__restrict__ z, int64_t k, int64_t ldz,
                              int64_t n_groups, const int64_t *__restrict__ gptr,
                              const int64_t *__restrict__ vptr,
                              const int64_t *__restrict__ vidx,
                              const double *__restrict__ vval) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < n_groups;
       g += nw) {
    for (int64_t vec = gptr[g]; vec < gptr[g + 1]; ++vec) {
      const int64_t s0 = vptr[vec], s1 = vptr[vec + 1];
      for (int64_t c = lane; c < k; c += 32) {
        // coeff = val @ cols[idx] (sequential over the support)
        double coeff = 0.0;
        for (int64_t t = s0; t < s1; ++t)
          coeff = __dadd_rn(coeff, __dmul_rn(vval[t], z[vidx[t] * ldz + c]));
        // cols[idx] -= outer(val, coeff)
        for (int64_t t = s0; t < s1; ++t) {
          double *zz = z + vidx[t] * ldz + c;
          *zz = __dsub_rn(*zz, __dmul_rn(vval[t], coeff));
        }
      }
    }
  }
}

}  // namespace kpm

using namespace kpm;

// Tensor maps of the recurrence blocks for the gather4 path: n x ld fp64,
// row stride 8*ld, box ld x 1 (ld <= 128, a multiple of 4).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static void encode_block_maps(kpm_run *r) {
  r->tm_ok = false;
  const kpm_graph *g = r->g;
  // ld % 4 == 0 keeps the second gather4 of a wave 128-byte aligned in shared memory
  if (g->n < 1 || g->n >= (int64_t)1 << 31 || (r->ld & 3) || r->ld > 128 || !r->a || !r->b) return;
  static EncodeTiledFn enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      enc = nullptr;
    cudaGetLastError();
  }
  if (!enc) return;
  const cuuint64_t dims[2] = {(cuuint64_t)r->ld, (cuuint64_t)g->n};
  const cuuint64_t strides[1] = {(cuuint64_t)r->ld * sizeof(double)};
  const cuuint32_t es[2] = {1, 1};
  double *blk[2] = {r->a, r->b};
  // box widths: [0] the whole row, [1] a 64-column tile, [2] the last partial tile
  const cuuint32_t widths[3] = {(cuuint32_t)r->ld, 64, (cuuint32_t)(r->ld % 64)};
  auto encode = [&](int q, int kind) {
    const cuuint32_t box[2] = {widths[kind], 1};
    return enc(&r->tm[q][kind], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, blk[q], dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  bool ok = true, tile_ok = r->ld > 64;
  for (int q = 0; q < 2; ++q) {
    ok = ok && encode(q, 0);
    if (tile_ok) tile_ok = encode(q, 1) && (widths[2] == 0 || encode(q, 2));
  }
  r->tm_ok = ok;
  r->tm_tile_ok = ok && tile_ok;
}

extern "C" {

// Large implicit graphs step on the gather-ordered twin (kpm_graph::relab):
// rows renumbered by degree, each row's neighbours hottest-first, so the
// popular rows of T_k stay in L2 (evict_first on everything else).  A row's
// sum then adds its neighbours in that order instead of ascending original
// id -- deterministic and independent of the probe count, but not the
// reference's rounding sequence; KPM_REORDER=0 keeps the reference's order
// (bit-identical T_k), KPM_REORDER=1 forces the twin.  Default: when one
// gathered column tile of T_k is >= 32x the L2.
static kpm_graph *stepping_graph(kpm_graph *g, int64_t k) {
  int want = -1;
  if (const char *e = getenv("KPM_REORDER")) want = atoi(e);
  const int cpl = k <= 32 ? 1 : (k <= 64 ? 2 : 4);
  const int64_t ld = (k + cpl - 1) / cpl * cpl;
  const double seg = (double)(cpl == 4 ? (ld < kTileW ? ld : kTileW) : ld);
  const bool big = 8.0 * seg * (double)g->n >= 32.0 * (double)g->ctx->l2_bytes;
  if (want == 1 || (want < 0 && big)) {
    if (kpm_graph *t = kpm::graph_relabelled(g)) return t;
  }
  return g;
}

int kpm_graph_prepare(kpm_graph *g, int64_t k, int32_t *twin) {
  KPM_CHECK_ARG(g && k >= 1, "bad arguments");
  KPM_CUDA(cudaSetDevice(g->ctx->device));
  kpm_graph *s = stepping_graph(g, k);
  if (twin) *twin = s != g ? 1 : 0;
  return KPM_OK;
}

int kpm_run_create(kpm_graph *g, int64_t k, int32_t mode, int32_t m_max,
                   int32_t flags, kpm_run **out) {
  KPM_CHECK_ARG(g && out, "bad arguments");
  KPM_CHECK_ARG(k >= 1, "need at least one probe column");
  KPM_CHECK_ARG(m_max >= 0, "m_max must be >= 0");
  KPM_CHECK_ARG(mode >= 0 && mode <= 2, "unknown mode %d", mode);
  KPM_CHECK_ARG(k <= 1024 || mode == KPM_MODE_LDOS,
                "at most 1024 probe columns per batch (got %lld)", (long long)k);
  KPM_CHECK_ARG(g->n_global == g->n || g->dinv_all || g->values,
                "partition graph needs kpm_graph_set_dinv first");
  KPM_CUDA(cudaSetDevice(g->ctx->device));
  kpm_run *r = new kpm_run();
  r->user_g = g;
  r->k = k;
  r->cpl = k <= 32 ? 1 : (k <= 64 ? 2 : 4);
  r->ld = (k + r->cpl - 1) / r->cpl * r->cpl;
  g = stepping_graph(g, k);
  r->g = g;
  r->mode = mode;
  r->m_max = m_max;
  r->flags = flags;
  r->total_steps = mode == KPM_MODE_DOS_DOUBLING ? (m_max + 1) / 2 : m_max;
  const size_t blk = sizeof(double) * (size_t)(g->n > 0 ? g->n : 1) * r->ld;
  cudaError_t e = cudaSuccess;
  auto A = [&](void **p, size_t b) { if (e == cudaSuccess) e = cudaMalloc(p, b); };
  A((void **)&r->a, blk);
  if (m_max >= 1) A((void **)&r->b, blk);
  if (mode != KPM_MODE_DOS_DOUBLING) A((void **)&r->z, blk);
  A((void **)&r->flag, sizeof(int32_t) * 4);
  A((void **)&r->queue, sizeof(unsigned long long));
  const int64_t nh = g->n_heavy > 0 ? g->n_heavy : 1;
  if (mode == KPM_MODE_LDOS) A((void **)&r->hldos, sizeof(double) * nh * ((r->ld + kSlice - 1) / kSlice));
  else A((void **)&r->hpart, sizeof(double) * nh * 2 * r->ld);
  if (mode == KPM_MODE_LDOS) {
    A((void **)&r->ldos, sizeof(double) * (size_t)(g->n > 0 ? g->n : 1) * (m_max + 1));
    A((void **)&r->den, sizeof(double) * (size_t)(g->n > 0 ? g->n : 1));
  } else {
    A((void **)&r->partial, sizeof(double) * (size_t)(g->n_chunks > 0 ? g->n_chunks : 1) * 2 * r->ld);
    A((void **)&r->gpart,
      sizeof(double) * (size_t)((g->n_chunks + 31) / 32 + 1) * 2 * r->ld);
    A((void **)&r->contrib, sizeof(double) * (size_t)(m_max + 1) * r->ld);
  }
  if (e == cudaSuccess) encode_block_maps(r);
  if (e != cudaSuccess) {
    cudaGetLastError();
    kpm_run_free(r);
    set_error("run allocation failed: %s", cudaGetErrorString(e));
    return KPM_ENOMEM;
  }
  *out = r;
  return KPM_OK;
}

static int run_after_probes(kpm_run *r) {
  cudaStream_t st = r->g->ctx->stream;
  const kpm_graph *g = r->g;
  if (r->ld > r->k && g->n > 0)
    zero_pad_cols<<<grid_of(g->n * (r->ld - r->k)), 256, 0, st>>>(r->a, g->n, r->k, r->ld);
  if (r->z && g->n > 0)
    KPM_CUDA(cudaMemcpyAsync(r->z, r->a, sizeof(double) * g->n * r->ld,
                             cudaMemcpyDeviceToDevice, st));
  int32_t init_flag[4] = {0, 0x7fffffff, 0, 0};
  KPM_CUDA(cudaMemcpyAsync(r->flag, init_flag, sizeof(init_flag), cudaMemcpyHostToDevice, st));
  if (r->contrib)
    KPM_CUDA(cudaMemsetAsync(r->contrib, 0, sizeof(double) * (r->m_max + 1) * r->ld, st));
  StepParams p = base_params(r);
  p.X = r->a;
  p.ldos_col = 0;
  KPM_CUDA(launch_step(r, p, true, true, st));
  if (r->mode != KPM_MODE_LDOS) KPM_CUDA(launch_finalize(r, 0, 0, st));
  KPM_CUDA(cudaStreamSynchronize(st));  // init_flag lives on this stack
  r->cur = r->a;
  r->prev = nullptr;
  r->k_index = 0;
  r->done_steps = 0;
  r->have_probes = true;
  r->finished = false;
  return KPM_OK;
}

int kpm_run_set_probes(kpm_run *r, const double *z, int64_t ldz) {
  kpm::Nvtx nvtx_range_("kpm_run_set_probes");
  KPM_CHECK_ARG(r && (z || r->g->n == 0), "bad arguments");
  KPM_CHECK_ARG(ldz >= r->k, "ldz < k");
  KPM_CUDA(cudaSetDevice(r->g->ctx->device));
  cudaStream_t st = r->g->ctx->stream;
  if (r->g->n > 0 && r->g->perm) {
    // the caller's rows -> the twin's order, staged through T_1's block
    double *tmp = r->b;
    if (!tmp) KPM_CUDA(cudaMalloc(&tmp, sizeof(double) * (size_t)r->g->n * r->ld));
    KPM_CUDA(cudaMemcpy2DAsync(tmp, sizeof(double) * r->ld, z, sizeof(double) * ldz,
                               sizeof(double) * r->k, r->g->n, cudaMemcpyDefault, st));
    permute_rows_kernel<<<grid_of(r->g->n * r->ld), 256, 0, st>>>(tmp, r->a, r->g->perm, r->g->n,
                                                                 r->ld, 0);
    KPM_CUDA(cudaGetLastError());
    if (!r->b) {
      KPM_CUDA(cudaStreamSynchronize(st));
      cudaFree(tmp);
    }
  } else if (r->g->n > 0) {
    KPM_CUDA(cudaMemcpy2DAsync(r->a, sizeof(double) * r->ld, z, sizeof(double) * ldz,
                               sizeof(double) * r->k, r->g->n, cudaMemcpyDefault, st));
  }
  return run_after_probes(r);
}

int kpm_run_set_rademacher(kpm_run *r, const uint64_t *keys) {
  kpm::Nvtx nvtx_range_("kpm_run_set_rademacher");
  KPM_CHECK_ARG(r && keys, "bad arguments");
  KPM_CUDA(cudaSetDevice(r->g->ctx->device));
  cudaStream_t st = r->g->ctx->stream;
  DevBuf tk;
  const void *dk;
  KPM_TRY(stage_in(st, keys, sizeof(uint64_t) * 2 * r->k, tk, &dk));
  const int64_t n = r->g->n;
  if (n > 0)
    rademacher_kernel<<<grid_of(((n + 15) / 8) * r->k), 256, 0, st>>>(
        n, r->k, (const uint64_t *)dk, r->a, r->ld, 0, r->g->row0, r->g->iperm);
  KPM_CUDA(cudaGetLastError());
  int rc = run_after_probes(r);
  return rc;
}

int kpm_run_total_steps(kpm_run *r) { return r ? r->total_steps : 0; }

int kpm_run_blocks(kpm_run *r, void **a, void **b) {
  KPM_CHECK_ARG(r, "run is NULL");
  if (a) *a = r->a;
  if (b) *b = r->b;
  return KPM_OK;
}

int kpm_run_set_partition(kpm_run *r, int nparts, const int64_t *part_lo, int me,
                          const void *const *peer_a, const void *const *peer_b) {
  KPM_CHECK_ARG(r && part_lo && peer_a && peer_b, "bad arguments");
  KPM_CHECK_ARG(nparts >= 1 && nparts <= KPM_MAX_PARTS, "1 <= nparts <= %d", KPM_MAX_PARTS);
  KPM_CHECK_ARG(me >= 0 && me < nparts, "bad partition index");
  KPM_CHECK_ARG(part_lo[me] == r->g->row0 && part_lo[me + 1] - part_lo[me] == r->g->n,
                "partition %d rows do not match the graph's rows", me);
  KPM_CHECK_ARG(part_lo[0] == 0 && part_lo[nparts] == r->g->n_global, "bad partition bounds");
  KPM_CHECK_ARG(peer_a[me] == r->a && peer_b[me] == r->b, "peer table must hold own blocks");
  KPM_CHECK_ARG(r->mode != KPM_MODE_LDOS || nparts == 1 || true, "");
  r->nparts = nparts;
  r->partitioned = true;
  r->me = me;
  for (int q = 0; q <= nparts; ++q) r->part_lo[q] = part_lo[q];
  for (int q = 0; q < nparts; ++q) {
    r->peer_a[q] = (const double *)peer_a[q];
    r->peer_b[q] = (const double *)peer_b[q];
  }
  return KPM_OK;
}

int kpm_run_advance(kpm_run *r, int32_t steps, int32_t *remaining) {
  kpm::Nvtx nvtx_range_("kpm_run_advance");
  KPM_CHECK_ARG(r, "run is NULL");
  KPM_CHECK_ARG(r->have_probes, "probes not set");
  cudaStream_t st = r->g->ctx->stream;
  for (int32_t s = 0; s < steps && r->done_steps < r->total_steps; ++s) {
    const bool first = r->k_index == 0;
    StepParams p = base_params(r);
    p.X = r->cur;
    p.Xprev = r->prev;
    if (r->nparts > 1) {
      const bool on_a = r->cur == r->a;
      for (int q = 0; q < r->nparts; ++q) p.xparts[q] = on_a ? r->peer_a[q] : r->peer_b[q];
    }
    double *dst = first ? r->b : r->prev;  // T_{k+1} overwrites T_{k-1}
    p.Y = dst;
    p.ldos_col = r->k_index + 1;
    if (r->timing) {
      if ((size_t)(2 * r->ev_used + 2) > r->ev.size()) {
        for (int q = 0; q < 2; ++q) {
          cudaEvent_t e;
          KPM_CUDA(cudaEventCreate(&e));
          r->ev.push_back(e);
        }
      }
      KPM_CUDA(cudaEventRecord(r->ev[2 * r->ev_used], st));
    }
    // KPM_TRACE=<file>: record the work items of step KPM_TRACE_STEP (default 2)
    const char *trace_path = getenv("KPM_TRACE");
    const int trace_step = getenv("KPM_TRACE_STEP") ? atoi(getenv("KPM_TRACE_STEP")) : 2;
    const int64_t trace_items = r->g->n_chunks + p.n_heavy_tasks;
    if (trace_path && r->done_steps == trace_step && trace_items > 0) {
      KPM_CUDA(cudaMallocAsync(&p.trace, sizeof(unsigned long long) * 3 * trace_items, st));
      p.fuse_tiles = 0;  // the trace layout is one item per chunk
    }
    // KPM_WINDOW_MB (experiment): persisting L2 access-policy window over the
    // first rows of the gathered block T_k (the highest-degree rows when the
    // graph is degree-relabelled)
    static const double window_mb = getenv("KPM_WINDOW_MB") ? atof(getenv("KPM_WINDOW_MB")) : 0.0;
    if (window_mb > 0.0) {
      size_t bytes = (size_t)(window_mb * 1048576.0);
      const size_t blk = sizeof(double) * (size_t)r->g->n * r->ld;
      if (bytes > blk) bytes = blk;
      static bool limit_set = false;
      if (!limit_set) {
        KPM_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, r->g->ctx->persist_max));
        limit_set = true;
      }
      cudaStreamAttrValue attr = {};
      attr.accessPolicyWindow.base_ptr = r->cur;
      attr.accessPolicyWindow.num_bytes = bytes;
      attr.accessPolicyWindow.hitRatio =
          bytes > r->g->ctx->persist_max ? (float)r->g->ctx->persist_max / (float)bytes : 1.0f;
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      KPM_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr));
    }
    KPM_CUDA(launch_step(r, p, false, first, st));
    if (p.trace) {
      std::vector<unsigned long long> tr(3 * trace_items);
      KPM_CUDA(cudaMemcpyAsync(tr.data(), p.trace, sizeof(unsigned long long) * tr.size(),
                               cudaMemcpyDeviceToHost, st));
      KPM_CUDA(cudaStreamSynchronize(st));
      KPM_CUDA(cudaFreeAsync(p.trace, st));
      if (FILE *fp = fopen(trace_path, "wb")) {
        const long long hdr[4] = {(long long)p.n_heavy_tasks, (long long)r->g->n_chunks,
                                  (long long)r->ld, (long long)r->g->n_heavy};
        fwrite(hdr, sizeof(hdr), 1, fp);
        fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
        std::vector<int32_t> cs(r->g->n_chunks + 1), co(r->g->n_chunks);
        std::vector<int64_t> rp(r->g->n + 1);
        cudaMemcpy(cs.data(), r->g->chunk_start, sizeof(int32_t) * cs.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(co.data(), r->g->chunk_order, sizeof(int32_t) * co.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(rp.data(), r->g->row_ptr, sizeof(int64_t) * rp.size(), cudaMemcpyDeviceToHost);
        // per chunk id: rows, nonzeros, empty rows
        std::vector<int64_t> cst(3 * (size_t)r->g->n_chunks);
        for (int32_t c = 0; c < r->g->n_chunks; ++c) {
          int64_t empty = 0;
          for (int32_t i = cs[c]; i < cs[c + 1]; ++i) empty += rp[i + 1] == rp[i];
          cst[3 * c] = cs[c + 1] - cs[c];
          cst[3 * c + 1] = rp[cs[c + 1]] - rp[cs[c]];
          cst[3 * c + 2] = empty;
        }
        fwrite(co.data(), sizeof(int32_t), co.size(), fp);
        fwrite(cst.data(), sizeof(int64_t), cst.size(), fp);
        fclose(fp);
      }
    }
    if (r->timing) KPM_CUDA(cudaEventRecord(r->ev[2 * r->ev_used++ + 1], st));
    const int m = r->k_index + 1;
    if (r->mode == KPM_MODE_LDOS && r->g->n_heavy > 0) {
      const int nsl = (int)((r->ld + kSlice - 1) / kSlice);
      ldos_heavy_kernel<<<(r->g->n_heavy + 127) / 128, 128, 0, st>>>(
          r->hldos, r->g->heavy_rows, r->g->n_heavy, nsl, r->ldos, r->m_max + 1, m, r->flag,
          r->g->perm);
      KPM_CUDA(cudaGetLastError());
    }
    if (r->mode == KPM_MODE_DOS_DOUBLING) KPM_CUDA(launch_finalize(r, 2, m, st));
    else if (r->mode == KPM_MODE_DOS_DIRECT) KPM_CUDA(launch_finalize(r, 1, m, st));
    r->prev = r->cur;
    r->cur = dst;
    r->k_index += 1;
    r->done_steps += 1;
  }
  if (remaining) *remaining = r->total_steps - r->done_steps;
  return KPM_OK;
}

int kpm_run_result(kpm_run *r, double *out, double trace_scale, int64_t *bad_node) {
  kpm::Nvtx nvtx_range_("kpm_run_result");
  KPM_CHECK_ARG(r && (out || r->mode == KPM_MODE_LDOS), "bad arguments");
  KPM_CHECK_ARG(r->have_probes, "probes not set");
  KPM_CHECK_ARG(r->done_steps == r->total_steps, "run not finished (%d of %d steps)",
                r->done_steps, r->total_steps);
  cudaStream_t st = r->g->ctx->stream;
  KPM_CUDA(cudaSetDevice(r->g->ctx->device));
  int32_t hflag[4];
  KPM_CUDA(cudaMemcpyAsync(hflag, r->flag, sizeof(hflag), cudaMemcpyDeviceToHost, st));
  if (r->mode == KPM_MODE_LDOS) {
    if (!(r->flags & KPM_LDOS_RAW) && r->g->n > 0 && !r->finished) {
      set_i32_kernel<<<1, 1, 0, st>>>(r->flag + 1, 0x7fffffff);
      first_zero_kernel<<<grid_of(r->g->n), 256, 0, st>>>(r->den, r->g->n, r->flag + 1);
      KPM_CUDA(cudaMemcpyAsync(hflag, r->flag, sizeof(hflag), cudaMemcpyDeviceToHost, st));
    }
    KPM_CUDA(cudaStreamSynchronize(st));
    if (hflag[0]) {
      set_error("Chebyshev recurrence overflowed; re-estimate the spectral range "
                "with a larger margin");
      return KPM_ENONFINITE;
    }
    if (!(r->flags & KPM_LDOS_RAW) && !r->finished && hflag[1] != 0x7fffffff) {
      if (bad_node) *bad_node = hflag[1];
      set_error("zero probe mass at node %d; its moments are unrecoverable", hflag[1]);
      return KPM_EZEROMASS;
    }
    if (r->g->n > 0 && !r->finished)
      ldos_finish<<<grid_of(r->g->n * (r->m_max + 1)), 256, 0, st>>>(
          r->ldos, r->den, r->g->n, r->m_max + 1, (r->flags & KPM_LDOS_RAW) != 0,
          trace_scale);
    KPM_CUDA(cudaGetLastError());
    r->finished = true;  // the num buffer now holds values
    if (r->g->n > 0 && out)
      KPM_CUDA(cudaMemcpyAsync(out, r->ldos,
                               sizeof(double) * (size_t)r->g->n * (r->m_max + 1),
                               cudaMemcpyDefault, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    return KPM_OK;
  }
  KPM_CUDA(cudaMemcpy2DAsync(out, sizeof(double) * r->k, r->contrib, sizeof(double) * r->ld,
                             sizeof(double) * r->k, r->m_max + 1, cudaMemcpyDefault, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  return KPM_OK;
}

int kpm_run_ldos_values(kpm_run *r, const double **values) {
  KPM_CHECK_ARG(r && values && r->mode == KPM_MODE_LDOS, "not an LDOS run");
  *values = r->ldos;
  return KPM_OK;
}

int kpm_run_accumulate(kpm_run *dst, kpm_run *src) {
  kpm::Nvtx nvtx_range_("kpm_run_accumulate");
  KPM_CHECK_ARG(dst && src && dst != src, "bad arguments");
  KPM_CHECK_ARG(dst->mode == KPM_MODE_LDOS && src->mode == KPM_MODE_LDOS,
                "accumulate combines LDOS runs");
  KPM_CHECK_ARG(dst->g->n == src->g->n && dst->m_max == src->m_max,
                "runs differ in n or m_max");
  KPM_CHECK_ARG(dst->have_probes && src->have_probes && !dst->finished && !src->finished &&
                    dst->done_steps == dst->total_steps && src->done_steps == src->total_steps,
                "both runs must be complete and not yet finished by kpm_run_result");
  const int64_t n = dst->g->n, cnt = n * (dst->m_max + 1);
  if (n == 0) return KPM_OK;
  // src's stream has produced its sums; dst's stream orders the rest
  KPM_CUDA(cudaSetDevice(src->g->ctx->device));
  KPM_CUDA(cudaStreamSynchronize(src->g->ctx->stream));
  KPM_CUDA(cudaSetDevice(dst->g->ctx->device));
  cudaStream_t st = dst->g->ctx->stream;
  const bool same = src->g->ctx->device == dst->g->ctx->device;
  const double *sl = src->ldos, *sd = src->den;
  const int32_t *sf = src->flag;
  char *tmp = nullptr;
  if (!same) {  // stage the peer device's sums (NVLink peer copy) on dst's device
    const size_t bytes = sizeof(double) * (size_t)(cnt + n) + 16;
    KPM_CUDA(cudaMallocAsync((void **)&tmp, bytes, st));
    KPM_CUDA(cudaMemcpyPeerAsync(tmp, dst->g->ctx->device, src->ldos, src->g->ctx->device,
                                 sizeof(double) * cnt, st));
    KPM_CUDA(cudaMemcpyPeerAsync(tmp + sizeof(double) * cnt, dst->g->ctx->device, src->den,
                                 src->g->ctx->device, sizeof(double) * n, st));
    KPM_CUDA(cudaMemcpyPeerAsync(tmp + sizeof(double) * (cnt + n), dst->g->ctx->device,
                                 src->flag, src->g->ctx->device, sizeof(int32_t), st));
    sl = (const double *)tmp;
    sd = sl + cnt;
    sf = (const int32_t *)(sd + n);
  }
  add_inplace_kernel<<<grid_of(cnt), 256, 0, st>>>(dst->ldos, sl, cnt);
  add_inplace_kernel<<<grid_of(n), 256, 0, st>>>(dst->den, sd, n);
  or_flag_kernel<<<1, 1, 0, st>>>(dst->flag, sf);
  KPM_CUDA(cudaGetLastError());
  if (tmp) KPM_CUDA(cudaFreeAsync(tmp, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  return KPM_OK;
}

int kpm_run_trim(kpm_run *r) {
  KPM_CHECK_ARG(r, "run is NULL");
  KPM_CHECK_ARG(r->done_steps == r->total_steps, "run not complete");
  KPM_CUDA(cudaSetDevice(r->g->ctx->device));
  KPM_CUDA(cudaStreamSynchronize(r->g->ctx->stream));
  double **bufs[] = {&r->a, &r->b, &r->z, &r->partial, &r->hpart, &r->hldos, &r->gpart};
  for (double **b : bufs) {
    cudaFree(*b);
    *b = nullptr;
  }
  r->cur = r->prev = nullptr;
  r->tm_ok = r->tm_tile_ok = false;
  return KPM_OK;
}

int kpm_run_block(kpm_run *r, const double **t_k, int64_t *ld, int32_t *k_index) {
  KPM_CHECK_ARG(r, "run is NULL");
  if (t_k) *t_k = r->cur;
  if (t_k && r->g->perm && r->cur && r->g->n > 0) {
    // a run on the twin: hand out T_k in the caller's row order
    KPM_CUDA(cudaSetDevice(r->g->ctx->device));
    cudaStream_t st = r->g->ctx->stream;
    if (!r->unperm) KPM_CUDA(cudaMalloc(&r->unperm, sizeof(double) * (size_t)r->g->n * r->ld));
    permute_rows_kernel<<<grid_of(r->g->n * r->ld), 256, 0, st>>>(r->cur, r->unperm, r->g->perm,
                                                                 r->g->n, r->ld, 1);
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaStreamSynchronize(st));
    *t_k = r->unperm;
  }
  if (ld) *ld = r->ld;
  if (k_index) *k_index = r->k_index;
  return KPM_OK;
}

void kpm_run_free(kpm_run *r) {
  if (!r) return;
  cudaSetDevice(r->g->ctx->device);
  cudaStreamSynchronize(r->g->ctx->stream);
  cudaFree(r->a);
  cudaFree(r->b);
  cudaFree(r->z);
  cudaFree(r->partial);
  cudaFree(r->contrib);
  cudaFree(r->ldos);
  cudaFree(r->den);
  cudaFree(r->flag);
  cudaFree(r->hpart);
  cudaFree(r->hldos);
  cudaFree(r->gpart);
  cudaFree(r->queue);
  cudaFree(r->unperm);
  for (cudaEvent_t e : r->ev) cudaEventDestroy(e);
  delete r;
}

int kpm_run_set_timing(kpm_run *r, int enable) {
  KPM_CHECK_ARG(r, "run is NULL");
  r->timing = enable != 0;
  r->ev_used = 0;
  return KPM_OK;
}

int kpm_run_kernel_time(kpm_run *r, double *ms, int32_t *launches) {
  KPM_CHECK_ARG(r && ms, "bad arguments");
  KPM_CUDA(cudaStreamSynchronize(r->g->ctx->stream));
  double tot = 0.0;
  for (int32_t i = 0; i < r->ev_used; ++i) {
    float t = 0.f;
    KPM_CUDA(cudaEventElapsedTime(&t, r->ev[2 * i], r->ev[2 * i + 1]));
    tot += t;
  }
  *ms = tot;
  if (launches) *launches = r->ev_used;
  r->ev_used = 0;
  return KPM_OK;
}

int kpm_dos_contrib(kpm_graph *g, const double *z, int64_t k, int32_t m_max,
                    int32_t doubling, double *contrib) {
  kpm_run *r = nullptr;
  KPM_TRY(kpm_run_create(g, k, doubling ? KPM_MODE_DOS_DOUBLING : KPM_MODE_DOS_DIRECT,
                         m_max, 0, &r));
  int rc = kpm_run_set_probes(r, z, k);
  if (rc == KPM_OK) rc = kpm_run_advance(r, r->total_steps, nullptr);
  if (rc == KPM_OK) rc = kpm_run_result(r, contrib, 0.0, nullptr);
  kpm_run_free(r);
  return rc;
}

int kpm_ldos(kpm_graph *g, const double *z, int64_t k, int32_t m_max, int32_t flags,
             double trace_scale, double *values, int64_t *bad_node) {
  kpm_run *r = nullptr;
  KPM_TRY(kpm_run_create(g, k, KPM_MODE_LDOS, m_max, flags, &r));
  int rc = kpm_run_set_probes(r, z, k);
  if (rc == KPM_OK) rc = kpm_run_advance(r, r->total_steps, nullptr);
  if (rc == KPM_OK) rc = kpm_run_result(r, values, trace_scale, bad_node);
  kpm_run_free(r);
  return rc;
}

int kpm_probes_rademacher(kpm_ctx *ctx, int64_t n, int64_t ncols, const uint64_t *keys,
                          double *z, int64_t ldz, int64_t col0) {
  KPM_CHECK_ARG(ctx && keys && z && n >= 0 && ncols >= 0 && col0 >= 0 && ldz >= col0 + ncols,
                "bad arguments");
  KPM_CHECK_ARG(is_device_ptr(z), "z must be a device buffer");
  KPM_CUDA(cudaSetDevice(ctx->device));
  DevBuf tk;
  const void *dk;
  KPM_TRY(stage_in(ctx->stream, keys, sizeof(uint64_t) * 2 * ncols, tk, &dk));
  if (n > 0 && ncols > 0)
    rademacher_kernel<<<grid_of(((n + 7) / 8) * ncols), 256, 0, ctx->stream>>>(
        n, ncols, (const uint64_t *)dk, z, ldz, col0, 0);
  KPM_CUDA(cudaGetLastError());
  KPM_CUDA(cudaStreamSynchronize(ctx->stream));  // tk is freed on return
  return KPM_OK;
}

int kpm_csr_matvec(kpm_ctx *ctx, int64_t n_rows, const int64_t *indptr,
                   const int64_t *indices, const double *data, int64_t nnz,
                   const double *x, int64_t n_x_rows, int64_t k, double *out) {
  kpm::Nvtx nvtx_range_("kpm_csr_matvec");
  KPM_CHECK_ARG(ctx && n_rows >= 0 && nnz >= 0 && k >= 0 && n_x_rows >= 0, "bad arguments");
  KPM_CHECK_ARG(indptr && (nnz == 0 || (indices && data)), "NULL CSR arrays");
  if (n_rows == 0 || k == 0) return KPM_OK;
  KPM_CHECK_ARG(out && (x || n_x_rows == 0), "NULL x/out");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf tp, ti, td, tx, to;
  const void *dp, *di, *dd, *dx;
  KPM_TRY(stage_in(st, indptr, sizeof(int64_t) * (n_rows + 1), tp, &dp));
  KPM_TRY(stage_in(st, indices, sizeof(int64_t) * nnz, ti, &di));
  KPM_TRY(stage_in(st, data, sizeof(double) * nnz, td, &dd));
  KPM_TRY(stage_in(st, x, sizeof(double) * n_x_rows * k, tx, &dx));
  double *dout = out;
  const bool out_dev = is_device_ptr(out);
  if (!out_dev) {
    KPM_CUDA(cudaMalloc(&to.ptr, sizeof(double) * n_rows * k));
    dout = (double *)to.ptr;
  }
  const int64_t warps = n_rows;
  csr_matvec_kernel<<<grid_of(warps * 32), 256, 0, st>>>(
      n_rows, (const int64_t *)dp, (const int64_t *)di, (const double *)dd,
      (const double *)dx, k, dout);
  KPM_CUDA(cudaGetLastError());
  if (!out_dev)
    KPM_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * n_rows * k, cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  return KPM_OK;
}

int kpm_filter_probes(kpm_ctx *ctx, int64_t n, int64_t k, double *z, int64_t ldz,
                      int64_t n_groups, const int64_t *group_ptr, const int64_t *vec_ptr,
                      const int64_t *vec_idx, const double *vec_val) {
  kpm::Nvtx nvtx_range_("kpm_filter_probes");
  KPM_CHECK_ARG(ctx && z && n >= 0 && k >= 0 && ldz >= k && n_groups >= 0, "bad arguments");
  if (n_groups == 0 || k == 0 || n == 0) return KPM_OK;
  KPM_CHECK_ARG(group_ptr && vec_ptr && vec_idx && vec_val, "NULL vector arrays");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  // group_ptr / vec_ptr are read on the host for the sizes
  int64_t nvec = 0, nent = 0;
  const bool gp_dev = is_device_ptr(group_ptr);
  if (gp_dev) {
    KPM_CUDA(cudaMemcpy(&nvec, group_ptr + n_groups, sizeof(int64_t), cudaMemcpyDeviceToHost));
  } else {
    nvec = group_ptr[n_groups];
  }
  if (is_device_ptr(vec_ptr)) {
    KPM_CUDA(cudaMemcpy(&nent, vec_ptr + nvec, sizeof(int64_t), cudaMemcpyDeviceToHost));
  } else {
    nent = vec_ptr[nvec];
  }
  DevBuf tg, tv, ti, tw, tz;
  const void *dg, *dv, *di, *dw;
  KPM_TRY(stage_in(st, group_ptr, sizeof(int64_t) * (n_groups + 1), tg, &dg));
  KPM_TRY(stage_in(st, vec_ptr, sizeof(int64_t) * (nvec + 1), tv, &dv));
  KPM_TRY(stage_in(st, vec_idx, sizeof(int64_t) * nent, ti, &di));
  KPM_TRY(stage_in(st, vec_val, sizeof(double) * nent, tw, &dw));
  double *dz = z;
  const bool z_dev = is_device_ptr(z);
  if (!z_dev) {
    KPM_CUDA(cudaMalloc(&tz.ptr, sizeof(double) * n * ldz));
    KPM_CUDA(cudaMemcpyAsync(tz.ptr, z, sizeof(double) * n * ldz, cudaMemcpyHostToDevice, st));
    dz = (double *)tz.ptr;
  }
  filter_kernel<<<grid_of(n_groups * 32), 256, 0, st>>>(
      dz, k, ldz, n_groups, (const int64_t *)dg, (const int64_t *)dv, (const int64_t *)di,
      (const double *)dw);
  KPM_CUDA(cudaGetLastError());
  if (!z_dev)
    KPM_CUDA(cudaMemcpyAsync(z, dz, sizeof(double) * n * ldz, cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  return KPM_OK;
}

}  // extern "C"
