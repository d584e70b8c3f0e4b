// Lanczos with full reorthogonalisation on the device.
//
// lanczos_factorize (lanczos.py:46-91) for k independent start vectors at
// once, driving every column in lockstep until it exhausts its Krylov space:
//   q_0 = z / ||z||
//   w = H q_j                      (bit-identical to the reference's apply:
//                                   CSR order, separate roundings, explicit
//                                   values or h_ij = dinv_i dinv_j, then
//                                   y -= shift x; y /= scale)
//   alpha_j = q_j . w
//   2x classical Gram-Schmidt: w -= Q (Q^T w)   (Q = q_0..q_j)
//   beta_j = ||w||; breakdown if beta_j <= 1e-12 max(hnorm, 1e-300)
//   q_{j+1} = w / beta_j
// The basis lives in HBM vector-major (column c, vector v, row i) so every
// pass over it is a coalesced stream: the Gram-Schmidt dots read one 2048-row
// tile of w into shared memory and each warp streams a subset of the basis
// vectors over it; the partial sums are reduced in a fixed order (the result
// is deterministic run to run; it differs from numpy's BLAS order in the
// last bits, so parity is a tolerance on alphas / betas / Ritz values).
// Host control per step: one D2H of (alpha, beta) per column for the
// NaN / breakdown decisions, exactly the reference's.
#include <cmath>
#include <vector>

#include "kpm_internal.cuh"

namespace kpm {

constexpr int kLzTile = 2048;   // rows per dot tile (8 per thread)
constexpr double kBreakdownRtol = 1e-12;  // lanczos.py:24

struct LzGraph {
  const int64_t *row_ptr;
  const int32_t *col;
  const double *vals;   // explicit values or nullptr (implicit dinv products)
  const double *dinv;
  double shift, scale;
  int64_t n;
};

// w_c = H q_c for every active column (warp per row, products formed in
// parallel, summed in CSR order by shuffles: the Cython kernel's order)
__global__ void lz_apply_kernel(LzGraph g, const double *__restrict__ Q, int64_t qstride,
                                double *__restrict__ W, const int8_t *__restrict__ active) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  const double *x = Q + c * qstride;
  double *y = W + c * g.n;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < g.n; i += nw) {
    const int64_t beg = g.row_ptr[i], end = g.row_ptr[i + 1];
    const double di = g.vals ? 0.0 : g.dinv[i];
    double acc = 0.0;
    for (int64_t base = beg; base < end; base += 32) {
      const int cnt = (int)min((int64_t)32, end - base);
      double prod = 0.0;
      if (lane < cnt) {
        const int j = g.col[base + lane];
        const double h = g.vals ? g.vals[base + lane] : __dmul_rn(di, g.dinv[j]);
        prod = __dmul_rn(h, x[j]);
      }
      for (int q = 0; q < cnt; ++q) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, q));
    }
    if (lane == 0) {
      double yv = acc;
      if (g.shift != 0.0) yv = __dsub_rn(yv, __dmul_rn(g.shift, x[i]));
      if (g.scale != 1.0) yv = __ddiv_rn(yv, g.scale);
      y[i] = yv;
    }
  }
}

// partial[c][tile][v] = sum over the tile's rows of Q_c[v0+v][i] * W_c[i]
__global__ void __launch_bounds__(256) lz_dots_kernel(
    const double *__restrict__ Q, int64_t qstride, int nvec, const double *__restrict__ W,
    int64_t n, const int8_t *__restrict__ active, double *__restrict__ partial, int64_t tiles,
    int pstride) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  __shared__ double ws[kLzTile];
  const int64_t r0 = (int64_t)blockIdx.x * kLzTile;
  const double *w = W + c * n;
  for (int r = threadIdx.x; r < kLzTile; r += blockDim.x)
    ws[r] = (r0 + r < n) ? w[r0 + r] : 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double *qc = Q + c * qstride;
  for (int v = warp; v < nvec; v += 8) {
    const double *q = qc + (int64_t)v * n + r0;
    double s = 0.0;
    for (int r = lane; r < kLzTile; r += 32)
      if (r0 + r < n) s = fma(q[r], ws[r], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) partial[((int64_t)c * tiles + blockIdx.x) * pstride + v] = s;
  }
}

// out[c][v] = sum_t partial[c][t][v] in a fixed order (warp per (c, v))
__global__ void lz_reduce_kernel(const double *__restrict__ partial, int64_t tiles, int pstride,
                                 int nvec, int k, const int8_t *__restrict__ active,
                                 double *__restrict__ out, int ostride) {
  const int lane = threadIdx.x & 31;
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (item >= (int64_t)k * nvec) return;
  const int c = (int)(item / nvec), v = (int)(item % nvec);
  if (!active[c]) return;
  double s = 0.0;
  for (int64_t t = lane; t < tiles; t += 32) s += partial[((int64_t)c * tiles + t) * pstride + v];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[(int64_t)c * ostride + v] = s;
}

// W_c[i] -= sum_v Q_c[v][i] * h_c[v]; optionally the tile's sum of W_c^2
__global__ void __launch_bounds__(256) lz_update_kernel(
    const double *__restrict__ Q, int64_t qstride, int nvec, const double *__restrict__ h,
    int hstride, double *__restrict__ W, int64_t n, const int8_t *__restrict__ active,
    double *__restrict__ norm_partial, int64_t tiles) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  const int64_t r0 = (int64_t)blockIdx.x * kLzTile;
  const double *qc = Q + c * qstride;
  const double *hc = h + (int64_t)c * hstride;
  double *w = W + c * n;
  double sq = 0.0;
  for (int r = threadIdx.x; r < kLzTile; r += blockDim.x) {
    const int64_t i = r0 + r;
    if (i >= n) break;
    double acc = 0.0;
    for (int v = 0; v < nvec; ++v) acc = fma(qc[(int64_t)v * n + i], hc[v], acc);
    const double x = w[i] - acc;
    w[i] = x;
    sq = fma(x, x, sq);
  }
  if (norm_partial) {
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < 8; ++q) s += red[q];
      norm_partial[(int64_t)c * tiles + blockIdx.x] = s;
    }
  }
}

// q_{j+1} = w / beta   (or q_0 = z / ||z||)
__global__ void lz_scale_kernel(const double *__restrict__ W, int64_t wstride,
                                const double *__restrict__ beta, double *__restrict__ Q,
                                int64_t qstride, int64_t n, const int8_t *__restrict__ active) {
  const int c = blockIdx.y;
  if (!active[c]) return;
  const double b = beta[c];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Q[c * qstride + i] = __ddiv_rn(W[c * wstride + i], b);
}

__global__ void lz_sqrt_kernel(double *x, int k) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < k) x[c] = sqrt(x[c]);
}

}  // namespace kpm

using namespace kpm;

extern "C" int kpm_lanczos(kpm_graph *g, const double *z, int64_t ldz, int64_t k, int32_t steps,
                           const double *z_norm, double *alphas, double *betas,
                           int32_t *taken, int32_t *exhausted, int32_t *status,
                           double *basis) {
  kpm::Nvtx nvtx_range_("kpm_lanczos");
  KPM_CHECK_ARG(g && z && z_norm && alphas && betas && taken && exhausted && status,
                "bad arguments");
  KPM_CHECK_ARG(k >= 1 && steps >= 1 && ldz >= k, "bad sizes");
  KPM_CHECK_ARG(g->row0 == 0 && (g->n_global == 0 || g->n_global == g->n),
                "row-partitioned graphs are not supported");
  const int64_t n = g->n;
  KPM_CHECK_ARG(n >= 1, "empty operator");
  const int S = (int)std::min<int64_t>(steps, n);
  kpm_ctx *ctx = g->ctx;
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int64_t tiles = (n + kLzTile - 1) / kLzTile;
  const int64_t qstride = (int64_t)S * n;  // per column
  DevBuf dq, dw, dpart, dred, dnorm, dact, dz, dzn, dscal;
  KPM_CUDA(cudaMalloc(&dq.ptr, sizeof(double) * (size_t)k * qstride));
  KPM_CUDA(cudaMalloc(&dw.ptr, sizeof(double) * (size_t)k * n));
  KPM_CUDA(cudaMalloc(&dpart.ptr, sizeof(double) * (size_t)k * tiles * S));
  KPM_CUDA(cudaMalloc(&dred.ptr, sizeof(double) * (size_t)k * S));
  KPM_CUDA(cudaMalloc(&dnorm.ptr, sizeof(double) * (size_t)k * tiles));
  KPM_CUDA(cudaMalloc(&dact.ptr, k));
  KPM_CUDA(cudaMalloc(&dscal.ptr, sizeof(double) * 2 * k));
  double *Q = (double *)dq.ptr, *W = (double *)dw.ptr, *part = (double *)dpart.ptr;
  double *red = (double *)dred.ptr, *npart = (double *)dnorm.ptr;
  double *alpha_d = (double *)dscal.ptr, *beta_d = alpha_d + k;
  int8_t *act = (int8_t *)dact.ptr;
  std::vector<int8_t> hact(k, 1);
  KPM_CUDA(cudaMemcpyAsync(act, hact.data(), k, cudaMemcpyHostToDevice, st));

  // q_0 = z / ||z|| (norms from the caller: the reference's np.linalg.norm)
  const void *zd, *znd;
  KPM_TRY(stage_in(st, z, sizeof(double) * (size_t)n * ldz, dz, &zd));
  KPM_TRY(stage_in(st, z_norm, sizeof(double) * k, dzn, &znd));
  {
    // z is n x ldz row-major: gather column c into W_c, then scale into Q_c[0]
    const double *zz = (const double *)zd;
    for (int64_t c = 0; c < k; ++c)
      KPM_CUDA(cudaMemcpy2DAsync(W + c * n, sizeof(double), zz + c, sizeof(double) * ldz,
                                 sizeof(double), n, cudaMemcpyDeviceToDevice, st));
    const dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), (unsigned)k);
    lz_scale_kernel<<<grid, 256, 0, st>>>(W, n, (const double *)znd, Q, qstride, n, act);
  }

  LzGraph lg{g->row_ptr, g->col_idx, g->values, g->dinv, g->shift, g->scale, n};
  const int apply_blocks = (int)std::min<int64_t>((n * 32 + 255) / 256, 148 * 64);
  const dim3 gapply(apply_blocks, (unsigned)k);
  const dim3 gtiles((unsigned)tiles, (unsigned)k);
  const dim3 gscale((unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), (unsigned)k);
  std::vector<double> ha(k), hb(k), hnorm(k, 0.0);
  std::vector<int32_t> done(k, 0);
  for (int64_t c = 0; c < k; ++c) {
    taken[c] = 0;
    exhausted[c] = 0;
    status[c] = 0;
  }
  int64_t live = k;
  for (int j = 0; j < S && live > 0; ++j) {
    lz_apply_kernel<<<gapply, 256, 0, st>>>(lg, Q + (int64_t)j * n, qstride, W, act);
    // pass 1 dots against q_0..q_j (v = j is alpha_j = q_j . w)
    const int nv = j + 1;
    lz_dots_kernel<<<gtiles, 256, 0, st>>>(Q, qstride, nv, W, n, act, part, tiles, S);
    lz_reduce_kernel<<<(unsigned)((k * nv * 32 + 255) / 256), 256, 0, st>>>(part, tiles, S, nv,
                                                                          (int)k, act, red, S);
    const bool last = (j == S - 1);
    if (!last) {
      // w -= Q h ; second pass ; beta^2 from the second update
      lz_update_kernel<<<gtiles, 256, 0, st>>>(Q, qstride, nv, red, S, W, n, act, nullptr,
                                                tiles);
    }
    // alpha_j out of the first pass
    KPM_CUDA(cudaMemcpy2DAsync(alpha_d, sizeof(double), red + j, sizeof(double) * S,
                               sizeof(double), k, cudaMemcpyDeviceToDevice, st));
    if (!last) {
      lz_dots_kernel<<<gtiles, 256, 0, st>>>(Q, qstride, nv, W, n, act, part, tiles, S);
      lz_reduce_kernel<<<(unsigned)((k * nv * 32 + 255) / 256), 256, 0, st>>>(
          part, tiles, S, nv, (int)k, act, red, S);
      lz_update_kernel<<<gtiles, 256, 0, st>>>(Q, qstride, nv, red, S, W, n, act, npart, tiles);
      lz_reduce_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, st>>>(npart, tiles, 1, 1,
                                                                        (int)k, act, beta_d, 1);
      lz_sqrt_kernel<<<(unsigned)((k + 127) / 128), 128, 0, st>>>(beta_d, (int)k);
    }
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaMemcpyAsync(ha.data(), alpha_d, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    if (!last)
      KPM_CUDA(cudaMemcpyAsync(hb.data(), beta_d, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    bool mask_changed = false;
    for (int64_t c = 0; c < k; ++c) {
      if (done[c]) continue;
      const double a = ha[c];
      alphas[c * S + j] = a;
      taken[c] = j + 1;
      if (!std::isfinite(a)) {  // lanczos.py:71-72
        status[c] = 1;
        done[c] = 1;
      } else {
        hnorm[c] = std::max(hnorm[c], std::fabs(a) + (j > 0 ? betas[c * (S - 1) + j - 1] : 0.0));
        if (last) {
          done[c] = 1;
        } else {
          const double b = hb[c];
          if (!std::isfinite(b)) {  // lanczos.py:80-81
            status[c] = 2;
            done[c] = 1;
          } else if (b <= kBreakdownRtol * std::max(hnorm[c], 1e-300)) {
            exhausted[c] = 1;  // lanczos.py:82-84
            done[c] = 1;
          } else {
            betas[c * (S - 1) + j] = b;
            hnorm[c] = std::max(hnorm[c], b);
          }
        }
      }
      if (done[c]) {
        hact[c] = 0;
        --live;
        mask_changed = true;
      }
    }
    if (mask_changed)
      KPM_CUDA(cudaMemcpyAsync(act, hact.data(), k, cudaMemcpyHostToDevice, st));
    if (!last && live > 0)
      lz_scale_kernel<<<gscale, 256, 0, st>>>(W, n, beta_d, Q + (int64_t)(j + 1) * n, qstride,
                                              n, act);
  }
  KPM_CUDA(cudaGetLastError());
  if (basis)
    KPM_CUDA(cudaMemcpyAsync(basis, Q, sizeof(double) * (size_t)k * qstride, cudaMemcpyDefault,
                             st));
  KPM_CUDA(cudaStreamSynchronize(st));
  return KPM_OK;
}
