// Per-node spectral histograms on the device.
//
// histogram_from_moments for per-node moments (density.py:63-108): with the
// closed-form bin table W[m, b] (density.py:51-60) and Jackson factors g_m,
//     masses[i, b] = sum_m (c[i, m] * g_m) * W[m, b],   norm[i] = c[i, 0] * g_0
// i.e. an (n x M+1) @ (M+1 x B) fp64 product (the reference's `coef @ table`,
// numpy/BLAS) -- 2 n (M+1) B flops over n (M+1) + n B doubles, so it is
// HBM-bound at C2 scale (808 MB of moments in, 400 MB of masses out).  The
// moments are read where the LDOS run left them (HBM), so only the (n, B)
// masses cross PCIe -- or nothing, when the caller keeps them on the device.
//
// One CTA computes a 64-row x 64-bin tile with 256 threads (4 x 4 outputs per
// thread, rows ty + 16 i and bins tx + 16 j: conflict-free shared reads),
// staging 16-moment slices of the damped moments and of W in shared memory.
// The damping product is rounded on its own as numpy's `coef * g` is; the
// accumulation uses fma (BLAS does too; its order is unspecified, so parity
// is the L1 tolerance of the histogram tests).
#include <cub/device/device_reduce.cuh>

#include "kpm_internal.cuh"

namespace kpm {

constexpr int kHB = 64;   // rows per tile
constexpr int kHN = 64;   // bins per tile
constexpr int kHK = 16;   // moments per slice

__global__ void __launch_bounds__(256) ldos_hist_kernel(
    const double *__restrict__ values, int64_t n, int64_t ld, int m1,
    const double *__restrict__ damp, const double *__restrict__ table, int bins,
    double *__restrict__ masses, double *__restrict__ norm, double *__restrict__ block_min) {
  __shared__ double As[kHK][kHB + 1];
  __shared__ double Bs[kHK][kHN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * kHB;
  const int bin0 = blockIdx.y * kHN;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  for (int m0 = 0; m0 < m1; m0 += kHK) {
    // damped moment slice: 64 rows x 16 moments, 4 per thread, coalesced
    // along the moment index of each row
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;
      const int r = e >> 4, k = e & 15;
      const int64_t row = row0 + r;
      double x = 0.0;
      if (row < n && m0 + k < m1) {
        x = values[row * ld + m0 + k];
        if (damp) x = __dmul_rn(x, damp[m0 + k]);
      }
      As[k][r] = x;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;
      const int k = e >> 6, b = e & 63;
      double w = 0.0;
      if (m0 + k < m1 && bin0 + b < bins) w = table[(int64_t)(m0 + k) * bins + bin0 + b];
      Bs[k][b] = w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kHK; ++k) {
      double a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = Bs[k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }

  double mn = INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = row0 + ty + 16 * i;
    if (row >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = bin0 + tx + 16 * j;
      if (b < bins) {
        const double x = acc[i][j];
        masses[row * bins + b] = x;
        mn = (x != x || mn != mn) ? NAN : fmin(mn, x);
      }
    }
  }
  if (norm && blockIdx.y == 0 && tid < kHB && row0 + tid < n) {
    const double c0 = values[(row0 + tid) * ld];
    norm[row0 + tid] = damp ? __dmul_rn(c0, damp[0]) : c0;
  }
  // block minimum (NaN-propagating like ndarray.min: a NaN wins)
  __shared__ double red[256];
  red[tid] = mn;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (tid < s) {
      const double o = red[tid + s], v = red[tid];
      red[tid] = (v != v || o != o) ? NAN : fmin(v, o);
    }
    __syncthreads();
  }
  if (tid == 0) block_min[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

struct NanMin {
  __device__ double operator()(double a, double b) const {
    return (a != a || b != b) ? NAN : fmin(a, b);
  }
};

}  // namespace kpm

using namespace kpm;

extern "C" int kpm_ldos_histogram(kpm_ctx *ctx, const double *values, int64_t n, int64_t ld,
                                  int32_t m_max, const double *damping, const double *table,
                                  int32_t bins, double *masses, double *norm,
                                  double *min_mass) {
  kpm::Nvtx nvtx_range_("kpm_ldos_histogram");
  KPM_CHECK_ARG(ctx && values && table && masses && n >= 0 && m_max >= 0 && bins >= 1 &&
                    ld >= m_max + 1,
                "bad arguments");
  KPM_CHECK_ARG(n < (int64_t(1) << 31) * kHB, "n too large");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  if (min_mass) *min_mass = INFINITY;
  if (n == 0) return KPM_OK;
  const int m1 = m_max + 1;
  DevBuf tv, td, tt, tm, tn, bmin, omin, tmp;
  const void *dv, *dd = nullptr, *dt;
  KPM_TRY(stage_in(st, values, sizeof(double) * (size_t)n * ld, tv, &dv));
  if (damping) KPM_TRY(stage_in(st, damping, sizeof(double) * m1, td, &dd));
  KPM_TRY(stage_in(st, table, sizeof(double) * (size_t)m1 * bins, tt, &dt));
  // outputs: device pointers in place, host pointers through a device buffer
  const bool masses_dev = is_device_ptr(masses);
  double *dm = masses;
  if (!masses_dev) {
    KPM_CUDA(cudaMalloc(&tm.ptr, sizeof(double) * (size_t)n * bins));
    dm = (double *)tm.ptr;
  }
  double *dn = norm;
  const bool norm_dev = norm && is_device_ptr(norm);
  if (norm && !norm_dev) {
    KPM_CUDA(cudaMalloc(&tn.ptr, sizeof(double) * n));
    dn = (double *)tn.ptr;
  }
  const dim3 grid((unsigned)((n + kHB - 1) / kHB), (unsigned)((bins + kHN - 1) / kHN));
  const int64_t nblk = (int64_t)grid.x * grid.y;
  KPM_CUDA(cudaMalloc(&bmin.ptr, sizeof(double) * nblk));
  KPM_CUDA(cudaMalloc(&omin.ptr, sizeof(double)));
  ldos_hist_kernel<<<grid, 256, 0, st>>>((const double *)dv, n, ld, m1, (const double *)dd,
                                         (const double *)dt, bins, dm, dn,
                                         (double *)bmin.ptr);
  KPM_CUDA(cudaGetLastError());
  size_t tb = 0;
  cub::DeviceReduce::Reduce(nullptr, tb, (double *)bmin.ptr, (double *)omin.ptr, nblk, NanMin{},
                            (double)INFINITY, st);
  KPM_CUDA(cudaMalloc(&tmp.ptr, tb));
  cub::DeviceReduce::Reduce(tmp.ptr, tb, (double *)bmin.ptr, (double *)omin.ptr, nblk, NanMin{},
                            (double)INFINITY, st);
  if (!masses_dev)
    KPM_CUDA(cudaMemcpyAsync(masses, dm, sizeof(double) * (size_t)n * bins,
                             cudaMemcpyDeviceToHost, st));
  if (norm && !norm_dev)
    KPM_CUDA(cudaMemcpyAsync(norm, dn, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  double hmin = INFINITY;
  KPM_CUDA(cudaMemcpyAsync(&hmin, omin.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  if (min_mass) *min_mass = hmin;
  return KPM_OK;
}
