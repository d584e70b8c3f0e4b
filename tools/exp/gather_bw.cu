// Gather roofline by segment size (round 2): what DRAM bandwidth do COLD row
// gathers reach on a B200 as a function of the gathered segment's size?
//
// The fused KPM step gathers one row segment of T_k per nonzero: 256 B for a
// 32-column shard (ld = 32), 512 B for a 64-column tile of a 128-column block
// (ld = 128).  MEASURED_PEAKS.json's hbm_gbs is a sequential copy; this
// program measures the same engine the step uses (TMA tile::gather4 into a
// per-warp shared-memory ring, one mbarrier per wave, 16 warps per SM, a
// consumer that reads every gathered byte once) on uniformly random rows of a
// block far larger than L2, so every gather is a DRAM miss.  Output: GB/s per
// (segment bytes, row stride, rows per wave, waves in flight).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gather_bw gather_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity)
      : "memory");
}

// W columns (fp64) per segment, WAVE rows per wave, D waves in flight per warp.
template <int W, int WAVE, int D>
__global__ void __launch_bounds__(256, 2)
gather_tma(const __grid_constant__ CUtensorMap tm, int64_t rows, int64_t waves_total,
           double *out) {
  extern __shared__ __align__(128) double smem[];
  constexpr int slot_d = WAVE * W;
  constexpr int warp_d = D * slot_d + (WAVE * D / 2 + 15) / 16 * 16 + 16;  // rows, ids (int32), barriers
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *base = smem + (size_t)warp * warp_d;
  int *ids = reinterpret_cast<int *>(base + D * slot_d);
  uint64_t *bars = reinterpret_cast<uint64_t *>(base + warp_d - 16);
  if (lane < D) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + lane)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t mine = (waves_total - gw + nwarps - 1) / nwarps;  // waves of this warp
  auto issue = [&](int64_t w) {
    const int sl = (int)(w % D);
    if (lane < WAVE)
      ids[sl * WAVE + lane] = (int)(mix((uint64_t)((gw + w * nwarps) * WAVE + lane)) % (uint64_t)rows);
    __syncwarp();
    if (elect_one()) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bar = smem_u32(bars + sl);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)(WAVE * W * 8))
                   : "memory");
      const uint32_t dst = smem_u32(base + sl * slot_d);
#pragma unroll
      for (int q = 0; q < WAVE / 4; ++q) {
        const int *j = ids + sl * WAVE + 4 * q;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst + 4 * q * W * 8),
            "l"(&tm), "r"(0), "r"(j[0]), "r"(j[1]), "r"(j[2]), "r"(j[3]), "r"(bar)
            : "memory");
      }
    }
  };
  for (int w = 0; w < D; ++w)
    if (w < mine) issue(w);
  uint32_t phase = 0;
  double acc = 0.0;
  for (int64_t w = 0; w < mine; ++w) {
    const int sl = (int)(w % D);
    mbar_wait(smem_u32(bars + sl), (phase >> sl) & 1u);
    phase ^= 1u << sl;
    const double *slot = base + sl * slot_d;
    // read every gathered byte once, the way the step's consumer does
#pragma unroll
    for (int k = 0; k < WAVE; ++k)
#pragma unroll
      for (int c = lane; c < W; c += 32) acc += slot[k * W + c];
    __syncwarp();
    if (w + D < mine) issue(w + D);
  }
  if (acc == 12345.678) out[0] = acc;
}

// The same gathers as coalesced LSU loads (each lane one 8/16-byte piece of the
// segment), U rows in flight per warp through registers.
template <int W, int U>
__global__ void __launch_bounds__(256, 4)
gather_lsu(const double *__restrict__ X, int64_t ld, int64_t rows, int64_t gathers, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t g = gw * U; g < gathers; g += nwarps * U) {
    double v[U][W / 32];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = (int64_t)(mix((uint64_t)(g + u)) % (uint64_t)rows);
#pragma unroll
      for (int c = 0; c < W / 32; ++c) v[u][c] = __ldg(X + j * ld + lane * (W / 32) + c);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < W / 32; ++c) acc += v[u][c];
  }
  if (acc == 12345.678) out[0] = acc;
}

static EncodeFn g_enc;
static double *g_X, *g_out;
static size_t g_bytes;

template <int W, int WAVE, int D>
static void run_tma(int64_t ld) {
  const int64_t rows = (int64_t)(g_bytes / (ld * 8));
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)W, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g_X, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return; }
  constexpr int warp_d = D * WAVE * W + (WAVE * D / 2 + 15) / 16 * 16 + 16;
  const size_t smem = (size_t)8 * warp_d * 8;
  auto kern = gather_tma<W, WAVE, D>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 256, smem);
  if (nb < 1) { printf("W=%d WAVE=%d D=%d: does not fit\n", W, WAVE, D); return; }
  const int grid = 148 * nb;
  const int64_t total_bytes = 200ll << 30;  // 200 GiB of gathers per launch
  const int64_t waves = total_bytes / (WAVE * W * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    kern<<<grid, 256, smem>>>(tm, rows, waves, g_out);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e != cudaSuccess) { printf("kernel error %s\n", cudaGetErrorString(e)); exit(1); }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("{\"engine\": \"tma_gather4\", \"segment_bytes\": %d, \"row_stride_bytes\": %lld, \"rows_per_wave\": %d, "
         "\"waves_in_flight\": %d, \"warps_per_sm\": %d, \"bytes_in_flight_per_sm\": %d, \"ms\": %.3f, \"GBs\": %.1f}\n",
         W * 8, (long long)ld * 8, WAVE, D, nb * 8, nb * 8 * D * WAVE * W * 8, best,
         (double)waves * WAVE * W * 8 / best * 1e-6);
  fflush(stdout);
}

template <int W, int U>
static void run_lsu(int64_t ld) {
  const int64_t rows = (int64_t)(g_bytes / (ld * 8));
  auto kern = gather_lsu<W, U>;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 256, 0);
  const int64_t gathers = (200ll << 30) / (W * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kern<<<148 * nb, 256>>>(g_X, ld, rows, gathers, g_out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  printf("{\"engine\": \"lsu\", \"segment_bytes\": %d, \"row_stride_bytes\": %lld, \"rows_in_flight_per_warp\": %d, "
         "\"warps_per_sm\": %d, \"ms\": %.3f, \"GBs\": %.1f}\n",
         W * 8, (long long)ld * 8, U, nb * 8, best, (double)gathers * W * 8 / best * 1e-6);
  fflush(stdout);
}

__global__ void fill(double *x, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] = (double)(i & 1023);
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&g_enc, cudaEnableDefault, &q);
  if (!g_enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  g_bytes = 32ull << 30;
  if (cudaMalloc(&g_X, g_bytes) != cudaSuccess || cudaMalloc(&g_out, 64) != cudaSuccess) {
    printf("alloc failed\n"); return 1;
  }
  fill<<<148 * 8, 256>>>(g_X, g_bytes / 8);
  cudaDeviceSynchronize();
  // 16-column (128 B), 32-column (256 B), 64-column (512 B) segments, packed
  // rows and 1 KB-stride rows (a tile of a 128-column block); 8 KB and 16 KB in
  // flight per warp
  run_tma<16, 32, 1>(16);  run_tma<16, 32, 2>(16);
  run_tma<32, 32, 1>(32);  run_tma<32, 16, 2>(32);  run_tma<32, 32, 2>(32);  run_tma<32, 16, 1>(32);
  run_tma<32, 32, 1>(128); run_tma<32, 32, 2>(128);
  run_tma<64, 16, 1>(64);  run_tma<64, 8, 2>(64);   run_tma<64, 16, 2>(64);
  run_tma<64, 16, 1>(128); run_tma<64, 16, 2>(128);
  run_tma<128, 8, 1>(128); run_tma<128, 8, 2>(128);
  run_lsu<32, 8>(32);  run_lsu<32, 16>(32);
  run_lsu<64, 8>(64);  run_lsu<64, 8>(128);
  run_lsu<128, 8>(128);
  return 0;
}
