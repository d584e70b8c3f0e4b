// Feasibility probe: TMA tile::gather4 of fp64 rows (sm_100a).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
template <int W>
__global__ void k(const __grid_constant__ CUtensorMap tm, const int* rows, double* out) {
  __shared__ alignas(128) double buf[4 * W];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(4 * W * 8));
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"((uint32_t)__cvta_generic_to_shared(buf)), "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(b) : "memory");
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" :: "r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * W; i += blockDim.x) out[i] = buf[i];
}
template <int W>
int run(EncodeFn enc, int ld, int boxrows) {
  const int n = 100000;
  std::vector<double> h((size_t)n * ld);
  for (size_t i = 0; i < (size_t)n; ++i) for (int c = 0; c < ld; ++c) h[i * ld + c] = i * 1000.0 + c;
  double *X, *out; int *rows;
  cudaMalloc(&X, h.size() * 8); cudaMalloc(&out, 4 * W * 8); cudaMalloc(&rows, 16);
  cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  int hr[4] = {5, 99999, 0, 17}; cudaMemcpy(rows, hr, 16, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)boxrows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("W=%d ld=%d boxrows=%d encode failed %d\n", W, ld, boxrows, (int)r); return 1; }
  k<W><<<1, 128>>>(tm, rows, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("W=%d kernel error %s\n", W, cudaGetErrorString(e)); return 1; }
  std::vector<double> o(4 * W); cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int q = 0; q < 4; ++q) for (int c = 0; c < W; ++c) if (o[q * W + c] != hr[q] * 1000.0 + c) ++bad;
  printf("W=%d ld=%d boxrows=%d bad=%d  o[0]=%g o[W]=%g o[2W]=%g o[3W+1]=%g\n", W, ld, boxrows, bad, o[0], o[W], o[2*W], o[3*W+1]);
  cudaFree(X); cudaFree(out); cudaFree(rows);
  return bad != 0;
}
int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no encode fn\n"); return 1; }
  run<32>(enc, 32, 1); run<64>(enc, 64, 1); run<128>(enc, 128, 1); run<32>(enc, 40, 1); run<32>(enc, 32, 4);
  return 0;
}
