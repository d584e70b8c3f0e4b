// L2 residency experiment (round 2): can a hot set of gathered rows be kept
// in the B200's L2 while a cold gather stream and row streams pass through?
//
// Synthetic version of the KPM step's access pattern: a 16 GiB block of
// 512-byte rows (one 64-column fp64 tile); each warp gathers rows, a fraction
// `p_hot` of them uniform over the first `hot_rows` rows (the "hub" rows), the
// rest uniform over the whole block; plus a streamed read of a second block
// (the own-row T_k / T_{k-1} streams).  Variants:
//   0 plain loads
//   1 hot rows ld.L2::cache_hint evict_last, everything else evict_first
//   2 persisting access-policy window over the hot rows (set-aside = max)
//   3 = 2 + evict_first on cold gathers and streams
//   4 hot evict_last only (cold/streams plain)
//   5 = 1 (reserved)
//   6 hot plain (evict_normal), cold gathers and streams evict_first, no window
//   7 hot evict_last, cold gathers evict_first, streams plain
//   10-13 the gathers as TMA bulk copies (see gather_tma)
// Every variant also writes one 512-byte row per 8 gathers (the T_{k+1} stream),
// with evict_first where the variant streams with evict_first.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2policy l2policy.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <int V>
__global__ void __launch_bounds__(256) gather(const double2 *__restrict__ blk, int64_t rows,
                                              int64_t hot_rows, uint32_t p_hot32,
                                              int64_t n_gathers, const double2 *__restrict__ strm,
                                              int64_t strm_rows, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t pl, pf;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  double acc = 0.0;
  const int64_t per = 8;  // gathers per stream row (~ degree 8 per own row)
  for (int64_t g0 = warp * per; g0 < n_gathers; g0 += nwarps * per) {
    // stream: own row of the second block
    const int64_t srow = (g0 / per) % strm_rows;
    double2 s;
    const double2 *sp = strm + srow * 32 + lane;
    constexpr bool SF = (V == 1 || V == 3 || V == 5 || V == 6);
    if (SF)
      asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                   : "=d"(s.x), "=d"(s.y) : "l"(sp), "l"(pf));
    else
      s = __ldg(sp);
    acc += s.x + s.y;
    {  // the written stream (second half of the stream block)
      double2 *wp = const_cast<double2 *>(strm) + (strm_rows + srow) * 32 + lane;
      if (SF)
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(wp), "d"(s.x),
                     "d"(s.y), "l"(pf) : "memory");
      else
        *wp = s;
    }
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const uint64_t h = mix((uint64_t)(g0 + q));
      const bool hot = (uint32_t)h < p_hot32;
      const int64_t row = hot ? (int64_t)((h >> 32) % (uint64_t)hot_rows)
                              : (int64_t)((h >> 32) % (uint64_t)rows);
      const double2 *rp = blk + row * 32 + lane;
      double2 v;
      if (V == 1 || V == 5 || V == 7) {
        const uint64_t pol = hot ? pl : pf;
        asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(v.x), "=d"(v.y) : "l"(rp), "l"(pol));
      } else if (V == 3 || V == 6) {
        if (hot) v = __ldg(rp);
        else
          asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                       : "=d"(v.x), "=d"(v.y) : "l"(rp), "l"(pf));
      } else if (V == 4) {
        if (hot)
          asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                       : "=d"(v.x), "=d"(v.y) : "l"(rp), "l"(pl));
        else v = __ldg(rp);
      } else {
        v = __ldg(rp);
      }
      acc += v.x * v.y;
    }
  }
  if (acc == 123.456) out[0] = acc;
}


// The same access pattern with the gathers issued as TMA bulk copies
// (cp.async.bulk global -> shared, one per row, completion on an mbarrier), as
// the step kernel's TMA paths do.  T: 10 plain, 11 hot evict_last / cold and
// streams evict_first (cache_hint operand; 15: the same with the persisting
// set-aside configured), 14 cold and streams evict_first only (16: with the
// set-aside), 12 persisting window + plain
// copies, 13 persisting window + evict_first on cold copies and streams.
template <int T>
__global__ void __launch_bounds__(256) gather_tma(const double2 *__restrict__ blk, int64_t rows,
                                                  int64_t hot_rows, uint32_t p_hot32,
                                                  int64_t n_gathers,
                                                  const double2 *__restrict__ strm,
                                                  int64_t strm_rows, double *out) {
  __shared__ alignas(128) double2 buf[8][8][32];
  __shared__ alignas(8) uint64_t bars[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  uint64_t pl, pf;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  double acc = 0.0;
  uint32_t phase = 0;
  const int64_t per = 8;
  constexpr bool SF = (T == 11 || T == 13 || T == 14 || T == 15 || T == 16);
  for (int64_t g0 = warp * per; g0 < n_gathers; g0 += nwarps * per) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4096)
                   : "memory");
    __syncwarp();
    if (lane < per) {
      const uint64_t h = mix((uint64_t)(g0 + lane));
      const bool hot = (uint32_t)h < p_hot32;
      const int64_t row = hot ? (int64_t)((h >> 32) % (uint64_t)hot_rows)
                              : (int64_t)((h >> 32) % (uint64_t)rows);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[w][lane][0]);
      const double2 *src = blk + row * 32;
      const bool hinted = (T == 11 || T == 15) || ((T == 13 || T == 14 || T == 16) && !hot);
      if (hinted) {
        const uint64_t pol = ((T == 11 || T == 15) && hot) ? pl : pf;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(dst), "l"(src), "r"(512), "r"(bar), "l"(pol)
            : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(dst), "l"(src), "r"(512), "r"(bar) : "memory");
      }
    }
    const int64_t srow = (g0 / per) % strm_rows;
    double2 s;
    const double2 *sp = strm + srow * 32 + lane;
    if (SF)
      asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                   : "=d"(s.x), "=d"(s.y) : "l"(sp), "l"(pf));
    else
      s = __ldg(sp);
    acc += s.x + s.y;
    double2 *wp = const_cast<double2 *>(strm) + (strm_rows + srow) * 32 + lane;
    if (SF)
      asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(wp), "d"(s.x),
                   "d"(s.y), "l"(pf) : "memory");
    else
      *wp = s;
    asm volatile(
        "{\n\t.reg .pred P;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(bar), "r"(phase) : "memory");
    phase ^= 1;
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const double2 v = buf[w][q][lane];
      acc += v.x * v.y;
    }
    __syncwarp();
  }
  if (acc == 123.456) out[0] = acc;
}

template <int T>
static float run_tma(const double2 *blk, int64_t rows, int64_t hot_rows, double p_hot, int64_t ng,
                     const double2 *strm, int64_t srows, double *out, int sms) {
  const uint32_t p32 = (uint32_t)(p_hot * 4294967296.0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather_tma<T><<<sms * 6, 256>>>(blk, rows, hot_rows, p32, ng / 4, strm, srows, out);  // warm
  cudaEventRecord(a);
  gather_tma<T><<<sms * 6, 256>>>(blk, rows, hot_rows, p32, ng, strm, srows, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

template <int V>
static float run(const double2 *blk, int64_t rows, int64_t hot_rows, double p_hot, int64_t ng,
                 const double2 *strm, int64_t srows, double *out, int sms) {
  const uint32_t p32 = (uint32_t)(p_hot * 4294967296.0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<V><<<sms * 8, 256>>>(blk, rows, hot_rows, p32, ng / 4, strm, srows, out);  // warm
  cudaEventRecord(a);
  gather<V><<<sms * 8, 256>>>(blk, rows, hot_rows, p32, ng, strm, srows, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main(int argc, char **argv) {
  const double hot_mb = argc > 1 ? atof(argv[1]) : 64.0;
  const double p_hot = argc > 2 ? atof(argv[2]) : 0.5;
  const int only = argc > 3 ? atoi(argv[3]) : -1;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  printf("L2 %d MB, persisting max %d MB, accessPolicyMaxWindowSize %d MB\n",
         prop.l2CacheSize >> 20, (int)(prop.persistingL2CacheMaxSize >> 20),
         prop.accessPolicyMaxWindowSize >> 20);
  const int64_t row_bytes = 512;
  const int64_t rows = (16ll << 30) / row_bytes;
  const int64_t srows = (4ll << 30) / row_bytes;  // read half; an equal written half follows
  const int64_t hot_rows = (int64_t)(hot_mb * (1 << 20)) / row_bytes;
  double2 *blk, *strm;
  double *out;
  if (cudaMalloc(&blk, rows * row_bytes) || cudaMalloc(&strm, 2 * srows * row_bytes) ||
      cudaMalloc(&out, 8)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(blk, 0, rows * row_bytes);
  cudaMemset(strm, 0, 2 * srows * row_bytes);
  const int64_t ng = 400ll << 20;  // gathers per timed launch (~200 GB)
  const double bytes = (double)ng * row_bytes * (1.0 + 2.0 / 8);
  for (int v = 0; v <= 16; ++v) {
    if (v == 5 || v == 8 || v == 9) continue;
    if (only >= 0 && v != only) continue;
    cudaStreamAttrValue attr = {};
    if (v == 15 || v == 16)  // set-aside only, no window
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize);
    if (v == 2 || v == 3 || v == 12 || v == 13) {
      size_t setaside = prop.persistingL2CacheMaxSize;
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside);
      attr.accessPolicyWindow.base_ptr = blk;
      size_t win = (size_t)hot_rows * row_bytes;
      if (win > (size_t)prop.accessPolicyMaxWindowSize) win = prop.accessPolicyMaxWindowSize;
      attr.accessPolicyWindow.num_bytes = win;
      attr.accessPolicyWindow.hitRatio = win > setaside ? (float)setaside / win : 1.0f;
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &attr);
    }
    float ms = 0;
    switch (v) {
      case 0: ms = run<0>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 1: ms = run<1>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 2: ms = run<2>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 3: ms = run<3>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 4: ms = run<4>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 6: ms = run<6>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 7: ms = run<7>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 10: ms = run_tma<10>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 11: ms = run_tma<11>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 12: ms = run_tma<12>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 13: ms = run_tma<13>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 14: ms = run_tma<14>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 15: ms = run_tma<15>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
      case 16: ms = run_tma<16>(blk, rows, hot_rows, p_hot, ng, strm, srows, out, prop.multiProcessorCount); break;
    }
    if (v == 2 || v == 3 || v == 12 || v == 13) {
      attr.accessPolicyWindow.num_bytes = 0;
      cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &attr);
      cudaCtxResetPersistingL2Cache();
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    }
    if (v == 15 || v == 16) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    cudaError_t e = cudaGetLastError();
    printf("variant %d hot %.0f MB p_hot %.2f: %.2f ms, %.0f GB/s requested, ideal DRAM share %.2f %s\n",
           v, hot_mb, p_hot, ms, bytes / ms / 1e6, 1.0 - p_hot * 8.0 / 10.0,
           e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
