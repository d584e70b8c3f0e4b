// Device graph loader: edges -> symmetric CSR with
// int64 row_ptr, int32 col_idx (sorted per row) and fp64 d^-1/2, plus the
// load-balanced row-chunk schedule used by the recurrence kernels.
//
// Reference semantics (paths relative to /root/reference/pkg/src/netdos/):
//   graph.py:69-81  _csr_from_canonical: both directions of each canonical
//                   pair (a loop once), lexsort by (row, col), row_ptr by
//                   counting + cumsum;
//   graph.py:130-160 build_csr: canonicalise + merge duplicates;
//   graph.py:47-54  degrees (unit weights, loop counted once);
//   operators.py:108-110 dinv = deg > 0 ? 1/sqrt(deg) : 0 (IEEE sqrt, div).
//
// B200 design: one 64-bit key per stored entry, key = row << s | col with
// 2^s > n, radix-sorted on exactly 2s bits (CUB onesweep over HBM), unique'd
// in place, then row_ptr from the row boundaries of the sorted keys -- no
// atomics, so the CSR is deterministic and bit-identical to the reference.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "kpm_internal.cuh"

namespace kpm {

static constexpr uint64_t kSentinel = ~0ull;

static int key_bits(int64_t n) {
  int s = 1;
  while ((int64_t(1) << s) <= n) ++s;  // 2^s > n: row 2^s-1 never occurs
  return s;
}

__global__ void edges_to_keys(const int64_t *__restrict__ u,
                              const int64_t *__restrict__ v, int64_t m,
                              int64_t n, int s, int keep_loops,
                              uint64_t *__restrict__ keys, int *bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[e], b = v[e];
    uint64_t k0 = kSentinel, k1 = kSentinel;
    if (a < 0 || b < 0 || a >= n || b >= n) {
      atomicOr(bad, 1);
    } else if (a == b) {
      if (keep_loops) k0 = ((uint64_t)a << s) | (uint64_t)a;
    } else {
      k0 = ((uint64_t)a << s) | (uint64_t)b;
      k1 = ((uint64_t)b << s) | (uint64_t)a;
    }
    keys[2 * e] = k0;
    keys[2 * e + 1] = k1;
  }
}

// Philox4x32-10 (Salmon et al., SC'11): the R-MAT harness generator.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0,
                                              uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ void rmat_draw(uint64_t e, int scale, uint32_t k0,
                                          uint32_t k1, uint32_t ta,
                                          uint32_t tab, uint32_t tabc,
                                          int64_t &a, int64_t &b) {
  uint32_t w[4];
  a = 0;
  b = 0;
  for (int l = 0; l < scale; ++l) {
    if ((l & 3) == 0) {
      w[0] = (uint32_t)e;
      w[1] = (uint32_t)(e >> 32);
      w[2] = (uint32_t)(l >> 2);
      w[3] = 0u;
      philox4x32_10(w, k0, k1);
    }
    uint32_t r = w[l & 3];
    int bu = r >= tab;
    int bv = (r >= ta && r < tab) || r >= tabc;
    a = (a << 1) | bu;
    b = (b << 1) | bv;
  }
}

__global__ void rmat_edges_kernel(int scale, uint64_t seed, uint32_t ta,
                                  uint32_t tab, uint32_t tabc, int64_t e0,
                                  int64_t count, int64_t *u, int64_t *v) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    rmat_draw((uint64_t)(e0 + t), scale, k0, k1, ta, tab, tabc, a, b);
    u[t] = a;
    v[t] = b;
  }
}

__global__ void rmat_keys_kernel(int scale, uint64_t seed, uint32_t ta,
                                 uint32_t tab, uint32_t tabc, int64_t m,
                                 int s, int64_t lo, int64_t hi,
                                 uint64_t *__restrict__ keys) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    rmat_draw((uint64_t)e, scale, k0, k1, ta, tab, tabc, a, b);
    uint64_t k0v = kSentinel, k1v = kSentinel;
    if (a != b) {  // rows outside [lo, hi) belong to other partitions
      if (a >= lo && a < hi) k0v = ((uint64_t)(a - lo) << s) | (uint64_t)b;
      if (b >= lo && b < hi) k1v = ((uint64_t)(b - lo) << s) | (uint64_t)a;
    }
    keys[2 * e] = k0v;
    keys[2 * e + 1] = k1v;
  }
}

// row_ptr[r] = index of the first key with row >= r (keys sorted, unique).
__global__ void keys_to_csr(const uint64_t *__restrict__ keys, int64_t nnz,
                            int s, int64_t *__restrict__ row_ptr,
                            int32_t *__restrict__ col) {
  const uint64_t mask = (uint64_t(1) << s) - 1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = keys[k];
    int64_t r = (int64_t)(key >> s);
    int64_t rp = k > 0 ? (int64_t)(keys[k - 1] >> s) : -1;
    for (int64_t q = rp + 1; q <= r; ++q) row_ptr[q] = k;
    col[k] = (int32_t)(key & mask);
  }
}

__global__ void fill_tail_rows(int64_t *row_ptr, int64_t from, int64_t n,
                               int64_t nnz) {
  for (int64_t q = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       q <= n; q += (int64_t)gridDim.x * blockDim.x)
    row_ptr[q] = nnz;
}

// graph.py:47-54 + operators.py:108-109 with IEEE-exact sqrt and division.
__global__ void dinv_kernel(const int64_t *__restrict__ row_ptr, int64_t n,
                            double *__restrict__ dinv,
                            unsigned long long *max_deg) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = row_ptr[i + 1] - row_ptr[i];
    dinv[i] = d > 0 ? __ddiv_rn(1.0, __dsqrt_rn((double)d)) : 0.0;
    if ((unsigned long long)d > local) local = (unsigned long long)d;
  }
  for (int o = 16; o > 0; o >>= 1)
    local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0) atomicMax(max_deg, local);
}

// Rows per floor(log2(degree)) bucket (degree >= 1): the step kernel's L2
// policy picks its "hot" (re-gathered) rows from it.
__global__ void deg_hist_kernel(const int64_t *__restrict__ row_ptr, int64_t n,
                                unsigned long long *__restrict__ hist) {
  __shared__ unsigned long long sh[kDegBuckets];
  for (int b = threadIdx.x; b < kDegBuckets; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = row_ptr[i + 1] - row_ptr[i];
    if (d > 0) atomicAdd(&sh[deg_bucket((unsigned long long)d)], 1ull);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kDegBuckets; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, sh[b]);
}

// Chunk c covers rows [start[c], start[c+1]); boundaries split the prefix of
// the per-row cost min(deg, heavy) + kRowCost evenly (heavy rows are worked
// by their own CTAs, kpm_step.cu).  Depends on the graph only.
static constexpr int64_t kRowCost = 8;
static constexpr int64_t kMaxChunkCost = 16384;

__global__ void row_cost_kernel(const int64_t *__restrict__ row_ptr, int64_t n,
                                int64_t heavy, int64_t *__restrict__ cost,
                                int32_t *__restrict__ is_heavy) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = row_ptr[i + 1] - row_ptr[i];
    bool h = d >= heavy;
    cost[i] = (h ? 0 : d) + kRowCost;
    is_heavy[i] = h ? 1 : 0;
  }
}

__global__ void chunk_bounds(const int64_t *__restrict__ prefix, int64_t n,
                             int32_t n_chunks, int64_t target,
                             int32_t *__restrict__ start) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_chunks) return;
  if (c == 0) { start[0] = 0; return; }
  if (c == n_chunks) { start[c] = (int32_t)n; return; }
  int64_t want = (int64_t)c * target;
  int64_t lo = 0, hi = n;  // first i with prefix(i) >= want
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (prefix[mid] >= want) hi = mid; else lo = mid + 1;
  }
  start[c] = (int32_t)lo;
}

// per-chunk largest light-row cost (for the work-queue order)
__global__ void chunk_maxdeg(const int64_t *__restrict__ row_ptr,
                             const int32_t *__restrict__ start, int32_t n_chunks,
                             int64_t heavy, int64_t *__restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_chunks;
       c += (int64_t)gridDim.x * blockDim.x) {
    int64_t mx = 0;
    for (int32_t i = start[c]; i < start[c + 1]; ++i) {
      int64_t d = row_ptr[i + 1] - row_ptr[i];
      if (d < heavy && d > mx) mx = d;
    }
    out[c] = mx;
  }
}

__global__ void gather_degrees(const int64_t *__restrict__ row_ptr,
                               const int32_t *__restrict__ rows, int64_t k,
                               int64_t *__restrict__ deg) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < k;
       t += (int64_t)gridDim.x * blockDim.x)
    deg[t] = row_ptr[rows[t] + 1] - row_ptr[rows[t]];
}

static int grid_for(int64_t work, int threads = 256) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return (int)b;
}

int finish_graph(kpm_graph *g) {
  cudaStream_t st = g->ctx->stream;
  const int64_t n = g->n;
  unsigned long long *dmax = nullptr;
  KPM_CUDA(cudaMallocAsync(&dmax, sizeof(unsigned long long), st));
  KPM_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
  if (n > 0)
    dinv_kernel<<<grid_for(n), 256, 0, st>>>(g->row_ptr, n, g->dinv, dmax);
  unsigned long long hmax = 0;
  KPM_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(hmax), cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaFreeAsync(dmax, st));
  {
    unsigned long long *dh = nullptr;
    KPM_CUDA(cudaMallocAsync(&dh, sizeof(unsigned long long) * kDegBuckets, st));
    KPM_CUDA(cudaMemsetAsync(dh, 0, sizeof(unsigned long long) * kDegBuckets, st));
    if (n > 0) deg_hist_kernel<<<grid_for(n), 256, 0, st>>>(g->row_ptr, n, dh);
    KPM_CUDA(cudaMemcpyAsync(g->deg_hist, dh, sizeof(unsigned long long) * kDegBuckets,
                             cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaFreeAsync(dh, st));
  }

  // capped row costs -> prefix (n+1) ; heavy-row flags
  // A row goes to the hub path (column slices on dedicated warps) only when one
  // warp walking it would set the span of the step: the slices gather 128-byte
  // pieces through cp.async and cost ~4x the light path per nonzero (work-item
  // traces, profiles/r02_ncu_summary.md section 6), so the bar is the degree at
  // which a single light row takes about half a step: nnz / 2048 (C3: 254k ->
  // only the 406k-degree row; C5: 1.03M), never below kHeavyDegree.  Graph-only.
  g->heavy_threshold = kHeavyDegree;
  if (g->nnz / 2048 > g->heavy_threshold) g->heavy_threshold = g->nnz / 2048;
  if (const char *e = getenv("KPM_HEAVY_DEGREE")) {  // tests force the hub path
    long long v = atoll(e);
    if (v > 0) g->heavy_threshold = v;
  }
  int64_t *prefix = nullptr;
  int32_t *flags = nullptr;
  KPM_CUDA(cudaMalloc(&prefix, sizeof(int64_t) * (n + 1)));
  KPM_CUDA(cudaMalloc(&flags, sizeof(int32_t) * (n > 0 ? n : 1)));
  KPM_CUDA(cudaMemsetAsync(prefix, 0, sizeof(int64_t) * (n + 1), st));
  if (n > 0) {
    row_cost_kernel<<<grid_for(n), 256, 0, st>>>(g->row_ptr, n, g->heavy_threshold, prefix,
                                                 flags);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, prefix, prefix, n + 1, st);
    void *tmp = nullptr;
    KPM_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, prefix, prefix, n + 1, st);
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaFreeAsync(tmp, st));
  }
  int64_t total = 0;
  KPM_CUDA(cudaMemcpyAsync(&total, prefix + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  // a fixed denominator (148 SMs x 128) keeps chunks independent of the device
  // and of the probe count, so reductions are reproducible.
  // Big graphs cap the chunk cost instead (more chunks): the last chunks of
  // the queue set the launch's tail, so a chunk must stay short next to the
  // step (C5: 14 ms chunks at 148*128 of them, profiles/r01_trace_report.json).
  int64_t target = (total + 148 * 128 - 1) / (148 * 128);
  int64_t cap = kMaxChunkCost;
  if (const char *e = getenv("KPM_CHUNK_COST")) cap = atoll(e);
  if (cap > 0 && target > cap) target = cap;
  if (target < 256) target = 256;
  int64_t nch = (total + target - 1) / target;
  if (nch < 1) nch = 1;
  std::vector<int32_t> bounds(nch + 1);
  {
    int32_t *dcs = nullptr;
    KPM_CUDA(cudaMalloc(&dcs, sizeof(int32_t) * (nch + 1)));
    chunk_bounds<<<(int)((nch + 1 + 255) / 256), 256, 0, st>>>(prefix, n, (int32_t)nch, target,
                                                                 dcs);
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaMemcpyAsync(bounds.data(), dcs, sizeof(int32_t) * (nch + 1),
                             cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    cudaFree(dcs);
  }
  std::vector<int32_t> heavy_sorted;

  // heavy rows, ordered by (degree desc, row asc): deterministic, graph-only
  g->n_heavy = 0;
  if (n > 0 && (int64_t)hmax >= g->heavy_threshold) {
    int32_t *sel = nullptr, *dnum = nullptr;
    KPM_CUDA(cudaMalloc(&sel, sizeof(int32_t) * n));
    KPM_CUDA(cudaMalloc(&dnum, sizeof(int32_t)));
    size_t tb = 0;
    thrust::counting_iterator<int32_t> rows(0);
    cub::DeviceSelect::Flagged(nullptr, tb, rows, flags, sel, dnum, (int)n, st);
    void *tmp = nullptr;
    KPM_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceSelect::Flagged(tmp, tb, rows, flags, sel, dnum, (int)n, st);
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaFreeAsync(tmp, st));
    int32_t nh = 0;
    KPM_CUDA(cudaMemcpyAsync(&nh, dnum, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> hrows(nh);
    std::vector<int64_t> hdeg(nh);
    if (nh > 0) {
      int64_t *ddeg = nullptr;
      KPM_CUDA(cudaMalloc(&ddeg, sizeof(int64_t) * nh));
      gather_degrees<<<grid_for(nh), 256, 0, st>>>(g->row_ptr, sel, nh, ddeg);
      KPM_CUDA(cudaMemcpyAsync(hrows.data(), sel, sizeof(int32_t) * nh, cudaMemcpyDeviceToHost, st));
      KPM_CUDA(cudaMemcpyAsync(hdeg.data(), ddeg, sizeof(int64_t) * nh, cudaMemcpyDeviceToHost, st));
      KPM_CUDA(cudaStreamSynchronize(st));
      cudaFree(ddeg);
      std::vector<int32_t> order(nh);
      for (int32_t t = 0; t < nh; ++t) order[t] = t;
      std::stable_sort(order.begin(), order.end(),
                       [&](int32_t a, int32_t b) { return hdeg[a] > hdeg[b]; });
      std::vector<int32_t> sorted(nh);
      for (int32_t t = 0; t < nh; ++t) sorted[t] = hrows[order[t]];
      KPM_CUDA(cudaMalloc(&g->heavy_rows, sizeof(int32_t) * nh));
      KPM_CUDA(cudaMemcpy(g->heavy_rows, sorted.data(), sizeof(int32_t) * nh,
                          cudaMemcpyHostToDevice));
      heavy_sorted = sorted;
    }
    g->n_heavy = nh;
    cudaFree(sel);
    cudaFree(dnum);
  }
  // every hub row becomes a singleton chunk (skipped by the light stream),
  // so a light chunk is a run of light rows whose nonzeros can be streamed
  for (int32_t h : heavy_sorted) {
    bounds.push_back(h);
    bounds.push_back(h + 1);
  }
  std::sort(bounds.begin(), bounds.end());
  bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
  nch = (int64_t)bounds.size() - 1;
  g->n_chunks = (int32_t)nch;
  KPM_CUDA(cudaMalloc(&g->chunk_start, sizeof(int32_t) * (nch + 1)));
  KPM_CUDA(cudaMemcpy(g->chunk_start, bounds.data(), sizeof(int32_t) * (nch + 1),
                      cudaMemcpyHostToDevice));
  {
    // queue order: chunks holding the longest rows first (ties by id), so a
    // long row never starts late; partial slots stay indexed by chunk id
    int64_t *dmx = nullptr;
    KPM_CUDA(cudaMalloc(&dmx, sizeof(int64_t) * (nch > 0 ? nch : 1)));
    if (nch > 0)
      chunk_maxdeg<<<grid_for(nch), 256, 0, st>>>(g->row_ptr, g->chunk_start, g->n_chunks,
                                                  g->heavy_threshold, dmx);
    std::vector<int64_t> mx(nch);
    KPM_CUDA(cudaMemcpyAsync(mx.data(), dmx, sizeof(int64_t) * nch, cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    cudaFree(dmx);
    std::vector<int32_t> order(nch);
    for (int64_t c = 0; c < nch; ++c) order[c] = (int32_t)c;
    // longest row first (row-id order measured slower, profiles/r01_chunk_order_exp.log)
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t x, int32_t y) { return mx[x] > mx[y]; });
    KPM_CUDA(cudaMalloc(&g->chunk_order, sizeof(int32_t) * (nch > 0 ? nch : 1)));
    KPM_CUDA(cudaMemcpy(g->chunk_order, order.data(), sizeof(int32_t) * nch,
                        cudaMemcpyHostToDevice));
  }
  KPM_CUDA(cudaStreamSynchronize(st));
  cudaFree(prefix);
  cudaFree(flags);
  g->max_degree = (int64_t)hmax;
  return KPM_OK;
}

// keys: 2m entries (sentinels allowed); consumes and frees keys/alt.
static int keys_to_graph(kpm_ctx *ctx, int64_t n, int s, uint64_t *keys,
                         uint64_t *alt, int64_t nkeys, kpm_graph **out,
                         int64_t row0 = 0, int64_t n_global = -1) {
  const int sort_bits = s + key_bits(n);
  cudaStream_t st = ctx->stream;
  int64_t nnz = 0;
  if (nkeys > 0) {
    cub::DoubleBuffer<uint64_t> db(keys, alt);
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, nkeys, 0, sort_bits, st);
    void *tmp = nullptr;
    KPM_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, nkeys, 0, sort_bits, st);
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaFreeAsync(tmp, st));
    uint64_t *sorted = db.Current(), *other = db.Alternate();
    int64_t *d_nsel = nullptr;
    KPM_CUDA(cudaMallocAsync(&d_nsel, sizeof(int64_t), st));
    tmp_bytes = 0;
    cub::DeviceSelect::Unique(nullptr, tmp_bytes, sorted, other, d_nsel, nkeys, st);
    KPM_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, other, d_nsel, nkeys, st);
    KPM_CUDA(cudaGetLastError());
    KPM_CUDA(cudaFreeAsync(tmp, st));
    int64_t nsel = 0;
    KPM_CUDA(cudaMemcpyAsync(&nsel, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaFreeAsync(d_nsel, st));
    uint64_t last = 0;
    KPM_CUDA(cudaStreamSynchronize(st));
    if (nsel > 0) {
      KPM_CUDA(cudaMemcpy(&last, other + nsel - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    }
    // the sentinel (all sorted bits set) sorts last and is not a real key
    nnz = (nsel > 0 && last == kSentinel) ? nsel - 1 : nsel;
    keys = other;  // unique keys live here now
    alt = sorted;
  }
  KPM_CHECK_ARG(n < (int64_t(1) << 31), "n must be < 2^31 (int32 col_idx)");
  kpm_graph *g = new kpm_graph();
  g->ctx = ctx;
  g->n = n;
  g->nnz = nnz;
  g->row0 = row0;
  g->n_global = n_global < 0 ? n : n_global;
  cudaError_t e1 = cudaMalloc(&g->row_ptr, sizeof(int64_t) * (n + 1));
  cudaError_t e2 = cudaMalloc(&g->col_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1));
  cudaError_t e3 = cudaMalloc(&g->dinv, sizeof(double) * (n > 0 ? n : 1));
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
    kpm_graph_free(g);
    set_error("graph allocation failed (n=%lld nnz=%lld)", (long long)n, (long long)nnz);
    return KPM_ENOMEM;
  }
  if (nnz > 0) {
    keys_to_csr<<<grid_for(nnz), 256, 0, st>>>(keys, nnz, s, g->row_ptr, g->col_idx);
    uint64_t lastkey = 0;
    KPM_CUDA(cudaMemcpyAsync(&lastkey, keys + nnz - 1, sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    int64_t last_row = (int64_t)(lastkey >> s);
    fill_tail_rows<<<grid_for(n - last_row), 256, 0, st>>>(g->row_ptr, last_row + 1, n, nnz);
  } else {
    fill_tail_rows<<<grid_for(n + 1), 256, 0, st>>>(g->row_ptr, 0, n, 0);
  }
  KPM_CUDA(cudaGetLastError());
  KPM_CUDA(cudaStreamSynchronize(st));
  if (keys) cudaFree(keys);
  if (alt) cudaFree(alt);
  int rc = finish_graph(g);
  if (rc != KPM_OK) {
    kpm_graph_free(g);
    return rc;
  }
  *out = g;
  return KPM_OK;
}

// ---- gather-ordered twin (degree-descending renumbering) -----------------
__global__ void relab_deg_keys(const int64_t *__restrict__ row_ptr, int64_t n,
                               uint32_t *__restrict__ deg, int32_t *__restrict__ row) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    deg[i] = (uint32_t)(row_ptr[i + 1] - row_ptr[i]);
    row[i] = (int32_t)i;
  }
}

__global__ void relab_invert(const int32_t *__restrict__ perm, int64_t n,
                             int32_t *__restrict__ iperm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    iperm[perm[i]] = (int32_t)i;
}

// one warp per (old) row: key = new_row << s | new_col
__global__ void relab_keys(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const int32_t *__restrict__ iperm, int64_t n, int s,
                           uint64_t *__restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t o = warp; o < n; o += nwarps) {
    const int64_t e0 = row_ptr[o], e1 = row_ptr[o + 1];
    if (e1 == e0) continue;
    const uint64_t hi = (uint64_t)(uint32_t)iperm[o] << s;
    for (int64_t e = e0 + lane; e < e1; e += 32) keys[e] = hi | (uint64_t)(uint32_t)iperm[col[e]];
  }
}

// The twin of an implicit, unpartitioned graph (see kpm_graph::relab); NULL
// when it cannot be built (explicit values, partitions, out of memory).
// Twin rows are degree-descending: thread e finds the first row whose degree is
// <= kDinvSteps - 1 - e (n when none) and that degree's d^-1/2.
__global__ void dinv_steps_kernel(const int64_t *__restrict__ row_ptr,
                                  const double *__restrict__ dinv, int64_t n,
                                  int32_t *__restrict__ step_id, double *__restrict__ step_val) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= kDinvSteps) return;
  const int64_t d = kDinvSteps - 1 - e;
  int64_t lo = 0, hi = n;  // first row in [0, n] with degree <= d
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (row_ptr[mid + 1] - row_ptr[mid] <= d) hi = mid;
    else lo = mid + 1;
  }
  step_id[e] = lo < n ? (int32_t)lo : 0x7fffffff;
  step_val[e] = lo < n ? dinv[lo] : 0.0;
}

kpm_graph *graph_relabelled(kpm_graph *g) {
  if (g->relab_state != 0) return g->relab;
  g->relab_state = -1;
  if (g->values || g->dinv_all || g->row0 != 0 || g->n_global != g->n || g->n < 2 || g->nnz < 1)
    return nullptr;
  cudaStream_t st = g->ctx->stream;
  const int64_t n = g->n, nnz = g->nnz;
  uint32_t *deg = nullptr, *deg2 = nullptr;
  int32_t *row = nullptr, *perm = nullptr, *iperm = nullptr;
  uint64_t *keys = nullptr, *alt = nullptr;
  void *tmp = nullptr;
  auto fail = [&]() -> kpm_graph * {
    cudaGetLastError();
    cudaFree(deg); cudaFree(deg2); cudaFree(row); cudaFree(perm); cudaFree(iperm);
    cudaFree(keys); cudaFree(alt); cudaFree(tmp);
    return nullptr;
  };
  if (cudaMalloc(&deg, 4 * n) || cudaMalloc(&deg2, 4 * n) || cudaMalloc(&row, 4 * n) ||
      cudaMalloc(&perm, 4 * n) || cudaMalloc(&iperm, 4 * n))
    return fail();
  relab_deg_keys<<<grid_for(n), 256, 0, st>>>(g->row_ptr, n, deg, row);
  size_t tb = 0;
  // stable: equal degrees keep ascending row ids
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, deg, deg2, row, perm, (int)n, 0, 32, st);
  if (cudaMalloc(&tmp, tb)) return fail();
  cub::DeviceRadixSort::SortPairsDescending(tmp, tb, deg, deg2, row, perm, (int)n, 0, 32, st);
  relab_invert<<<grid_for(n), 256, 0, st>>>(perm, n, iperm);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail();
  cudaFree(tmp); tmp = nullptr;
  cudaFree(deg); deg = nullptr;
  cudaFree(deg2); deg2 = nullptr;
  cudaFree(row); row = nullptr;
  if (cudaMalloc(&keys, 8 * nnz) || cudaMalloc(&alt, 8 * nnz)) return fail();
  const int s = key_bits(n);
  relab_keys<<<grid_for(n * 32), 256, 0, st>>>(g->row_ptr, g->col_idx, iperm, n, s, keys);
  if (cudaGetLastError() != cudaSuccess) return fail();
  kpm_graph *t = nullptr;
  const int rc = keys_to_graph(g->ctx, n, s, keys, alt, nnz, &t);  // frees keys / alt
  keys = alt = nullptr;
  if (rc != KPM_OK || !t || t->nnz != nnz) {
    if (t) kpm_graph_free(t);
    return fail();
  }
  t->perm = perm;
  t->iperm = iperm;
  t->relab_state = -1;  // a twin has no twin
  if (cudaMalloc(&t->dstep_id, sizeof(int32_t) * kDinvSteps) == cudaSuccess &&
      cudaMalloc(&t->dstep_val, sizeof(double) * kDinvSteps) == cudaSuccess) {
    dinv_steps_kernel<<<(kDinvSteps + 127) / 128, 128, 0, st>>>(t->row_ptr, t->dinv, n,
                                                                 t->dstep_id, t->dstep_val);
    if (cudaMemcpyAsync(&t->dstep_h, t->dstep_id, sizeof(int32_t), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(t->dstep_id); cudaFree(t->dstep_val);
      t->dstep_id = nullptr; t->dstep_val = nullptr;
      t->dstep_h = 0x7fffffff;
    }
  } else {
    cudaGetLastError();
    cudaFree(t->dstep_id);
    t->dstep_id = nullptr;
  }
  g->relab = t;
  g->relab_state = 1;
  return t;
}

__global__ void idx64_to_32(const int64_t *__restrict__ in, int64_t m,
                            int64_t n, int32_t *__restrict__ out, int *bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = in[e];
    if (x < 0 || x >= n) atomicOr(bad, 1);
    out[e] = (int32_t)x;
  }
}

__global__ void idx32_check(const int32_t *__restrict__ in, int64_t m, int64_t n, int *bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = in[e];
    if (x < 0 || x >= n) atomicOr(bad, 1);
  }
}

}  // namespace kpm

using namespace kpm;

extern "C" {

int kpm_graph_from_edges(kpm_ctx *ctx, int64_t n, const int64_t *u,
                         const int64_t *v, int64_t m, int keep_loops,
                         kpm_graph **out) {
  kpm::Nvtx nvtx_range_("kpm_graph_from_edges");
  KPM_CHECK_ARG(ctx && out && n >= 0 && m >= 0, "bad arguments");
  KPM_CHECK_ARG(m == 0 || (u && v), "u/v are NULL");
  KPM_CHECK_ARG(n < (int64_t(1) << 31), "n must be < 2^31 (int32 col_idx)");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  int s = key_bits(n);
  uint64_t *keys = nullptr, *alt = nullptr;
  if (m > 0) {
    DevBuf tu, tv;
    const void *du, *dv;
    KPM_TRY(stage_in(st, u, sizeof(int64_t) * m, tu, &du));
    KPM_TRY(stage_in(st, v, sizeof(int64_t) * m, tv, &dv));
    KPM_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * 2 * m));
    KPM_CUDA(cudaMalloc(&alt, sizeof(uint64_t) * 2 * m));
    int *bad = nullptr;
    KPM_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
    KPM_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    edges_to_keys<<<grid_for(m), 256, 0, st>>>((const int64_t *)du, (const int64_t *)dv,
                                               m, n, s, keep_loops, keys, bad);
    int hbad = 0;
    KPM_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaFreeAsync(bad, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    if (hbad) {
      cudaFree(keys);
      cudaFree(alt);
      set_error("node ids must be in [0, n)");
      return KPM_EINVAL;
    }
  }
  return keys_to_graph(ctx, n, s, keys, alt, 2 * m, out);
}

int kpm_graph_rmat(kpm_ctx *ctx, int scale, int64_t n_edges, uint64_t seed,
                   uint32_t ta, uint32_t tab, uint32_t tabc, kpm_graph **out) {
  kpm::Nvtx nvtx_range_("kpm_graph_rmat");
  KPM_CHECK_ARG(ctx && out && scale >= 1 && scale <= 30 && n_edges >= 0,
                "bad arguments");
  KPM_CUDA(cudaSetDevice(ctx->device));
  int64_t n = int64_t(1) << scale;
  int s = key_bits(n);
  uint64_t *keys = nullptr, *alt = nullptr;
  if (n_edges > 0) {
    KPM_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * 2 * n_edges));
    KPM_CUDA(cudaMalloc(&alt, sizeof(uint64_t) * 2 * n_edges));
    rmat_keys_kernel<<<grid_for(n_edges), 256, 0, ctx->stream>>>(
        scale, seed, ta, tab, tabc, n_edges, s, 0, n, keys);
    KPM_CUDA(cudaGetLastError());
  }
  return keys_to_graph(ctx, n, s, keys, alt, 2 * n_edges, out);
}

int kpm_graph_rmat_part(kpm_ctx *ctx, int scale, int64_t n_edges, uint64_t seed,
                        uint32_t ta, uint32_t tab, uint32_t tabc, int64_t row_lo,
                        int64_t row_hi, kpm_graph **out) {
  KPM_CHECK_ARG(ctx && out && scale >= 1 && scale <= 30 && n_edges >= 0, "bad arguments");
  const int64_t n = int64_t(1) << scale;
  KPM_CHECK_ARG(0 <= row_lo && row_lo <= row_hi && row_hi <= n, "bad row range");
  KPM_CUDA(cudaSetDevice(ctx->device));
  int s = key_bits(n);
  uint64_t *keys = nullptr, *alt = nullptr;
  if (n_edges > 0) {
    KPM_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * 2 * n_edges));
    KPM_CUDA(cudaMalloc(&alt, sizeof(uint64_t) * 2 * n_edges));
    rmat_keys_kernel<<<grid_for(n_edges), 256, 0, ctx->stream>>>(
        scale, seed, ta, tab, tabc, n_edges, s, row_lo, row_hi, keys);
    KPM_CUDA(cudaGetLastError());
  }
  return keys_to_graph(ctx, row_hi - row_lo, s, keys, alt, 2 * n_edges, out, row_lo, n);
}

int kpm_rmat_edges(kpm_ctx *ctx, int scale, uint64_t seed, uint32_t ta,
                   uint32_t tab, uint32_t tabc, int64_t e0, int64_t count,
                   int64_t *u, int64_t *v) {
  KPM_CHECK_ARG(ctx && u && v && scale >= 1 && scale <= 30 && e0 >= 0 && count >= 0,
                "bad arguments");
  KPM_CHECK_ARG(is_device_ptr(u) && is_device_ptr(v), "u/v must be device buffers");
  KPM_CUDA(cudaSetDevice(ctx->device));
  if (count > 0)
    rmat_edges_kernel<<<grid_for(count), 256, 0, ctx->stream>>>(scale, seed, ta, tab,
                                                                tabc, e0, count, u, v);
  KPM_CUDA(cudaGetLastError());
  return KPM_OK;
}

static int graph_from_csr_impl(kpm_ctx *ctx, int64_t n, int64_t n_cols, int64_t row0,
                               const int64_t *indptr, const void *indices, int idx_bytes,
                               int64_t nnz, const double *values, double shift, double scale,
                               kpm_graph **out);

int kpm_graph_from_csr(kpm_ctx *ctx, int64_t n, const int64_t *indptr,
                       const int64_t *indices, int64_t nnz,
                       const double *values, double shift, double scale,
                       kpm_graph **out) {
  return graph_from_csr_impl(ctx, n, n, 0, indptr, indices, 8, nnz, values, shift, scale, out);
}

int kpm_graph_from_csr32(kpm_ctx *ctx, int64_t n, const int64_t *indptr,
                         const int32_t *indices, int64_t nnz, const double *values,
                         double shift, double scale, kpm_graph **out) {
  return graph_from_csr_impl(ctx, n, n, 0, indptr, indices, 4, nnz, values, shift, scale, out);
}

int kpm_graph_from_csr_part(kpm_ctx *ctx, int64_t n_global, int64_t row_lo, int64_t n_local,
                            const int64_t *indptr, const int64_t *indices, int64_t nnz,
                            const double *values, double shift, double scale,
                            kpm_graph **out) {
  KPM_CHECK_ARG(row_lo >= 0 && n_local >= 0 && row_lo + n_local <= n_global,
                "bad partition rows");
  return graph_from_csr_impl(ctx, n_local, n_global, row_lo, indptr, indices, 8, nnz, values,
                             shift, scale, out);
}

int kpm_graph_set_dinv(kpm_graph *g, const double *dinv_global) {
  KPM_CHECK_ARG(g && dinv_global, "bad arguments");
  KPM_CUDA(cudaSetDevice(g->ctx->device));
  if (!g->dinv_all) KPM_CUDA(cudaMalloc(&g->dinv_all, sizeof(double) * (g->n_global + 1)));
  KPM_CUDA(cudaMemcpyAsync(g->dinv_all, dinv_global, sizeof(double) * g->n_global,
                           cudaMemcpyDefault, g->ctx->stream));
  KPM_CUDA(cudaStreamSynchronize(g->ctx->stream));
  return KPM_OK;
}

static int graph_from_csr_impl(kpm_ctx *ctx, int64_t n, int64_t n_cols, int64_t row0,
                               const int64_t *indptr, const void *indices, int idx_bytes,
                               int64_t nnz, const double *values, double shift, double scale,
                               kpm_graph **out) {
  kpm::Nvtx nvtx_range_("kpm_graph_from_csr");
  KPM_CHECK_ARG(ctx && out && n >= 0 && nnz >= 0 && indptr, "bad arguments");
  KPM_CHECK_ARG(nnz == 0 || indices, "indices is NULL");
  KPM_CHECK_ARG(n < (int64_t(1) << 31), "n must be < 2^31 (int32 col_idx)");
  KPM_CHECK_ARG(values || (shift == 0.0 && scale == 1.0),
                "implicit normalized adjacency takes shift 0, scale 1");
  KPM_CHECK_ARG(scale != 0.0, "scale must be nonzero");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  kpm_graph *g = new kpm_graph();
  g->ctx = ctx;
  g->n = n;
  g->nnz = nnz;
  g->shift = shift;
  g->scale = scale;
  g->row0 = row0;
  g->n_global = n_cols;
  auto fail = [&](int rc) { kpm_graph_free(g); return rc; };
  if (cudaMalloc(&g->row_ptr, sizeof(int64_t) * (n + 1)) != cudaSuccess ||
      cudaMalloc(&g->col_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess ||
      cudaMalloc(&g->dinv, sizeof(double) * (n > 0 ? n : 1)) != cudaSuccess ||
      (values && cudaMalloc(&g->values, sizeof(double) * (nnz > 0 ? nnz : 1)) != cudaSuccess)) {
    set_error("graph allocation failed");
    return fail(KPM_ENOMEM);
  }
  cudaError_t e = cudaMemcpyAsync(g->row_ptr, indptr, sizeof(int64_t) * (n + 1),
                                  cudaMemcpyDefault, st);
  if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return fail(KPM_ECUDA); }
  int64_t ends[2] = {0, 0};
  e = cudaMemcpyAsync(ends, g->row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ends + 1, g->row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return fail(KPM_ECUDA); }
  if (ends[0] != 0 || ends[1] != nnz) {
    set_error("indptr must start at 0 and end at nnz");
    return fail(KPM_EINVAL);
  }
  if (nnz > 0) {
    DevBuf ti;
    const void *di = nullptr;
    if (idx_bytes == 8) {
      int rc = stage_in(st, indices, sizeof(int64_t) * nnz, ti, &di);
      if (rc != KPM_OK) return fail(rc);
    } else {
      e = cudaMemcpyAsync(g->col_idx, indices, sizeof(int32_t) * nnz, cudaMemcpyDefault, st);
      if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return fail(KPM_ECUDA); }
    }
    int *bad = nullptr;
    cudaMalloc(&bad, sizeof(int));
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (idx_bytes == 8)
      idx64_to_32<<<grid_for(nnz), 256, 0, st>>>((const int64_t *)di, nnz, n_cols, g->col_idx,
                                                 bad);
    else
      idx32_check<<<grid_for(nnz), 256, 0, st>>>(g->col_idx, nnz, n_cols, bad);
    int hbad = 0;
    cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    cudaFree(bad);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return fail(KPM_ECUDA); }
    if (hbad) { set_error("column index out of range"); return fail(KPM_EINVAL); }
    if (values) {
      e = cudaMemcpyAsync(g->values, values, sizeof(double) * nnz, cudaMemcpyDefault, st);
      if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return fail(KPM_ECUDA); }
    }
  }
  int rc = finish_graph(g);
  if (rc != KPM_OK) return fail(rc);
  *out = g;
  return KPM_OK;
}

int kpm_graph_replicate(kpm_graph *src, kpm_ctx *ctx, kpm_graph **out) {
  kpm::Nvtx nvtx_range_("kpm_graph_replicate");
  KPM_CHECK_ARG(src && ctx && out, "bad arguments");
  KPM_CHECK_ARG(src->row0 == 0 && src->n_global == src->n && !src->dinv_all,
                "row-partition graphs are not replicated");
  // the source's stream has built the arrays; the copies run on ctx's stream
  KPM_CUDA(cudaSetDevice(src->ctx->device));
  KPM_CUDA(cudaStreamSynchronize(src->ctx->stream));
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const int64_t n = src->n, nnz = src->nnz;
  kpm_graph *g = new kpm_graph();
  g->ctx = ctx;
  g->n = n;
  g->nnz = nnz;
  g->shift = src->shift;
  g->scale = src->scale;
  g->n_global = n;
  auto fail = [&](int rc) { kpm_graph_free(g); return rc; };
  if (cudaMalloc(&g->row_ptr, sizeof(int64_t) * (n + 1)) != cudaSuccess ||
      cudaMalloc(&g->col_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1)) != cudaSuccess ||
      cudaMalloc(&g->dinv, sizeof(double) * (n > 0 ? n : 1)) != cudaSuccess ||
      (src->values &&
       cudaMalloc(&g->values, sizeof(double) * (nnz > 0 ? nnz : 1)) != cudaSuccess)) {
    set_error("graph allocation failed");
    return fail(KPM_ENOMEM);
  }
  const int sd = src->ctx->device, dd = ctx->device;
  cudaError_t e = cudaMemcpyPeerAsync(g->row_ptr, dd, src->row_ptr, sd,
                                      sizeof(int64_t) * (n + 1), st);
  if (e == cudaSuccess && nnz > 0)
    e = cudaMemcpyPeerAsync(g->col_idx, dd, src->col_idx, sd, sizeof(int32_t) * nnz, st);
  if (e == cudaSuccess && nnz > 0 && src->values)
    e = cudaMemcpyPeerAsync(g->values, dd, src->values, sd, sizeof(double) * nnz, st);
  if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); return fail(KPM_ECUDA); }
  // d^-1/2 and the schedule are recomputed from row_ptr: bit-identical
  int rc = finish_graph(g);
  if (rc != KPM_OK) return fail(rc);
  *out = g;
  return KPM_OK;
}

int kpm_graph_part_info(kpm_graph *g, int64_t *row0, int64_t *n_global) {
  KPM_CHECK_ARG(g, "graph is NULL");
  if (row0) *row0 = g->row0;
  if (n_global) *n_global = g->n_global;
  return KPM_OK;
}

int kpm_graph_info(kpm_graph *g, int64_t *n, int64_t *nnz, int64_t *max_degree) {
  KPM_CHECK_ARG(g, "graph is NULL");
  if (n) *n = g->n;
  if (nnz) *nnz = g->nnz;
  if (max_degree) *max_degree = g->max_degree;
  return KPM_OK;
}

int kpm_graph_export(kpm_graph *g, int64_t *row_ptr, int32_t *col_idx,
                     double *dinv) {
  KPM_CHECK_ARG(g, "graph is NULL");
  cudaStream_t st = g->ctx->stream;
  KPM_CUDA(cudaSetDevice(g->ctx->device));
  if (row_ptr)
    KPM_CUDA(cudaMemcpyAsync(row_ptr, g->row_ptr, sizeof(int64_t) * (g->n + 1),
                             cudaMemcpyDefault, st));
  if (col_idx && g->nnz)
    KPM_CUDA(cudaMemcpyAsync(col_idx, g->col_idx, sizeof(int32_t) * g->nnz,
                             cudaMemcpyDefault, st));
  if (dinv && g->n)
    KPM_CUDA(cudaMemcpyAsync(dinv, g->dinv, sizeof(double) * g->n, cudaMemcpyDefault, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  return KPM_OK;
}

void kpm_graph_free(kpm_graph *g) {
  if (!g) return;
  if (g->ctx) {
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
  }
  cudaFree(g->row_ptr);
  cudaFree(g->col_idx);
  cudaFree(g->dinv);
  cudaFree(g->values);
  cudaFree(g->chunk_start);
  cudaFree(g->heavy_rows);
  cudaFree(g->chunk_order);
  cudaFree(g->dinv_all);
  cudaFree(g->perm);
  cudaFree(g->iperm);
  cudaFree(g->dstep_id);
  cudaFree(g->dstep_val);
  if (g->relab) kpm_graph_free(g->relab);
  delete g;
}

}  // extern "C"
