// Internal types and helpers shared by the libkpm translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/kpm.h"

#include <nvtx3/nvToolsExt.h>

namespace kpm {

void set_error(const char *fmt, ...);

// NVTX range per C-ABI phase (graph load, probes, steps, result, ...): shows
// up in nsys / ncu --nvtx timelines; header-only NVTX v3, no link dependency.
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx &) = delete;
  Nvtx &operator=(const Nvtx &) = delete;
};

#define KPM_CUDA(expr)                                                         \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      kpm::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                     cudaGetErrorString(_e));                                  \
      return _e == cudaErrorMemoryAllocation ? KPM_ENOMEM : KPM_ECUDA;         \
    }                                                                          \
  } while (0)

#define KPM_CHECK_ARG(cond, ...)                                               \
  do {                                                                         \
    if (!(cond)) {                                                             \
      kpm::set_error(__VA_ARGS__);                                             \
      return KPM_EINVAL;                                                       \
    }                                                                          \
  } while (0)

#define KPM_TRY(expr)                                                          \
  do {                                                                         \
    int _s = (expr);                                                           \
    if (_s != KPM_OK) return _s;                                               \
  } while (0)

// true when p is device (or managed) memory usable in kernels
bool is_device_ptr(const void *p);

// Stage a host-or-device input array on the device: returns a device pointer
// (p itself when already on the device; otherwise a temporary owned by tmp).
struct DevBuf {
  void *ptr = nullptr;
  ~DevBuf() { if (ptr) cudaFree(ptr); }
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
};
int stage_in(cudaStream_t s, const void *p, size_t bytes, DevBuf &tmp,
             const void **dev);

}  // namespace kpm

struct kpm_ctx {
  int device = 0;
  int sm_count = 148;
  size_t persist_max = 0;  // cudaDeviceProp::persistingL2CacheMaxSize
  size_t l2_bytes = 126u << 20;  // cudaDeviceProp::l2CacheSize
  cudaStream_t stream = nullptr;
};

// Device CSR: int64 row_ptr, int32 col_idx, fp64 dinv (implicit normalized
// adjacency) or fp64 values + (shift, scale) (explicit operator).
// degree buckets of the hot-row rule: 8 per octave (3 mantissa bits)
static constexpr int kDegBuckets = 512;
__host__ __device__ inline int deg_bucket(unsigned long long d) {  // d >= 1
#ifdef __CUDA_ARCH__
  const int e = 63 - __clzll((long long)d);
#else
  int e = 0;
  for (unsigned long long t = d; t > 1; t >>= 1) ++e;
#endif
  const unsigned long long m = e >= 3 ? (d >> (e - 3)) & 7ull : (d << (3 - e)) & 7ull;
  return 8 * e + (int)m;
}
inline double deg_bucket_lo(int b) {
  const int e = b >> 3, m = b & 7;
  double lo = 1.0;
  for (int q = 0; q < e; ++q) lo *= 2.0;
  return lo * (1.0 + m / 8.0);
}

struct kpm_graph {
  kpm_ctx *ctx = nullptr;
  int64_t n = 0, nnz = 0, max_degree = 0;
  int64_t *row_ptr = nullptr;   // n+1
  int32_t *col_idx = nullptr;   // nnz
  double *dinv = nullptr;       // n (always computed from row degree)
  double *values = nullptr;     // nnz, explicit mode only
  double shift = 0.0, scale = 1.0;
  // load-balanced schedule (depends on the graph only, never on k)
  int32_t n_chunks = 0;
  int32_t *chunk_start = nullptr;  // n_chunks+1 row boundaries
  int32_t *chunk_order = nullptr;  // work-queue order of the chunks
  // rows with degree >= heavy_threshold are split over column slices and
  // worked by dedicated warps (degree-desc order); chunks skip them
  int64_t heavy_threshold = 0;
  int32_t n_heavy = 0;
  int32_t *heavy_rows = nullptr;
  // row partition (rows [row0, row0+n) of an n_global-row graph; col ids are
  // global).  dinv_all: d^-1/2 of all n_global rows (NULL = dinv, unpartitioned)
  int64_t row0 = 0, n_global = 0;
  double *dinv_all = nullptr;
  // rows per degree bucket, 8 buckets per octave (bucket b holds degrees
  // [deg_bucket_lo(b), deg_bucket_lo(b + 1)); finish_graph): hot-row L2 policy
  unsigned long long deg_hist[kDegBuckets] = {};
  // gather-ordered twin (kpm_graph_relabelled): the same graph with vertices
  // renumbered by degree descending (ties by id) and every row's neighbour list
  // sorted by the new ids, i.e. hottest neighbours first; built on demand for
  // large implicit graphs, owned by this graph.  In the twin, perm[new] = old
  // and iperm[old] = new.
  kpm_graph *relab = nullptr;
  int relab_state = 0;  // 0 not tried, 1 built, -1 unavailable
  int32_t *perm = nullptr, *iperm = nullptr;
  // twin only: d^-1/2 as a step function of the (degree-ranked) id.  Ids
  // >= dstep_id[0] have degree < kDinvSteps; dstep_id[e] is the first id with
  // degree <= kDinvSteps - 1 - e (ascending in e), dstep_val[e] that degree's
  // dinv (copied from dinv, bit-identical).  The step kernel looks the cold
  // ids' dinv_j up in this table (shared memory) instead of gathering 8 bytes
  // per nonzero from the n-entry array (a DRAM sector each at R-MAT scale).
  int32_t *dstep_id = nullptr;
  double *dstep_val = nullptr;
  int32_t dstep_h = 0x7fffffff;  // = dstep_id[0]
};
static constexpr int kDinvSteps = 512;

namespace kpm {
kpm_graph *graph_relabelled(kpm_graph *g);  // kpm_graph.cu; NULL when unavailable
}

#define KPM_MAX_PARTS 16

// lowest degree from which a row can be a "heavy" (hub) row; finish_graph raises
// the bar to nnz / 2048 on large graphs (graph-only)
static constexpr int64_t kHeavyDegree = 65536;

struct kpm_run {
  kpm_graph *g = nullptr;       // the graph the step kernels walk (user_g or its twin)
  kpm_graph *user_g = nullptr;  // the graph the caller passed
  double *unperm = nullptr;     // kpm_run_block scratch: T_k in the caller's row order
  int64_t k = 0;      // probes in this batch
  int64_t ld = 0;     // padded row stride (doubles)
  int cpl = 1;        // columns per lane (1, 2, 4)
  int32_t mode = 0, m_max = 0, flags = 0;
  int32_t total_steps = 0, done_steps = 0;
  bool have_probes = false;
  bool finished = false;      // LDOS: kpm_run_result turned the sums into values
  double *z = nullptr;        // probes (DIRECT/LDOS), n x ld
  double *a = nullptr, *b = nullptr;  // recurrence blocks
  double *cur = nullptr, *prev = nullptr;  // T_k (gather source), T_{k-1}
  int32_t k_index = 0;        // index of the block in `cur`
  double *partial = nullptr;  // n_chunks x 2 x ld
  double *contrib = nullptr;  // (m_max+1) x ld (global modes)
  double *ldos = nullptr;     // n x (m_max+1) (LDOS)
  double *den = nullptr;      // n (LDOS)
  double *hpart = nullptr;    // n_heavy x 2 x ld (global modes)
  double *hldos = nullptr;    // n_heavy x slices (LDOS)
  double *gpart = nullptr;    // chunk-group partials (level-1 reduction)
  unsigned long long *queue = nullptr;  // persistent-kernel work counter
  // row partitions: this run owns partition `me`; peer_a/peer_b[q] are the
  // a/b recurrence blocks of partition q (peer memory or same device)
  int nparts = 1, me = 0;
  bool partitioned = false;  // kpm_run_set_partition called: raw global sums
  int64_t part_lo[KPM_MAX_PARTS + 1] = {0};
  const double *peer_a[KPM_MAX_PARTS] = {nullptr};
  const double *peer_b[KPM_MAX_PARTS] = {nullptr};
  int32_t *flag = nullptr;    // [0]: non-finite seen; [1..2]: zero-mass node
  // optional per-launch timing of the step kernel (roofline evidence)
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // pairs (start, stop), reused
  int32_t ev_used = 0;
  // TMA tensor maps of the two recurrence blocks (n x ld fp64, box ld x 1) for
  // the gather4 light path (kpm_step.cu light_g4); tm_ok when encodable
  CUtensorMap tm[2][3];  // [block][box: whole row, 64-column tile, last partial tile]
  bool tm_ok = false, tm_tile_ok = false;
};
