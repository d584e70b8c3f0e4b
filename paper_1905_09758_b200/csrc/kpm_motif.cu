// Device motif scan ("device motif detection").
//
// Reference semantics (motifs.py:189-311): open twins are nodes with identical
// neighbour lists (no self-loop); closed twins are adjacent nodes whose
// neighbourhoods agree outside the pair (identical closed neighbourhoods);
// dangling two-chains are pendant paths x - b - hub (deg x = 1, deg b = 2).
// Candidate classes come from a commutative hash of per-node labels over the
// neighbourhood and are then verified EXACTLY, so no false positives.
//
// B200 design: one warp per row forms two independent 64-bit label sums over
// the row (labels are splitmix64 of the node id -- no label array), the
// (signature, row) pairs are radix-sorted on the device (stable: members of a
// run stay in row order), and one thread per sorted position verifies its row
// against the run head entry by entry.  The host receives n-sized arrays and
// extracts classes with O(n) numpy.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kpm_internal.cuh"

namespace kpm {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t lab1(int64_t j) { return splitmix64((uint64_t)j * 2 + 1); }
__device__ __forceinline__ uint64_t lab2(int64_t j) {
  return splitmix64((uint64_t)j * 2 + 0x5851F42D4C957F2Dull);
}

__device__ __forceinline__ uint64_t mix_key(uint64_t h1, uint64_t h2, int64_t deg) {
  uint64_t k = h1 ^ splitmix64(h2 ^ ((uint64_t)deg * 0xD6E8FEB86659FD93ull));
  return k == ~0ull ? k - 1 : k;  // ~0 marks excluded rows
}

// keys for open (N(i)) and closed (N(i) + {i}) signatures; rows with a self
// loop are excluded from both (the difference vectors are not eigenvectors)
__global__ void motif_hash_kernel(const int64_t *__restrict__ row_ptr,
                                  const int32_t *__restrict__ col, int64_t n,
                                  uint64_t *__restrict__ kopen, uint64_t *__restrict__ kclosed,
                                  int64_t *__restrict__ ids_open,
                                  int64_t *__restrict__ ids_closed) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    uint64_t h1 = 0, h2 = 0;
    int loop = 0;
    for (int64_t k = b + lane; k < e; k += 32) {
      const int32_t j = col[k];
      h1 += lab1(j);
      h2 += lab2(j);
      loop |= (j == i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      h1 += __shfl_xor_sync(0xffffffffu, h1, o);
      h2 += __shfl_xor_sync(0xffffffffu, h2, o);
    }
    loop = __any_sync(0xffffffffu, loop);
    if (lane == 0) {
      const int64_t deg = e - b;
      kopen[i] = loop ? ~0ull : mix_key(h1, h2, deg);
      kclosed[i] = (loop || deg == 0) ? ~0ull : mix_key(h1 + lab1(i), h2 + lab2(i), deg + 1);
      ids_open[i] = i;
      ids_closed[i] = i;
    }
  }
}

// ok[p] = row srt[p] has the same neighbour list as its run head (open)
__global__ void verify_open_kernel(const int64_t *__restrict__ row_ptr,
                                   const int32_t *__restrict__ col,
                                   const uint64_t *__restrict__ key,
                                   const int64_t *__restrict__ srt, int64_t n,
                                   const int64_t *__restrict__ head, int8_t *__restrict__ ok) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = head[p];
    int8_t good = 1;
    if (key[p] == ~0ull) {
      good = 0;
    } else if (h != p) {
      const int64_t i = srt[p], r = srt[h];
      const int64_t bi = row_ptr[i], ei = row_ptr[i + 1], br = row_ptr[r], er = row_ptr[r + 1];
      if (ei - bi != er - br) {
        good = 0;
      } else {
        for (int64_t t = 0; t < ei - bi; ++t)
          if (col[bi + t] != col[br + t]) { good = 0; break; }
      }
    }
    ok[p] = good;
  }
}

// closed: i ~ r and N(i) \ {r} == N(r) \ {i} (unit weights)
__global__ void verify_closed_kernel(const int64_t *__restrict__ row_ptr,
                                     const int32_t *__restrict__ col,
                                     const uint64_t *__restrict__ key,
                                     const int64_t *__restrict__ srt, int64_t n,
                                     const int64_t *__restrict__ head, int8_t *__restrict__ ok) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = head[p];
    int8_t good = 1;
    if (key[p] == ~0ull) {
      good = 0;
    } else if (h != p) {
      const int64_t i = srt[p], r = srt[h];
      int64_t a = row_ptr[i], ae = row_ptr[i + 1], b = row_ptr[r], be = row_ptr[r + 1];
      bool adj = false;
      for (int64_t t = a; t < ae; ++t) adj |= (col[t] == r);
      if (!adj || ae - a != be - b) {
        good = 0;
      } else {
        while (true) {  // merge-walk both lists, skipping r in N(i), i in N(r)
          while (a < ae && col[a] == r) ++a;
          while (b < be && col[b] == i) ++b;
          if (a == ae || b == be) {
            if (a != ae || b != be) good = 0;
            break;
          }
          if (col[a] != col[b]) { good = 0; break; }
          ++a;
          ++b;
        }
      }
    }
    ok[p] = good;
  }
}

// run starts: p if key[p] != key[p-1] else 0; an inclusive max-scan of this
// gives head[p] = first position of p's run (runs can be millions long)
__global__ void run_starts_kernel(const uint64_t *__restrict__ key, int64_t n,
                                  int64_t *__restrict__ start) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    start[p] = (p == 0 || key[p] != key[p - 1]) ? p : 0;
}

struct MaxOp {
  __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const {
    return a > b ? a : b;
  }
};

// pendant paths x - b - h (motifs.py:243-260): chain_hub[x] = h, mid[x] = b
__global__ void chain_kernel(const int64_t *__restrict__ row_ptr,
                             const int32_t *__restrict__ col, int64_t n,
                             int64_t *__restrict__ hub, int64_t *__restrict__ mid) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    int64_t hh = -1, bb = -1;
    if (row_ptr[x + 1] - row_ptr[x] == 1) {
      const int64_t b = col[row_ptr[x]];
      if (row_ptr[b + 1] - row_ptr[b] == 2) {
        const int64_t n0 = col[row_ptr[b]], n1 = col[row_ptr[b] + 1];
        const bool one = (n0 == x) != (n1 == x);
        const int64_t other = n0 == x ? n1 : n0;
        if (one && other != x) {
          hh = other;
          bb = b;
        }
      }
    }
    hub[x] = hh;
    mid[x] = bb;
  }
}

static int grid_n(int64_t work) {
  int64_t b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

}  // namespace kpm

using namespace kpm;

extern "C" int kpm_motif_scan(kpm_graph *g, int64_t *open_rows, int8_t *open_ok,
                              int64_t *open_head, int64_t *closed_rows, int8_t *closed_ok,
                              int64_t *closed_head, int64_t *chain_hub, int64_t *chain_mid) {
  kpm::Nvtx nvtx_range_("kpm_motif_scan");
  KPM_CHECK_ARG(g && open_rows && open_ok && open_head && closed_rows && closed_ok &&
                    closed_head && chain_hub && chain_mid,
                "bad arguments");
  KPM_CHECK_ARG(g->values == nullptr && g->n_global == g->n,
                "motif scan needs an unpartitioned unit-weight graph");
  KPM_CUDA(cudaSetDevice(g->ctx->device));
  cudaStream_t st = g->ctx->stream;
  const int64_t n = g->n;
  if (n == 0) return KPM_OK;
  uint64_t *k[2] = {nullptr, nullptr}, *ks[2] = {nullptr, nullptr};
  int64_t *id[2] = {nullptr, nullptr}, *ids[2] = {nullptr, nullptr}, *head = nullptr;
  int64_t *dh = nullptr, *dm = nullptr;
  int8_t *ok = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = KPM_OK;
  auto cleanup = [&]() {
    for (int q = 0; q < 2; ++q) {
      cudaFree(k[q]);
      cudaFree(ks[q]);
      cudaFree(id[q]);
      cudaFree(ids[q]);
    }
    cudaFree(head);
    cudaFree(ok);
    cudaFree(dh);
    cudaFree(dm);
    cudaFree(tmp);
  };
  do {
    bool fail = false;
    for (int q = 0; q < 2 && !fail; ++q)
      fail = cudaMalloc(&k[q], 8 * n) != cudaSuccess || cudaMalloc(&ks[q], 8 * n) != cudaSuccess ||
             cudaMalloc(&id[q], 8 * n) != cudaSuccess || cudaMalloc(&ids[q], 8 * n) != cudaSuccess;
    if (fail || cudaMalloc(&head, 8 * n) != cudaSuccess || cudaMalloc(&ok, n) != cudaSuccess ||
        cudaMalloc(&dh, 8 * n) != cudaSuccess || cudaMalloc(&dm, 8 * n) != cudaSuccess) {
      cudaGetLastError();
      set_error("motif scan: device allocation failed");
      rc = KPM_ENOMEM;
      break;
    }
    motif_hash_kernel<<<grid_n(32 * n), 256, 0, st>>>(g->row_ptr, g->col_idx, n, k[0], k[1],
                                                      id[0], id[1]);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k[0], ks[0], id[0], ids[0], n, 0, 64, st);
    size_t scan_bytes = 0;
    cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, dh, head, MaxOp(), n, st);
    if (scan_bytes > tmp_bytes) tmp_bytes = scan_bytes;
    if (cudaMalloc(&tmp, tmp_bytes) != cudaSuccess) {
      set_error("motif scan: temp allocation failed");
      rc = KPM_ENOMEM;
      break;
    }
    int64_t *out_rows[2] = {open_rows, closed_rows}, *out_head[2] = {open_head, closed_head};
    int8_t *out_ok[2] = {open_ok, closed_ok};
    for (int q = 0; q < 2; ++q) {
      size_t tb = tmp_bytes;
      cub::DeviceRadixSort::SortPairs(tmp, tb, k[q], ks[q], id[q], ids[q], n, 0, 64, st);
      run_starts_kernel<<<grid_n(n), 256, 0, st>>>(ks[q], n, dh);
      tb = tmp_bytes;
      cub::DeviceScan::InclusiveScan(tmp, tb, dh, head, MaxOp(), n, st);
      if (q == 0)
        verify_open_kernel<<<grid_n(n), 256, 0, st>>>(g->row_ptr, g->col_idx, ks[q], ids[q], n,
                                                      head, ok);
      else
        verify_closed_kernel<<<grid_n(n), 256, 0, st>>>(g->row_ptr, g->col_idx, ks[q], ids[q],
                                                        n, head, ok);
      if (cudaMemcpyAsync(out_rows[q], ids[q], 8 * n, cudaMemcpyDefault, st) != cudaSuccess ||
          cudaMemcpyAsync(out_head[q], head, 8 * n, cudaMemcpyDefault, st) != cudaSuccess ||
          cudaMemcpyAsync(out_ok[q], ok, n, cudaMemcpyDefault, st) != cudaSuccess ||
          cudaStreamSynchronize(st) != cudaSuccess) {
        set_error("motif scan: %s", cudaGetErrorString(cudaGetLastError()));
        rc = KPM_ECUDA;
        break;
      }
    }
    if (rc != KPM_OK) break;
    chain_kernel<<<grid_n(n), 256, 0, st>>>(g->row_ptr, g->col_idx, n, dh, dm);
    if (cudaMemcpyAsync(chain_hub, dh, 8 * n, cudaMemcpyDefault, st) != cudaSuccess ||
        cudaMemcpyAsync(chain_mid, dm, 8 * n, cudaMemcpyDefault, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      set_error("motif scan: %s", cudaGetErrorString(cudaGetLastError()));
      rc = KPM_ECUDA;
    }
  } while (false);
  cudaGetLastError();
  cleanup();
  return rc;
}
