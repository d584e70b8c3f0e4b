// Device graph ingest: text edge lists / Matrix Market
// bodies parsed on the B200, then handed to the sort-based loader (K1-K3).
//
// Reference semantics (fileio.py:28-128): whitespace-separated `u v [w]` lines,
// blank lines and lines starting with '#' or '%' skipped, 2 or 3 tokens per
// line, integer node ids; Matrix Market bodies use 1-based indices.
//
// Design: the file bytes are copied to HBM once; one pass flags line starts,
// an exclusive scan numbers them, and one thread per line tokenises its line
// and parses the two integer ids (a third token is recorded as "weighted" --
// decimal->double parsing is left to the host so weights stay bit-exact with
// Python's float()).  Malformed lines are reported by (1-based) line number.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/discard_iterator.h>

#include "kpm_internal.cuh"

namespace kpm {

// Bytes the device tokenizer does not model exactly (Python's text-mode
// reader and str.split/int would): non-ASCII (UTF-8 decoding), control
// characters Python treats as whitespace (0x1c-0x1f), NUL / DEL, and a bare
// '\r' (universal newlines split lines on it).  Any of them -> host parse.
__global__ void byte_class_kernel(const char *__restrict__ buf, int64_t len,
                                  int32_t *__restrict__ unusual) {
  int found = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < len;
       p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned char c = (unsigned char)buf[p];
    if (c >= 0x7f || (c < 0x20 && c != '\t' && c != '\n' && c != '\v' && c != '\f' && c != '\r'))
      found = 1;
    else if (c == '\r' && (p + 1 >= len || buf[p + 1] != '\n'))
      found = 1;
  }
  if (__syncthreads_or(found) && threadIdx.x == 0) atomicOr(unusual, 1);
}

struct IsLineStart {
  const char *b;
  __device__ bool operator()(int64_t p) const { return p == 0 || b[p - 1] == '\n'; }
};

__device__ __forceinline__ bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

// status: 0 skip (blank/comment), 2 or 3 = token count, -1 malformed,
// -2 the host must decide (see byte_class_kernel / long or '_' tokens)
__global__ void parse_lines_kernel(const char *__restrict__ buf, int64_t len,
                                   const int64_t *__restrict__ starts, int64_t nlines,
                                   int64_t base, int hash_comments, int64_t *__restrict__ u,
                                   int64_t *__restrict__ v, int8_t *__restrict__ status) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nlines;
       l += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = starts[l];
    const int64_t end = (l + 1 < nlines) ? starts[l + 1] : len;
    while (p < end && (is_ws(buf[p]) || buf[p] == '\n')) ++p;
    int8_t st = 0;
    int64_t vals[2] = {0, 0};
    if (p < end && buf[p] != '%' && !(hash_comments && buf[p] == '#')) {
      int ntok = 0;
      bool bad = false, host = false;
      while (p < end && buf[p] != '\n') {
        if (is_ws(buf[p])) { ++p; continue; }
        const int64_t t0 = p;
        while (p < end && buf[p] != '\n' && !is_ws(buf[p])) ++p;
        if (ntok < 2) {  // an integer token: [+-]digits
          int64_t q = t0, x = 0;
          bool neg = false;
          if (buf[q] == '+' || buf[q] == '-') { neg = buf[q] == '-'; ++q; }
          if (q == p) bad = true;
          if (p - q > 18) host = true;  // may overflow int64: Python's int() decides
          for (; q < p && !host; ++q) {
            const char c = buf[q];
            if (c == '_') { host = true; break; }  // int('1_0') == 10
            if (c < '0' || c > '9') { bad = true; break; }
            x = x * 10 + (c - '0');
          }
          vals[ntok] = neg ? -x : x;
        }
        ++ntok;
      }
      st = (ntok != 2 && ntok != 3) ? -1 : host ? -2 : bad ? -1 : (int8_t)ntok;
    }
    status[l] = st;
    u[l] = vals[0] - base;
    v[l] = vals[1] - base;
  }
}

__global__ void line_flags_kernel(const int8_t *__restrict__ status, int64_t nlines,
                                  int8_t *__restrict__ keep, int32_t *__restrict__ info) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nlines;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int8_t s = status[l];
    keep[l] = s >= 2;
    if (s == 3) atomicOr(info + 0, 1);
    if (s == -2) atomicOr(info + 0, 2);
    if (s < 0) atomicMin(info + 3, (int32_t)min(l, (int64_t)0x7ffffffe));
  }
}

__global__ void concat_kernel(const int64_t *__restrict__ u, const int64_t *__restrict__ v,
                              int64_t m, int64_t *__restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    out[e] = u[e];
    out[m + e] = v[e];
  }
}

// u, v -> position in the sorted unique id list; range / loop checks
__global__ void remap_kernel(int64_t *__restrict__ u, int64_t *__restrict__ v, int64_t m,
                             const int64_t *__restrict__ ids, int64_t n, int compact,
                             int32_t *__restrict__ info) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[e], b = v[e];
    if (compact) {
      int64_t lo = 0, hi = n;
      while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (ids[mid] < a) lo = mid + 1; else hi = mid; }
      a = lo;
      lo = 0; hi = n;
      while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (ids[mid] < b) lo = mid + 1; else hi = mid; }
      b = lo;
      u[e] = a;
      v[e] = b;
    }
    if (a < 0 || b < 0 || a >= n || b >= n) atomicOr(info + 4, 1);
    if (a == b) atomicOr(info + 1, 1);
  }
}

__global__ void directed_keys_kernel(const int64_t *__restrict__ u, const int64_t *__restrict__ v,
                                     int64_t m, int s, uint64_t *__restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    keys[e] = ((uint64_t)u[e] << s) | (uint64_t)v[e];
}

static int grid_p(int64_t work) {
  int64_t b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

}  // namespace kpm

using namespace kpm;

extern "C" int kpm_parse_edges(kpm_ctx *ctx, const char *text, int64_t len, int64_t base,
                               int flags, int64_t *nlines_out, int64_t **u_out,
                               int64_t **v_out, int8_t **status_out, int32_t *unusual_out) {
  kpm::Nvtx nvtx_range_("kpm_parse_edges");
  KPM_CHECK_ARG(ctx && (text || len == 0) && len >= 0 && nlines_out && u_out && v_out &&
                    status_out && unusual_out,
                "bad arguments");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  *nlines_out = 0;
  *u_out = *v_out = nullptr;
  *status_out = nullptr;
  *unusual_out = 0;
  if (len == 0) return KPM_OK;
  DevBuf dbuf, cnt, tmp, startsb, unus;
  const void *dtext;
  KPM_TRY(stage_in(st, text, (size_t)len, dbuf, &dtext));
  const char *b = (const char *)dtext;
  KPM_CUDA(cudaMalloc(&unus.ptr, sizeof(int32_t)));
  KPM_CUDA(cudaMemsetAsync(unus.ptr, 0, sizeof(int32_t), st));
  byte_class_kernel<<<grid_p(len), 256, 0, st>>>(b, len, (int32_t *)unus.ptr);
  // line starts = positions p with p == 0 or buf[p-1] == '\n' (8 B per line)
  KPM_CUDA(cudaMalloc(&cnt.ptr, sizeof(int64_t)));
  int64_t nl_bound = 0;
  {
    thrust::counting_iterator<int64_t> it(0);
    size_t tb = 0;
    cub::DeviceSelect::If(nullptr, tb, it, (int64_t *)nullptr, (int64_t *)cnt.ptr, len,
                          IsLineStart{b}, st);
    KPM_CUDA(cudaMalloc(&tmp.ptr, tb));
    // count first (discard output) so the starts buffer is exact
    cub::DeviceSelect::If(tmp.ptr, tb, it, thrust::make_discard_iterator(), (int64_t *)cnt.ptr,
                          len, IsLineStart{b}, st);
    KPM_CUDA(cudaMemcpyAsync(&nl_bound, cnt.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    KPM_CUDA(cudaMalloc(&startsb.ptr, sizeof(int64_t) * nl_bound));
    cub::DeviceSelect::If(tmp.ptr, tb, it, (int64_t *)startsb.ptr, (int64_t *)cnt.ptr, len,
                          IsLineStart{b}, st);
  }
  const int64_t nlines = nl_bound;
  const int64_t *starts = (const int64_t *)startsb.ptr;
  int64_t *du = nullptr, *dv = nullptr;
  int8_t *ds = nullptr;
  cudaError_t e1 = cudaMalloc(&du, sizeof(int64_t) * nlines);
  cudaError_t e2 = cudaMalloc(&dv, sizeof(int64_t) * nlines);
  cudaError_t e3 = cudaMalloc(&ds, nlines);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
    cudaFree(du);
    cudaFree(dv);
    cudaFree(ds);
    set_error("ingest: device allocation failed");
    return KPM_ENOMEM;
  }
  parse_lines_kernel<<<grid_p(nlines), 256, 0, st>>>(b, len, starts, nlines, base,
                                                     (flags & KPM_PARSE_HASH_COMMENTS) ? 1 : 0,
                                                     du, dv, ds);
  int32_t unusual = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&unusual, unus.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    cudaFree(du);
    cudaFree(dv);
    cudaFree(ds);
    set_error("ingest: %s", cudaGetErrorString(e));
    return KPM_ECUDA;
  }
  *nlines_out = nlines;
  *u_out = du;
  *v_out = dv;
  *status_out = ds;
  *unusual_out = unusual;
  return KPM_OK;
}

// Compact the parsed lines into an edge list (device), map node ids onto
// 0..n-1 (sorted unique ids, as fileio.py:122-126) or check them against n,
// and report what needs the host's build_csr semantics.
// info: [0] a line had a weight token, [1] a self-loop, [2] a repeated
// (same-direction) edge -- build_csr would sum its weight --, [3] first
// malformed line (0-based) or INT32_MAX, [4] id out of range.
extern "C" int kpm_edges_finalize(kpm_ctx *ctx, int64_t nlines, int64_t *u, int64_t *v,
                                  const int8_t *status, int compact_ids, int64_t n_declared,
                                  int64_t *m_out, int64_t *n_out, int64_t **eu_out,
                                  int64_t **ev_out, int64_t **ids_out, int32_t *info) {
  kpm::Nvtx nvtx_range_("kpm_edges_finalize");
  KPM_CHECK_ARG(ctx && m_out && n_out && eu_out && ev_out && ids_out && info, "bad arguments");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  int32_t hinfo[5] = {0, 0, 0, 0x7fffffff, 0};
  *m_out = *n_out = 0;
  *eu_out = *ev_out = *ids_out = nullptr;
  if (nlines == 0) {
    for (int q = 0; q < 5; ++q) info[q] = hinfo[q];
    return KPM_OK;
  }
  DevBuf dinfo, keep, nsel, tmp, cat, catsorted, ukeys;
  KPM_CUDA(cudaMalloc(&dinfo.ptr, sizeof(hinfo)));
  KPM_CUDA(cudaMemcpyAsync(dinfo.ptr, hinfo, sizeof(hinfo), cudaMemcpyHostToDevice, st));
  int32_t *di = (int32_t *)dinfo.ptr;
  KPM_CUDA(cudaMalloc(&keep.ptr, nlines));
  line_flags_kernel<<<grid_p(nlines), 256, 0, st>>>(status, nlines, (int8_t *)keep.ptr, di);
  int64_t *eu = nullptr, *ev = nullptr;
  KPM_CUDA(cudaMalloc(&eu, sizeof(int64_t) * nlines));
  KPM_CUDA(cudaMalloc(&ev, sizeof(int64_t) * nlines));
  KPM_CUDA(cudaMalloc(&nsel.ptr, sizeof(int64_t)));
  size_t tb = 0;
  cub::DeviceSelect::Flagged(nullptr, tb, u, (int8_t *)keep.ptr, eu, (int64_t *)nsel.ptr, nlines, st);
  KPM_CUDA(cudaMalloc(&tmp.ptr, tb));
  cub::DeviceSelect::Flagged(tmp.ptr, tb, u, (int8_t *)keep.ptr, eu, (int64_t *)nsel.ptr, nlines, st);
  cub::DeviceSelect::Flagged(tmp.ptr, tb, v, (int8_t *)keep.ptr, ev, (int64_t *)nsel.ptr, nlines, st);
  int64_t m = 0;
  KPM_CUDA(cudaMemcpyAsync(&m, nsel.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  int64_t n = n_declared, *ids = nullptr;
  if (m > 0 && compact_ids) {
    KPM_CUDA(cudaMalloc(&cat.ptr, sizeof(int64_t) * 2 * m));
    KPM_CUDA(cudaMalloc(&catsorted.ptr, sizeof(int64_t) * 2 * m));
    concat_kernel<<<grid_p(m), 256, 0, st>>>(eu, ev, m, (int64_t *)cat.ptr);
    DevBuf t2;
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb2, (int64_t *)cat.ptr, (int64_t *)catsorted.ptr,
                                   2 * m, 0, 64, st);
    size_t tb3 = 0;
    cub::DeviceSelect::Unique(nullptr, tb3, (int64_t *)catsorted.ptr, (int64_t *)cat.ptr,
                              (int64_t *)nsel.ptr, 2 * m, st);
    KPM_CUDA(cudaMalloc(&t2.ptr, tb2 > tb3 ? tb2 : tb3));
    cub::DeviceRadixSort::SortKeys(t2.ptr, tb2, (int64_t *)cat.ptr, (int64_t *)catsorted.ptr,
                                   2 * m, 0, 64, st);
    cub::DeviceSelect::Unique(t2.ptr, tb3, (int64_t *)catsorted.ptr, (int64_t *)cat.ptr,
                              (int64_t *)nsel.ptr, 2 * m, st);
    KPM_CUDA(cudaMemcpyAsync(&n, nsel.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KPM_CUDA(cudaStreamSynchronize(st));
    KPM_CUDA(cudaMalloc(&ids, sizeof(int64_t) * (n > 0 ? n : 1)));
    KPM_CUDA(cudaMemcpyAsync(ids, cat.ptr, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st));
  }
  if (m > 0) {
    remap_kernel<<<grid_p(m), 256, 0, st>>>(eu, ev, m, ids, n, compact_ids, di);
    // same-direction repeats (build_csr sums their weights -> host path)
    int s = 1;
    while ((int64_t(1) << s) <= n) ++s;
    if (2 * s <= 64 && n > 0) {
      KPM_CUDA(cudaMalloc(&ukeys.ptr, sizeof(uint64_t) * 2 * m));
      uint64_t *k0 = (uint64_t *)ukeys.ptr, *k1 = k0 + m;
      directed_keys_kernel<<<grid_p(m), 256, 0, st>>>(eu, ev, m, s, k0);
      DevBuf t4;
      size_t tb4 = 0, tb5 = 0;
      cub::DeviceRadixSort::SortKeys(nullptr, tb4, k0, k1, m, 0, 2 * s, st);
      cub::DeviceSelect::Unique(nullptr, tb5, k1, k0, (int64_t *)nsel.ptr, m, st);
      KPM_CUDA(cudaMalloc(&t4.ptr, tb4 > tb5 ? tb4 : tb5));
      cub::DeviceRadixSort::SortKeys(t4.ptr, tb4, k0, k1, m, 0, 2 * s, st);
      cub::DeviceSelect::Unique(t4.ptr, tb5, k1, k0, (int64_t *)nsel.ptr, m, st);
      int64_t nu = 0;
      KPM_CUDA(cudaMemcpyAsync(&nu, nsel.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      KPM_CUDA(cudaStreamSynchronize(st));
      if (nu != m) hinfo[2] = 1;
    }
  }
  int32_t dinfo_h[5];
  KPM_CUDA(cudaMemcpyAsync(dinfo_h, di, sizeof(dinfo_h), cudaMemcpyDeviceToHost, st));
  KPM_CUDA(cudaStreamSynchronize(st));
  info[0] = dinfo_h[0];
  info[1] = dinfo_h[1];
  info[2] = hinfo[2];
  info[3] = dinfo_h[3];
  info[4] = dinfo_h[4];
  *m_out = m;
  *n_out = n;
  *eu_out = eu;
  *ev_out = ev;
  *ids_out = ids;
  return KPM_OK;
}
