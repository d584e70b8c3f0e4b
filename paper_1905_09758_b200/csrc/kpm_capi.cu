// libkpm C-ABI: context, memory and error plumbing (include/kpm.h).
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <thread>
#include <vector>

#include "kpm_internal.cuh"

namespace kpm {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int stage_in(cudaStream_t s, const void *p, size_t bytes, DevBuf &tmp,
             const void **dev) {
  if (bytes == 0 || p == nullptr) {
    *dev = p;
    return KPM_OK;
  }
  if (is_device_ptr(p)) {
    *dev = p;
    return KPM_OK;
  }
  KPM_CUDA(cudaMalloc(&tmp.ptr, bytes));
  KPM_CUDA(cudaMemcpyAsync(tmp.ptr, p, bytes, cudaMemcpyHostToDevice, s));
  *dev = tmp.ptr;
  return KPM_OK;
}

}  // namespace kpm

using namespace kpm;

extern "C" {

int kpm_abi_version(void) { return KPM_ABI_VERSION; }

const char *kpm_last_error(void) { return g_err; }

int kpm_device_count(int *count) {
  KPM_CHECK_ARG(count, "count is NULL");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return KPM_OK;
}

int kpm_init(int device, kpm_ctx **out) {
  KPM_CHECK_ARG(out, "out is NULL");
  int count = 0;
  kpm_device_count(&count);
  if (count <= 0) {
    set_error("no CUDA device visible");
    return KPM_ENODEV;
  }
  KPM_CHECK_ARG(device >= 0 && device < count, "device %d out of range (%d)",
                device, count);
  KPM_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  KPM_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    set_error("device %d is sm_%d%d; libkpm is built for sm_100a only", device,
              prop.major, prop.minor);
    return KPM_ENODEV;
  }
  kpm_ctx *c = new kpm_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->persist_max = prop.persistingL2CacheMaxSize;
  c->l2_bytes = prop.l2CacheSize;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    set_error("cudaStreamCreate: %s", cudaGetErrorString(e));
    return KPM_ECUDA;
  }
  *out = c;
  return KPM_OK;
}

void kpm_finalize(kpm_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

void *kpm_ctx_stream(kpm_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int kpm_ctx_synchronize(kpm_ctx *ctx) {
  KPM_CHECK_ARG(ctx, "ctx is NULL");
  KPM_CUDA(cudaStreamSynchronize(ctx->stream));
  KPM_CUDA(cudaGetLastError());
  return KPM_OK;
}

int kpm_device_alloc(kpm_ctx *ctx, int64_t bytes, void **out) {
  KPM_CHECK_ARG(ctx && out && bytes >= 0, "bad arguments");
  *out = nullptr;
  if (bytes == 0) return KPM_OK;
  KPM_CUDA(cudaSetDevice(ctx->device));
  KPM_CUDA(cudaMalloc(out, (size_t)bytes));
  return KPM_OK;
}

int kpm_device_free(kpm_ctx *ctx, void *ptr) {
  KPM_CHECK_ARG(ctx, "ctx is NULL");
  if (ptr) {
    KPM_CUDA(cudaStreamSynchronize(ctx->stream));
    KPM_CUDA(cudaFree(ptr));
  }
  return KPM_OK;
}

int kpm_memcpy(kpm_ctx *ctx, void *dst, const void *src, int64_t bytes,
               int kind) {
  KPM_CHECK_ARG(ctx && bytes >= 0 && kind >= 0 && kind <= 2, "bad arguments");
  if (bytes == 0) return KPM_OK;
  cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                     : kind == 1 ? cudaMemcpyDeviceToHost
                                 : cudaMemcpyDeviceToDevice;
  KPM_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, k, ctx->stream));
  return KPM_OK;
}

int kpm_host_alloc(int64_t bytes, void **out) {
  KPM_CHECK_ARG(out && bytes >= 0, "bad arguments");
  *out = nullptr;
  if (bytes == 0) return KPM_OK;
  KPM_CUDA(cudaMallocHost(out, (size_t)bytes));
  return KPM_OK;
}

int kpm_mem_info(kpm_ctx *ctx, int64_t *free_bytes, int64_t *total_bytes) {
  KPM_CHECK_ARG(ctx, "ctx is NULL");
  KPM_CUDA(cudaSetDevice(ctx->device));
  size_t f = 0, t = 0;
  KPM_CUDA(cudaMemGetInfo(&f, &t));
  if (free_bytes) *free_bytes = (int64_t)f;
  if (total_bytes) *total_bytes = (int64_t)t;
  return KPM_OK;
}

int kpm_ipc_get_handle(const void *dptr, void *handle) {
  KPM_CHECK_ARG(dptr && handle, "bad arguments");
  cudaIpcMemHandle_t h;
  KPM_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(dptr)));
  memcpy(handle, &h, sizeof(h));
  return KPM_OK;
}

int kpm_ipc_open_handle(kpm_ctx *ctx, const void *handle, void **dptr) {
  KPM_CHECK_ARG(ctx && handle && dptr, "bad arguments");
  KPM_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  KPM_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return KPM_OK;
}

int kpm_ipc_close(void *dptr) {
  if (dptr) KPM_CUDA(cudaIpcCloseMemHandle(dptr));
  return KPM_OK;
}

int kpm_host_free(void *ptr) {
  if (ptr) KPM_CUDA(cudaFreeHost(ptr));
  return KPM_OK;
}

}  // extern "C"

int kpm_host_prefault(void *ptr, int64_t bytes, int threads) {
  KPM_CHECK_ARG(bytes >= 0, "negative size");
  if (!ptr || bytes == 0) return KPM_OK;
  const uintptr_t pg = 4096, a = (uintptr_t)ptr, e = a + (uintptr_t)bytes;
  const uintptr_t lo = (a + pg - 1) & ~(pg - 1), hi = e & ~(pg - 1);
  if (hi > lo) madvise((void *)lo, hi - lo, MADV_HUGEPAGE);  // advisory only
  if (threads <= 0) {
    const unsigned hc = std::thread::hardware_concurrency();
    threads = (int)(hc == 0 ? 1 : (hc < 16 ? hc : 16));
  }
  const uintptr_t base = a & ~(pg - 1);
  const int64_t pages = (int64_t)((e - base + pg - 1) / pg);  // pages the buffer spans
  if (pages < 4 * threads) threads = 1;
  auto touch = [=](int64_t p0, int64_t p1) {
    volatile char *c = (volatile char *)ptr;
    for (int64_t q = p0; q < p1; ++q) {
      const uintptr_t at = base + (uintptr_t)q * pg;
      c[(at > a ? at : a) - a] = 0;  // first byte of page q inside the buffer
    }
  };
  if (threads == 1) {
    touch(0, pages);
    return KPM_OK;
  }
  std::vector<std::thread> ts;
  int64_t done = 0;  // pages [0, done) are covered by started threads
  try {
    for (int t = 0; t < threads; ++t) {
      const int64_t p0 = pages * t / threads, p1 = pages * (t + 1) / threads;
      ts.emplace_back(touch, p0, p1);
      done = p1;
    }
  } catch (...) {  // no thread available: the caller's thread finishes the rest
  }
  touch(done, pages);
  for (auto &t : ts) t.join();
  return KPM_OK;
}
