// Stream-ordered device allocation for per-evaluation buffers (see common.cuh).
#include <cstdint>
#include <mutex>
#include <unordered_set>

#include "common.cuh"

namespace hmgp_gpu {
namespace {
thread_local cudaStream_t t_alloc_stream = nullptr;
std::mutex g_mu;
std::unordered_set<void*> g_async;  // pointers from cudaMallocAsync

void pool_setup() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;  // keep freed blocks cached for the next evaluation
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

void trim_pool() {
  cudaGetLastError();
  cudaDeviceSynchronize();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
}
}  // namespace

void dev_pool_trim() { trim_pool(); }

// Last resort before reporting out-of-memory: whoever keeps device workspaces
// between calls (the persistent θ-batch workers, pipeline.cu) registers a
// callback that gives them back.  Declared here (not in common.cuh) on purpose:
// only pipeline.cu sets it.
void (*g_low_memory_hook)() = nullptr;
static bool reclaim() {
  if (!g_low_memory_hook) return false;
  g_low_memory_hook();
  trim_pool();
  return true;
}

AllocScope::AllocScope(cudaStream_t s) : prev(t_alloc_stream) {
  pool_setup();
  t_alloc_stream = s;
}
AllocScope::~AllocScope() { t_alloc_stream = prev; }

cudaError_t dev_malloc_plain(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    trim_pool();
    e = cudaMalloc(p, bytes);
  }
  if (e == cudaErrorMemoryAllocation && reclaim()) e = cudaMalloc(p, bytes);
  return e;
}

void* dev_alloc(size_t bytes) {
  void* p = nullptr;
  if (t_alloc_stream) {
    cudaError_t e = cudaMallocAsync(&p, bytes, t_alloc_stream);
    if (e == cudaErrorMemoryAllocation) {
      trim_pool();
      e = cudaMallocAsync(&p, bytes, t_alloc_stream);
    }
    if (e == cudaErrorMemoryAllocation && reclaim()) e = cudaMallocAsync(&p, bytes, t_alloc_stream);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      // a capacity failure, not a CUDA fault: θ-batch workers hand the θ back to the
      // caller's thread, which runs it once the others have released their share
      throw Error(6 /* HMGP_ECAPACITY */, "device memory exhausted (per-evaluation buffer)");
    }
    HMGP_CUDA(e);
    std::lock_guard<std::mutex> lk(g_mu);
    g_async.insert(p);
    return p;
  }
  const cudaError_t e = dev_malloc_plain(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(6 /* HMGP_ECAPACITY */, "device memory exhausted");
  }
  HMGP_CUDA(e);
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  bool async = false;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    async = g_async.erase(p) > 0;
  }
  if (async && t_alloc_stream)
    cudaFreeAsync(p, t_alloc_stream);
  else
    cudaFree(p);
}

}  // namespace hmgp_gpu
