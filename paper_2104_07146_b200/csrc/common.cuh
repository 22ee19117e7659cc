// Shared device/host helpers for the hmgp B200 library (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace hmgp_gpu {

// NVTX phase range (SURVEY.md §5 tracing): visible in Nsight Systems / ncu --nvtx,
// a no-op costing one load when no tool is attached (header-only NVTX3).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


// Error raised inside the library; mapped to a C-ABI status code.
struct Error : std::runtime_error {
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
  int code;
};

}  // namespace hmgp_gpu

#define HMGP_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw hmgp_gpu::Error(5 /*HMGP_ECUDA*/, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace hmgp_gpu {
// Number of device kernels this library has launched (reported by bench.py as
// gpu_launches; incremented at every launch site through HMGP_LAUNCH_CHECK).
extern std::atomic<uint64_t> g_launches;
}
#define HMGP_LAUNCH_CHECK()                  \
  do {                                       \
    hmgp_gpu::g_launches.fetch_add(1);       \
    HMGP_CUDA(cudaGetLastError());           \
  } while (0)

namespace hmgp_gpu {

// Device memory for per-evaluation buffers (alloc.cu).  Inside an AllocScope
// (one L(θ) evaluation on its stream) buffers come from the device's
// stream-ordered pool (cudaMallocAsync / cudaFreeAsync on that stream): freeing
// them never synchronises the device, so concurrent θ workers do not serialise
// each other on cudaFree.  Outside a scope: cudaMalloc / cudaFree.  Allocation
// failures trim the pool's cached memory and retry once.
void* dev_alloc(size_t bytes);
void dev_free(void* p);
template <class T>
T* dev_alloc_n(size_t count) {
  return static_cast<T*>(dev_alloc((count ? count : 1) * sizeof(T)));
}
struct AllocScope {
  cudaStream_t prev;
  explicit AllocScope(cudaStream_t s);
  ~AllocScope();
};
// plain cudaMalloc with the same trim-and-retry on failure (persistent buffers)
cudaError_t dev_malloc_plain(void** p, size_t bytes);
// release the pool's cached (freed) blocks to the device (synchronises the device)
void dev_pool_trim();

constexpr int kSMs = 148;  // B200

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024); result broadcast.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = threadIdx.x < nw ? red[threadIdx.x] : 0.0;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// Block-wide argmax of |v| with the LOWEST index winning ties (the reference's
// strict '>' scans, hmatrix.cpp:36,84).  Entries with idx < 0 are ignored.
// Returns the best index (or -1) and writes the best value through *best.
__device__ __forceinline__ int block_argmax(double a, int idx, double* redv, int* redi,
                                            double* best) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (idx < 0) a = -1.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double a2 = __shfl_xor_sync(0xffffffffu, a, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (a2 > a || (a2 == a && i2 >= 0 && (idx < 0 || i2 < idx))) {
      a = a2;
      idx = i2;
    }
  }
  __syncthreads();
  if (lane == 0) {
    redv[w] = a;
    redi[w] = idx;
  }
  __syncthreads();
  if (w == 0) {
    a = lane < nw ? redv[lane] : -1.0;
    idx = lane < nw ? redi[lane] : -1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double a2 = __shfl_xor_sync(0xffffffffu, a, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (a2 > a || (a2 == a && i2 >= 0 && (idx < 0 || i2 < idx))) {
        a = a2;
        idx = i2;
      }
    }
    if (lane == 0) {
      redv[0] = a;
      redi[0] = idx;
    }
  }
  __syncthreads();
  const int r = redi[0];
  *best = redv[0];
  __syncthreads();
  return r;
}

}  // namespace hmgp_gpu
