// Device-side phase timing (CUDA events on the library stream) and algorithmic
// work counters, used by bench.py for the roofline and the per-phase share.
#pragma once
#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "matern.cuh"

namespace hmgp_gpu {

enum Phase {
  PH_START = 0,
  PH_GEOMETRY = 1,   // K1 + K2
  PH_DENSE = 2,      // K3 dense Matérn leaves
  PH_ACA = 3,        // K4 ACA + K5 truncation
  PH_LAYOUT = 4,     // pool layout, copies, coarsening
  PH_FACTOR = 5,     // K6-K9 H-LDL / H-Cholesky
  PH_LOGDET = 6,     // K11 log-determinant
  PH_FWD = 7,        // K10 forward solve + quadratic form
  PH_BWD = 8,        // K10 backward solve
  PH_CROSS = 9,      // K12 kriging cross-covariance
  PH_COUNT = 10
};

struct PhaseTimer {
  cudaStream_t st = nullptr;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  void begin(cudaStream_t s) {
    st = s;
    marks.clear();
    used = 0;
  }
  void mark(int phase) {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    cudaEvent_t e = pool[used++];
    cudaEventRecord(e, st);
    marks.push_back({phase, e});
  }
  // per-phase device milliseconds between consecutive marks (after a sync)
  void collect(double* ms) {
    for (int i = 0; i < PH_COUNT; ++i) ms[i] = 0.0;
    cudaStreamSynchronize(st);
    for (size_t k = 1; k < marks.size(); ++k) {
      float t = 0.f;
      cudaEventElapsedTime(&t, marks[k - 1].second, marks[k].second);
      ms[marks[k].first] += t;
    }
  }
  ~PhaseTimer() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// Active timer of the calling thread (set by the pipeline entry points).
extern thread_local PhaseTimer* t_phase;
inline void phase_mark(int i) {
  if (t_phase) t_phase->mark(i);
}

// Work counters (host side accumulators filled from device counters).
struct WorkCounters {
  double dense_entries = 0, aca_entries = 0, kernel_flops = 0;
  double gemm_flops = 0, trsm_flops = 0, leaf_flops = 0, trunc_flops = 0, trunc_items = 0;
  double arena_peak = 0, factor_attempts = 0;
};
extern WorkCounters g_work;
extern bool g_count_kernel_flops;  // run the (untimed) Matérn flop-count pass

// per-translation-unit device counters -> host
void linalg_counters_read_reset(double* gemm, double* trsm, double* leaf);
void truncate_counters_read_reset(double* flops, double* items);
double aca_entries_read_reset();
double dense_kernel_flops(const void* items, int count, const MaternDev& p, const double* xt,
                          int n_pts, int dim, cudaStream_t st);

}  // namespace hmgp_gpu
