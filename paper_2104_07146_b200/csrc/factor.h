// H-factor object and entry points (hfactor.hpp:34-77).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "hmgp_internal.h"
#include "linalg.cuh"

namespace hmgp_gpu {

struct Trip {  // sub_product target and operands: C -= A diag(d) B^T
  int c, a, b;
};

struct Factor {
  Geometry* g = nullptr;  // non-owning, like HFactor::tree_ (hfactor.hpp:63)
  bool ldl = true;
  double eps = 1e-6;
  std::vector<HNode> nodes;
  std::vector<int> leaf_node;
  std::vector<LeafDev> leaf;
  double* pool = nullptr;
  LeafDev* d_leaf = nullptr;
  int* d_rank = nullptr;
  int* d_compact = nullptr;
  double* d_d = nullptr;  // D (LDL) or L_ii (Cholesky), tree order
  LeafFactorStatus* d_status = nullptr;
  double clamp_tol = 0.0;
  int clamped = 0, negative = 0, fail_pos = 0;
  double min_pivot = 0.0, fail_val = 0.0;
  std::vector<int> rank_host;
  std::vector<int> diag_leaf, diag_base, fwd_off, bwd_off;
  void* d_fwd = nullptr;
  void* d_bwd = nullptr;
  double* d_work = nullptr;
  // persistent-sweep solve plans (factor.cu, K10)
  void* d_fsteps = nullptr;
  void* d_funits = nullptr;
  void* d_bsteps = nullptr;
  void* d_bunits = nullptr;
  double* d_part = nullptr;
  int solve_stride = 1;
  size_t arena_peak = 0;
  bool borrowed = false;  // pool / rank arrays / d_d / d_status belong to the thread's graph cache
  ~Factor();
};

void factorize(Factor& F, HMat& H, double eps_f, bool ldl, cudaStream_t st, size_t arena_bytes);
void forward_solve(const Factor& F, double* v, cudaStream_t st);
void backward_solve(const Factor& F, double* v, cudaStream_t st);
double factor_log_det(const Factor& F, cudaStream_t st);
double factor_quad_form_dev(const Factor& F, const double* d_b, cudaStream_t st);
void factor_solve_dev(const Factor& F, const double* d_b, double* d_x, bool full, cudaStream_t st);
double factor_storage_bytes(const Factor& F);
// frees the calling host thread's persistent device arena (the next
// factorization on this thread allocates it again)
void release_thread_workspace();
// device arena of the next factorizations on this host thread (0: automatic)
extern thread_local size_t t_arena_bytes;
// arena peak and H-matrix payload bytes of this thread's last factorization
extern thread_local size_t t_last_arena_peak, t_last_pool_bytes;
// factorizations on this thread use only their own stream (θ-batch workers:
// concurrency comes from the other workers, and fewer streams per worker keep
// the hardware work queues from being shared)
extern thread_local bool t_one_stream;
// the factor of the next factorize() on this thread is ephemeral (destroyed before
// the thread factorizes again): its launch sequence may be captured / replayed as a
// CUDA graph over buffers the thread keeps (factor.cu, "captured factorization")
extern thread_local bool t_graph_ok;

}  // namespace hmgp_gpu
