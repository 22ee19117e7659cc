// Opaque handle definitions behind include/hmgp_cuda.h and the internal entry
// points the C ABI dispatches to.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../../include/hmgp_cuda.h"
#include "hmgp_internal.h"
#include "phases.h"

struct hmgp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  hmgp_gpu::PhaseTimer timer;
  double phase_ms[hmgp_gpu::PH_COUNT] = {};
};

// Times the phases of one pipeline call on the context's stream.
struct PhaseScope {
  hmgp_ctx* c;
  explicit PhaseScope(hmgp_ctx* ctx) : c(ctx) {
    c->timer.begin(c->stream);
    hmgp_gpu::t_phase = &c->timer;
    hmgp_gpu::phase_mark(hmgp_gpu::PH_START);
  }
  void finish() {
    hmgp_gpu::t_phase = nullptr;
    c->timer.collect(c->phase_ms);
  }
  ~PhaseScope() { hmgp_gpu::t_phase = nullptr; }
};
struct hmgp_geom {
  hmgp_gpu::Geometry g;
};
struct hmgp_hmat {
  hmgp_gpu::HMat h;
  // from_dense (hmatrix.cpp:223-242): the H-matrix owns its one-cluster tree;
  // factors of it share the ownership (the reference's owned_tree_)
  std::shared_ptr<hmgp_geom> owned_geom;
  bool symmetric = true;
};
namespace hmgp_gpu {
struct Factor;
}
struct hmgp_factor {
  std::unique_ptr<hmgp_gpu::Factor> f;
  std::shared_ptr<hmgp_geom> owned_geom;
  ~hmgp_factor();
};

void hmgp_set_pivot(int idx, double v);
void hmgp_validate_matern(const hmgp_matern* p);

namespace hmgp_gpu {
double normal_quantile_host(double p);
bool device_all_finite(const double* d_x, size_t count, cudaStream_t st);
void kernel_pairs(cudaStream_t st, const double* coords, int n, int dim, const MaternDev& p,
                  const int32_t* ii, const int32_t* jj, int64_t count, double* out);
void at_distance(cudaStream_t st, const MaternDev& p, const double* h, int64_t count, double* out);
// sample_grf (simgen.cpp:125-141): z = chol(cov_dense) w, host buffers
void sample_grf_dense(cudaStream_t st, const double* coords, int n, int dim, const MaternDev& p,
                      const double* w, double* out);
// kriging_variance_dense (krige.cpp:46-74) / mloe_mmom (metrics.cpp:17-69), dense,
// n <= 4096, host buffers; idx = the m sampled targets
void kriging_variance_dense(cudaStream_t st, const double* train, int n, const double* test, int m, int dim,
                            const MaternDev& p, double* out);
void mloe_mmom(cudaStream_t st, const double* x, int n, int dim, const MaternDev& pt, const MaternDev& pa,
               const int* idx, int m, double* mloe, double* mmom);
void matern_batch(cudaStream_t st, const double* h, int64_t count, double sigma2, double ell, double nu,
                  double tau2, int generic, double* out);
void bessel_batch(cudaStream_t st, const double* nu, const double* x, int64_t count, int generic,
                  double* out);
void hmat_matvec(cudaStream_t st, const HMat& h, const double* x, double* y);
// the same product with device vectors (original order); plan cached per H-matrix (matvec.cu)
void hmat_matvec_device(cudaStream_t st, const HMat& h, const double* d_x, double* d_y);
void hmat_matvec_forget(const HMat* h);
// dense diagnostics, n <= 4096 (hmatrix.cpp:274-297, hfactor.cpp:421-449), host out
void hmat_to_dense(cudaStream_t st, const HMat& h, double* out);              // original order
void factor_lower_dense(cudaStream_t st, const Factor& F, double* out);       // tree order
void factor_reconstruct(cudaStream_t st, const Factor& F, double* out);       // original order
// K12: d_out[i] = sum_j at_distance(|test_i - train_j|) d_w[j] (all device, AoS coords)
void cross_apply(cudaStream_t st, const double* d_train, int n, int dim, const double* d_w,
                 const double* d_test, int m, const MaternDev& p, double* d_out);
}  // namespace hmgp_gpu
