// Entry-level kernels (parity hooks), H-matvec, K12 kriging cross-covariance,
// and host-side input utilities.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "hmgp_api.h"
#include "hmgp_internal.h"

namespace hmgp_gpu {

namespace {
template <class T>
struct DBuf {
  T* p = nullptr;
  explicit DBuf(size_t n) { p = hmgp_gpu::dev_alloc_n<T>(n); }
  ~DBuf() { hmgp_gpu::dev_free(p); }
};
}  // namespace

__global__ void k_all_finite(const double* __restrict__ x, size_t count, int* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) *bad = 1;
}

bool device_all_finite(const double* d_x, size_t count, cudaStream_t st) {
  DBuf<int> bad(1);
  HMGP_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
  k_all_finite<<<kSMs * 4, 256, 0, st>>>(d_x, count, bad.p);
  HMGP_LAUNCH_CHECK();
  int h = 0;
  HMGP_CUDA(cudaMemcpyAsync(&h, bad.p, 4, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  return h == 0;
}

__global__ void k_kernel_pairs(const double* __restrict__ x, int dim, MaternDev p,
                               const int* __restrict__ ii, const int* __restrict__ jj,
                               int64_t count, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int a = ii[t], b = jj[t];
    if (a == b) {
      out[t] = p.sigma2 + p.tau2;
      continue;
    }
    const double* pa = x + (size_t)a * dim;
    const double* pb = x + (size_t)b * dim;
    const double h = dim == 2 ? dist2d(pa[0], pa[1], pb[0], pb[1])
                              : dist3d(pa[0], pa[1], pa[2], pb[0], pb[1], pb[2]);
    out[t] = matern_at(p, h);
  }
}

void kernel_pairs(cudaStream_t st, const double* coords, int n, int dim, const MaternDev& p,
                  const int32_t* ii, const int32_t* jj, int64_t count, double* out) {
  if (count <= 0) return;
  DBuf<double> dx((size_t)n * dim), dout(count);
  DBuf<int> di(count), dj(count);
  HMGP_CUDA(cudaMemcpyAsync(dx.p, coords, 8ull * n * dim, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(di.p, ii, 4ull * count, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(dj.p, jj, 4ull * count, cudaMemcpyHostToDevice, st));
  k_kernel_pairs<<<kSMs * 8, 256, 0, st>>>(dx.p, dim, p, di.p, dj.p, count, dout.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(out, dout.p, 8ull * count, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

__global__ void k_at_distance(MaternDev p, const double* __restrict__ h, int64_t count,
                              double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = matern_at(p, h[t]);
}

void at_distance(cudaStream_t st, const MaternDev& p, const double* h, int64_t count, double* out) {
  if (count <= 0) return;
  DBuf<double> dh(count), dout(count);
  HMGP_CUDA(cudaMemcpyAsync(dh.p, h, 8ull * count, cudaMemcpyHostToDevice, st));
  k_at_distance<<<kSMs * 8, 256, 0, st>>>(p, dh.p, count, dout.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(out, dout.p, 8ull * count, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

__global__ void k_bessel(const double* __restrict__ nu, const double* __restrict__ x, int64_t count,
                         int generic, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double v = nu[t], z = x[t];
    const double hs = v - 0.5;
    if (!generic && hs == floor(hs) && hs >= 0.0)  // covkernel.cpp:200-202
      out[t] = bessel_half((int)hs, z);
    else
      out[t] = bessel_k_generic_dev(v, z);
  }
}

void bessel_batch(cudaStream_t st, const double* nu, const double* x, int64_t count, int generic,
                  double* out) {
  if (count <= 0) return;
  DBuf<double> dn(count), dx(count), dout(count);
  HMGP_CUDA(cudaMemcpyAsync(dn.p, nu, 8ull * count, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(dx.p, x, 8ull * count, cudaMemcpyHostToDevice, st));
  k_bessel<<<kSMs * 8, 256, 0, st>>>(dn.p, dx.p, count, generic, dout.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(out, dout.p, 8ull * count, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

// matern(h, p) / detail::matern_generic (covkernel.cpp:184-194, 206-214): the
// public entry point uses pref * t^nu * K_nu(t) (no closed forms), K_nu with the
// half-integer shortcut unless `generic`.  pref = sigma2 2^(1-nu) / Gamma(nu) is
// computed on the host, as the reference does.
__global__ void k_matern_values(const double* __restrict__ h, int64_t count, double sigma2,
                                double ell, double nu, double tau2, double pref, int generic,
                                double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double hv = h[t];
    if (hv == 0.0) {
      out[t] = sigma2 + tau2;
      continue;
    }
    const double x = hv / ell;
    if (x < 1e-10) {
      out[t] = sigma2;
      continue;
    }
    const double hs = nu - 0.5;
    const double k = (!generic && hs == floor(hs) && hs >= 0.0) ? bessel_half((int)hs, x)
                                                                : bessel_k_generic_dev(nu, x);
    out[t] = pref * pow(x, nu) * k;
  }
}

void matern_batch(cudaStream_t st, const double* h, int64_t count, double sigma2, double ell, double nu,
                  double tau2, int generic, double* out) {
  if (count <= 0) return;
  const double pref = sigma2 * std::pow(2.0, 1.0 - nu) / std::tgamma(nu);
  DBuf<double> dh(count), dout(count);
  HMGP_CUDA(cudaMemcpyAsync(dh.p, h, 8ull * count, cudaMemcpyHostToDevice, st));
  k_matern_values<<<kSMs * 8, 256, 0, st>>>(dh.p, count, sigma2, ell, nu, tau2, pref, generic, dout.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(out, dout.p, 8ull * count, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------------- H-matvec ---
// One CTA per stored leaf; y (tree order) accumulated with FP64 atomics.
__global__ void k_leaf_matvec(const LeafDev* __restrict__ lf, const int* __restrict__ rank,
                              const int* __restrict__ r0, const int* __restrict__ c0,
                              const double* __restrict__ xt, double* __restrict__ yt,
                              double* __restrict__ scratch, int sym_stride) {
  const int k = blockIdx.x;
  const LeafDev L = lf[k];
  const int rb = r0[k], cb = c0[k];
  const bool mirror = rb != cb;
  double* t = scratch + (size_t)k * sym_stride;  // 2 * cap doubles
  if (L.kind == DENSE) {
    for (int i = threadIdx.x; i < L.m; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < L.n; ++j) s += L.a[(size_t)j * L.m + i] * xt[cb + j];
      atomicAdd(&yt[rb + i], s);
    }
    if (mirror)
      for (int j = threadIdx.x; j < L.n; j += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < L.m; ++i) s += L.a[(size_t)j * L.m + i] * xt[rb + i];
        atomicAdd(&yt[cb + j], s);
      }
    return;
  }
  const int r = rank[k];
  if (r <= 0) return;
  for (int l = threadIdx.x; l < r; l += blockDim.x) {
    double s = 0.0, s2 = 0.0;
    for (int j = 0; j < L.n; ++j) s += L.b[(size_t)l * L.n + j] * xt[cb + j];
    for (int i = 0; i < L.m; ++i) s2 += L.a[(size_t)l * L.m + i] * xt[rb + i];
    t[l] = s;
    t[L.cap + l] = s2;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < L.m; i += blockDim.x) {
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += L.a[(size_t)l * L.m + i] * t[l];
    atomicAdd(&yt[rb + i], s);
  }
  if (mirror)
    for (int j = threadIdx.x; j < L.n; j += blockDim.x) {
      double s = 0.0;
      for (int l = 0; l < r; ++l) s += L.b[(size_t)l * L.n + j] * t[L.cap + l];
      atomicAdd(&yt[cb + j], s);
    }
}

__global__ void k_permute_in(const double* __restrict__ x, const int* __restrict__ perm, int n,
                             double* __restrict__ xt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) xt[k] = x[perm[k]];
}
__global__ void k_permute_out(const double* __restrict__ yt, const int* __restrict__ perm, int n,
                              double* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[perm[k]] = yt[k];
}

void hmat_matvec(cudaStream_t st, const HMat& h, const double* x, double* y) {
  const Geometry& G = *h.g;
  const int n = G.n, L = (int)h.leaf.size();
  if (!getenv("HMGP_MATVEC_LEGACY")) {  // HBM-oriented deterministic pass (matvec.cu)
    DBuf<double> dx(n), dy(n);
    HMGP_CUDA(cudaMemcpyAsync(dx.p, x, 8ull * n, cudaMemcpyHostToDevice, st));
    hmat_matvec_device(st, h, dx.p, dy.p);
    HMGP_CUDA(cudaMemcpyAsync(y, dy.p, 8ull * n, cudaMemcpyDeviceToHost, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
    return;
  }
  NvtxRange nvtx_range("hmgp:matvec(legacy)");
  std::vector<int> r0(L), c0(L);
  int maxcap = 1;
  for (int k = 0; k < L; ++k) {
    const HNode& nd = h.nodes[h.leaf_node[k]];
    r0[k] = G.nbeg[nd.row];
    c0[k] = G.nbeg[nd.col];
    maxcap = std::max(maxcap, h.leaf[k].cap);
  }
  DBuf<double> dx(n), dxt(n), dyt(n), scratch((size_t)L * 2 * maxcap);
  DBuf<int> dr0(L), dc0(L);
  HMGP_CUDA(cudaMemcpyAsync(dx.p, x, 8ull * n, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(dr0.p, r0.data(), 4ull * L, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(dc0.p, c0.data(), 4ull * L, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemsetAsync(dyt.p, 0, 8ull * n, st));
  k_permute_in<<<(n + 255) / 256, 256, 0, st>>>(dx.p, G.d_perm, n, dxt.p);
  HMGP_LAUNCH_CHECK();
  k_leaf_matvec<<<L, 128, 0, st>>>(h.d_leaf, h.d_rank, dr0.p, dc0.p, dxt.p, dyt.p, scratch.p,
                                   2 * maxcap);
  HMGP_LAUNCH_CHECK();
  k_permute_out<<<(n + 255) / 256, 256, 0, st>>>(dyt.p, G.d_perm, n, dx.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(y, dx.p, 8ull * n, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------- AS241 (host) -----
// Wichura AS241 PPND16 (simgen.cpp:9-106); published coefficients.
double normal_quantile_host(double p) {
  if (!(p > 0.0 && p < 1.0)) throw std::domain_error("std_normal_quantile: p must be in (0, 1)");
  const double q = p - 0.5;
  auto horner = [](const double* c, double r) {
    double v = c[7];
    for (int k = 6; k >= 0; --k) v = v * r + c[k];
    return v;
  };
  if (std::fabs(q) <= 0.425) {
    static const double a[8] = {3.3871328727963666080e+0, 1.3314166789178437745e+2,
                                1.9715909503065514427e+3, 1.3731693765509461125e+4,
                                4.5921953931549871457e+4, 6.7265770927008700853e+4,
                                3.3430575583588128105e+4, 2.5090809287301226727e+3};
    static const double b[8] = {1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2,
                                5.3941960214247511077e+3, 2.1213794301586595867e+4,
                                3.9307895800092710610e+4, 2.8729085735721942674e+4,
                                5.226495278852545609e+3};
    const double r = 0.180625 - q * q;
    return q * horner(a, r) / horner(b, r);
  }
  double r = q < 0.0 ? p : 1.0 - p;
  r = std::sqrt(-std::log(r));
  double x;
  if (r <= 5.0) {
    static const double c[8] = {1.42343711074968357734e+0, 4.63033784615654529590e+0,
                                5.76949722146069140550e+0, 3.64784832476320460504e+0,
                                1.27045825245236838258e+0, 2.41780725177450611770e-1,
                                2.27238449892691845833e-2, 7.74545014278341407640e-4};
    static const double d[8] = {1.0, 2.05319162663775882187e+0, 1.67638483018380384940e+0,
                                6.89767334985100004550e-1, 1.48103976427480074590e-1,
                                1.51986665636164571966e-2, 5.47593808499534494600e-4,
                                1.05075007164441684324e-9};
    r -= 1.6;
    x = horner(c, r) / horner(d, r);
  } else {
    static const double e[8] = {6.65790464350110377720e+0, 5.46378491116411436990e+0,
                                1.78482653991729133580e+0, 2.96560571828504891230e-1,
                                2.65321895265761230930e-2, 1.24266094738807843860e-3,
                                2.71155556874348757815e-5, 2.01033439929228813265e-7};
    static const double f[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,
                                1.48753612908506148525e-2, 7.868691311456132591e-4,
                                1.8463183175100546818e-5, 1.4215117583164458887e-7,
                                2.04426310338993978564e-15};
    r -= 5.0;
    x = horner(e, r) / horner(f, r);
  }
  return q < 0.0 ? -x : x;
}

}  // namespace hmgp_gpu

// ------------------------------------------------- exact GRF sample (dense) --
// sample_grf (simgen.cpp:125-141) on device, beyond the reference's n <= 16384
// guard: dense covariance (cov_dense, covkernel.cpp:262-275:
// diagonal sigma2 + tau2, off-diagonal at_distance), lower Cholesky, z = L w with
// w the AS241 normals of `seed` drawn on the host exactly as the reference does.
// A data-generation utility, not the measured path: the factorization is the
// library dense POTRF (cuSOLVER 64-bit API), the triangular product cuBLAS TRMV.
namespace hmgp_gpu {

__global__ void k_cov_dense_lower(const double* __restrict__ x, int n, int dim, MaternDev p,
                                  double* __restrict__ C, int j0) {
  // column-major n x n, lower triangle (j <= i); one thread per (i, j), i fastest
  const int j = j0 + blockIdx.y;
  for (int i = j + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v;
    if (i == j) {
      v = p.sigma2 + p.tau2;
    } else {
      const double* pa = x + (size_t)i * dim;
      const double* pb = x + (size_t)j * dim;
      const double h = dim == 2 ? dist2d(pa[0], pa[1], pb[0], pb[1])
                                : dist3d(pa[0], pa[1], pa[2], pb[0], pb[1], pb[2]);
      v = matern_at(p, h);
    }
    C[(size_t)j * n + i] = v;
  }
}

void sample_grf_dense(cudaStream_t st, const double* coords, int n, int dim, const MaternDev& p,
                      const double* w, double* out) {
  DBuf<double> dx((size_t)n * dim), dC((size_t)n * n), dw(n);
  HMGP_CUDA(cudaMemcpyAsync(dx.p, coords, 8ull * n * dim, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(dw.p, w, 8ull * n, cudaMemcpyHostToDevice, st));
  for (int j0 = 0; j0 < n; j0 += 65535) {  // grid.y limit
    const int nj = std::min(65535, n - j0);
    const int gx = std::min((n - j0 + 255) / 256, 64);
    dim3 grid(gx, nj);  // block (x, y) handles column j0 + y
    k_cov_dense_lower<<<grid, 256, 0, st>>>(dx.p, n, dim, p, dC.p, j0);
    HMGP_LAUNCH_CHECK();
  }
  // blocked right-looking Cholesky, nb = 4096: POTRF of each diagonal block
  // (cuSOLVER), TRSM of the panel below it and SYRK of the trailing matrix
  // (cuBLAS 64-bit API) -- every library call stays far below 2^31 elements
  // per operand dimension product except the GEMM-like updates, which take
  // 64-bit sizes
  cusolverDnHandle_t sh = nullptr;
  cusolverDnParams_t prm = nullptr;
  cublasHandle_t bh = nullptr;
  if (cusolverDnCreate(&sh) != CUSOLVER_STATUS_SUCCESS) throw Error(HMGP_ECUDA, "cusolverDnCreate failed");
  if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) {
    cusolverDnDestroy(sh);
    throw Error(HMGP_ECUDA, "cublasCreate failed");
  }
  cusolverDnSetStream(sh, st);
  cublasSetStream(bh, st);
  cusolverDnCreateParams(&prm);
  const int64_t nb = 4096, ld = n;
  bool lib_ok = true;
  int info = 0;
  {
    size_t dbytes = 0, hbytes = 0;
    const int64_t b0 = std::min<int64_t>(nb, n);
    lib_ok = cusolverDnXpotrf_bufferSize(sh, prm, CUBLAS_FILL_MODE_LOWER, b0, CUDA_R_64F, dC.p, ld, CUDA_R_64F,
                                         &dbytes, &hbytes) == CUSOLVER_STATUS_SUCCESS;
    DBuf<char> dwork(std::max<size_t>(dbytes, 1));
    std::vector<char> hwork(std::max<size_t>(hbytes, 1));
    DBuf<int> dinfo(1);
    for (int64_t k0 = 0; lib_ok && k0 < n; k0 += nb) {
      const int64_t kb = std::min<int64_t>(nb, n - k0), rest = n - k0 - kb;
      double* A11 = dC.p + (size_t)k0 * ld + k0;
      lib_ok = cusolverDnXpotrf(sh, prm, CUBLAS_FILL_MODE_LOWER, kb, CUDA_R_64F, A11, ld, CUDA_R_64F, dwork.p,
                                dbytes, hwork.data(), hbytes, dinfo.p) == CUSOLVER_STATUS_SUCCESS;
      HMGP_CUDA(cudaMemcpyAsync(&info, dinfo.p, 4, cudaMemcpyDeviceToHost, st));
      HMGP_CUDA(cudaStreamSynchronize(st));
      if (!lib_ok || info != 0) break;
      if (rest > 0) {
        double* A21 = A11 + kb;
        double* A22 = A21 + (size_t)kb * ld;
        const double one = 1.0, mone = -1.0;
        lib_ok = cublasDtrsm_64(bh, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                                rest, kb, &one, A11, ld, A21, ld) == CUBLAS_STATUS_SUCCESS &&
                 cublasDsyrk_64(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, rest, kb, &mone, A21, ld, &one, A22,
                                ld) == CUBLAS_STATUS_SUCCESS;
      }
    }
  }
  cusolverDnDestroyParams(prm);
  cusolverDnDestroy(sh);
  if (!lib_ok) {
    cublasDestroy(bh);
    throw Error(HMGP_ECUDA, "sample_grf: cuSOLVER/cuBLAS call failed");
  }
  if (info != 0) {
    cublasDestroy(bh);
    throw std::runtime_error("sample_grf: covariance not SPD; increase nugget tau2");
  }
  const cublasStatus_t bs =
      cublasDtrmv_64(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, dC.p, n, dw.p, 1);
  HMGP_CUDA(cudaMemcpyAsync(out, dw.p, 8ull * n, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  cublasDestroy(bh);
  if (bs != CUBLAS_STATUS_SUCCESS) throw Error(HMGP_ECUDA, "cublasDtrmv failed");
}

}  // namespace hmgp_gpu

// ------------------------------------------------ dense diagnostics (n <= 4096)
// HMatrix::to_dense (hmatrix.cpp:274-297), HFactor::lower_dense / reconstruct
// (hfactor.cpp:421-449): leaves expanded on the device into a dense tree-order
// matrix (one CTA per stored leaf; low-rank leaves as U V^T), then permuted to
// the original order.  SURVEY.md §8f row 3.
#include "factor.h"
namespace hmgp_gpu {

// mode bit 0: symmetric H-matrix (also write the mirror of off-diagonal leaves);
// bit 1: factor (diagonal leaves: strict upper triangle zero, diagonal = 1 for
// LDL or the stored L_ii (diag != nullptr) for Cholesky)
__global__ void k_expand_leaves(const LeafDev* __restrict__ leaf, const int* __restrict__ rank,
                                const int* __restrict__ r0, const int* __restrict__ c0, int n, int mode,
                                const double* __restrict__ diag, double* __restrict__ T) {
  const int k = blockIdx.x;
  const LeafDev L = leaf[k];
  const int rb = r0[k], cb = c0[k];
  const bool on_diag = rb == cb;
  const int r = L.kind == DENSE ? 0 : rank[k];
  for (int e = threadIdx.x; e < L.m * L.n; e += blockDim.x) {
    const int i = e % L.m, j = e / L.m;
    double v;
    if (L.kind == DENSE) {
      v = L.a[(size_t)j * L.m + i];
    } else {
      v = 0.0;
      for (int q = 0; q < r; ++q) v += L.a[(size_t)q * L.m + i] * L.b[(size_t)q * L.n + j];
    }
    if ((mode & 2) && on_diag) {
      if (i < j) v = 0.0;
      if (i == j) v = diag ? diag[rb + i] : 1.0;
    }
    T[(size_t)(cb + j) * n + rb + i] = v;
    if ((mode & 1) && !on_diag) T[(size_t)(rb + i) * n + cb + j] = v;
  }
}

__global__ void k_permute_dense(const double* __restrict__ T, const int* __restrict__ perm, int n,
                                double* __restrict__ out) {
  // out(perm[i], perm[j]) = T(i, j), column-major
  const int j = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[(size_t)perm[j] * n + perm[i]] = T[(size_t)j * n + i];
}

__global__ void k_scale_cols(const double* __restrict__ A, const double* __restrict__ d, int n,
                             double* __restrict__ W) {
  const int j = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    W[(size_t)j * n + i] = A[(size_t)j * n + i] * d[j];
}

static void expand(cudaStream_t st, const Geometry& G, const std::vector<HNode>& nodes,
                   const std::vector<int>& leaf_node, const LeafDev* d_leaf, const int* d_rank, int mode,
                   const double* d_diag, double* d_T) {
  const int n = G.n, L = (int)leaf_node.size();
  std::vector<int> r0(L), c0(L);
  for (int k = 0; k < L; ++k) {
    r0[k] = G.nbeg[nodes[leaf_node[k]].row];
    c0[k] = G.nbeg[nodes[leaf_node[k]].col];
  }
  DBuf<int> dr0(L), dc0(L);
  HMGP_CUDA(cudaMemcpyAsync(dr0.p, r0.data(), 4ull * L, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(dc0.p, c0.data(), 4ull * L, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemsetAsync(d_T, 0, 8ull * n * n, st));
  if (L > 0) {
    k_expand_leaves<<<L, 256, 0, st>>>(d_leaf, d_rank, dr0.p, dc0.p, n, mode, d_diag, d_T);
    HMGP_LAUNCH_CHECK();
  }
  HMGP_CUDA(cudaStreamSynchronize(st));
}

static void check_dense_n(int n, const char* what) {
  if (n > 4096) throw std::invalid_argument(std::string(what) + ": refused beyond n = 4096");
}

void hmat_to_dense(cudaStream_t st, const HMat& h, double* out) {
  const Geometry& G = *h.g;
  const int n = G.n;
  check_dense_n(n, "to_dense");
  DBuf<double> T((size_t)n * n), O((size_t)n * n);
  expand(st, G, h.nodes, h.leaf_node, h.d_leaf, h.d_rank, 1, nullptr, T.p);
  k_permute_dense<<<dim3((n + 255) / 256, n), 256, 0, st>>>(T.p, G.d_perm, n, O.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(out, O.p, 8ull * n * n, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

void factor_lower_dense(cudaStream_t st, const Factor& F, double* out) {
  const int n = F.g->n;
  check_dense_n(n, "lower_dense");
  DBuf<double> T((size_t)n * n);
  expand(st, *F.g, F.nodes, F.leaf_node, F.d_leaf, F.d_rank, 2, F.ldl ? nullptr : F.d_d, T.p);
  HMGP_CUDA(cudaMemcpyAsync(out, T.p, 8ull * n * n, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

void factor_reconstruct(cudaStream_t st, const Factor& F, double* out) {
  const int n = F.g->n;
  check_dense_n(n, "reconstruct");
  DBuf<double> T((size_t)n * n), W((size_t)n * n), M((size_t)n * n);
  expand(st, *F.g, F.nodes, F.leaf_node, F.d_leaf, F.d_rank, 2, F.ldl ? nullptr : F.d_d, T.p);
  const double* Lw = T.p;
  if (F.ldl) {  // W = L diag(d)
    k_scale_cols<<<dim3((n + 255) / 256, n), 256, 0, st>>>(T.p, F.d_d, n, W.p);
    HMGP_LAUNCH_CHECK();
    Lw = W.p;
  }
  cublasHandle_t bh = nullptr;
  if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) throw Error(HMGP_ECUDA, "cublasCreate failed");
  cublasSetStream(bh, st);
  const double one = 1.0, zero = 0.0;  // M = Lw L^T (tree order)
  const cublasStatus_t bs =
      cublasDgemm(bh, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, Lw, n, T.p, n, &zero, M.p, n);
  cublasDestroy(bh);
  if (bs != CUBLAS_STATUS_SUCCESS) throw Error(HMGP_ECUDA, "cublasDgemm failed");
  k_permute_dense<<<dim3((n + 255) / 256, n), 256, 0, st>>>(M.p, F.g->d_perm, n, W.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(out, W.p, 8ull * n * n, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
}

}  // namespace hmgp_gpu

// ------------------------------------ dense kriging variance / MLOE-MMOM (§8f 4)
// kriging_variance_dense (krige.cpp:46-74) and mloe_mmom (metrics.cpp:17-69): the
// reference's dense small-n diagnostics (n <= 4096), on the device.  Covariance
// and cross-covariance entries come from the same Matérn kernel as the hot path;
// the dense LLT / triangular solves / SYMM are library calls (cuSOLVER POTRF +
// POTRS, cuBLAS DSYMM) since these are diagnostics outside every timed region.
namespace hmgp_gpu {

namespace {
struct DenseLib {
  cusolverDnHandle_t sh = nullptr;
  cusolverDnParams_t prm = nullptr;
  cublasHandle_t bh = nullptr;
  explicit DenseLib(cudaStream_t st) {
    if (cusolverDnCreate(&sh) != CUSOLVER_STATUS_SUCCESS) throw Error(HMGP_ECUDA, "cusolverDnCreate failed");
    if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) {
      cusolverDnDestroy(sh);
      throw Error(HMGP_ECUDA, "cublasCreate failed");
    }
    cusolverDnSetStream(sh, st);
    cublasSetStream(bh, st);
    cusolverDnCreateParams(&prm);
  }
  ~DenseLib() {
    cusolverDnDestroyParams(prm);
    cusolverDnDestroy(sh);
    cublasDestroy(bh);
  }
  // in-place lower Cholesky of the n x n column-major A; false if not SPD
  bool potrf(cudaStream_t st, double* A, int64_t n) {
    size_t db = 0, hb = 0;
    if (cusolverDnXpotrf_bufferSize(sh, prm, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, &db, &hb) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(HMGP_ECUDA, "cusolverDnXpotrf_bufferSize failed");
    DBuf<char> dw(std::max<size_t>(db, 1));
    std::vector<char> hw(std::max<size_t>(hb, 1));
    DBuf<int> dinfo(1);
    if (cusolverDnXpotrf(sh, prm, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, dw.p, db, hw.data(), hb,
                         dinfo.p) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HMGP_ECUDA, "cusolverDnXpotrf failed");
    int info = 0;
    HMGP_CUDA(cudaMemcpyAsync(&info, dinfo.p, 4, cudaMemcpyDeviceToHost, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
    return info == 0;
  }
  // B <- A^-1 B with A = L L^T from potrf, B n x k
  void potrs(cudaStream_t st, const double* L, int64_t n, double* B, int64_t k) {
    DBuf<int> dinfo(1);
    if (cusolverDnXpotrs(sh, prm, CUBLAS_FILL_MODE_LOWER, n, k, CUDA_R_64F, L, n, CUDA_R_64F, B, n, dinfo.p) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(HMGP_ECUDA, "cusolverDnXpotrs failed");
  }
};

void cov_lower(cudaStream_t st, const double* d_x, int n, int dim, const MaternDev& p, double* d_C) {
  k_cov_dense_lower<<<dim3(std::min((n + 255) / 256, 64), n), 256, 0, st>>>(d_x, n, dim, p, d_C, 0);
  HMGP_LAUNCH_CHECK();
}
}  // namespace

// C(j, k) = at_distance(|test_k - train_j|), column-major n x m (one column per
// new location, the reference's c vector)
__global__ void k_cov_cross(const double* __restrict__ train, int n, const double* __restrict__ test, int dim,
                            MaternDev p, double* __restrict__ Cnm) {
  const int k = blockIdx.y;
  const double* pa = test + (size_t)k * dim;
  const double ax = pa[0], ay = pa[1], az = dim == 3 ? pa[2] : 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double* pb = train + (size_t)j * dim;
    const double h = dim == 2 ? dist2d(ax, ay, pb[0], pb[1]) : dist3d(ax, ay, az, pb[0], pb[1], pb[2]);
    Cnm[(size_t)k * n + j] = matern_at(p, h);
  }
}

template <int NT>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[NT / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;  // valid on thread 0
}

// out[k] = prior - c_k . x_k with the reference's (-1e-9, 0) -> 0 clamp
__global__ void k_kvar_finish(const double* __restrict__ Cnm, const double* __restrict__ X, int n, double prior,
                              double* __restrict__ out) {
  const int k = blockIdx.x;
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += 256) s += Cnm[(size_t)k * n + j] * X[(size_t)k * n + j];
  s = block_sum<256>(s);
  if (threadIdx.x == 0) {
    double v = prior - s;
    if (v < 0.0 && v > -1e-9) v = 0.0;
    out[k] = v;
  }
}

void kriging_variance_dense(cudaStream_t st, const double* train, int n, const double* test, int m, int dim,
                            const MaternDev& p, double* out) {
  if (m == 0) return;
  DBuf<double> dx((size_t)n * dim), dL((size_t)n * n);
  HMGP_CUDA(cudaMemcpyAsync(dx.p, train, 8ull * n * dim, cudaMemcpyHostToDevice, st));
  cov_lower(st, dx.p, n, dim, p, dL.p);
  DenseLib lib(st);
  if (!lib.potrf(st, dL.p, n))
    throw std::runtime_error("kriging_variance_dense: C11 not SPD; increase nugget tau2");
  const int mb = std::min(m, 4096);
  DBuf<double> dt((size_t)mb * dim), dC((size_t)n * mb), dX((size_t)n * mb), dv(mb);
  const double prior = p.sigma2 + p.tau2;
  for (int k0 = 0; k0 < m; k0 += mb) {
    const int kb = std::min(mb, m - k0);
    HMGP_CUDA(cudaMemcpyAsync(dt.p, test + (size_t)k0 * dim, 8ull * kb * dim, cudaMemcpyHostToDevice, st));
    k_cov_cross<<<dim3(std::min((n + 255) / 256, 16), kb), 256, 0, st>>>(dx.p, n, dt.p, dim, p, dC.p);
    HMGP_LAUNCH_CHECK();
    HMGP_CUDA(cudaMemcpyAsync(dX.p, dC.p, 8ull * n * kb, cudaMemcpyDeviceToDevice, st));
    lib.potrs(st, dL.p, n, dX.p, kb);
    k_kvar_finish<<<kb, 256, 0, st>>>(dC.p, dX.p, n, prior, dv.p);
    HMGP_LAUNCH_CHECK();
    HMGP_CUDA(cudaMemcpyAsync(out + k0, dv.p, 8ull * kb, cudaMemcpyDeviceToHost, st));
  }
  HMGP_CUDA(cudaStreamSynchronize(st));
}

// E(idx[k], k) = 1 in a zeroed n x m matrix
__global__ void k_unit_cols(const int* __restrict__ idx, int n, int m, double* __restrict__ E) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) E[(size_t)k * n + idx[k]] = 1.0;
}

// ga_diag(k) = G_a(idx[k], k); G_a(:, k) *= -1 / ga_diag(k)
__global__ void k_loo_weights(const int* __restrict__ idx, int n, double* __restrict__ Ga, double* __restrict__ gd) {
  const int k = blockIdx.x;
  double* col = Ga + (size_t)k * n;
  const double d = col[idx[k]];
  __syncthreads();  // every thread has read the diagonal before it is scaled
  const double s = -1.0 / d;
  for (int i = threadIdx.x; i < n; i += 256) col[i] *= s;
  if (threadIdx.x == 0) gd[k] = d;
}

// per target k: terms[2k] = E_t[(Zhat_a - Z)^2] / E_t[(Zhat_t - Z)^2] - 1 (MLOE),
// terms[2k+1] = E_a[(Zhat_a - Z)^2] / E_t[(Zhat_a - Z)^2] - 1 (MMOM)
__global__ void k_mloe_terms(const int* __restrict__ idx, int n, const double* __restrict__ Gt,
                             const double* __restrict__ Ga, const double* __restrict__ CtW,
                             const double* __restrict__ gd, double* __restrict__ terms) {
  const int k = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += Ga[(size_t)k * n + i] * CtW[(size_t)k * n + i];
  s = block_sum<256>(s);
  if (threadIdx.x == 0) {
    const double e_tt = 1.0 / Gt[(size_t)k * n + idx[k]], e_aa = 1.0 / gd[k], e_ta = s;
    terms[2 * k] = e_ta / e_tt - 1.0;
    terms[2 * k + 1] = e_aa / e_ta - 1.0;
  }
}

void mloe_mmom(cudaStream_t st, const double* x, int n, int dim, const MaternDev& pt, const MaternDev& pa,
               const int* idx, int m, double* mloe, double* mmom) {
  DBuf<double> dx((size_t)n * dim), dCt((size_t)n * n), dLt((size_t)n * n), dLa((size_t)n * n);
  DBuf<double> dGt((size_t)n * m), dGa((size_t)n * m), dW((size_t)n * m), dgd(m), dterms(2ull * m);
  DBuf<int> didx(m);
  HMGP_CUDA(cudaMemcpyAsync(dx.p, x, 8ull * n * dim, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(didx.p, idx, 4ull * m, cudaMemcpyHostToDevice, st));
  cov_lower(st, dx.p, n, dim, pt, dCt.p);
  HMGP_CUDA(cudaMemcpyAsync(dLt.p, dCt.p, 8ull * n * n, cudaMemcpyDeviceToDevice, st));
  cov_lower(st, dx.p, n, dim, pa, dLa.p);
  DenseLib lib(st);
  if (!lib.potrf(st, dLt.p, n) || !lib.potrf(st, dLa.p, n))
    throw std::runtime_error("mloe_mmom: covariance not SPD; increase nugget tau2");
  HMGP_CUDA(cudaMemsetAsync(dGt.p, 0, 8ull * n * m, st));
  k_unit_cols<<<(m + 255) / 256, 256, 0, st>>>(didx.p, n, m, dGt.p);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaMemcpyAsync(dGa.p, dGt.p, 8ull * n * m, cudaMemcpyDeviceToDevice, st));
  lib.potrs(st, dLt.p, n, dGt.p, m);
  lib.potrs(st, dLa.p, n, dGa.p, m);
  k_loo_weights<<<m, 256, 0, st>>>(didx.p, n, dGa.p, dgd.p);
  HMGP_LAUNCH_CHECK();
  const double one = 1.0, zero = 0.0;  // W = C_t G_a (C_t symmetric, lower stored)
  if (cublasDsymm(lib.bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, n, m, &one, dCt.p, n, dGa.p, n, &zero, dW.p,
                  n) != CUBLAS_STATUS_SUCCESS)
    throw Error(HMGP_ECUDA, "cublasDsymm failed");
  k_mloe_terms<<<m, 256, 0, st>>>(didx.p, n, dGt.p, dGa.p, dW.p, dgd.p, dterms.p);
  HMGP_LAUNCH_CHECK();
  std::vector<double> t(2ull * m);
  HMGP_CUDA(cudaMemcpyAsync(t.data(), dterms.p, 16ull * m, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  double lo = 0.0, mo = 0.0;  // summed in target order, as the reference does
  for (int k = 0; k < m; ++k) {
    lo += t[2 * k];
    mo += t[2 * k + 1];
  }
  *mloe = lo / m;
  *mmom = mo / m;
}

}  // namespace hmgp_gpu
