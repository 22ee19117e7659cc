// K5: batched low-rank recompression (U V^T) <- trunc_eps(U V^T).
//
// Restates hblock.cpp:127-162 (join_truncate) for the case every reference call
// site uses (P, Q empty: fill_leaf hmatrix.cpp:159-161, compress_low_rank
// hblock.cpp:164-170, product_low_rank hfactor.cpp:170-171,187-188):
//   Householder QR of U and V, core = R_u R_v^T, SVD, keep sigma_i > eps*sigma_0
//   (and > 0), U <- Q_u [X_k S_k; 0], V <- Q_v [Y_k; 0].
// One CTA per item; the item's condition (watermark rules of the reference) is
// evaluated ON DEVICE against the device-resident column count, so the host
// never has to read ranks back.  The SVD is a parallel (round-robin) one-sided
// Jacobi; the reference uses Eigen's two-sided JacobiSVD / dgesdd — the same
// singular triplets up to rounding, so the kept rank only differs when a
// singular value sits within rounding of the cut.
#include "common.cuh"
#include "hmgp_internal.h"

namespace hmgp_gpu {

constexpr int kTruncThreads = 256;
constexpr int kMaxTruncCols = 1024;

__device__ double d_cnt_trunc, d_cnt_titems;

void truncate_counters_read_reset(double* flops, double* items) {
  double z = 0.0;
  HMGP_CUDA(cudaMemcpyFromSymbol(flops, d_cnt_trunc, 8));
  HMGP_CUDA(cudaMemcpyFromSymbol(items, d_cnt_titems, 8));
  HMGP_CUDA(cudaMemcpyToSymbol(d_cnt_trunc, &z, 8));
  HMGP_CUDA(cudaMemcpyToSymbol(d_cnt_titems, &z, 8));
}

// LAPACK dgeqrf flop count for an m x r panel
__device__ __forceinline__ double qr_flops(double m, double r) {
  return m >= r ? 2.0 * m * r * r - 2.0 / 3.0 * r * r * r : 2.0 * r * m * m - 2.0 / 3.0 * m * m * m;
}

size_t trunc_ws_doubles(int m, int n, int rcap) {
  const size_t kq = (size_t)min(min(m, n), rcap);
  return (size_t)(m + n) * rcap + 2 * (size_t)rcap + (size_t)rcap * kq + kq * kq;
}

// In-place Householder QR of A (m x r, ld m) inside one CTA; tau[min(m,r)].
__device__ void cta_householder(double* A, int m, int r, double* tau, double* red) {
  const int kmax = min(m, r);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double s_beta, s_t, s_inv;
  for (int k = 0; k < kmax; ++k) {
    double* col = A + (size_t)k * m;
    double part = 0.0;
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) part += col[i] * col[i];
    const double tail2 = block_sum(part, red);
    if (threadIdx.x == 0) {
      const double c0 = col[k];
      if (tail2 <= 2.2250738585072014e-308) {
        s_t = 0.0;
        s_beta = c0;
        s_inv = 0.0;
      } else {
        double beta = sqrt(c0 * c0 + tail2);
        if (c0 >= 0.0) beta = -beta;
        s_inv = 1.0 / (c0 - beta);
        s_t = (beta - c0) / beta;
        s_beta = beta;
      }
    }
    __syncthreads();
    const double t = s_t, inv = s_inv;
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) col[i] = (t == 0.0) ? 0.0 : col[i] * inv;
    __syncthreads();
    if (threadIdx.x == 0) {
      col[k] = s_beta;
      tau[k] = t;
    }
    __syncthreads();
    if (t != 0.0) {
      for (int j = k + 1 + w; j < r; j += nw) {
        double* cj = A + (size_t)j * m;
        double s = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) s += col[i] * cj[i];
        s = warp_sum(s);
        s = (s + cj[k]) * t;
        for (int i = k + 1 + lane; i < m; i += 32) cj[i] -= s * col[i];
        if (lane == 0) cj[k] -= s;
      }
    }
    __syncthreads();
  }
}

// E <- Q E with Q = H_0 ... H_{kq-1} from cta_householder(QR); E m x c (ld m).
__device__ void cta_apply_q(const double* QR, int m, int kq, const double* tau, double* E, int c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = kq - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t != 0.0) {
      const double* v = QR + (size_t)k * m;
      for (int j = w; j < c; j += nw) {
        double* e = E + (size_t)j * m;
        double s = 0.0;
        for (int i = k + 1 + lane; i < m; i += 32) s += v[i] * e[i];
        s = warp_sum(s);
        s = (s + e[k]) * t;
        for (int i = k + 1 + lane; i < m; i += 32) e[i] -= s * v[i];
        if (lane == 0) e[k] -= s;
      }
    }
    __syncthreads();
  }
}

// One-sided Jacobi on W (p x q, ld p, p >= q); J (q x q) accumulates rotations.
// Returns the algorithmic flops (6p per pair inspected, 6(p+q) per rotation).
__device__ double cta_jacobi(double* W, int p, int q, double* J) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int idx = threadIdx.x; idx < q * q; idx += blockDim.x) J[idx] = (idx % (q + 1) == 0) ? 1.0 : 0.0;
  __syncthreads();
  if (q < 2) return 0.0;
  const int qq = q + (q & 1);
  const int m1 = qq - 1;
  __shared__ int s_rot;
  __shared__ unsigned s_nrot;
  if (threadIdx.x == 0) s_nrot = 0;
  int sweeps = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    ++sweeps;
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < m1; ++round) {
      for (int t = w; t < qq / 2; t += nw) {
        int a, b;
        if (t == 0) {
          a = qq - 1;
          b = round;
        } else {
          a = (round + t) % m1;
          b = (round + m1 - t) % m1;
        }
        if (a > b) {
          const int tmp = a;
          a = b;
          b = tmp;
        }
        if (b >= q) continue;
        double* wj = W + (size_t)a * p;
        double* wk = W + (size_t)b * p;
        double sa = 0, sb = 0, sc = 0;
        for (int i = lane; i < p; i += 32) {
          const double x = wj[i], y = wk[i];
          sa += x * x;
          sb += y * y;
          sc += x * y;
        }
        sa = warp_sum(sa);
        sb = warp_sum(sb);
        sc = warp_sum(sc);
        if (fabs(sc) <= 1e-15 * sqrt(sa * sb) || sc == 0.0) continue;
        if (lane == 0) {
          s_rot = 1;
          atomicAdd(&s_nrot, 1u);
        }
        const double zeta = (sb - sa) / (2.0 * sc);
        const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
        for (int i = lane; i < p; i += 32) {
          const double x = wj[i], y = wk[i];
          wj[i] = cs * x - sn * y;
          wk[i] = sn * x + cs * y;
        }
        double* jj = J + (size_t)a * q;
        double* jk = J + (size_t)b * q;
        for (int i = lane; i < q; i += 32) {
          const double x = jj[i], y = jk[i];
          jj[i] = cs * x - sn * y;
          jk[i] = sn * x + cs * y;
        }
      }
      __syncthreads();
    }
    const int rot = s_rot;
    __syncthreads();
    if (!rot) break;
  }
  return (double)sweeps * (0.5 * q * (q - 1)) * 6.0 * p + (double)s_nrot * 6.0 * (p + q);
}

__global__ void __launch_bounds__(kTruncThreads) k_truncate(const TruncItem* __restrict__ items,
                                                            double eps, int* err) {
  const TruncItem it = items[blockIdx.x];
  __shared__ double red[32];
  __shared__ double s_sig[kMaxTruncCols];
  __shared__ int s_ord[kMaxTruncCols];
  const int r0 = *it.rank;
  const int add = it.P ? (it.addp ? *it.addp : it.addv) : 0;
  const int r = r0 + add;
  bool go;
  switch (it.cond) {
    case 1:
      go = r > 16;
      break;
    case 2:
      go = r > *it.compact + 16;
      break;
    case 3:
      go = r > 48;
      break;
    case 4:
      go = false;
      break;
    default:
      go = r > 0;
      break;
  }
  if (!go) {  // plain append of the new columns
    if (add > 0) {
      if (r > it.cap) {
        if (threadIdx.x == 0) atomicOr(err, 2);
        return;
      }
      for (size_t e = threadIdx.x; e < (size_t)it.m * add; e += blockDim.x) {
        const int i = (int)(e % it.m), k = (int)(e / it.m), pi = i - it.pro;
        it.U[(size_t)(r0 + k) * it.m + i] =
            (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)k * it.ldp + pi] : 0.0;
      }
      for (size_t e = threadIdx.x; e < (size_t)it.n * add; e += blockDim.x) {
        const int i = (int)(e % it.n), k = (int)(e / it.n), qi = i - it.qro;
        it.V[(size_t)(r0 + k) * it.n + i] =
            (qi >= 0 && qi < it.qr) ? it.Q[(size_t)k * it.ldq + qi] : 0.0;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *it.rank = r;
      if (it.cond == 0 && it.compact) *it.compact = r;
    }
    return;
  }
  if (r > it.rcap || r > kMaxTruncCols) {
    if (threadIdx.x == 0) atomicOr(err, 1);
    return;
  }
  const int m = it.m, n = it.n;
  double* WU = it.ws;
  double* WV = WU + (size_t)m * it.rcap;
  double* tu = WV + (size_t)n * it.rcap;
  double* tv = tu + it.rcap;
  double* C = tv + it.rcap;
  double* J = C + (size_t)it.rcap * min(min(m, n), it.rcap);
  for (size_t i = threadIdx.x; i < (size_t)m * r0; i += blockDim.x) WU[i] = it.U[i];
  for (size_t i = threadIdx.x; i < (size_t)n * r0; i += blockDim.x) WV[i] = it.V[i];
  for (size_t e = threadIdx.x; e < (size_t)m * add; e += blockDim.x) {
    const int i = (int)(e % m), k = (int)(e / m), pi = i - it.pro;
    WU[(size_t)(r0 + k) * m + i] = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)k * it.ldp + pi] : 0.0;
  }
  for (size_t e = threadIdx.x; e < (size_t)n * add; e += blockDim.x) {
    const int i = (int)(e % n), k = (int)(e / n), qi = i - it.qro;
    WV[(size_t)(r0 + k) * n + i] = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)k * it.ldq + qi] : 0.0;
  }
  __syncthreads();
  cta_householder(WU, m, r, tu, red);
  cta_householder(WV, n, r, tv, red);
  const int ku = min(m, r), kv = min(n, r);
  const bool swapped = ku < kv;
  const int p = swapped ? kv : ku, q = swapped ? ku : kv;
  // core(i,j) = sum_{l >= max(i,j)} Ru(i,l) Rv(j,l); stored as W (p x q)
  for (int idx = threadIdx.x; idx < ku * kv; idx += blockDim.x) {
    const int i = idx % ku, j = idx / ku;
    double s = 0.0;
    for (int l = max(i, j); l < r; ++l) s += WU[(size_t)l * m + i] * WV[(size_t)l * n + j];
    if (!swapped)
      C[(size_t)j * p + i] = s;
    else
      C[(size_t)i * p + j] = s;
  }
  __syncthreads();
  const double jac_flops = cta_jacobi(C, p, q, J);
  // singular values = column norms of W; order descending (ties by index)
  for (int c = threadIdx.x; c < q; c += blockDim.x) {
    const double* wc = C + (size_t)c * p;
    double s = 0.0;
    for (int i = 0; i < p; ++i) s += wc[i] * wc[i];
    s_sig[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < q; c += blockDim.x) {
    const double sc = s_sig[c];
    int rk = 0;
    for (int d = 0; d < q; ++d) rk += (s_sig[d] > sc) || (s_sig[d] == sc && d < c);
    s_ord[rk] = c;
  }
  __syncthreads();
  const double smax = q > 0 ? s_sig[s_ord[0]] : 0.0;
  __shared__ int s_keep;
  if (threadIdx.x == 0) {
    int keep = 0;
    while (keep < q && s_sig[s_ord[keep]] > eps * smax && s_sig[s_ord[keep]] > 0.0) ++keep;
    s_keep = keep;
  }
  __syncthreads();
  const int keep = s_keep;
  if (keep > it.cap) {
    if (threadIdx.x == 0) atomicOr(err, 4);
    return;
  }
  // E_u (m x keep) -> it.U, E_v (n x keep) -> it.V, then apply Q_u, Q_v.
  for (int idx = threadIdx.x; idx < m * keep; idx += blockDim.x) {
    const int i = idx % m, c = idx / m;
    const int src = s_ord[c];
    double v = 0.0;
    if (i < ku) v = swapped ? J[(size_t)src * q + i] * s_sig[src] : C[(size_t)src * p + i];
    it.U[idx] = v;
  }
  for (int idx = threadIdx.x; idx < n * keep; idx += blockDim.x) {
    const int i = idx % n, c = idx / n;
    const int src = s_ord[c];
    double v = 0.0;
    if (i < kv) v = swapped ? C[(size_t)src * p + i] / s_sig[src] : J[(size_t)src * q + i];
    it.V[idx] = v;
  }
  __syncthreads();
  cta_apply_q(WU, m, ku, tu, it.U, keep);
  cta_apply_q(WV, n, kv, tv, it.V, keep);
  if (threadIdx.x == 0) {
    *it.rank = keep;
    if (it.compact) *it.compact = keep;
    const double fl = qr_flops(m, r) + qr_flops(n, r) + (double)ku * kv * r + jac_flops +
                      4.0 * keep * ((double)m * ku + (double)n * kv);
    atomicAdd(&d_cnt_trunc, fl);
    atomicAdd(&d_cnt_titems, 1.0);
  }
}

void launch_truncate(const TruncItem* d_items, int count, double eps, int* d_err, cudaStream_t st) {
  if (count <= 0) return;
  k_truncate<<<count, kTruncThreads, 0, st>>>(d_items, eps, d_err);
  HMGP_LAUNCH_CHECK();
}

}  // namespace hmgp_gpu
