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
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "hmgp_internal.h"

namespace hmgp_gpu {

constexpr int kTruncThreads = 512;
constexpr int kMaxTruncCols = 1024;
constexpr int kChunk = 8;              // factor columns staged per pass when forming W
constexpr int kMaxSmemW = 16384;       // W = [U|aP][V|Q]^T in shared memory (128 KB)
constexpr int kMaxSmemMN = 1024;       // m + n bound of the staged column chunks (64 KB)

__device__ double d_cnt_trunc, d_cnt_titems;

// (stats mode) per-path histogram of recompressions by max(m, n) and column
// count r: item count and summed SM cycles.  path 0 small (W in smem), 1 large
// single CTA, 2 cluster.
constexpr int kHM = 10, kHR = 10;
__device__ unsigned long long d_hist_n[4][kHM][kHR], d_hist_cyc[4][kHM][kHR];
__device__ int d_hist_on;
__device__ __forceinline__ int hbucket(int v) {
  int b = 0;
  while (b < kHM - 1 && (16 << b) < v) ++b;
  return b;
}
// (stats mode) per-launch maxima: slowest item and slowest target sequence
constexpr int kLaunchSlots = 1 << 17;
__device__ int d_lidx;
__device__ unsigned long long d_lmax[kLaunchSlots], d_lseq[kLaunchSlots];
__device__ __forceinline__ void seq_done(long long ts) {
  if (!d_hist_on || threadIdx.x != 0) return;
  atomicMax(&d_lseq[d_lidx & (kLaunchSlots - 1)], (unsigned long long)(clock64() - ts));
}
void truncate_launch_slot(int idx, cudaStream_t st) {
  HMGP_CUDA(cudaMemcpyToSymbolAsync(d_lidx, &idx, 4, 0, cudaMemcpyHostToDevice, st));
}
void truncate_launch_read(std::vector<unsigned long long>& mx, std::vector<unsigned long long>& sq) {
  mx.resize(kLaunchSlots);
  sq.resize(kLaunchSlots);
  HMGP_CUDA(cudaMemcpyFromSymbol(mx.data(), d_lmax, kLaunchSlots * 8));
  HMGP_CUDA(cudaMemcpyFromSymbol(sq.data(), d_lseq, kLaunchSlots * 8));
}
__device__ __forceinline__ void hist_add(int path, int m, int n, int r, long long t0) {
  if (!d_hist_on || threadIdx.x != 0) return;
  atomicMax(&d_lmax[d_lidx & (kLaunchSlots - 1)], (unsigned long long)(clock64() - t0));
  const int bm = hbucket(max(m, n)), br = min(hbucket(r), kHR - 1);
  atomicAdd(&d_hist_n[path][bm][br], 1ull);
  atomicAdd(&d_hist_cyc[path][bm][br], (unsigned long long)(clock64() - t0));
}
// (stats mode) per-stage SM cycles of the single-CTA paths: [path][stage]
// stages: 0 stage-in / W formation, 1 Householder QR of the factors, 2 RRQR of
// the core, 3 Jacobi, 4 Q application / write-back; d_stage_sweeps counts sweeps
__device__ unsigned long long d_stage_cyc[3][5], d_stage_sweeps[3], d_stage_jac[3];
// (stats mode) global cluster path stages: stage-in, QR U, QR V, core SVD, write, apply U, apply V
__device__ unsigned long long d_clu_cyc[7];
__device__ unsigned long long d_qr_cyc[5];  // clu_qr phases (rank 0, thread 0): partials, barrier, gather+update, syncthreads, steps
__device__ __forceinline__ void stage_add(int path, int st, long long& t) {
  if (!d_hist_on || threadIdx.x != 0) return;
  const long long now = clock64();
  atomicAdd(&d_stage_cyc[path][st], (unsigned long long)(now - t));
  t = now;
}
void truncate_hist_enable(bool on) {
  const int v = on ? 1 : 0;
  HMGP_CUDA(cudaMemcpyToSymbol(d_hist_on, &v, 4));
}
void truncate_hist_print() {
  static unsigned long long hn[4][kHM][kHR], hc[4][kHM][kHR];
  HMGP_CUDA(cudaMemcpyFromSymbol(hn, d_hist_n, sizeof(hn)));
  HMGP_CUDA(cudaMemcpyFromSymbol(hc, d_hist_cyc, sizeof(hc)));
  static unsigned long long sc[3][5], sw[3], sj[3];
  HMGP_CUDA(cudaMemcpyFromSymbol(sc, d_stage_cyc, sizeof(sc)));
  HMGP_CUDA(cudaMemcpyFromSymbol(sw, d_stage_sweeps, sizeof(sw)));
  HMGP_CUDA(cudaMemcpyFromSymbol(sj, d_stage_jac, sizeof(sj)));
  for (int p = 0; p < 3; ++p)
    fprintf(stderr,
            "[hmgp]   trunc %s stages (s, SM clock): stage-in %.2f qr %.2f rrqr %.2f jacobi %.2f apply %.2f;"
            " jacobi calls %llu, sweeps/call %.2f\n",
            p == 2 ? "pair" : p ? "large" : "small", sc[p][0] / 1.9e9, sc[p][1] / 1.9e9, sc[p][2] / 1.9e9, sc[p][3] / 1.9e9,
            sc[p][4] / 1.9e9, sj[p], sj[p] ? (double)sw[p] / sj[p] : 0.0);
  {
    static unsigned long long cc[7];
    HMGP_CUDA(cudaMemcpyFromSymbol(cc, d_clu_cyc, sizeof(cc)));
    unsigned long long qc[5];
    HMGP_CUDA(cudaMemcpyFromSymbol(qc, d_qr_cyc, sizeof(qc)));
    if (qc[4])
      fprintf(stderr, "[hmgp]   cluster QR per column step (cycles, rank 0 thread 0): partials %.0f barrier %.0f "
              "gather+update %.0f syncthreads %.0f (%llu steps)\n", (double)qc[0] / qc[4], (double)qc[1] / qc[4],
              (double)qc[2] / qc[4], (double)qc[3] / qc[4], qc[4]);
    fprintf(stderr,
            "[hmgp]   trunc cluster(global) stages (s): stage-in %.3f qr %.3f core-form %.3f core-svd %.3f write %.3f "
            "applyU %.3f applyV %.3f\n",
            cc[0] / 1.9e9, cc[1] / 1.9e9, cc[2] / 1.9e9, cc[3] / 1.9e9, cc[4] / 1.9e9, cc[5] / 1.9e9,
            cc[6] / 1.9e9);
  }
  static const char* nm[4] = {"small", "large", "cluster", "pair"};
  for (int p = 0; p < 4; ++p)
    for (int a = 0; a < kHM; ++a)
      for (int b = 0; b < kHR; ++b)
        if (hn[p][a][b])
          fprintf(stderr, "[hmgp]   trunc %-7s max(m,n)<=%6d r<=%5d: %8llu items, %8.1f us/item (SM clock)\n",
                  nm[p], 16 << a, 16 << b, hn[p][a][b], hc[p][a][b] / (double)hn[p][a][b] / 1.9e3);
}

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
  const size_t mn = (size_t)min(m, n);
  const size_t kq = std::min(mn, (size_t)rcap), rc = (size_t)rcap;
  if ((size_t)m * n <= (size_t)kMaxSmemW && m + n <= kMaxSmemMN)  // small-block path only
    return 4 * (size_t)n + (size_t)n * kq + kq * kq;
  return (size_t)(m + n) * rc + 6 * rc + rc * rc + 2 * rc * kq + kq * kq;
}

void trunc_smem_dims(int m, int n, int* smem_w, int* smem_mn) {
  if ((size_t)m * n <= (size_t)kMaxSmemW && m + n <= kMaxSmemMN) {
    *smem_w = std::max(*smem_w, m * n);
    *smem_mn = std::max(*smem_mn, m + n);
  }
}

// Apply H = I - t v v^T (v = [1; col[k+1:m]]) to columns [j0, j1) of A (ld m):
// one warp per column group of 4, four independent dot products in flight per
// warp so the L1/L2 load latency of one column overlaps the others.
__device__ __forceinline__ void reflect_cols(double* A, int m, int k, const double* col, double t,
                                             int j0, int j1, int lane, int w, int nw) {
  for (int jb = j0 + 4 * w; jb < j1; jb += 4 * nw) {
    double* c[4];
    double s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = A + (size_t)min(jb + u, j1 - 1) * m;
      s[u] = 0.0;
    }
    for (int i = k + 1 + lane; i < m; i += 32) {
      const double v = col[i];
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += v * c[u][i];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = warp_sum(s[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = (s[u] + c[u][k]) * t;
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (jb + u >= j1) continue;
      for (int i = k + 1 + lane; i < m; i += 32) c[u][i] -= s[u] * col[i];
      if (lane == 0) c[u][k] -= s[u];
    }
  }
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
    if (t != 0.0) reflect_cols(A, m, k, col, t, k + 1, r, lane, w, nw);
    __syncthreads();
  }
}

// E <- Q E with Q = H_0 ... H_{kq-1} from cta_householder(QR); E m x c (ld m).
__device__ void cta_apply_q(const double* QR, int m, int kq, const double* tau, double* E, int c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = kq - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t != 0.0) reflect_cols(E, m, k, QR + (size_t)k * m, t, 0, c, lane, w, nw);
    __syncthreads();
  }
}

// One-sided Jacobi on W (p x q, ld p, p >= q); J (q x q) accumulates rotations.
// Returns the algorithmic flops (6p per pair inspected, 6(p+q) per rotation).
__device__ double cta_jacobi(double* W, int p, int q, double* J, int* sweeps_out = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int idx = threadIdx.x; idx < q * q; idx += blockDim.x) J[idx] = (idx % (q + 1) == 0) ? 1.0 : 0.0;
  __syncthreads();
  if (q < 2) {
    if (sweeps_out && threadIdx.x == 0) *sweeps_out = 0;
    return 0.0;
  }
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
  if (sweeps_out && threadIdx.x == 0) *sweeps_out = sweeps;
  return (double)sweeps * (0.5 * q * (q - 1)) * 6.0 * p + (double)s_nrot * 6.0 * (p + q);
}

struct RS {
  int kq, keep;
  double flops;
};

// Rank-revealing truncated SVD of W (p x q, ld p; destroyed): Businger-Golub
// column-pivoted Householder QR stopped once the Frobenius norm of the trailing
// block is <= 1e-3*eps*(largest column norm) <= 1e-3*eps*sigma_max — every
// singular value it drops is three decades below the reference's cut
// eps*sigma_max — then a one-sided Jacobi SVD of the small k' x q factor.
// Output: kq = k', reflectors in W / tau, G (q x kq, ld q) with columns Y*S
// (unpermuted rows), J (kq x kq) = X, s_sig / s_ord sorted descending and
// keep = #{sigma_i > eps*sigma_0, sigma_i > 0} (hblock.cpp:151-153).
__device__ RS cta_rrqr_svd(double* W, int p, int q, double eps, double* tau, int* piv, double* cn,
                           double* G, double* J, double* s_sig, int* s_ord, double* red,
                           int path = 0, long long* tclk = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double redv[32];
  __shared__ int redi[32];
  __shared__ double s_beta, s_t, s_inv, s_thresh;
  __shared__ int s_stop;
  double flops = 0.0;
  for (int j = w; j < q; j += nw) {
    const double* c = W + (size_t)j * p;
    double s = 0.0;
    for (int i = lane; i < p; i += 32) s += c[i] * c[i];
    s = warp_sum(s);
    if (lane == 0) {
      cn[j] = s;
      piv[j] = j;
    }
  }
  __syncthreads();
  flops += 2.0 * p * q;
  {
    double a = -1.0;
    int ia = -1;
    for (int j = threadIdx.x; j < q; j += blockDim.x)
      if (cn[j] > a) {
        a = cn[j];
        ia = j;
      }
    double best;
    block_argmax(a, ia, redv, redi, &best);
    if (threadIdx.x == 0) s_thresh = 1e-3 * eps * sqrt(fmax(best, 0.0));
    __syncthreads();
  }
  const int kmax = min(p, q);
  int k = 0;
  __shared__ double s_part[32];
  for (; k < kmax; ++k) {
    double part = 0.0, a = -1.0;
    int ia = -1;
    for (int j = k + threadIdx.x; j < q; j += blockDim.x) {
      part += cn[j];
      if (cn[j] > a) {
        a = cn[j];
        ia = j;
      }
    }
    // one fused reduction: trailing Frobenius norm^2 and the pivot column
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    double best;
    const int jm = block_argmax(a, ia, redv, redi, &best);  // contains the barrier
    if (threadIdx.x == 0) {
      double resid = 0.0;
      for (int q2 = 0; q2 < nw; ++q2) resid += s_part[q2];
      s_stop = !(sqrt(resid) > s_thresh) || jm < 0;
    }
    __syncthreads();
    if (s_stop) break;
    if (jm != k) {  // swap columns k <-> jm
      double* ck = W + (size_t)k * p;
      double* cm = W + (size_t)jm * p;
      for (int i = threadIdx.x; i < p; i += blockDim.x) {
        const double t = ck[i];
        ck[i] = cm[i];
        cm[i] = t;
      }
      if (threadIdx.x == 0) {
        const double t = cn[k];
        cn[k] = cn[jm];
        cn[jm] = t;
        const int pt = piv[k];
        piv[k] = piv[jm];
        piv[jm] = pt;
      }
      __syncthreads();
    }
    double* col = W + (size_t)k * p;
    double tp = 0.0;
    for (int i = k + 1 + threadIdx.x; i < p; i += blockDim.x) tp += col[i] * col[i];
    const double tail2 = block_sum(tp, red);
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
    for (int i = k + 1 + threadIdx.x; i < p; i += blockDim.x) col[i] = (t == 0.0) ? 0.0 : col[i] * inv;
    __syncthreads();
    if (threadIdx.x == 0) {
      col[k] = s_beta;
      tau[k] = t;
    }
    __syncthreads();
    // apply H_k and refresh the trailing norms, 4 columns per warp in flight
    for (int jb = k + 1 + 4 * w; jb < q; jb += 4 * nw) {
      double* c4[4];
      double s[4], s2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c4[u] = W + (size_t)min(jb + u, q - 1) * p;
        s[u] = 0.0;
        s2[u] = 0.0;
      }
      if (t != 0.0) {
        for (int i = k + 1 + lane; i < p; i += 32) {
          const double v = col[i];
#pragma unroll
          for (int u = 0; u < 4; ++u) s[u] += v * c4[u][i];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = (warp_sum(s[u]) + c4[u][k]) * t;
      }
      __syncwarp();
      for (int i = k + 1 + lane; i < p; i += 32) {
        const double v = col[i];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (jb + u >= q) continue;
          const double x = c4[u][i] - s[u] * v;
          c4[u][i] = x;
          s2[u] += x * x;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) s2[u] = warp_sum(s2[u]);
      if (lane == 0)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (jb + u < q) {
            c4[u][k] -= s[u];
            cn[jb + u] = s2[u];
          }
    }
    __syncthreads();
    flops += 6.0 * (p - k) * (q - k);
  }
  const int kq = k;
  if (tclk) stage_add(path, 2, *tclk);
  // G = (R P^T)^T : q x kq, row piv[j] holds R(:, j)
  for (int e = threadIdx.x; e < q * kq; e += blockDim.x) {
    const int j = e % q, i = e / q;
    G[(size_t)i * q + piv[j]] = (j >= i) ? W[(size_t)j * p + i] : 0.0;
  }
  __syncthreads();
  __shared__ int s_sweeps;
  flops += cta_jacobi(G, q, kq, J, &s_sweeps);
  if (tclk) {
    stage_add(path, 3, *tclk);
    if (d_hist_on && threadIdx.x == 0) {
      atomicAdd(&d_stage_sweeps[path], (unsigned long long)s_sweeps);
      atomicAdd(&d_stage_jac[path], 1ull);
    }
  }
  for (int c = threadIdx.x; c < kq; c += blockDim.x) {
    const double* gc = G + (size_t)c * q;
    double s = 0.0;
    for (int i = 0; i < q; ++i) s += gc[i] * gc[i];
    s_sig[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kq; c += blockDim.x) {
    const double sc = s_sig[c];
    int rk = 0;
    for (int d = 0; d < kq; ++d) rk += (s_sig[d] > sc) || (s_sig[d] == sc && d < c);
    s_ord[rk] = c;
  }
  __syncthreads();
  __shared__ int s_keep;
  if (threadIdx.x == 0) {
    const double smax = kq > 0 ? s_sig[s_ord[0]] : 0.0;
    int keep = 0;
    while (keep < kq && s_sig[s_ord[keep]] > eps * smax && s_sig[s_ord[keep]] > 0.0) ++keep;
    s_keep = keep;
  }
  __syncthreads();
  return RS{kq, s_keep, flops};
}

#include "trunc_lean.cuh"

__device__ void lr_update(const TruncItem& it, double eps, int* err, int smem_w, int smem_mn);

// Fused trsm_lower_t post-op (hfactor.cpp:198-202): V <- L^{-1} V, V /= d.
// One warp per column, lanes over rows; L read through L1/L2.
// n <= 32*NB: the column is held in registers (lane l owns rows l, l+32, ...),
// one shuffle broadcast per step, reciprocal diagonal precomputed, L columns
// read through L1 (every warp walks the same L).
template <int NB>
__device__ void lr_post_solve_reg(const TruncItem& it, double* s_inv) {
  const int cols = *it.rank, n = it.n, ld = it.post_ldl_ld;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* L = it.post_L;
  for (int j = threadIdx.x; j < 32 * NB; j += blockDim.x) s_inv[j] = j < n ? 1.0 / L[(size_t)j * ld + j] : 0.0;
  __syncthreads();
  for (int c = w; c < cols; c += nw) {
    double* x = it.V + (size_t)c * n;
    double xr[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) xr[k] = (k * 32 + lane < n) ? x[k * 32 + lane] : 0.0;
#pragma unroll
    for (int kb = 0; kb < NB; ++kb)
#pragma unroll 4
      for (int jj = 0; jj < 32; ++jj) {
        const int j = kb * 32 + jj;
        if (j >= n) break;
        const double* lc = L + (size_t)j * ld;
        double lv[NB];
#pragma unroll
        for (int k = kb; k < NB; ++k) lv[k] = (k * 32 + lane < n) ? lc[k * 32 + lane] : 0.0;
        if (lane == jj) xr[kb] *= s_inv[j];
        const double xj = __shfl_sync(0xffffffffu, xr[kb], jj);
        if (lane > jj) xr[kb] -= lv[kb] * xj;
#pragma unroll
        for (int k = kb + 1; k < NB; ++k) xr[k] -= lv[k] * xj;
      }
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k * 32 + lane < n) x[k * 32 + lane] = it.post_d ? xr[k] / it.post_d[k * 32 + lane] : xr[k];
  }
  __syncthreads();
}

__device__ void lr_post_solve(const TruncItem& it) {
  __shared__ double s_inv[128];
  if (it.n <= 32) return lr_post_solve_reg<1>(it, s_inv);
  if (it.n <= 64) return lr_post_solve_reg<2>(it, s_inv);
  if (it.n <= 96) return lr_post_solve_reg<3>(it, s_inv);
  if (it.n <= 128) return lr_post_solve_reg<4>(it, s_inv);
  const int cols = *it.rank, n = it.n, ld = it.post_ldl_ld;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* L = it.post_L;
  for (int c = w; c < cols; c += nw) {
    double* x = it.V + (size_t)c * n;
    for (int j = 0; j < n; ++j) {
      const double xj = x[j] / L[(size_t)j * ld + j];
      __syncwarp();
      if (lane == 0) x[j] = xj;
      const double* lc = L + (size_t)j * ld;
      for (int i = j + 1 + lane; i < n; i += 32) x[i] -= lc[i] * xj;
      __syncwarp();
    }
    if (it.post_d)
      for (int i = lane; i < n; i += 32) x[i] /= it.post_d[i];
  }
}

__global__ void __launch_bounds__(kTruncThreads) k_truncate(const TruncItem* __restrict__ items,
                                                            double eps, int* err, int smem_w,
                                                            int smem_mn) {
  const long long ts = clock64();
  const TruncItem& it = items[blockIdx.x];
  lr_update(it, eps, err, smem_w, smem_mn);
  if (it.post_L) {
    __syncthreads();
    lr_post_solve(it);
  }
  seq_done(ts);
}

// One CTA per target: its updates items[off[b] .. off[b+1]) run in order (the
// reference's per-target sequence and watermark decisions), all targets at once.
__global__ void __launch_bounds__(kTruncThreads) k_truncate_seq(const TruncItem* __restrict__ items,
                                                                const int* __restrict__ off,
                                                                double eps, int* err, int smem_w,
                                                                int smem_mn) {
  const long long ts = clock64();
  for (int i = off[blockIdx.x]; i < off[blockIdx.x + 1]; ++i) {
    lr_update(items[i], eps, err, smem_w, smem_mn);
    __syncthreads();
  }
  seq_done(ts);
}

__device__ void lr_update(const TruncItem& it, double eps, int* err, int smem_w, int smem_mn) {
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
  const long long t0 = clock64();
  extern __shared__ double dsm[];
  if ((size_t)m * n <= (size_t)smem_w && m + n <= smem_mn) {
    // ---- small block: W = [U | aP][V | Q]^T explicitly, rank-revealing SVD of W.
    // W has exactly the singular values of the reference's core R_u R_v^T.
    double* W = dsm;
    double* sU = dsm + (size_t)m * n;
    double* sV = sU + (size_t)m * kChunk;
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) W[e] = 0.0;
    for (int l0 = 0; l0 < r; l0 += kChunk) {
      const int lc = min(kChunk, r - l0);
      __syncthreads();
      for (int e = threadIdx.x; e < m * lc; e += blockDim.x) {
        const int i = e % m, l = l0 + e / m;
        double v;
        if (l < r0) {
          v = it.U[(size_t)l * m + i];
        } else {
          const int pi = i - it.pro;
          v = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)(l - r0) * it.ldp + pi] : 0.0;
        }
        sU[(size_t)(e / m) * m + i] = v;
      }
      for (int e = threadIdx.x; e < n * lc; e += blockDim.x) {
        const int j = e % n, l = l0 + e / n;
        double v;
        if (l < r0) {
          v = it.V[(size_t)l * n + j];
        } else {
          const int qi = j - it.qro;
          v = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)(l - r0) * it.ldq + qi] : 0.0;
        }
        sV[(size_t)(e / n) * n + j] = v;
      }
      __syncthreads();
      // W += sU sV^T in 4 x 4 register tiles (8 shared loads per 16 FMAs)
      const int tmi = (m + 3) >> 2, tiles = tmi * ((n + 3) >> 2);
      for (int tt = threadIdx.x; tt < tiles; tt += blockDim.x) {
        const int i0 = (tt % tmi) << 2, j0 = (tt / tmi) << 2;
        double acc[4][4];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int a = 0; a < 4; ++a) acc[b][a] = 0.0;
        for (int l = 0; l < lc; ++l) {
          double u[4], v[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            u[a] = (i0 + a < m) ? sU[(size_t)l * m + i0 + a] : 0.0;
            v[a] = (j0 + a < n) ? sV[(size_t)l * n + j0 + a] : 0.0;
          }
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[b][a] += u[a] * v[b];
        }
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int a = 0; a < 4; ++a)
            if (i0 + a < m && j0 + b < n) W[(size_t)(j0 + b) * m + i0 + a] += acc[b][a];
      }
    }
    __syncthreads();
    double* ws = it.ws;
    double* tau = ws;
    double* cn = tau + n;                                 // 2n (double-buffered in rrqr2)
    int* piv = reinterpret_cast<int*>(cn + 2 * n);        // n ints
    int* stepof = piv + n;                                // n ints
    double* G = cn + 3 * n;
    const int kqmax = min(min(m, n), it.rcap);  // rank(W) <= r <= rcap
    double* J = G + (size_t)n * kqmax;
    long long tc = t0;
    stage_add(0, 0, tc);
    const bool lean = n <= 128 && blockDim.x == 512;
    const RS rs = lean ? cta_rrqr_svd2(W, m, n, eps, tau, piv, cn, stepof, G, J, s_sig, s_ord, 0, &tc)
                       : cta_rrqr_svd(W, m, n, eps, tau, piv, cn, G, J, s_sig, s_ord, red, 0, &tc);
    if (rs.keep > it.cap) {
      if (threadIdx.x == 0) atomicOr(err, 4);
      return;
    }
    const int keep = rs.keep, kq = rs.kq;
    for (int idx = threadIdx.x; idx < m * keep; idx += blockDim.x) {
      const int i = idx % m, c = idx / m, src = s_ord[c];
      it.U[idx] = i < kq ? J[(size_t)src * kq + i] * s_sig[src] : 0.0;
    }
    for (int idx = threadIdx.x; idx < n * keep; idx += blockDim.x) {
      const int i = idx % n, c = idx / n, src = s_ord[c];
      it.V[idx] = G[(size_t)src * n + i] / s_sig[src];
    }
    __syncthreads();
    if (lean)
      cta_apply_q_map(W, m, m, kq, tau, piv, it.U, keep);
    else
      cta_apply_q(W, m, kq, tau, it.U, keep);
    stage_add(0, 4, tc);
    if (threadIdx.x == 0) {
      *it.rank = keep;
      if (it.compact) *it.compact = keep;
      atomicAdd(&d_cnt_trunc, 2.0 * m * n * r + rs.flops + 4.0 * keep * (double)m * kq);
      atomicAdd(&d_cnt_titems, 1.0);
    }
    hist_add(0, m, n, r, t0);
    return;
  }
  // ---- large block: Householder QR of both stacked factors, core R_u R_v^T,
  // then the same rank-revealing SVD on the core (hblock.cpp:144-161).
  double* WU = it.ws;
  double* WV = WU + (size_t)m * it.rcap;
  double* tu = WV + (size_t)n * it.rcap;
  double* tv = tu + it.rcap;
  double* C = tv + it.rcap;
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
  long long tc = t0;
  stage_add(1, 0, tc);
  {
    __shared__ double s_tail2[2];
    smem_qr(WU, m, m, r, tu, s_tail2);  // one barrier per column (generic memory)
    smem_qr(WV, n, n, r, tv, s_tail2);
  }
  stage_add(1, 1, tc);
  const int ku = min(m, r), kv = min(n, r);
  // core(i,j) = sum_{l >= max(i,j)} Ru(i,l) Rv(j,l)  (ku x kv, ld ku)
  for (int idx = threadIdx.x; idx < ku * kv; idx += blockDim.x) {
    const int i = idx % ku, j = idx / ku;
    double s = 0.0;
    for (int l = max(i, j); l < r; ++l) s += WU[(size_t)l * m + i] * WV[(size_t)l * n + j];
    C[(size_t)j * ku + i] = s;
  }
  __syncthreads();
  const int kqmax = min(ku, kv);
  double* tau = C + (size_t)ku * kv;
  double* cn = tau + kv;                            // 2 kv
  int* piv = reinterpret_cast<int*>(cn + 2 * kv);   // kv ints
  int* stepof = piv + kv;                           // kv ints
  double* G = cn + 3 * kv;
  double* J = G + (size_t)kv * kqmax;
  double* Uc = J + (size_t)kqmax * kqmax;
  const bool lean = kv <= 128 && blockDim.x == 512;
  const RS rs = lean ? cta_rrqr_svd2(C, ku, kv, eps, tau, piv, cn, stepof, G, J, s_sig, s_ord, 1, &tc)
                     : cta_rrqr_svd(C, ku, kv, eps, tau, piv, cn, G, J, s_sig, s_ord, red, 1, &tc);
  if (rs.keep > it.cap) {
    if (threadIdx.x == 0) atomicOr(err, 4);
    return;
  }
  const int keep = rs.keep, kq = rs.kq;
  // U_core = Q_core [J S; 0] (ku x keep)
  for (int idx = threadIdx.x; idx < ku * keep; idx += blockDim.x) {
    const int i = idx % ku, c = idx / ku, src = s_ord[c];
    Uc[idx] = i < kq ? J[(size_t)src * kq + i] * s_sig[src] : 0.0;
  }
  __syncthreads();
  if (lean)
    cta_apply_q_map(C, ku, ku, kq, tau, piv, Uc, keep);
  else
    cta_apply_q(C, ku, kq, tau, Uc, keep);
  // E_u = [U_core; 0] -> it.U, E_v = [Y; 0] -> it.V, then apply Q_u, Q_v.
  for (int idx = threadIdx.x; idx < m * keep; idx += blockDim.x) {
    const int i = idx % m, c = idx / m;
    it.U[idx] = i < ku ? Uc[(size_t)c * ku + i] : 0.0;
  }
  for (int idx = threadIdx.x; idx < n * keep; idx += blockDim.x) {
    const int i = idx % n, c = idx / n, src = s_ord[c];
    it.V[idx] = i < kv ? G[(size_t)src * kv + i] / s_sig[src] : 0.0;
  }
  __syncthreads();
  cta_apply_q(WU, m, ku, tu, it.U, keep);
  cta_apply_q(WV, n, kv, tv, it.V, keep);
  stage_add(1, 4, tc);
  if (threadIdx.x == 0) {
    *it.rank = keep;
    if (it.compact) *it.compact = keep;
    const double fl = qr_flops(m, r) + qr_flops(n, r) + (double)ku * kv * r + rs.flops +
                      4.0 * keep * ((double)m * ku + (double)n * kv + (double)ku * kq);
    atomicAdd(&d_cnt_trunc, fl);
    atomicAdd(&d_cnt_titems, 1.0);
  }
  hist_add(1, m, n, r, t0);
}

// ===================================================================== //
// Large blocks: one thread-block CLUSTER of kClu CTAs per target.  CTA c owns
// the row slice [c*ms, (c+1)*ms) of the stacked factors; Householder QR and
// the Q application run column by column with the per-column reductions
// exchanged through distributed shared memory (2 cluster barriers per column,
// double-buffered partials).  The small core R_u R_v^T goes through the same
// rank-revealing SVD as the single-CTA path, on CTA 0.
// ===================================================================== //
constexpr int kClu = 8;
constexpr int kCluMaxR = 1024;

namespace cg = cooperative_groups;

constexpr int kGather = 64;  // remote partials fetched per chunk (per rank)

struct CluShared {
  double part[2][kCluMaxR + 2];  // per column step: [0] tail norm^2, [1] row-k value, [2..] dots
  double gb[kClu][kGather];      // local copy of the ranks' partials being summed
};

// Distributed Householder QR of A (m x r, ld m) over the row slices of a group
// of gs ranks starting at rank g0 (the U and V factors run at once on the two
// halves of the cluster).  Every rank executes the same barrier sequence: kit
// column steps (the larger of the two groups' min(m, r)), two cluster barriers
// each, whether or not its group has work at that step.
__device__ void clu_qr_2b(cg::cluster_group& cl, CluShared& sh, double* A, int m, int r, double* tau, int g0,
                          int gs, int kit) {
  double (*gb)[kGather] = sh.gb;
  const int rank = cl.block_rank();
  const int ms = (m + gs - 1) / gs, lo = (rank - g0) * ms, hi = min(m, lo + ms);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double red[32];
  const int kmax = min(m, r);
  for (int k = 0; k < kit; ++k) {
    const bool act = k < kmax;
    double* P = sh.part[k & 1];
    double* col = A + (size_t)k * m;
    // (a) partial tail norm^2 over own rows > k; owner of row k publishes A(k,k)
    double part = 0.0;
    if (act)
      for (int i = max(lo, k + 1) + threadIdx.x; i < hi; i += blockDim.x) part += col[i] * col[i];
    part = block_sum(part, red);
    if (threadIdx.x == 0) {
      P[0] = part;
      P[1] = (act && k >= lo && k < hi) ? col[k] : 0.0;
    }
    cl.sync();
    // (b) every rank of the group forms the same reflector from the group sums
    // (remote values fetched once, in parallel, summed in rank order)
    if (threadIdx.x < 2 * gs) gb[0][threadIdx.x] = cl.map_shared_rank(P, g0 + threadIdx.x % gs)[threadIdx.x / gs];
    __syncthreads();
    double tail2 = 0.0, c0 = 0.0;
    for (int c = 0; c < gs; ++c) {
      tail2 += gb[0][c];
      c0 += gb[0][gs + c];
    }
    double t = 0.0, beta = c0, inv = 0.0;
    if (tail2 > 2.2250738585072014e-308) {
      beta = sqrt(c0 * c0 + tail2);
      if (c0 >= 0.0) beta = -beta;
      inv = 1.0 / (c0 - beta);
      t = (beta - c0) / beta;
    }
    if (act)
      for (int i = max(lo, k + 1) + threadIdx.x; i < hi; i += blockDim.x) col[i] = (t == 0.0) ? 0.0 : col[i] * inv;
    __syncthreads();
    if (act && threadIdx.x == 0) {
      if (k >= lo && k < hi) col[k] = beta;
      if (rank == g0) tau[k] = t;
    }
    const bool up = act && t != 0.0;
    // (c) partial dots v^T A(:, j) over own rows for the trailing columns
    if (up)
      for (int j = k + 1 + w; j < r; j += nw) {
        const double* cj = A + (size_t)j * m;
        double s = 0.0;
        for (int i = max(lo, k + 1) + lane; i < hi; i += 32) s += col[i] * cj[i];
        s = warp_sum(s);
        if (lane == 0) P[2 + j] = s + ((k >= lo && k < hi) ? cj[k] : 0.0);
      }
    cl.sync();
    // (d) full dots from the group (remote partials gathered in chunks of
    // kGather columns, summed in rank order), update own rows
    if (up)
      for (int jc = k + 1; jc < r; jc += kGather) {
        const int nj = min(kGather, r - jc);
        if (threadIdx.x < gs * kGather) {
          const int cc = threadIdx.x / kGather, jj = threadIdx.x % kGather;
          if (jj < nj) gb[cc][jj] = cl.map_shared_rank(P, g0 + cc)[2 + jc + jj];
        }
        __syncthreads();
        for (int j = jc + w; j < jc + nj; j += nw) {
          double s = 0.0;
          for (int c = 0; c < gs; ++c) s += gb[c][j - jc];
          s *= t;
          double* cj = A + (size_t)j * m;
          for (int i = max(lo, k + 1) + lane; i < hi; i += 32) cj[i] -= s * col[i];
          if (lane == 0 && k >= lo && k < hi) cj[k] -= s;
        }
        __syncthreads();
      }
  }
  cl.sync();
}

// One cluster barrier per column (r <= kCluMaxR / 2): at step k every rank
// publishes, for its own rows, the partial tail norm^2 of the UNNORMALISED
// column x = A(:, k) and the partial dots x_tail . A(:, j) for j > k; the owner
// of row k also publishes the heads A(k, k..r-1).  After the barrier every warp
// forms the reflector scalars (t, beta, inv) from the group sums itself and the
// full dots as s_j = t (A(k, j) + inv D_j) -- the same reflector as the
// two-barrier variant, v = [1; inv x_tail] -- and updates its columns' own
// rows.  Column k is normalised one step late (nobody reads it then), so the
// only intra-CTA barrier is the one that makes step k's updates visible to
// step k+1's partials.  Partials are double-buffered by step parity: a rank
// overwrites buffer k&1 only after passing step k+1's barrier, i.e. after every
// rank has finished reading it at step k.
// lda: column stride of A.  A may be a shared-memory row slice addressed with
// global row indices (A = slice - lo, lda = slice height): only own rows are
// touched.
// kQrRows: rows per lane held in registers (the slice height / 32, rounded up
// to 2, 4 or 8; taller slices fall back to row loops).
template <int kQrRows>
__device__ void clu_qr_t(cg::cluster_group& cl, CluShared& sh, double* A, int m, int r, double* tau, int g0,
                         int gs, int kit, int lda) {
  const int rank = cl.block_rank();
  const int ms = (m + gs - 1) / gs, lo = (rank - g0) * ms, hi = min(m, lo + ms);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kmax = min(m, r);
  double pt = 0.0, pinv = 0.0, pbeta = 0.0;  // previous step's scalars (lagged normalisation)
  const bool prof = d_hist_on && rank == 0 && threadIdx.x == 0;
  long long tq = prof ? clock64() : 0;
  auto qmark = [&](int i) {
    if (!prof) return;
    const long long now = clock64();
    atomicAdd(&d_qr_cyc[i], (unsigned long long)(now - tq));
    tq = now;
  };
  for (int k = 0; k < kit; ++k) {
    const bool act = k < kmax;
    double* P = sh.part[k & 1];
    // lagged normalisation of column k-1 (own rows), by the last warp
    if (k > 0 && k - 1 < kmax && w == nw - 1) {
      double* xp = A + (size_t)(k - 1) * lda;
      for (int i = max(lo, k) + lane; i < hi; i += 32) xp[i] = (pt == 0.0) ? 0.0 : xp[i] * pinv;
      if (lane == 0 && k - 1 >= lo && k - 1 < hi) xp[k - 1] = pbeta;
    }
    const double* x = A + (size_t)k * lda;
    const bool own_k = k >= lo && k < hi;
    // this lane's rows of the step (i0 + 32 t, t < nrow); with at most kQrRows
    // per lane (slices <= 256 rows) x's tail stays in registers for the step and
    // each four-column group issues all its loads before any arithmetic / store
    // (one memory round trip per group instead of one per row)
    const int i0 = max(lo, k + 1) + lane;
    const int nrow = i0 < hi ? (hi - i0 + 31) / 32 : 0;
    const bool regs = (hi - lo + 31) / 32 <= kQrRows;
    double xv[kQrRows];
#pragma unroll
    for (int t = 0; t < kQrRows; ++t) xv[t] = (regs && act && t < nrow) ? x[i0 + 32 * t] : 0.0;
    if (act) {
      // virtual column q = 0: norm of x's tail; q >= 1: dot with column k + q.
      // Four columns per warp pass: their loads and shuffle reductions overlap.
      for (int q0 = w; q0 < r - k; q0 += 4 * nw) {
        const double* c[4];
        bool on[4];
        double sd[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + u * nw;
          on[u] = q < r - k;
          c[u] = (on[u] && q > 0) ? A + (size_t)(k + q) * lda : x;
          sd[u] = 0.0;
        }
        if (regs) {
          double cv[4][kQrRows];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int t = 0; t < kQrRows; ++t) cv[u][t] = t < nrow ? c[u][i0 + 32 * t] : 0.0;
#pragma unroll
          for (int t = 0; t < kQrRows; ++t)
#pragma unroll
            for (int u = 0; u < 4; ++u) sd[u] += xv[t] * cv[u][t];
        } else {
          for (int i = i0; i < hi; i += 32) {
            const double xi = x[i];
#pragma unroll
            for (int u = 0; u < 4; ++u) sd[u] += xi * c[u][i];
          }
        }
        warp_sum_n<4>(sd);
        if (lane == 0)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = q0 + u * nw;
            if (!on[u]) continue;
            if (q == 0) {
              P[0] = sd[u];
              P[1] = own_k ? x[k] : 0.0;
            } else {
              P[2 + k + q] = sd[u];                   // dots at P[2 + j] (j = k + q)
              if (own_k) P[2 + r + k + q] = c[u][k];  // heads at P[2 + r + j]
            }
          }
      }
    }
    qmark(0);
    cl.sync();
    qmark(1);
    if (act) {
      // reflector scalars from the group sums (every warp, identical arithmetic)
      const int owner = g0 + min(k / ms, gs - 1);
      double part = 0.0;
      if (lane < gs) part = cl.map_shared_rank(P, g0 + lane)[0];
      else if (lane == gs) part = cl.map_shared_rank(P, owner)[1];
      double tail2 = 0.0;
      for (int c = 0; c < gs; ++c) tail2 += __shfl_sync(0xffffffffu, part, c);
      const double c0 = __shfl_sync(0xffffffffu, part, gs);
      double t = 0.0, beta = c0, inv = 0.0;
      if (tail2 > 2.2250738585072014e-308) {
        beta = sqrt(c0 * c0 + tail2);
        if (c0 >= 0.0) beta = -beta;
        inv = 1.0 / (c0 - beta);
        t = (beta - c0) / beta;
      }
      if (rank == g0 && threadIdx.x == 0) tau[k] = t;
      if (t != 0.0) {
        // lanes < gs read rank lane's dot partials, lane gs the owner's heads;
        // four columns' remote loads are in flight at once
        const double* Prem = lane < gs ? cl.map_shared_rank(P, g0 + lane) : cl.map_shared_rank(P, owner);
        const int off = lane < gs ? 2 : 2 + r;
        for (int j0 = k + 1 + w; j0 < r; j0 += 4 * nw) {
          double dp[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * nw;
            dp[u] = (j < r && lane <= gs) ? Prem[off + j] : 0.0;
          }
          double sj[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            double D = 0.0;
            for (int c = 0; c < gs; ++c) D += __shfl_sync(0xffffffffu, dp[u], c);
            const double head = __shfl_sync(0xffffffffu, dp[u], gs);
            sj[u] = t * (head + inv * D);
          }
          if (regs) {
            double* cjp[4];
            double cv[4][kQrRows];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              cjp[u] = A + (size_t)min(j0 + u * nw, r - 1) * lda;
#pragma unroll
              for (int t2 = 0; t2 < kQrRows; ++t2)
                cv[u][t2] = (j0 + u * nw < r && t2 < nrow) ? cjp[u][i0 + 32 * t2] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (j0 + u * nw >= r) continue;
#pragma unroll
              for (int t2 = 0; t2 < kQrRows; ++t2)
                if (t2 < nrow) cjp[u][i0 + 32 * t2] = cv[u][t2] - sj[u] * (inv * xv[t2]);
              if (lane == 0 && own_k) cjp[u][k] -= sj[u];
            }
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = j0 + u * nw;
              if (j >= r) continue;
              double* cj = A + (size_t)j * lda;
              for (int i = i0; i < hi; i += 32) cj[i] -= sj[u] * (inv * x[i]);
              if (lane == 0 && own_k) cj[k] -= sj[u];
            }
          }
        }
      }
      pt = t;
      pinv = inv;
      pbeta = beta;
    }
    qmark(2);
    __syncthreads();
    qmark(3);
    if (prof) atomicAdd(&d_qr_cyc[4], 1ull);
  }
  // normalise the last factored column
  if (kit > 0 && kit - 1 < kmax && w == nw - 1) {
    double* xp = A + (size_t)(kit - 1) * lda;
    for (int i = max(lo, kit) + lane; i < hi; i += 32) xp[i] = (pt == 0.0) ? 0.0 : xp[i] * pinv;
    if (lane == 0 && kit - 1 >= lo && kit - 1 < hi) xp[kit - 1] = pbeta;
  }
  cl.sync();
}

// E <- Q E over a group's row slices (Q from clu_qr with the same group), E m x c
// (ld m); kit reflector steps for every rank (uniform barrier sequence).
template <int kQrRows>
__device__ void clu_apply_q_t(cg::cluster_group& cl, CluShared& sh, const double* A, int m, int kq,
                              const double* tau, double* E, int c, int g0, int gs, int kit, int lda, int lde) {
  const int rank = cl.block_rank();
  const int ms = (m + gs - 1) / gs, lo = (rank - g0) * ms, hi = min(m, lo + ms);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = kit - 1; k >= 0; --k) {
    const double t = k < kq ? tau[k] : 0.0;
    const bool up = t != 0.0;
    const bool own_k = k >= lo && k < hi;
    double* P = sh.part[k & 1];
    const double* v = A + (size_t)k * lda;
    // register-held rows as in clu_qr: v's tail once per step, all loads of a
    // four-column group issued before its arithmetic / stores
    const int i0 = max(lo, k + 1) + lane;
    const int nrow = i0 < hi ? (hi - i0 + 31) / 32 : 0;
    const bool regs = (hi - lo + 31) / 32 <= kQrRows;
    double vv[kQrRows];
#pragma unroll
    for (int q = 0; q < kQrRows; ++q) vv[q] = (regs && up && q < nrow) ? v[i0 + 32 * q] : 0.0;
    // partial dots v . E(:, j) over own rows (+ the unit head on the owner);
    // column j is handled by the same warp in both phases, so E needs no
    // intra-CTA barrier, only the cluster barrier for the partials
    if (up)
      for (int j0 = w; j0 < c; j0 += 4 * nw) {
        double sd[4];
        const double* e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = min(j0 + u * nw, c - 1);
          e[u] = E + (size_t)j * lde;
          sd[u] = 0.0;
        }
        if (regs) {
          double ev[4][kQrRows];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < kQrRows; ++q) ev[u][q] = q < nrow ? e[u][i0 + 32 * q] : 0.0;
#pragma unroll
          for (int q = 0; q < kQrRows; ++q)
#pragma unroll
            for (int u = 0; u < 4; ++u) sd[u] += vv[q] * ev[u][q];
        } else {
          for (int i = i0; i < hi; i += 32) {
            const double vi = v[i];
#pragma unroll
            for (int u = 0; u < 4; ++u) sd[u] += vi * e[u][i];
          }
        }
        warp_sum_n<4>(sd);
        if (lane == 0)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u * nw < c) P[2 + j0 + u * nw] = sd[u] + (own_k ? e[u][k] : 0.0);
      }
    cl.sync();
    if (up) {
      const double* Prem = cl.map_shared_rank(P, g0 + min(lane, gs - 1));
      for (int j0 = w; j0 < c; j0 += 4 * nw) {
        double dp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * nw;
          dp[u] = (j < c && lane < gs) ? Prem[2 + j] : 0.0;
        }
        double sj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double su = 0.0;
          for (int q = 0; q < gs; ++q) su += __shfl_sync(0xffffffffu, dp[u], q);  // rank order
          sj[u] = su * t;
        }
        if (regs) {
          double* ep[4];
          double ev[4][kQrRows];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ep[u] = E + (size_t)min(j0 + u * nw, c - 1) * lde;
#pragma unroll
            for (int q = 0; q < kQrRows; ++q) ev[u][q] = (j0 + u * nw < c && q < nrow) ? ep[u][i0 + 32 * q] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (j0 + u * nw >= c) continue;
#pragma unroll
            for (int q = 0; q < kQrRows; ++q)
              if (q < nrow) ep[u][i0 + 32 * q] = ev[u][q] - sj[u] * vv[q];
            if (lane == 0 && own_k) ep[u][k] -= sj[u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * nw;
            if (j >= c) continue;
            double* e = E + (size_t)j * lde;
            for (int i = i0; i < hi; i += 32) e[i] -= sj[u] * v[i];
            if (lane == 0 && own_k) e[k] -= sj[u];
          }
        }
      }
    }
    // the next step overwrites the other parity buffer only after every rank
    // passed this step's barrier, so one barrier per step suffices here
  }
  cl.sync();
}

__device__ void clu_qr(cg::cluster_group& cl, CluShared& sh, double* A, int m, int r, double* tau, int g0,
                       int gs, int kit, int lda) {
  if (2 * r > kCluMaxR) {  // (only reached with lda == m: see lr_update_cluster)
    clu_qr_2b(cl, sh, A, m, r, tau, g0, gs, kit);
    return;
  }
  const int rpl = ((m + gs - 1) / gs + 31) / 32;
  if (rpl <= 2)
    clu_qr_t<2>(cl, sh, A, m, r, tau, g0, gs, kit, lda);
  else if (rpl <= 4)
    clu_qr_t<4>(cl, sh, A, m, r, tau, g0, gs, kit, lda);
  else
    clu_qr_t<8>(cl, sh, A, m, r, tau, g0, gs, kit, lda);
}

__device__ void clu_apply_q(cg::cluster_group& cl, CluShared& sh, const double* A, int m, int kq,
                            const double* tau, double* E, int c, int g0, int gs, int kit, int lda, int lde) {
  const int rpl = ((m + gs - 1) / gs + 31) / 32;
  if (rpl <= 2)
    clu_apply_q_t<2>(cl, sh, A, m, kq, tau, E, c, g0, gs, kit, lda, lde);
  else if (rpl <= 4)
    clu_apply_q_t<4>(cl, sh, A, m, kq, tau, E, c, g0, gs, kit, lda, lde);
  else
    clu_apply_q_t<8>(cl, sh, A, m, kq, tau, E, c, g0, gs, kit, lda, lde);
}

__device__ void lr_update_cluster(cg::cluster_group& cl, CluShared& sh, const TruncItem& it,
                                  double eps, int* err, int r0) {
  const int rank = cl.block_rank();
  __shared__ double red[32];
  __shared__ double s_sig[kMaxTruncCols];
  __shared__ int s_ord[kMaxTruncCols];
  __shared__ int s_kq;
  const int add = it.P ? (it.addp ? *it.addp : it.addv) : 0;
  const int r = r0 + add;
  bool go;
  switch (it.cond) {
    case 1: go = r > 16; break;
    case 2: go = r > *it.compact + 16; break;
    case 3: go = r > 48; break;
    case 4: go = false; break;
    default: go = r > 0; break;
  }
  const int m = it.m, n = it.n;
  const int msu = (m + kClu - 1) / kClu, mlo = rank * msu, mhi = min(m, mlo + msu);
  const int msv = (n + kClu - 1) / kClu, nlo = rank * msv, nhi = min(n, nlo + msv);
  if (!go) {
    if (add > 0 && r > it.cap) {
      if (rank == 0 && threadIdx.x == 0) atomicOr(err, 2);
      cl.sync();
      return;
    }
    for (int k = 0; k < add; ++k) {
      for (int i = mlo + threadIdx.x; i < mhi; i += blockDim.x) {
        const int pi = i - it.pro;
        it.U[(size_t)(r0 + k) * m + i] = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)k * it.ldp + pi] : 0.0;
      }
      for (int i = nlo + threadIdx.x; i < nhi; i += blockDim.x) {
        const int qi = i - it.qro;
        it.V[(size_t)(r0 + k) * n + i] = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)k * it.ldq + qi] : 0.0;
      }
    }
    cl.sync();
    if (rank == 0 && threadIdx.x == 0) {
      *it.rank = r;
      if (it.cond == 0 && it.compact) *it.compact = r;
    }
    cl.sync();
    return;
  }
  if (r > it.rcap || r > kCluMaxR) {
    if (rank == 0 && threadIdx.x == 0) atomicOr(err, 1);
    cl.sync();
    return;
  }
  const long long t0 = clock64();
  long long tcl = t0;
  auto cstage = [&](int i) {
    if (!d_hist_on || rank != 0 || threadIdx.x != 0) return;
    const long long now = clock64();
    atomicAdd(&d_clu_cyc[i], (unsigned long long)(now - tcl));
    tcl = now;
  };
  double* WU = it.ws;
  double* WV = WU + (size_t)m * it.rcap;
  double* tu = WV + (size_t)n * it.rcap;
  double* tv = tu + it.rcap;
  double* C = tv + it.rcap;
  const int ku = min(m, r), kv = min(n, r);
  // stage [U | aP] and [V | Q] (own row slices)
  for (int l = 0; l < r; ++l) {
    for (int i = mlo + threadIdx.x; i < mhi; i += blockDim.x) {
      double v;
      if (l < r0) {
        v = it.U[(size_t)l * m + i];
      } else {
        const int pi = i - it.pro;
        v = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)(l - r0) * it.ldp + pi] : 0.0;
      }
      WU[(size_t)l * m + i] = v;
    }
    for (int i = nlo + threadIdx.x; i < nhi; i += blockDim.x) {
      double v;
      if (l < r0) {
        v = it.V[(size_t)l * n + i];
      } else {
        const int qi = i - it.qro;
        v = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)(l - r0) * it.ldq + qi] : 0.0;
      }
      WV[(size_t)l * n + i] = v;
    }
  }
  cl.sync();
  cstage(0);
  {  // U on ranks 0-3, V on ranks 4-7, at once
    const int kit = max(min(m, r), min(n, r));
    if (rank < kClu / 2) {
      clu_qr(cl, sh, WU, m, r, tu, 0, kClu / 2, kit, m);
    } else {
      clu_qr(cl, sh, WV, n, r, tv, kClu / 2, kClu / 2, kit, n);
    }
  }
  cstage(1);
  const int kqmax = min(ku, kv);
  double* tau = C + (size_t)ku * kv;
  double* cn = tau + kv;                                // 2 kv (double-buffered norms)
  int* phys = reinterpret_cast<int*>(cn + 2 * kv);      // kv ints
  int* stepof = phys + kv;                              // kv ints
  double* G = cn + 3 * kv;
  double* J = G + (size_t)kv * kqmax;
  double* Uc = J + (size_t)kqmax * kqmax;
  double* gsig = Uc + (size_t)ku * kqmax;  // exported sigma / order for the other CTAs
  int* gord = reinterpret_cast<int*>(gsig + kqmax);
  RS rs{0, 0, 0.0};
  {  // core(i,j) = sum_{l >= max(i,j)} Ru(i,l) Rv(j,l), 32x32 tiles spread over all
     // ranks of the cluster and staged through shared memory (sh.part is free
     // between the QR and the Q application).  Every entry accumulates l in
     // ascending order from a start <= max(i,j); the masked entries below the
     // diagonals contribute exact zeros, so C is bit-identical to the
     // one-rank formula it replaces.
    double* As = &sh.part[0][0];  // [l][i], 32 x 32
    double* Bs = As + 1024;       // [l][j]
    const int ti = (ku + 31) / 32, tj = (kv + 31) / 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, nty = blockDim.x >> 5;
    for (int t = rank; t < ti * tj; t += kClu) {
      const int i0 = (t % ti) * 32, j0 = (t / ti) * 32;
      double acc[2] = {0.0, 0.0};
      for (int l0 = max(i0, j0); l0 < r; l0 += 32) {
        __syncthreads();
        for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
          const int a = e & 31, gl = l0 + (e >> 5), gi = i0 + a, gj = j0 + a;
          As[e] = (gl < r && gi < ku && gi <= gl) ? WU[(size_t)gl * m + gi] : 0.0;
          Bs[e] = (gl < r && gj < kv && gj <= gl) ? WV[(size_t)gl * n + gj] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
          const double a = As[l * 32 + tx];
          for (int q = 0; q < 2; ++q)
            if (ty + q * nty < 32) acc[q] += a * Bs[l * 32 + ty + q * nty];
        }
      }
      for (int q = 0; q < 2; ++q) {
        const int i = i0 + tx, j = j0 + ty + q * nty;
        if (ty + q * nty < 32 && i < ku && j < kv) C[(size_t)j * ku + i] = acc[q];
      }
    }
    cl.sync();
  }
  cstage(2);
  if (rank == 0) {
    // lean rank-revealing SVD (virtual pivoting, one barrier per step)
    const bool lean = kv <= 128;  // the lean variant's pivot bitmask covers 128 columns
    long long tcs = clock64();    // HMGP_STATS: rrqr / jacobi / core-Q split in path 1's slots
    if (lean) {
      rs = cta_rrqr_svd2(C, ku, kv, eps, tau, phys, cn, stepof, G, J, s_sig, s_ord, 1, &tcs);
    } else {
      rs = cta_rrqr_svd(C, ku, kv, eps, tau, phys, cn, G, J, s_sig, s_ord, red);
      for (int j = threadIdx.x; j < kv; j += blockDim.x) phys[j] = j;  // explicit swaps: identity map
      __syncthreads();
    }
    for (int idx = threadIdx.x; idx < ku * rs.keep; idx += blockDim.x) {
      const int i = idx % ku, c = idx / ku, src = s_ord[c];
      Uc[idx] = i < rs.kq ? J[(size_t)src * rs.kq + i] * s_sig[src] : 0.0;
    }
    __syncthreads();
    cta_apply_q_map(C, ku, ku, rs.kq, tau, phys, Uc, rs.keep);
    stage_add(1, 4, tcs);
    for (int c = threadIdx.x; c < rs.keep; c += blockDim.x) {
      gsig[c] = s_sig[s_ord[c]];
      gord[c] = s_ord[c];
    }
    if (threadIdx.x == 0) {
      s_kq = rs.kq;
      gord[kqmax] = rs.keep;  // published to the cluster through global memory
    }
    __syncthreads();
  }
  cl.sync();
  cstage(3);
  const int keep = gord[kqmax];
  if (keep > it.cap) {
    if (rank == 0 && threadIdx.x == 0) atomicOr(err, 4);
    cl.sync();
    return;
  }
  // E_u = [U_core; 0] -> it.U, E_v = [Y; 0] -> it.V (own row slices)
  {
    for (int c = 0; c < keep; ++c) {
      for (int i = mlo + threadIdx.x; i < mhi; i += blockDim.x)
        it.U[(size_t)c * m + i] = i < ku ? Uc[(size_t)c * ku + i] : 0.0;
      const int src = gord[c];
      const double sg = gsig[c];
      for (int i = nlo + threadIdx.x; i < nhi; i += blockDim.x)
        it.V[(size_t)c * n + i] = i < kv ? G[(size_t)src * kv + i] / sg : 0.0;
    }
  }
  cl.sync();
  cstage(4);
  {
    const int kit = max(ku, kv);
    if (rank < kClu / 2) {
      clu_apply_q(cl, sh, WU, m, ku, tu, it.U, keep, 0, kClu / 2, kit, m, m);
    } else {
      clu_apply_q(cl, sh, WV, n, kv, tv, it.V, keep, kClu / 2, kClu / 2, kit, n, n);
    }
  }
  cstage(5);
  cstage(6);
  if (rank == 0 && threadIdx.x == 0) {
    *it.rank = keep;
    if (it.compact) *it.compact = keep;
    const double fl = qr_flops(m, r) + qr_flops(n, r) + (double)ku * kv * r + rs.flops +
                      4.0 * keep * ((double)m * ku + (double)n * kv + (double)ku * s_kq);
    atomicAdd(&d_cnt_trunc, fl);
    atomicAdd(&d_cnt_titems, 1.0);
  }
  if (rank == 0) hist_add(2, m, n, r, t0);
  cl.sync();
}


// ===================================================================== //
// Medium blocks: a CTA PAIR (cluster of 2) per target.  CTA 0 owns the U side,
// CTA 1 the V side; each keeps its stacked factor [U | aP] or [V | Q] resident
// in shared memory, so both Householder QRs run at once with one barrier per
// column (the next column's tail norm is produced by the update that touches
// it).  The r x r core R_u R_v^T is formed and decomposed redundantly by both
// CTAs (identical arithmetic, identical results), and each side applies its Q
// in compact WY form, I - Y T Y^T, with one pass that writes the new factor to
// global memory.  Items whose factors do not fit fall back, on device, to the
// single-CTA global-memory path run by CTA 0.
// ===================================================================== //
constexpr int kPairMaxR = 128;


// out (mm x c, ld mm, global) = Q [E0; 0] with Q = H_0 ... H_{k-1} from
// smem_qr(A) in compact WY form Q = I - Y T Y^T (T upper triangular, the
// forward column-wise recurrence of dlarft).  E0 is k x c (ld k).  Scratch: S
// and T (k x k), X (k x c); S may alias X's storage only after T is built, so
// the caller passes distinct buffers for S/Z and T/X1 pairs as documented.
__device__ void wy_apply(const double* A, int mm, int lda, int k, const double* tau, const double* E0,
                         int c, double* out, double* S, double* T, double* X1) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // S(l, q) = v_l^T v_q for l < q (ld k), four dots per warp in flight
  const int np = k * (k - 1) / 2;
  for (int pb = 4 * w; pb < np; pb += 4 * nw) {
    int ls[4], qs[4];
    double s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int p = min(pb + u, np - 1);
      // pair index p -> (l, q) with q = floor((1 + sqrt(1 + 8p)) / 2)
      int q = (int)((1.0 + sqrt(1.0 + 8.0 * p)) * 0.5);
      while (q * (q - 1) / 2 > p) --q;
      while ((q + 1) * q / 2 <= p) ++q;
      ls[u] = p - q * (q - 1) / 2;
      qs[u] = q;
      s[u] = 0.0;
    }
    int qmin = qs[0];
#pragma unroll
    for (int u = 1; u < 4; ++u) qmin = min(qmin, qs[u]);
    for (int i = qmin + 1 + lane; i < mm; i += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i > qs[u]) s[u] += A[(size_t)ls[u] * lda + i] * A[(size_t)qs[u] * lda + i];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = warp_sum(s[u]);
      if (lane == 0 && pb + u < np) S[(size_t)qs[u] * k + ls[u]] = v + A[(size_t)ls[u] * lda + qs[u]];
    }
  }
  __syncthreads();
  // T recurrence: T(q,q) = tau_q, T(0:q, q) = -tau_q T(0:q, 0:q) S(0:q, q)
  for (int q = 0; q < k; ++q) {
    const double tq = tau[q];
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
      double s = 0.0;
      for (int l = i; l < q; ++l) s += T[(size_t)l * k + i] * S[(size_t)q * k + l];
      T[(size_t)q * k + i] = -tq * s;
    }
    if (threadIdx.x == 0) T[(size_t)q * k + q] = tq;
    for (int i = q + 1 + threadIdx.x; i < k; i += blockDim.x) T[(size_t)q * k + i] = 0.0;
    __syncthreads();
  }
  // X1 = Y1^T E0 (Y1 = unit lower k x k top of Y), then Z = T X1 into S's storage
  for (int e = threadIdx.x; e < k * c; e += blockDim.x) {
    const int l = e % k, cc = e / k;
    const double* ec = E0 + (size_t)cc * k;
    double s = ec[l];
    for (int i = l + 1; i < k; ++i) s += A[(size_t)l * lda + i] * ec[i];
    X1[e] = s;
  }
  __syncthreads();
  double* Z = S;
  for (int e = threadIdx.x; e < k * c; e += blockDim.x) {
    const int l = e % k, cc = e / k;
    const double* xc = X1 + (size_t)cc * k;
    double s = 0.0;
    for (int j = l; j < k; ++j) s += T[(size_t)j * k + l] * xc[j];
    Z[e] = s;
  }
  __syncthreads();
  // out(i, cc) = [E0; 0](i, cc) - sum_{l <= min(i, k-1)} Y(i, l) Z(l, cc)
  for (int e = threadIdx.x; e < mm * c; e += blockDim.x) {
    const int i = e % mm, cc = e / mm;
    const double* zc = Z + (size_t)cc * k;
    double s = (i < k) ? E0[(size_t)cc * k + i] - zc[i] : 0.0;  // Y(i,i) = 1 term
    const int lmax = min(i, k);
    for (int l = 0; l < lmax; ++l) s -= A[(size_t)l * lda + i] * zc[l];
    out[(size_t)cc * mm + i] = s;
  }
}

// shared-memory doubles the pair path needs for an m x n target with r columns
__host__ __device__ __forceinline__ size_t pair_smem_doubles(int m, int n, int r) {
  return (size_t)(max(m, n) | 1) * r + 4 * (size_t)r * r + 5 * (size_t)r + 8;
}

// the pair path covers the item: columns, shared memory, register QR shape
__device__ __forceinline__ bool pair_fits(int m, int n, int r, int cap_dbl) {
  return r <= kPairMaxR && pair_smem_doubles(m, n, r) <= (size_t)cap_dbl && !(max(m, n) > 256 && r > 32) &&
         max(m, n) <= 512;
}

// Pair-path recompression of one item.  The caller has read the item's rank
// (r0) in every CTA of its cluster and synchronised the cluster.  `active` is
// true on the two CTAs doing the work (cluster ranks 0: U side, 1: V side);
// inside the 8-CTA cluster kernel the other ranks call it with active = false
// and only take part in the cluster barriers (the barrier sequence depends
// only on item data, identical in every rank).  Returns false (nothing done)
// when the item does not fit and may_defer is set.  kFallback: run items that
// do not fit on CTA 0's single-CTA paths (the cluster kernel never passes such
// items).
template <bool kFallback>
__device__ bool lr_update_pair(cg::cluster_group& cl, const TruncItem& it, double eps, int* err,
                               int cap_dbl, double* sm, bool may_defer, int r0, bool active) {
  const int side = (int)cl.block_rank() & 1;  // 0: U side, 1: V side
  const bool lead = cl.block_rank() == 0 && threadIdx.x == 0;
  __shared__ double s_sig[kPairMaxR];
  __shared__ int s_ord[kPairMaxR];
  __shared__ double s_tail[2];
  const int add = it.P ? (it.addp ? *it.addp : it.addv) : 0;
  const int r = r0 + add;
  bool go;
  switch (it.cond) {
    case 1: go = r > 16; break;
    case 2: go = r > *it.compact + 16; break;
    case 3: go = r > 48; break;
    case 4: go = false; break;
    default: go = r > 0; break;
  }
  const int m = it.m, n = it.n;
  const int mm = side ? n : m;
  double* X = side ? it.V : it.U;
  if (!go) {
    if (add > 0 && r > it.cap) {
      if (lead) atomicOr(err, 2);
      cl.sync();
      return true;
    }
    if (active)
      for (size_t e = threadIdx.x; e < (size_t)mm * add; e += blockDim.x) {
        const int i = (int)(e % mm), k = (int)(e / mm);
        double v;
        if (side == 0) {
          const int pi = i - it.pro;
          v = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)k * it.ldp + pi] : 0.0;
        } else {
          const int qi = i - it.qro;
          v = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)k * it.ldq + qi] : 0.0;
        }
        X[(size_t)(r0 + k) * mm + i] = v;
      }
    if (lead) {
      *it.rank = r;
      if (it.cond == 0 && it.compact) *it.compact = r;
    }
    cl.sync();
    return true;
  }
  if (r > it.rcap) {
    if (lead) atomicOr(err, 1);
    cl.sync();
    return true;
  }
  if (!pair_fits(m, n, r, cap_dbl)) {
    if (may_defer) return false;
    // single-CTA paths on CTA 0 (W in shared memory when it fits, else global)
    if (kFallback && cl.block_rank() == 0) lr_update(it, eps, err, kMaxSmemW, kMaxSmemMN);
    cl.sync();
    return true;
  }
  const long long t0 = clock64();
  long long tc = t0;
  const int ku = min(m, r), kv = min(n, r);
  const int kme = side ? kv : ku, ko = side ? ku : kv, mo = side ? m : n;
  const int lda = mm | 1, ldo = mo | 1;    // odd strides: conflict-free row-varying access
  double* A = sm;                          // mm x r (ld lda)
  double* Ro = A + (size_t)lda * r;        // other side's R (ko x r), later G, later X1
  double* C = Ro + (size_t)r * r;          // core ku x kv, later T
  double* J = C + (size_t)r * r;           // kq x kq, later S / Z
  double* E0 = J + (size_t)r * r;          // kme x keep
  double* tau = E0 + (size_t)r * r;        // r
  double* tau_c = tau + r;                 // r
  double* cn = tau_c + r;                  // 2r (double-buffered trailing norms)
  int* phys = reinterpret_cast<int*>(cn + 2 * r);  // r ints: core pivot order
  int* stepof = phys + r;                          // r ints
  if (active) {
    // stage [X | added] (mm x r)
    for (size_t e = threadIdx.x; e < (size_t)mm * r; e += blockDim.x) {
      const int i = (int)(e % mm), l = (int)(e / mm);
      double v;
      if (l < r0) {
        v = X[e];
      } else if (side == 0) {
        const int pi = i - it.pro;
        v = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)(l - r0) * it.ldp + pi] : 0.0;
      } else {
        const int qi = i - it.qro;
        v = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)(l - r0) * it.ldq + qi] : 0.0;
      }
      A[(size_t)l * lda + i] = v;
    }
    __syncthreads();
    stage_add(2, 0, tc);
    __shared__ double s_vbuf[2 * 512];
    __shared__ double s_sbuf[2];
    if (!reg_qr_any(A, mm, lda, r, tau, s_vbuf, s_sbuf)) smem_qr(A, mm, lda, r, tau, s_tail);
    stage_add(2, 1, tc);
  }
  cl.sync();
  int keep = 0;
  RS rs{0, 0, 0.0};
  if (active) {
    {  // other side's R through distributed shared memory
      const double* Aot = cl.map_shared_rank(A, side ^ 1);
      for (int e = threadIdx.x; e < ko * r; e += blockDim.x) {
        const int i = e % ko, l = e / ko;
        Ro[e] = (i <= l) ? Aot[(size_t)l * ldo + i] : 0.0;
      }
    }
    __syncthreads();
    // core(i,j) = sum_{l >= max(i,j)} Ru(i,l) Rv(j,l)  (ku x kv, ld ku); both sides
    // form it with identical arithmetic
    {
      const double* Ru = side ? Ro : A;
      const double* Rv = side ? A : Ro;
      const int ldu = side ? ku : lda, ldv = side ? lda : kv;
      for (int idx = threadIdx.x; idx < ku * kv; idx += blockDim.x) {
        const int i = idx % ku, j = idx / ku;
        double s = 0.0;
        for (int l = max(i, j); l < r; ++l) s += Ru[(size_t)l * ldu + i] * Rv[(size_t)l * ldv + j];
        C[(size_t)j * ku + i] = s;
      }
    }
    __syncthreads();
    rs = cta_rrqr_svd2(C, ku, kv, eps, tau_c, phys, cn, stepof, Ro, J, s_sig, s_ord, 2, &tc);
    keep = rs.keep;
    const int kq = rs.kq;
    if (keep > it.cap) {
      if (lead) atomicOr(err, 4);
    } else {
      if (side == 0) {  // U_core = Q_core [J S; 0] (ku x keep)
        for (int idx = threadIdx.x; idx < ku * keep; idx += blockDim.x) {
          const int i = idx % ku, c = idx / ku, src = s_ord[c];
          E0[idx] = i < kq ? J[(size_t)src * kq + i] * s_sig[src] : 0.0;
        }
        __syncthreads();
        cta_apply_q_map(C, ku, ku, kq, tau_c, phys, E0, keep);
      } else {  // Y (kv x keep)
        for (int idx = threadIdx.x; idx < kv * keep; idx += blockDim.x) {
          const int i = idx % kv, c = idx / kv, src = s_ord[c];
          E0[idx] = Ro[(size_t)src * kv + i] / s_sig[src];
        }
      }
      __syncthreads();
      wy_apply(A, mm, lda, kme, tau, E0, keep, X, J, C, Ro);
      stage_add(2, 4, tc);
    }
  }
  cl.sync();
  if (lead && keep <= it.cap) {
    *it.rank = keep;
    if (it.compact) *it.compact = keep;
    const double fl = qr_flops(m, r) + qr_flops(n, r) + (double)ku * kv * r + rs.flops +
                      4.0 * keep * ((double)m * ku + (double)n * kv + (double)ku * rs.kq);
    atomicAdd(&d_cnt_trunc, fl);
    atomicAdd(&d_cnt_titems, 1.0);
  }
  if (cl.block_rank() == 0) hist_add(3, m, n, r, t0);
  cl.sync();
  return true;
}

// cluster b (CTA pair 2b, 2b+1) runs target b's sequence in order
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTruncThreads)
    k_truncate_pair(const TruncItem* __restrict__ items, const int* __restrict__ off, double eps,
                    int* err, int cap_dbl, int* defer) {
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double psm[];
  const int b = blockIdx.x / 2;
  const bool lead = cl.block_rank() == 0 && threadIdx.x == 0;
  const long long ts = clock64();
  if (defer && lead) defer[b] = -1;
  for (int i = off[b]; i < off[b + 1]; ++i) {
    const TruncItem& it = items[i];
    const int r0 = *it.rank;
    cl.sync();  // both CTAs have read rank / compact before either may change them
    if (!lr_update_pair<true>(cl, it, eps, err, cap_dbl, psm, defer != nullptr, r0, true)) {
      if (lead) defer[b] = i;  // items[i..] go to the cluster kernel, in order
      break;
    }
    if (it.post_L) {
      if (cl.block_rank() == 1) lr_post_solve(it);
      cl.sync();
    }
  }
  if (cl.block_rank() == 0) seq_done(ts);
}

#include "trunc_dist.cuh"

// cluster b (CTAs b*kClu .. b*kClu+kClu-1) runs target b's sequence in order
__global__ void __cluster_dims__(kClu, 1, 1) __launch_bounds__(kTruncThreads)
    k_truncate_cluster(const TruncItem* __restrict__ items, const int* __restrict__ off, double eps,
                       int* err, const int* __restrict__ defer, int cap_dbl) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ CluShared sh;
  __shared__ double s_sig_d[64];
  __shared__ int s_ord_d[64];
  extern __shared__ double csm[];
  // the register path's exchange area sits at the end of the dynamic region
  // (same offset in every CTA, so DSMEM addresses line up)
  constexpr int kDsDbl = (int)((sizeof(DistShared) + 7) / 8);
  DistShared& dsh = *reinterpret_cast<DistShared*>(csm + max(cap_dbl - kDsDbl, 0));
  const int cap_dist = cap_dbl - kDsDbl;
  const long long ts = clock64();
  const int b = blockIdx.x / kClu;
  int start = off[b];
  if (defer) {  // only the sequence tail the pair kernel handed over
    start = defer[b];
    if (start < 0) return;
  }
  for (int i = start; i < off[b + 1]; ++i) {
    const TruncItem& it = items[i];
    const int r0 = *it.rank;
    // every rank has read rank / compact before any may change them (the
    // cluster path itself writes them only after its own cluster barriers)
    if (cap_dbl > 0) cl.sync();
    // with a shared-memory carve-out (cap_dbl > 0), items whose actual column
    // count fits run on ranks 0-1 as a pair, or register-resident over all
    // eight ranks; the rest take the global-memory cluster path
    bool pair = false, dist = false;
    if (cap_dbl > 0) {
      const int add = it.P ? (it.addp ? *it.addp : it.addv) : 0;
      const int r = r0 + add;
      bool go;
      switch (it.cond) {
        case 1: go = r > 16; break;
        case 2: go = r > *it.compact + 16; break;
        case 3: go = r > 48; break;
        case 4: go = false; break;
        default: go = r > 0; break;
      }
      if (go && r <= it.rcap) {
        pair = pair_fits(it.m, it.n, r, cap_dbl);
        dist = !pair && dist_fits(it.m, it.n, r, cap_dist);
        if (dist) lr_update_dist_any(cl, it, eps, err, r0, r, add, csm, dsh, s_sig_d, s_ord_d);
      }
    }
    if (pair)
      lr_update_pair<false>(cl, it, eps, err, cap_dbl, csm, false, r0, cl.block_rank() < 2);
    else if (!dist)
      lr_update_cluster(cl, sh, it, eps, err, r0);
    if (it.post_L) {
      if (cl.block_rank() == (pair ? 1 : 0)) lr_post_solve(it);
      cl.sync();
    }
  }
  if (cl.block_rank() == 0) seq_done(ts);
}

static int g_pair_cap = -1;
static size_t g_pair_bytes = 0;
void launch_truncate_pair(const TruncItem* d_items, const int* d_off, int targets, double eps,
                          int* d_err, cudaStream_t st, int* d_defer) {
  if (targets <= 0) return;
  if (g_pair_cap < 0) {
    cudaFuncAttributes fa;
    HMGP_CUDA(cudaFuncGetAttributes(&fa, k_truncate_pair));
    int dev = 0, optin = 0;
    HMGP_CUDA(cudaGetDevice(&dev));
    HMGP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    g_pair_bytes = (size_t)optin - fa.sharedSizeBytes - 1024;
    HMGP_CUDA(cudaFuncSetAttribute(k_truncate_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)g_pair_bytes));
    g_pair_cap = (int)(g_pair_bytes / 8);
  }
  int* dfr = d_defer;  // per-target hand-over index (targets ints), or nullptr
  k_truncate_pair<<<targets * 2, kTruncThreads, g_pair_bytes, st>>>(d_items, d_off, eps, d_err,
                                                                   g_pair_cap, dfr);
  HMGP_LAUNCH_CHECK();
  if (dfr) {
    k_truncate_cluster<<<targets * kClu, kTruncThreads, 0, st>>>(d_items, d_off, eps, d_err, dfr, 0);
    HMGP_LAUNCH_CHECK();
  }
}

size_t trunc_ws_doubles_pair(int m, int n, int rcap) {  // the single-CTA fallbacks (either path)
  const size_t rc = (size_t)rcap, kq = std::min((size_t)std::min(m, n), rc);
  return std::max(trunc_ws_doubles(m, n, rcap),
                  (size_t)(m + n) * rc + 6 * rc + rc * rc + 2 * rc * kq + kq * kq);
}

bool trunc_use_pair(int m, int n, int rcap) {
  (void)rcap;
  if ((size_t)m * n <= (size_t)kMaxSmemW / 4) return false;
  return std::max(m, n) <= 256;
}

// 1: pair (device fallback to one CTA), 3: pair with hand-over of items that
// do not fit (rank known only on device) to the 8-CTA cluster kernel,
// 2: cluster, 0: one CTA
int trunc_route(int m, int n, int rcap) {
  if (trunc_use_pair(m, n, rcap)) return 1;
  if (trunc_use_cluster(m, n)) return 2;  // (the cluster kernel runs fitting items as a pair)
  return 0;
}

size_t trunc_ws_for(int m, int n, int rcap) {
  switch (trunc_route(m, n, rcap)) {
    case 3:
    case 2: return trunc_ws_doubles_cluster(m, n, rcap);
    case 1: return trunc_ws_doubles_pair(m, n, rcap);
    default: return trunc_ws_doubles(m, n, rcap);
  }
}

size_t trunc_ws_doubles_cluster(int m, int n, int rcap) {
  const size_t rc = (size_t)rcap, kq = std::min((size_t)std::min(m, n), rc);
  return (size_t)(m + n) * rc + 5 * rc + rc * rc + 3 * rc * kq + kq * kq + 2 * kq + 2;
}

bool trunc_cluster_resident(int m, int n) { return std::max(m, n) <= 2048; }

bool trunc_use_cluster(int m, int n) {
  return !((size_t)m * n <= (size_t)kMaxSmemW && m + n <= kMaxSmemMN) && std::max(m, n) >= 512;
}

void launch_truncate_cluster(const TruncItem* d_items, const int* d_off, int targets, double eps,
                             int* d_err, cudaStream_t st, bool resident) {
  if (targets <= 0) return;
  // resident = false: no shared-memory carve-out (cap_dbl = 0), everything on the
  // global-memory cluster path, which depends on L1 holding its row slices.
  // resident = true: pair / register-resident dispatch per item (targets up to
  // 2048 rows, where most items fit).
  static int cap = -1;
  static size_t bytes = 0;
  if (resident && cap < 0) {
    cudaFuncAttributes fa;
    HMGP_CUDA(cudaFuncGetAttributes(&fa, k_truncate_cluster));
    int dev = 0, optin = 0;
    HMGP_CUDA(cudaGetDevice(&dev));
    HMGP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // ~112 KB: enough for the register path's slices (ms <= 256 at r <= 32,
    // ms <= 128 at r <= 40) while leaving L1 for the items that fall back to
    // the global-memory path (measured: a 200 KB carve-out holding the global
    // path's row slices in shared memory instead was 20 % slower per item --
    // the rank-0 core SVD then misses L1)
    bytes = std::min((size_t)optin - fa.sharedSizeBytes - 1024, (size_t)14336 * 8);
    HMGP_CUDA(cudaFuncSetAttribute(k_truncate_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)bytes));
    cap = (int)(bytes / 8);
  }
  k_truncate_cluster<<<targets * kClu, kTruncThreads, resident ? bytes : 0, st>>>(
      d_items, d_off, eps, d_err, nullptr, resident ? cap : 0);
  HMGP_LAUNCH_CHECK();
}

void launch_truncate(const TruncItem* d_items, int count, double eps, int* d_err, cudaStream_t st,
                     int smem_w, int smem_mn) {
  if (count <= 0) return;
  if (smem_w > kMaxSmemW || smem_mn > kMaxSmemMN) {
    smem_w = 0;
    smem_mn = 0;
  }
  const size_t bytes = ((size_t)smem_w + (size_t)kChunk * smem_mn) * 8;
  static bool configured = false;
  if (!configured) {
    const int mx = (int)((kMaxSmemW + (size_t)kChunk * kMaxSmemMN) * 8);
    HMGP_CUDA(cudaFuncSetAttribute(k_truncate, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    HMGP_CUDA(cudaFuncSetAttribute(k_truncate_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    configured = true;
  }
  k_truncate<<<count, kTruncThreads, bytes, st>>>(d_items, eps, d_err, smem_w, smem_mn);
  HMGP_LAUNCH_CHECK();
}

void launch_truncate_seq(const TruncItem* d_items, const int* d_off, int targets, double eps,
                         int* d_err, cudaStream_t st, int smem_w, int smem_mn) {
  if (targets <= 0) return;
  if (smem_w > kMaxSmemW || smem_mn > kMaxSmemMN) {
    smem_w = 0;
    smem_mn = 0;
  }
  const size_t bytes = ((size_t)smem_w + (size_t)kChunk * smem_mn) * 8;
  static bool configured = false;
  if (!configured) {
    const int mx = (int)((kMaxSmemW + (size_t)kChunk * kMaxSmemMN) * 8);
    HMGP_CUDA(cudaFuncSetAttribute(k_truncate, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    HMGP_CUDA(cudaFuncSetAttribute(k_truncate_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    configured = true;
  }
  k_truncate_seq<<<targets, kTruncThreads, bytes, st>>>(d_items, d_off, eps, d_err, smem_w, smem_mn);
  HMGP_LAUNCH_CHECK();
}

}  // namespace hmgp_gpu
