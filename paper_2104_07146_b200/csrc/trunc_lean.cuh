// Latency-lean CTA building blocks for the recompression kernels (included by
// truncate.cu after RS / stage_add are defined): one barrier per Householder
// column, per pivoted-QR step and per Jacobi round.  Reductions of several
// independent values are interleaved level by level so their shuffle
// latencies overlap.
#pragma once

template <int N>
__device__ __forceinline__ void warp_sum_n(double (&v)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int u = 0; u < N; ++u) v[u] += __shfl_xor_sync(0xffffffffu, v[u], o);
  }
}

// Householder scalars of a column with head c0 and tail norm^2 tail2 (the
// convention of cta_householder: v = [1; inv * x], H = I - t v v^T).
__device__ __forceinline__ void hh_scalars(double c0, double tail2, double& t, double& beta,
                                           double& inv) {
  if (tail2 <= 2.2250738585072014e-308) {
    t = 0.0;
    beta = c0;
    inv = 0.0;
  } else {
    beta = sqrt(c0 * c0 + tail2);
    if (c0 >= 0.0) beta = -beta;
    inv = 1.0 / (c0 - beta);
    t = (beta - c0) / beta;
  }
}

// Apply the reflector given by the raw column x (rows > k) and its scalars to
// up to four columns c[u] (rows >= k) owned by one warp.  With tail != nullptr
// also returns the new tail norm^2 (rows > k+1) of c[0].
__device__ __forceinline__ void warp_reflect4(const double* x, double* (&c)[4], const bool (&on)[4], int k,
                                              int mm, double t, double inv, int lane, double* tail) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  if (t != 0.0) {
    for (int i = k + 1 + lane; i < mm; i += 32) {
      const double v = x[i];
#pragma unroll
      for (int u = 0; u < 4; ++u) s[u] += v * c[u][i];
    }
    warp_sum_n<4>(s);
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = (c[u][k] + inv * s[u]) * t;
  }
  double q = 0.0;
  if (t != 0.0) {
    for (int i = k + 1 + lane; i < mm; i += 32) {
      const double v = x[i] * inv;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!on[u]) continue;
        const double y = c[u][i] - s[u] * v;
        c[u][i] = y;
        if (u == 0 && i > k + 1) q += y * y;
      }
    }
  } else {
    for (int i = k + 2 + lane; i < mm; i += 32) q += c[0][i] * c[0][i];
  }
  if (tail) *tail = warp_sum(q);
  __syncwarp();
  if (lane == 0 && t != 0.0)
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (on[u]) c[u][k] -= s[u];
  __syncwarp();
}

// In-place Householder QR of A (mm x r, ld lda, shared memory); reflectors
// normalised v = [1; A(k+1:, k)], R on and above the diagonal, tau[min(mm,r)].
// Warp 0 updates column k+1 alone and produces its tail norm for the next step;
// the other warps take the remaining trailing columns, four per pass; the
// normalisation of a reflector is applied one step late (nobody reads it then).
__device__ void smem_qr(double* A, int mm, int lda, int r, double* tau, double* s_tail) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kmax = min(mm, r);
  if (kmax <= 0) return;
  if (w == 0) {
    double s = 0.0;
    for (int i = 1 + lane; i < mm; i += 32) s += A[i] * A[i];
    s = warp_sum(s);
    if (lane == 0) s_tail[0] = s;
  }
  __syncthreads();
  double pt = 0.0, pinv = 0.0, pbeta = 0.0;
  const int nt = nw - 1;  // warps sharing columns k+2..
  for (int k = 0; k < kmax; ++k) {
    const double* x = A + (size_t)k * lda;
    double t, beta, inv;
    hh_scalars(x[k], s_tail[k & 1], t, beta, inv);
    if (w == 0) {
      if (k + 1 < r) {
        double* c[4];
        const bool on[4] = {true, false, false, false};
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = A + (size_t)(k + 1) * lda;
        double tail;
        warp_reflect4(x, c, on, k, mm, t, inv, lane, &tail);
        if (lane == 0) s_tail[(k + 1) & 1] = tail;
      }
    } else {
      if (w == nw - 1 && k > 0) {  // lagged normalisation of column k-1
        double* xp = A + (size_t)(k - 1) * lda;
        for (int i = k + lane; i < mm; i += 32) xp[i] = (pt == 0.0) ? 0.0 : xp[i] * pinv;
        if (lane == 0) {
          xp[k - 1] = pbeta;
          tau[k - 1] = pt;
        }
      }
      for (int jb = k + 2 + (w - 1); jb < r; jb += 4 * nt) {
        double* c[4];
        bool on[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = jb + u * nt;
          on[u] = j < r;
          c[u] = A + (size_t)(on[u] ? j : jb) * lda;
        }
        warp_reflect4(x, c, on, k, mm, t, inv, lane, nullptr);
      }
    }
    pt = t;
    pinv = inv;
    pbeta = beta;
    __syncthreads();
  }
  if (w == nw - 1) {
    double* xp = A + (size_t)(kmax - 1) * lda;
    for (int i = kmax + lane; i < mm; i += 32) xp[i] = (pt == 0.0) ? 0.0 : xp[i] * pinv;
    if (lane == 0) {
      xp[kmax - 1] = pbeta;
      tau[kmax - 1] = pt;
    }
  }
  __syncthreads();
}

// E <- Q E with Q = H_0 ... H_{kq-1}; reflector s lives in column map[s] of QR
// (ld ldq; rows > s, unit head at row s).  E is m x c (ld m).
__device__ void cta_apply_q_map(const double* QR, int m, int ldq, int kq, const double* tau,
                                const int* map, double* E, int c) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = kq - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t != 0.0) {
      const double* v = QR + (size_t)map[k] * ldq;
      for (int jb = 4 * w; jb < c; jb += 4 * nw) {
        double* cc[4];
        bool on[4];
        double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          on[u] = jb + u < c;
          cc[u] = E + (size_t)(on[u] ? jb + u : jb) * m;
        }
        for (int i = k + 1 + lane; i < m; i += 32) {
          const double vi = v[i];
#pragma unroll
          for (int u = 0; u < 4; ++u) s[u] += vi * cc[u][i];
        }
        warp_sum_n<4>(s);
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = (s[u] + cc[u][k]) * t;
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (!on[u]) continue;
          for (int i = k + 1 + lane; i < m; i += 32) cc[u][i] -= s[u] * v[i];
        }
        __syncwarp();
        if (lane == 0)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (on[u]) cc[u][k] -= s[u];
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

// One-sided Jacobi with the rotations and stopping rule of cta_jacobi, one
// barrier per round.  A pair is handled by a group of G lanes (G sized to the
// column length p: 8 lanes for p <= 64, ...), so a warp works on 32/G pairs at
// once and the three dot products of a pair reduce over log2(G) shuffle levels
// -- the round is bound by instruction issue, not by latency, and this cuts
// the instructions per pair by ~32/G.
// tol: rotate a pair while |w_a . w_b| > tol * |w_a| |w_b|.  R = J G^T holds
// exactly whatever the convergence state, so the truncation error is bounded by
// the norms of the dropped columns in any case; a tolerance tied to the cut
// (tol <= 1e-4 eps) only spares the final sweeps.
template <int G>
__device__ bool jacobi_round(double* W, int p, int q, double* J, int qq, int m1, int round, double tol2,
                             unsigned& nrot) {
  constexpr int kGpw = 32 / G;  // pairs per warp at once
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gi = lane / G, gl = lane % G;
  bool rot = false;
  for (int base = w * kGpw; base < qq / 2; base += nw * kGpw) {
    const int t = base + gi;
    bool act = t < qq / 2;
    int a = 0, b = 0;
    if (act) {
      if (t == 0) {
        a = qq - 1;
        b = round;
      } else {  // (round + t) mod m1 and (round - t) mod m1 without divisions
        a = round + t;
        if (a >= m1) a -= m1;
        b = round - t;
        if (b < 0) b += m1;
      }
      if (a > b) {
        const int tmp = a;
        a = b;
        b = tmp;
      }
      if (b >= q) act = false;
    }
    double sa = 0.0, sb = 0.0, sc = 0.0;
    double* wj = W + (size_t)a * p;
    double* wk = W + (size_t)b * p;
    if (act)
      for (int i = gl; i < p; i += G) {
        const double x = wj[i], y = wk[i];
        sa += x * x;
        sb += y * y;
        sc += x * y;
      }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
      sc += __shfl_xor_sync(0xffffffffu, sc, o);
    }
    // |sc| <= tol sqrt(sa sb), squared (sa, sb >= 0)
    if (!act || sc * sc <= tol2 * (sa * sb) || sc == 0.0) continue;
    rot = true;
    if (gl == 0) ++nrot;
    // Rotation from cos 2phi = |dd| / sqrt(dd^2 + 4 sc^2), |phi| <= pi/4:
    //   cos^2 phi = (1 + cos 2phi) / 2,  sin phi = sin 2phi / (2 cos phi)
    // — the same angle as tan phi = 2 sc sign(dd) / (|dd| + sqrt(dd^2 + 4 sc^2)), but
    // the dependent chain is two reciprocal square roots instead of a square root, a
    // division and a reciprocal square root (every pair of a round waits on it, and
    // a dependent FP64 op costs ~40 cycles here).  sin phi is formed from sc itself,
    // so small angles keep full relative accuracy.
    const double dd = sb - sa;
    const double rz = rsqrt(dd * dd + 4.0 * sc * sc);
    const double c2h = 0.5 + 0.5 * fabs(dd) * rz;  // cos^2 phi in [1/2, 1]
    const double rc = rsqrt(c2h);
    const double cs = c2h * rc, sn = (dd >= 0.0 ? sc : -sc) * rz * rc;
    for (int i = gl; i < p; i += G) {
      const double x = wj[i], y = wk[i];
      wj[i] = cs * x - sn * y;
      wk[i] = sn * x + cs * y;
    }
    double* jj = J + (size_t)a * q;
    double* jk = J + (size_t)b * q;
    for (int i = gl; i < q; i += G) {
      const double x = jj[i], y = jk[i];
      jj[i] = cs * x - sn * y;
      jk[i] = sn * x + cs * y;
    }
  }
  return rot;
}

__device__ double cta_jacobi2(double* W, int p, int q, double* J, int* sweeps_out, double tol) {
  const int lane = threadIdx.x & 31;
  for (int idx = threadIdx.x; idx < q * q; idx += blockDim.x) J[idx] = (idx % (q + 1) == 0) ? 1.0 : 0.0;
  __shared__ unsigned s_nrot2;
  if (threadIdx.x == 0) s_nrot2 = 0;
  __syncthreads();
  if (q < 2) {
    if (threadIdx.x == 0) *sweeps_out = 0;
    return 0.0;
  }
  const int qq = q + (q & 1);
  const int m1 = qq - 1;
  const double tol2 = tol * tol;
  unsigned nrot = 0;
  int sweeps = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    ++sweeps;
    bool rot = false;
    for (int round = 0; round < m1; ++round) {
      if (p <= 32)
        rot |= jacobi_round<4>(W, p, q, J, qq, m1, round, tol2, nrot);
      else if (p <= 64)
        rot |= jacobi_round<8>(W, p, q, J, qq, m1, round, tol2, nrot);
      else if (p <= 128)
        rot |= jacobi_round<16>(W, p, q, J, qq, m1, round, tol2, nrot);
      else
        rot |= jacobi_round<32>(W, p, q, J, qq, m1, round, tol2, nrot);
      __syncthreads();
    }
    if (!__syncthreads_or(rot)) break;
  }
  nrot += __shfl_xor_sync(0xffffffffu, nrot, 16);
  nrot += __shfl_xor_sync(0xffffffffu, nrot, 8);
  nrot += __shfl_xor_sync(0xffffffffu, nrot, 4);
  nrot += __shfl_xor_sync(0xffffffffu, nrot, 2);
  nrot += __shfl_xor_sync(0xffffffffu, nrot, 1);
  if (lane == 0 && nrot) atomicAdd(&s_nrot2, nrot);
  __syncthreads();
  if (threadIdx.x == 0) *sweeps_out = sweeps;
  return (double)sweeps * (0.5 * q * (q - 1)) * 6.0 * p + (double)s_nrot2 * 6.0 * (p + q);
}

// Rank-revealing truncated SVD of W (p x q, ld p, destroyed; q <= 128) with the
// contract of cta_rrqr_svd, except that pivoting is virtual: step s factors the
// physical column phys[s] (no column swaps) and every warp re-derives the pivot
// (largest remaining trailing norm, lowest index on ties) and the reflector
// scalars redundantly, so one step costs one barrier.  G (q x kq) is (R P^T)^T
// in physical column order, as cta_rrqr_svd returns it; the Q of the core is
// applied with cta_apply_q_map(W, ..., phys, ...).  cn holds 2q doubles: the
// trailing norms are double-buffered so a warp that runs ahead into the update
// never changes what a slower warp is still reading for its pivot choice.
__device__ RS cta_rrqr_svd2(double* W, int p, int q, double eps, double* tau, int* phys, double* cn,
                            int* stepof, double* G, double* J, double* s_sig, int* s_ord, int path,
                            long long* tclk) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double flops = 0.0;
  for (int j = w; j < q; j += nw) {
    const double* c = W + (size_t)j * p;
    double s = 0.0;
    for (int i = lane; i < p; i += 32) s += c[i] * c[i];
    s = warp_sum(s);
    if (lane == 0) {
      cn[j] = s;
      stepof[j] = INT_MAX;
    }
  }
  __syncthreads();
  flops += 2.0 * p * q;
  double thresh;
  {
    double a = 0.0;
    for (int j = lane; j < q; j += 32) a = fmax(a, cn[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    thresh = 1e-3 * eps * sqrt(fmax(a, 0.0));
  }
  unsigned long long ch[2] = {0ull, 0ull};  // chosen columns (identical in every thread)
  const int kmax = min(p, q);
  double pt = 0.0, pinv = 0.0, pbeta = 0.0;
  int pj = -1, k = 0;
  for (; k < kmax; ++k) {
    // (a) pivot and trailing Frobenius norm, redundantly in every warp
    const double* cnr = cn + (k & 1) * q;
    double* cnw = cn + ((k + 1) & 1) * q;
    double best = -1.0, resid = 0.0;
    int jb = -1;
    for (int j = lane; j < q; j += 32) {
      if ((ch[j >> 6] >> (j & 63)) & 1ull) continue;
      const double v = cnr[j];
      resid += v;
      if (v > best) {
        best = v;
        jb = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int j2 = __shfl_xor_sync(0xffffffffu, jb, o);
      resid += __shfl_xor_sync(0xffffffffu, resid, o);
      if (b2 > best || (b2 == best && j2 >= 0 && (jb < 0 || j2 < jb))) {
        best = b2;
        jb = j2;
      }
    }
    // lagged normalisation of the previous pivot column
    if (k > 0 && w == nw - 1) {
      double* xp = W + (size_t)pj * p;
      for (int i = k + lane; i < p; i += 32) xp[i] = (pt == 0.0) ? 0.0 : xp[i] * pinv;
      if (lane == 0) {
        xp[k - 1] = pbeta;
        tau[k - 1] = pt;
        phys[k - 1] = pj;
        stepof[pj] = k - 1;
      }
    }
    if (!(sqrt(resid) > thresh) || jb < 0) break;
    const int jm = jb;
    ch[jm >> 6] |= 1ull << (jm & 63);
    const double* x = W + (size_t)jm * p;
    double tail2 = 0.0;
    for (int i = k + 1 + lane; i < p; i += 32) tail2 += x[i] * x[i];
    tail2 = warp_sum(tail2);
    double t, beta, inv;
    hh_scalars(x[k], tail2, t, beta, inv);
    // (b) apply H_k to the remaining columns (physical j = w mod nw) and refresh
    // their trailing norms (rows > k)
    {
      int js[4], nj = 0;
      for (int j = w; j < q; j += nw) {
        const bool skip = (ch[j >> 6] >> (j & 63)) & 1ull;
        if (!skip) js[nj++] = j;
        if (nj == 4 || (j + nw >= q && nj > 0)) {
          double* c[4];
          bool on[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            on[u] = u < nj;
            c[u] = W + (size_t)(on[u] ? js[u] : js[0]) * p;
          }
          double s[4] = {0.0, 0.0, 0.0, 0.0};
          if (t != 0.0) {
            for (int i = k + 1 + lane; i < p; i += 32) {
              const double v = x[i];
#pragma unroll
              for (int u = 0; u < 4; ++u) s[u] += v * c[u][i];
            }
            warp_sum_n<4>(s);
#pragma unroll
            for (int u = 0; u < 4; ++u) s[u] = (c[u][k] + inv * s[u]) * t;
          }
          double s2[4] = {0.0, 0.0, 0.0, 0.0};
          for (int i = k + 1 + lane; i < p; i += 32) {
            const double v = x[i] * inv;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (!on[u]) continue;
              const double y = (t != 0.0) ? c[u][i] - s[u] * v : c[u][i];
              c[u][i] = y;
              s2[u] += y * y;
            }
          }
          warp_sum_n<4>(s2);
          __syncwarp();
          if (lane == 0)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (on[u]) {
                if (t != 0.0) c[u][k] -= s[u];
                cnw[js[u]] = s2[u];
              }
          __syncwarp();
          nj = 0;
        }
      }
    }
    flops += 6.0 * (p - k) * (q - k);
    pt = t;
    pinv = inv;
    pbeta = beta;
    pj = jm;
    __syncthreads();
  }
  if (k > 0 && k == kmax && w == nw - 1) {  // ran to the end: normalise the last pivot
    double* xp = W + (size_t)pj * p;
    for (int i = k + lane; i < p; i += 32) xp[i] = (pt == 0.0) ? 0.0 : xp[i] * pinv;
    if (lane == 0) {
      xp[k - 1] = pbeta;
      tau[k - 1] = pt;
      phys[k - 1] = pj;
      stepof[pj] = k - 1;
    }
  }
  __syncthreads();
  const int kq = k;
  if (tclk) stage_add(path, 2, *tclk);
  // G = (R P^T)^T : q x kq in physical column order
  for (int e = threadIdx.x; e < q * kq; e += blockDim.x) {
    const int c = e % q, i = e / q;
    const int sc = stepof[c];
    G[(size_t)i * q + c] = (sc == INT_MAX || i <= sc) ? W[(size_t)c * p + i] : 0.0;
  }
  __syncthreads();
  __shared__ int s_sweeps2;
  flops += cta_jacobi2(G, q, kq, J, &s_sweeps2, fmax(1e-15, fmin(1e-10, 1e-4 * eps)));
  if (tclk) {
    stage_add(path, 3, *tclk);
    if (d_hist_on && threadIdx.x == 0) {
      atomicAdd(&d_stage_sweeps[path], (unsigned long long)s_sweeps2);
      atomicAdd(&d_stage_jac[path], 1ull);
    }
  }
  for (int c = w; c < kq; c += nw) {
    const double* gc = G + (size_t)c * q;
    double s = 0.0;
    for (int i = lane; i < q; i += 32) s += gc[i] * gc[i];
    s = warp_sum(s);
    if (lane == 0) s_sig[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kq; c += blockDim.x) {
    const double sc = s_sig[c];
    int rk = 0;
    for (int d = 0; d < kq; ++d) rk += (s_sig[d] > sc) || (s_sig[d] == sc && d < c);
    s_ord[rk] = c;
  }
  __syncthreads();
  const double smax = kq > 0 ? s_sig[s_ord[0]] : 0.0;
  int keep = 0;
  while (keep < kq && s_sig[s_ord[keep]] > eps * smax && s_sig[s_ord[keep]] > 0.0) ++keep;
  return RS{kq, keep, flops};
}

// Register-resident Householder QR of A (mm x r, ld lda, shared memory) for
// mm <= 32*RT, r <= 16*CT, 512 threads: lane l holds rows l + 32*ii, warp w
// holds columns w + 16*cc.  Step k: every warp reads the published reflector
// v_k (explicit unit head and zeros above it, so the loops carry no bounds),
// forms its dot products with one interleaved warp reduction and updates its
// columns; the warp owning column k+1 then forms and publishes v_{k+1}.  One
// barrier per column; A is written back (R above, reflectors below) at the end.
template <int RT, int CT>
__device__ void reg_qr(double* A, int mm, int lda, int r, double* tau, double* vbuf, double* sbuf) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = 16;
  double a[CT][RT];
#pragma unroll
  for (int cc = 0; cc < CT; ++cc)
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      const int j = w + NW * cc, i = lane + 32 * ii;
      a[cc][ii] = (j < r && i < mm) ? A[(size_t)j * lda + i] : 0.0;
    }
  const int kmax = min(mm, r);
  // the owner warp of column k (w == k % NW) forms and publishes reflector k
  auto publish = [&](int k) {
    const int cs = k / NW;
    double x[RT];
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      x[ii] = 0.0;
#pragma unroll
      for (int cc = 0; cc < CT; ++cc)
        if (cc == cs) x[ii] = a[cc][ii];
    }
    double tail = 0.0, xk = 0.0;
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      const int i = lane + 32 * ii;
      if (i > k) tail += x[ii] * x[ii];
      if (ii == (k >> 5)) xk = x[ii];
    }
    tail = warp_sum(tail);
    const double c0 = __shfl_sync(0xffffffffu, xk, k & 31);
    double t, beta, inv;
    hh_scalars(c0, tail, t, beta, inv);
    double* vb = vbuf + (size_t)(k & 1) * (32 * RT);
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      const int i = lane + 32 * ii;
      const double v = (i > k) ? ((t == 0.0) ? 0.0 : x[ii] * inv) : (i == k ? 1.0 : 0.0);
      vb[i] = v;
      const double st = (i > k) ? v : (i == k ? beta : x[ii]);
#pragma unroll
      for (int cc = 0; cc < CT; ++cc)
        if (cc == cs) a[cc][ii] = st;
    }
    if (lane == 0) {
      sbuf[k & 1] = t;
      tau[k] = t;
    }
  };
  if (kmax > 0 && w == 0) publish(0);
  __syncthreads();
  for (int k = 0; k < kmax; ++k) {
    const double t = sbuf[k & 1];
    if (t != 0.0) {
      const double* vb = vbuf + (size_t)(k & 1) * (32 * RT);
      double vr[RT];
#pragma unroll
      for (int ii = 0; ii < RT; ++ii) vr[ii] = vb[lane + 32 * ii];
      double d[CT];
#pragma unroll
      for (int cc = 0; cc < CT; ++cc) {
        d[cc] = 0.0;
        if (w + NW * cc > k)
#pragma unroll
          for (int ii = 0; ii < RT; ++ii) d[cc] += vr[ii] * a[cc][ii];
      }
      warp_sum_n<CT>(d);
#pragma unroll
      for (int cc = 0; cc < CT; ++cc) {
        if (w + NW * cc <= k) continue;
        const double s = d[cc] * t;
#pragma unroll
        for (int ii = 0; ii < RT; ++ii) a[cc][ii] -= s * vr[ii];
      }
    }
    if (k + 1 < kmax && w == (k + 1) % NW) publish(k + 1);
    __syncthreads();
  }
#pragma unroll
  for (int cc = 0; cc < CT; ++cc)
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      const int j = w + NW * cc, i = lane + 32 * ii;
      if (j < r && i < mm) A[(size_t)j * lda + i] = a[cc][ii];
    }
  __syncthreads();
}

// dispatch on (rows, columns); returns false when the shape is not covered
__device__ __forceinline__ bool reg_qr_any(double* A, int mm, int lda, int r, double* tau, double* vbuf,
                                           double* sbuf) {
  if (blockDim.x != 512 || r > 64 || mm > 512) return false;
  const int ct = (r + 15) / 16;
  if (mm > 256) {
    if (ct > 2) return false;
    if (ct == 1) reg_qr<16, 1>(A, mm, lda, r, tau, vbuf, sbuf);
    else reg_qr<16, 2>(A, mm, lda, r, tau, vbuf, sbuf);
    return true;
  }
  if (mm <= 128) {
    switch (ct) {
      case 1: reg_qr<4, 1>(A, mm, lda, r, tau, vbuf, sbuf); return true;
      case 2: reg_qr<4, 2>(A, mm, lda, r, tau, vbuf, sbuf); return true;
      case 3: reg_qr<4, 3>(A, mm, lda, r, tau, vbuf, sbuf); return true;
      default: reg_qr<4, 4>(A, mm, lda, r, tau, vbuf, sbuf); return true;
    }
  }
  switch (ct) {
    case 1: reg_qr<8, 1>(A, mm, lda, r, tau, vbuf, sbuf); return true;
    case 2: reg_qr<8, 2>(A, mm, lda, r, tau, vbuf, sbuf); return true;
    case 3: reg_qr<8, 3>(A, mm, lda, r, tau, vbuf, sbuf); return true;
    default: reg_qr<8, 4>(A, mm, lda, r, tau, vbuf, sbuf); return true;
  }
}
