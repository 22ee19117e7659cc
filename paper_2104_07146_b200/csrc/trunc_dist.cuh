// Large-block recompression with the stacked factors resident in REGISTERS of
// an 8-CTA cluster (included by truncate.cu after the pair path).
//
// Cluster ranks 0-3 hold row slices of [U | aP], ranks 4-7 row slices of
// [V | Q] (kDistS CTAs per side, slice s = rows [s*ms, (s+1)*ms)).  Inside a CTA
// lanes run over the slice's rows and warps over columns, as in reg_qr.
// Householder step k (both sides in lockstep, two cluster barriers):
//   X_k  every CTA reads the kDistS partial tail norms / heads of column k
//        through DSMEM and derives the same reflector scalars; the owner warp
//        normalises its slice of v_k and shares it in shared memory;
//        partial dots v_k . a_j of every local column go to shared memory;
//   Y_k  every CTA sums the kDistS partial dots (DSMEM) and updates its
//        columns; the owner of column k+1 posts its partial tail norm.
// The side leaders (ranks 0 and 4, whose slices hold the R factors) then form
// the core R_u R_v^T, take its rank-revealing SVD (identical arithmetic on
// both), and each side applies its Q in WY form: the Gram of the reflectors
// is summed from per-slice partials, T and Z = T Y_1^T E0 are built on the
// leader, and every CTA writes its own rows of [E0; 0] - Y Z.
#pragma once

constexpr int kDistS = 4;  // CTAs per side

struct DistShared {
  double P[2][2];          // partial tail norm^2 and head of the pending column
  double D[2][64];         // partial dot products per column
  double vb[2][512];       // this slice of the current reflector
  double tau[64];          // reflector scalars (identical in every CTA of a side)
  int keep, kq, ok;
};

// shared-memory doubles of the dynamic region: slice (ld ms|1) + 5 r x r + 8 r
__host__ __device__ __forceinline__ size_t dist_smem_doubles(int ms, int r) {
  return (size_t)(ms | 1) * r + 5 * (size_t)r * r + 8 * (size_t)r + 16;
}

template <int RT, int CT>
__device__ void lr_update_dist(cg::cluster_group& cl, const TruncItem& it, double eps, int* err, int r0,
                               int r, int add, double* sm, DistShared& ds, double* s_sig, int* s_ord) {
  const int rank = (int)cl.block_rank();
  const int side = rank / kDistS, srank = rank % kDistS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = 16;
  const int m = it.m, n = it.n;
  const int mm = side ? n : m;
  const int ms = (max(m, n) + kDistS - 1) / kDistS;  // slice height (same on both sides)
  const int lo = srank * ms;
  const int kme = min(mm, r), ku = min(m, r), kv = min(n, r);
  const int ksteps = max(ku, kv);
  const long long t0 = clock64();
  double* X = side ? it.V : it.U;
  // ---- stage this slice (global -> registers, coalesced over rows)
  double a[CT][RT];
#pragma unroll
  for (int cc = 0; cc < CT; ++cc)
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      const int j = w + NW * cc, il = lane + 32 * ii, i = lo + il;
      double v = 0.0;
      if (j < r && il < ms && i < mm) {
        if (j < r0) {
          v = X[(size_t)j * mm + i];
        } else if (side == 0) {
          const int pi = i - it.pro;
          v = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)(j - r0) * it.ldp + pi] : 0.0;
        } else {
          const int qi = i - it.qro;
          v = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)(j - r0) * it.ldq + qi] : 0.0;
        }
      }
      a[cc][ii] = v;
    }
  // owner warp of column k posts this slice's tail norm^2 (rows > k) and head
  auto post = [&](int k) {
    const int cs = k / NW;
    double tail = 0.0, xk = 0.0;
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      double x = 0.0;
#pragma unroll
      for (int cc = 0; cc < CT; ++cc)
        if (cc == cs) x = a[cc][ii];
      const int i = lo + lane + 32 * ii;
      if (i > k) tail += x * x;
      if (i == k) xk = x;
    }
    tail = warp_sum(tail);
    xk = warp_sum(xk);  // at most one lane holds row k
    if (lane == 0) {
      ds.P[k & 1][0] = tail;
      ds.P[k & 1][1] = xk;
    }
  };
  if (ku > 0 && w == 0) post(0);
  for (int k = 0; k < ksteps; ++k) {
    cl.sync();  // X_k
    const bool act = k < kme;
    double t = 0.0;
    if (act) {
      double tail = 0.0, c0 = 0.0;
#pragma unroll
      for (int s = 0; s < kDistS; ++s) {
        const double* Pr = cl.map_shared_rank(&ds.P[k & 1][0], side * kDistS + s);
        tail += Pr[0];
        c0 += Pr[1];
      }
      double beta, inv;
      hh_scalars(c0, tail, t, beta, inv);
      if (w == k % NW) {  // normalise this slice of column k: v below, beta at row k
        const int cs = k / NW;
#pragma unroll
        for (int ii = 0; ii < RT; ++ii) {
          const int il = lane + 32 * ii, i = lo + il;
          double x = 0.0;
#pragma unroll
          for (int cc = 0; cc < CT; ++cc)
            if (cc == cs) x = a[cc][ii];
          const double v = (i > k) ? ((t == 0.0) ? 0.0 : x * inv) : (i == k ? 1.0 : 0.0);
          if (il < 512) ds.vb[k & 1][il] = (il < ms) ? v : 0.0;
          const double st = (i > k) ? v : (i == k ? beta : x);
#pragma unroll
          for (int cc = 0; cc < CT; ++cc)
            if (cc == cs) a[cc][ii] = st;
        }
      }
      if (threadIdx.x == 0) ds.tau[k] = t;
    }
    __syncthreads();
    double vr[RT];
    if (act && t != 0.0) {
#pragma unroll
      for (int ii = 0; ii < RT; ++ii) vr[ii] = ds.vb[k & 1][lane + 32 * ii];
      double d[CT];
#pragma unroll
      for (int cc = 0; cc < CT; ++cc) {
        d[cc] = 0.0;
#pragma unroll
        for (int ii = 0; ii < RT; ++ii) d[cc] += vr[ii] * a[cc][ii];
      }
      warp_sum_n<CT>(d);
      if (lane == 0)
#pragma unroll
        for (int cc = 0; cc < CT; ++cc) {
          const int j = w + NW * cc;
          if (j > k && j < r) ds.D[k & 1][j] = d[cc];
        }
    }
    cl.sync();  // Y_k
    if (act && t != 0.0) {
#pragma unroll
      for (int cc = 0; cc < CT; ++cc) {
        const int j = w + NW * cc;
        if (j <= k || j >= r) continue;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kDistS; ++q) s += cl.map_shared_rank(&ds.D[k & 1][0], side * kDistS + q)[j];
        s *= t;
#pragma unroll
        for (int ii = 0; ii < RT; ++ii) a[cc][ii] -= s * vr[ii];
      }
    }
    if (k + 1 < kme && w == (k + 1) % NW) post(k + 1);
  }
  long long tc = t0;
  if (rank == 0) stage_add(2, 1, tc);
  // ---- slice to shared memory: Y (reflectors below the diagonal), R above
  const int lds = ms | 1;
  double* Y = sm;                            // ms x r (ld lds)
  double* Sp = Y + (size_t)lds * r;          // partial Gram, r x r
  double* Ro = Sp + (size_t)r * r;           // leader: other R, later G, later X1; others: Z copy
  double* C = Ro + (size_t)r * r;            // leader: core, later T
  double* J = C + (size_t)r * r;             // leader: Jacobi X, later S, later Z
  double* E0 = J + (size_t)r * r;            // leader: kme x keep
  double* tau_c = E0 + (size_t)r * r;        // r
  double* cn = tau_c + r;                    // 2r
  int* phys = reinterpret_cast<int*>(cn + 2 * r);
  int* stepof = phys + r;
#pragma unroll
  for (int cc = 0; cc < CT; ++cc)
#pragma unroll
    for (int ii = 0; ii < RT; ++ii) {
      const int j = w + NW * cc, il = lane + 32 * ii;
      if (j < r && il < ms) Y[(size_t)j * lds + il] = a[cc][ii];
    }
  cl.sync();  // Z0: every slice stored
  const bool leader = srank == 0;
  RS rs{0, 0, 0.0};
  if (leader) {
    // other side's R (ko x r) through DSMEM; the leader slice holds rows [0, ms) >= r
    const int ko = side ? ku : kv;
    const double* Yo = cl.map_shared_rank(Y, (side ^ 1) * kDistS);
    for (int e = threadIdx.x; e < ko * r; e += blockDim.x) {
      const int i = e % ko, l = e / ko;
      Ro[e] = (i <= l) ? Yo[(size_t)l * lds + i] : 0.0;
    }
    __syncthreads();
    const double* Ru = side ? Ro : Y;
    const double* Rv = side ? Y : Ro;
    const int ldu = side ? ku : lds, ldv = side ? lds : kv;
    for (int idx = threadIdx.x; idx < ku * kv; idx += blockDim.x) {
      const int i = idx % ku, j = idx / ku;
      double s = 0.0;
      for (int l = max(i, j); l < r; ++l) s += Ru[(size_t)l * ldu + i] * Rv[(size_t)l * ldv + j];
      C[(size_t)j * ku + i] = s;
    }
    __syncthreads();
    rs = cta_rrqr_svd2(C, ku, kv, eps, tau_c, phys, cn, stepof, Ro, J, s_sig, s_ord, 2,
                       rank == 0 ? &tc : nullptr);
    const int keep = rs.keep, kq = rs.kq;
    if (keep <= it.cap) {
      if (side == 0) {  // U_core = Q_core [J S; 0]
        for (int idx = threadIdx.x; idx < ku * keep; idx += blockDim.x) {
          const int i = idx % ku, c = idx / ku, src = s_ord[c];
          E0[idx] = i < kq ? J[(size_t)src * kq + i] * s_sig[src] : 0.0;
        }
        __syncthreads();
        cta_apply_q_map(C, ku, ku, kq, tau_c, phys, E0, keep);
      } else {
        for (int idx = threadIdx.x; idx < kv * keep; idx += blockDim.x) {
          const int i = idx % kv, c = idx / kv, src = s_ord[c];
          E0[idx] = Ro[(size_t)src * kv + i] / s_sig[src];
        }
      }
    }
    if (threadIdx.x == 0) {
      ds.keep = keep;
      ds.kq = kq;
      ds.ok = keep <= it.cap;
      if (keep > it.cap && side == 0) atomicOr(err, 4);
    }
  }
  // partial Gram of this slice's reflectors: Sp(l, q) for l < q < kme
  {
    const int np = kme * (kme - 1) / 2;
    for (int pb = 4 * w; pb < np; pb += 4 * NW) {
      int ls[4], qs[4];
      double s[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = min(pb + u, max(np - 1, 0));
        int q = (int)((1.0 + sqrt(1.0 + 8.0 * p)) * 0.5);
        while (q * (q - 1) / 2 > p) --q;
        while ((q + 1) * q / 2 <= p) ++q;
        ls[u] = p - q * (q - 1) / 2;
        qs[u] = q;
        s[u] = 0.0;
      }
      for (int il = lane; il < ms; il += 32) {
        const int i = lo + il;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (i < qs[u]) continue;
          const double yl = Y[(size_t)ls[u] * lds + il];
          const double yq = (i == qs[u]) ? 1.0 : Y[(size_t)qs[u] * lds + il];
          s[u] += yl * yq;
        }
      }
      warp_sum_n<4>(s);
      if (lane == 0)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (pb + u < np) Sp[(size_t)qs[u] * kme + ls[u]] = s[u];
    }
  }
  cl.sync();  // Z1
  const int keep = cl.map_shared_rank(&ds.keep, side * kDistS)[0];
  const int okk = cl.map_shared_rank(&ds.ok, side * kDistS)[0];
  if (leader && okk) {
    // S = sum of the slices' partial Grams (into J), then T (into C)
    double* S = J;
    for (int e = threadIdx.x; e < kme * kme; e += blockDim.x) {
      const int l = e % kme, q = e / kme;
      if (l >= q) continue;
      double s = 0.0;
#pragma unroll
      for (int t2 = 0; t2 < kDistS; ++t2) s += cl.map_shared_rank(Sp, side * kDistS + t2)[(size_t)q * kme + l];
      S[(size_t)q * kme + l] = s;
    }
    __syncthreads();
    double* T = C;
    for (int q = 0; q < kme; ++q) {
      const double tq = ds.tau[q];
      for (int i = threadIdx.x; i < q; i += blockDim.x) {
        double s = 0.0;
        for (int l = i; l < q; ++l) s += T[(size_t)l * kme + i] * S[(size_t)q * kme + l];
        T[(size_t)q * kme + i] = -tq * s;
      }
      if (threadIdx.x == 0) T[(size_t)q * kme + q] = tq;
      for (int i = q + 1 + threadIdx.x; i < kme; i += blockDim.x) T[(size_t)q * kme + i] = 0.0;
      __syncthreads();
    }
    // X1 = Y1^T E0 (into Ro), Z = T X1 (into J)
    double* X1 = Ro;
    for (int e = threadIdx.x; e < kme * keep; e += blockDim.x) {
      const int l = e % kme, cc = e / kme;
      const double* ec = E0 + (size_t)cc * kme;
      double s = ec[l];
      for (int i = l + 1; i < kme; ++i) s += Y[(size_t)l * lds + i] * ec[i];
      X1[e] = s;
    }
    __syncthreads();
    double* Z = J;
    for (int e = threadIdx.x; e < kme * keep; e += blockDim.x) {
      const int l = e % kme, cc = e / kme;
      const double* xc = X1 + (size_t)cc * kme;
      double s = 0.0;
      for (int j = l; j < kme; ++j) s += T[(size_t)j * kme + l] * xc[j];
      Z[e] = s;
    }
  }
  cl.sync();  // Z2: Z ready on the leaders
  if (okk) {
    const double* Z = leader ? J : Ro;
    if (!leader) {
      const double* Zr = cl.map_shared_rank(J, side * kDistS);
      for (int e = threadIdx.x; e < kme * keep; e += blockDim.x) Ro[e] = Zr[e];
      __syncthreads();
    }
    // own rows of [E0; 0] - Y Z
    for (int e = threadIdx.x; e < ms * keep; e += blockDim.x) {
      const int il = e % ms, cc = e / ms, i = lo + il;
      if (i >= mm) continue;
      const double* zc = Z + (size_t)cc * kme;
      double s = 0.0;
      if (i < kme) s = E0[(size_t)cc * kme + i] - zc[i];  // only the leader slice has i < kme
      const int lmax = min(i, kme);
      for (int l = 0; l < lmax; ++l) s -= Y[(size_t)l * lds + il] * zc[l];
      X[(size_t)cc * mm + i] = s;
    }
  }
  cl.sync();  // Z3: outputs written, leaders' buffers free
  if (rank == 0 && threadIdx.x == 0 && okk) {
    *it.rank = keep;
    if (it.compact) *it.compact = keep;
    const double fl = qr_flops(m, r) + qr_flops(n, r) + (double)ku * kv * r + rs.flops +
                      4.0 * keep * ((double)m * ku + (double)n * kv + (double)ku * ds.kq);
    atomicAdd(&d_cnt_trunc, fl);
    atomicAdd(&d_cnt_titems, 1.0);
  }
  if (rank == 0) {
    stage_add(2, 4, tc);
    hist_add(2, m, n, r, t0);
  }
  (void)add;
  cl.sync();
}

// covered shapes: slice height ms = ceil(max(m,n)/4) <= 32*RT, r <= 16*CT,
// RT*CT <= 32 registers of factor per thread, the leader slice holds all of R
__device__ __forceinline__ bool dist_fits(int m, int n, int r, int cap_dbl) {
  const int ms = (max(m, n) + kDistS - 1) / kDistS;
  if (r > 64 || ms < r || ms > 512) return false;
  const int rt = (ms + 31) / 32 <= 4 ? 4 : (ms + 31) / 32 <= 8 ? 8 : 16;
  const int ct = (r + 15) / 16;
  if (rt * ct > 16) return false;
  return dist_smem_doubles(ms, r) <= (size_t)cap_dbl;
}

__device__ __forceinline__ void lr_update_dist_any(cg::cluster_group& cl, const TruncItem& it, double eps,
                                                   int* err, int r0, int r, int add, double* sm,
                                                   DistShared& ds, double* s_sig, int* s_ord) {
  const int ms = (max(it.m, it.n) + kDistS - 1) / kDistS;
  const int ct = (r + 15) / 16;
  if ((ms + 31) / 32 <= 4) {
    switch (ct) {
      case 1: lr_update_dist<4, 1>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord); return;
      case 2: lr_update_dist<4, 2>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord); return;
      case 3: lr_update_dist<4, 3>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord); return;
      default: lr_update_dist<4, 4>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord); return;
    }
  }
  if ((ms + 31) / 32 <= 8) {
    if (ct == 1) lr_update_dist<8, 1>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord);
    else lr_update_dist<8, 2>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord);
    return;
  }
  lr_update_dist<16, 1>(cl, it, eps, err, r0, r, add, sm, ds, s_sig, s_ord);
}
