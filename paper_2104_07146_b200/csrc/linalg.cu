// Batched FP64 building blocks of the H-factorization (see linalg.cuh).
//   GEMM      hblk::apply / multiply / add_low_rank dense update (hblock.cpp:46-92,181-184)
//   TRSM      solveInPlace variants (hfactor.cpp:78,92,109,201,205)
//   leaf LDL  dense_ldl_leaf / dense_cholesky_leaf (hfactor.cpp:22-73)
#include <climits>

#include "common.cuh"
#include "linalg.cuh"

namespace hmgp_gpu {

// algorithmic flop counters (one atomic per item; read by bench.py)
__device__ double d_cnt_gemm, d_cnt_trsm, d_cnt_leaf;

void linalg_counters_read_reset(double* g, double* t, double* l) {
  double z = 0.0;
  HMGP_CUDA(cudaMemcpyFromSymbol(g, d_cnt_gemm, 8));
  HMGP_CUDA(cudaMemcpyFromSymbol(t, d_cnt_trsm, 8));
  HMGP_CUDA(cudaMemcpyFromSymbol(l, d_cnt_leaf, 8));
  HMGP_CUDA(cudaMemcpyToSymbol(d_cnt_gemm, &z, 8));
  HMGP_CUDA(cudaMemcpyToSymbol(d_cnt_trsm, &z, 8));
  HMGP_CUDA(cudaMemcpyToSymbol(d_cnt_leaf, &z, 8));
}

// ----------------------------------------------------------------- GEMM ---
// FP64 tensor cores (DMMA.8x8x4, mma.sync.m8n8k4.f64).  64x64 output tile per
// CTA iteration, k-slabs of 16 staged in shared memory, 8 warps as 2 x 4, each
// warp a 32x16 sub-tile = 4 x 2 DMMA accumulators (16 doubles per thread).
// Fragments (PTX m8n8k4 .f64): A a0 at (row lane/4, k lane%4); B b0 at
// (k lane%4, col lane/4); C c0,c1 at (row lane/4, col 2*(lane%4) + {0,1}).
// Dimensions may live on device.
constexpr int GT = 64, GK = 16;

__device__ void gemm_item(const GemmItem& it, int tile0, int tstride, bool count);

__global__ void __launch_bounds__(256) k_gemm(const GemmItem* __restrict__ items) {
  gemm_item(items[blockIdx.x], blockIdx.y, gridDim.y, blockIdx.y == 0);
}

// One CTA per target: its GEMM updates items[off[b] .. off[b+1]) in order.
__global__ void __launch_bounds__(256) k_gemm_seq(const GemmItem* __restrict__ items,
                                                  const int* __restrict__ off) {
  for (int i = off[blockIdx.x]; i < off[blockIdx.x + 1]; ++i) {
    gemm_item(items[i], 0, 1, true);
    __syncthreads();
  }
}

void launch_gemm_seq(const GemmItem* d_items, const int* d_off, int targets, cudaStream_t st) {
  if (targets <= 0) return;
  k_gemm_seq<<<targets, 256, 0, st>>>(d_items, d_off);
  HMGP_LAUNCH_CHECK();
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ void gemm_item(const GemmItem& it, int tile0, int tstride, bool count) {
  const int M = it.M.get(), N = it.N.get(), K = it.K.get();
  if (M <= 0 || N <= 0) return;
  if (count && threadIdx.x == 0) atomicAdd(&d_cnt_gemm, 2.0 * M * N * K);
  const int tm = (M + GT - 1) / GT, tn = (N + GT - 1) / GT;
  // k-slabs are double-buffered in shared memory: the global loads of slab s+1 are
  // issued into registers before the DMMA work on slab s and stored afterwards, so
  // their latency overlaps the math and a slab costs ONE barrier.  The summation
  // order of every output element is unchanged (k ascending).
  __shared__ double sA[2][GK][GT + 1];
  __shared__ double sB[2][GK][GT + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = (w >> 2) * 32, wc = (w & 3) * 16;  // warp sub-tile origin
  const int fr = lane >> 2, fk = lane & 3;           // fragment row / k index
  // No split-K inside an item and no atomics: every output element is written
  // by exactly one CTA with a fixed summation order (bit-reproducible).  Long
  // contractions are split by the host into K-range items writing separate
  // slabs, summed in a fixed order by k_slab_sum.
  const int T = tm * tn;
  const int tbeg = tile0, tstep = tstride, kbeg = 0, kend = K;
  constexpr int kPer = GK * GT / 256;  // elements of each operand slab per thread
  // this thread's element e -> (kk, ii) of the A slab and (kk, jj) of the B slab
  int akk[kPer], aii[kPer], bkk[kPer], bjj[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = threadIdx.x + q * 256;
    if (!it.ta) {
      aii[q] = e % GT;
      akk[q] = e / GT;
    } else {
      akk[q] = e % GK;
      aii[q] = e / GK;
    }
    if (!it.tb) {
      bkk[q] = e % GK;
      bjj[q] = e / GK;
    } else {
      bjj[q] = e % GT;
      bkk[q] = e / GT;
    }
  }
  for (int tile = tbeg; tile < T; tile += tstep) {
    const int i0 = (tile % tm) * GT, j0 = (tile / tm) * GT;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double ra[kPer], rb2[kPer];
    auto fetch = [&](int k0) {
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int gi = i0 + aii[q], gk = k0 + akk[q];
        ra[q] = (gi < M && gk < kend)
                    ? (it.ta ? it.A[(size_t)gi * it.lda + gk] : it.A[(size_t)gk * it.lda + gi])
                    : 0.0;
        const int gj = j0 + bjj[q], gk2 = k0 + bkk[q];
        rb2[q] = (gj < N && gk2 < kend)
                     ? (it.tb ? it.B[(size_t)gk2 * it.ldb + gj] : it.B[(size_t)gj * it.ldb + gk2])
                     : 0.0;
      }
    };
    auto stash = [&](int buf) {
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        sA[buf][akk[q]][aii[q]] = ra[q];
        sB[buf][bkk[q]][bjj[q]] = rb2[q];
      }
    };
    __syncthreads();  // the previous tile's readers are done with both buffers
    if (kbeg < kend) {
      fetch(kbeg);
      stash(0);
    }
    __syncthreads();
    int buf = 0;
    for (int k0 = kbeg; k0 < kend; k0 += GK, buf ^= 1) {
      const bool more = k0 + GK < kend;
      if (more) fetch(k0 + GK);
#pragma unroll
      for (int ks = 0; ks < GK; ks += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) af[rb] = sA[buf][ks + fk][wr + rb * 8 + fr];
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) bf[cb] = sB[buf][ks + fk][wc + cb * 8 + fr];
#pragma unroll
        for (int rb = 0; rb < 4; ++rb)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb) dmma884(acc[rb][cb], af[rb], bf[cb]);
      }
      if (more) stash(buf ^ 1);  // nobody reads buf^1 during this slab
      __syncthreads();
    }
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = j0 + wc + cb * 8 + 2 * fk + h;
        if (gj >= N) continue;
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int gi = i0 + wr + rb * 8 + fr;
          if (gi >= M) continue;
          const double v = acc[rb][cb][h];
          if (it.atomic == 2)
            it.C[(size_t)gj * it.ldc + gi] = it.alpha * v;
          else
            it.C[(size_t)gj * it.ldc + gi] += it.alpha * v;
        }
      }
  }
}

void launch_gemm(const GemmItem* d_items, int count, int max_tiles, cudaStream_t st) {
  if (count <= 0) return;
  const int ty = max(1, min(max_tiles, 128));
  k_gemm<<<dim3(count, ty), 256, 0, st>>>(d_items);
  HMGP_LAUNCH_CHECK();
}

// ----------------------------------------------------------------- TRSM ---
// Left: one warp per right-hand-side column, lanes over rows (coalesced).
__global__ void k_trsm_left(const TrsmLItem* __restrict__ items) {
  const TrsmLItem it = items[blockIdx.x];
  const int cols = it.cols.get();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int b = it.b;
  if (blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&d_cnt_trsm, (double)b * b * cols);
  for (int c = blockIdx.y * nw + w; c < cols; c += gridDim.y * nw) {
    double* x = it.M + (size_t)c * it.ldm;
    if (!it.trans) {
      for (int j = 0; j < b; ++j) {
        const double xj = x[j] / it.L[(size_t)j * it.ldl + j];
        __syncwarp();
        if (lane == 0) x[j] = xj;
        const double* lc = it.L + (size_t)j * it.ldl;
        for (int i = j + 1 + lane; i < b; i += 32) x[i] -= lc[i] * xj;
        __syncwarp();
      }
    } else {
      for (int j = b - 1; j >= 0; --j) {
        const double* lc = it.L + (size_t)j * it.ldl;
        double s = 0.0;
        for (int i = j + 1 + lane; i < b; i += 32) s += lc[i] * x[i];
        s = warp_sum(s);
        if (lane == 0) x[j] = (x[j] - s) / lc[j];
        __syncwarp();
      }
    }
  }
}

// Shared-memory variant: the CTA stages L (b x b) once; each warp solves one
// right-hand side column out of shared memory (lanes over rows).
__global__ void __launch_bounds__(512) k_trsm_left_smem(const TrsmLItem* __restrict__ items) {
  const TrsmLItem it = items[blockIdx.x];
  const int cols = it.cols.get();
  const int b = it.b;
  if (cols <= 0 || blockIdx.y * (blockDim.x >> 5) >= cols) return;
  extern __shared__ double sm[];
  double* L = sm;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) L[e] = it.L[(size_t)(e / b) * it.ldl + e % b];
  if (blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&d_cnt_trsm, (double)b * b * cols);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = blockIdx.y * nw + w; c < cols; c += gridDim.y * nw) {
    double* x = it.M + (size_t)c * it.ldm;
    if (!it.trans) {
      for (int j = 0; j < b; ++j) {
        const double xj = x[j] / L[(size_t)j * b + j];
        __syncwarp();
        if (lane == 0) x[j] = xj;
        for (int i = j + 1 + lane; i < b; i += 32) x[i] -= L[(size_t)j * b + i] * xj;
        __syncwarp();
      }
    } else {
      for (int j = b - 1; j >= 0; --j) {
        double s = 0.0;
        for (int i = j + 1 + lane; i < b; i += 32) s += L[(size_t)j * b + i] * x[i];
        s = warp_sum(s);
        if (lane == 0) x[j] = (x[j] - s) / L[(size_t)j * b + j];
        __syncwarp();
      }
    }
  }
}

// Register-resident substitutions for diagonal leaves of up to 32*NB rows:
// L staged in shared memory once per CTA (padded ld, 16-byte loads), the
// reciprocal diagonal precomputed, and each warp solves one right-hand side
// held in registers (lane l owns rows l, l+32, ...): one shuffle broadcast and
// NB FMAs per column instead of a division and two warp barriers.
template <int NB>
__device__ __forceinline__ void stage_tri(const double* __restrict__ Lg, int ldl, int b, double* L, double* inv) {
  constexpr int S = 32 * NB, LD = S + 1;
#pragma unroll 4
  for (int e = threadIdx.x; e < S * S; e += blockDim.x) {
    const int c = e / S, r = e % S;
    L[c * LD + r] = (c < b && r < b) ? Lg[(size_t)c * ldl + r] : 0.0;
  }
  for (int j = threadIdx.x; j < S; j += blockDim.x) inv[j] = j < b ? 1.0 / Lg[(size_t)j * ldl + j] : 0.0;
}
// x <- L^{-1} x (forward) for one warp's register vector
template <int NB>
__device__ __forceinline__ void warp_fwd(double (&xr)[NB], const double* L, const double* inv, int lane) {
  constexpr int LD = 32 * NB + 1;
#pragma unroll
  for (int kb = 0; kb < NB; ++kb)
    for (int jj = 0; jj < 32; ++jj) {
      const int j = kb * 32 + jj;
      if (lane == jj) xr[kb] *= inv[j];
      const double xj = __shfl_sync(0xffffffffu, xr[kb], jj);
      const double* Lc = L + (size_t)j * LD;
      if (lane > jj) xr[kb] -= Lc[kb * 32 + lane] * xj;
#pragma unroll
      for (int k = kb + 1; k < NB; ++k) xr[k] -= Lc[k * 32 + lane] * xj;
    }
}
// x <- L^{-T} x (backward)
template <int NB>
__device__ __forceinline__ void warp_bwd(double (&xr)[NB], const double* L, const double* inv, int lane) {
  constexpr int LD = 32 * NB + 1;
#pragma unroll
  for (int kb = NB - 1; kb >= 0; --kb)
    for (int jj = 31; jj >= 0; --jj) {
      const int j = kb * 32 + jj;
      if (lane == jj) xr[kb] *= inv[j];
      const double xj = __shfl_sync(0xffffffffu, xr[kb], jj);
      if (lane < jj) xr[kb] -= L[(size_t)(kb * 32 + lane) * LD + j] * xj;
#pragma unroll
      for (int k = 0; k < kb; ++k) xr[k] -= L[(size_t)(k * 32 + lane) * LD + j] * xj;
    }
}

template <int NB>
__global__ void __launch_bounds__(512) k_trsm_left_reg(const TrsmLItem* __restrict__ items) {
  const TrsmLItem it = items[blockIdx.x];
  const int cols = it.cols.get();
  const int b = it.b;
  const int nw = blockDim.x >> 5;
  if (cols <= 0 || (int)blockIdx.y * nw >= cols) return;
  extern __shared__ double sm[];
  constexpr int S = 32 * NB;
  double* L = sm;
  double* inv = sm + (size_t)S * (S + 1);
  stage_tri<NB>(it.L, it.ldl, b, L, inv);
  if (blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&d_cnt_trsm, (double)b * b * cols);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = blockIdx.y * nw + w; c < cols; c += gridDim.y * nw) {
    double* x = it.M + (size_t)c * it.ldm;
    double xr[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) xr[k] = (k * 32 + lane < b) ? x[k * 32 + lane] : 0.0;
    if (!it.trans)
      warp_fwd<NB>(xr, L, inv, lane);
    else
      warp_bwd<NB>(xr, L, inv, lane);
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k * 32 + lane < b) x[k * 32 + lane] = xr[k];
  }
}

// X (s x t) <- X L^{-T} (D^{-1}): every row of X is a forward substitution
// with L; rows are staged 32 at a time through shared memory (coalesced) and
// solved one per warp in registers.
template <int NB>
__global__ void __launch_bounds__(512) k_trsm_right_reg(const TrsmRItem* __restrict__ items) {
  const TrsmRItem it = items[blockIdx.x];
  const int t = it.t;
  extern __shared__ double sm[];
  constexpr int S = 32 * NB;
  double* L = sm;
  double* inv = sm + (size_t)S * (S + 1);
  double* X = inv + S;  // 32 rows x S, ld 33 (row r, column c at c * 33 + r)
  stage_tri<NB>(it.L, it.ldl, t, L, inv);
  if (blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&d_cnt_trsm, (double)t * t * it.s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r0 = blockIdx.y * 32; r0 < it.s; r0 += gridDim.y * 32) {
    const int rows = min(32, it.s - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * S; e += blockDim.x) {
      const int r = e & 31, c = e >> 5;
      X[c * 33 + r] = (r < rows && c < t) ? it.X[(size_t)c * it.ldx + r0 + r] : 0.0;
    }
    __syncthreads();
    for (int r = w; r < rows; r += nw) {
      double xr[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) xr[k] = X[(k * 32 + lane) * 33 + r];
      warp_fwd<NB>(xr, L, inv, lane);
#pragma unroll
      for (int k = 0; k < NB; ++k) X[(k * 32 + lane) * 33 + r] = xr[k];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * S; e += blockDim.x) {
      const int r = e & 31, c = e >> 5;
      if (r < rows && c < t) it.X[(size_t)c * it.ldx + r0 + r] = it.d ? X[c * 33 + r] / it.d[c] : X[c * 33 + r];
    }
  }
}

template <class K>
static void set_smem_once(K kern, size_t bytes, bool& done) {
  if (!done) {
    HMGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done = true;
  }
}

void launch_trsm_left(const TrsmLItem* d_items, int count, int max_cols, cudaStream_t st,
                      int max_b) {
  if (count <= 0) return;
  if (max_b > 0 && max_b <= 128) {
    const int gy = max(1, min((max_cols + 15) / 16, 32));
    const int nb = (max_b + 31) / 32;
    const size_t by = ((size_t)32 * nb * (32 * nb + 1) + 32 * nb) * 8;
    static bool c1 = false, c2 = false, c3 = false, c4 = false;
    switch (nb) {
      case 1: set_smem_once(k_trsm_left_reg<1>, by, c1); k_trsm_left_reg<1><<<dim3(count, gy), 512, by, st>>>(d_items); break;
      case 2: set_smem_once(k_trsm_left_reg<2>, by, c2); k_trsm_left_reg<2><<<dim3(count, gy), 512, by, st>>>(d_items); break;
      case 3: set_smem_once(k_trsm_left_reg<3>, by, c3); k_trsm_left_reg<3><<<dim3(count, gy), 512, by, st>>>(d_items); break;
      default: set_smem_once(k_trsm_left_reg<4>, by, c4); k_trsm_left_reg<4><<<dim3(count, gy), 512, by, st>>>(d_items); break;
    }
    HMGP_LAUNCH_CHECK();
    return;
  }
  const size_t bytes = (size_t)max_b * max_b * 8;
  if (max_b > 0 && bytes <= 200 * 1024) {
    static bool configured = false;
    if (!configured) {
      HMGP_CUDA(cudaFuncSetAttribute(k_trsm_left_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
      configured = true;
    }
    const int gy = max(1, min((max_cols + 15) / 16, 32));
    k_trsm_left_smem<<<dim3(count, gy), 512, bytes, st>>>(d_items);
  } else {
    const int gy = max(1, min((max_cols + 7) / 8, 32));
    k_trsm_left<<<dim3(count, gy), 256, 0, st>>>(d_items);
  }
  HMGP_LAUNCH_CHECK();
}

// Right: X <- X L^{-T}, one thread per row of X.
__global__ void k_trsm_right(const TrsmRItem* __restrict__ items) {
  const TrsmRItem it = items[blockIdx.x];
  if (blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&d_cnt_trsm, (double)it.t * it.t * it.s);
  for (int r = blockIdx.y * blockDim.x + threadIdx.x; r < it.s; r += gridDim.y * blockDim.x) {
    for (int j = 0; j < it.t; ++j) {
      const double xj = it.X[(size_t)j * it.ldx + r] / it.L[(size_t)j * it.ldl + j];
      it.X[(size_t)j * it.ldx + r] = xj;
      const double* lc = it.L + (size_t)j * it.ldl;
      for (int c = j + 1; c < it.t; ++c) it.X[(size_t)c * it.ldx + r] -= xj * lc[c];
    }
    if (it.d)
      for (int j = 0; j < it.t; ++j) it.X[(size_t)j * it.ldx + r] /= it.d[j];
  }
}

// Shared-memory variant: L (t x t) and a 64-row tile of X staged on chip; the
// substitution runs column by column with all threads on the tile.
constexpr int kTrsmRTile = 64;
__global__ void __launch_bounds__(256) k_trsm_right_smem(const TrsmRItem* __restrict__ items) {
  const TrsmRItem it = items[blockIdx.x];
  extern __shared__ double sm[];
  const int t = it.t;
  double* L = sm;
  double* X = sm + (size_t)t * t;  // kTrsmRTile x t, ld kTrsmRTile
  for (int e = threadIdx.x; e < t * t; e += blockDim.x) L[e] = it.L[(size_t)(e / t) * it.ldl + e % t];
  for (int r0 = blockIdx.y * kTrsmRTile; r0 < it.s; r0 += gridDim.y * kTrsmRTile) {
    const int rows = min(kTrsmRTile, it.s - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < kTrsmRTile * t; e += blockDim.x) {
      const int r = e % kTrsmRTile, c = e / kTrsmRTile;
      X[e] = r < rows ? it.X[(size_t)c * it.ldx + r0 + r] : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < t; ++j) {
      if (threadIdx.x < kTrsmRTile) X[(size_t)j * kTrsmRTile + threadIdx.x] /= L[(size_t)j * t + j];
      __syncthreads();
      const int w = t - j - 1;
      for (int e = threadIdx.x; e < kTrsmRTile * w; e += blockDim.x) {
        const int r = e % kTrsmRTile, c = j + 1 + e / kTrsmRTile;
        X[(size_t)c * kTrsmRTile + r] -= X[(size_t)j * kTrsmRTile + r] * L[(size_t)j * t + c];
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < kTrsmRTile * t; e += blockDim.x) {
      const int r = e % kTrsmRTile, c = e / kTrsmRTile;
      if (r < rows) it.X[(size_t)c * it.ldx + r0 + r] = it.d ? X[e] / it.d[c] : X[e];
    }
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) atomicAdd(&d_cnt_trsm, (double)t * t * it.s);
}

void launch_trsm_right(const TrsmRItem* d_items, int count, int max_rows, cudaStream_t st,
                       int max_t) {
  if (count <= 0) return;
  if (max_t > 0 && max_t <= 128) {
    const int gy = max(1, min((max_rows + 31) / 32, 32));
    const int nb = (max_t + 31) / 32;
    const size_t by = ((size_t)32 * nb * (32 * nb + 1) + 32 * nb + (size_t)33 * 32 * nb) * 8;
    static bool c1 = false, c2 = false, c3 = false, c4 = false;
    switch (nb) {
      case 1: set_smem_once(k_trsm_right_reg<1>, by, c1); k_trsm_right_reg<1><<<dim3(count, gy), 512, by, st>>>(d_items); break;
      case 2: set_smem_once(k_trsm_right_reg<2>, by, c2); k_trsm_right_reg<2><<<dim3(count, gy), 512, by, st>>>(d_items); break;
      case 3: set_smem_once(k_trsm_right_reg<3>, by, c3); k_trsm_right_reg<3><<<dim3(count, gy), 512, by, st>>>(d_items); break;
      default: set_smem_once(k_trsm_right_reg<4>, by, c4); k_trsm_right_reg<4><<<dim3(count, gy), 512, by, st>>>(d_items); break;
    }
    HMGP_LAUNCH_CHECK();
    return;
  }
  const size_t bytes = ((size_t)max_t * max_t + (size_t)kTrsmRTile * max_t) * 8;
  if (bytes <= 200 * 1024) {
    static bool configured = false;
    if (!configured) {
      HMGP_CUDA(cudaFuncSetAttribute(k_trsm_right_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
      configured = true;
    }
    const int gy = max(1, min((max_rows + kTrsmRTile - 1) / kTrsmRTile, 32));
    k_trsm_right_smem<<<dim3(count, gy), 256, bytes, st>>>(d_items);
  } else {
    const int gy = max(1, min((max_rows + 127) / 128, 64));
    k_trsm_right<<<dim3(count, gy), 128, 0, st>>>(d_items);
  }
  HMGP_LAUNCH_CHECK();
}

// ----------------------------------------------------------- copy/scale ---
__global__ void k_copy_scale(const CopyScaleItem* __restrict__ items) {
  const CopyScaleItem it = items[blockIdx.x];
  const int cols = it.cols.get();
  if (it.set_cols && blockIdx.y == 0 && threadIdx.x == 0) *it.set_cols = cols;
  const size_t tot = (size_t)it.rows * cols;
  for (size_t e = blockIdx.y * (size_t)blockDim.x + threadIdx.x; e < tot;
       e += (size_t)gridDim.y * blockDim.x) {
    const int i = (int)(e % it.rows), j = (int)(e / it.rows);
    double v;
    if (it.src)
      v = it.trans ? it.src[(size_t)i * it.lds + j] : it.src[(size_t)j * it.lds + i];
    else
      v = (i == j) ? 1.0 : 0.0;
    v *= it.alpha;
    switch (it.mode) {
      case 1:
        v *= it.d[i];
        break;
      case 2:
        v /= it.d[i];
        break;
      case 3:
        v *= it.d[j];
        break;
      case 4:
        v /= it.d[j];
        break;
      default:
        break;
    }
    if (it.accum)
      it.dst[(size_t)j * it.ldd + i] += v;
    else
      it.dst[(size_t)j * it.ldd + i] = v;
  }
}

void launch_copy_scale(const CopyScaleItem* d_items, int count, int max_elems, cudaStream_t st) {
  if (count <= 0) return;
  const int gy = max(1, min((max_elems + 255) / 256, 64));
  k_copy_scale<<<dim3(count, gy), 256, 0, st>>>(d_items);
  HMGP_LAUNCH_CHECK();
}

// ------------------------------------------------------ ordered adds ---
// y[i, c] += alpha * sum over the interval's segments, in segment order (the
// reference's DFS order of hblk::apply over a branch, hblock.cpp:46-60).  The
// host cuts the rows of every target into intervals covered by the same
// segments, so intervals are independent and every element has one writer.
__global__ void k_ordered_add(const OrdIv* __restrict__ ivs, const OrdSeg* __restrict__ segs) {
  const OrdIv iv = ivs[blockIdx.x];
  const int cols = iv.cols.get(), len = iv.i1 - iv.i0;
  const size_t tot = (size_t)len * cols;
  for (size_t e = blockIdx.y * (size_t)blockDim.x + threadIdx.x; e < tot;
       e += (size_t)gridDim.y * blockDim.x) {
    const int i = iv.i0 + (int)(e % len), c = (int)(e / len);
    double v = iv.y[(size_t)c * iv.ldy + i];
    for (int l = iv.l0; l < iv.l1; ++l) {
      const OrdSeg sg = segs[l];
      v += iv.alpha * sg.src[(size_t)c * sg.lds + (i - sg.r0)];
    }
    iv.y[(size_t)c * iv.ldy + i] = v;
  }
}

void launch_ordered_add(const OrdIv* d_iv, int count, const OrdSeg* d_segs, int max_elems,
                        cudaStream_t st) {
  if (count <= 0) return;
  const int gy = max(1, min((max_elems + 255) / 256, 32));
  k_ordered_add<<<dim3(count, gy), 256, 0, st>>>(d_iv, d_segs);
  HMGP_LAUNCH_CHECK();
}

// slab 0 <- slab 0 + slab 1 + ... + slab (nslab-1), fixed order (split-K partials)
__global__ void k_slab_sum(const SlabSumItem* __restrict__ items) {
  const SlabSumItem it = items[blockIdx.x];
  const int rows = it.rows.get(), cols = it.cols.get();
  const size_t tot = (size_t)rows * cols;
  for (size_t e = blockIdx.y * (size_t)blockDim.x + threadIdx.x; e < tot;
       e += (size_t)gridDim.y * blockDim.x) {
    const size_t o = (e / rows) * it.ld + (e % rows);
    double v = it.p[o];
    for (int s = 1; s < it.nslab; ++s) v += it.p[s * it.slab + o];
    it.p[o] = v;
  }
}

void launch_slab_sum(const SlabSumItem* d_items, int count, int max_elems, cudaStream_t st) {
  if (count <= 0) return;
  const int gy = max(1, min((max_elems + 255) / 256, 16));
  k_slab_sum<<<dim3(count, gy), 256, 0, st>>>(d_items);
  HMGP_LAUNCH_CHECK();
}

// --------------------------------------------------------------- append ---
// hblock.cpp:186-199: U(:, r0:r0+add) = [0; alpha P; 0], V(:, r0:r0+add) = [0; Q; 0]
__global__ void k_append(const AppendItem* __restrict__ items, int* err) {
  const AppendItem it = items[blockIdx.x];
  const int r0 = *it.rank, add = it.add.get();
  if (add <= 0) return;
  if (r0 + add > it.cap) {
    if (blockIdx.y == 0 && threadIdx.x == 0) atomicOr(err, 2);
    return;
  }
  const size_t tu = (size_t)it.um * add, tv = (size_t)it.vn * add;
  for (size_t e = blockIdx.y * (size_t)blockDim.x + threadIdx.x; e < tu + tv;
       e += (size_t)gridDim.y * blockDim.x) {
    if (e < tu) {
      const int i = (int)(e % it.um), k = (int)(e / it.um);
      const int pi = i - it.pro;
      const double v = (pi >= 0 && pi < it.pr) ? it.alpha * it.P[(size_t)k * it.ldp + pi] : 0.0;
      it.U[(size_t)(r0 + k) * it.um + i] = v;
    } else {
      const size_t f = e - tu;
      const int i = (int)(f % it.vn), k = (int)(f / it.vn);
      const int qi = i - it.qro;
      const double v = (qi >= 0 && qi < it.qr) ? it.Q[(size_t)k * it.ldq + qi] : 0.0;
      it.V[(size_t)(r0 + k) * it.vn + i] = v;
    }
  }
}

// rank update after all CTAs of the item are done: separate tiny kernel
__global__ void k_append_commit(const AppendItem* __restrict__ items, int count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const AppendItem it = items[t];
  const int r0 = *it.rank, add = it.add.get();
  if (add > 0 && r0 + add <= it.cap) *it.rank = r0 + add;
}

void launch_append(const AppendItem* d_items, int count, int max_elems, int* d_err, cudaStream_t st) {
  if (count <= 0) return;
  const int gy = max(1, min((max_elems + 255) / 256, 64));
  k_append<<<dim3(count, gy), 256, 0, st>>>(d_items, d_err);
  HMGP_LAUNCH_CHECK();
  k_append_commit<<<(count + 127) / 128, 128, 0, st>>>(d_items, count);
  HMGP_LAUNCH_CHECK();
}

// ------------------------------------------------------------ leaf LDL ----
__device__ __forceinline__ void atomic_min_double(double* addr, double v) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(addr);
  unsigned long long old = *a;
  while (v < __longlong_as_double(old)) {
    const unsigned long long prev = atomicCAS(a, old, __double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

// Unblocked left-looking column factorization, the reference's loop order
// (hfactor.cpp:22-73); the leaf lives in dynamic shared memory when it fits.
__global__ void k_leaf_factor(double* __restrict__ Dg, int b, int base, int ldl, double* __restrict__ d,
                              double clamp_tol, LeafFactorStatus* st, int use_smem) {
  if (clamp_tol < 0.0) clamp_tol = st->clamp_tol;  // per-evaluation value (graph replay)
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ double s_piv;
  double* A = use_smem ? sm : Dg;
  if (threadIdx.x == 0) atomicAdd(&d_cnt_leaf, (double)b * b * b / 3.0);
  if (use_smem)
    for (int e = threadIdx.x; e < b * b; e += blockDim.x) A[e] = Dg[e];
  __syncthreads();
  // Right-looking: the trailing lower triangle already holds every update of
  // the previous columns, so the pivot is A(j,j) (same value as the reference's
  // left-looking s = m(j,j) - sum_k m(j,k)^2 d_k, different summation order).
  (void)red;
  for (int j = 0; j < b; ++j) {
    if (threadIdx.x == 0) {
      double s = A[(size_t)j * b + j];
      atomic_min_double(&st->min_pivot, s);
      bool failed;
      if (ldl) {
        failed = (s == 0.0);
        if (s < 0.0) {
          if (-s <= clamp_tol) {
            s = clamp_tol;
            atomicAdd(&st->clamped, 1);
          } else {
            atomicAdd(&st->negative, 1);
          }
        }
      } else {
        failed = !(s > 0.0);
      }
      if (failed) {
        const int pos = base + j;
        if (atomicMin(&st->fail_pos, pos) > pos) st->fail_val = s;
      }
      s_piv = s;
    }
    __syncthreads();
    const double s = s_piv;
    const double piv = ldl ? s : sqrt(s);
    if (threadIdx.x == 0) {
      if (ldl) d[base + j] = s;
      A[(size_t)j * b + j] = ldl ? 1.0 : piv;
    }
    for (int i = j + 1 + threadIdx.x; i < b; i += blockDim.x) A[(size_t)j * b + i] /= piv;
    __syncthreads();
    const int t = b - j - 1;
    const double w = ldl ? s : 1.0;
    for (int e = threadIdx.x; e < t * t; e += blockDim.x) {
      const int i = j + 1 + e % t, k = j + 1 + e / t;
      if (i >= k) A[(size_t)k * b + i] -= A[(size_t)j * b + i] * A[(size_t)j * b + k] * w;
    }
    __syncthreads();
  }
  // zero the strict upper triangle (hfactor.cpp:41,72)
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e % b, j = e / b;
    const double v = i < j ? 0.0 : A[e];
    Dg[e] = v;
  }
}

// Register-resident right-looking variant for b <= 128: thread t owns row
// i = t % b and the columns k = t / b + q*G (G = 1024 / b groups), held in
// registers.  Column j is exchanged through shared memory once per step; the
// update A(i,k) -= c_i c_k / s is the same for LDL (l = c/s, d = s) and
// Cholesky (l = c/sqrt(s)).  Two barriers per column.
// BMAX (32, 64 or 128) is a compile-time bound on b so every register slot and
// shared-memory offset is static.
constexpr int kLeafRegThreads = 512;
// Register-resident leaf LDL / Cholesky (dense_ldl_leaf / dense_cholesky_leaf,
// hfactor.cpp:22-73): thread (i, g) holds row i of the columns g, g + G, ...;
// column j is published to a double-buffered shared vector and every thread
// derives the (clamped) pivot from it redundantly, so each column costs one
// barrier.  Pivot bookkeeping (min pivot, clamps, negatives, first failure)
// is kept by thread 0 and committed with one set of atomics at the end.
template <int BMAX>
__global__ void __launch_bounds__(kLeafRegThreads) k_leaf_factor_reg(double* __restrict__ Dg, int b,
                                                                     int base, int ldl,
                                                                     double* __restrict__ d,
                                                                     double clamp_tol,
                                                                     LeafFactorStatus* st) {
  if (clamp_tol < 0.0) clamp_tol = st->clamp_tol;  // per-evaluation value (graph replay)
  constexpr int G = kLeafRegThreads / BMAX;
  constexpr int kLeafRegMaxK = BMAX / G;  // columns per thread
  __shared__ double col[2][BMAX];
  const int t = threadIdx.x;
  const int i = t % BMAX, g = t / BMAX;
  const bool active = i < b;
  double a[kLeafRegMaxK];
#pragma unroll
  for (int q = 0; q < kLeafRegMaxK; ++q) {
    const int k = g + q * G;
    a[q] = (active && k < b) ? Dg[(size_t)k * b + i] : 0.0;
  }
  double minp = INFINITY, failv = 0.0;
  int nclamp = 0, nneg = 0, failpos = INT_MAX;
  for (int j = 0; j < b; ++j) {
    double* cj = col[j & 1];
    // owners of column j (group g = j % G, slot qj = j / G) publish it
    const int qj = j / G;
    const bool own = active && g == j % G;
    double aj = 0.0;
#pragma unroll
    for (int q = 0; q < kLeafRegMaxK; ++q)
      if (q == qj) aj = a[q];
    if (own) cj[i] = aj;
    __syncthreads();
    double s = cj[j];
    const double s_raw = s;
    bool failed;
    bool clamped = false, negative = false;
    if (ldl) {
      failed = (s == 0.0);
      if (s < 0.0) {
        if (-s <= clamp_tol) {
          s = clamp_tol;
          clamped = true;
        } else {
          negative = true;
        }
      }
    } else {
      failed = !(s > 0.0);
    }
    if (t == 0) {
      minp = fmin(minp, s_raw);
      nclamp += clamped;
      nneg += negative;
      if (failed && failpos == INT_MAX) {
        failpos = base + j;
        failv = s;
      }
      if (ldl) d[base + j] = s;
    }
    // One reciprocal (LDL) or reciprocal square root (Cholesky) of the pivot per
    // step, shared by the trailing update and the column scaling: a division, a
    // square root and a second division used to sit on every step's dependent chain
    // (the owner warps of column j hold the barrier of step j + 1).  x * rsqrt(s)
    // differs from x / sqrt(s) by at most an ulp or two.
    const double rp = ldl ? 1.0 / s : rsqrt(s);  // 1/s  or  1/sqrt(s)
    const double rs = ldl ? rp : rp * rp;         // 1/s
    // trailing update of the columns k > j this thread owns (rows i > j only are
    // ever read again, so the strict upper part may hold stale values)
    if (active && i > j) {
      const double ci = cj[i] * rs;
      const int qmin = j >= g ? (j - g) / G + 1 : 0;  // first q with g + q*G > j
#pragma unroll
      for (int q = 0; q < kLeafRegMaxK; ++q)
        if (q >= qmin) a[q] -= ci * cj[g + q * G];
    }
    // finalize column j in its owners' registers
    if (own) {
      const double v = (i == j) ? (ldl ? 1.0 : s * rp) : (i > j ? aj * rp : 0.0);  // s * rsqrt(s) = sqrt(s)
#pragma unroll
      for (int q = 0; q < kLeafRegMaxK; ++q)
        if (q == qj) a[q] = v;
    }
  }
#pragma unroll
  for (int q = 0; q < kLeafRegMaxK; ++q) {
    const int k = g + q * G;
    if (active && k < b) Dg[(size_t)k * b + i] = (i < k) ? 0.0 : a[q];
  }
  if (t == 0) {
    atomicAdd(&d_cnt_leaf, (double)b * b * b / 3.0);
    atomic_min_double(&st->min_pivot, minp);
    if (nclamp) atomicAdd(&st->clamped, nclamp);
    if (nneg) atomicAdd(&st->negative, nneg);
    if (failpos != INT_MAX && atomicMin(&st->fail_pos, failpos) > failpos) st->fail_val = failv;
  }
}

void launch_leaf_factor(double* D, int b, int base, int ldl, double* d, double clamp_tol,
                        LeafFactorStatus* status, cudaStream_t st) {
  if (b <= 128) {
    if (b <= 32)
      k_leaf_factor_reg<32><<<1, kLeafRegThreads, 0, st>>>(D, b, base, ldl, d, clamp_tol, status);
    else if (b <= 64)
      k_leaf_factor_reg<64><<<1, kLeafRegThreads, 0, st>>>(D, b, base, ldl, d, clamp_tol, status);
    else
      k_leaf_factor_reg<128><<<1, kLeafRegThreads, 0, st>>>(D, b, base, ldl, d, clamp_tol, status);
    HMGP_LAUNCH_CHECK();
    return;
  }
  const size_t bytes = (size_t)b * b * 8;
  const int use_smem = bytes <= 200 * 1024;
  if (use_smem && bytes > 48 * 1024)
    HMGP_CUDA(cudaFuncSetAttribute(k_leaf_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)bytes));
  k_leaf_factor<<<1, 256, use_smem ? bytes : 0, st>>>(D, b, base, ldl, d, clamp_tol, status,
                                                       use_smem);
  HMGP_LAUNCH_CHECK();
}

}  // namespace hmgp_gpu
