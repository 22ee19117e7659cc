// H-matrix times vector, y = C x, for the symmetric lower-stored H-matrix
// (hmatrix.cpp:244-272 / hblock.cpp:36-75) — an HBM-bound pass: every stored
// payload byte is needed once (4 GB at C3), the arithmetic is 2 flop per 8 bytes.
//
// Layout of the pass:
//   k_mv_leaf    one CTA per stored leaf that fits one CTA: a dense leaf is read
//                once, column-major coalesced, and yields BOTH its products (A x_c
//                for the row range and, off the diagonal, A^T x_r for the mirrored
//                column range) from the same registers; a low-rank leaf forms
//                t = V^T x_c, t2 = U^T x_r (warp per column) and then U t, V t2 with
//                its factors still in L1 / L2.
//   k_mv_chunk_* low-rank leaves too tall for one CTA, cut into 1024-row chunks:
//                partial dots, a fixed-order sum over the chunks, then U t / V t2.
//   k_mv_gather  every product goes to a private segment; the rows of one leaf
//                cluster then sum the segments that cover them in a fixed (DFS)
//                order — no atomics, so y is bit-reproducible
//                (tests/test_hmatrix.cpp:165-171).
// The plan (offsets, chunk lists, gather lists) depends only on the block layout
// and is kept for the H-matrix it was built for.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "hmgp_api.h"
#include "hmgp_internal.h"

namespace hmgp_gpu {
namespace {

constexpr int kMvThreads = 128;
constexpr int kChunkRows = 1024;
constexpr size_t kFusedMax = (size_t)96 * 1024;  // (m + n) * cap doubles handled by one CTA

struct MvLeaf {
  const double* a;
  const double* b;
  int m, n, kind, cap;
  int rb, cb;         // tree positions of the row / column range
  long long seg_r;    // private output segment of a x_c (m doubles)
  long long seg_c;    // of a^T x_r (n doubles), -1 on the diagonal
  int rank_idx;       // index into d_rank
  int t_off;          // chunked leaves: offset of their t / t2 vectors (2 * cap doubles)
};

struct MvChunk {
  int leaf;   // index into the MvLeaf table
  int side;   // 0: rows of U (x_r side), 1: rows of V (x_c side)
  int r0, r1; // row range of the chunk within the factor
  int part;   // index of this chunk's partial vector (cap doubles each)
};

struct MvRed {  // sum of a chunked leaf-side's partials, in chunk order
  int t_dst;    // offset into tbuf
  int part0, nparts, cap, rank_idx;
};

struct MvUnit {  // one leaf cluster's rows and the segments covering them
  int begin, len, e0, e1;
};

__global__ void __launch_bounds__(kMvThreads) k_mv_leaf(const MvLeaf* __restrict__ leaves,
                                                        const int* __restrict__ ids,
                                                        const int* __restrict__ rank,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ ypart) {
  const MvLeaf L = leaves[ids[blockIdx.x]];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = kMvThreads / 32;
  const bool mirror = L.seg_c >= 0;
  __shared__ double s_t[2][1024];
  if (L.kind == DENSE) {
    // rows in strips of 128: thread = row, all columns; the mirrored product is a
    // CTA-wide column sum of the same loaded value
    __shared__ double s_col[kMvThreads / 32][132];
    double* yr = ypart + L.seg_r;
    double* yc = mirror ? ypart + L.seg_c : nullptr;
    for (int j0 = 0; j0 < L.n; j0 += 128) {
      const int nj = min(128, L.n - j0);
      double colacc = 0.0;  // thread j (< nj) accumulates column j0 + j over the row strips
      for (int i0 = 0; i0 < L.m; i0 += kMvThreads) {
        const int i = i0 + threadIdx.x;
        const bool on = i < L.m;
        const double xr = (mirror && on) ? x[L.rb + i] : 0.0;
        double acc = 0.0;
        const double* ap = L.a + (size_t)j0 * L.m + i;
        for (int jb = 0; jb < nj; jb += 4) {
          double av[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) av[u] = (on && jb + u < nj) ? ap[(size_t)(jb + u) * L.m] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (jb + u < nj) acc += av[u] * x[L.cb + j0 + jb + u];
          if (mirror) {
            double pv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) pv[u] = av[u] * xr;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
              for (int u = 0; u < 4; ++u) pv[u] += __shfl_xor_sync(0xffffffffu, pv[u], o);
            }
            if (lane == 0) {
#pragma unroll
              for (int u = 0; u < 4; ++u) s_col[w][jb + u] = pv[u];
            }
          }
        }
        if (on) {
          if (j0 == 0) yr[i] = acc;
          else yr[i] += acc;  // same thread, same row: ordered
        }
        if (mirror) {
          __syncthreads();
          if (threadIdx.x < nj) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < nw; ++q) s += s_col[q][threadIdx.x];
            colacc += s;
          }
          __syncthreads();
        }
      }
      if (mirror && threadIdx.x < nj) yc[j0 + threadIdx.x] = colacc;
    }
    return;
  }
  // low-rank leaf handled by one CTA
  const int r = rank[L.rank_idx];
  double* yr = ypart + L.seg_r;
  double* yc = mirror ? ypart + L.seg_c : nullptr;
  if (r <= 0) {
    for (int i = threadIdx.x; i < L.m; i += kMvThreads) yr[i] = 0.0;
    if (mirror)
      for (int j = threadIdx.x; j < L.n; j += kMvThreads) yc[j] = 0.0;
    return;
  }
  for (int l0 = 0; l0 < r; l0 += 1024) {  // (ranks beyond 1024 in slabs; never in practice)
    const int rl = min(1024, r - l0);
    for (int l = w; l < rl; l += nw) {
      const double* v = L.b + (size_t)(l0 + l) * L.n;
      double s = 0.0;
      for (int j = lane; j < L.n; j += 32) s += v[j] * x[L.cb + j];
      s = warp_sum(s);
      double s2 = 0.0;
      if (mirror) {
        const double* u = L.a + (size_t)(l0 + l) * L.m;
        for (int i = lane; i < L.m; i += 32) s2 += u[i] * x[L.rb + i];
        s2 = warp_sum(s2);
      }
      if (lane == 0) {
        s_t[0][l] = s;
        s_t[1][l] = s2;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < L.m; i += kMvThreads) {
      double s = 0.0;
      for (int l = 0; l < rl; ++l) s += L.a[(size_t)(l0 + l) * L.m + i] * s_t[0][l];
      if (l0 == 0) yr[i] = s;
      else yr[i] += s;
    }
    if (mirror)
      for (int j = threadIdx.x; j < L.n; j += kMvThreads) {
        double s = 0.0;
        for (int l = 0; l < rl; ++l) s += L.b[(size_t)(l0 + l) * L.n + j] * s_t[1][l];
        if (l0 == 0) yc[j] = s;
        else yc[j] += s;
      }
    __syncthreads();
  }
}

// chunked low-rank leaves, pass 1: partial t (side 1: V^T x_c) / t2 (side 0: U^T x_r)
__global__ void __launch_bounds__(kMvThreads) k_mv_chunk_dots(const MvLeaf* __restrict__ leaves,
                                                              const MvChunk* __restrict__ chunks,
                                                              const int* __restrict__ rank,
                                                              const double* __restrict__ x,
                                                              double* __restrict__ parts, int cap_stride) {
  const MvChunk c = chunks[blockIdx.x];
  const MvLeaf L = leaves[c.leaf];
  const int r = rank[L.rank_idx];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = kMvThreads / 32;
  const double* F = c.side ? L.b : L.a;
  const int ld = c.side ? L.n : L.m;
  const double* xv = x + (c.side ? L.cb : L.rb);
  double* out = parts + (size_t)c.part * cap_stride;
  if (c.side == 0 && L.seg_c < 0) return;  // no mirrored product on the diagonal
  for (int l = w; l < r; l += nw) {
    const double* f = F + (size_t)l * ld;
    double s = 0.0;
    for (int i = c.r0 + lane; i < c.r1; i += 32) s += f[i] * xv[i];
    s = warp_sum(s);
    if (lane == 0) out[l] = s;
  }
}

__global__ void k_mv_chunk_reduce(const MvRed* __restrict__ reds, const int* __restrict__ rank,
                                  const double* __restrict__ parts, int cap_stride,
                                  double* __restrict__ tbuf) {
  const MvRed R = reds[blockIdx.x];
  const int r = rank[R.rank_idx];
  for (int l = threadIdx.x; l < r; l += blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < R.nparts; ++p) s += parts[(size_t)(R.part0 + p) * cap_stride + l];
    tbuf[R.t_dst + l] = s;
  }
}

// pass 2: rows of the chunk: y_r = U t (side 0), y_c = V t2 (side 1)
__global__ void __launch_bounds__(kMvThreads) k_mv_chunk_apply(const MvLeaf* __restrict__ leaves,
                                                               const MvChunk* __restrict__ chunks,
                                                               const int* __restrict__ rank,
                                                               const double* __restrict__ tbuf,
                                                               double* __restrict__ ypart) {
  const MvChunk c = chunks[blockIdx.x];
  const MvLeaf L = leaves[c.leaf];
  const int r = rank[L.rank_idx];
  if (c.side == 1 && L.seg_c < 0) return;
  const double* F = c.side ? L.b : L.a;
  const int ld = c.side ? L.n : L.m;
  // U rows take t = V^T x_c (stored first), V rows take t2 = U^T x_r
  const double* t = tbuf + L.t_off + (c.side ? L.cap : 0);
  double* out = ypart + (c.side ? L.seg_c : L.seg_r);
  __shared__ double s_t[1024];
  for (int l0 = 0; l0 < max(r, 1); l0 += 1024) {
    const int rl = min(1024, r - l0);
    __syncthreads();
    for (int l = threadIdx.x; l < rl; l += kMvThreads) s_t[l] = t[l0 + l];
    __syncthreads();
    for (int i = c.r0 + threadIdx.x; i < c.r1; i += kMvThreads) {
      double s = 0.0;
      for (int l = 0; l < rl; ++l) s += F[(size_t)(l0 + l) * ld + i] * s_t[l];
      if (l0 == 0) out[i] = s;
      else out[i] += s;
    }
  }
}

__global__ void k_mv_gather(const MvUnit* __restrict__ units, const long long* __restrict__ ent,
                            const double* __restrict__ ypart, double* __restrict__ y) {
  const MvUnit u = units[blockIdx.x];
  for (int i = threadIdx.x; i < u.len; i += blockDim.x) {
    double s = 0.0;
    for (int e = u.e0; e < u.e1; ++e) s += ypart[ent[e] + i];
    y[u.begin + i] = s;
  }
}

__global__ void k_mv_permute_in(const double* __restrict__ x, const int* __restrict__ perm, int n,
                                double* __restrict__ xt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) xt[k] = x[perm[k]];
}
__global__ void k_mv_permute_out(const double* __restrict__ yt, const int* __restrict__ perm, int n,
                                 double* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) y[perm[k]] = yt[k];
}

struct Plan {
  const HMat* owner = nullptr;
  const double* pool = nullptr;
  uint64_t sig = 0;
  int n_fused = 0, n_chunks = 0, n_reds = 0, n_units = 0, cap_stride = 1;
  size_t ypart_doubles = 0, parts_doubles = 0, tbuf_doubles = 0;
  MvLeaf* d_leaves = nullptr;
  int* d_fused = nullptr;
  MvChunk* d_chunks = nullptr;
  MvRed* d_reds = nullptr;
  MvUnit* d_units = nullptr;
  long long* d_ent = nullptr;
  double *d_ypart = nullptr, *d_parts = nullptr, *d_tbuf = nullptr, *d_xt = nullptr, *d_yt = nullptr;
  void free_all() {
    cudaFree(d_leaves);
    cudaFree(d_fused);
    cudaFree(d_chunks);
    cudaFree(d_reds);
    cudaFree(d_units);
    cudaFree(d_ent);
    cudaFree(d_ypart);
    cudaFree(d_parts);
    cudaFree(d_tbuf);
    cudaFree(d_xt);
    cudaFree(d_yt);
    *this = Plan();
  }
};
Plan g_plan;
std::mutex g_plan_mu;

uint64_t layout_sig(const HMat& h) {
  uint64_t s = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    s ^= v;
    s *= 1099511628211ull;
  };
  mix(h.leaf.size());
  for (const LeafDev& l : h.leaf) {
    mix((uint64_t)(uintptr_t)l.a);
    mix(((uint64_t)l.m << 40) ^ ((uint64_t)l.n << 16) ^ ((uint64_t)l.kind << 12) ^ (uint64_t)l.cap);
  }
  return s;
}

template <class T>
T* upload(const std::vector<T>& v, cudaStream_t st) {
  T* d = nullptr;
  HMGP_CUDA(dev_malloc_plain((void**)&d, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) HMGP_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return d;
}

void build_plan(Plan& P, const HMat& h, cudaStream_t st) {
  P.free_all();
  const Geometry& G = *h.g;
  const int L = (int)h.leaf.size();
  std::vector<MvLeaf> leaves(L);
  std::vector<int> fused;
  std::vector<MvChunk> chunks;
  std::vector<MvRed> reds;
  long long seg = 0;
  int tnext = 0, pnext = 0, cap_stride = 1;
  // leaf clusters = row ranges of the diagonal leaves (they partition [0, n))
  std::vector<int> ubeg;
  for (int k = 0; k < L; ++k) {
    const HNode& nd = h.nodes[h.leaf_node[k]];
    const LeafDev& l = h.leaf[k];
    MvLeaf& m = leaves[k];
    m.a = l.a;
    m.b = l.b;
    m.m = l.m;
    m.n = l.n;
    m.kind = l.kind;
    m.cap = l.cap;
    m.rb = G.nbeg[nd.row];
    m.cb = G.nbeg[nd.col];
    m.rank_idx = k;
    m.seg_r = seg;
    seg += l.m;
    m.seg_c = -1;
    if (m.rb != m.cb) {
      m.seg_c = seg;
      seg += l.n;
    } else {
      ubeg.push_back(m.rb);
    }
    m.t_off = -1;
    const bool chunked = l.kind == LOWRANK && (size_t)(l.m + l.n) * l.cap > kFusedMax;
    if (!chunked) {
      fused.push_back(k);
      continue;
    }
    m.t_off = tnext;
    tnext += 2 * l.cap;
    cap_stride = std::max(cap_stride, l.cap);
    for (int side = 0; side < 2; ++side) {
      const int rows = side ? l.n : l.m;
      MvRed rd{m.t_off + (side ? 0 : l.cap), pnext, 0, l.cap, k};  // side 1 (V) -> t, side 0 (U) -> t2
      for (int r0 = 0; r0 < rows; r0 += kChunkRows) {
        chunks.push_back(MvChunk{k, side, r0, std::min(rows, r0 + kChunkRows), pnext++});
        ++rd.nparts;
      }
      reds.push_back(rd);
    }
  }
  std::sort(ubeg.begin(), ubeg.end());
  std::vector<std::vector<long long>> cover(ubeg.size());
  auto unit_of = [&](int pos) { return (int)(std::upper_bound(ubeg.begin(), ubeg.end(), pos) - ubeg.begin()) - 1; };
  for (int k = 0; k < L; ++k) {  // DFS leaf order; direct before mirrored
    const MvLeaf& m = leaves[k];
    for (int u = unit_of(m.rb); u < (int)ubeg.size() && ubeg[u] < m.rb + m.m; ++u)
      cover[u].push_back(m.seg_r + (ubeg[u] - m.rb));
    if (m.seg_c >= 0)
      for (int u = unit_of(m.cb); u < (int)ubeg.size() && ubeg[u] < m.cb + m.n; ++u)
        cover[u].push_back(m.seg_c + (ubeg[u] - m.cb));
  }
  std::vector<MvUnit> units(ubeg.size());
  std::vector<long long> ent;
  for (size_t u = 0; u < ubeg.size(); ++u) {
    const int end = u + 1 < ubeg.size() ? ubeg[u + 1] : G.n;
    units[u] = MvUnit{ubeg[u], end - ubeg[u], (int)ent.size(), 0};
    ent.insert(ent.end(), cover[u].begin(), cover[u].end());
    units[u].e1 = (int)ent.size();
  }
  P.n_fused = (int)fused.size();
  P.n_chunks = (int)chunks.size();
  P.n_reds = (int)reds.size();
  P.n_units = (int)units.size();
  P.cap_stride = cap_stride;
  P.ypart_doubles = (size_t)seg;
  P.parts_doubles = (size_t)std::max(pnext, 1) * cap_stride;
  P.tbuf_doubles = (size_t)std::max(tnext, 1);
  P.d_leaves = upload(leaves, st);
  P.d_fused = upload(fused, st);
  P.d_chunks = upload(chunks, st);
  P.d_reds = upload(reds, st);
  P.d_units = upload(units, st);
  P.d_ent = upload(ent, st);
  HMGP_CUDA(dev_malloc_plain((void**)&P.d_ypart, std::max<size_t>(1, P.ypart_doubles) * 8));
  HMGP_CUDA(dev_malloc_plain((void**)&P.d_parts, P.parts_doubles * 8));
  HMGP_CUDA(dev_malloc_plain((void**)&P.d_tbuf, P.tbuf_doubles * 8));
  HMGP_CUDA(dev_malloc_plain((void**)&P.d_xt, 8ull * G.n));
  HMGP_CUDA(dev_malloc_plain((void**)&P.d_yt, 8ull * G.n));
  HMGP_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
  P.owner = &h;
  P.pool = h.pool;
  P.sig = layout_sig(h);
}

}  // namespace

// y = C x with device vectors in ORIGINAL order (the permutation is applied here)
void hmat_matvec_device(cudaStream_t st, const HMat& h, const double* d_x, double* d_y) {
  NvtxRange nvtx_range("hmgp:matvec");
  std::lock_guard<std::mutex> lk(g_plan_mu);
  const Geometry& G = *h.g;
  const int n = G.n;
  Plan& P = g_plan;
  if (P.owner != &h || P.pool != h.pool || P.sig != layout_sig(h)) build_plan(P, h, st);
  k_mv_permute_in<<<(n + 255) / 256, 256, 0, st>>>(d_x, G.d_perm, n, P.d_xt);
  HMGP_LAUNCH_CHECK();
  if (P.n_fused) {
    k_mv_leaf<<<P.n_fused, kMvThreads, 0, st>>>(P.d_leaves, P.d_fused, h.d_rank, P.d_xt, P.d_ypart);
    HMGP_LAUNCH_CHECK();
  }
  if (P.n_chunks) {
    k_mv_chunk_dots<<<P.n_chunks, kMvThreads, 0, st>>>(P.d_leaves, P.d_chunks, h.d_rank, P.d_xt, P.d_parts,
                                                       P.cap_stride);
    HMGP_LAUNCH_CHECK();
    k_mv_chunk_reduce<<<P.n_reds, 128, 0, st>>>(P.d_reds, h.d_rank, P.d_parts, P.cap_stride, P.d_tbuf);
    HMGP_LAUNCH_CHECK();
    k_mv_chunk_apply<<<P.n_chunks, kMvThreads, 0, st>>>(P.d_leaves, P.d_chunks, h.d_rank, P.d_tbuf, P.d_ypart);
    HMGP_LAUNCH_CHECK();
  }
  k_mv_gather<<<P.n_units, 128, 0, st>>>(P.d_units, P.d_ent, P.d_ypart, P.d_yt);
  HMGP_LAUNCH_CHECK();
  k_mv_permute_out<<<(n + 255) / 256, 256, 0, st>>>(P.d_yt, G.d_perm, n, d_y);
  HMGP_LAUNCH_CHECK();
}

// drop the cached plan if it belongs to this H-matrix (called when it is destroyed)
void hmat_matvec_forget(const HMat* h) {
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (g_plan.owner == h) g_plan.free_all();
}

}  // namespace hmgp_gpu
