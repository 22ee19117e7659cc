// H-matrix assembly on the GPU (hmatrix.cpp:108-221):
//   payload tree        build_payload_tree, lower triangle only (hmatrix.cpp:108-139)
//   K3 dense leaves     fill_leaf dense branch (hmatrix.cpp:147-153): one CTA per
//                       leaf, row/col coordinates staged in shared memory from the
//                       tree-ordered SoA copy, column-major coalesced stores
//   K4 batched ACA      detail::aca (hmatrix.cpp:13-102): one CTA per admissible
//                       block, CTA-wide pivot searches with lowest-index ties,
//                       residual rows/columns against U, V in global memory
//   K5 truncation       rank > 16 -> join_truncate (hmatrix.cpp:159-161)
//   coarsening          (m+n) r >= m n -> dense U V^T (hmatrix.cpp:164-169)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "hmgp_internal.h"
#include "phases.h"

namespace hmgp_gpu {

MaternDev make_matern(double sigma2, double ell, double nu, double tau2) {
  MaternDev p{};
  p.sigma2 = sigma2;
  p.ell = ell;
  p.nu = nu;
  p.tau2 = tau2;
  p.pref = sigma2 * std::pow(2.0, 1.0 - nu) / std::tgamma(nu);  // covkernel.cpp:219
  p.closed = nu == 0.5 ? 0 : nu == 1.5 ? 1 : nu == 2.5 ? 2 : -1;
  const double hs = nu - 0.5;
  p.half = (hs == std::floor(hs) && hs >= 0.0) ? static_cast<int>(hs) : -1;
  return p;
}

// entry (tree positions a, b): nugget on index equality (covkernel.hpp:45-48)
__device__ __forceinline__ double kentry(const MaternDev& p, const double* __restrict__ xt, int n,
                                         int dim, int a, int b) {
  if (a == b) return p.sigma2 + p.tau2;
  const double h = dim == 2 ? dist2d(xt[a], xt[n + a], xt[b], xt[n + b])
                            : dist3d(xt[a], xt[n + a], xt[2 * n + a], xt[b], xt[n + b], xt[2 * n + b]);
  return matern_at(p, h);
}

struct DenseItem {
  double* D;
  int r0, c0, m, n;
};

__global__ void __launch_bounds__(256) k_dense_leaves(const DenseItem* __restrict__ items,
                                                      MaternDev p, const double* __restrict__ xt,
                                                      int n_pts, int dim) {
  const DenseItem it = items[blockIdx.x];
  __shared__ double sr[3][256], sc[3][256];
  for (int tile_j = 0; tile_j < it.n; tile_j += 256)
    for (int tile_i = 0; tile_i < it.m; tile_i += 256) {
      const int mi = min(256, it.m - tile_i), nj = min(256, it.n - tile_j);
      __syncthreads();
      for (int t = threadIdx.x; t < mi; t += blockDim.x)
        for (int d = 0; d < dim; ++d) sr[d][t] = xt[(size_t)d * n_pts + it.r0 + tile_i + t];
      for (int t = threadIdx.x; t < nj; t += blockDim.x)
        for (int d = 0; d < dim; ++d) sc[d][t] = xt[(size_t)d * n_pts + it.c0 + tile_j + t];
      __syncthreads();
      for (int idx = threadIdx.x; idx < mi * nj; idx += blockDim.x) {
        const int i = idx % mi, j = idx / mi;
        const int a = it.r0 + tile_i + i, b = it.c0 + tile_j + j;
        double v;
        if (a == b) {
          v = p.sigma2 + p.tau2;
        } else {
          const double h = dim == 2 ? dist2d(sr[0][i], sr[1][i], sc[0][j], sc[1][j])
                                    : dist3d(sr[0][i], sr[1][i], sr[2][i], sc[0][j], sc[1][j], sc[2][j]);
          v = matern_at(p, h);
        }
        it.D[(size_t)(tile_j + j) * it.m + tile_i + i] = v;
      }
    }
}

// Untimed counting pass: algorithmic flops of all dense-leaf entries.
__global__ void k_dense_flops(const DenseItem* __restrict__ items, MaternDev p,
                              const double* __restrict__ xt, int n_pts, int dim, double* out) {
  const DenseItem it = items[blockIdx.x];
  __shared__ double red[32];
  double acc = 0.0;
  for (int idx = threadIdx.x; idx < it.m * it.n; idx += blockDim.x) {
    const int a = it.r0 + idx % it.m, b = it.c0 + idx / it.m;
    if (a == b) continue;
    const double h = dim == 2 ? dist2d(xt[a], xt[n_pts + a], xt[b], xt[n_pts + b])
                              : dist3d(xt[a], xt[n_pts + a], xt[2 * n_pts + a], xt[b],
                                       xt[n_pts + b], xt[2 * n_pts + b]);
    acc += matern_flops(p, h);
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) atomicAdd(out, acc);
}

__device__ double d_cnt_aca;

double aca_entries_read_reset() {
  double v = 0.0, z = 0.0;
  HMGP_CUDA(cudaMemcpyFromSymbol(&v, d_cnt_aca, 8));
  HMGP_CUDA(cudaMemcpyToSymbol(d_cnt_aca, &z, 8));
  return v;
}

struct AcaItem {
  double* U;  // m x cap
  double* V;  // n x cap
  int r0, c0, m, n;
  int cap;        // column capacity of U, V in this pass
  int max_terms;  // min(m, n, max_rank[, k])  (hmatrix.cpp:15-16)
  int* rank;      // out; -1 = capacity reached before the stopping rule (redo)
  unsigned* flags;  // (m + n) bits: used rows then used cols, zero-initialised
};

constexpr int kAcaThreads = 256;

__global__ void __launch_bounds__(kAcaThreads) k_aca(const AcaItem* __restrict__ items, MaternDev p,
                                                     const double* __restrict__ xt, int n_pts,
                                                     int dim, double eps, int fixed) {
  const AcaItem it = items[blockIdx.x];
  const int m = it.m, n = it.n;
  unsigned* rused = it.flags;
  unsigned* cused = it.flags + (m + 31) / 32;
  __shared__ double redv[32];
  __shared__ int redi[32];
  __shared__ double s_coef[256 + 1];
  __shared__ double s_du[256], s_dv[256];
  __shared__ int s_next, s_fresh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int max_terms = it.max_terms;
  double fro2 = 0.0, scale0 = 0.0, ne = 0.0;
  int ip = 0, k = 0;
  if (threadIdx.x == 0) s_fresh = 1;
  __syncthreads();
  while (k < max_terms) {
    if (k >= it.cap) {  // pass capacity reached before the stopping rule: redo later
      if (threadIdx.x == 0) *it.rank = -1;
      return;
    }
    // residual row r_j = A(ip, j) - sum_l U(ip,l) V(j,l)  -> stored in V(:, k)
    for (int l = threadIdx.x; l < k; l += blockDim.x) s_coef[l] = it.U[(size_t)l * m + ip];
    __syncthreads();
    double* r = it.V + (size_t)k * n;
    ne += n;
    int jb = -1;
    double ab = -1.0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double v = kentry(p, xt, n_pts, dim, it.r0 + ip, it.c0 + j);
      for (int l = 0; l < k; ++l) v -= s_coef[l] * it.V[(size_t)l * n + j];
      r[j] = v;
      if (!((cused[j >> 5] >> (j & 31)) & 1u)) {
        const double a = fabs(v);
        if (a > ab) {  // strict: first (lowest) index per thread
          ab = a;
          jb = j;
        }
      }
    }
    double best;
    const int jp = block_argmax(ab, jb, redv, redi, &best);
    if (jp < 0) break;
    if (best <= 1e-15 * scale0 || best == 0.0) {
      // retire the row; next fresh row (hmatrix.cpp:42-56)
      if (threadIdx.x == 0) {
        rused[ip >> 5] |= 1u << (ip & 31);
        int nx = -1, fr = s_fresh;
        while (fr < m) {
          if (!((rused[fr >> 5] >> (fr & 31)) & 1u)) {
            nx = fr;
            break;
          }
          ++fr;
        }
        s_fresh = fr;
        s_next = nx;
      }
      __syncthreads();
      const int nx = s_next;
      __syncthreads();
      if (nx < 0) break;
      ip = nx;
      continue;
    }
    if (scale0 == 0.0) scale0 = best;
    const double piv = r[jp];
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) r[j] = r[j] / piv;
    // column u_i = A(i, jp) - sum_l V(jp,l) U(i,l) -> U(:, k)
    for (int l = threadIdx.x; l < k; l += blockDim.x) s_coef[l] = it.V[(size_t)l * n + jp];
    __syncthreads();
    double* u = it.U + (size_t)k * m;
    ne += m;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      double v = kentry(p, xt, n_pts, dim, it.r0 + i, it.c0 + jp);
      for (int l = 0; l < k; ++l) v -= s_coef[l] * it.U[(size_t)l * m + i];
      u[i] = v;
    }
    if (threadIdx.x == 0) {
      rused[ip >> 5] |= 1u << (ip & 31);
      cused[jp >> 5] |= 1u << (jp & 31);
    }
    __syncthreads();
    // norms and cross terms
    double pu = 0.0, pv = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) pu += u[i] * u[i];
    for (int j = threadIdx.x; j < n; j += blockDim.x) pv += r[j] * r[j];
    const double u2 = block_sum(pu, redv);
    const double v2 = block_sum(pv, redv);
    for (int l = w; l < k; l += nw) {
      const double* ul = it.U + (size_t)l * m;
      const double* vl = it.V + (size_t)l * n;
      double a = 0.0, b = 0.0;
      for (int i = lane; i < m; i += 32) a += ul[i] * u[i];
      for (int j = lane; j < n; j += 32) b += vl[j] * r[j];
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0) {
        s_du[l] = a;
        s_dv[l] = b;
      }
    }
    __syncthreads();
    double cross = 0.0;
    for (int l = 0; l < k; ++l) cross += s_du[l] * s_dv[l];
    fro2 += 2.0 * cross + u2 * v2;
    ++k;
    if (!fixed && u2 * v2 <= eps * eps * fro2) break;
    // next row = argmax |u_i| over unused rows
    int ib = -1;
    ab = -1.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      if ((rused[i >> 5] >> (i & 31)) & 1u) continue;
      const double a = fabs(u[i]);
      if (a > ab) {
        ab = a;
        ib = i;
      }
    }
    const int inx = block_argmax(ab, ib, redv, redi, &best);
    if (inx < 0) break;
    ip = inx;
  }
  if (threadIdx.x == 0) {
    *it.rank = k;
    atomicAdd(&d_cnt_aca, ne);
  }
}

// C (m x n) = U (m x r) V^T (n x r), r from device; one CTA per item.
struct OuterItem {
  const double* U;
  const double* V;
  double* C;
  int m, n;
  const int* rank;
};
__global__ void k_outer(const OuterItem* __restrict__ items) {
  const OuterItem it = items[blockIdx.x];
  const int r = *it.rank;
  for (int idx = threadIdx.x; idx < it.m * it.n; idx += blockDim.x) {
    const int i = idx % it.m, j = idx / it.m;
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += it.U[(size_t)l * it.m + i] * it.V[(size_t)l * it.n + j];
    it.C[idx] = s;
  }
}

struct CopyItem {
  const double* src;
  double* dst;
  size_t count;
};
__global__ void k_copy(const CopyItem* __restrict__ items) {
  const CopyItem it = items[blockIdx.x];
  for (size_t i = threadIdx.x; i < it.count; i += blockDim.x) it.dst[i] = it.src[i];
}

__global__ void k_diag_max(const LeafDev* __restrict__ lf, const int* __restrict__ diag_leaves,
                           int count, double* out) {
  double mx = 0.0;
  for (int t = threadIdx.x; t < count; t += blockDim.x) {
    const LeafDev L = lf[diag_leaves[t]];
    for (int i = 0; i < L.m; ++i) mx = fmax(mx, L.a[(size_t)i * L.m + i]);
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) mx = fmax(mx, red[q]);
    *out = mx;
  }
}

namespace {
template <class T>
T* dmalloc(size_t count) {
  T* p = nullptr;
  p = dev_alloc_n<T>(count);
  return p;
}
template <class T>
T* upload(const std::vector<T>& v, cudaStream_t st) {
  T* p = dmalloc<T>(v.size());
  if (!v.empty())
    HMGP_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return p;
}

int build_payload(HMat& h, const Geometry& g, int bn, bool sym) {
  const int id = static_cast<int>(h.nodes.size());
  h.nodes.emplace_back();
  const BlockNodeRec& b = g.bnodes[bn];
  h.nodes[id].row = b.row;
  h.nodes[id].col = b.col;
  h.nodes[id].kr = g.nleft[b.row] < 0 ? 1 : 2;
  h.nodes[id].kc = g.nleft[b.col] < 0 ? 1 : 2;
  if (b.tag == 1 || b.tag == 0) {
    h.nodes[id].kind = b.tag == 1 ? DENSE : LOWRANK;
    h.nodes[id].leaf = static_cast<int>(h.leaf_node.size());
    h.leaf_node.push_back(id);
    return id;
  }
  h.nodes[id].kind = BRANCH;
  const int kr = h.nodes[id].kr, kc = h.nodes[id].kc;
  const auto& kids = g.bkids[bn];
  for (int i = 0; i < kr; ++i)
    for (int j = 0; j < kc; ++j) {
      if (sym && b.row == b.col && j > i) continue;  // mirror implied (hmatrix.cpp:131)
      const int c = build_payload(h, g, kids[i * kc + j], sym);
      h.nodes[id].kids[i * kc + j] = c;
    }
  return id;
}
}  // namespace

void hmat_matvec_forget(const HMat* h);  // matvec.cu: drops the plan cached for this H-matrix
HMat::~HMat() {
  hmat_matvec_forget(this);
  dev_free(d_leaf);
  dev_free(d_rank);
  dev_free(d_compact);
  dev_free(pool);
}

// Column capacity of a stored low-rank leaf for the factorization: its assembled
// rank plus headroom, plus the +16 watermark slack (hblock.cpp:200).
static int lr_capacity(int m, int n, int rank) {
  const int mn = std::min(m, n);
  const int want = std::max(2 * rank + 32, 64);
  return std::min(mn, want) + 16;
}

// Greedy prefix split: range p ends at the first leaf whose prefix cost reaches
// (p+1)/parts of the total, so every range is contiguous in DFS order.
void balanced_ranges(const double* cost, int L, int parts, int* bounds) {
  double total = 0.0;
  for (int k = 0; k < L; ++k) total += cost[k];
  bounds[0] = 0;
  double acc = 0.0;
  int k = 0;
  for (int q = 1; q < parts; ++q) {
    const double target = total * q / parts;
    while (k < L && acc + 0.5 * cost[k] < target) acc += cost[k++];
    bounds[q] = k;
  }
  bounds[parts] = L;
}

void assemble(HMat& h, Geometry& g, const MaternDev& p, double eps, bool fixed_rank, int rank_k,
              int max_rank, cudaStream_t st, double* stats, int shard, int n_shards) {
  NvtxRange nvtx_range("hmgp:assemble(K3-K5)");
  h.g = &g;
  h.p = p;
  h.eps = eps;
  h.fixed_rank = fixed_rank;
  h.rank_k = rank_k;
  h.max_rank = max_rank;
  h.nodes.clear();
  h.leaf_node.clear();
  build_payload(h, g, 0, true);
  const int L = static_cast<int>(h.leaf_node.size());

  // ---- ACA over admissible leaves, in chunks bounded by workspace size ----
  std::vector<int> rank(L, -1);
  std::vector<int> mm(L), nn(L), r0v(L), c0v(L);
  for (int k = 0; k < L; ++k) {
    const HNode& nd = h.nodes[h.leaf_node[k]];
    r0v[k] = g.nbeg[nd.row];
    c0v[k] = g.nbeg[nd.col];
    mm[k] = g.nend[nd.row] - r0v[k];
    nn[k] = g.nend[nd.col] - c0v[k];
  }
  h.leaf_begin = 0;
  h.leaf_end = -1;
  if (n_shards > 1) {  // cost: dense m n entries, admissible (m + n) r with r ~ 16
    std::vector<double> cost(L);
    for (int k = 0; k < L; ++k)
      cost[k] = h.nodes[h.leaf_node[k]].kind == LOWRANK ? 16.0 * (mm[k] + nn[k]) : (double)mm[k] * nn[k];
    std::vector<int> b(n_shards + 1);
    balanced_ranges(cost.data(), L, n_shards, b.data());
    h.leaf_begin = b[shard];
    h.leaf_end = b[shard + 1];
  }
  std::vector<int> adm, den;
  for (int k = 0; k < L; ++k)
    if (h.in_shard(k)) (h.nodes[h.leaf_node[k]].kind == LOWRANK ? adm : den).push_back(k);
  int* d_rank_tmp = dmalloc<int>(L);
  HMGP_CUDA(cudaMemsetAsync(d_rank_tmp, 0, (size_t)L * 4, st));
  int* d_err = dmalloc<int>(1);
  HMGP_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
  // Device staging buffers per chunk; results copied into the final pool after
  // the ranks are known.  We keep all chunk buffers alive until the pool copy.
  // Pass 1 gives every block a 64-column ACA capacity; a block that reaches it
  // without meeting the stopping rule is recomputed from scratch in pass 2 with
  // the full max_terms (ACA is deterministic, so the result is the same as a
  // single run with full capacity).
  struct Chunk {
    std::vector<int> leaves;
    std::vector<char> valid;
    double* buf = nullptr;
    std::vector<size_t> offU, offV;
    std::vector<int> cap;
    double* ws = nullptr;
  };
  std::vector<Chunk> chunks;
  const size_t kChunkDoubles = (size_t)1 << 30;  // 8 GiB of U/V staging per chunk
  auto max_terms_of = [&](int k) {
    int mt = std::min({mm[k], nn[k], max_rank});
    if (fixed_rank) mt = std::min(mt, rank_k);
    return mt;
  };
  auto run_pass = [&](const std::vector<int>& list, int capmax) {
    size_t i = 0;
    while (i < list.size()) {
      Chunk c;
      size_t tot = 0;
      while (i < list.size()) {
        const int k = list[i];
        const int cap = std::min(max_terms_of(k), capmax);
        const size_t need = (size_t)(mm[k] + nn[k]) * cap;
        if (!c.leaves.empty() && tot + need > kChunkDoubles) break;
        c.leaves.push_back(k);
        c.offU.push_back(tot);
        c.offV.push_back(tot + (size_t)mm[k] * cap);
        c.cap.push_back(cap);
        tot += need;
        ++i;
      }
      c.buf = dmalloc<double>(tot);
      // flags
      size_t fl = 0;
      std::vector<size_t> foff;
      for (int k : c.leaves) {
        foff.push_back(fl);
        fl += (mm[k] + 31) / 32 + (nn[k] + 31) / 32;
      }
      unsigned* d_flags = dmalloc<unsigned>(fl);
      HMGP_CUDA(cudaMemsetAsync(d_flags, 0, std::max<size_t>(1, fl) * 4, st));
      std::vector<AcaItem> items;
      for (size_t t = 0; t < c.leaves.size(); ++t) {
        const int k = c.leaves[t];
        items.push_back(AcaItem{c.buf + c.offU[t], c.buf + c.offV[t], r0v[k], c0v[k], mm[k], nn[k],
                                c.cap[t], max_terms_of(k), d_rank_tmp + k, d_flags + foff[t]});
      }
      AcaItem* d_items = upload(items, st);
      k_aca<<<(int)items.size(), kAcaThreads, 0, st>>>(d_items, p, g.d_xt, g.n, g.dim, eps,
                                                       fixed_rank ? 1 : 0);
      HMGP_LAUNCH_CHECK();
      // K5: rank > 16 -> join_truncate (FixedAccuracy only)
      if (!fixed_rank) {
        size_t wsd = 0;
        std::vector<size_t> woff;
        for (size_t t = 0; t < c.leaves.size(); ++t) {
          const int k = c.leaves[t];
          woff.push_back(wsd);
          wsd += c.cap[t] <= 16 ? 0 : trunc_ws_for(mm[k], nn[k], c.cap[t]);
        }
        c.ws = dmalloc<double>(wsd);
        std::vector<TruncItem> ti;
        for (size_t t = 0; t < c.leaves.size(); ++t) {
          const int k = c.leaves[t];
          if (c.cap[t] <= 16) continue;
          TruncItem x{};
          x.U = c.buf + c.offU[t];
          x.V = c.buf + c.offV[t];
          x.m = mm[k];
          x.n = nn[k];
          x.rank = d_rank_tmp + k;
          x.cond = 1;
          x.cap = c.cap[t];
          x.rcap = c.cap[t];
          x.ws = c.ws + woff[t];
          ti.push_back(x);
        }
        std::vector<TruncItem> tbig, tsmall, tmid, tdef;
        for (const TruncItem& x : ti) {
          const int rt = trunc_route(x.m, x.n, x.rcap);
          (rt == 2 ? tbig : rt == 1 ? tmid : rt == 3 ? tdef : tsmall).push_back(x);
        }
        for (int pass = 0; pass < 2; ++pass) {  // medium blocks: one CTA pair each
          std::vector<TruncItem>& tm = pass ? tdef : tmid;
          if (tm.empty()) continue;
          TruncItem* d_tm = upload(tm, st);
          std::vector<int> off(tm.size() + 1);
          for (size_t q = 0; q <= tm.size(); ++q) off[q] = (int)q;
          int* d_off = upload(off, st);
          int* d_dfr = nullptr;
          if (pass == 1) d_dfr = dev_alloc_n<int>(tm.size());
          launch_truncate_pair(d_tm, d_off, (int)tm.size(), eps, d_err, st, d_dfr);
          HMGP_CUDA(cudaStreamSynchronize(st));
          dev_free(d_tm);
          dev_free(d_off);
          dev_free(d_dfr);
        }
        if (!tbig.empty()) {  // large blocks: one 8-CTA cluster each
          TruncItem* d_tb = upload(tbig, st);
          std::vector<int> off(tbig.size() + 1);
          for (size_t q = 0; q <= tbig.size(); ++q) off[q] = (int)q;
          int* d_off = upload(off, st);
          launch_truncate_cluster(d_tb, d_off, (int)tbig.size(), eps, d_err, st, false);
          HMGP_CUDA(cudaStreamSynchronize(st));
          dev_free(d_tb);
          dev_free(d_off);
        }
        if (!tsmall.empty()) {
          TruncItem* d_ti = upload(tsmall, st);
          int sw = 0, smn = 0;
          for (const TruncItem& x : tsmall) trunc_smem_dims(x.m, x.n, &sw, &smn);
          launch_truncate(d_ti, (int)tsmall.size(), eps, d_err, st, sw, smn);
          HMGP_CUDA(cudaStreamSynchronize(st));
          dev_free(d_ti);
        }
        dev_free(c.ws);
        c.ws = nullptr;
      }
      HMGP_CUDA(cudaStreamSynchronize(st));
      dev_free(d_items);
      dev_free(d_flags);
      c.valid.assign(c.leaves.size(), 1);
      chunks.push_back(std::move(c));
    }
  };
  run_pass(adm, 64);
  {
    HMGP_CUDA(cudaMemcpyAsync(rank.data(), d_rank_tmp, (size_t)L * 4, cudaMemcpyDeviceToHost, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
    std::vector<int> redo;
    for (Chunk& c : chunks)
      for (size_t t = 0; t < c.leaves.size(); ++t)
        if (rank[c.leaves[t]] < 0) {
          c.valid[t] = 0;
          redo.push_back(c.leaves[t]);
        }
    if (!redo.empty()) run_pass(redo, 1 << 30);
  }
  {
  }
  phase_mark(PH_ACA);
  HMGP_CUDA(cudaMemcpyAsync(rank.data(), d_rank_tmp, (size_t)L * 4, cudaMemcpyDeviceToHost, st));
  int herr = 0;
  HMGP_CUDA(cudaMemcpyAsync(&herr, d_err, 4, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  if (herr) throw Error(6, "assemble: truncation workspace overflow");

  // ---- coarsening decision + final pool layout ----
  h.leaf.assign(L, LeafDev{});
  std::vector<int> kind(L);
  size_t total = 0;
  std::vector<size_t> off(L);
  for (int k = 0; k < L; ++k) {
    const int m = mm[k], n = nn[k];
    int kd = h.nodes[h.leaf_node[k]].kind;
    if (kd == LOWRANK && static_cast<long>(m + n) * rank[k] >= static_cast<long>(m) * n) kd = DENSE;
    kind[k] = kd;
    off[k] = total;
    if (!h.in_shard(k)) {  // outside this shard: no payload
      if (kd == LOWRANK) rank[k] = 0;
      continue;
    }
    if (kd == DENSE) {
      total += (size_t)m * n;
    } else {
      const int cap = lr_capacity(m, n, rank[k]);
      h.leaf[k].cap = cap;
      total += (size_t)(m + n) * cap;
    }
  }
  h.pool = dmalloc<double>(total);
  h.pool_doubles = total;
  HMGP_CUDA(cudaMemsetAsync(h.pool, 0, total * 8, st));
  std::vector<int> compact(L, 0);
  h.n_dense_leaves = h.n_lr_leaves = 0;
  for (int k = 0; k < L; ++k) {
    LeafDev& lf = h.leaf[k];
    lf.m = mm[k];
    lf.n = nn[k];
    lf.kind = kind[k];
    lf.a = h.pool + off[k];
    if (kind[k] == DENSE) {
      lf.b = nullptr;
      lf.cap = 0;
      ++h.n_dense_leaves;
    } else {
      lf.b = lf.a + (size_t)lf.m * lf.cap;
      compact[k] = rank[k];
      ++h.n_lr_leaves;
    }
    h.nodes[h.leaf_node[k]].kind = kind[k];
    if (kind[k] == DENSE) rank[k] = -1;
  }
  // dense leaves (K3)
  {
    std::vector<DenseItem> di;
    for (int k : den) di.push_back(DenseItem{h.leaf[k].a, r0v[k], c0v[k], mm[k], nn[k]});
    if (!di.empty()) {
      DenseItem* d_di = upload(di, st);
      phase_mark(PH_LAYOUT);
      k_dense_leaves<<<(int)di.size(), 256, 0, st>>>(d_di, p, g.d_xt, g.n, g.dim);
      HMGP_LAUNCH_CHECK();
      phase_mark(PH_DENSE);
      if (g_count_kernel_flops) {  // untimed counting pass (bench roofline)
        double* d_f = dmalloc<double>(1);
        HMGP_CUDA(cudaMemsetAsync(d_f, 0, 8, st));
        k_dense_flops<<<(int)di.size(), 256, 0, st>>>(d_di, p, g.d_xt, g.n, g.dim, d_f);
        HMGP_LAUNCH_CHECK();
        double fl = 0;
        HMGP_CUDA(cudaMemcpyAsync(&fl, d_f, 8, cudaMemcpyDeviceToHost, st));
        HMGP_CUDA(cudaStreamSynchronize(st));
        g_work.kernel_flops += fl;
        dev_free(d_f);
        phase_mark(PH_LAYOUT);
      }
      HMGP_CUDA(cudaStreamSynchronize(st));
      dev_free(d_di);
    }
    for (int k : den) g_work.dense_entries += (double)mm[k] * nn[k];
  }
  // ACA results -> pool (copy, or coarsen to dense U V^T)
  for (Chunk& c : chunks) {
    std::vector<CopyItem> cp;
    std::vector<OuterItem> oi;
    for (size_t t = 0; t < c.leaves.size(); ++t) {
      if (!c.valid[t]) continue;  // superseded by the full-capacity pass
      const int k = c.leaves[t];
      const double* U = c.buf + c.offU[t];
      const double* V = c.buf + c.offV[t];
      if (kind[k] == DENSE) {
        oi.push_back(OuterItem{U, V, h.leaf[k].a, mm[k], nn[k], d_rank_tmp + k});
      } else if (rank[k] > 0) {
        cp.push_back(CopyItem{U, h.leaf[k].a, (size_t)mm[k] * rank[k]});
        cp.push_back(CopyItem{V, h.leaf[k].b, (size_t)nn[k] * rank[k]});
      }
    }
    if (!cp.empty()) {
      CopyItem* d = upload(cp, st);
      k_copy<<<(int)cp.size(), 256, 0, st>>>(d);
      HMGP_LAUNCH_CHECK();
      HMGP_CUDA(cudaStreamSynchronize(st));
      dev_free(d);
    }
    if (!oi.empty()) {
      OuterItem* d = upload(oi, st);
      k_outer<<<(int)oi.size(), 256, 0, st>>>(d);
      HMGP_LAUNCH_CHECK();
      HMGP_CUDA(cudaStreamSynchronize(st));
      dev_free(d);
    }
    dev_free(c.buf);
    c.buf = nullptr;
  }
  phase_mark(PH_LAYOUT);
  dev_free(d_rank_tmp);
  dev_free(d_err);
  h.d_leaf = upload(h.leaf, st);
  h.d_rank = upload(rank, st);
  h.d_compact = upload(compact, st);
  h.rank_host = rank;
  // max diagonal of the dense diagonal leaves (hmatrix.cpp:306-313)
  {
    std::vector<int> diag;
    for (int k = 0; k < L; ++k) {
      const HNode& nd = h.nodes[h.leaf_node[k]];
      if (nd.row == nd.col && kind[k] == DENSE && h.in_shard(k)) diag.push_back(k);
    }
    int* d_diag = upload(diag, st);
    double* d_out = dmalloc<double>(1);
    k_diag_max<<<1, 256, 0, st>>>(h.d_leaf, d_diag, (int)diag.size(), d_out);
    HMGP_LAUNCH_CHECK();
    HMGP_CUDA(cudaMemcpyAsync(&h.max_diag, d_out, 8, cudaMemcpyDeviceToHost, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
    dev_free(d_diag);
    dev_free(d_out);
  }
  if (stats) {
    double entries_dense = 0;
    for (int k : den) entries_dense += (double)mm[k] * nn[k];
    stats[0] = entries_dense;
    stats[1] = (double)adm.size();
  }
}

}  // namespace hmgp_gpu
