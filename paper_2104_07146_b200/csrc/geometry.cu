// K1 cluster tree + K2 block-cluster tree on the GPU, bit-exact with the
// reference (geometry.cpp:26-154).
//
// K1 (ClusterTree::build, geometry.cpp:56-78).  The tree SHAPE depends only on
// (n, leaf_size): node [b, e) splits at b + (e-b)/2 while e-b > leaf_size.  So the
// host lays out the nodes once and the device only has to produce, per level,
// (a) every node's bounding box and split axis and (b) the new permutation.
// The reference sorts each segment by (coordinate, original index) with -0 == +0;
// that order equals the order of a per-axis GLOBAL rank computed once by a stable
// radix sort of the canonicalised coordinate bits (values in index order).  Each
// level is then ONE 64-bit radix sort keyed by (segment begin << 32 | axis rank),
// finished-leaf positions keyed by their own position so they stay put.
// Bounding boxes are (value, position)-lexicographic min / max reductions: the
// reference keeps the FIRST of equal values (std::min / std::max), which matters
// only for the sign of zero, and we reproduce even that.
//
// K2 (BlockClusterTree::build, geometry.cpp:100-154).  Level-synchronous frontier
// expansion; every node carries its base-4 DFS path key (child index i*nc+j at
// each depth), so sorting the emitted leaves by key restores the reference's
// DFS pre-order exactly.  The admissibility test dist > 0 && min(diam) <= eta*dist
// uses explicit _rn intrinsics (no FMA contraction), matching the x86-64 build.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "hmgp_internal.h"

namespace hmgp_gpu {

__device__ __forceinline__ uint64_t canon_key(double v) {
  if (v == 0.0) v = 0.0;  // -0 -> +0 (the reference compare treats them equal)
  uint64_t b = __double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_axis_keys(const double* __restrict__ x, int n, int dim, int axis,
                            uint64_t* __restrict__ keys, int* __restrict__ vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = canon_key(x[(size_t)i * dim + axis]);
  vals[i] = i;
}

__global__ void k_scatter_rank(const int* __restrict__ sorted_idx, int n, int* __restrict__ rank) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) rank[sorted_idx[k]] = k;
}

// One CTA per node of the level: bbox (first-occurrence min/max) and axis.
__global__ void k_level_bbox(const double* __restrict__ x, int dim, const int* __restrict__ perm,
                             const int* __restrict__ lvl_nodes, const int* __restrict__ nbeg,
                             const int* __restrict__ nend, double* __restrict__ box,
                             int* __restrict__ axis_out) {
  const int node = lvl_nodes[blockIdx.x];
  const int b = nbeg[node], e = nend[node];
  __shared__ double sv[2][3][32];
  __shared__ int sp[2][3][32];
  double lo[3], hi[3];
  int plo[3], phi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = 0;
    hi[d] = 0;
    plo[d] = 0x7fffffff;
    phi[d] = 0x7fffffff;
  }
  for (int k = b + threadIdx.x; k < e; k += blockDim.x) {
    const double* p = x + (size_t)perm[k] * dim;
    for (int d = 0; d < dim; ++d) {
      const double v = p[d];
      if (plo[d] == 0x7fffffff || v < lo[d]) {  // strictly smaller, or first seen
        lo[d] = v;
        plo[d] = k;
      }
      if (phi[d] == 0x7fffffff || v > hi[d]) {
        hi[d] = v;
        phi[d] = k;
      }
    }
  }
  // warp reduce: lexicographic (value, position); equal values keep the lower position
  for (int d = 0; d < dim; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      double v2 = __shfl_xor_sync(0xffffffffu, lo[d], o);
      int p2 = __shfl_xor_sync(0xffffffffu, plo[d], o);
      if (p2 != 0x7fffffff && (plo[d] == 0x7fffffff || v2 < lo[d] || (v2 == lo[d] && p2 < plo[d]))) {
        lo[d] = v2;
        plo[d] = p2;
      }
      v2 = __shfl_xor_sync(0xffffffffu, hi[d], o);
      p2 = __shfl_xor_sync(0xffffffffu, phi[d], o);
      if (p2 != 0x7fffffff && (phi[d] == 0x7fffffff || v2 > hi[d] || (v2 == hi[d] && p2 < phi[d]))) {
        hi[d] = v2;
        phi[d] = p2;
      }
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0)
    for (int d = 0; d < dim; ++d) {
      sv[0][d][w] = lo[d];
      sp[0][d][w] = plo[d];
      sv[1][d][w] = hi[d];
      sp[1][d][w] = phi[d];
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int d = 0; d < dim; ++d) {
      double l = 0, h = 0;
      int pl = 0x7fffffff, ph = 0x7fffffff;
      for (int q = 0; q < nw; ++q) {
        const double a = sv[0][d][q], c = sv[1][d][q];
        const int pa = sp[0][d][q], pc = sp[1][d][q];
        if (pa != 0x7fffffff && (pl == 0x7fffffff || a < l || (a == l && pa < pl))) {
          l = a;
          pl = pa;
        }
        if (pc != 0x7fffffff && (ph == 0x7fffffff || c > h || (c == h && pc < ph))) {
          h = c;
          ph = pc;
        }
      }
      box[node * 6 + d] = l;
      box[node * 6 + 3 + d] = h;
    }
    for (int d = dim; d < 3; ++d) box[node * 6 + d] = box[node * 6 + 3 + d] = 0.0;
    // longest axis, ties to the lower axis (geometry.cpp:64-66)
    int ax = 0;
    double ext = __dsub_rn(box[node * 6 + 3], box[node * 6 + 0]);
    for (int d = 1; d < dim; ++d) {
      const double e2 = __dsub_rn(box[node * 6 + 3 + d], box[node * 6 + d]);
      if (e2 > ext) {
        ext = e2;
        ax = d;
      }
    }
    axis_out[node] = ax;
  }
}

__global__ void k_default_keys(int n, uint64_t* __restrict__ keys) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) keys[k] = (uint64_t)k << 32;
}

// Keys for the positions of splitting nodes: (begin << 32) | rank_axis(perm[k]).
__global__ void k_split_keys(const int* __restrict__ perm, const int* __restrict__ split_nodes,
                             const int* __restrict__ nbeg, const int* __restrict__ nend,
                             const int* __restrict__ axis, const int* __restrict__ ranks, int n,
                             uint64_t* __restrict__ keys) {
  const int node = split_nodes[blockIdx.x];
  const int b = nbeg[node], e = nend[node];
  const int* rk = ranks + (size_t)axis[node] * n;
  for (int k = b + threadIdx.x; k < e; k += blockDim.x)
    keys[k] = ((uint64_t)b << 32) | (uint32_t)rk[perm[k]];
}

__global__ void k_inverse_perm(const int* __restrict__ perm, int n, int* __restrict__ iperm) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) iperm[perm[k]] = k;
}

__global__ void k_gather_coords(const double* __restrict__ x, const int* __restrict__ perm, int n,
                                int dim, double* __restrict__ xt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int p = perm[k];
  for (int d = 0; d < dim; ++d) xt[(size_t)d * n + k] = x[(size_t)p * dim + d];  // SoA
}

// ---------------------------------------------------------------- K2 ------
struct FrontItem {
  int row, col;
  uint64_t key;
  int depth;
};

__device__ __forceinline__ double box_diam(const double* b, int dim) {
  double s = 0.0;
  for (int d = 0; d < dim; ++d) {
    const double e = __dsub_rn(b[3 + d], b[d]);
    s = __dadd_rn(s, __dmul_rn(e, e));
  }
  return __dsqrt_rn(s);
}
__device__ __forceinline__ double box_dist(const double* a, const double* b, int dim) {
  double s = 0.0;
  for (int d = 0; d < dim; ++d) {
    const double g = fmax(0.0, fmax(__dsub_rn(b[d], a[3 + d]), __dsub_rn(a[d], b[3 + d])));
    s = __dadd_rn(s, __dmul_rn(g, g));
  }
  return __dsqrt_rn(s);
}

// Expand one frontier level.  Every node is also recorded (for the host-side
// payload structure); leaves additionally go to the leaf list.
__global__ void k_block_expand(const FrontItem* __restrict__ cur, int ncur,
                               const double* __restrict__ box, const int* __restrict__ left,
                               const int* __restrict__ right, int dim, double eta, int maxdepth,
                               FrontItem* __restrict__ next, int* __restrict__ nnext,
                               BlockNodeRec* __restrict__ all, int* __restrict__ nall) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ncur) return;
  const FrontItem it = cur[t];
  const double* rb = box + it.row * 6;
  const double* cb = box + it.col * 6;
  const double dist = box_dist(rb, cb, dim);
  const double dmin = fmin(box_diam(rb, dim), box_diam(cb, dim));
  const bool rleaf = left[it.row] < 0, cleaf = left[it.col] < 0;
  int tag;
  if (dist > 0.0 && dmin <= __dmul_rn(eta, dist))
    tag = 0;
  else if (rleaf && cleaf)
    tag = 1;
  else
    tag = 2;
  const int slot = atomicAdd(nall, 1);
  all[slot] = BlockNodeRec{it.row, it.col, tag, it.depth, it.key};
  if (tag != 2) return;
  int rp[2] = {it.row, -1}, cp[2] = {it.col, -1};
  int nr = 1, nc = 1;
  if (!rleaf) {
    rp[0] = left[it.row];
    rp[1] = right[it.row];
    nr = 2;
  }
  if (!cleaf) {
    cp[0] = left[it.col];
    cp[1] = right[it.col];
    nc = 2;
  }
  const int base = atomicAdd(nnext, nr * nc);
  const int shift = 2 * (maxdepth - 1 - it.depth);
  for (int i = 0; i < nr; ++i)
    for (int j = 0; j < nc; ++j) {
      const uint64_t digit = (uint64_t)(i * nc + j);
      next[base + i * nc + j] = FrontItem{rp[i], cp[j], it.key | (digit << shift), it.depth + 1};
    }
}

// ------------------------------------------------------------ host side ----
namespace {
template <class T>
T* dalloc(size_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  HMGP_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

int host_layout(Geometry& g, int b, int e, int level) {
  const int id = static_cast<int>(g.nbeg.size());
  g.nbeg.push_back(b);
  g.nend.push_back(e);
  g.nleft.push_back(-1);
  g.nright.push_back(-1);
  g.nlevel.push_back(level);
  if (e - b <= g.leaf_size) return id;
  const int mid = b + (e - b) / 2;
  const int l = host_layout(g, b, mid, level + 1);
  const int r = host_layout(g, mid, e, level + 1);
  g.nleft[id] = l;
  g.nright[id] = r;
  return id;
}
}  // namespace

// Level-synchronous K2 frontier from the root pair (root_row, root_col) over the
// node arrays box/left/right (one tree, or two trees concatenated for a
// rectangular block tree); returns every node in DFS pre-order (geometry.cpp:
// 100-154).  maxdepth bounds the block depth (<= deeper tree's depth + 1).
std::vector<BlockNodeRec> block_frontier(const double* d_box, const int* d_left, const int* d_right,
                                         int dim, double eta, int maxdepth, int root_row,
                                         int root_col, cudaStream_t st) {
  std::vector<FrontItem> root{FrontItem{root_row, root_col, 0ull, 0}};
  size_t cap_front = 16, cap_all = 64;
  FrontItem* f_cur = dalloc<FrontItem>(cap_front);
  FrontItem* f_next = dalloc<FrontItem>(cap_front);
  HMGP_CUDA(cudaMemcpyAsync(f_cur, root.data(), sizeof(FrontItem), cudaMemcpyHostToDevice, st));
  BlockNodeRec* d_all = dalloc<BlockNodeRec>(cap_all);
  int* d_cnt = dalloc<int>(2);
  int ncur = 1, nall = 0;
  for (int level = 0; ncur > 0; ++level) {
    // capacity: each item emits <= 4 children and 1 record
    if ((size_t)ncur * 4 > cap_front) {
      size_t nc = std::max<size_t>((size_t)ncur * 4, cap_front * 2);
      FrontItem* a = dalloc<FrontItem>(nc);
      FrontItem* b = dalloc<FrontItem>(nc);
      HMGP_CUDA(cudaMemcpyAsync(a, f_cur, ncur * sizeof(FrontItem), cudaMemcpyDeviceToDevice, st));
      HMGP_CUDA(cudaStreamSynchronize(st));
      cudaFree(f_cur);
      cudaFree(f_next);
      f_cur = a;
      f_next = b;
      cap_front = nc;
    }
    if ((size_t)nall + ncur > cap_all) {
      size_t nc = std::max<size_t>((size_t)nall + ncur, cap_all * 2);
      BlockNodeRec* a = dalloc<BlockNodeRec>(nc);
      HMGP_CUDA(cudaMemcpyAsync(a, d_all, nall * sizeof(BlockNodeRec), cudaMemcpyDeviceToDevice, st));
      HMGP_CUDA(cudaStreamSynchronize(st));
      cudaFree(d_all);
      d_all = a;
      cap_all = nc;
    }
    int init[2] = {0, nall};
    HMGP_CUDA(cudaMemcpyAsync(d_cnt, init, 8, cudaMemcpyHostToDevice, st));
    k_block_expand<<<(ncur + 127) / 128, 128, 0, st>>>(f_cur, ncur, d_box, d_left, d_right, dim, eta,
                                                       maxdepth, f_next, d_cnt, d_all, d_cnt + 1);
    HMGP_LAUNCH_CHECK();
    int out[2];
    HMGP_CUDA(cudaMemcpyAsync(out, d_cnt, 8, cudaMemcpyDeviceToHost, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
    ncur = out[0];
    nall = out[1];
    std::swap(f_cur, f_next);
  }
  // DFS pre-order of all nodes: sort by (key, depth) -> parent before first child.
  std::vector<BlockNodeRec> nodes(nall);
  HMGP_CUDA(cudaMemcpyAsync(nodes.data(), d_all, nall * sizeof(BlockNodeRec), cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  std::sort(nodes.begin(), nodes.end(), [](const BlockNodeRec& a, const BlockNodeRec& b) {
    return a.key != b.key ? a.key < b.key : a.depth < b.depth;
  });
  cudaFree(f_cur);
  cudaFree(f_next);
  cudaFree(d_all);
  cudaFree(d_cnt);
  return nodes;
}

// Rectangular block tree BlockClusterTree(rows, cols, eta) (geometry.cpp:100-154)
// over two cluster trees: their node arrays are concatenated (column-tree ids
// offset by the row tree's node count) and the same frontier kernel runs from
// the pair of roots.  Leaves in DFS order as hmgp_block rows (tree positions).
void block_tree_rect(const Geometry& R, const Geometry& Cg, double eta, std::vector<int>& out5,
                     int& n_adm, int& n_dense, cudaStream_t st) {
  if (R.dim != Cg.dim) throw std::invalid_argument("block tree: row and column trees differ in dimension");
  const int nr = static_cast<int>(R.nbeg.size()), nc = static_cast<int>(Cg.nbeg.size()), dim = R.dim;
  std::vector<int> left(nr + nc), right(nr + nc);
  for (int i = 0; i < nr; ++i) {
    left[i] = R.nleft[i];
    right[i] = R.nright[i];
  }
  for (int i = 0; i < nc; ++i) {
    left[nr + i] = Cg.nleft[i] < 0 ? -1 : Cg.nleft[i] + nr;
    right[nr + i] = Cg.nright[i] < 0 ? -1 : Cg.nright[i] + nr;
  }
  int* d_l = dalloc<int>(nr + nc);
  int* d_r = dalloc<int>(nr + nc);
  double* d_b = dalloc<double>((size_t)(nr + nc) * 6);
  HMGP_CUDA(cudaMemcpyAsync(d_l, left.data(), 4ull * (nr + nc), cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(d_r, right.data(), 4ull * (nr + nc), cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(d_b, R.d_box, 48ull * nr, cudaMemcpyDeviceToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(d_b + (size_t)nr * 6, Cg.d_box, 48ull * nc, cudaMemcpyDeviceToDevice, st));
  const std::vector<BlockNodeRec> nodes =
      block_frontier(d_b, d_l, d_r, dim, eta, std::max(R.depth, Cg.depth) + 1, 0, nr, st);
  cudaFree(d_l);
  cudaFree(d_r);
  cudaFree(d_b);
  out5.clear();
  n_adm = n_dense = 0;
  for (const BlockNodeRec& b : nodes) {
    if (b.tag == 2) continue;
    const int c = b.col - nr;
    out5.insert(out5.end(), {R.nbeg[b.row], R.nend[b.row], Cg.nbeg[c], Cg.nend[c], b.tag});
    (b.tag == 0 ? n_adm : n_dense)++;
  }
}

void geometry_build(Geometry& g, cudaStream_t st) {
  NvtxRange nvtx_range("hmgp:geometry(K1-K2)");
  const int n = g.n, dim = g.dim;
  // ---- host tree shape (pre-order ids, like the reference's recursion) ----
  g.nbeg.clear();
  g.nend.clear();
  g.nleft.clear();
  g.nright.clear();
  g.nlevel.clear();
  host_layout(g, 0, n, 0);
  const int nn = static_cast<int>(g.nbeg.size());
  int depth = 0;
  for (int l : g.nlevel) depth = std::max(depth, l);
  g.depth = depth;
  std::vector<std::vector<int>> lv(depth + 1), sp(depth + 1);
  for (int i = 0; i < nn; ++i) {
    lv[g.nlevel[i]].push_back(i);
    if (g.nleft[i] >= 0) sp[g.nlevel[i]].push_back(i);
  }

  int* d_nbeg = dalloc<int>(nn);
  int* d_nend = dalloc<int>(nn);
  int* d_left = dalloc<int>(nn);
  int* d_right = dalloc<int>(nn);
  int* d_axis = dalloc<int>(nn);
  int* d_lvl = dalloc<int>(nn);
  HMGP_CUDA(cudaMemcpyAsync(d_nbeg, g.nbeg.data(), nn * 4, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(d_nend, g.nend.data(), nn * 4, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(d_left, g.nleft.data(), nn * 4, cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(d_right, g.nright.data(), nn * 4, cudaMemcpyHostToDevice, st));
  g.d_box = dalloc<double>((size_t)nn * 6);

  // ---- per-axis global ranks (stable radix sort, values in index order) ----
  uint64_t *k0 = dalloc<uint64_t>(n), *k1 = dalloc<uint64_t>(n);
  int *v0 = dalloc<int>(n), *v1 = dalloc<int>(n);
  int* d_ranks = dalloc<int>((size_t)n * dim);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, v1, n, 0, 64, st);
  void* d_tmp = dalloc<char>(tmp_bytes);
  const int TB = 256, GB = (n + TB - 1) / TB;
  for (int a = 0; a < dim; ++a) {
    k_axis_keys<<<GB, TB, 0, st>>>(g.d_x, n, dim, a, k0, v0);
    HMGP_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, k0, k1, v0, v1, n, 0, 64, st));
    k_scatter_rank<<<GB, TB, 0, st>>>(v1, n, d_ranks + (size_t)a * n);
  }
  HMGP_LAUNCH_CHECK();

  // ---- level sweep ----
  int* d_perm = dalloc<int>(n);
  int* d_perm2 = dalloc<int>(n);
  {
    std::vector<int> iota(n);
    for (int i = 0; i < n; ++i) iota[i] = i;
    HMGP_CUDA(cudaMemcpyAsync(d_perm, iota.data(), (size_t)n * 4, cudaMemcpyHostToDevice, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
  }
  for (int l = 0; l <= depth; ++l) {
    HMGP_CUDA(cudaMemcpyAsync(d_lvl, lv[l].data(), lv[l].size() * 4, cudaMemcpyHostToDevice, st));
    k_level_bbox<<<(int)lv[l].size(), 256, 0, st>>>(g.d_x, dim, d_perm, d_lvl, d_nbeg, d_nend,
                                                    g.d_box, d_axis);
    if (sp[l].empty()) {
      HMGP_CUDA(cudaStreamSynchronize(st));
      continue;
    }
    HMGP_CUDA(cudaMemcpyAsync(d_lvl, sp[l].data(), sp[l].size() * 4, cudaMemcpyHostToDevice, st));
    k_default_keys<<<GB, TB, 0, st>>>(n, k0);
    k_split_keys<<<(int)sp[l].size(), 256, 0, st>>>(d_perm, d_lvl, d_nbeg, d_nend, d_axis,
                                                    d_ranks, n, k0);
    HMGP_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, k0, k1, d_perm, d_perm2, n, 0, 64,
                                              st));
    std::swap(d_perm, d_perm2);
    HMGP_CUDA(cudaStreamSynchronize(st));  // d_lvl is reused next level
  }
  HMGP_LAUNCH_CHECK();
  g.d_perm = d_perm;
  g.d_iperm = dalloc<int>(n);
  k_inverse_perm<<<GB, TB, 0, st>>>(d_perm, n, g.d_iperm);
  g.d_xt = dalloc<double>((size_t)n * dim);
  k_gather_coords<<<GB, TB, 0, st>>>(g.d_x, d_perm, n, dim, g.d_xt);
  HMGP_LAUNCH_CHECK();

  // ---- K2: block tree frontier ----
  g.bnodes = block_frontier(g.d_box, d_left, d_right, dim, g.eta, depth + 1, 0, 0, st);
  const int nall = static_cast<int>(g.bnodes.size());
  // link children: a stack walk over the pre-order
  g.bkids.assign(nall, {});
  {
    std::vector<int> stack;
    for (int i = 0; i < nall; ++i) {
      while (!stack.empty() && g.bnodes[stack.back()].depth >= g.bnodes[i].depth) stack.pop_back();
      if (!stack.empty()) g.bkids[stack.back()].push_back(i);
      if (g.bnodes[i].tag == 2) stack.push_back(i);
    }
  }
  g.leaves.clear();
  g.n_adm = g.n_dense = 0;
  for (int i = 0; i < nall; ++i)
    if (g.bnodes[i].tag != 2) {
      g.leaves.push_back(i);
      (g.bnodes[i].tag == 0 ? g.n_adm : g.n_dense)++;
    }

  // keep node arrays on device for later kernels
  g.d_nbeg = d_nbeg;
  g.d_nend = d_nend;
  g.d_left = d_left;
  g.d_right = d_right;
  g.axis.resize(nn);
  HMGP_CUDA(cudaMemcpyAsync(g.axis.data(), d_axis, nn * 4, cudaMemcpyDeviceToHost, st));
  g.box.resize((size_t)nn * 6);
  HMGP_CUDA(cudaMemcpyAsync(g.box.data(), g.d_box, (size_t)nn * 6 * 8, cudaMemcpyDeviceToHost, st));
  g.perm.resize(n);
  HMGP_CUDA(cudaMemcpyAsync(g.perm.data(), d_perm, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  g.iperm.resize(n);
  for (int k = 0; k < n; ++k) g.iperm[g.perm[k]] = k;

  cudaFree(d_axis);
  cudaFree(d_lvl);
  cudaFree(k0);
  cudaFree(k1);
  cudaFree(v0);
  cudaFree(v1);
  cudaFree(d_ranks);
  cudaFree(d_tmp);
  cudaFree(d_perm2);
}

void geometry_free(Geometry& g) {
  cudaFree(g.d_x);
  cudaFree(g.d_xt);
  cudaFree(g.d_perm);
  cudaFree(g.d_iperm);
  cudaFree(g.d_box);
  cudaFree(g.d_nbeg);
  cudaFree(g.d_nend);
  cudaFree(g.d_left);
  cudaFree(g.d_right);
  g.d_x = g.d_xt = g.d_box = nullptr;
  g.d_perm = g.d_iperm = g.d_nbeg = g.d_nend = g.d_left = g.d_right = nullptr;
}

}  // namespace hmgp_gpu
