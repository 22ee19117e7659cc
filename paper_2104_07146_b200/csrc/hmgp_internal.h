// Internal (non-ABI) data structures of the hmgp B200 library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <memory>
#include <vector>

#include "matern.cuh"

namespace hmgp_gpu {

// Block-tree node as emitted by the device frontier expansion (K2).
struct BlockNodeRec {
  int row, col;
  int tag;  // 0 admissible, 1 dense, 2 split
  int depth;
  uint64_t key;  // base-4 DFS path key
};

// Cluster tree + block tree for one point set (θ-independent).
struct Geometry {
  int n = 0, dim = 2, leaf_size = 32, depth = 0;
  double eta = 2.0;
  // host tree (pre-order node ids, same numbering as the reference recursion)
  std::vector<int> nbeg, nend, nleft, nright, nlevel, axis;
  std::vector<double> box;  // 6 per node: lo[3], hi[3]
  std::vector<int> perm, iperm;
  // block tree in DFS pre-order; bkids[i] row-major children
  std::vector<BlockNodeRec> bnodes;
  std::vector<std::vector<int>> bkids;
  std::vector<int> leaves;  // indices into bnodes, DFS order
  int n_adm = 0, n_dense = 0;
  // device
  double* d_x = nullptr;   // AoS input coordinates (original order)
  double* d_xt = nullptr;  // SoA coordinates in tree order: xt[d*n + k]
  int *d_perm = nullptr, *d_iperm = nullptr;
  double* d_box = nullptr;
  int *d_nbeg = nullptr, *d_nend = nullptr, *d_left = nullptr, *d_right = nullptr;
};

void geometry_build(Geometry& g, cudaStream_t st);
void geometry_free(Geometry& g);
// rectangular BlockClusterTree(rows, cols, eta): leaves in DFS order, 5 ints each
// (row_begin, row_end, col_begin, col_end, tag 0 admissible / 1 dense)
void block_tree_rect(const Geometry& rows, const Geometry& cols, double eta, std::vector<int>& out5,
                     int& n_adm, int& n_dense, cudaStream_t st);

// ---------------------------------------------------------------- H-matrix --
enum Kind { BRANCH = 0, DENSE = 1, LOWRANK = 2 };

// Device-side description of one stored leaf.  Dense: a = D (m x n, ld m).
// Low-rank: a = U (m x cap, ld m), b = V (n x cap, ld n); rank/compact live in
// separate device int arrays so kernels can grow/shrink them without the host.
struct LeafDev {
  double* a;
  double* b;
  int m, n;
  int kind;
  int cap;
};

// Host payload node (mirror of HBlock, hblock.hpp:17-45).
struct HNode {
  int kind = BRANCH;
  int row = 0, col = 0;     // cluster node ids
  int kids[4] = {-1, -1, -1, -1};  // row-major, -1 = null (upper mirror)
  int kr = 1, kc = 1;
  int leaf = -1;  // index into the leaf table (stored leaves)
};

struct DeviceArena;

struct HMat {
  Geometry* g = nullptr;
  MaternDev p{};
  double eps = 1e-6;
  bool fixed_rank = false;
  int rank_k = 16, max_rank = 256;
  std::vector<HNode> nodes;  // node 0 = root
  std::vector<int> leaf_node;  // stored leaf -> node id (DFS order)
  std::vector<LeafDev> leaf;   // host copy of the table
  LeafDev* d_leaf = nullptr;   // device copy
  int* d_rank = nullptr;       // per stored leaf (low-rank: rank; dense: -1)
  int* d_compact = nullptr;
  std::vector<int> rank_host;  // snapshot after assembly
  double* pool = nullptr;      // one allocation for all payload
  size_t pool_doubles = 0;
  double max_diag = 0.0;
  int n_dense_leaves = 0, n_lr_leaves = 0;
  // leaf-range shard: only stored leaves [leaf_begin, leaf_end)
  // carry payload; a partial H-matrix is refused by matvec / factorize / to_dense
  int leaf_begin = 0, leaf_end = -1;
  bool partial() const { return leaf_begin != 0 || (leaf_end >= 0 && leaf_end != (int)leaf.size()); }
  bool in_shard(int k) const { return k >= leaf_begin && (leaf_end < 0 || k < leaf_end); }
  ~HMat();
};

// Assembly (K3 dense leaves, K4 batched ACA + K5 truncation), hmatrix.cpp:174-221.
// shard/n_shards > 1: assemble only the shard-th of n_shards contiguous,
// cost-balanced ranges of the DFS-ordered stored-leaf list (balanced_ranges).
void assemble(HMat& h, Geometry& g, const MaternDev& p, double eps, bool fixed_rank, int rank_k,
              int max_rank, cudaStream_t st, double* stats, int shard = 0, int n_shards = 1);
// bounds[0..parts]: contiguous ranges of cost[0..L) with near-equal sums
void balanced_ranges(const double* cost, int L, int parts, int* bounds);

MaternDev make_matern(double sigma2, double ell, double nu, double tau2);

// ------------------------------------------------------------ kernels API --
// Batched low-rank update / recompression item (one CTA each).  The target
// holds U (m x cap, ld m), V (n x cap, ld n) with *rank current columns.  Optional
// appended columns alpha*P (rows [pro, pro+pr) of U) and Q (rows [qro, qro+qr) of V)
// with `add` columns (hblock.cpp:186-199).  With cols = rank + add the condition
// decides between a plain append and a recompression of the concatenation
// (hblock.cpp:127-162 with empty P, Q — every reference call site):
//   cond 0: cols > 0 (compress_low_rank)   1: cols > 16 (fill_leaf)
//   cond 2: cols > compact + 16 (watermark) 3: cols > 48 (product accumulation)
//   cond 4: never (pure append)
struct TruncItem {
  double* U;
  double* V;
  int m, n;
  int* rank;
  int* compact;  // optional; set to the new column count after the op when cond 0/2
  int cond;
  int cap;  // target column capacity
  const double* P;
  const double* Q;
  int ldp, ldq, pr, qr, pro, qro;
  const int* addp;  // device column count of P (nullptr -> addv)
  int addv;
  double alpha;
  int rcap;    // workspace column capacity (>= rank + add)
  double* ws;  // trunc_ws_doubles(m, n, rcap)
  // optional fused post-op (trsm_lower_t with a dense leaf, hfactor.cpp:198-202):
  // V <- L^{-1} V (L n x n lower, stored diagonal), then V rows /= d (LDL)
  const double* post_L;
  int post_ldl_ld;
  const double* post_d;
};
size_t trunc_ws_doubles(int m, int n, int rcap);
// grow the per-launch shared-memory dims for an item that can take the small-block path
void trunc_smem_dims(int m, int n, int* smem_w, int* smem_mn);
void launch_truncate(const TruncItem* d_items, int count, double eps, int* d_err, cudaStream_t st,
                     int smem_w, int smem_mn);
// large blocks: one 8-CTA cluster per target sequence (distributed Householder)
bool trunc_use_cluster(int m, int n);
size_t trunc_ws_doubles_cluster(int m, int n, int rcap);
void launch_truncate_cluster(const TruncItem* d_items, const int* d_off, int targets, double eps,
                             int* d_err, cudaStream_t st, bool resident = false);
// launch cluster targets of this size with the resident (pair / register) dispatch
bool trunc_cluster_resident(int m, int n);
// medium blocks: one CTA pair (U side, V side) per target sequence, factors in smem
bool trunc_use_pair(int m, int n, int rcap);
size_t trunc_ws_doubles_pair(int m, int n, int rcap);
// d_defer: nullptr, or `targets` device ints: items that do not fit the pair
// layout are handed over to the 8-CTA cluster kernel (same launch sequence)
void launch_truncate_pair(const TruncItem* d_items, const int* d_off, int targets, double eps,
                          int* d_err, cudaStream_t st, int* d_defer = nullptr);
// 0 single CTA (small), 1 CTA pair, 2 8-CTA cluster, 3 pair handing over to the
// cluster kernel what does not fit; workspace for that route
int trunc_route(int m, int n, int rcap);
size_t trunc_ws_for(int m, int n, int rcap);
void truncate_hist_enable(bool on);
void truncate_launch_slot(int idx, cudaStream_t st);
void truncate_launch_read(std::vector<unsigned long long>& mx, std::vector<unsigned long long>& sq);
void truncate_hist_print();
// per-target ordered sequences: CTA b runs items[off[b]..off[b+1]) in order
void launch_truncate_seq(const TruncItem* d_items, const int* d_off, int targets, double eps,
                         int* d_err, cudaStream_t st, int smem_w, int smem_mn);

}  // namespace hmgp_gpu
