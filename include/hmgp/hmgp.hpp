// hmgp/hmgp.hpp — header-only C++ drop-in for the reference's hot-path API
// (/root/reference/proj/include/hmgp/{geometry,covkernel,hmatrix,hfactor,
// pipeline,loglik,krige}.hpp), implemented over the C ABI in ../hmgp_cuda.h.
//
// Same names, argument meaning and exception types as the reference:
//   std::invalid_argument, std::domain_error, std::out_of_range, hmgp::FactorError.
// Eigen is not required: vectors are hmgp::Vector (= std::vector<double>).
// Lifetimes follow the reference: an HMatrix / HFactor must not outlive the
// ClusterTree/BlockClusterTree it was built from (hmatrix.hpp:77-78).
#pragma once
#include <cmath>
#include <algorithm>
#include <cstdint>
#include <memory>
#include <utility>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../hmgp_cuda.h"

namespace hmgp {

using Vector = std::vector<double>;

// Dense column-major matrix for the n <= 4096 diagnostics (stands in for
// Eigen::MatrixXd in to_dense / lower_dense / reconstruct).
struct Matrix {
  int n_rows = 0, n_cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(int r, int c) : n_rows(r), n_cols(c), data(static_cast<size_t>(r) * c) {}
  int rows() const { return n_rows; }
  int cols() const { return n_cols; }
  double operator()(int i, int j) const { return data[static_cast<size_t>(j) * n_rows + i]; }
  double& operator()(int i, int j) { return data[static_cast<size_t>(j) * n_rows + i]; }
};

struct Location {  // geometry.hpp:11-14
  double x = 0.0;
  double y = 0.0;
};

inline double distance(const Location& a, const Location& b) {
  const double dx = a.x - b.x, dy = a.y - b.y;
  return std::sqrt(dx * dx + dy * dy);
}

struct FactorError : std::runtime_error {  // hfactor.hpp:17-22
  FactorError(const std::string& msg, int index, double value)
      : std::runtime_error(msg), pivot_index(index), pivot_value(value) {}
  int pivot_index;
  double pivot_value;
};

namespace detail {
inline void check(int rc) {
  if (rc == HMGP_OK) return;
  const std::string msg = hmgp_last_error();
  switch (rc) {
    case HMGP_EINVAL:
      throw std::invalid_argument(msg);
    case HMGP_EDOMAIN:
      throw std::domain_error(msg);
    case HMGP_ERANGE:
      throw std::out_of_range(msg);
    case HMGP_ENOTSPD:
      throw FactorError(msg, hmgp_last_pivot_index(), hmgp_last_pivot_value());
    default:
      throw std::runtime_error(msg);
  }
}
inline hmgp_ctx* context() {
  static std::shared_ptr<hmgp_ctx> ctx = [] {
    hmgp_ctx* c = nullptr;
    check(hmgp_ctx_create(0, &c));
    return std::shared_ptr<hmgp_ctx>(c, hmgp_ctx_destroy);
  }();
  return ctx.get();
}
inline std::vector<double> flat(std::span<const Location> p) {
  std::vector<double> v(2 * p.size());
  for (size_t i = 0; i < p.size(); ++i) {
    v[2 * i] = p[i].x;
    v[2 * i + 1] = p[i].y;
  }
  return v;
}
}  // namespace detail

struct MaternParams {  // covkernel.hpp:11-19
  double sigma2 = 1.0, ell = 0.1, nu = 0.5, tau2 = 0.0;
  bool valid() const {
    return std::isfinite(sigma2) && std::isfinite(ell) && std::isfinite(nu) &&
           std::isfinite(tau2) && sigma2 > 0.0 && ell > 0.0 && nu > 0.0 && tau2 >= 0.0;
  }
  void validate() const {
    if (!valid())
      throw std::invalid_argument(
          "invalid Matern parameters: need sigma2 > 0, ell > 0, nu > 0, tau2 >= 0");
  }
  hmgp_matern c() const { return hmgp_matern{sigma2, ell, nu, tau2}; }
};

struct RankControl {  // hmatrix.hpp:17-36
  enum class Mode { FixedAccuracy, FixedRank };
  Mode mode = Mode::FixedAccuracy;
  double eps = 1e-6;
  int rank = 16;
  int max_rank = 256;
  static RankControl fixed_accuracy(double e) {
    RankControl r;
    r.eps = e;
    return r;
  }
  static RankControl fixed_rank(int k) {
    RankControl r;
    r.mode = Mode::FixedRank;
    r.rank = k;
    return r;
  }
  hmgp_rank_control c() const {
    return hmgp_rank_control{mode == Mode::FixedRank ? 1 : 0, eps, rank, max_rank};
  }
};

enum class FactorForm { Cholesky, Ldl };

struct HConfig {  // pipeline.hpp:13-25
  double eta = 2.0;
  int leaf_size = 32;
  RankControl rank = RankControl::fixed_accuracy(1e-6);
  double eps_factor = -1.0;
  FactorForm form = FactorForm::Ldl;
  int threads = 1;
  double factor_eps() const {
    if (eps_factor > 0.0) return eps_factor;
    return rank.mode == RankControl::Mode::FixedAccuracy ? rank.eps : 1e-6;
  }
  hmgp_config c() const {
    return hmgp_config{eta, leaf_size, rank.c(), eps_factor, form == FactorForm::Ldl ? 1 : 0,
                       threads};
  }
};

// --------------------------------------------------------------- kernel ----
// covkernel.hpp:24-69.  Every value is computed on the device (C ABI); the
// host only validates and marshals, with the reference's exception types.
inline double bessel_k(double nu, double x) {  // covkernel.cpp:196-204
  double out = 0.0;
  detail::check(hmgp_bessel_k(detail::context(), &nu, &x, 1, 0, &out));
  return out;
}

namespace detail {
inline double bessel_k_generic(double nu, double x) {  // covkernel.cpp:170-182
  double out = 0.0;
  check(hmgp_bessel_k(context(), &nu, &x, 1, 1, &out));
  return out;
}
inline double matern_generic(double h, const MaternParams& p) {  // covkernel.cpp:184-194
  p.validate();
  const hmgp_matern m = p.c();
  double out = 0.0;
  check(hmgp_matern_values(context(), &m, &h, 1, 1, &out));
  return out;
}
}  // namespace detail

inline double matern(double h, const MaternParams& p) {  // covkernel.cpp:206-214
  p.validate();
  const hmgp_matern m = p.c();
  double out = 0.0;
  detail::check(hmgp_matern_values(detail::context(), &m, &h, 1, 0, &out));
  return out;
}

// KernelEvaluator (covkernel.hpp:41-61): entries by original index, the nugget on
// index equality only.  operator() is one device evaluation per call (API
// parity); entries() evaluates many index pairs in one launch.
class KernelEvaluator {
 public:
  KernelEvaluator(std::span<const Location> locations, const MaternParams& p)
      : xy_(detail::flat(locations)), n_(static_cast<int>(locations.size())), p_(p) {
    p.validate();
  }
  double operator()(int i, int j) const {
    double out = 0.0;
    entries(&i, &j, 1, &out);
    return out;
  }
  double at_distance(double h) const {
    const hmgp_matern m = p_.c();
    double out = 0.0;
    detail::check(hmgp_at_distance(detail::context(), &m, &h, 1, &out));
    return out;
  }
  void entries(const int* ii, const int* jj, int64_t count, double* out) const {
    const hmgp_matern m = p_.c();
    detail::check(hmgp_kernel_pairs(detail::context(), xy_.data(), n_, 2, &m, ii, jj, count, out));
  }
  const MaternParams& params() const { return p_; }

 private:
  std::vector<double> xy_;
  int n_;
  MaternParams p_;
};

// cov_block / cov_dense (covkernel.cpp:248-275)
inline Matrix cov_block(std::span<const int> rows, std::span<const int> cols,
                        std::span<const Location> locations, const MaternParams& p) {
  const KernelEvaluator k(locations, p);
  const int n = static_cast<int>(locations.size());
  for (int i : rows)
    if (i < 0 || i >= n) throw std::out_of_range("cov_block: row index out of range");
  for (int j : cols)
    if (j < 0 || j >= n) throw std::out_of_range("cov_block: col index out of range");
  Matrix block(static_cast<int>(rows.size()), static_cast<int>(cols.size()));
  std::vector<int> ii, jj;
  ii.reserve(block.data.size());
  jj.reserve(block.data.size());
  for (size_t b = 0; b < cols.size(); ++b)
    for (size_t a = 0; a < rows.size(); ++a) {
      ii.push_back(rows[a]);
      jj.push_back(cols[b]);
    }
  if (!ii.empty()) k.entries(ii.data(), jj.data(), static_cast<int64_t>(ii.size()), block.data.data());
  return block;
}

inline Matrix cov_dense(std::span<const Location> locations, const MaternParams& p) {
  const int n = static_cast<int>(locations.size());
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  return cov_block(idx, idx, locations, p);  // symmetric by construction (same pairs)
}

// ------------------------------------------------------------- geometry ----
struct Box {  // geometry.hpp:23-29, geometry.cpp:9-22
  double lo[2] = {0.0, 0.0};
  double hi[2] = {0.0, 0.0};
  double diameter() const {
    const double dx = hi[0] - lo[0], dy = hi[1] - lo[1];
    return std::sqrt(dx * dx + dy * dy);
  }
  static double distance(const Box& a, const Box& b) {
    double s = 0.0;
    for (int d = 0; d < 2; ++d) {
      const double gap = std::max({0.0, b.lo[d] - a.hi[d], a.lo[d] - b.hi[d]});
      s += gap * gap;
    }
    return std::sqrt(s);
  }
};

struct Cluster {  // geometry.hpp:33-42 (ranges of the tree permutation)
  int begin = 0;
  int end = 0;
  Box box;
  std::unique_ptr<Cluster> left;
  std::unique_ptr<Cluster> right;
  int size() const { return end - begin; }
  bool is_leaf() const { return left == nullptr; }
};

class ClusterTree {  // geometry.hpp:44-66 (built on the GPU; perm bit-exact)
 public:
  ClusterTree(std::span<const Location> points, int leaf_size, double eta = 2.0)
      : coords_(detail::flat(points)), leaf_size_(leaf_size), eta_(eta) {
    hmgp_geom* g = nullptr;
    detail::check(hmgp_geometry_build(detail::context(), coords_.data(),
                                      static_cast<int>(points.size()), 2, leaf_size, eta, &g));
    geom_.reset(g, hmgp_geometry_destroy);
    perm_.resize(points.size());
    inv_.resize(points.size());
    detail::check(hmgp_geometry_perm(g, perm_.data(), inv_.data()));
    // cluster nodes in the reference's pre-order (begin, end, left, right, box)
    const int cap = 2 * static_cast<int>(points.size()) + 1;
    std::vector<int32_t> n4(4 * static_cast<size_t>(cap));
    std::vector<double> b6(6 * static_cast<size_t>(cap));
    int cnt = 0;
    detail::check(hmgp_geometry_clusters(g, n4.data(), b6.data(), cap, &cnt));
    root_ = make(n4, b6, 0);
  }
  const Cluster& root() const { return *root_; }
  int size() const { return static_cast<int>(perm_.size()); }
  int leaf_size() const { return leaf_size_; }
  const std::vector<int>& perm() const { return perm_; }
  const std::vector<int>& inverse_perm() const { return inv_; }
  std::vector<const Cluster*> leaves() const {  // geometry.cpp:80-94 (left to right)
    std::vector<const Cluster*> out;
    std::vector<const Cluster*> stack{root_.get()};
    while (!stack.empty()) {
      const Cluster* c = stack.back();
      stack.pop_back();
      if (c->is_leaf()) {
        out.push_back(c);
      } else {
        stack.push_back(c->right.get());
        stack.push_back(c->left.get());
      }
    }
    return out;
  }
  hmgp_geom* handle() const { return geom_.get(); }
  double eta() const { return eta_; }
  const std::vector<double>& coords() const { return coords_; }

 private:
  static std::unique_ptr<Cluster> make(const std::vector<int32_t>& n4, const std::vector<double>& b6, int id) {
    auto c = std::make_unique<Cluster>();
    c->begin = n4[4 * id];
    c->end = n4[4 * id + 1];
    c->box.lo[0] = b6[6 * id];
    c->box.lo[1] = b6[6 * id + 1];
    c->box.hi[0] = b6[6 * id + 3];
    c->box.hi[1] = b6[6 * id + 4];
    if (n4[4 * id + 2] >= 0) {
      c->left = make(n4, b6, n4[4 * id + 2]);
      c->right = make(n4, b6, n4[4 * id + 3]);
    }
    return c;
  }
  std::vector<double> coords_;
  int leaf_size_;
  double eta_;
  std::shared_ptr<hmgp_geom> geom_;
  std::vector<int> perm_, inv_;
  std::unique_ptr<Cluster> root_;
};

inline ClusterTree build_cluster_tree(std::span<const Location> locations, int leaf_size = 32) {
  return ClusterTree(locations, leaf_size);
}

// BlockClusterTree (geometry.hpp:72-106).  The partition is built on the GPU
// (square: with the cluster tree; rectangular rows != cols: hmgp_block_tree_rect);
// the Node tree is rebuilt on the host from the DFS leaf list and the two
// cluster trees with the reference's split rule (geometry.cpp:119-154).
class BlockClusterTree {
 public:
  struct Node {
    enum class Tag { Admissible, Dense, Split };
    const Cluster* row = nullptr;
    const Cluster* col = nullptr;
    Tag tag = Tag::Dense;
    std::vector<std::unique_ptr<Node>> children;  // row-major over child pairs
    bool is_leaf() const { return tag != Tag::Split; }
  };
  struct Leaf {  // flat DFS leaf record (tree positions)
    int row_begin, row_end, col_begin, col_end;
    bool admissible;
  };
  BlockClusterTree(const ClusterTree& rows, const ClusterTree& cols, double eta)
      : rows_(&rows), cols_(&cols), eta_(eta) {
    if (!(eta > 0.0)) throw std::invalid_argument("eta must be positive");
    std::vector<hmgp_block> b;
    int64_t cnt = 0;
    if (&rows == &cols) {
      hmgp_geom* g = rows.handle();
      if (eta != rows.eta()) {  // same tree, different admissibility: rebuild on device
        hmgp_geom* g2 = nullptr;
        detail::check(hmgp_geometry_build(detail::context(), rows.coords().data(), rows.size(), 2,
                                          rows.leaf_size(), eta, &g2));
        own_.reset(g2, hmgp_geometry_destroy);
        g = g2;
      }
      geom_ = g;
      detail::check(hmgp_geometry_block_count(g, &cnt, &adm_, &dense_));
      b.resize(static_cast<size_t>(cnt));
      detail::check(hmgp_geometry_blocks(g, b.data(), cnt));
    } else {
      detail::check(hmgp_block_tree_rect(detail::context(), rows.handle(), cols.handle(), eta, nullptr, 0,
                                         &cnt, &adm_, &dense_));
      b.resize(static_cast<size_t>(cnt));
      detail::check(hmgp_block_tree_rect(detail::context(), rows.handle(), cols.handle(), eta, b.data(),
                                         cnt, &cnt, &adm_, &dense_));
    }
    for (const auto& x : b) blocks_.push_back(Leaf{x.row_begin, x.row_end, x.col_begin, x.col_end, x.tag == 0});
    size_t next = 0;
    root_ = rebuild(rows.root(), cols.root(), next);
    if (next != blocks_.size()) throw std::runtime_error("BlockClusterTree: inconsistent leaf list");
  }
  const Node& root() const { return *root_; }
  const ClusterTree& rows() const { return *rows_; }
  const ClusterTree& cols() const { return *cols_; }
  double eta() const { return eta_; }
  bool square_symmetric() const { return rows_ == cols_; }
  const std::vector<const Node*>& leaves() const { return leaves_; }
  int admissible_count() const { return adm_; }
  int dense_count() const { return dense_; }
  const std::vector<Leaf>& blocks() const { return blocks_; }
  hmgp_geom* handle() const {
    if (!geom_) throw std::invalid_argument("GPU H-matrix: rectangular block trees are not supported");
    return geom_;
  }

 private:
  std::unique_ptr<Node> rebuild(const Cluster& r, const Cluster& c, size_t& next) {
    auto nd = std::make_unique<Node>();
    nd->row = &r;
    nd->col = &c;
    if (next < blocks_.size()) {
      const Leaf& l = blocks_[next];
      if (l.row_begin == r.begin && l.row_end == r.end && l.col_begin == c.begin && l.col_end == c.end) {
        nd->tag = l.admissible ? Node::Tag::Admissible : Node::Tag::Dense;
        ++next;
        leaves_.push_back(nd.get());
        return nd;
      }
    }
    if (r.is_leaf() && c.is_leaf()) throw std::runtime_error("BlockClusterTree: leaf list does not cover the tree");
    nd->tag = Node::Tag::Split;
    const Cluster* rp[2] = {&r, nullptr};
    const Cluster* cp[2] = {&c, nullptr};
    int nr = 1, nc = 1;
    if (!r.is_leaf()) {
      rp[0] = r.left.get();
      rp[1] = r.right.get();
      nr = 2;
    }
    if (!c.is_leaf()) {
      cp[0] = c.left.get();
      cp[1] = c.right.get();
      nc = 2;
    }
    for (int i = 0; i < nr; ++i)
      for (int j = 0; j < nc; ++j) nd->children.push_back(rebuild(*rp[i], *cp[j], next));
    return nd;
  }
  const ClusterTree* rows_;
  const ClusterTree* cols_;
  double eta_;
  hmgp_geom* geom_ = nullptr;
  std::shared_ptr<hmgp_geom> own_;
  std::vector<Leaf> blocks_;
  std::unique_ptr<Node> root_;
  std::vector<const Node*> leaves_;
  int adm_ = 0, dense_ = 0;
};

inline BlockClusterTree build_block_tree(const ClusterTree& rows, const ClusterTree& cols,
                                         double eta = 2.0) {
  return BlockClusterTree(rows, cols, eta);
}

// ------------------------------------------------------------- H-matrix ----
enum class BlockKind { Branch, Dense, LowRank };

// Host view of the payload tree (hblock.hpp:17-45), materialised on first
// HMatrix::root() call from the device payload: lower triangle only (null
// upper-mirror slots), Dense = dense, LowRank = U V^T.
struct HBlock {
  BlockKind kind = BlockKind::Branch;
  const Cluster* row = nullptr;
  const Cluster* col = nullptr;
  Matrix dense;
  Matrix U, V;
  int compact_cols = 0;
  std::vector<std::unique_ptr<HBlock>> children;
  int nrows() const { return row->size(); }
  int ncols() const { return col->size(); }
  int rank() const { return U.cols(); }
  int child_rows() const { return row->is_leaf() ? 1 : 2; }
  int child_cols() const { return col->is_leaf() ? 1 : 2; }
  const HBlock* child(int i, int j) const { return children[i * child_cols() + j].get(); }
  const Cluster* row_part(int i) const { return row->is_leaf() ? row : (i == 0 ? row->left.get() : row->right.get()); }
  const Cluster* col_part(int j) const { return col->is_leaf() ? col : (j == 0 ? col->left.get() : col->right.get()); }
  std::size_t payload_bytes() const {
    if (kind == BlockKind::Dense) return sizeof(double) * dense.data.size();
    if (kind == BlockKind::LowRank) return sizeof(double) * (U.data.size() + V.data.size());
    return 0;
  }
};

class HMatrix;
HMatrix from_dense(const Matrix& m);

class HMatrix {  // hmatrix.hpp:44-83
 public:
  struct Storage {
    std::size_t bytes = 0;
    double ratio = 0.0;
  };
  HMatrix(const BlockClusterTree& bt, const MaternParams& p, const RankControl& rc)
      : n_(bt.rows().size()), bt_(&bt), rows_(&bt.rows()), rc_(rc) {
    const hmgp_matern m = p.c();
    const hmgp_rank_control r = rc.c();
    hmgp_hmat* h = nullptr;
    detail::check(hmgp_assemble(detail::context(), bt.handle(), &m, &r, &h));
    h_.reset(h, hmgp_hmat_destroy);
  }
  // one GPU's share of a sharded assembly: stored leaves
  // [leaf_range().first, leaf_range().second) only; leaf queries only
  HMatrix(const BlockClusterTree& bt, const MaternParams& p, const RankControl& rc, int shard, int n_shards)
      : n_(bt.rows().size()), bt_(&bt), rows_(&bt.rows()), rc_(rc) {
    const hmgp_matern m = p.c();
    const hmgp_rank_control r = rc.c();
    hmgp_hmat* h = nullptr;
    int b = 0, e = 0;
    detail::check(hmgp_assemble_shard(detail::context(), bt.handle(), &m, &r, shard, n_shards, &h, &b, &e));
    h_.reset(h, hmgp_hmat_destroy);
    range_ = {b, e};
    partial_ = true;
  }
  // stored leaves [first, second): the whole list for a full H-matrix
  std::pair<int, int> leaf_range() const {
    if (partial_) return range_;
    return {0, leaf_count()};
  }
  bool is_shard() const { return partial_; }
  int rows() const { return n_; }
  int cols() const { return n_; }
  bool symmetric() const {
    int s = 1;
    detail::check(hmgp_hmat_symmetric(h_.get(), &s));
    return s != 0;
  }
  const ClusterTree& row_tree() const { return *rows_; }
  const ClusterTree& col_tree() const { return *rows_; }
  const RankControl& rank_control() const { return rc_; }
  const HBlock& root() const {  // materialised on first use
    if (!root_) build_root();
    return *root_;
  }
  Vector matvec(const Vector& x) const {
    if (static_cast<int>(x.size()) != n_) throw std::invalid_argument("matvec: dimension mismatch");
    Vector y(n_);
    detail::check(hmgp_hmat_matvec(detail::context(), h_.get(), x.data(), y.data()));
    return y;
  }
  Storage storage() const {
    whole("storage");
    double b = 0, md = 0;
    int r = 0;
    detail::check(hmgp_hmat_stats(h_.get(), &b, &r, &md));
    return Storage{static_cast<std::size_t>(b), b / (8.0 * n_ * n_)};
  }
  double max_diagonal() const {
    whole("max_diagonal");
    double b = 0, md = 0;
    int r = 0;
    detail::check(hmgp_hmat_stats(h_.get(), &b, &r, &md));
    return md;
  }
  int max_leaf_rank() const {
    whole("max_leaf_rank");
    double b = 0, md = 0;
    int r = 0;
    detail::check(hmgp_hmat_stats(h_.get(), &b, &r, &md));
    return r;
  }
  // hmatrix.cpp:274-297 (original index order; refused beyond n = 4096)
  Matrix to_dense() const {
    if (n_ > 4096) throw std::invalid_argument("to_dense: refused beyond n = 4096");
    Matrix out(n_, n_);
    detail::check(hmgp_hmat_to_dense(detail::context(), h_.get(), out.data.data()));
    return out;
  }
  // stored leaves in DFS order (row_begin, row_end, col_begin, col_end, kind 1/2, rank;
  // rank -2 outside a shard's range) and one leaf's payload (dense, or U and V)
  struct LeafInfo {
    int row_begin, row_end, col_begin, col_end, kind, rank;
  };
  std::vector<LeafInfo> leaves() const {
    std::vector<LeafInfo> out(static_cast<size_t>(leaf_count()));
    int64_t cnt = 0;
    if (!out.empty())
      detail::check(hmgp_hmat_leaves(h_.get(), reinterpret_cast<int32_t*>(out.data()),
                                     static_cast<int64_t>(out.size()), &cnt));
    return out;
  }
  int leaf_count() const {
    int64_t cnt = 0;
    detail::check(hmgp_hmat_leaves(h_.get(), nullptr, 0, &cnt));
    return static_cast<int>(cnt);
  }
  void leaf_data(int k, Matrix* a, Matrix* b) const {
    const auto lv = leaves();
    if (k < 0 || k >= static_cast<int>(lv.size())) throw std::out_of_range("leaf_data: index");
    const LeafInfo& l = lv[k];
    if (l.rank == -2) throw std::invalid_argument("leaf_data: leaf outside this shard");
    const int m = l.row_end - l.row_begin, n = l.col_end - l.col_begin;
    if (l.kind == 1) {
      *a = Matrix(m, n);
      detail::check(hmgp_hmat_leaf_data(h_.get(), k, a->data.data(), nullptr));
    } else {
      *a = Matrix(m, l.rank);
      *b = Matrix(n, l.rank);
      std::vector<double> ua(std::max<size_t>(1, a->data.size())), vb(std::max<size_t>(1, b->data.size()));
      detail::check(hmgp_hmat_leaf_data(h_.get(), k, ua.data(), vb.data()));
      std::copy(ua.begin(), ua.begin() + a->data.size(), a->data.begin());
      std::copy(vb.begin(), vb.begin() + b->data.size(), b->data.begin());
    }
  }
  hmgp_hmat* handle() const { return h_.get(); }

 private:
  friend HMatrix from_dense(const Matrix& m);
  HMatrix() = default;
  void whole(const char* what) const {
    if (partial_) throw std::invalid_argument(std::string(what) + ": H-matrix is a leaf-range shard");
  }
  void build_root() const {
    whole("root");
    const auto lv = leaves();
    size_t k = 0;
    if (!bt_) {  // from_dense: one dense leaf over the owned tree's root
      auto r = std::make_unique<HBlock>();
      r->kind = BlockKind::Dense;
      r->row = r->col = &rows_->root();
      leaf_data(0, &r->dense, nullptr);
      root_ = std::move(r);
      return;
    }
    root_ = payload(bt_->root(), lv, k);
  }
  // build_payload_tree (hmatrix.cpp:108-139): the upper mirror of diagonal nodes is null
  std::unique_ptr<HBlock> payload(const BlockClusterTree::Node& nd, const std::vector<LeafInfo>& lv,
                                  size_t& k) const {
    auto b = std::make_unique<HBlock>();
    b->row = nd.row;
    b->col = nd.col;
    if (nd.is_leaf()) {
      const int idx = static_cast<int>(k++);
      if (lv[idx].kind == 1) {
        b->kind = BlockKind::Dense;
        leaf_data(idx, &b->dense, nullptr);
      } else {
        b->kind = BlockKind::LowRank;
        leaf_data(idx, &b->U, &b->V);
        b->compact_cols = lv[idx].rank;  // fill_leaf (hmatrix.cpp:162)
      }
      return b;
    }
    b->kind = BlockKind::Branch;
    const int nr = b->child_rows(), nc = b->child_cols();
    b->children.resize(static_cast<size_t>(nr) * nc);
    for (int i = 0; i < nr; ++i)
      for (int j = 0; j < nc; ++j) {
        if (nd.row == nd.col && j > i) continue;
        b->children[i * nc + j] = payload(*nd.children[i * nc + j], lv, k);
      }
    return b;
  }
  int n_ = 0;
  const BlockClusterTree* bt_ = nullptr;
  const ClusterTree* rows_ = nullptr;
  std::shared_ptr<const ClusterTree> owned_tree_;
  RankControl rc_;
  std::pair<int, int> range_{0, 0};
  bool partial_ = false;
  std::shared_ptr<hmgp_hmat> h_;
  mutable std::unique_ptr<HBlock> root_;
};

// from_dense (hmatrix.cpp:223-242): one Dense leaf over a self-owned one-cluster tree
inline HMatrix from_dense(const Matrix& m) {
  if (m.rows() != m.cols() || m.rows() < 1)
    throw std::invalid_argument("from_dense: need a nonempty square matrix");
  const int n = m.rows();
  std::vector<Location> line(n);
  for (int i = 0; i < n; ++i) line[i] = {static_cast<double>(i) / n, 0.0};
  HMatrix h;
  h.n_ = n;
  h.owned_tree_ = std::make_shared<ClusterTree>(line, n);
  h.rows_ = h.owned_tree_.get();
  hmgp_hmat* p = nullptr;
  detail::check(hmgp_hmat_from_dense(detail::context(), m.data.data(), n, &p));
  h.h_.reset(p, hmgp_hmat_destroy);
  return h;
}

inline HMatrix assemble_shard(const BlockClusterTree& block_tree, const MaternParams& params,
                              const RankControl& rc, int shard, int n_shards) {
  params.validate();
  return HMatrix(block_tree, params, rc, shard, n_shards);
}

// assemble (hmatrix.hpp:88-89, hmatrix.cpp:174-221).  `locations` must be the
// points the block tree's cluster tree was built from (checked); `threads` is
// accepted for API parity (the GPU path is one batched pass).
inline HMatrix assemble(const BlockClusterTree& block_tree, std::span<const Location> locations,
                        const MaternParams& params, const RankControl& rc, int threads = 1) {
  (void)threads;
  if (rc.mode == RankControl::Mode::FixedAccuracy && !(rc.eps > 0.0))
    throw std::invalid_argument("assemble: eps must be positive");
  if (rc.mode == RankControl::Mode::FixedRank && rc.rank < 1)
    throw std::invalid_argument("assemble: fixed rank must be >= 1");
  if (!block_tree.square_symmetric())
    throw std::invalid_argument("GPU assemble: rectangular block trees are not supported");
  if (static_cast<int>(locations.size()) != block_tree.rows().size() ||
      detail::flat(locations) != block_tree.rows().coords())
    throw std::invalid_argument("assemble: locations differ from the block tree's points");
  params.validate();
  return HMatrix(block_tree, params, rc);
}

// AssembledCov / assemble_covariance (pipeline.hpp:29-36, loglik.cpp:9-16)
struct AssembledCov {
  std::unique_ptr<ClusterTree> tree;
  std::unique_ptr<BlockClusterTree> blocks;
  HMatrix matrix;
};

inline AssembledCov assemble_covariance(std::span<const Location> locations, const MaternParams& params,
                                        const HConfig& cfg);

struct FactorInfo {  // hfactor.hpp:24-29
  double eps = 0.0;
  int clamped = 0, negative = 0;
  double min_pivot = 0.0;
};

class HFactor {  // hfactor.hpp:34-68
 public:
  HFactor(const HMatrix& h, double eps_f, FactorForm form) : n_(h.rows()), form_(form) {
    hmgp_factor* f = nullptr;
    hmgp_factor_info info{};
    detail::check(hmgp_factorize(detail::context(), h.handle(), eps_f,
                                 form == FactorForm::Ldl ? 1 : 0, &f, &info));
    f_.reset(f, hmgp_factor_destroy);
    info_ = FactorInfo{info.eps, info.clamped, info.negative, info.min_pivot};
    bytes_ = static_cast<std::size_t>(info.storage_bytes);
  }
  FactorForm form() const { return form_; }
  const FactorInfo& info() const { return info_; }
  int size() const { return n_; }
  Vector solve_lower(const Vector& b) const { return run(b, hmgp_solve_lower, "solve_lower"); }
  Vector solve_factored(const Vector& b) const {
    return run(b, hmgp_solve_factored, "solve_factored");
  }
  double quad_form(const Vector& b) const {
    if (static_cast<int>(b.size()) != n_) throw std::invalid_argument("quad_form: dimension mismatch");
    double q = 0;
    detail::check(hmgp_quad_form(detail::context(), f_.get(), b.data(), &q));
    return q;
  }
  double log_det() const {
    double v = 0;
    detail::check(hmgp_log_det(detail::context(), f_.get(), &v));
    return v;
  }
  Vector diagonal() const {
    Vector d(n_);
    detail::check(hmgp_factor_diagonal(detail::context(), f_.get(), d.data()));
    return d;
  }
  std::size_t storage_bytes() const { return bytes_; }
  // hfactor.cpp:421-434 (tree order) and 436-449 (L D L^T or L L^T, original order)
  Matrix lower_dense() const {
    if (n_ > 4096) throw std::invalid_argument("lower_dense: refused beyond n = 4096");
    Matrix out(n_, n_);
    detail::check(hmgp_factor_lower_dense(detail::context(), f_.get(), out.data.data()));
    return out;
  }
  Matrix reconstruct() const {
    if (n_ > 4096) throw std::invalid_argument("lower_dense: refused beyond n = 4096");
    Matrix out(n_, n_);
    detail::check(hmgp_factor_reconstruct(detail::context(), f_.get(), out.data.data()));
    return out;
  }

 private:
  using SolveFn = int (*)(hmgp_ctx*, const hmgp_factor*, const double*, double*);
  Vector run(const Vector& b, SolveFn fn, const char* what) const {
    if (static_cast<int>(b.size()) != n_)
      throw std::invalid_argument(std::string(what) + ": dimension mismatch");
    Vector x(n_);
    detail::check(fn(detail::context(), f_.get(), b.data(), x.data()));
    return x;
  }
  int n_;
  FactorForm form_;
  FactorInfo info_;
  std::size_t bytes_ = 0;
  std::shared_ptr<hmgp_factor> f_;
};

inline HFactor factorize(const HMatrix& h, double eps_f, FactorForm form) {
  if (!(eps_f > 0.0)) throw std::invalid_argument("factorize: eps_f must be positive");
  return HFactor(h, eps_f, form);
}
inline HFactor h_cholesky(const HMatrix& h, double eps_f) {
  return factorize(h, eps_f, FactorForm::Cholesky);
}
inline HFactor h_ldl(const HMatrix& h, double eps_f) { return factorize(h, eps_f, FactorForm::Ldl); }

// ------------------------------------------------------------- pipeline ----
inline AssembledCov assemble_covariance(std::span<const Location> locations, const MaternParams& params,
                                        const HConfig& cfg) {
  params.validate();
  auto tree = std::make_unique<ClusterTree>(locations, cfg.leaf_size, cfg.eta);
  auto blocks = std::make_unique<BlockClusterTree>(*tree, *tree, cfg.eta);
  HMatrix m = assemble(*blocks, locations, params, cfg.rank, cfg.threads);
  return AssembledCov{std::move(tree), std::move(blocks), std::move(m)};
}

struct LogLikResult {  // loglik.hpp:10-17
  double loglik = 0.0, logdet = 0.0, quad_form = 0.0;
  int n = 0;
  double seconds = 0.0;
  enum class Status { Success, Clamped } factor_status = Status::Success;
};

inline LogLikResult evaluate_loglik(std::span<const Location> locations, const Vector& z,
                                    const MaternParams& params, const HConfig& cfg = {}) {
  params.validate();
  const int n = static_cast<int>(locations.size());
  if (n < 1) throw std::invalid_argument("evaluate_loglik: empty dataset");
  if (static_cast<int>(z.size()) != n) throw std::invalid_argument("evaluate_loglik: |z| != n");
  const auto xy = detail::flat(locations);
  const hmgp_matern m = params.c();
  const hmgp_config c = cfg.c();
  hmgp_loglik_result r{};
  detail::check(hmgp_loglik(detail::context(), xy.data(), n, 2, z.data(), &m, &c, &r));
  LogLikResult out;
  out.loglik = r.loglik;
  out.logdet = r.logdet;
  out.quad_form = r.quad_form;
  out.n = r.n;
  out.seconds = r.seconds;
  out.factor_status = r.status == 1 ? LogLikResult::Status::Clamped : LogLikResult::Status::Success;
  return out;
}

struct PredictionResult {  // krige.hpp:10-13
  Vector z2_hat;
  double seconds = 0.0;
};

inline PredictionResult predict(std::span<const Location> train, const Vector& z1,
                                std::span<const Location> new_locations,
                                const MaternParams& params, const HConfig& cfg = {}) {
  params.validate();
  if (train.empty()) throw std::invalid_argument("predict: empty training set");
  if (z1.size() != train.size()) throw std::invalid_argument("predict: |z1| != n");
  const auto tr = detail::flat(train);
  const auto te = detail::flat(new_locations);
  const hmgp_matern m = params.c();
  const hmgp_config c = cfg.c();
  PredictionResult res;
  res.z2_hat.resize(new_locations.size());
  detail::check(hmgp_predict(detail::context(), tr.data(), static_cast<int>(train.size()), 2,
                             z1.data(), te.data(), static_cast<int>(new_locations.size()), &m, &c,
                             res.z2_hat.data(), &res.seconds));
  return res;
}

// krige.hpp kriging_variance_dense (krige.cpp:46-74) on the GPU, dense, n <= 4096
inline Vector kriging_variance_dense(std::span<const Location> train,
                                     std::span<const Location> new_locations,
                                     const MaternParams& params) {
  params.validate();
  const auto tr = detail::flat(train);
  const auto te = detail::flat(new_locations);
  const hmgp_matern m = params.c();
  Vector out(new_locations.size());
  detail::check(hmgp_kriging_variance_dense(detail::context(), tr.data(), static_cast<int>(train.size()), 2,
                                            te.data(), static_cast<int>(new_locations.size()), &m,
                                            out.data()));
  return out;
}

// metrics.hpp (metrics.cpp:11-69): rmse on the host, mloe_mmom dense on the GPU
inline double rmse(const Vector& z_hat, const Vector& z_true) {
  if (z_hat.size() != z_true.size()) throw std::invalid_argument("rmse: length mismatch");
  if (z_hat.size() == 0) throw std::invalid_argument("rmse: empty input");
  double s = 0.0;
  for (size_t i = 0; i < z_hat.size(); ++i) s += (z_hat[i] - z_true[i]) * (z_hat[i] - z_true[i]);
  return std::sqrt(s / static_cast<double>(z_hat.size()));
}

struct MetricConfig {
  int M = 1000;  // evaluation locations, clamped to n
  std::uint64_t seed = 0;
  int dense_guard = 4096;
};

struct MloeMmom {
  double mloe = 0.0;
  double mmom = 0.0;
};

inline MloeMmom mloe_mmom(std::span<const Location> locations, const MaternParams& theta_true,
                          const MaternParams& theta_approx, const MetricConfig& cfg = {}) {
  theta_true.validate();
  theta_approx.validate();
  const auto xy = detail::flat(locations);
  const hmgp_matern mt = theta_true.c(), ma = theta_approx.c();
  MloeMmom r;
  detail::check(hmgp_mloe_mmom(detail::context(), xy.data(), static_cast<int>(locations.size()), 2, &mt, &ma,
                               cfg.M, cfg.seed, cfg.dense_guard, &r.mloe, &r.mmom));
  return r;
}

// simgen.hpp data utilities over the C ABI
inline std::vector<Location> random_locations(int n, std::uint64_t seed) {  // simgen.cpp:114-123
  if (n < 1) throw std::invalid_argument("random_locations: n must be >= 1");
  std::vector<double> xy(2 * static_cast<size_t>(n));
  detail::check(hmgp_random_locations(n, 2, seed, xy.data()));
  std::vector<Location> out(n);
  for (int i = 0; i < n; ++i) out[i] = Location{xy[2 * i], xy[2 * i + 1]};
  return out;
}

// simgen.cpp:125-141 on the GPU (dense FP64 Cholesky; n <= 65536 instead of
// the reference's 16384).  std::runtime_error if the covariance is not SPD.
inline Vector sample_grf(std::span<const Location> locations, const MaternParams& params,
                         std::uint64_t seed) {
  params.validate();
  if (locations.empty()) throw std::invalid_argument("sample_grf: empty dataset");
  const auto xy = detail::flat(locations);
  const hmgp_matern m = params.c();
  Vector z(locations.size());
  detail::check(hmgp_sample_grf(detail::context(), xy.data(), static_cast<int>(locations.size()), 2, &m,
                                seed, z.data()));
  return z;
}

}  // namespace hmgp
