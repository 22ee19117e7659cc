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

// ------------------------------------------------------------- geometry ----
class ClusterTree {  // geometry.hpp:44-66 (GPU-built; perm bit-exact)
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
  }
  int size() const { return static_cast<int>(perm_.size()); }
  int leaf_size() const { return leaf_size_; }
  const std::vector<int32_t>& perm() const { return perm_; }
  const std::vector<int32_t>& inverse_perm() const { return inv_; }
  hmgp_geom* handle() const { return geom_.get(); }
  double eta() const { return eta_; }
  const std::vector<double>& coords() const { return coords_; }

 private:
  std::vector<double> coords_;
  int leaf_size_;
  double eta_;
  std::shared_ptr<hmgp_geom> geom_;
  std::vector<int32_t> perm_, inv_;
};

inline ClusterTree build_cluster_tree(std::span<const Location> locations, int leaf_size = 32) {
  return ClusterTree(locations, leaf_size);
}

class BlockClusterTree {  // geometry.hpp:72-106 (square symmetric trees)
 public:
  struct Leaf {
    int row_begin, row_end, col_begin, col_end;
    bool admissible;
  };
  BlockClusterTree(const ClusterTree& rows, const ClusterTree& cols, double eta)
      : tree_(&rows), eta_(eta) {
    if (&rows != &cols)
      throw std::invalid_argument("GPU block tree: rows and cols must be the same tree");
    if (!(eta > 0.0)) throw std::invalid_argument("eta must be positive");
    hmgp_geom* g = rows.handle();
    if (eta != rows.eta()) {  // same tree, different admissibility: rebuild on device
      hmgp_geom* g2 = nullptr;
      detail::check(hmgp_geometry_build(detail::context(), rows.coords().data(), rows.size(), 2,
                                        rows.leaf_size(), eta, &g2));
      own_.reset(g2, hmgp_geometry_destroy);
      g = g2;
    }
    geom_ = g;
    int64_t cnt = 0;
    detail::check(hmgp_geometry_block_count(g, &cnt, &adm_, &dense_));
    std::vector<hmgp_block> b(static_cast<size_t>(cnt));
    detail::check(hmgp_geometry_blocks(g, b.data(), cnt));
    for (const auto& x : b)
      leaves_.push_back(Leaf{x.row_begin, x.row_end, x.col_begin, x.col_end, x.tag == 0});
  }
  const std::vector<Leaf>& leaves() const { return leaves_; }
  int admissible_count() const { return adm_; }
  int dense_count() const { return dense_; }
  bool square_symmetric() const { return true; }
  double eta() const { return eta_; }
  const ClusterTree& rows() const { return *tree_; }
  hmgp_geom* handle() const { return geom_; }

 private:
  const ClusterTree* tree_;
  double eta_;
  hmgp_geom* geom_ = nullptr;
  std::shared_ptr<hmgp_geom> own_;
  std::vector<Leaf> leaves_;
  int adm_ = 0, dense_ = 0;
};

inline BlockClusterTree build_block_tree(const ClusterTree& rows, const ClusterTree& cols,
                                         double eta = 2.0) {
  return BlockClusterTree(rows, cols, eta);
}

// ------------------------------------------------------------- H-matrix ----
class HMatrix {  // hmatrix.hpp:44-83
 public:
  struct Storage {
    std::size_t bytes = 0;
    double ratio = 0.0;
  };
  HMatrix(const BlockClusterTree& bt, const MaternParams& p, const RankControl& rc) : n_(bt.rows().size()) {
    const hmgp_matern m = p.c();
    const hmgp_rank_control r = rc.c();
    hmgp_hmat* h = nullptr;
    detail::check(hmgp_assemble(detail::context(), bt.handle(), &m, &r, &h));
    h_.reset(h, hmgp_hmat_destroy);
  }
  // one GPU's share of a sharded assembly: stored leaves
  // [leaf_range().first, leaf_range().second) only; leaf queries only
  HMatrix(const BlockClusterTree& bt, const MaternParams& p, const RankControl& rc, int shard, int n_shards)
      : n_(bt.rows().size()) {
    const hmgp_matern m = p.c();
    const hmgp_rank_control r = rc.c();
    hmgp_hmat* h = nullptr;
    detail::check(hmgp_assemble_shard(detail::context(), bt.handle(), &m, &r, shard, n_shards, &h,
                                      &range_.first, &range_.second));
    h_.reset(h, hmgp_hmat_destroy);
  }
  std::pair<int, int> leaf_range() const { return range_; }  // (0, -1): the whole matrix
  int rows() const { return n_; }
  int cols() const { return n_; }
  bool symmetric() const { return true; }
  Vector matvec(const Vector& x) const {
    if (static_cast<int>(x.size()) != n_) throw std::invalid_argument("matvec: dimension mismatch");
    Vector y(n_);
    detail::check(hmgp_hmat_matvec(detail::context(), h_.get(), x.data(), y.data()));
    return y;
  }
  Storage storage() const {
    double b = 0, md = 0;
    int r = 0;
    detail::check(hmgp_hmat_stats(h_.get(), &b, &r, &md));
    return Storage{static_cast<std::size_t>(b), b / (8.0 * n_ * n_)};
  }
  double max_diagonal() const {
    double b = 0, md = 0;
    int r = 0;
    detail::check(hmgp_hmat_stats(h_.get(), &b, &r, &md));
    return md;
  }
  int max_leaf_rank() const {
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
  hmgp_hmat* handle() const { return h_.get(); }

 private:
  int n_;
  std::pair<int, int> range_{0, -1};
  std::shared_ptr<hmgp_hmat> h_;
};

inline HMatrix assemble_shard(const BlockClusterTree& block_tree, const MaternParams& params,
                              const RankControl& rc, int shard, int n_shards) {
  params.validate();
  return HMatrix(block_tree, params, rc, shard, n_shards);
}

inline HMatrix assemble(const BlockClusterTree& block_tree, std::span<const Location>,
                        const MaternParams& params, const RankControl& rc, int threads = 1) {
  (void)threads;
  params.validate();
  return HMatrix(block_tree, params, rc);
}

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
