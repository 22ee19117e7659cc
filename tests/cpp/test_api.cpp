// Drop-in check of include/hmgp/hmgp.hpp: the reference's own hand cases and
// API contracts (tests/test_geometry.cpp, test_hfactor.cpp, test_loglik_mle.cpp,
// test_krige_metrics.cpp under /root/reference/proj) through the C++ mirror
// that a reference user would compile against.  Prints one line per check and
// exits non-zero on any failure.  Run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "hmgp/hmgp.hpp"

using namespace hmgp;

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool ok_ = false;            \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      ok_ = true;                \
    } catch (...) {              \
    }                            \
    CHECK(ok_);                  \
  } while (0)

// random_locations (simgen.cpp:114-123) comes from hmgp/hmgp.hpp


static double rel_err(double a, double b) { return std::abs(a - b) / std::abs(b); }

// covkernel.hpp through the drop-in (test_covkernel.cpp:29-187 ported)
static void covkernel_cases() {
  {
    MaternParams p{2.0, 0.3, 0.7, 0.25};
    CHECK(matern(0.0, p) == 2.25);
    MaternParams q{1.5, 0.1, 1.2, 0.0};
    CHECK(matern(0.0, q) == 1.5);
  }
  CHECK(rel_err(matern(1.0, {1.0, 1.0, 0.5, 0.0}), 0.36787944117144233) < 1e-13);
  CHECK(rel_err(detail::matern_generic(1.0, {1.0, 1.0, 0.5, 0.0}), 0.36787944117144233) < 1e-12);
  CHECK(rel_err(matern(1.0, {1.0, 1.0, 1.5, 0.0}), 0.73575888234288464) < 1e-13);
  CHECK(rel_err(detail::matern_generic(1.0, {1.0, 1.0, 1.5, 0.0}), 0.73575888234288464) < 1e-12);
  CHECK(rel_err(matern(0.7, {1.3, 0.2, 0.6, 0.0}), 0.050105793549337933) < 1e-12);
  CHECK(rel_err(matern(0.05, {2.0, 0.1, 2.5, 0.0}), 1.9206804224233392) < 1e-13);
  CHECK(rel_err(matern(0.3, {1.0, 0.1, 1.5, 0.0}), 0.19914827347145577) < 1e-13);
  CHECK(rel_err(bessel_k(0.5, 1.0), 0.46106850444789456) < 1e-14);
  for (double x : {0.02, 0.7, 1.9, 3.5, 20.0, 300.0}) {
    const double kh = std::sqrt(M_PI / (2.0 * x)) * std::exp(-x);
    CHECK(rel_err(bessel_k(0.5, x), kh) < 1e-14);
    CHECK(rel_err(bessel_k(1.5, x), kh * (1.0 + 1.0 / x)) < 1e-14);
    CHECK(rel_err(detail::bessel_k_generic(0.5, x), kh) < 1e-12);
    CHECK(rel_err(detail::bessel_k_generic(1.5, x), kh * (1.0 + 1.0 / x)) < 1e-12);
  }
  const double refs[][3] = {
      {1.0, 1.0, 0.60190723019723457},   {0.3, 0.5, 0.97647412438178792},
      {0.6, 1.0, 0.47971569489286612},   {1.0, 1e-6, 999999.99999278428},
      {2.7, 3.2, 0.072917852205606608},  {5.5, 10.0, 7.3304530079850216e-5},
      {10.0, 0.01, 1.8579404390480640e+28}, {25.0, 30.0, 3.7775319791336277e-10},
      {0.9, 650.0, 2.5140676518253439e-284}, {7.3, 2.0, 543.63827738445926},
      {12.6, 0.37, 1.4985106123100319e+17}, {3.0, 1e-8, 7.9999999999999999e+24},
      {0.01, 0.02, 4.0298381770492421},  {24.5, 1e-8, 1.4946625757169951e+226},
      {1.9, 700.0, 4.6818247046354968e-306}};
  for (const auto& r : refs) {
    CHECK(rel_err(bessel_k(r[0], r[1]), r[2]) < 1e-12);
    CHECK(rel_err(detail::bessel_k_generic(r[0], r[1]), r[2]) < 1e-12);
  }
  CHECK_THROWS_AS(bessel_k(0.5, 0.0), std::domain_error);
  CHECK_THROWS_AS(bessel_k(0.5, -1.0), std::domain_error);
  CHECK_THROWS_AS(bessel_k(-1.0, 1.0), std::domain_error);
  CHECK(bessel_k(0.5, 800.0) >= 0.0 && bessel_k(0.5, 800.0) < 1e-300);
  for (double nu : {0.37, 0.5, 1.1, 2.5, 4.8}) {  // positive, non-increasing
    MaternParams p{1.0, 0.2, nu, 0.0};
    double prev = matern(1e-9, p);
    for (int i = 1; i <= 50; ++i) {
      const double v = matern(10.0 * i / 50.0, p);
      CHECK(v > 0.0 && v <= prev * (1.0 + 1e-14) && v <= p.sigma2 + p.tau2);
      prev = v;
    }
  }
  {  // cov_block basics
    std::vector<Location> pts{{0.2, 0.2}, {0.2, 0.2}, {0.5, 0.2}};
    MaternParams p{2.0, 0.3, 0.5, 0.5};
    const std::vector<int> one{1}, r{0}, c{1}, bad{7};
    CHECK(cov_block(one, one, pts, p)(0, 0) == 2.5);
    CHECK(std::abs(cov_block(r, c, pts, p)(0, 0) - 2.0) <= 2e-14);
    CHECK_THROWS_AS(cov_block(bad, c, pts, p), std::out_of_range);
  }
  {  // Toeplitz exponential block
    std::vector<Location> pts{{0.0, 0.0}, {0.1, 0.0}, {0.2, 0.0}};
    std::vector<int> all{0, 1, 2};
    const Matrix b = cov_block(all, all, pts, {1.3, 0.1, 0.5, 0.0});
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) CHECK(rel_err(b(i, j), 1.3 * std::exp(-std::abs(i - j))) < 1e-13);
  }
  {  // cov_dense symmetric, nugget on the diagonal
    const auto pts = random_locations(40, 42);
    const Matrix c = cov_dense(pts, {1.0, 0.1, 1.5, 1e-8});
    for (int i = 0; i < 40; ++i) {
      CHECK(c(i, i) == 1.0 + 1e-8);
      for (int j = 0; j < 40; ++j) CHECK(c(i, j) == c(j, i));
    }
  }
  CHECK_THROWS_AS(matern(1.0, {0.0, 1.0, 0.5, 0.0}), std::invalid_argument);
  CHECK_THROWS_AS(matern(1.0, {1.0, -1.0, 0.5, 0.0}), std::invalid_argument);
  CHECK_THROWS_AS(matern(1.0, {1.0, 1.0, 0.0, 0.0}), std::invalid_argument);
  CHECK_THROWS_AS(matern(1.0, {1.0, 1.0, 0.5, -0.1}), std::invalid_argument);
  CHECK_THROWS_AS(matern(std::nan(""), {1.0, 1.0, 0.5, 0.0}), std::invalid_argument);
  {  // KernelEvaluator matches matern
    const auto pts = random_locations(50, 8);
    for (double nu : {0.5, 1.5, 2.5, 3.5, 0.82}) {
      MaternParams p{1.4, 0.07, nu, 0.3};
      KernelEvaluator k(pts, p);
      for (int i = 0; i < 50; i += 7)
        for (int j = 0; j < 50; j += 5) {
          const double want = i == j ? p.sigma2 + p.tau2 : matern(distance(pts[i], pts[j]), p);
          CHECK(rel_err(k(i, j), want) < 1e-13);
        }
      CHECK(k.at_distance(0.0) == p.sigma2);
    }
  }
}

// geometry.hpp / hmatrix.hpp / pipeline.hpp structure through the drop-in
static void structure_cases() {
  const auto pts = random_locations(1500, 3);
  ClusterTree t(pts, 32);
  {  // Cluster tree: root covers everything, children partition, leaves left to right
    CHECK(t.root().begin == 0 && t.root().end == 1500 && !t.root().is_leaf());
    const auto lv = t.leaves();
    int pos = 0;
    for (const Cluster* c : lv) {
      CHECK(c->is_leaf() && c->begin == pos && c->size() <= 32 && c->size() > 0);
      pos = c->end;
      for (int k = c->begin; k < c->end; ++k) {  // box containment (test_geometry.cpp:48-64)
        const Location& p = pts[t.perm()[k]];
        CHECK(p.x >= c->box.lo[0] && p.x <= c->box.hi[0] && p.y >= c->box.lo[1] && p.y <= c->box.hi[1]);
      }
    }
    CHECK(pos == 1500);
    Box a{{0, 0}, {1, 1}}, b{{2, 0}, {3, 1}};
    CHECK(a.diameter() == std::sqrt(2.0) && Box::distance(a, b) == 1.0 && Box::distance(a, a) == 0.0);
  }
  BlockClusterTree bt(t, t, 2.0);
  {  // Node tree: DFS leaves = flat list; admissibility rule; square_symmetric
    CHECK(bt.square_symmetric() && &bt.rows() == &t && &bt.cols() == &t);
    CHECK(bt.leaves().size() == bt.blocks().size());
    CHECK(static_cast<int>(bt.leaves().size()) == bt.admissible_count() + bt.dense_count());
    for (size_t k = 0; k < bt.leaves().size(); ++k) {
      const auto* l = bt.leaves()[k];
      CHECK(l->row->begin == bt.blocks()[k].row_begin && l->col->end == bt.blocks()[k].col_end);
      if (l->tag == BlockClusterTree::Node::Tag::Admissible) {
        const double d = Box::distance(l->row->box, l->col->box);
        CHECK(d > 0.0 && std::min(l->row->box.diameter(), l->col->box.diameter()) <= 2.0 * d);
      } else {
        CHECK(l->row->is_leaf() && l->col->is_leaf());
      }
    }
    CHECK(!bt.root().is_leaf() && bt.root().children.size() == 4);
  }
  {  // rectangular block tree (two different cluster trees): tiles rows x cols exactly
    const auto q = random_locations(700, 5);
    ClusterTree t2(q, 16);
    BlockClusterTree rb(t, t2, 2.0);
    CHECK(!rb.square_symmetric());
    long long area = 0;
    for (const auto* l : rb.leaves()) area += (long long)l->row->size() * l->col->size();
    CHECK(area == 1500LL * 700);
    CHECK(rb.admissible_count() > 0);
    CHECK_THROWS_AS(assemble(rb, pts, MaternParams{}, RankControl::fixed_accuracy(1e-6)), std::invalid_argument);
  }
  {  // assemble honours `locations`; HMatrix structure accessors; root() payload view
    const MaternParams p{1.0, 0.1, 0.5, 0.01};
    auto moved = pts;
    moved[3].x += 1e-3;
    CHECK_THROWS_AS(assemble(bt, moved, p, RankControl::fixed_accuracy(1e-6)), std::invalid_argument);
    const HMatrix h = assemble(bt, pts, p, RankControl::fixed_accuracy(1e-6));
    CHECK(&h.row_tree() == &t && &h.col_tree() == &t && h.rank_control().eps == 1e-6 && h.symmetric());
    CHECK(h.leaf_range().first == 0 && h.leaf_range().second == h.leaf_count());
    const HBlock& r = h.root();
    CHECK(r.kind == BlockKind::Branch && r.nrows() == 1500 && r.child(0, 1) == nullptr);
    // payload bytes of the view == storage(); U V^T of one low-rank leaf == matvec action
    std::size_t bytes = 0;
    std::vector<const HBlock*> st{&r};
    const HBlock* lr = nullptr;
    while (!st.empty()) {
      const HBlock* b = st.back();
      st.pop_back();
      bytes += b->payload_bytes();
      if (b->kind == BlockKind::LowRank && !lr) lr = b;
      for (const auto& c : b->children)
        if (c) st.push_back(c.get());
    }
    CHECK(bytes == h.storage().bytes);
    CHECK(lr && lr->U.rows() == lr->nrows() && lr->V.rows() == lr->ncols() && lr->compact_cols == lr->rank());
  }
  {  // AssembledCov / assemble_covariance (loglik.cpp:9-16)
    HConfig cfg;
    cfg.leaf_size = 32;
    const AssembledCov ac = assemble_covariance(pts, MaternParams{1.0, 0.1, 0.5, 0.01}, cfg);
    CHECK(ac.tree->size() == 1500 && ac.blocks->square_symmetric() && ac.matrix.rows() == 1500);
    CHECK(ac.tree->perm() == t.perm());
  }
  {  // from_dense (hmatrix.cpp:223-242): [[4,2],[2,5]] -> LDL L21 = 0.5, D = (4, 4)
    Matrix m(2, 2);
    m(0, 0) = 4;
    m(1, 0) = 2;
    m(0, 1) = 2;
    m(1, 1) = 5;
    const HMatrix h = from_dense(m);
    CHECK(h.symmetric() && h.rows() == 2 && h.root().kind == BlockKind::Dense);
    const HFactor f = h_ldl(h, 1e-10);
    const Vector d = f.diagonal();
    CHECK(d[0] == 4.0 && d[1] == 4.0);
    CHECK(f.lower_dense()(1, 0) == 0.5);
    Matrix one(1, 1);
    one(0, 0) = 4.0;
    CHECK(h_cholesky(from_dense(one), 1e-10).diagonal()[0] == 2.0);  // 1x1 Cholesky => 2
    Matrix ns(2, 2);
    ns(0, 0) = 1;
    ns(1, 0) = 0.5;
    ns(1, 1) = 1;
    CHECK(!from_dense(ns).symmetric());
    CHECK_THROWS_AS(factorize(from_dense(ns), 1e-6, FactorForm::Ldl), std::invalid_argument);
    CHECK_THROWS_AS(from_dense(Matrix(2, 3)), std::invalid_argument);
  }
}

int main() {
  covkernel_cases();
  structure_cases();
  {  // single point tree (test_geometry.cpp:20-27)
    std::vector<Location> pts{{0.3, 0.7}};
    ClusterTree t(pts, 32);
    CHECK(t.size() == 1 && t.perm()[0] == 0);
  }
  {  // 8x8 grid partitions exactly; perm round trip (test_geometry.cpp:29-46, 83-94)
    std::vector<Location> pts;
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) pts.push_back({i / 8.0, j / 8.0});
    ClusterTree t(pts, 16);
    std::vector<int> seen(64, 0);
    for (int k = 0; k < 64; ++k) seen[t.perm()[k]]++;
    for (int s : seen) CHECK(s == 1);
    for (int i = 0; i < 64; ++i) CHECK(t.perm()[t.inverse_perm()[i]] == i);
  }
  {  // block leaves tile n^2 exactly once, diagonal never admissible (test_geometry.cpp:132-143)
    const auto pts = random_locations(256, 11);
    ClusterTree t(pts, 16);
    BlockClusterTree bt(t, t, 2.0);
    std::vector<int> cnt(256 * 256, 0);
    for (const BlockClusterTree::Node* l : bt.leaves()) {
      for (int i = l->row->begin; i < l->row->end; ++i)
        for (int j = l->col->begin; j < l->col->end; ++j) cnt[i * 256 + j]++;
      if (l->row == l->col) CHECK(l->tag != BlockClusterTree::Node::Tag::Admissible);
    }
    for (int c : cnt) CHECK(c == 1);
    CHECK(bt.admissible_count() + bt.dense_count() == static_cast<int>(bt.leaves().size()));
  }
  {  // invalid inputs (test_geometry.cpp:96-101)
    std::vector<Location> none;
    CHECK_THROWS_AS(ClusterTree(none, 32), std::invalid_argument);
    std::vector<Location> bad{{0.1, std::nan("")}};
    CHECK_THROWS_AS(ClusterTree(bad, 32), std::invalid_argument);
  }
  {  // L(θ) hand cases (test_loglik_mle.cpp:13-33)
    std::vector<Location> one{{0.5, 0.5}};
    const auto r = evaluate_loglik(one, Vector{0.0}, MaternParams{0.75, 0.1, 0.5, 0.25});
    CHECK(std::abs(r.loglik - -0.9189385332046727) < 1e-14);
    CHECK(r.quad_form == 0.0);
    std::vector<Location> two{{0.0, 0.0}, {1.0, 1.0}};
    const auto r2 = evaluate_loglik(two, Vector{1.0, 1.0}, MaternParams{0.5, 1e-3, 0.5, 0.5});
    CHECK(std::abs(r2.loglik - (-std::log(2.0 * M_PI) - 1.0)) < 1e-10);
    CHECK_THROWS_AS(evaluate_loglik(one, Vector{0.0, 1.0}, MaternParams{}), std::invalid_argument);
  }
  {  // identical points -> FactorError with the nugget hint (test_loglik_mle.cpp:89-94)
    std::vector<Location> same(6, Location{0.25, 0.75});
    bool caught = false;
    try {
      evaluate_loglik(same, Vector(6, 1.0), MaternParams{1.0, 0.1, 0.5, 0.0});
    } catch (const FactorError& e) {
      caught = std::string(e.what()).find("nugget") != std::string::npos && e.pivot_index >= 0 &&
               e.pivot_index < 6;
    }
    CHECK(caught);
  }
  {  // assemble -> factorize -> solve inverts matvec (test_hfactor.cpp:126-134)
    const auto pts = random_locations(700, 8);
    ClusterTree t(pts, 32);
    BlockClusterTree bt(t, t, 2.0);
    const MaternParams p{1.0, 0.1, 1.5, 0.01};
    const HMatrix h = assemble(bt, pts, p, RankControl::fixed_accuracy(1e-6));
    CHECK(h.storage().ratio <= 1.0);
    const HFactor f = h_ldl(h, 1e-6);
    const Vector rhs = h.matvec(Vector(700, 1.0));
    const Vector x = f.solve_factored(rhs);
    double e2 = 0;
    for (double v : x) e2 += (v - 1) * (v - 1);
    CHECK(std::sqrt(e2 / 700) <= 1e-4);
    const HFactor fc = h_cholesky(h, 1e-6);
    CHECK(std::abs(fc.log_det() - f.log_det()) <= 1e-8 * std::abs(f.log_det()));
    CHECK_THROWS_AS(factorize(h, -1.0, FactorForm::Ldl), std::invalid_argument);
  }
  {  // prediction: empty set, linearity (test_krige_metrics.cpp:24-29, 62-78)
    const auto all = random_locations(300, 5);
    std::vector<Location> tr(all.begin(), all.begin() + 256), te(all.begin() + 256, all.end());
    std::vector<Location> none;
    const MaternParams p{1.0, 0.1, 1.5, 1e-2};
    CHECK(predict(tr, Vector(256, 1.0), none, p).z2_hat.empty());
    std::mt19937_64 g(7);
    Vector z1(256), z2(256), mix(256);
    for (int i = 0; i < 256; ++i) {
      z1[i] = ((g() >> 11) + 0.5) * 0x1.0p-53 - 0.5;
      z2[i] = ((g() >> 11) + 0.5) * 0x1.0p-53 - 0.5;
      mix[i] = 1.7 * z1[i] - 0.4 * z2[i];
    }
    const auto a = predict(tr, z1, te, p).z2_hat, b = predict(tr, z2, te, p).z2_hat;
    const auto c = predict(tr, mix, te, p).z2_hat;
    double worst = 0;
    for (size_t i = 0; i < c.size(); ++i) worst = std::max(worst, std::abs(c[i] - (1.7 * a[i] - 0.4 * b[i])));
    CHECK(worst <= 1e-10);
  }
  {  // dense diagnostics (test_hmatrix.cpp:91-98, test_hfactor.cpp:71-99)
    std::vector<Location> one{{0.4, 0.6}};
    ClusterTree t1(one, 32);
    BlockClusterTree b1(t1, t1, 2.0);
    const HMatrix h1 = assemble(b1, one, MaternParams{1.2, 0.1, 0.5, 0.3}, RankControl::fixed_accuracy(1e-6));
    CHECK(std::abs(h1.to_dense()(0, 0) - 1.5) <= 1.5e-14);
    const auto pts = random_locations(512, 31);
    ClusterTree t(pts, 32);
    BlockClusterTree b(t, t, 2.0);
    const MaternParams p{1.0, 0.1, 0.5, 0.01};
    const HMatrix h = assemble(b, pts, p, RankControl::fixed_accuracy(1e-6));
    const Matrix d = h.to_dense();
    const HFactor fc = h_cholesky(h, 1e-6);
    const Matrix rc = fc.reconstruct();
    double num = 0, den = 0;
    for (size_t e = 0; e < d.data.size(); ++e) {
      num += (rc.data[e] - d.data[e]) * (rc.data[e] - d.data[e]);
      den += d.data[e] * d.data[e];
    }
    CHECK(std::sqrt(num / den) <= 1e-4);
    const Matrix l = h_ldl(h, 1e-6).lower_dense();
    CHECK(l(0, 0) == 1.0 && l(0, 1) == 0.0);
  }
  {  // kriging variance and MLOE/MMOM (test_krige_metrics.cpp:80-91, 137-145, 212-244)
    const auto train = random_locations(256, 9);
    const MaternParams p{2.0, 0.1, 1.5, 0.0};
    std::vector<Location> test{train[17], {123.0, -55.0}};
    const Vector var = kriging_variance_dense(train, test, p);
    CHECK(std::abs(var[0]) <= 1e-10);
    CHECK(std::abs(var[1] - 2.0) <= 2e-12);
    const auto pts = random_locations(64, 20);
    MetricConfig cfg;
    cfg.M = 64;
    const MaternParams t{1.5, 0.1, 0.5, 0.0};
    const MloeMmom m = mloe_mmom(pts, t, t, cfg);
    CHECK(std::abs(m.mloe) <= 1e-8 && std::abs(m.mmom) <= 1e-8);
    const auto pts30 = random_locations(64, 30);
    const MloeMmom v = mloe_mmom(pts30, t, MaternParams{0.6, 0.1, 0.5, 0.0}, cfg);
    CHECK(std::abs(v.mloe) <= 1e-10 && std::abs(v.mmom) > 0.1);
    MetricConfig bad;
    bad.M = 0;
    CHECK_THROWS_AS(mloe_mmom(random_locations(8, 1), t, t, bad), std::invalid_argument);
    bad.M = 4;
    bad.dense_guard = 4;
    CHECK_THROWS_AS(mloe_mmom(random_locations(8, 1), t, t, bad), std::invalid_argument);
    CHECK(std::abs(rmse(Vector{1, 2, 3}, Vector{0, 0, 0}) - 2.1602468994692869) <= 1e-14);
    CHECK_THROWS_AS(rmse(Vector{1, 1}, Vector{1, 1, 1}), std::invalid_argument);
  }
  {  // sharded assembly: contiguous ranges, shards refuse matvec
    const auto pts = random_locations(2000, 8);
    ClusterTree t(pts, 32);
    BlockClusterTree b(t, t, 2.0);
    const MaternParams p{1.0, 0.1, 0.5, 0.01};
    const HMatrix s0 = assemble_shard(b, p, RankControl::fixed_accuracy(1e-6), 0, 2);
    const HMatrix s1 = assemble_shard(b, p, RankControl::fixed_accuracy(1e-6), 1, 2);
    CHECK(s0.leaf_range().first == 0 && s0.leaf_range().second == s1.leaf_range().first);
    CHECK(s1.leaf_range().second > s1.leaf_range().first);
    CHECK_THROWS_AS(s0.matvec(Vector(2000, 1.0)), std::invalid_argument);
  }
  {  // θ-sweep / kriging shards through the C ABI alone (csrc/sweep.cu)
    const auto pts = random_locations(1500, 3);
    ClusterTree t(pts, 64);
    Vector z(1500);
    for (int i = 0; i < 1500; ++i) z[i] = std::sin(0.37 * i);
    HConfig cfg;
    cfg.leaf_size = 64;
    const hmgp_config hc = cfg.c();
    const hmgp_matern th[5] = {{1.0, 0.1, 0.5, 0.01}, {1.2, 0.07, 1.1, 0.001}, {0.8, 0.12, 1.5, 0.01},
                               {1.0, 0.05, 0.3, 0.01}, {1.5, 0.1, 0.7, 0.001}};
    // shards partition the list, nu-major round-robin
    int32_t i0[5], i1[5];
    int c0 = 0, c1 = 0;
    CHECK(hmgp_sweep_shard(th, 5, 0, 2, i0, &c0) == HMGP_OK && hmgp_sweep_shard(th, 5, 1, 2, i1, &c1) == HMGP_OK);
    CHECK(c0 + c1 == 5 && c0 == 3);
    // the sweep equals single evaluations bit for bit
    hmgp_loglik_result rows[5];
    CHECK(hmgp_loglik_sweep(detail::context(), t.handle(), z.data(), th, 5, &hc, rows) == HMGP_OK);
    for (int k = 0; k < 5; ++k) {
      const LogLikResult one = evaluate_loglik(pts, z, MaternParams{th[k].sigma2, th[k].ell, th[k].nu, th[k].tau2}, cfg);
      CHECK(rows[k].loglik == one.loglik && rows[k].logdet == one.logdet);
    }
    // world-1 communicator: gather = scatter by index; rows nobody evaluated keep status -2
    hmgp_comm* comm = nullptr;
    char id[128] = {};
    CHECK(hmgp_comm_create(detail::context(), id, 0, 1, &comm) == HMGP_OK);
    hmgp_loglik_result table[5];
    const int32_t mine[2] = {3, 1};
    CHECK(hmgp_sweep_gather(detail::context(), comm, mine, rows, 2, 5, table) == HMGP_OK);
    CHECK(table[3].loglik == rows[0].loglik && table[1].loglik == rows[1].loglik && table[0].status == -2);
    int b = -1, e = -1;
    CHECK(hmgp_predict_range(10, 1, 4, &b, &e) == HMGP_OK && b == 2 && e == 5);
    double loc[3] = {1, 2, 3}, out[3] = {};
    CHECK(hmgp_predict_gather(detail::context(), comm, loc, 3, out) == HMGP_OK && out[2] == 3.0);
    hmgp_comm_destroy(comm);
    hmgp_release_workspace();
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
