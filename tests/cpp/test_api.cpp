// Drop-in check of include/hmgp/hmgp.hpp: the reference's own hand cases and
// API contracts (tests/test_geometry.cpp, test_hfactor.cpp, test_loglik_mle.cpp,
// test_krige_metrics.cpp under /root/reference/proj) through the C++ mirror
// that a reference user would compile against.  Prints one line per check and
// exits non-zero on any failure.  Run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
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

int main() {
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
    for (const auto& l : bt.leaves()) {
      for (int i = l.row_begin; i < l.row_end; ++i)
        for (int j = l.col_begin; j < l.col_end; ++j) cnt[i * 256 + j]++;
      if (l.row_begin == l.col_begin && l.row_end == l.col_end) CHECK(!l.admissible);
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
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
