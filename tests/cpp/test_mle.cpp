// Drop-in check of include/hmgp/mle.hpp: the reference's MLE test cases
// (/root/reference/proj/tests/test_loglik_mle.cpp:96-215) through the C++
// mirror.  `--host-only` runs the cases that need no GPU (reparameterisation,
// Brent); without it the fit cases run too (GPU L(θ), GPU sample_grf).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>

#include "hmgp/mle.hpp"

using namespace hmgp;

static int g_fail = 0;
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                               \
    }                                                         \
  } while (0)

static bool close_rel(double a, double b, double r) { return std::abs(a - b) <= r * std::max(std::abs(b), 1.0); }

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
  {  // reparameterization maps (96-108)
    const MaternParams z = reparam_to_params({0.0, 0.0, 0.0, 0.0});
    CHECK(z.sigma2 == 4.0 && z.ell == 1.0 && z.nu == 1.0 && z.tau2 == 1.0);
    const MaternParams i = reparam_to_params({2.0, 2.0, 1.0, 15.0});
    CHECK(std::abs(i.sigma2 - 2.73205382146028) <= 1e-12 * 2.73205382146028);
    CHECK(std::abs(i.ell - 1.0 / 2.25) <= 1e-14);
    CHECK(std::abs(i.nu - 1.0 / 1.2) <= 1e-14);
    CHECK(std::abs(i.tau2 - 9.31322574615479e-10) <= 1e-12 * 9.31322574615479e-10);
  }
  {  // round trips (110-122)
    for (const ReparamPoint p0 : {ReparamPoint{0, 0, 0, 0}, ReparamPoint{2, 2, 1, 15},
                                  ReparamPoint{-3.5, 4.2, -1.1, 7.7}}) {
      const ReparamPoint b = params_to_reparam(reparam_to_params(p0));
      for (int k = 0; k < 4; ++k) CHECK(close_rel(b[k], p0[k], 1e-12));
    }
    CHECK(reparam_to_params({50.0, -40.0, 30.0, 60.0}).valid());
  }
  {  // Brent (124-147)
    auto r = brent_max_1d([](double x) { return -(x - 1.0) * (x - 1.0); }, -4.0, 4.0, 1e-8, 200);
    CHECK(std::abs(r.x - 1.0) <= 1e-7 && r.evals <= 200);
    r = brent_max_1d([](double x) { return -std::abs(x); }, -3.0, 2.0, 1e-6, 200);
    CHECK(std::abs(r.x) <= 1e-5);
    r = brent_max_1d([](double x) { return x < 0.0 ? std::nan("") : -(x - 2.0) * (x - 2.0); }, -1.0, 5.0,
                     1e-8, 200);
    CHECK(std::abs(r.x - 2.0) <= 1e-6);
    bool threw = false;
    try {
      brent_max_1d([](double) { return std::nan(""); }, 0.0, 1.0, 1e-8, 50);
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
      brent_max_1d([](double x) { return x; }, 1.0, 0.0, 1e-8, 50);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  if (!host_only) {
    {  // small fit beats the truth likelihood and ascends (180-199)
      const auto pts = random_locations(256, 8);
      const MaternParams truth{1.5, 0.1, 0.5, 0.0};
      const Vector z = sample_grf(pts, truth, 12);
      OptimizerConfig cfg;
      cfg.h.rank = RankControl::fixed_accuracy(1e-4);
      cfg.brent_max_evals = 20;
      const FitReport rep = fit(pts, z, cfg);
      CHECK(rep.iterations <= cfg.max_iters);
      double prev = -std::numeric_limits<double>::infinity();
      for (const FitTraceEntry& t : rep.trace) {
        CHECK(t.loglik >= prev);
        prev = t.loglik;
      }
      CHECK(rep.loglik_at_opt >= evaluate_loglik(pts, z, truth, cfg.h).loglik - 1e-3);
      CHECK(rep.theta_hat.valid());
      std::printf("fit n=256: %d iterations, %d L(theta) probes, %.3f s, L=%.10f theta=(%.6f %.6f %.6f %.3g)\n",
                  rep.iterations, rep.evaluations, rep.seconds, rep.loglik_at_opt, rep.theta_hat.sigma2,
                  rep.theta_hat.ell, rep.theta_hat.nu, rep.theta_hat.tau2);
    }
    {  // fit is bit-reproducible (201-215)
      const auto pts = random_locations(200, 14);
      const Vector z = sample_grf(pts, {1.0, 0.1, 0.5, 0.0}, 3);
      OptimizerConfig cfg;
      cfg.h.rank = RankControl::fixed_accuracy(1e-4);
      cfg.max_iters = 12;
      const FitReport a = fit(pts, z, cfg), b = fit(pts, z, cfg);
      CHECK(a.trace.size() == b.trace.size());
      for (size_t i = 0; i < a.trace.size() && i < b.trace.size(); ++i) {
        CHECK(a.trace[i].loglik == b.trace[i].loglik);
        CHECK(a.trace[i].point.sigma0 == b.trace[i].point.sigma0);
        CHECK(a.trace[i].point.tau0 == b.trace[i].point.tau0);
      }
      CHECK(a.loglik_at_opt == b.loglik_at_opt);
    }
    {  // argument checks (154-158)
      const auto pts = random_locations(4, 1);
      bool threw = false;
      try {
        fit(pts, Vector(3, 0.0));
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      CHECK(threw);
    }
  }
  if (g_fail == 0) std::printf("ALL PASSED\n");
  return g_fail == 0 ? 0 : 1;
}
