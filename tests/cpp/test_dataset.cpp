// Host-only port of /root/reference/proj/tests/test_io.cpp:28-150 against
// include/hmgp/dataset.hpp (point CSV, dataset split, fit report v1).
#include <unistd.h>

#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <random>

#include "hmgp/dataset.hpp"

using namespace hmgp;

static int g_fail = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++g_fail;                                                    \
    }                                                              \
  } while (0)
#define CHECK_THROWS_RT(expr)                     \
  do {                                            \
    bool ok_ = false;                             \
    try {                                         \
      (void)(expr);                               \
    } catch (const std::runtime_error&) {         \
      ok_ = true;                                 \
    }                                             \
    CHECK(ok_);                                   \
  } while (0)

static std::string slurp(const std::string& p) {
  std::ifstream f(p, std::ios::binary);
  return std::string((std::istreambuf_iterator<char>(f)), {});
}

int main() {
  const auto dir = std::filesystem::temp_directory_path() / ("hmgp_io_" + std::to_string(::getpid()));
  std::filesystem::create_directories(dir);
  auto file = [&](const char* n) { return (dir / n).string(); };
  {  // round trip, exact values, byte-identical rewrite
    PointSet ps;
    ps.locations = random_locations(1000, 5);
    ps.has_values = true;
    std::mt19937_64 g(9);
    std::normal_distribution<double> nd;
    for (int i = 0; i < 1000; ++i) ps.values.push_back(nd(g) * 1e3);
    write_points_csv(file("pts.csv"), ps);
    const PointSet back = read_points_csv(file("pts.csv"));
    CHECK(back.locations.size() == 1000 && back.has_values);
    bool same = true;
    for (int i = 0; i < 1000; ++i)
      same = same && back.locations[i].x == ps.locations[i].x && back.locations[i].y == ps.locations[i].y &&
             back.values[i] == ps.values[i];
    CHECK(same);
    write_points_csv(file("pts2.csv"), back);
    CHECK(slurp(file("pts.csv")) == slurp(file("pts2.csv")));
  }
  {  // header only; locations-only schema; CRLF
    std::ofstream(file("empty.csv")) << "x,y,z\n";
    const PointSet e = read_points_csv(file("empty.csv"));
    CHECK(e.locations.empty() && e.has_values);
    std::ofstream(file("loc.csv")) << "x,y\r\n0.5,0.25\r\n\r\n";
    const PointSet l = read_points_csv(file("loc.csv"));
    CHECK(l.locations.size() == 1 && !l.has_values && l.locations[0].x == 0.5);
  }
  {  // malformed input with line number, missing header, missing file, field counts
    std::ofstream(file("bad.csv")) << "x,y,z\n0.1,0.2,0.3\n0.4,oops,0.6\n";
    bool has_line = false;
    try {
      read_points_csv(file("bad.csv"));
    } catch (const std::runtime_error& e) {
      has_line = std::string(e.what()).find(":3") != std::string::npos;
    }
    CHECK(has_line);
    std::ofstream(file("nohdr.csv")) << "0.1,0.2,0.3\n";
    CHECK_THROWS_RT(read_points_csv(file("nohdr.csv")));
    CHECK_THROWS_RT(read_points_csv(file("missing.csv")));
    std::ofstream(file("short.csv")) << "x,y,z\n0.1,0.2\n";
    CHECK_THROWS_RT(read_points_csv(file("short.csv")));
    std::ofstream(file("trail.csv")) << "x,y\n0.1,0.2,\n";
    CHECK_THROWS_RT(read_points_csv(file("trail.csv")));
    std::ofstream(file("inf.csv")) << "x,y\n0.1,inf\n";
    CHECK_THROWS_RT(read_points_csv(file("inf.csv")));
  }
  {  // fit report round trip
    FitReportFile rep;
    rep.theta = {1.4523e-3, 0.077, 1.51, 9.3e-10};
    rep.reparam = {2.5, 1.75, -0.25, 15.0};
    rep.loglik = -1234.5678901234567;
    rep.iterations = 37;
    rep.converged = true;
    rep.final_sweep_delta = 5.5e-5;
    rep.seconds = 12.25;
    rep.trace.push_back({1, 0, {2.0, 2.0, 1.0, 15.0}, -2000.0});
    rep.trace.push_back({2, 1, {2.5, 1.9, 1.0, 15.0}, -1500.0});
    write_fit_report(file("fit.txt"), rep);
    const FitReportFile b = read_fit_report(file("fit.txt"));
    CHECK(b.theta.sigma2 == rep.theta.sigma2 && b.theta.ell == rep.theta.ell && b.theta.nu == rep.theta.nu &&
          b.theta.tau2 == rep.theta.tau2);
    CHECK(b.reparam.sigma0 == rep.reparam.sigma0 && b.reparam.tau0 == 15.0);
    CHECK(b.loglik == rep.loglik && b.iterations == 37 && b.converged);
    CHECK(b.eps == 1e-6 && b.seconds == 12.25 && b.leaf_size == 32);
    CHECK(slurp(file("fit.txt")).find("trace:\niter coord sigma0 ell0 nu0 tau0 loglik\n1 0 2 2 1 15 -2000\n") !=
          std::string::npos);
    std::ofstream(file("junk.txt")) << "not a report\n";
    CHECK_THROWS_RT(read_fit_report(file("junk.txt")));
  }
  {  // dataset split io
    Dataset ds;
    ds.train.locations = random_locations(90, 3);
    ds.train.has_values = true;
    for (int i = 0; i < 90; ++i) ds.train.values.push_back(i / 89.0);
    ds.test.locations = random_locations(10, 4);
    write_dataset(ds, file("tr.csv"), file("te.csv"));
    const Dataset back = read_dataset(file("tr.csv"), file("te.csv"));
    CHECK(back.train.locations.size() == 90 && back.train.has_values);
    CHECK(back.test.locations.size() == 10 && !back.test.has_values);
  }
  std::filesystem::remove_all(dir);
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
  return g_fail ? 1 : 0;
}
