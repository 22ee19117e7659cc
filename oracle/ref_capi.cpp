// extern "C" shim over the UNMODIFIED reference sources
//   /root/reference/proj/src/geometry.cpp   (ClusterTree, BlockClusterTree)
//   /root/reference/proj/src/covkernel.cpp  (bessel_k, matern, KernelEvaluator)
// compiled straight from /root/reference by oracle/Makefile into
// oracle/_ref/libhmgp_ref.so.  TEST INFRASTRUCTURE ONLY: tests/ and bench.py's
// cpu_baseline leg load it as the checker; the product never links it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include "hmgp/covkernel.hpp"
#include "hmgp/geometry.hpp"

using namespace hmgp;

namespace {
thread_local char g_err[512];
int fail(const std::exception& e, int code) {
  std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
  return code;
}
// 1 = invalid_argument, 2 = domain_error, 3 = out_of_range, 9 = other
#define REF_GUARD(...)                                   \
  try {                                                   \
    __VA_ARGS__;                                          \
    return 0;                                             \
  } catch (const std::invalid_argument& e) {              \
    return fail(e, 1);                                    \
  } catch (const std::domain_error& e) {                  \
    return fail(e, 2);                                    \
  } catch (const std::out_of_range& e) {                  \
    return fail(e, 3);                                    \
  } catch (const std::exception& e) {                     \
    return fail(e, 9);                                    \
  }

std::vector<Location> to_locs(const double* xy, int n) {
  std::vector<Location> p(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) p[i] = {xy[2 * i], xy[2 * i + 1]};
  return p;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

// perm[n]; node arrays in pre-order (begin, end, box lo/hi x/y)
int ref_cluster_tree(const double* xy, int n, int leaf, int32_t* perm, int32_t* inv_perm,
                     int* n_leaves) {
  REF_GUARD({
    const auto pts = to_locs(xy, n);
    ClusterTree t(pts, leaf);
    for (int i = 0; i < n; ++i) {
      perm[i] = t.perm()[i];
      inv_perm[i] = t.inverse_perm()[i];
    }
    *n_leaves = static_cast<int>(t.leaves().size());
  })
}

// Block leaves in the reference's DFS order: (row_begin,row_end,col_begin,col_end,tag)
// tag 0 = admissible, 1 = dense.  cap = capacity of `out` in blocks.
int ref_block_tree(const double* xy, int n, int leaf, double eta, int32_t* out, int64_t cap,
                   int64_t* count, int* n_adm, int* n_dense) {
  REF_GUARD({
    const auto pts = to_locs(xy, n);
    ClusterTree t(pts, leaf);
    BlockClusterTree bt(t, t, eta);
    const auto& lv = bt.leaves();
    *count = static_cast<int64_t>(lv.size());
    *n_adm = bt.admissible_count();
    *n_dense = bt.dense_count();
    if (static_cast<int64_t>(lv.size()) > cap) throw std::out_of_range("ref_block_tree: cap");
    for (size_t k = 0; k < lv.size(); ++k) {
      out[5 * k + 0] = lv[k]->row->begin;
      out[5 * k + 1] = lv[k]->row->end;
      out[5 * k + 2] = lv[k]->col->begin;
      out[5 * k + 3] = lv[k]->col->end;
      out[5 * k + 4] = lv[k]->tag == BlockClusterTree::Node::Tag::Admissible ? 0 : 1;
    }
  })
}

int ref_bessel_k(double nu, double x, double* out) { REF_GUARD(*out = bessel_k(nu, x)) }
int ref_bessel_k_generic(double nu, double x, double* out) {
  REF_GUARD(*out = detail::bessel_k_generic(nu, x))
}
int ref_matern(double h, const double* theta, double* out) {
  REF_GUARD({
    MaternParams p{theta[0], theta[1], theta[2], theta[3]};
    *out = matern(h, p);
  })
}
int ref_matern_generic(double h, const double* theta, double* out) {
  REF_GUARD({
    MaternParams p{theta[0], theta[1], theta[2], theta[3]};
    *out = detail::matern_generic(h, p);
  })
}

// KernelEvaluator(i, j) over index pairs (original indices).
int ref_kernel_pairs(const double* xy, int n, const double* theta, const int32_t* ii,
                     const int32_t* jj, int64_t count, double* out) {
  REF_GUARD({
    const auto pts = to_locs(xy, n);
    MaternParams p{theta[0], theta[1], theta[2], theta[3]};
    KernelEvaluator k(pts, p);
    for (int64_t t = 0; t < count; ++t) out[t] = k(ii[t], jj[t]);
  })
}

// KernelEvaluator::at_distance over a distance list.
int ref_at_distance(const double* theta, const double* h, int64_t count, double* out) {
  REF_GUARD({
    std::vector<Location> none;
    MaternParams p{theta[0], theta[1], theta[2], theta[3]};
    KernelEvaluator k(none, p);
    for (int64_t t = 0; t < count; ++t) out[t] = k.at_distance(h[t]);
  })
}

// cov_block(rows, cols) column-major.
int ref_cov_block(const double* xy, int n, const double* theta, const int32_t* rows, int nr,
                  const int32_t* cols, int nc, double* out) {
  REF_GUARD({
    const auto pts = to_locs(xy, n);
    MaternParams p{theta[0], theta[1], theta[2], theta[3]};
    std::vector<int> r(rows, rows + nr), c(cols, cols + nc);
    const auto b = cov_block(r, c, pts, p);
    std::memcpy(out, b.data(), sizeof(double) * static_cast<size_t>(nr) * nc);
  })
}

}  // extern "C"
