/* hmgp CPU oracle C API — TEST INFRASTRUCTURE ONLY (see hmgp_oracle.cpp). */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_EDOMAIN = 2, ORC_ERANGE = 3, ORC_ENOTSPD = 4, ORC_EOTHER = 9 };

typedef struct orc_config {
  double eta;        /* HConfig::eta */
  int leaf_size;     /* HConfig::leaf_size */
  double eps;        /* RankControl::eps (FixedAccuracy) */
  int fixed_rank;    /* > 0: RankControl::fixed_rank(k) */
  int max_rank;      /* RankControl::max_rank (256) */
  double eps_factor; /* HConfig::eps_factor (< 0: reuse eps) */
  int ldl;           /* 1 = FactorForm::Ldl, 0 = Cholesky */
  int threads;       /* assembly threads (0 = hardware concurrency) */
} orc_config;

typedef struct orc_factor_info {
  int clamped, negative;
  double min_pivot, storage_bytes;
} orc_factor_info;

typedef struct orc_loglik_result {
  double loglik, logdet, quad_form;
  int n, clamped;
  double seconds, t_tree, t_assemble, t_factor;
} orc_loglik_result;

typedef struct orc_problem orc_problem;

const char* orc_last_error(void);
int orc_last_pivot_index(void);
double orc_last_pivot_value(void);
void orc_counters(double* out11);
void orc_counters_reset(void);

int orc_cluster_tree(const double* x, int n, int dim, int leaf, int32_t* perm, int* n_nodes);
int orc_block_tree(const double* x, int n, int dim, int leaf, double eta, int32_t* out, int64_t cap,
                   int64_t* count, int* n_adm, int* n_dense);
int orc_bessel_k(double nu, double x, int generic, double* out);
int orc_matern(double h, const double* theta, int generic, double* out);
int orc_at_distance(const double* theta, const double* h, int64_t count, double* out);
int orc_kernel_pairs(const double* x, int n, int dim, const double* theta, const int32_t* ii,
                     const int32_t* jj, int64_t count, double* out);

int orc_problem_create(const double* x, int n, int dim, int leaf, double eta, orc_problem** out);
void orc_problem_destroy(orc_problem* p);
int orc_assemble(orc_problem* p, const double* theta, const orc_config* cfg, double* seconds);
int orc_leaves(orc_problem* p, int32_t* out, int64_t cap, int64_t* count);
int orc_leaf_data(orc_problem* p, int64_t k, double* a, double* b);
int orc_hmat_stats(orc_problem* p, double* bytes, int* max_rank, double* max_diag);
int orc_matvec(orc_problem* p, const double* x, double* y);
int orc_factorize(orc_problem* p, double eps_f, int ldl, orc_factor_info* info, double* seconds);
int orc_log_det(orc_problem* p, double* out);
int orc_quad_form(orc_problem* p, const double* z, double* out);
int orc_solve_factored(orc_problem* p, const double* b, double* x);
int orc_solve_lower(orc_problem* p, const double* b, double* x);
int orc_factor_diag(orc_problem* p, double* out);

int orc_loglik(const double* x, int n, int dim, const double* z, const double* theta,
               const orc_config* cfg, orc_loglik_result* res);
int orc_predict(const double* train, int n, int dim, const double* z1, const double* test, int m,
                const double* theta, const orc_config* cfg, double* out, double* seconds);
int orc_cross_apply(const double* train, int n, int dim, const double* w, const double* test, int m,
                    const double* theta, int threads, double* out);
int orc_dense_loglik(const double* x, int n, int dim, const double* z, const double* theta,
                     int threads, double* loglik, double* logdet, double* quad);
int orc_dense_predict(const double* train, int n, int dim, const double* z1, const double* test,
                      int m, const double* theta, int threads, double* out);
int orc_sample_grf(const double* x, int n, int dim, const double* theta, uint64_t seed, int threads,
                   double* z);
int orc_normal_quantile(double p, double* out);
int orc_random_locations(int n, int dim, uint64_t seed, double* out);
int orc_jittered_grid(int g, uint64_t seed, double* out);
int orc_kriging_variance_dense(const double* train, int n, int dim, const double* test, int m,
                               const double* th, double* out);
int orc_mloe_mmom(const double* x, int n, int dim, const double* tt, const double* ta, int M,
                  uint64_t seed, int dense_guard, double* mloe, double* mmom);
int orc_normals(int n, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
