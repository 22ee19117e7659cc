/*
 * hmgp_cuda.h — C ABI of the B200-native hmgp hot path (Gaussian log-likelihood
 * and kriging through an H-matrix LDL^T / Cholesky, arXiv 2104.07146).
 *
 * This is the drop-in boundary: plain pointers and sizes, int status codes, no
 * torch or C++ types.  Every entry point replaces one reference C++ interface
 * (paths relative to /root/reference/proj) and keeps its argument meaning and
 * error behaviour; the C++ shim include/hmgp/hmgp.hpp maps the status codes
 * back onto the reference's exception types.
 *
 * Conventions: coordinates are AoS FP64 (x, y[, z]) per point in ORIGINAL
 * order (dim = 2 as in the reference; dim = 3 extends it for BASELINE config C5);
 * vectors are FP64 in original index order; all pointers are HOST pointers
 * unless the name starts with d_ (device).  Functions are thread-safe per
 * context; one context = one device + one stream.
 */
#ifndef HMGP_CUDA_H
#define HMGP_CUDA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (reference exception in brackets) */
enum {
  HMGP_OK = 0,
  HMGP_EINVAL = 1,    /* std::invalid_argument */
  HMGP_EDOMAIN = 2,   /* std::domain_error (bessel_k domain, indefinite log_det) */
  HMGP_ERANGE = 3,    /* std::out_of_range (cov_block indices) */
  HMGP_ENOTSPD = 4,   /* hmgp::FactorError (pivot_index / pivot_value set) */
  HMGP_ECUDA = 5,     /* CUDA runtime failure */
  HMGP_ECAPACITY = 6, /* a device workspace bound was exceeded */
  HMGP_ERUNTIME = 7   /* std::runtime_error (sample_grf: covariance not SPD) */
};

typedef struct hmgp_ctx hmgp_ctx;
typedef struct hmgp_geom hmgp_geom;
typedef struct hmgp_hmat hmgp_hmat;
typedef struct hmgp_factor hmgp_factor;

/* hmgp::MaternParams (covkernel.hpp:11-19) */
typedef struct hmgp_matern {
  double sigma2, ell, nu, tau2;
} hmgp_matern;

/* hmgp::RankControl (hmatrix.hpp:17-36): mode 0 = FixedAccuracy(eps), 1 = FixedRank(rank) */
typedef struct hmgp_rank_control {
  int mode;
  double eps;
  int rank;
  int max_rank;
} hmgp_rank_control;

/* hmgp::HConfig (pipeline.hpp:13-25); form 1 = Ldl (default), 0 = Cholesky */
typedef struct hmgp_config {
  double eta;
  int leaf_size;
  hmgp_rank_control rank;
  double eps_factor;
  int form;
  int threads; /* accepted for API parity; the GPU path ignores it */
} hmgp_config;

/* one block-tree leaf in the reference's DFS order (geometry.cpp:100-117) */
typedef struct hmgp_block {
  int32_t row_begin, row_end, col_begin, col_end;
  int32_t tag; /* 0 = Admissible, 1 = Dense */
} hmgp_block;

/* hmgp::FactorInfo (hfactor.hpp:24-29) + HFactor::storage_bytes (hfactor.cpp:412-419) */
typedef struct hmgp_factor_info {
  double eps;
  int clamped, negative;
  double min_pivot;
  double storage_bytes;
} hmgp_factor_info;

/* hmgp::LogLikResult (loglik.hpp:10-17); status 0 = Success, 1 = Clamped */
typedef struct hmgp_loglik_result {
  double loglik, logdet, quad_form;
  int n;
  double seconds;
  int status;
} hmgp_loglik_result;

/* ------------------------------------------------------------- context --- */
int hmgp_ctx_create(int device, hmgp_ctx** out);
void hmgp_ctx_destroy(hmgp_ctx* ctx);
const char* hmgp_last_error(void);          /* thread-local message of the last failure */
int hmgp_last_pivot_index(void);            /* FactorError::pivot_index (original index) */
double hmgp_last_pivot_value(void);         /* FactorError::pivot_value */
uint64_t hmgp_kernel_launches(hmgp_ctx* ctx);  /* device kernels launched by this context */
void hmgp_default_config(hmgp_config* cfg);    /* HConfig{} defaults */

/* ------------------------------------------------------------ geometry --- */
/* ClusterTree(points, leaf_size) + BlockClusterTree(tree, tree, eta):
 * geometry.cpp:41-54, 100-117 / build_cluster_tree, build_block_tree (geometry.hpp:68,108) */
int hmgp_geometry_build(hmgp_ctx* ctx, const double* coords, int n, int dim, int leaf_size,
                        double eta, hmgp_geom** out);
/* same, coordinates already in device memory (AoS) */
int hmgp_geometry_build_device(hmgp_ctx* ctx, const double* d_coords, int n, int dim,
                               int leaf_size, double eta, hmgp_geom** out);
/* ClusterTree::perm / inverse_perm (geometry.hpp:53-55) */
int hmgp_geometry_perm(const hmgp_geom* g, int32_t* perm, int32_t* inv_perm);
/* cluster nodes in the reference's pre-order: begin, end, left, right (-1 = leaf) and
 * box lo[3], hi[3] (Cluster, geometry.hpp:33-42) */
int hmgp_geometry_clusters(const hmgp_geom* g, int32_t* out4, double* box6, int cap,
                           int* count);
/* BlockClusterTree::leaves / admissible_count / dense_count (geometry.hpp:92-94) */
int hmgp_geometry_block_count(const hmgp_geom* g, int64_t* count, int* n_admissible,
                              int* n_dense);
int hmgp_geometry_blocks(const hmgp_geom* g, hmgp_block* out, int64_t cap);
/* BlockClusterTree(rows, cols, eta) for two different cluster trees (geometry.cpp:100-154,
 * geometry.hpp:76): leaves in DFS order; out == NULL returns the count only */
int hmgp_block_tree_rect(hmgp_ctx* ctx, const hmgp_geom* rows, const hmgp_geom* cols, double eta,
                         hmgp_block* out, int64_t cap, int64_t* count, int* n_adm, int* n_dense);
void hmgp_geometry_destroy(hmgp_geom* g);

/* -------------------------------------------------------------- kernel --- */
/* KernelEvaluator(i, j) over index pairs (covkernel.hpp:45-48); coords host AoS */
int hmgp_kernel_pairs(hmgp_ctx* ctx, const double* coords, int n, int dim,
                      const hmgp_matern* theta, const int32_t* ii, const int32_t* jj,
                      int64_t count, double* out);
/* KernelEvaluator::at_distance (covkernel.cpp:230-246) */
int hmgp_at_distance(hmgp_ctx* ctx, const hmgp_matern* theta, const double* h, int64_t count,
                     double* out);
/* bessel_k (covkernel.cpp:196-204) and detail::bessel_k_generic (170-182), on device */
int hmgp_bessel_k(hmgp_ctx* ctx, const double* nu, const double* x, int64_t count, int generic,
                  double* out);

/* matern(h, params) (covkernel.cpp:206-214: pref * t^nu * bessel_k, no closed forms) and
 * detail::matern_generic (generic = 1: bessel_k_generic, covkernel.cpp:184-194), on device */
int hmgp_matern_values(hmgp_ctx* ctx, const hmgp_matern* theta, const double* h, int64_t count, int generic,
                       double* out);

/* ------------------------------------------------------------ H-matrix --- */
/* assemble(block_tree, locations, params, rc) (hmatrix.hpp:88-89) */
int hmgp_assemble(hmgp_ctx* ctx, hmgp_geom* g, const hmgp_matern* theta,
                  const hmgp_rank_control* rc, hmgp_hmat** out);
/* HMatrix::storage / max_leaf_rank / max_diagonal (hmatrix.hpp:60-66) */
int hmgp_hmat_stats(const hmgp_hmat* h, double* bytes, int* max_rank, double* max_diag);
/* stored leaves in assembly order: row_begin,row_end,col_begin,col_end,kind(1 dense, 2 low-rank),rank
 * (out6 == NULL: *count only) */
int hmgp_hmat_leaves(const hmgp_hmat* h, int32_t* out6, int64_t cap, int64_t* count);
/* payload of stored leaf k: dense -> a (m x n col-major); low-rank -> a = U, b = V */
int hmgp_hmat_leaf_data(const hmgp_hmat* h, int64_t k, double* a, double* b);
/* HMatrix::matvec (hmatrix.cpp:244-272), original order */
int hmgp_hmat_matvec(hmgp_ctx* ctx, const hmgp_hmat* h, const double* x, double* y);
/* the same product with DEVICE vectors (original order), enqueued on the context's
   stream without a synchronisation: the HBM-bound pass alone (bench roofline) */
int hmgp_hmat_matvec_device(hmgp_ctx* ctx, const hmgp_hmat* h, const double* d_x, double* d_y);
/* from_dense(m) (hmatrix.cpp:223-242): single Dense leaf, self-contained tree; a is n x n
 * column-major (host).  hmgp_hmat_symmetric: HMatrix::symmetric() (isApprox(m, m^T)) */
int hmgp_hmat_from_dense(hmgp_ctx* ctx, const double* a, int n, hmgp_hmat** out);
int hmgp_hmat_symmetric(const hmgp_hmat* h, int* out);
void hmgp_hmat_destroy(hmgp_hmat* h);

/* -------------------------------------------------------------- factor --- */
/* factorize(h, eps_f, form) (hfactor.hpp:70-77).  HMGP_ENOTSPD -> FactorError */
int hmgp_factorize(hmgp_ctx* ctx, hmgp_hmat* h, double eps_f, int form, hmgp_factor** out,
                   hmgp_factor_info* info);
/* HFactor::log_det / quad_form / solve_factored / solve_lower / diagonal (hfactor.hpp:40-50) */
int hmgp_log_det(hmgp_ctx* ctx, const hmgp_factor* f, double* out);
int hmgp_quad_form(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* out);
int hmgp_solve_factored(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* x);
int hmgp_solve_lower(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* x);
int hmgp_factor_diagonal(hmgp_ctx* ctx, const hmgp_factor* f, double* out);
/* Dense diagnostics, n <= 4096 (HMGP_EINVAL beyond), out n x n column-major:
   HMatrix::to_dense (hmatrix.cpp:274-297, original order),
   HFactor::lower_dense (hfactor.cpp:421-434, tree order),
   HFactor::reconstruct (hfactor.cpp:436-449, L D L^T / L L^T, original order) */
/* Leaf-range shard of assemble for multi-GPU assembly: the
   DFS-ordered stored-leaf list is cut into n_shards contiguous ranges of near-equal
   cost (dense m·n, admissible 16·(m+n); hmgp_balanced_ranges) and only range
   `shard` is assembled — its leaves are bit-identical to a full hmgp_assemble.
   The result is for leaf queries only (hmgp_hmat_leaves reports rank -2 outside
   the range; matvec / factorize / to_dense refuse it). */
int hmgp_assemble_shard(hmgp_ctx* ctx, hmgp_geom* g, const hmgp_matern* theta, const hmgp_rank_control* rc,
                        int shard, int n_shards, hmgp_hmat** out, int* leaf_begin, int* leaf_end);
/* bounds[0..parts]: contiguous ranges of cost[0..count) with near-equal sums (host) */
int hmgp_balanced_ranges(const double* cost, int count, int parts, int* bounds);
int hmgp_hmat_to_dense(hmgp_ctx* ctx, const hmgp_hmat* h, double* out);
int hmgp_factor_lower_dense(hmgp_ctx* ctx, const hmgp_factor* f, double* out);
int hmgp_factor_reconstruct(hmgp_ctx* ctx, const hmgp_factor* f, double* out);
void hmgp_factor_destroy(hmgp_factor* f);

/* ------------------------------------------------------------ pipeline --- */
/* evaluate_loglik(locations, z, params, cfg) (loglik.hpp:22-23), host buffers */
int hmgp_loglik(hmgp_ctx* ctx, const double* coords, int n, int dim, const double* z,
                const hmgp_matern* theta, const hmgp_config* cfg, hmgp_loglik_result* res);
/* same L(θ) chain on a prebuilt geometry with device-resident z (original order) */
int hmgp_loglik_geom(hmgp_ctx* ctx, hmgp_geom* g, const double* d_z, const hmgp_matern* theta,
                     const hmgp_config* cfg, hmgp_loglik_result* res);
/* θ-batch: one geometry, many θ (C4 sweep); failures give status -1 and loglik = -inf */
int hmgp_loglik_batch(hmgp_ctx* ctx, hmgp_geom* g, const double* d_z, const hmgp_matern* thetas,
                      int ntheta, const hmgp_config* cfg, hmgp_loglik_result* res);
/* predict(train, z1, new_locations, params, cfg) (krige.hpp:19-21), host buffers */
int hmgp_predict(hmgp_ctx* ctx, const double* train, int n, int dim, const double* z1,
                 const double* test, int m, const hmgp_matern* theta, const hmgp_config* cfg,
                 double* out, double* seconds);
/* K12 alone: out_i = sum_j at_distance(|s_i - x_j|) w_j (krige.cpp:30-41), device buffers */
int hmgp_cross_apply_device(hmgp_ctx* ctx, const double* d_train, int n, int dim,
                            const double* d_w, const double* d_test, int m,
                            const hmgp_matern* theta, double* d_out);

/* ------------------------------------------- θ-sweep / kriging shards (§8e) */
/* One rank's share of a θ list on its GPU, z in HOST memory (uploaded once):
   the independent probes of the reference's MLE (mle.cpp:152-158).  Same result
   rows and failure mapping as hmgp_loglik_batch. */
int hmgp_loglik_sweep(hmgp_ctx* ctx, hmgp_geom* g, const double* z, const hmgp_matern* thetas,
                      int ntheta, const hmgp_config* cfg, hmgp_loglik_result* res);
/* Indices of the θ that `rank` of `world` evaluates: round-robin over the list
   sorted ν-major (stable), returned ascending.  idx may be NULL (count only). */
int hmgp_sweep_shard(const hmgp_matern* thetas, int ntheta, int rank, int world, int32_t* idx,
                     int* count);
/* Contiguous [begin, end) of m new locations predicted by `rank` of `world`. */
int hmgp_predict_range(int m, int rank, int world, int* begin, int* end);
/* NCCL plumbing for the two result gathers (libnccl resolved at first use).
   id128: a 128-byte ncclUniqueId made on one rank and sent to the others by the
   caller's launcher (MPI, torch.distributed, a file). */
typedef struct hmgp_comm hmgp_comm;
int hmgp_comm_unique_id(void* id128);
int hmgp_comm_create(hmgp_ctx* ctx, const void* id128, int rank, int world, hmgp_comm** out);
void hmgp_comm_destroy(hmgp_comm* comm);
/* ONE all-gather of this rank's rows into the θ-ordered table (ntheta rows) on
   every rank; rows nobody evaluated keep status -2 and loglik NaN.  comm == NULL
   or world 1: local scatter, no collective. */
int hmgp_sweep_gather(hmgp_ctx* ctx, hmgp_comm* comm, const int32_t* idx, const hmgp_loglik_result* local,
                      int count, int ntheta, hmgp_loglik_result* table);
/* ONE all-gather of the prediction slices (hmgp_predict_range) into out[m] on
   every rank; m == 0 returns without a collective. */
int hmgp_predict_gather(hmgp_ctx* ctx, hmgp_comm* comm, const double* local, int m, double* out);

/* Free the device workspaces the library keeps between calls: the calling
   thread's temporary arena and captured factorization, and those of the
   persistent θ-batch workers.  The next call allocates them again. */
void hmgp_release_workspace(void);

/* ------------------------------------------------------- instrumentation */
/* the context's CUDA stream (cudaStream_t), for event timing by callers */
int hmgp_ctx_stream(hmgp_ctx* ctx, void** stream);
/* per-phase device milliseconds of the last loglik / predict call on ctx:
 * [0] start [1] geometry [2] dense leaves K3 [3] ACA K4+K5 [4] layout/copies
 * [5] factorization K6-K9 [6] logdet [7] forward solve + quad [8] backward solve [9] K12 */
int hmgp_last_phases(hmgp_ctx* ctx, double* ms, int cap);
/* algorithmic work since the last reset: [0] dense entries [1] ACA entries
 * [2] Matérn flops of dense leaves (only when counting is on) [3] GEMM flops
 * [4] TRSM flops [5] leaf factor flops [6] recompression flops [7] recompressions */
int hmgp_work_counters(double* out, int cap, int reset);
/* enable the untimed Matérn flop-count pass inside assembly */
void hmgp_set_flop_counting(int on);
/* measured FP64 FMA-pipe peak of the device (TFLOP/s), FMA-chain microbenchmark */
int hmgp_fp64_peak(hmgp_ctx* ctx, double* tflops);

/* --------------------------------------------------------- data utilities */
/* simgen conventions (simgen.cpp:108-123): mt19937_64 + ((x>>11)+0.5)*2^-53 */
int hmgp_random_locations(int n, int dim, uint64_t seed, double* out);
/* jittered g x g grid */
int hmgp_jittered_grid(int g, uint64_t seed, double* out);
/* iid standard normals via AS241 (simgen.cpp:9-112) */
int hmgp_normals(int n, uint64_t seed, double* out);
/* sample_grf(locations, params, seed) (simgen.cpp:125-141): z = chol(cov_dense) w,
   w = AS241 normals of `seed`; dense on device, n <= 65536 (the reference caps at
   16384); HMGP_ERUNTIME when the covariance is not SPD.  Host buffers. */
int hmgp_sample_grf(hmgp_ctx* ctx, const double* coords, int n, int dim, const hmgp_matern* theta,
                    uint64_t seed, double* out);

/* ------------------------------------------- dense diagnostics */
/* kriging_variance_dense(train, new_locations, params) (krige.hpp / krige.cpp:46-74):
   out_i = σ²+τ² − c_iᵀ C11⁻¹ c_i, dense FP64 on device, n <= 4096 (HMGP_EINVAL beyond),
   HMGP_ERUNTIME when C11 is not SPD.  Host buffers. */
int hmgp_kriging_variance_dense(hmgp_ctx* ctx, const double* train, int n, int dim, const double* test, int m,
                                const hmgp_matern* theta, double* out);
/* mloe_mmom(locations, theta_true, theta_approx, MetricConfig{M, seed, dense_guard})
   (metrics.hpp:24-31 / metrics.cpp:17-69): leave-one-out kriging MLOE / MMOM closed
   forms, dense FP64 on device, n <= min(dense_guard, 32768).  Host buffers. */
int hmgp_mloe_mmom(hmgp_ctx* ctx, const double* coords, int n, int dim, const hmgp_matern* theta_true,
                   const hmgp_matern* theta_approx, int M, uint64_t seed, int dense_guard, double* mloe,
                   double* mmom);

#ifdef __cplusplus
}
#endif
#endif /* HMGP_CUDA_H */
