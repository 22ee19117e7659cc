// Batched FP64 kernels for the H-factorization.  Every item carries its own
// pointers and may take a dimension from device memory (a low-rank block's
// current rank), so the host recursion never has to read ranks back.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hmgp_gpu {

// "int value or device pointer" dimension
struct Dim {
  int v;
  const int* p;
  __host__ __device__ int get() const { return p ? *p : v; }
};
inline Dim dimv(int v) { return Dim{v, nullptr}; }
inline Dim dimp(const int* p, int cap) { return Dim{cap, p}; }

// C (M x N, ldc) += alpha * op(A) * op(B); op(A) is M x K, op(B) is K x N.
struct GemmItem {
  const double* A;
  const double* B;
  double* C;
  int lda, ldb, ldc;
  Dim M, N, K;
  int ta, tb;
  double alpha;
  int atomic;  // 0: C += ..., 2: C = ... (overwrite; the item owns its C).  (No FP64
               // atomics: shared targets go through k_ordered_add, split-K through
               // separate slabs + k_slab_sum, so results are bit-reproducible.)
};

// M (b x cols) <- L^{-1} M (trans = 0) or L^{-T} M (trans = 1); L b x b lower,
// its stored diagonal used (unit for LDL since the diagonal holds 1.0).
struct TrsmLItem {
  const double* L;
  int ldl, b;
  double* M;
  int ldm;
  Dim cols;
  int trans;
};

// X (s x t) <- X L^{-T}
struct TrsmRItem {
  const double* L;
  int ldl, t;
  double* X;
  int ldx, s;
  const double* d;  // optional: then column j /= d[j] (LDL, hfactor.cpp:205-207)
};

// dst (rows x cols) = alpha * op(src) [.* scale], scale by d on rows (mode 1 mul,
// 2 div) or columns (3 mul, 4 div), mode 0 none.  src == nullptr -> fill with
// alpha * I (identity) or zero (alpha == 0).  Optionally sets *dst_cols.
struct CopyScaleItem {
  const double* src;
  int lds;
  double* dst;
  int ldd;
  int rows;
  Dim cols;
  int trans;  // dst = src^T
  double alpha;
  const double* d;
  int mode;
  int* set_cols;  // if not null: *set_cols = cols
  int accum;      // dst += value instead of dst = value
};

// Append alpha*P (pr x add) at row offset pro into U (um rows, ld um) after its
// current `*rank` columns, and Q (qr x add) at row qro into V; zero elsewhere;
// rank += add.  If cap < rank + add: error flag.
struct AppendItem {
  double* U;
  double* V;
  int um, vn;
  const double* P;
  const double* Q;
  int ldp, ldq, pr, qr, pro, qro;
  Dim add;
  double alpha;
  int* rank;
  int cap;
};

// ordered accumulation (see k_ordered_add)
struct OrdSeg {
  const double* src;  // rows [r0, r0 + rows) of the target, column stride lds
  int lds, r0;
};
struct OrdIv {
  double* y;
  int ldy;
  Dim cols;
  double alpha;
  int i0, i1;  // target rows of the interval
  int l0, l1;  // its segments (in order) in the segment array
};
// p[0 .. rows x cols, ld] += sum_{s >= 1} p[s * slab + ...]
struct SlabSumItem {
  double* p;
  int ld;
  Dim rows, cols;
  int nslab;
  size_t slab;
};

struct LeafFactorStatus {
  int fail_pos;  // min tree position of a failing pivot (INT_MAX if none)
  int clamped, negative;
  int pad;
  double fail_val;
  double min_pivot;
  // pivot clamp 1e-14 * max_diag (hfactor.cpp:349), set per evaluation: the leaf
  // kernels read it here when launched with clamp_tol < 0, so that a captured
  // launch sequence carries no θ-dependent scalar
  double clamp_tol;
};

void launch_gemm(const GemmItem* d_items, int count, int max_tiles, cudaStream_t st);
// per-target ordered sequences: CTA b runs items[off[b]..off[b+1]) in order
void launch_gemm_seq(const GemmItem* d_items, const int* d_off, int targets, cudaStream_t st);
void launch_ordered_add(const OrdIv* d_iv, int count, const OrdSeg* d_segs, int max_elems,
                        cudaStream_t st);
void launch_slab_sum(const SlabSumItem* d_items, int count, int max_elems, cudaStream_t st);
void launch_trsm_left(const TrsmLItem* d_items, int count, int max_cols, cudaStream_t st,
                      int max_b);
void launch_trsm_right(const TrsmRItem* d_items, int count, int max_rows, cudaStream_t st,
                       int max_t);
void launch_copy_scale(const CopyScaleItem* d_items, int count, int max_elems, cudaStream_t st);
void launch_append(const AppendItem* d_items, int count, int max_elems, int* d_err, cudaStream_t st);
// one diagonal leaf (b x b at D, ld b), tree rows [base, base+b); LDL writes d[base..]
void launch_leaf_factor(double* D, int b, int base, int ldl, double* d, double clamp_tol,
                        LeafFactorStatus* status, cudaStream_t st);

}  // namespace hmgp_gpu
