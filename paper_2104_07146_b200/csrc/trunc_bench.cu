// Developer hook (not part of include/hmgp_cuda.h): time the batched
// recompression kernels on synthetic items so the truncation paths can be
// tuned in isolation (scripts/bench_trunc.py).
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "hmgp_internal.h"

namespace hmgp_gpu {
namespace {
uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  return x ^ (x >> 33);
}
double urand(uint64_t& s) {
  s = mix(s + 0x9e3779b97f4a7c15ULL);
  return (double)(s >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}
}  // namespace
}  // namespace hmgp_gpu

using namespace hmgp_gpu;

extern "C" int hmgp_debug_trunc_bench(int m, int n, int r0, int add, int count, int route, int reps,
                                      double eps, double decay, double* ms_out, int* keep_out) {
  try {
    const int r = r0 + add;
    uint64_t seed = 12345;
    // U (m x r), V (n x r) hold the current factor in the first r0 columns; P, Q the
    // appended ones.  Column l scaled by decay^l so the product is numerically low rank.
    std::vector<double> U((size_t)count * m * r), V((size_t)count * n * r), P((size_t)count * m * add + 1),
        Q((size_t)count * n * add + 1);
    for (int it = 0; it < count; ++it) {
      for (int l = 0; l < r; ++l) {
        const double sc = std::pow(decay, l);
        for (int i = 0; i < m; ++i) {
          const double v = sc * urand(seed);
          if (l < r0) U[(size_t)it * m * r + (size_t)l * m + i] = v;
          else P[(size_t)it * m * add + (size_t)(l - r0) * m + i] = v;
        }
        for (int i = 0; i < n; ++i) {
          const double v = urand(seed);
          if (l < r0) V[(size_t)it * n * r + (size_t)l * n + i] = v;
          else Q[(size_t)it * n * add + (size_t)(l - r0) * n + i] = v;
        }
      }
    }
    double *dU, *dV, *dP, *dQ, *dU0, *dV0, *ws;
    int *drank, *dcomp, *derr, *doff;
    const size_t wsd = std::max(std::max(trunc_ws_doubles(m, n, r), trunc_ws_doubles_pair(m, n, r)),
                                  trunc_ws_doubles_cluster(m, n, r)) + 64;
    HMGP_CUDA(cudaMalloc(&dU, U.size() * 8));
    HMGP_CUDA(cudaMalloc(&dV, V.size() * 8));
    HMGP_CUDA(cudaMalloc(&dU0, U.size() * 8));
    HMGP_CUDA(cudaMalloc(&dV0, V.size() * 8));
    HMGP_CUDA(cudaMalloc(&dP, P.size() * 8));
    HMGP_CUDA(cudaMalloc(&dQ, Q.size() * 8));
    HMGP_CUDA(cudaMalloc(&ws, wsd * count * 8));
    HMGP_CUDA(cudaMalloc(&drank, count * 4));
    HMGP_CUDA(cudaMalloc(&dcomp, count * 4));
    HMGP_CUDA(cudaMalloc(&derr, 4));
    HMGP_CUDA(cudaMalloc(&doff, (count + 1) * 4));
    HMGP_CUDA(cudaMemcpy(dU0, U.data(), U.size() * 8, cudaMemcpyHostToDevice));
    HMGP_CUDA(cudaMemcpy(dV0, V.data(), V.size() * 8, cudaMemcpyHostToDevice));
    HMGP_CUDA(cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice));
    HMGP_CUDA(cudaMemcpy(dQ, Q.data(), Q.size() * 8, cudaMemcpyHostToDevice));
    std::vector<int> off(count + 1), rk(count, r0);
    for (int i = 0; i <= count; ++i) off[i] = i;
    HMGP_CUDA(cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
    std::vector<TruncItem> items(count);
    for (int it = 0; it < count; ++it) {
      TruncItem& t = items[it];
      t = TruncItem{};
      t.U = dU + (size_t)it * m * r;
      t.V = dV + (size_t)it * n * r;
      t.m = m;
      t.n = n;
      t.rank = drank + it;
      t.compact = dcomp + it;
      t.cond = 0;
      t.cap = r;
      if (add > 0) {
        t.P = dP + (size_t)it * m * add;
        t.Q = dQ + (size_t)it * n * add;
        t.ldp = m;
        t.ldq = n;
        t.pr = m;
        t.qr = n;
        t.addv = add;
      }
      t.alpha = -1.0;
      t.rcap = r;
      t.ws = ws + wsd * it;
    }
    TruncItem* ditems;
    HMGP_CUDA(cudaMalloc(&ditems, count * sizeof(TruncItem)));
    HMGP_CUDA(cudaMemcpy(ditems, items.data(), count * sizeof(TruncItem), cudaMemcpyHostToDevice));
    cudaStream_t st;
    HMGP_CUDA(cudaStreamCreate(&st));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sw = 0, smn = 0;
    trunc_smem_dims(m, n, &sw, &smn);
    if (getenv("HMGP_STATS")) truncate_hist_enable(true);
    int* ddfr = nullptr;
    HMGP_CUDA(cudaMalloc(&ddfr, (size_t)count * 4));
    double best = 1e30;
    for (int rep = 0; rep < reps; ++rep) {
      HMGP_CUDA(cudaMemcpyAsync(dU, dU0, U.size() * 8, cudaMemcpyDeviceToDevice, st));
      HMGP_CUDA(cudaMemcpyAsync(dV, dV0, V.size() * 8, cudaMemcpyDeviceToDevice, st));
      HMGP_CUDA(cudaMemcpyAsync(drank, rk.data(), count * 4, cudaMemcpyHostToDevice, st));
      HMGP_CUDA(cudaMemsetAsync(derr, 0, 4, st));
      cudaEventRecord(e0, st);
      if (route == 2)
        launch_truncate_cluster(ditems, doff, count, eps, derr, st, trunc_cluster_resident(m, n));
      else if (route == 1 || route == 3)
        launch_truncate_pair(ditems, doff, count, eps, derr, st, route == 3 ? ddfr : nullptr);
      else
        launch_truncate(ditems, count, eps, derr, st, sw, smn);
      cudaEventRecord(e1, st);
      HMGP_CUDA(cudaStreamSynchronize(st));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 || reps == 1) best = std::min(best, (double)ms);
    }
    int err = 0;
    HMGP_CUDA(cudaMemcpy(&err, derr, 4, cudaMemcpyDeviceToHost));
    std::vector<int> kr(count);
    HMGP_CUDA(cudaMemcpy(kr.data(), drank, count * 4, cudaMemcpyDeviceToHost));
    if (getenv("HMGP_STATS")) truncate_hist_print();
    *ms_out = best;
    *keep_out = kr[0];
    cudaFree(dU);
    cudaFree(dV);
    cudaFree(dU0);
    cudaFree(dV0);
    cudaFree(dP);
    cudaFree(dQ);
    cudaFree(ws);
    cudaFree(ddfr);
    cudaFree(drank);
    cudaFree(dcomp);
    cudaFree(derr);
    cudaFree(doff);
    cudaFree(ditems);
    cudaStreamDestroy(st);
    return err ? 100 + err : 0;
  } catch (const std::exception& e) {
    fprintf(stderr, "trunc_bench: %s\n", e.what());
    return 1;
  }
}
