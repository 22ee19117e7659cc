// θ-sweep and kriging shards over the GPUs of one box: the C-ABI
// entry points a C++ caller uses — no Python, no torch.
//
//   hmgp_loglik_sweep   one rank's share of a θ list on its GPU (host z, uploaded once)
//   hmgp_sweep_shard    which θ a rank evaluates (ν-major round-robin)
//   hmgp_predict_range  which new locations a rank predicts (contiguous)
//   hmgp_comm_*         NCCL communicator plumbing (ncclGetUniqueId / ncclCommInitRank)
//   hmgp_sweep_gather   ONE ncclAllGather of the per-θ {L, logdet, quad, status} rows
//   hmgp_predict_gather ONE ncclAllGather of the prediction slices
//
// The path has no data-path collective: every rank builds the θ-independent
// geometry itself, evaluates independent L(θ) (the reference's probes are
// independent, mle.cpp:152-158; evaluate_loglik is reentrant) and
// only the results are gathered.  NCCL is resolved at first use with
// dlopen("libnccl.so.2") so that single-GPU users need no NCCL at all.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "hmgp_api.h"

int hmgp_fail(int code, const char* msg);

#define SWEEP_GUARD(...)                                    \
  try {                                                     \
    __VA_ARGS__;                                            \
    return HMGP_OK;                                         \
  } catch (const hmgp_gpu::Error& e) {                      \
    return hmgp_fail(e.code, e.what());                     \
  } catch (const std::invalid_argument& e) {                \
    return hmgp_fail(HMGP_EINVAL, e.what());                \
  } catch (const std::exception& e) {                       \
    return hmgp_fail(HMGP_ECUDA, e.what());                 \
  }

using namespace hmgp_gpu;

namespace {
template <class T>
struct DBuf {
  T* p = nullptr;
  explicit DBuf(size_t n) { p = hmgp_gpu::dev_alloc_n<T>(n); }
  ~DBuf() { hmgp_gpu::dev_free(p); }
};
struct Id128 {  // ncclUniqueId (passed by value)
  char b[128];
};
// the five NCCL entry points this file needs, bound at first use
struct Nccl {
  void* lib = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, Id128, int) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
Nccl& nccl() {
  static Nccl n;
  if (n.lib) return n;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    n.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (n.lib) break;
  }
  if (!n.lib) throw std::runtime_error("NCCL not found (dlopen libnccl.so.2)");
  auto sym = [&](const char* s) {
    void* p = dlsym(n.lib, s);
    if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + s);
    return p;
  };
  n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
  n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
  n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
  n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  return n;
}
void nccl_check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(rc));
}
constexpr int kNcclChar = 0;  // ncclInt8 / ncclChar
}  // namespace

struct hmgp_comm {
  void* comm = nullptr;  // ncclComm_t
  int rank = 0, world = 1;
};

extern "C" {

int hmgp_loglik_sweep(hmgp_ctx* ctx, hmgp_geom* g, const double* z, const hmgp_matern* thetas,
                      int ntheta, const hmgp_config* cfg, hmgp_loglik_result* res) {
  if (ntheta <= 0) return HMGP_OK;
  double* dz = nullptr;
  int rc = HMGP_OK;
  try {
    HMGP_CUDA(cudaSetDevice(ctx->device));
    const int n = g->g.n;
    HMGP_CUDA(cudaMalloc(&dz, 8ull * n));
    HMGP_CUDA(cudaMemcpyAsync(dz, z, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    rc = hmgp_loglik_batch(ctx, g, dz, thetas, ntheta, cfg, res);
  } catch (const std::exception& e) {
    rc = hmgp_fail(HMGP_ECUDA, e.what());
  }
  if (dz) cudaFree(dz);
  return rc;
}

int hmgp_sweep_shard(const hmgp_matern* thetas, int ntheta, int rank, int world, int32_t* idx,
                     int* count) {
  SWEEP_GUARD({
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("sweep_shard: bad rank / world");
    std::vector<int> order(std::max(ntheta, 0));
    std::iota(order.begin(), order.end(), 0);
    // ν-major (stable), so the much cheaper closed-form ν points spread evenly
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return thetas[a].nu < thetas[b].nu; });
    std::vector<int32_t> mine;
    for (int k = rank; k < ntheta; k += world) mine.push_back(order[k]);
    std::sort(mine.begin(), mine.end());
    if (idx) std::copy(mine.begin(), mine.end(), idx);
    *count = (int)mine.size();
  })
}

int hmgp_predict_range(int m, int rank, int world, int* begin, int* end) {
  SWEEP_GUARD({
    if (world < 1 || rank < 0 || rank >= world || m < 0) throw std::invalid_argument("predict_range: bad arguments");
    *begin = (int)(((long long)m * rank) / world);
    *end = (int)(((long long)m * (rank + 1)) / world);
  })
}

int hmgp_comm_unique_id(void* id128) {
  SWEEP_GUARD({ nccl_check(nccl().GetUniqueId(id128), "ncclGetUniqueId"); })
}

int hmgp_comm_create(hmgp_ctx* ctx, const void* id128, int rank, int world, hmgp_comm** out) {
  SWEEP_GUARD({
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm_create: bad rank / world");
    HMGP_CUDA(cudaSetDevice(ctx->device));
    auto c = new hmgp_comm();
    c->rank = rank;
    c->world = world;
    if (world > 1) {
      Id128 id;
      std::memcpy(id.b, id128, 128);
      const int rc = nccl().CommInitRank(&c->comm, world, id, rank);
      if (rc != 0) {
        delete c;
        nccl_check(rc, "ncclCommInitRank");
      }
    }
    *out = c;
  })
}

void hmgp_comm_destroy(hmgp_comm* c) {
  if (!c) return;
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
}

// Rows {index, loglik, logdet, quad_form, status} of fixed capacity per rank, one
// all-gather, then scattered into the θ-ordered table on every rank.
int hmgp_sweep_gather(hmgp_ctx* ctx, hmgp_comm* comm, const int32_t* idx, const hmgp_loglik_result* local,
                      int count, int ntheta, hmgp_loglik_result* table) {
  SWEEP_GUARD({
    const int world = comm ? comm->world : 1;
    for (int t = 0; t < ntheta; ++t) {
      table[t] = hmgp_loglik_result{std::numeric_limits<double>::quiet_NaN(), 0, 0, 0, 0, -2};
    }
    if (world == 1) {
      for (int k = 0; k < count; ++k) table[idx[k]] = local[k];
      return HMGP_OK;
    }
    HMGP_CUDA(cudaSetDevice(ctx->device));
    struct Row {
      int64_t idx;
      hmgp_loglik_result r;
    };
    const int cap = (ntheta + world - 1) / world + 1;
    if (count > cap) throw std::invalid_argument("sweep_gather: more local rows than the shard capacity");
    std::vector<Row> send(cap, Row{-1, {}}), recv((size_t)cap * world);
    for (int k = 0; k < count; ++k) send[k] = Row{idx[k], local[k]};
    DBuf<char> ds(sizeof(Row) * cap), dr(sizeof(Row) * cap * world);
    HMGP_CUDA(cudaMemcpyAsync(ds.p, send.data(), sizeof(Row) * cap, cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(nccl().AllGather(ds.p, dr.p, sizeof(Row) * cap, kNcclChar, comm->comm, ctx->stream), "ncclAllGather");
    HMGP_CUDA(cudaMemcpyAsync(recv.data(), dr.p, sizeof(Row) * cap * world, cudaMemcpyDeviceToHost, ctx->stream));
    HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (const Row& r : recv)
      if (r.idx >= 0 && r.idx < ntheta) table[r.idx] = r.r;
  })
}

int hmgp_predict_gather(hmgp_ctx* ctx, hmgp_comm* comm, const double* local, int m, double* out) {
  SWEEP_GUARD({
    const int world = comm ? comm->world : 1, rank = comm ? comm->rank : 0;
    int lo = 0, hi = m;
    hmgp_predict_range(m, rank, world, &lo, &hi);
    if (world == 1) {
      if (m > 0) std::memcpy(out, local, 8ull * m);
      return HMGP_OK;
    }
    if (m == 0) return HMGP_OK;  // empty input: no collective (every rank agrees on m)
    HMGP_CUDA(cudaSetDevice(ctx->device));
    const int cap = (m + world - 1) / world;
    std::vector<double> send(cap, 0.0), recv((size_t)cap * world);
    std::copy(local, local + (hi - lo), send.begin());
    DBuf<double> ds(cap), dr((size_t)cap * world);
    HMGP_CUDA(cudaMemcpyAsync(ds.p, send.data(), 8ull * cap, cudaMemcpyHostToDevice, ctx->stream));
    nccl_check(nccl().AllGather(ds.p, dr.p, 8ull * cap, kNcclChar, comm->comm, ctx->stream), "ncclAllGather");
    HMGP_CUDA(cudaMemcpyAsync(recv.data(), dr.p, 8ull * cap * world, cudaMemcpyDeviceToHost, ctx->stream));
    HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < world; ++r) {
      int b = 0, e = 0;
      hmgp_predict_range(m, r, world, &b, &e);
      std::copy(recv.begin() + (size_t)r * cap, recv.begin() + (size_t)r * cap + (e - b), out + b);
    }
  })
}

}  // extern "C"
