// Pipeline entry points of the C ABI: factorize / solves / L(θ) / θ-batch /
// predict, and K12 (the streamed kriging cross-covariance product).
//   evaluate_loglik  loglik.cpp:18-38      predict  krige.cpp:9-44
#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <mutex>
#include <condition_variable>
#include <functional>
#include <thread>
#include <climits>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "../../include/hmgp_cuda.h"
#include "common.cuh"
#include "factor.h"
#include "hmgp_api.h"

namespace hmgp_gpu {
extern void (*g_low_memory_hook)();  // alloc.cu: called before an allocation reports out-of-memory
}
using namespace hmgp_gpu;

hmgp_factor::~hmgp_factor() = default;

namespace {
template <class T>
struct DBuf {
  T* p = nullptr;
  explicit DBuf(size_t n) { p = hmgp_gpu::dev_alloc_n<T>(n); }
  ~DBuf() { hmgp_gpu::dev_free(p); }
};

}  // namespace
namespace hmgp_gpu {
thread_local size_t t_arena_bytes = 0;
}
namespace {

size_t arena_bytes_for(const HMat& h) {
  if (t_arena_bytes) return t_arena_bytes;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  // room for the factor copy of the payload + solve work, keep 2 GiB spare
  const size_t need = h.pool_doubles * 8 + ((size_t)2 << 30);
  const size_t avail = fr > need + ((size_t)1 << 30) ? fr - need : ((size_t)1 << 30);
  // the task-flow factorization splits the arena into 4 rotating sub-arenas
  const size_t want = std::max<size_t>((size_t)112 << 30, h.pool_doubles * 8 * 3);
  return std::min(avail, want);
}

double factor_eps(const hmgp_config* c) {  // pipeline.hpp:21-24
  if (c->eps_factor > 0.0) return c->eps_factor;
  return c->rank.mode == 0 ? c->rank.eps : 1e-6;
}

// run factorize and translate a failing pivot into FactorError semantics
std::unique_ptr<Factor> do_factorize(HMat& h, double eps_f, bool ldl, cudaStream_t st) {
  if (!(eps_f > 0.0)) throw std::invalid_argument("factorize: eps_f must be positive");
  auto f = std::make_unique<Factor>();
  try {
    factorize(*f, h, eps_f, ldl, st, arena_bytes_for(h));
  } catch (const Error& e) {
    // the temporaries did not fit in what the parked θ-batch workers left free:
    // take their workspaces back and run once more with the full arena
    if (e.code != HMGP_ECAPACITY || !hmgp_gpu::g_low_memory_hook) throw;
    hmgp_gpu::g_low_memory_hook();
    release_thread_workspace();
    dev_pool_trim();
    const bool ok = t_graph_ok;
    f = std::make_unique<Factor>();
    t_graph_ok = ok;
    factorize(*f, h, eps_f, ldl, st, arena_bytes_for(h));
  }
  if (f->fail_pos != INT_MAX) {
    hmgp_set_pivot(h.g->perm[f->fail_pos], f->fail_val);
    throw Error(HMGP_ENOTSPD, "matrix not numerically SPD; increase nugget tau2");
  }
  return f;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct GraphOkScope {
  GraphOkScope() { t_graph_ok = true; }
  ~GraphOkScope() { t_graph_ok = false; }
};

// Persistent θ-batch workers: host threads that outlive one hmgp_loglik_batch
// call, each with its own stream, temporary arena and captured factorization
// (factor.cu), so that the next batch on the same block structure replays the
// workers' CUDA graphs instead of walking the recursion again.
static thread_local bool t_pool_worker = false;
static thread_local bool t_in_batch = false;  // this thread holds BatchPool::batch_mu_
void pool_low_memory();

class BatchPool {
 public:
  static BatchPool& get() {
    // never destroyed: its workers stay parked on the condition variable until the
    // process ends, and destroying a condition variable with waiters blocks exit
    static BatchPool* p = new BatchPool();
    return *p;
  }
  // run job(ctx) on workers [0, T) and wait for all of them
  void run(int T, int device, const std::function<void(hmgp_ctx*)>& job) {
    std::unique_lock<std::mutex> lk(mu_);
    while ((int)ws_.size() < T) {
      ws_.emplace_back(new Worker());
      Worker* w = ws_.back().get();
      w->th = std::thread([this, w, device] { loop(w, device); });
      w->th.detach();  // parked for the life of the process
    }
    pending_ = T;
    for (int i = 0; i < T; ++i) {
      ws_[i]->job = job;
      ws_[i]->has_job = true;
    }
    cv_.notify_all();
    done_.wait(lk, [&] { return pending_ == 0; });
  }
  bool busy() const { return pending_ > 0; }
  // every worker frees its arena, graph and stream-ordered buffers
  void release() {
    if (ws_.empty()) return;
    const int T = (int)ws_.size();
    run(T, -1, [](hmgp_ctx*) { release_thread_workspace(); });
    key_ = 0;
    share_ = 0;
    per_ = 0;
    warm_ = 0;
  }
  int size() const { return (int)ws_.size(); }
  uint64_t key_ = 0;   // structure the workers' workspaces were sized for
  size_t share_ = 0;   // arena bytes per worker
  size_t per_ = 0;     // device bytes per worker (arena + payloads)
  int warm_ = 0;       // workers holding a workspace
  std::mutex batch_mu_;

 private:
  struct Worker {
    std::thread th;
    std::function<void(hmgp_ctx*)> job;
    bool has_job = false;
    hmgp_ctx ctx;
  };
  void loop(Worker* w, int device) {
    t_pool_worker = true;
    if (device >= 0) cudaSetDevice(device);
    w->ctx.device = device;
    cudaStreamCreateWithFlags(&w->ctx.stream, cudaStreamNonBlocking);
    for (;;) {
      std::function<void(hmgp_ctx*)> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return w->has_job || stop_; });
        if (stop_) return;
        job = w->job;
        w->has_job = false;
      }
      job(&w->ctx);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  ~BatchPool() = delete;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::vector<std::unique_ptr<Worker>> ws_;
  int pending_ = 0;
  bool stop_ = false;
};

// L(θ) on a built geometry with device z (original order)
void loglik_on_geom(hmgp_ctx* ctx, Geometry& g, const double* d_z, const hmgp_matern* th,
                    const hmgp_config* cfg, hmgp_loglik_result* res) {
  hmgp_validate_matern(th);
  if (cfg->rank.mode == 0 && !(cfg->rank.eps > 0.0))
    throw std::invalid_argument("assemble: eps must be positive");
  AllocScope as(ctx->stream);  // per-evaluation buffers: stream-ordered (declared before h, f)
  HMat h;
  assemble(h, g, make_matern(th->sigma2, th->ell, th->nu, th->tau2), cfg->rank.eps,
           cfg->rank.mode == 1, cfg->rank.rank, cfg->rank.max_rank > 0 ? cfg->rank.max_rank : 256,
           ctx->stream, nullptr);
  std::unique_ptr<Factor> f;
  {
    GraphOkScope ephemeral;  // f dies before this thread factorizes again
    f = do_factorize(h, factor_eps(cfg), cfg->form == 1, ctx->stream);
  }
  const int n = g.n;
  res->n = n;
  res->logdet = factor_log_det(*f, ctx->stream);
  phase_mark(PH_LOGDET);
  res->quad_form = factor_quad_form_dev(*f, d_z, ctx->stream);
  phase_mark(PH_FWD);
  res->loglik = -0.5 * n * std::log(2.0 * M_PI) - 0.5 * res->logdet - 0.5 * res->quad_form;
  res->status = f->clamped > 0 ? 1 : 0;
}
}  // namespace

#define API_GUARD2(...)                                     \
  try {                                                     \
    __VA_ARGS__;                                            \
    return HMGP_OK;                                         \
  } catch (const hmgp_gpu::Error& e) {                      \
    return hmgp_fail(e.code, e.what());                     \
  } catch (const std::invalid_argument& e) {                \
    return hmgp_fail(HMGP_EINVAL, e.what());                \
  } catch (const std::domain_error& e) {                    \
    return hmgp_fail(HMGP_EDOMAIN, e.what());               \
  } catch (const std::out_of_range& e) {                    \
    return hmgp_fail(HMGP_ERANGE, e.what());                \
  } catch (const std::exception& e) {                       \
    return hmgp_fail(HMGP_ECUDA, e.what());                 \
  }

int hmgp_fail(int code, const char* msg);

namespace hmgp_gpu {
// ------------------------------------------------------------------- K12 --
// Each CTA: 256 test points (one per thread) x one slice of the training set,
// training points streamed through shared memory in tiles of 512 (coordinates
// + weights); partial sums per slice, reduced in a fixed order afterwards.
constexpr int kCrossTile = 512;

__global__ void __launch_bounds__(256) k_cross_apply(const double* __restrict__ train, int n, int dim,
                                                     const double* __restrict__ w,
                                                     const double* __restrict__ test, int m,
                                                     MaternDev p, int slice, double* __restrict__ part) {
  __shared__ double sx[kCrossTile], sy[kCrossTile], sz[kCrossTile], sw[kCrossTile];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.y * slice, j1 = min(n, j0 + slice);
  double tx = 0, ty = 0, tz = 0;
  if (i < m) {
    tx = test[(size_t)i * dim];
    ty = test[(size_t)i * dim + 1];
    if (dim == 3) tz = test[(size_t)i * dim + 2];
  }
  double acc = 0.0;
  for (int b = j0; b < j1; b += kCrossTile) {
    const int cnt = min(kCrossTile, j1 - b);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      sx[t] = train[(size_t)(b + t) * dim];
      sy[t] = train[(size_t)(b + t) * dim + 1];
      sz[t] = dim == 3 ? train[(size_t)(b + t) * dim + 2] : 0.0;
      sw[t] = w[b + t];
    }
    __syncthreads();
    if (i < m)
      for (int t = 0; t < cnt; ++t) {
        const double h = dim == 2 ? dist2d(tx, ty, sx[t], sy[t]) : dist3d(tx, ty, tz, sx[t], sy[t], sz[t]);
        acc += matern_at(p, h) * sw[t];
      }
  }
  if (i < m) part[(size_t)blockIdx.y * m + i] = acc;
}

__global__ void k_cross_reduce(const double* __restrict__ part, int m, int slices,
                               double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int q = 0; q < slices; ++q) s += part[(size_t)q * m + i];
  out[i] = s;
}

void cross_apply(cudaStream_t st, const double* d_train, int n, int dim, const double* d_w,
                 const double* d_test, int m, const MaternDev& p, double* d_out) {
  NvtxRange nvtx_range("hmgp:cross_apply(K12)");
  if (m <= 0) return;
  const int bx = (m + 255) / 256;
  int slices = std::max(1, (kSMs * 4 + bx - 1) / bx);
  slices = std::min(slices, std::max(1, n / kCrossTile));
  const int slice = (n + slices - 1) / slices;
  DBuf<double> part((size_t)slices * m);
  k_cross_apply<<<dim3(bx, slices), 256, 0, st>>>(d_train, n, dim, d_w, d_test, m, p, slice, part.p);
  HMGP_LAUNCH_CHECK();
  k_cross_reduce<<<bx, 256, 0, st>>>(part.p, m, slices, d_out);
  HMGP_LAUNCH_CHECK();
  HMGP_CUDA(cudaStreamSynchronize(st));
}
}  // namespace hmgp_gpu

extern "C" {

int hmgp_factorize(hmgp_ctx* ctx, hmgp_hmat* h, double eps_f, int form, hmgp_factor** out,
                   hmgp_factor_info* info) {
  API_GUARD2({
    if (h->h.partial()) throw std::invalid_argument("factorize: H-matrix is a leaf-range shard");
    if (!h->symmetric) throw std::invalid_argument("factorize: requires a symmetric H-matrix");  // hfactor.cpp:333-334
    HMGP_CUDA(cudaSetDevice(ctx->device));
    auto f = do_factorize(h->h, eps_f, form == 1, ctx->stream);
    if (info) {
      info->eps = eps_f;
      info->clamped = f->clamped;
      info->negative = f->negative;
      info->min_pivot = f->min_pivot;
      info->storage_bytes = factor_storage_bytes(*f);
    }
    auto r = new hmgp_factor();
    r->owned_geom = h->owned_geom;
    r->f = std::move(f);
    *out = r;
  })
}

int hmgp_log_det(hmgp_ctx* ctx, const hmgp_factor* f, double* out) {
  API_GUARD2({ *out = factor_log_det(*f->f, ctx->stream); })
}

int hmgp_quad_form(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* out) {
  API_GUARD2({
    const int n = f->f->g->n;
    DBuf<double> db(n);
    HMGP_CUDA(cudaMemcpyAsync(db.p, b, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    *out = factor_quad_form_dev(*f->f, db.p, ctx->stream);
  })
}

static int solve_common(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* x, bool full) {
  API_GUARD2({
    const int n = f->f->g->n;
    DBuf<double> db(n), dx(n);
    HMGP_CUDA(cudaMemcpyAsync(db.p, b, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    factor_solve_dev(*f->f, db.p, dx.p, full, ctx->stream);
    HMGP_CUDA(cudaMemcpyAsync(x, dx.p, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
    HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
  })
}
int hmgp_solve_factored(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* x) {
  return solve_common(ctx, f, b, x, true);
}
int hmgp_solve_lower(hmgp_ctx* ctx, const hmgp_factor* f, const double* b, double* x) {
  return solve_common(ctx, f, b, x, false);
}

int hmgp_factor_diagonal(hmgp_ctx* ctx, const hmgp_factor* f, double* out) {
  API_GUARD2({
    const Factor& F = *f->f;
    const int n = F.g->n;
    std::vector<double> d(n);
    HMGP_CUDA(cudaMemcpyAsync(d.data(), F.d_d, 8ull * n, cudaMemcpyDeviceToHost, ctx->stream));
    HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < n; ++k) out[F.g->perm[k]] = d[k];
  })
}

int hmgp_hmat_to_dense(hmgp_ctx* ctx, const hmgp_hmat* h, double* out) {
  API_GUARD2({
    if (h->h.partial()) throw std::invalid_argument("to_dense: H-matrix is a leaf-range shard");
    HMGP_CUDA(cudaSetDevice(ctx->device));
    hmat_to_dense(ctx->stream, h->h, out);
  })
}

int hmgp_factor_lower_dense(hmgp_ctx* ctx, const hmgp_factor* f, double* out) {
  API_GUARD2({
    HMGP_CUDA(cudaSetDevice(ctx->device));
    factor_lower_dense(ctx->stream, *f->f, out);
  })
}

int hmgp_factor_reconstruct(hmgp_ctx* ctx, const hmgp_factor* f, double* out) {
  API_GUARD2({
    HMGP_CUDA(cudaSetDevice(ctx->device));
    factor_reconstruct(ctx->stream, *f->f, out);
  })
}

void hmgp_factor_destroy(hmgp_factor* f) { delete f; }

int hmgp_loglik(hmgp_ctx* ctx, const double* coords, int n, int dim, const double* z,
                const hmgp_matern* theta, const hmgp_config* cfg, hmgp_loglik_result* res) {
  API_GUARD2({
    hmgp_validate_matern(theta);  // loglik.cpp:20-23
    if (n < 1) throw std::invalid_argument("evaluate_loglik: empty dataset");
    HMGP_CUDA(cudaSetDevice(ctx->device));
    const double t0 = now();
    PhaseScope ps(ctx);
    hmgp_geom* g = nullptr;
    const int rc = hmgp_geometry_build(ctx, coords, n, dim, cfg->leaf_size, cfg->eta, &g);
    if (rc != HMGP_OK) return rc;
    std::unique_ptr<hmgp_geom, void (*)(hmgp_geom*)> guard(g, hmgp_geometry_destroy);
    DBuf<double> dz(n);
    HMGP_CUDA(cudaMemcpyAsync(dz.p, z, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    phase_mark(PH_GEOMETRY);
    loglik_on_geom(ctx, g->g, dz.p, theta, cfg, res);
    ps.finish();
    res->seconds = now() - t0;
  })
}

int hmgp_loglik_geom(hmgp_ctx* ctx, hmgp_geom* g, const double* d_z, const hmgp_matern* theta,
                     const hmgp_config* cfg, hmgp_loglik_result* res) {
  API_GUARD2({
    HMGP_CUDA(cudaSetDevice(ctx->device));
    const double t0 = now();
    PhaseScope ps(ctx);
    loglik_on_geom(ctx, g->g, d_z, theta, cfg, res);
    ps.finish();
    res->seconds = now() - t0;
  })
}

// Independent θ run concurrently (evaluate_loglik is reentrant):
// the first θ alone on the caller's stream (it sizes the device workspace), the
// rest on up to HMGP_BATCH_THREADS (default 8) host workers, each with its own
// stream and arena, pulling θ indices from a shared counter.  One L(θ) is a
// chain of latency-bound launches that keeps only part of the GPU busy, so
// concurrent θ fill the idle SMs.
int hmgp_loglik_batch(hmgp_ctx* ctx, hmgp_geom* g, const double* d_z, const hmgp_matern* thetas,
                      int ntheta, const hmgp_config* cfg, hmgp_loglik_result* res) {
  API_GUARD2({
    HMGP_CUDA(cudaSetDevice(ctx->device));
    // θ whose worker ran out of device workspace: re-run on the caller thread
    // with the full workspace afterwards (never scored -inf for lack of memory)
    std::mutex retry_mu;
    std::vector<int> retry;
    auto one = [&](hmgp_ctx* c, int t) {
      const double t0 = now();
      try {  // fit() maps numerical failures to -inf (mle.cpp:152-158)
        loglik_on_geom(c, g->g, d_z, &thetas[t], cfg, &res[t]);
      } catch (const hmgp_gpu::Error& e) {
        if (e.code == HMGP_ECAPACITY && c != ctx) {
          std::lock_guard<std::mutex> lk(retry_mu);
          retry.push_back(t);
          return;
        }
        if (e.code != HMGP_ENOTSPD) throw;
        res[t] = hmgp_loglik_result{-std::numeric_limits<double>::infinity(), 0, 0, g->g.n, 0, -1};
      } catch (const std::domain_error&) {
        res[t] = hmgp_loglik_result{-std::numeric_limits<double>::infinity(), 0, 0, g->g.n, 0, -1};
      }
      res[t].seconds = now() - t0;
    };
    if (ntheta <= 0) return HMGP_OK;
    BatchPool& pool = BatchPool::get();
    std::lock_guard<std::mutex> one_batch(pool.batch_mu_);  // batches of different callers take turns
    struct InBatch {
      InBatch() { t_in_batch = true; }
      ~InBatch() { t_in_batch = false; }
    } in_batch;
    hmgp_gpu::g_low_memory_hook = pool_low_memory;
    // structure of this batch (workers keep workspaces sized for one structure)
    const uint64_t bkey = ((uint64_t)g->g.n << 32) ^ ((uint64_t)g->g.nbeg.size() << 8) ^ (uint64_t)cfg->leaf_size ^
                          ((uint64_t)(cfg->form == 1) << 7);
    if (pool.key_ != 0 && pool.key_ != bkey) {
      pool.release();
      dev_pool_trim();
    }
    int T = 16;
    if (const char* e = getenv("HMGP_BATCH_THREADS")) T = std::max(1, atoi(e));
    // workers that already hold a workspace for this structure take the whole
    // batch; otherwise the first θ runs alone on the caller's stream and sizes it
    const bool warm_start = pool.key_ == bkey && pool.warm_ > 0 && ntheta > 1 && T > 1;
    int first = 0;
    size_t share = pool.share_, per = pool.per_;
    if (!warm_start) {
      one(ctx, 0);
      first = 1;
      T = std::min(T, ntheta - 1);
      if (T <= 1) {
        for (int t = 1; t < ntheta; ++t) one(ctx, t);
        return HMGP_OK;
      }
      // per worker: the first θ's arena peak with headroom, plus the H-matrix and
      // factor payloads
      // (a first θ that failed before its factorization leaves no peak: assume 8 GiB)
      const size_t peak = t_last_arena_peak ? t_last_arena_peak : ((size_t)8 << 30);
      const size_t pl = t_last_pool_bytes;
      HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
      // (the temporaries are sized by the structure and the capacities, not by θ:
      // a small margin suffices, and a worker that still runs out hands its θ
      // back to the caller's full workspace)
      share = peak + peak / 6 + ((size_t)256 << 20);
      // H-matrix payload, factor pool (captured: +25 % capacities), descriptor store
      per = share + pl * 4 + ((size_t)768 << 20);
      if (pool.key_ == bkey && pool.share_ < share) {  // workspaces too small for this batch
        pool.release();
        pool.warm_ = 0;
        dev_pool_trim();
      }
    } else {
      T = std::min(T, ntheta);
    }
    size_t fr = 0, tot = 0;
    HMGP_CUDA(cudaMemGetInfo(&fr, &tot));
    const size_t reserve = (size_t)6 << 30;
    // the caller's own arena is only needed again for the retries: release it if
    // the workers would otherwise not fit
    const int warm = pool.key_ == bkey ? pool.warm_ : 0;
    auto fit_T = [&](size_t free_now) {
      const size_t usable = free_now > reserve ? free_now - reserve : 0;
      return (int)std::max<size_t>(1, std::min<size_t>(T, warm + usable / per));
    };
    if (fit_T(fr) < T) {
      release_thread_workspace();
      dev_pool_trim();
      HMGP_CUDA(cudaMemGetInfo(&fr, &tot));
    }
    T = fit_T(fr);
    pool.key_ = bkey;
    pool.share_ = std::max(pool.share_, share);
    pool.per_ = std::max(pool.per_, per);
    const size_t wshare = pool.share_;
    pool.warm_ = std::max(warm, T);
    std::atomic<int> next{first};
    std::vector<std::exception_ptr> errs(T);
    std::atomic<int> widx{0};
    pool.run(T, ctx->device, [&](hmgp_ctx* c) {
      const int w = widx.fetch_add(1);
      try {
        HMGP_CUDA(cudaSetDevice(ctx->device));
        t_arena_bytes = wshare;
        t_one_stream = getenv("HMGP_BATCH_SECTIONS") == nullptr;
        for (int t; (t = next.fetch_add(1)) < ntheta;) one(c, t);
        HMGP_CUDA(cudaStreamSynchronize(c->stream));
      } catch (...) {
        errs[w] = std::current_exception();
      }
    });
    // keep the workers' workspaces (arena + captured factorization) for the next
    // batch on this structure while they are small next to the device memory;
    // large ones (C3: ~30 GB per worker) go back right away
    {
      // kept by default: an allocation that would otherwise fail takes them back
      // (g_low_memory_hook), so holding them costs later calls nothing but a retry
      bool keep = true;
      if (const char* e = getenv("HMGP_BATCH_KEEP")) keep = atoi(e) != 0;
      if (!keep) {
        pool.release();
        pool.warm_ = 0;
        dev_pool_trim();
      }
    }
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    std::sort(retry.begin(), retry.end());
    if (!retry.empty()) dev_pool_trim();
    for (int t : retry) one(ctx, t);  // caller thread, full workspace (arena_bytes_for)
  })
}

// out-of-memory on some thread: idle workers give their workspaces back (never
// from a worker itself, and never while a batch is running — then the failing
// θ is retried on the caller thread instead)
}  // extern "C"
namespace {
void pool_low_memory() {
  if (t_pool_worker || t_in_batch) return;
  BatchPool& pool = BatchPool::get();
  if (!pool.batch_mu_.try_lock()) return;
  std::lock_guard<std::mutex> lk(pool.batch_mu_, std::adopt_lock);
  if (pool.busy()) return;
  pool.release();
}
}  // namespace
extern "C" {

void hmgp_release_workspace(void) {
  try {
    std::lock_guard<std::mutex> one_batch(BatchPool::get().batch_mu_);
    t_in_batch = true;
    BatchPool::get().release();
    t_in_batch = false;
    release_thread_workspace();
    dev_pool_trim();
  } catch (...) {
  }
}

int hmgp_predict(hmgp_ctx* ctx, const double* train, int n, int dim, const double* z1,
                 const double* test, int m, const hmgp_matern* theta, const hmgp_config* cfg,
                 double* out, double* seconds) {
  API_GUARD2({
    hmgp_validate_matern(theta);  // krige.cpp:12-15
    if (n < 1) throw std::invalid_argument("predict: empty training set");
    const double t0 = now();
    if (m == 0) {
      if (seconds) *seconds = now() - t0;
      return HMGP_OK;
    }
    HMGP_CUDA(cudaSetDevice(ctx->device));
    PhaseScope ps(ctx);
    hmgp_geom* g = nullptr;
    const int rc = hmgp_geometry_build(ctx, train, n, dim, cfg->leaf_size, cfg->eta, &g);
    if (rc != HMGP_OK) return rc;
    std::unique_ptr<hmgp_geom, void (*)(hmgp_geom*)> guard(g, hmgp_geometry_destroy);
    phase_mark(PH_GEOMETRY);
    HMat h;
    assemble(h, g->g, make_matern(theta->sigma2, theta->ell, theta->nu, theta->tau2), cfg->rank.eps,
             cfg->rank.mode == 1, cfg->rank.rank, cfg->rank.max_rank > 0 ? cfg->rank.max_rank : 256,
             ctx->stream, nullptr);
    std::unique_ptr<Factor> f;
    {
      GraphOkScope ephemeral;
      f = do_factorize(h, factor_eps(cfg), cfg->form == 1, ctx->stream);
    }
    DBuf<double> dz(n), dw(n), dtest((size_t)m * dim), dout(m);
    // The new locations are visited in Morton order: the 32 lanes of a warp then hold
    // neighbouring points, whose distances to one training point — hence the Bessel
    // branch (Temme / Steed) and iteration counts of the general-ν path — are close,
    // instead of diverging lane by lane.  Each prediction's own sum is unchanged
    // (same training order), so the values are bit-identical to the unsorted pass.
    std::vector<int> order(m);
    std::vector<double> tsorted((size_t)m * dim), osorted(m);
    {
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int k = 0; k < m; ++k)
        for (int d = 0; d < dim; ++d) {
          lo[d] = std::min(lo[d], test[(size_t)k * dim + d]);
          hi[d] = std::max(hi[d], test[(size_t)k * dim + d]);
        }
      std::vector<uint64_t> key(m);
      for (int k = 0; k < m; ++k) {
        uint64_t code = 0;
        for (int d = 0; d < dim; ++d) {
          const double span = hi[d] > lo[d] ? hi[d] - lo[d] : 1.0;
          uint64_t q = (uint64_t)std::min(65535.0, std::max(0.0, (test[(size_t)k * dim + d] - lo[d]) / span * 65535.0));
          for (int b = 0; b < 16; ++b) code |= ((q >> b) & 1ull) << (b * dim + d);
        }
        key[k] = code;
        order[k] = k;
      }
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key[a] < key[b]; });
      for (int k = 0; k < m; ++k)
        for (int d = 0; d < dim; ++d) tsorted[(size_t)k * dim + d] = test[(size_t)order[k] * dim + d];
    }
    HMGP_CUDA(cudaMemcpyAsync(dz.p, z1, 8ull * n, cudaMemcpyHostToDevice, ctx->stream));
    HMGP_CUDA(cudaMemcpyAsync(dtest.p, tsorted.data(), 8ull * m * dim, cudaMemcpyHostToDevice, ctx->stream));
    factor_solve_dev(*f, dz.p, dw.p, true, ctx->stream);
    phase_mark(PH_BWD);
    cross_apply(ctx->stream, g->g.d_x, n, dim, dw.p, dtest.p, m,
                make_matern(theta->sigma2, theta->ell, theta->nu, theta->tau2), dout.p);
    phase_mark(PH_CROSS);
    HMGP_CUDA(cudaMemcpyAsync(osorted.data(), dout.p, 8ull * m, cudaMemcpyDeviceToHost, ctx->stream));
    HMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int k = 0; k < m; ++k) out[order[k]] = osorted[k];
    ps.finish();
    if (seconds) *seconds = now() - t0;
  })
}

int hmgp_cross_apply_device(hmgp_ctx* ctx, const double* d_train, int n, int dim, const double* d_w,
                            const double* d_test, int m, const hmgp_matern* theta, double* d_out) {
  API_GUARD2({
    hmgp_validate_matern(theta);
    HMGP_CUDA(cudaSetDevice(ctx->device));
    cross_apply(ctx->stream, d_train, n, dim, d_w, d_test, m,
                make_matern(theta->sigma2, theta->ell, theta->nu, theta->tau2), d_out);
  })
}

}  // extern "C"
