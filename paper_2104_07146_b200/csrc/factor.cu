// H-LDL^T / H-Cholesky on the GPU (hfactor.cpp:22-363), column-sweep H-solves,
// log-determinant and quadratic form (hfactor.cpp:365-403).
//
// Design.  The reference factorization is a deep recursion over the payload tree
// (factor_diag -> trsm_lower_t / sub_product -> product_low_rank / add_low_rank).
// Its loops over row children (trsm_lower_t's `for i`, sub_product's `for ii, jj`)
// touch disjoint targets, so the host walks the SAME recursion but with LISTS of
// independent items: every elementary operation (GEMM, TRSM, scaling, append /
// recompression, leaf factorization) becomes ONE batched kernel launch over all
// items that the reference would have executed one after the other.  Per-target
// operation order is unchanged, so each block sees exactly the reference's
// sequence of updates.  Ranks never leave the device: every kernel reads its
// low-rank widths from device ints and the watermark rules (hblock.cpp:200,
// hfactor.cpp:170) are evaluated inside the update kernel.  Temporaries come from
// a stream-ordered stack arena with structural capacity bounds.
#include <cooperative_groups.h>

#include <algorithm>
#include <functional>
#include <climits>
#include <cmath>
#include <cstring>
#include <array>
#include <chrono>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "dag.h"
#include "factor.h"
#include "hmgp_api.h"
#include "linalg.cuh"
#include "phases.h"

namespace hmgp_gpu {
namespace cg = cooperative_groups;


// ------------------------------------------------------------ utilities ---
extern thread_local bool t_one_stream;
constexpr int kSubArenaFull = 1007;  // internal: task-flow sub-arenas too small -> serial redo
constexpr int kArenaFull = 1008;     // internal: arena too small with side streams -> one-stream redo

struct Arena {
  char* base = nullptr;
  size_t cap = 0, top = 0, peak = 0, total = 0;
  // Task-flow mode: K sub-arenas (stacks); consecutive frames rotate over them so
  // that independent frames do not reuse each other's memory right away (reuse
  // is still safe: the task flow fences it).  Marks are kept on a stack.
  static constexpr int kMaxSub = 8;
  int K = 1, cur = 0;
  size_t sub_cap = 0;
  size_t tops[kMaxSub] = {};
  std::vector<std::array<size_t, kMaxSub + 1>> marks;
  Dag* dag = nullptr;  // set in task-flow mode: allocations are registered
  void init(size_t bytes, int k = 1) {  // persistent: reallocate only to grow
    top = peak = total = 0;
    hold = 0;
    K = std::max(1, std::min(k, kMaxSub));
    cur = 0;
    marks.clear();
    if (!(base && cap >= bytes)) {
      if (base) cudaFree(base);  // persistent (plain cudaMalloc)
      base = nullptr;
      cap = bytes;
      if (dev_malloc_plain((void**)&base, cap) != cudaSuccess) {
        // less free memory than planned (e.g. after a pool regrowth): take what
        // is there minus 1 GiB; device-detected overflow still reports cleanly
        cudaGetLastError();
        base = nullptr;
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        cap = fr > ((size_t)2 << 30) ? fr - ((size_t)1 << 30) : fr / 2;
        HMGP_CUDA(dev_malloc_plain((void**)&base, cap));
      }
    }
    sub_cap = (cap / K) & ~size_t(255);
    for (int i = 0; i < K; ++i) tops[i] = i * sub_cap;
  }
  int hold = 0;  // > 0 while a side-stream section is being enqueued: no reuse
  size_t mark() {
    if (K == 1) return top;
    std::array<size_t, kMaxSub + 1> m{};
    for (int i = 0; i < K; ++i) m[i] = tops[i];
    m[kMaxSub] = marks.size();
    marks.push_back(m);
    cur = (cur + 1) % K;
    return marks.size() - 1;
  }
  void release(size_t m) {
    if (hold) return;
    if (K == 1) {
      top = m;
      return;
    }
    for (int i = 0; i < K; ++i) tops[i] = marks[m][i];
    marks.resize(m);
  }
  void* raw(size_t bytes) {
    if (K == 1) {
      const size_t a = (top + 255) & ~size_t(255);
      if (a + bytes > cap) throw Error(kArenaFull, "factorize: device temporary arena exhausted");
      top = a + bytes;
      peak = std::max(peak, top);
      total += bytes;
      if (dag) dag->on_alloc((uintptr_t)(base + a), (uintptr_t)(base + a + bytes));
      return base + a;
    }
    for (int j = 0; j < K; ++j) {
      const int i = (cur + j) % K;
      const size_t a = (tops[i] + 255) & ~size_t(255);
      if (a + bytes > (i + 1) * sub_cap) continue;
      tops[i] = a + bytes;
      peak = std::max(peak, tops[i] - i * sub_cap);
      total += bytes;
      if (dag) dag->on_alloc((uintptr_t)(base + a), (uintptr_t)(base + a + bytes));
      return base + a;
    }
    throw Error(kSubArenaFull, "factorize: device temporary sub-arenas exhausted");
  }
  double* dbl(size_t n) { return static_cast<double*>(raw(std::max<size_t>(n, 1) * 8)); }
  int* ints(size_t n) { return static_cast<int*>(raw(std::max<size_t>(n, 1) * 4)); }
  void free_all() {
    if (base) cudaFree(base);
    base = nullptr;
    cap = 0;
  }
  ~Arena() { free_all(); }
};

// Descriptor storage of a captured factorization (CUDA graph): the item lists are
// uploaded once, on a stream of their own (outside the capture), into chunks that
// live as long as the graph; replays read them in place.
struct DescStore {
  struct Chunk {
    char* h = nullptr;
    char* d = nullptr;
    size_t cap = 0, used = 0;
  };
  std::vector<Chunk> chunks;
  size_t cur = 0;  // chunk being filled (chunks are kept and re-used by the next capture:
                   // cudaMalloc / cudaFree / cudaMallocHost synchronise the whole device,
                   // which stalls every other θ-batch worker)
  size_t off = 0, bytes = 0;
  cudaStream_t up = nullptr;
  static constexpr size_t kChunk = (size_t)32 << 20;
  void* put(const void* src, size_t n) {
    const size_t a = (n + 255) & ~size_t(255);
    while (cur < chunks.size() && off + a > chunks[cur].cap) {
      ++cur;
      off = 0;
      if (cur < chunks.size()) chunks[cur].used = 0;
    }
    if (cur >= chunks.size()) {
      Chunk c;
      c.cap = std::max(kChunk, a);
      if (cudaMallocHost(&c.h, c.cap) != cudaSuccess || dev_malloc_plain((void**)&c.d, c.cap) != cudaSuccess) {
        cudaGetLastError();
        if (c.h) cudaFreeHost(c.h);
        throw Error(6, "descriptor store: out of memory");  // the capture is abandoned (stream path)
      }
      chunks.push_back(c);
      cur = chunks.size() - 1;
      off = 0;
    }
    Chunk& c = chunks[cur];
    std::memcpy(c.h + off, src, n);  // uploaded chunk-wise by finish_upload()
    void* r = c.d + off;
    off += a;
    c.used = off;
    bytes += a;
    return r;
  }
  void finish_upload() {  // after the capture: one copy per chunk, then wait
    if (!up) HMGP_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    for (size_t k = 0; k <= cur && k < chunks.size(); ++k)
      if (chunks[k].used)
        HMGP_CUDA(cudaMemcpyAsync(chunks[k].d, chunks[k].h, chunks[k].used, cudaMemcpyHostToDevice, up));
    HMGP_CUDA(cudaStreamSynchronize(up));
  }
  void rewind() {  // the next capture overwrites the chunks in place
    if (up) cudaStreamSynchronize(up);
    cur = 0;
    off = bytes = 0;
    if (!chunks.empty()) chunks[0].used = 0;
  }
  void clear() {
    if (up) cudaStreamSynchronize(up);
    for (Chunk& c : chunks) {
      if (c.h) cudaFreeHost(c.h);
      if (c.d) cudaFree(c.d);
    }
    chunks.clear();
    cur = 0;
    off = bytes = 0;
  }
  ~DescStore() {
    clear();
    if (up) cudaStreamDestroy(up);
  }
};

// Pinned host ring -> device ring for item descriptors (stream ordered).
struct Stager {
  DescStore* store = nullptr;  // set while a factorization is being captured
  char* h = nullptr;
  char* d = nullptr;
  size_t cap = 0, off = 0;
  int wraps = 0;
  double wrap_ms = 0;
  cudaStream_t st = nullptr;          // stream of the next copy (the engine's current one)
  std::vector<cudaStream_t> used;     // streams that may still read the ring
  void use(cudaStream_t s) {
    st = s;
    if (store) return;
    if (std::find(used.begin(), used.end(), s) == used.end()) used.push_back(s);
  }
  void init(size_t bytes, cudaStream_t s) {  // persistent across factorizations
    st = s;
    used.assign(1, s);
    off = 0;
    wraps = 0;
    wrap_ms = 0;
    if (h) return;
    cap = bytes;
    // Descriptors are copied into a device ring (one cudaMemcpyAsync per batch).
    // HMGP_DESC_ZEROCOPY=1 lets the kernels read them in place from mapped pinned
    // host memory instead: measured on B200 (profiles/r2_exp_desc.txt) that is 6 %
    // slower for one C3 L(θ) (11.2 s vs 10.5 s) and no faster for concurrent θ, so
    // the copy-engine FIFO is not what limits θ-batch concurrency.
    zero_copy = getenv("HMGP_DESC_ZEROCOPY") != nullptr;
    HMGP_CUDA(cudaHostAlloc(&h, cap, cudaHostAllocMapped | cudaHostAllocPortable));
    if (zero_copy) {
      HMGP_CUDA(cudaHostGetDevicePointer((void**)&d, h, 0));
    } else {
      HMGP_CUDA(cudaMalloc(&d, cap));
    }
  }
  bool zero_copy = false;
  ~Stager() {
    if (d && !zero_copy) cudaFree(d);
    if (h) cudaFreeHost(h);
  }
  template <class T>
  const T* put(const std::vector<T>& v) {
    if (store) return static_cast<const T*>(store->put(v.data(), v.size() * sizeof(T)));
    const size_t bytes = (v.size() * sizeof(T) + 255) & ~size_t(255);
    if (bytes > cap) throw Error(6, "item batch exceeds staging ring");
    if (off + bytes > cap) {  // wrap: every stream that read the ring must be done
      const auto w0 = std::chrono::steady_clock::now();
      for (cudaStream_t s : used) HMGP_CUDA(cudaStreamSynchronize(s));
      wrap_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
      ++wraps;
      used.assign(1, st);
      off = 0;
    }
    std::memcpy(h + off, v.data(), v.size() * sizeof(T));
    if (!zero_copy)
      HMGP_CUDA(cudaMemcpyAsync(d + off, h + off, v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    const T* r = reinterpret_cast<const T*>(d + off);
    off += bytes;
    return r;
  }
};

// device matrix view: rows x cols (cols possibly on device; .cols.v = capacity)
struct MV {
  double* p = nullptr;
  int ld = 0, rows = 0;
  Dim cols{0, nullptr};
};
static MV rows_of(MV m, int r0, int cnt) {
  m.p += r0;
  m.rows = cnt;
  return m;
}
static MV cols_of(MV m, int c0, int cnt) {  // structural columns only
  m.p += (size_t)c0 * m.ld;
  m.cols = dimv(cnt);
  return m;
}

// ----------------------------------------------------------- the engine ---
// Per host thread (evaluate_loglik is reentrant): device
// temporaries reused by every factorization of the thread (grows), and the
// item-descriptor ring.
// per host thread: side streams / events of the in-order schedule (destroyed
// with the thread, so θ-batch workers do not leak them)
struct SidePool {
  static constexpr int kSide = 7, kPool = 12;
  cudaStream_t side[kSide] = {};
  cudaEvent_t evf = nullptr, evj[kSide] = {};
  cudaStream_t pool[kPool] = {};
  int next = 0;
  std::vector<cudaEvent_t> evs;
  ~SidePool() {
    for (cudaStream_t x : side)
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t x : evj)
      if (x) cudaEventDestroy(x);
    if (evf) cudaEventDestroy(evf);
    for (cudaStream_t x : pool)
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t x : evs) cudaEventDestroy(x);
  }
};

// cudaMalloc-or-pool allocation that reports failure instead of throwing
static bool try_alloc(double** p, size_t bytes) {
  try {
    *p = static_cast<double*>(dev_alloc(bytes));
    return false;
  } catch (const Error&) {
    cudaGetLastError();
    *p = nullptr;
    return true;
  }
}

thread_local Arena g_arena;
thread_local Stager g_stager;
thread_local Dag g_dag;
thread_local SidePool g_side;

thread_local size_t t_last_arena_peak = 0, t_last_pool_bytes = 0;
thread_local bool t_one_stream = false;

// release this host thread's factorization temporaries (θ-batch workers); the
// captured factorization (below) lives in the arena, so it goes first
void drop_thread_graph();
void release_thread_workspace() {
  drop_thread_graph();
  g_arena.free_all();
}

struct Engine {
  Factor& F;
  const Geometry& G;
  cudaStream_t st;
  Arena& ar;
  Stager& sg;
  bool ldl;
  double eps;
  int* d_err = nullptr;
  int TCAP;  // width capacity of product temporaries; overflow is detected on device
  Dag* dag = nullptr;  // task-flow mode (dag.h); nullptr: in-order stream + sections
  cudaEvent_t fork_ev = nullptr;

  Engine(Factor& f, cudaStream_t s, size_t arena_bytes, int tcap, bool use_dag)
      : F(f), G(*f.g), st(s), ar(g_arena), sg(g_stager), ldl(f.ldl), eps(f.eps), TCAP(tcap) {
    ar.dag = nullptr;
    ar.init(arena_bytes, use_dag ? 4 : 1);
    sg.init(use_dag ? ((size_t)512 << 20) : ((size_t)64 << 20), s);
    if (use_dag) {
      sections_on = false;
      dag = &g_dag;
      dag->serial = getenv("HMGP_DAG_DIAG") != nullptr;
      const int L = (int)F.leaf.size();
      std::vector<uintptr_t> lb(L), le(L);
      for (int k = 0; k < L; ++k) {
        const LeafDev& l = F.leaf[k];
        lb[k] = (uintptr_t)l.a;
        le[k] = (uintptr_t)(l.a + (l.kind == DENSE ? (size_t)l.m * l.n : (size_t)(l.m + l.n) * l.cap));
      }
      std::vector<int> pobj(G.n, -1);
      for (int k = 0; k < L; ++k) {
        const HNode& nd = F.nodes[F.leaf_node[k]];
        if (nd.row == nd.col)
          for (int i = G.nbeg[nd.row]; i < G.nend[nd.row]; ++i) pobj[i] = k;
      }
      dag->reset(lb, le, F.d_rank, F.d_compact, F.d_d, pobj, (uintptr_t)ar.base, (uintptr_t)(ar.base + ar.cap));
      ar.dag = dag;
      HMGP_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    }
    d_err = ar.ints(1);
    HMGP_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
    if (dag) dag->fork_from(st, fork_ev);
  }
  ~Engine() {
    ar.dag = nullptr;
    if (fork_ev) cudaEventDestroy(fork_ev);
  }

  // --- task flow: accesses of the next launch (object, write)
  std::vector<std::pair<int, char>> accs;
  void A(const void* p, bool w) {
    if (!dag || !p) return;
    const int o = dag->lookup(p);
    if (o >= 0) accs.push_back({o, (char)w});
  }
  void acc(const GemmItem& g) {
    A(g.A, 0);
    A(g.B, 0);
    A(g.C, 1);
    A(g.M.p, 0);
    A(g.N.p, 0);
    A(g.K.p, 0);
  }
  void acc(const TruncItem& t) {
    A(t.U, 1);
    A(t.V, 1);
    A(t.rank, 1);
    A(t.compact, 1);
    A(t.ws, 1);
    A(t.P, 0);
    A(t.Q, 0);
    A(t.addp, 0);
    A(t.post_L, 0);
    A(t.post_d, 0);
  }
  void acc(const CopyScaleItem& c) {
    A(c.src, 0);
    if (c.mode) A(c.d, 0);
    A(c.dst, 1);
    A(c.cols.p, 0);
    A(c.set_cols, 1);
  }
  void acc(const TrsmLItem& x) {
    A(x.L, 0);
    A(x.M, 1);
    A(x.cols.p, 0);
  }
  void acc(const TrsmRItem& x) {
    A(x.L, 0);
    A(x.X, 1);
    A(x.d, 0);
  }
  template <class T>
  void acc_all(const std::vector<T>& v) {
    if (dag)
      for (const T& x : v) acc(x);
  }
  std::vector<std::pair<int, char>> take_accs() {
    std::vector<std::pair<int, char>> r;
    r.swap(accs);
    return r;
  }
  // launch fn(stream) now: as a task (task flow) or on the current stream
  template <class Fn>
  void run(const char* label, Fn&& fn) {
    if (!dag) {
      fn(st);
      return;
    }
    dag->label = label;
    dag->launch(accs, [&](cudaStream_t s) {
      sg.use(s);
      fn(s);
    });
    accs.clear();
  }

  // --- node helpers
  const HNode& N(int id) const { return F.nodes[id]; }
  int kind(int id) const { return F.nodes[id].kind; }
  int rb(int id) const { return G.nbeg[N(id).row]; }
  int cb(int id) const { return G.nbeg[N(id).col]; }
  int nr(int id) const { return G.nend[N(id).row] - G.nbeg[N(id).row]; }
  int nc(int id) const { return G.nend[N(id).col] - G.nbeg[N(id).col]; }
  int kid(int id, int i, int j) const { return N(id).kids[i * N(id).kc + j]; }
  const LeafDev& LF(int id) const { return F.leaf[N(id).leaf]; }
  int* rankp(int id) const { return F.d_rank + N(id).leaf; }
  int* compp(int id) const { return F.d_compact + N(id).leaf; }
  MV Uv(int id) const {
    const LeafDev& l = LF(id);
    return MV{l.a, l.m, l.m, dimp(rankp(id), l.cap)};
  }
  MV Vv(int id) const {
    const LeafDev& l = LF(id);
    return MV{l.b, l.n, l.n, dimp(rankp(id), l.cap)};
  }
  MV Dv(int id) const {
    const LeafDev& l = LF(id);
    return MV{l.a, l.m, l.m, dimv(l.n)};
  }
  const double* dseg(int begin) const { return F.d_d + begin; }

  MV temp(int rows, Dim cols) {
    MV m;
    m.rows = rows;
    m.ld = std::max(rows, 1);
    m.cols = cols;
    m.p = ar.dbl((size_t)m.ld * std::max(cols.v, 1));
    return m;
  }

  // --- launch statistics (HMGP_STATS=1 prints them after the factorization)
  enum { S_GEMM, S_COPY, S_TRUNC, S_TRSML, S_TRSMR, S_LEAF, S_N };
  long long st_launch[S_N] = {}, st_items[S_N] = {};
  // (stats mode) device time per primitive: an event after every launch, the
  // gap to the previous event is charged to the primitive just launched.
  bool stats_on = getenv("HMGP_STATS") != nullptr;
  std::vector<std::pair<int, cudaEvent_t>> st_ev;
  cudaEvent_t st_prev = nullptr;
  std::vector<std::array<int, 5>> st_meta;  // per event: max m, max n, items, max seq length, slot
  std::array<int, 5> st_next{};
  int st_slot = 0;
  // (stats mode) give the next truncation launch its own per-launch maxima slot
  void tslot() {
    if (stats_on) {
      ++st_slot;
      truncate_launch_slot(st_slot, st);
    }
  }
  void stat(int k, size_t items) {
    ++st_launch[k];
    st_items[k] += (long long)items;
    if (stats_on) {
      st_next[4] = k == S_TRUNC ? st_slot : 0;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      st_ev.push_back({k, e});
      st_meta.push_back(st_next);
      st_next = {};
    }
  }
  void stats_begin() {
    if (stats_on) {
      truncate_hist_enable(true);
      cudaEventCreate(&st_prev);
      cudaEventRecord(st_prev, st);
    }
  }

  // --- batched primitive launchers
  void gemm(std::vector<GemmItem>& v) {
    if (v.empty()) return;
    int tiles = 1;
    for (auto& g : v) {
      const int t = ((g.M.v + 63) / 64) * ((g.N.v + 63) / 64);
      tiles = std::max(tiles, std::min(128, t));
    }
    acc_all(v);
    const char* lab = "gemm";
    if (dag && dag->serial) {  // (diagnostics) size class of the launch
      static std::set<std::string> pool;
      int mm = 0, nn = 0, kk = 0;
      for (auto& g : v) {
        mm = std::max(mm, g.M.v);
        nn = std::max(nn, g.N.v);
        kk = std::max(kk, g.K.v);
      }
      auto p2 = [](int x) { int p = 1; while (p < x) p <<= 1; return p; };
      char buf[96];
      snprintf(buf, sizeof buf, "gemm:%s M<=%d N<=%d K<=%d n<=%d", site, p2(mm), p2(nn), p2(kk), p2((int)v.size()));
      lab = pool.insert(buf).first->c_str();
    }
    run(lab, [&](cudaStream_t s) { launch_gemm(sg.put(v), (int)v.size(), tiles, s); });
    stat(S_GEMM, v.size());
    v.clear();
  }
  void copy(std::vector<CopyScaleItem>& v) {
    if (v.empty()) return;
    int mx = 1;
    for (auto& c : v) mx = std::max<long long>(mx, std::min<long long>((long long)c.rows * c.cols.v, 1 << 24));
    acc_all(v);
    run("copy", [&](cudaStream_t s) { launch_copy_scale(sg.put(v), (int)v.size(), mx, s); });
    stat(S_COPY, v.size());
    v.clear();
  }
  void note_dims(int m, int n, int items, int seq) {
    st_next[0] = std::max(st_next[0], m);
    st_next[1] = std::max(st_next[1], n);
    st_next[2] = items;
    st_next[3] = std::max(st_next[3], seq);
  }
  // Independent launches (disjoint targets) queued as jobs: job 0 runs on the
  // main stream, the others on side streams forked from it and joined back
  // through events, so one step costs its slowest group rather than the sum.
  // Stats mode runs them in order on the main stream so that the per-launch
  // timing stays attributable.
  // A job enqueues its own descriptors (sg.put) and launch on the stream it is
  // given; in task-flow mode every job is a task with the accesses collected
  // (accs) when it was queued.
  struct Job {
    std::function<void(cudaStream_t)> fn;
    std::vector<std::pair<int, char>> acc;
    const char* label;
  };
  std::vector<Job> jobs;
  const char* site = "";  // (task-flow diagnostics) call site of the next truncation jobs
  // (task-flow diagnostics) label with size class: max(m, n) and longest sequence
  const char* cls(const char* base, const std::vector<TruncItem>& v, const std::vector<int>* off) {
    if (!dag || !dag->serial) return base;
    static std::set<std::string> pool;
    int mx = 0, sq = 1;
    for (const TruncItem& t : v) mx = std::max(mx, std::max(t.m, t.n));
    if (off)
      for (size_t b = 0; b + 1 < off->size(); ++b) sq = std::max(sq, (*off)[b + 1] - (*off)[b]);
    int pm = 1, ps = 1;
    while (pm < mx) pm <<= 1;
    while (ps < sq) ps <<= 1;
    char buf[96];
    snprintf(buf, sizeof buf, "%s:%s m<=%d seq<=%d", site, base, pm, ps);
    return pool.insert(buf).first->c_str();
  }
  template <class Fn>
  void add_job(const char* label, Fn&& fn) {
    jobs.push_back(Job{std::function<void(cudaStream_t)>(std::forward<Fn>(fn)), take_accs(), label});
  }
  void run_jobs() {
    if (jobs.empty()) return;
    if (dag) {
      for (Job& j : jobs) {
        dag->label = j.label;
        dag->launch(j.acc, [&](cudaStream_t s) {
          sg.use(s);
          j.fn(s);
        });
      }
      jobs.clear();
      return;
    }
    if (jobs.size() == 1 || stats_on || t_one_stream) {
      for (auto& j : jobs) j.fn(st);
      jobs.clear();
      return;
    }
    constexpr int kSide = SidePool::kSide;
    SidePool& sp = g_side;
    if (!sp.side[0]) {
      HMGP_CUDA(cudaEventCreateWithFlags(&sp.evf, cudaEventDisableTiming));
      for (int i = 0; i < kSide; ++i) {
        HMGP_CUDA(cudaStreamCreateWithFlags(&sp.side[i], cudaStreamNonBlocking));
        HMGP_CUDA(cudaEventCreateWithFlags(&sp.evj[i], cudaEventDisableTiming));
      }
    }
    cudaStream_t* side = sp.side;
    cudaEvent_t evf = sp.evf;
    cudaEvent_t* evj = sp.evj;
    const int ns = std::min((int)jobs.size() - 1, kSide);
    HMGP_CUDA(cudaEventRecord(evf, st));
    for (int i = 0; i < ns; ++i) HMGP_CUDA(cudaStreamWaitEvent(side[i], evf, 0));
    for (size_t k = 1; k < jobs.size(); ++k) {
      const cudaStream_t s = side[(k - 1) % kSide];
      sg.use(s);
      jobs[k].fn(s);
    }
    sg.use(st);
    for (int i = 0; i < ns; ++i) HMGP_CUDA(cudaEventRecord(evj[i], side[i]));
    jobs[0].fn(st);
    for (int i = 0; i < ns; ++i) HMGP_CUDA(cudaStreamWaitEvent(st, evj[i], 0));
    jobs.clear();
  }

  // Side-stream sections: independent parts of a recursion step (disjoint
  // targets) are enqueued on their own stream, forked from the current one,
  // and joined back before the step returns.  While a section is enqueued the
  // arena does not reuse memory (its kernels may still run); the caller
  // releases after the join.  Stats mode runs everything in order.
  struct Sec {
    cudaStream_t s;
    cudaEvent_t done;
  };
  bool sections_on = !stats_on && getenv("HMGP_SERIAL") == nullptr && !t_one_stream;
  cudaStream_t sec_stream() {
    constexpr int kPool = SidePool::kPool;
    cudaStream_t& s = g_side.pool[g_side.next];
    g_side.next = (g_side.next + 1) % kPool;
    if (!s) HMGP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
  }
  static std::vector<cudaEvent_t>& ev_pool() { return g_side.evs; }
  cudaEvent_t ev_get() {
    auto& p = ev_pool();
    if (p.empty()) {
      cudaEvent_t e;
      HMGP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      return e;
    }
    cudaEvent_t e = p.back();
    p.pop_back();
    return e;
  }
  void ev_put(cudaEvent_t e) { ev_pool().push_back(e); }
  template <class Fn>
  void section(std::vector<Sec>& secs, Fn&& fn) {
    if (!sections_on) {
      fn();
      return;
    }
    cudaEvent_t fe = ev_get();
    HMGP_CUDA(cudaEventRecord(fe, st));
    const cudaStream_t s = sec_stream();
    HMGP_CUDA(cudaStreamWaitEvent(s, fe, 0));
    ev_put(fe);  // the wait captured the record; the event may be recorded again
    const cudaStream_t saved = st;
    st = s;
    sg.use(s);
    ++ar.hold;
    fn();
    --ar.hold;
    cudaEvent_t de = ev_get();
    HMGP_CUDA(cudaEventRecord(de, s));
    st = saved;
    sg.use(saved);
    secs.push_back(Sec{s, de});
  }
  void join(std::vector<Sec>& secs) {
    for (const Sec& x : secs) {
      HMGP_CUDA(cudaStreamWaitEvent(st, x.done, 0));
      ev_put(x.done);
    }
    secs.clear();
  }

  // Cluster targets: those up to 2048 rows with the resident (pair / register)
  // dispatch, larger ones on the global-memory path without a shared-memory
  // carve-out; queued as two independent jobs.
  void cluster_jobs(const std::vector<TruncItem>& items, const std::vector<int>& off) {
    std::vector<TruncItem> ir, ig;
    std::vector<int> offr{0}, offg{0};
    for (size_t b = 0; b + 1 < off.size(); ++b) {
      const TruncItem& h = items[off[b]];
      const bool res = trunc_cluster_resident(h.m, h.n);
      std::vector<TruncItem>& dst = res ? ir : ig;
      for (int i = off[b]; i < off[b + 1]; ++i) dst.push_back(items[i]);
      (res ? offr : offg).push_back((int)dst.size());
    }
    const double e = eps;
    int* er = d_err;
    if (!ir.empty()) {
      const int nr = (int)offr.size() - 1;
      acc_all(ir);
      add_job(cls("cluster-res", ir, &offr), [=](cudaStream_t s) { launch_truncate_cluster(sg.put(ir), sg.put(offr), nr, e, er, s, true); });
    }
    if (!ig.empty()) {
      const int ng = (int)offg.size() - 1;
      acc_all(ig);
      add_job(cls("cluster-glb", ig, &offg), [=](cudaStream_t s) { launch_truncate_cluster(sg.put(ig), sg.put(offg), ng, e, er, s, false); });
    }
  }

  // Ordered sequences of updates, one target per sequence (e.g. the kk = 0, 1
  // accumulations of a product part): one job per route, every sequence runs in
  // order on its CTA(s), the targets concurrently.  Workspaces from the arena
  // (the caller releases).
  void lrupd_seq(const std::vector<std::vector<TruncItem>>& seqs) {
    std::vector<TruncItem> t, tp, tb;
    std::vector<int> toff{0}, tpoff{0}, tboff{0};
    int sw = 0, smn = 0;
    size_t nitems = 0;
    for (const auto& sq : seqs) {
      if (sq.empty()) continue;
      const TruncItem& h = sq[0];
      int rcap = 0;
      bool append_only = true;
      for (const TruncItem& x : sq) {
        rcap = std::max(rcap, x.rcap);
        append_only = append_only && x.cond == 4;
      }
      const int rt = append_only ? 0 : trunc_route(h.m, h.n, rcap);
      double* ws = append_only ? nullptr : ar.dbl(trunc_ws_for(h.m, h.n, rcap));
      std::vector<TruncItem>& dst = rt == 2 ? tb : rt == 1 || rt == 3 ? tp : t;
      for (TruncItem x : sq) {
        x.ws = ws;
        dst.push_back(x);
        if (x.cond != 4 && rt == 0) trunc_smem_dims(x.m, x.n, &sw, &smn);
      }
      (rt == 2 ? tboff : rt == 1 || rt == 3 ? tpoff : toff).push_back((int)dst.size());
      nitems += sq.size();
    }
    if (!nitems) return;
    const double e = eps;
    int* er = d_err;
    if (!tb.empty()) cluster_jobs(tb, tboff);
    if (!tp.empty()) {
      const int cnt = (int)tpoff.size() - 1;
      acc_all(tp);
      add_job(cls("pair", tp, &tpoff), [=](cudaStream_t s) { launch_truncate_pair(sg.put(tp), sg.put(tpoff), cnt, e, er, s); });
    }
    if (!t.empty()) {
      const int cnt = (int)toff.size() - 1;
      acc_all(t);
      add_job(cls("seq", t, &toff), [=](cudaStream_t s) { launch_truncate_seq(sg.put(t), sg.put(toff), cnt, e, er, s, sw, smn); });
    }
    tslot();
    run_jobs();
    st_next = {};
    st_next[2] = (int)nitems;
    stat(S_TRUNC, nitems);
  }

  void lrupd(std::vector<TruncItem>& v0) {
    if (v0.empty()) return;
    // large blocks -> one 8-CTA cluster each, medium -> one CTA pair each, the
    // rest -> one CTA each; the groups touch disjoint targets and run as jobs
    std::vector<TruncItem> v, big, mid, dfr;
    for (const TruncItem& t : v0) {
      const int rt = t.cond == 4 ? 0 : trunc_route(t.m, t.n, t.rcap);
      (rt == 2 ? big : rt == 1 ? mid : rt == 3 ? dfr : v).push_back(t);
    }
    v0.clear();
    const double e = eps;
    int* er = d_err;
    size_t nitems = 0;
    std::array<int, 5> mt{};
    for (int pass = 0; pass < 3; ++pass) {
      std::vector<TruncItem>& grp = pass == 2 ? dfr : pass ? mid : big;
      if (grp.empty()) continue;
      std::vector<int> off(grp.size() + 1);
      for (size_t i = 0; i <= grp.size(); ++i) off[i] = (int)i;
      if (pass) {
        const int cnt = (int)grp.size();
        int* dfr = pass == 2 ? ar.ints(cnt) : nullptr;
        acc_all(grp);
        A(dfr, 1);
        add_job(cls(dfr ? "pair-dfr" : "pair", grp, nullptr), [=, g = grp](cudaStream_t s) { launch_truncate_pair(sg.put(g), sg.put(off), cnt, e, er, s, dfr); });
      } else {
        cluster_jobs(grp, off);
      }
      for (const TruncItem& t : grp) {
        mt[0] = std::min(mt[0], -t.m);
        mt[1] = std::max(mt[1], t.n);
      }
      nitems += grp.size();
    }
    if (!v.empty()) {
      int sw = 0, smn = 0;
      for (const TruncItem& t : v) {
        if (t.cond != 4) trunc_smem_dims(t.m, t.n, &sw, &smn);
        mt[0] = mt[0] < 0 ? mt[0] : std::max(mt[0], t.m);
        mt[1] = std::max(mt[1], t.n);
      }
      const int cnt = (int)v.size();
      acc_all(v);
      add_job(cls("small", v, nullptr), [=](cudaStream_t s) { launch_truncate(sg.put(v), cnt, e, er, s, sw, smn); });
      nitems += v.size();
      v.clear();
    }
    if (jobs.empty()) return;
    tslot();
    run_jobs();
    mt[2] = (int)nitems;
    mt[3] = 1;
    st_next = mt;
    stat(S_TRUNC, nitems);
  }
  void print_stats() const {
    static const char* nm[S_N] = {"gemm", "copy", "lrupd", "trsm_left", "trsm_right", "leaf"};
    double ms[S_N] = {};
    cudaStreamSynchronize(st);
    cudaEvent_t prev = st_prev;
    std::vector<std::pair<float, size_t>> tr;
    for (size_t i = 0; i < st_ev.size(); ++i) {
      const auto& pe = st_ev[i];
      float t = 0.f;
      if (prev) cudaEventElapsedTime(&t, prev, pe.second);
      ms[pe.first] += t;
      if (pe.first == S_TRUNC) tr.push_back({t, i});
      prev = pe.second;
    }
    truncate_hist_print();
    {  // launch wall time vs its slowest item / slowest target sequence, by size class
      std::vector<unsigned long long> mx, sq;
      truncate_launch_read(mx, sq);
      std::map<int, std::array<double, 4>> agg;
      cudaEvent_t pv = st_prev;
      for (size_t i = 0; i < st_ev.size(); ++i) {
        float t = 0.f;
        if (pv) cudaEventElapsedTime(&t, pv, st_ev[i].second);
        pv = st_ev[i].second;
        if (st_ev[i].first != S_TRUNC) continue;
        const auto& mt = st_meta[i];
        int b = 1;
        while (b < std::max(std::abs(mt[0]), mt[1])) b <<= 1;
        auto& a = agg[mt[0] < 0 ? -b : b];
        const int sl = mt[4] & ((1 << 17) - 1);
        a[0] += t;
        a[1] += mx[sl] / 1.9e6;
        a[2] += sq[sl] / 1.9e6;
        a[3] += 1;
      }
      for (const auto& kv : agg)
        fprintf(stderr,
                "[hmgp]   lrupd %s max-dim <= %6d: wall %8.1f ms, sum of slowest item %8.1f ms, "
                "slowest sequence %8.1f ms (%d launches)\n",
                kv.first < 0 ? "cluster" : "cta    ", std::abs(kv.first), kv.second[0], kv.second[1],
                kv.second[2], (int)kv.second[3]);
    }
    std::sort(tr.begin(), tr.end(), [](auto& a, auto& b) { return a.first > b.first; });
    for (size_t q = 0; q < tr.size() && q < 12; ++q) {
      const auto& m = st_meta[tr[q].second];
      fprintf(stderr, "[hmgp]   lrupd launch %8.2f ms: max m %d, max n %d, items %d, longest seq %d\n",
              tr[q].first, m[0], m[1], m[2], m[3]);
    }
    // histogram of lrupd time by max(m, n)
    // (cluster launches carry a negative m)
    std::map<int, std::pair<double, int>> hist, shist;
    for (const auto& x : tr) {
      const auto& m = st_meta[x.second];
      int b = 1;
      while (b < std::max(std::abs(m[0]), m[1])) b <<= 1;
      auto& h = hist[m[0] < 0 ? -b : b];
      h.first += x.first;
      h.second += 1;
      int s = 1;
      while (s < m[3]) s <<= 1;
      auto& hs = shist[m[0] < 0 ? -s : s];
      hs.first += x.first;
      hs.second += 1;
    }
    for (const auto& h : hist)
      fprintf(stderr, "[hmgp]   lrupd %s max-dim <= %6d: %6d launches %9.1f ms\n",
              h.first < 0 ? "cluster" : "cta    ", std::abs(h.first), h.second.second, h.second.first);
    for (const auto& h : shist)
      fprintf(stderr, "[hmgp]   lrupd %s longest seq <= %5d: %6d launches %9.1f ms\n",
              h.first < 0 ? "cluster" : "cta    ", std::abs(h.first), h.second.second, h.second.first);
    for (int k = 0; k < S_N; ++k)
      fprintf(stderr, "[hmgp] %-10s launches %9lld items %10lld (%.1f/launch) %10.1f ms\n", nm[k],
              st_launch[k], st_items[k], st_launch[k] ? (double)st_items[k] / st_launch[k] : 0.0,
              ms[k]);
  }
  CopyScaleItem cpy(const double* src, int lds, MV dst, Dim cols, int trans, double alpha,
                    const double* d, int mode) {
    CopyScaleItem c{};
    c.src = src;
    c.lds = lds;
    c.dst = dst.p;
    c.ldd = dst.ld;
    c.rows = dst.rows;
    c.cols = cols;
    c.trans = trans;
    c.alpha = alpha;
    c.d = d;
    c.mode = ldl ? mode : 0;
    c.set_cols = nullptr;
    return c;
  }
  // fused LR update / recompression item for a target (U, V, rank, compact)
  TruncItem lritem(double* U, double* V, int m, int n, int* rank, int* compact, int cond, int cap,
                   const MV* P, const MV* Q, int pro, int qro, double alpha, int rcap) {
    TruncItem t{};
    t.U = U;
    t.V = V;
    t.m = m;
    t.n = n;
    t.rank = rank;
    t.compact = compact;
    t.cond = cond;
    t.cap = cap;
    if (P) {
      t.P = P->p;
      t.Q = Q->p;
      t.ldp = P->ld;
      t.ldq = Q->ld;
      t.pr = P->rows;
      t.qr = Q->rows;
      t.pro = pro;
      t.qro = qro;
      t.addp = P->cols.p;
      t.addv = P->cols.v;
    }
    t.alpha = alpha;
    t.rcap = rcap;
    t.ws = nullptr;
    return t;
  }
  // assign workspaces (from the arena; caller releases) and launch
  void lrupd_ws(std::vector<TruncItem>& v) {
    for (auto& t : v) {
      if (t.cond == 4) continue;
      t.ws = ar.dbl(trunc_ws_for(t.m, t.n, t.rcap));
    }
    lrupd(v);
  }

  // --- compress_low_rank on a list of LR blocks (hblock.cpp:164-170)
  void compress(const std::vector<int>& ids) {
    if (ids.empty()) return;
    const size_t mk = ar.mark();
    std::vector<TruncItem> v;
    for (int x : ids) {
      const LeafDev& l = LF(x);
      v.push_back(lritem(l.a, l.b, l.m, l.n, rankp(x), compp(x), 0, l.cap, nullptr, nullptr, 0, 0,
                         1.0, l.cap));
    }
    site = "compress";
    lrupd_ws(v);
    ar.release(mk);
  }

  // ------------------------------------------------------- hblk::apply ----
  struct Ap {
    int b;      // H-block node
    MV x, y;    // y (+)= alpha op(B) x
    double alpha;
    int trans;  // 0: B, 1: B^T
  };
  // Flatten a branch into its stored leaves (null children are structural
  // zeros, hblock.cpp:43-45), with the matching x / y sub-views.
  void flatten(const Ap& a, std::vector<Ap>& out) {
    if (kind(a.b) != BRANCH) {
      out.push_back(a);
      return;
    }
    const HNode& nd = N(a.b);
    for (int pos = 0; pos < nd.kr * nd.kc; ++pos) {
      const int c = nd.kids[pos];
      if (c < 0) continue;
      Ap s = a;
      s.b = c;
      if (!a.trans) {
        s.x = rows_of(a.x, cb(c) - cb(a.b), nc(c));
        s.y = rows_of(a.y, rb(c) - rb(a.b), nr(c));
      } else {
        s.x = rows_of(a.x, rb(c) - rb(a.b), nr(c));
        s.y = rows_of(a.y, cb(c) - cb(a.b), nc(c));
      }
      flatten(s, out);
    }
  }

  // y += alpha op(B) x for a list of (B, x, y); every H-block is flattened to
  // its leaves, so any block costs a fixed number of launches: dense leaves,
  // the two low-rank stages and one ordered add.  Leaves of a branch share y
  // rows: each writes its own temporary, and k_ordered_add applies them to y in
  // the reference's DFS leaf order (hblock.cpp:46-60) — no FP64 atomics, so the
  // result is bit-reproducible.  Long contractions V^T x (K >= 2048) are split
  // into K-range items on separate slabs summed in a fixed order.
  void apply(const std::vector<Ap>& its0) {
    if (its0.empty()) return;
    site = "apply";
    const size_t mk = ar.mark();
    std::vector<Ap> its;
    std::vector<int> grp;  // index into its0 for branch leaves, -1 otherwise
    for (size_t q = 0; q < its0.size(); ++q) {
      const Ap& a = its0[q];
      const size_t before = its.size();
      flatten(a, its);
      for (size_t i = before; i < its.size(); ++i) grp.push_back(kind(a.b) == BRANCH ? (int)q : -1);
    }
    // branch leaves: redirect y to a private temporary (alpha applied in the ordered add)
    std::vector<OrdSeg> seg(its.size(), OrdSeg{nullptr, 0, 0});
    for (size_t i = 0; i < its.size(); ++i) {
      if (grp[i] < 0) continue;
      Ap& a = its[i];
      const MV t = temp(a.y.rows, a.y.cols);
      seg[i] = OrdSeg{t.p, t.ld, (int)(a.y.p - its0[grp[i]].y.p)};
      a.y.p = t.p;
      a.y.ld = t.ld;
      a.alpha = 1.0;
    }
    auto own = [&](size_t i) { return grp[i] >= 0; };  // y is a private temporary: overwrite
    std::vector<GemmItem> g;
    std::vector<size_t> lr;
    for (size_t ii = 0; ii < its.size(); ++ii) {
      const Ap& a = its[ii];
      if (kind(a.b) == DENSE) {
        const LeafDev& l = LF(a.b);
        GemmItem gi{};
        gi.A = l.a;
        gi.lda = l.m;
        gi.ta = a.trans;
        gi.B = a.x.p;
        gi.ldb = a.x.ld;
        gi.tb = 0;
        gi.C = a.y.p;
        gi.ldc = a.y.ld;
        gi.M = dimv(a.trans ? l.n : l.m);
        gi.N = a.x.cols;
        gi.K = dimv(a.trans ? l.m : l.n);
        gi.alpha = a.alpha;
        gi.atomic = own(ii) ? 2 : 0;
        g.push_back(gi);
      } else {
        lr.push_back(ii);
      }
    }
    gemm(g);
    if (!lr.empty()) {
      std::vector<MV> T;
      std::vector<SlabSumItem> ss;
      for (size_t i : lr) {  // T = (trans ? U : V)^T x   (rank x c)
        const Ap& a = its[i];
        const LeafDev& l = LF(a.b);
        const int kk = a.trans ? l.m : l.n;
        const int ns = kk >= 2048 ? std::min(32, (kk + 1023) / 1024) : 1;
        const int kc = (kk + ns - 1) / ns;
        MV t = temp(l.cap, Dim{a.x.cols.v * ns, nullptr});
        t.cols = a.x.cols;
        T.push_back(t);
        const size_t slab = (size_t)t.ld * std::max(a.x.cols.v, 1);
        for (int s = 0; s < ns; ++s) {
          const int k0 = s * kc, k1 = std::min(kk, k0 + kc);
          GemmItem gi{};
          gi.A = (a.trans ? l.a : l.b) + k0;
          gi.lda = kk;
          gi.ta = 1;
          gi.B = a.x.p + k0;
          gi.ldb = a.x.ld;
          gi.C = t.p + s * slab;
          gi.ldc = t.ld;
          gi.M = dimp(rankp(a.b), l.cap);
          gi.N = a.x.cols;
          gi.K = dimv(k1 - k0);
          gi.alpha = 1.0;
          gi.atomic = 2;  // every slab is written by exactly one item
          g.push_back(gi);
        }
        if (ns > 1) ss.push_back(SlabSumItem{t.p, t.ld, dimp(rankp(a.b), l.cap), a.x.cols, ns, slab});
      }
      gemm(g);
      if (!ss.empty()) {
        int mx = 1;
        for (auto& x : ss) mx = std::max(mx, x.rows.v * x.cols.v);
        for (auto& x : ss) A(x.p, 1);
        run("slab-sum", [&](cudaStream_t s) { launch_slab_sum(sg.put(ss), (int)ss.size(), mx, s); });
        stat(S_COPY, ss.size());
      }
      for (size_t q = 0; q < lr.size(); ++q) {  // y += alpha (trans ? V : U) T
        const Ap& a = its[lr[q]];
        const LeafDev& l = LF(a.b);
        GemmItem gi{};
        gi.A = a.trans ? l.b : l.a;
        gi.lda = a.trans ? l.n : l.m;
        gi.B = T[q].p;
        gi.ldb = T[q].ld;
        gi.C = a.y.p;
        gi.ldc = a.y.ld;
        gi.M = dimv(a.trans ? l.n : l.m);
        gi.N = a.x.cols;
        gi.K = dimp(rankp(a.b), l.cap);
        gi.alpha = a.alpha;
        gi.atomic = own(lr[q]) ? 2 : 0;
        g.push_back(gi);
      }
      gemm(g);
    }
    // ordered application of the branch leaves' temporaries
    std::vector<OrdIv> iv;
    std::vector<OrdSeg> sl;
    int mx = 1;
    for (size_t q = 0; q < its0.size(); ++q) {
      if (kind(its0[q].b) != BRANCH) continue;
      std::vector<size_t> mine;
      std::vector<int> cut;
      for (size_t i = 0; i < its.size(); ++i)
        if (grp[i] == (int)q) {
          mine.push_back(i);
          cut.push_back(seg[i].r0);
          cut.push_back(seg[i].r0 + its[i].y.rows);
        }
      if (mine.empty()) continue;
      std::sort(cut.begin(), cut.end());
      cut.erase(std::unique(cut.begin(), cut.end()), cut.end());
      std::vector<std::vector<int>> lists(cut.size());
      for (size_t i : mine) {  // DFS order is the order of `mine`
        const int a0 = (int)(std::lower_bound(cut.begin(), cut.end(), seg[i].r0) - cut.begin());
        const int a1 = (int)(std::lower_bound(cut.begin(), cut.end(), seg[i].r0 + its[i].y.rows) - cut.begin());
        for (int k = a0; k < a1; ++k) lists[k].push_back((int)i);
      }
      const Ap& root = its0[q];
      for (size_t k = 0; k + 1 < cut.size(); ++k) {
        if (lists[k].empty()) continue;
        OrdIv v{root.y.p, root.y.ld, root.x.cols, root.alpha, cut[k], cut[k + 1], (int)sl.size(), 0};
        for (int i : lists[k]) sl.push_back(seg[i]);
        v.l1 = (int)sl.size();
        iv.push_back(v);
        mx = std::max(mx, (cut[k + 1] - cut[k]) * root.x.cols.v);
        A(root.y.p, 1);
      }
      for (size_t i : mine) A(seg[i].src, 0);
    }
    if (!iv.empty()) {
      run("ordered-add", [&](cudaStream_t s) {
        const OrdSeg* ds = sg.put(sl);
        launch_ordered_add(sg.put(iv), (int)iv.size(), ds, mx, s);
      });
      stat(S_COPY, iv.size());
    }
    ar.release(mk);
  }

  // multiply(B, X) into preallocated Y (zeroed here), hblock.cpp:89-92
  void multiply_into(const std::vector<int>& bs, const std::vector<MV>& xs, const std::vector<MV>& ys) {
    std::vector<CopyScaleItem> z;
    std::vector<Ap> ap;
    for (size_t i = 0; i < bs.size(); ++i) {
      z.push_back(cpy(nullptr, 0, ys[i], xs[i].cols, 0, 0.0, nullptr, 0));
      ap.push_back(Ap{bs[i], xs[i], ys[i], 1.0, 0});
    }
    copy(z);
    apply(ap);
  }

  // -------------------------------------------------- solve_lower_multi ---
  void solve_lower_multi(int l, const std::vector<MV>& ms) {
    if (ms.empty()) return;
    if (kind(l) == DENSE) {
      const LeafDev& L = LF(l);
      std::vector<TrsmLItem> v;
      int mc = 1;
      for (const MV& m : ms) {
        v.push_back(TrsmLItem{L.a, L.m, L.m, m.p, m.ld, m.cols, 0});
        mc = std::max(mc, m.cols.v);
      }
      acc_all(v);
      run("trsm_left", [&](cudaStream_t s) { launch_trsm_left(sg.put(v), (int)v.size(), mc, s, L.m); });
      stat(S_TRSML, v.size());
      return;
    }
    const int l00 = kid(l, 0, 0), l10 = kid(l, 1, 0), l11 = kid(l, 1, 1);
    const int n1 = nr(l00);
    std::vector<MV> top, bot;
    for (const MV& m : ms) {
      top.push_back(rows_of(m, 0, n1));
      bot.push_back(rows_of(m, n1, m.rows - n1));
    }
    solve_lower_multi(l00, top);
    std::vector<Ap> ap;
    for (size_t i = 0; i < ms.size(); ++i) ap.push_back(Ap{l10, top[i], bot[i], -1.0, 0});
    apply(ap);
    solve_lower_multi(l11, bot);
  }

  // ----------------------------------------------------- trsm_dense_block -
  // x <- x L^{-T} (D^{-1}), hfactor.cpp:107-123
  void trsm_dense(const std::vector<MV>& xs, int l) {
    if (xs.empty()) return;
    if (kind(l) == DENSE) {
      const LeafDev& L = LF(l);
      std::vector<TrsmRItem> v;
      int mr = 1;
      for (const MV& x : xs) {  // X <- X L^{-T} D^{-1} in one launch
        v.push_back(TrsmRItem{L.a, L.m, L.m, x.p, x.ld, x.rows, ldl ? dseg(rb(l)) : nullptr});
        mr = std::max(mr, x.rows);
      }
      acc_all(v);
      run("trsm_right", [&](cudaStream_t s) { launch_trsm_right(sg.put(v), (int)v.size(), mr, s, L.m); });
      stat(S_TRSMR, v.size());
      return;
    }
    const int l00 = kid(l, 0, 0), l10 = kid(l, 1, 0), l11 = kid(l, 1, 1);
    const int n1 = nr(l00), t = nr(l);
    std::vector<MV> x1, x2;
    for (const MV& x : xs) {
      x1.push_back(cols_of(x, 0, n1));
      x2.push_back(cols_of(x, n1, t - n1));
    }
    trsm_dense(x1, l00);
    const size_t mk = ar.mark();
    std::vector<MV> wt, pr;
    std::vector<CopyScaleItem> c;
    std::vector<int> bs;
    for (size_t i = 0; i < xs.size(); ++i) {
      MV w = temp(n1, dimv(xs[i].rows));  // wt = x1^T, rows scaled by d
      c.push_back(cpy(x1[i].p, x1[i].ld, w, dimv(xs[i].rows), 1, 1.0, dseg(rb(l00)), 1));
      wt.push_back(w);
      pr.push_back(temp(t - n1, dimv(xs[i].rows)));
      bs.push_back(l10);
    }
    copy(c);
    multiply_into(bs, wt, pr);
    for (size_t i = 0; i < xs.size(); ++i) {  // x2 -= pr^T
      CopyScaleItem a = cpy(pr[i].p, pr[i].ld, x2[i], dimv(t - n1), 1, -1.0, nullptr, 0);
      a.accum = 1;
      c.push_back(a);
    }
    copy(c);
    ar.release(mk);
    trsm_dense(x2, l11);
  }

  // -------------------------------------------------------- trsm_lower_t --
  void trsm(const std::vector<int>& xs, int l) {
    if (xs.empty()) return;
    std::vector<int> lr, dn, br;
    for (int x : xs) (kind(x) == LOWRANK ? lr : kind(x) == DENSE ? dn : br).push_back(x);
    // the low-rank, dense and branch targets are disjoint: the first two run as
    // side-stream sections while the branch recursion proceeds on this stream
    const size_t mk0 = ar.mark();
    std::vector<Sec> secs;
    const int parts = !lr.empty() + !dn.empty() + !br.empty();
    auto part = [&](bool last, auto&& fn) {
      if (parts > 1 && !last)
        section(secs, fn);
      else
        fn();
    };
    if (kind(l) == DENSE) {
      const LeafDev& L = LF(l);
      if (!lr.empty())
        part(dn.empty() && br.empty(), [&] {
          // compress_low_rank + V <- L^{-1} V (+ D^{-1}) fused in one launch
          const size_t mk = ar.mark();
          std::vector<TruncItem> v;
          for (int x : lr) {
            const LeafDev& lx = LF(x);
            TruncItem t = lritem(lx.a, lx.b, lx.m, lx.n, rankp(x), compp(x), 0, lx.cap, nullptr,
                                 nullptr, 0, 0, 1.0, lx.cap);
            t.post_L = L.a;
            t.post_ldl_ld = L.m;
            t.post_d = ldl ? dseg(rb(l)) : nullptr;
            v.push_back(t);
          }
          site = "trsm-lr";
          lrupd_ws(v);
          ar.release(mk);
        });
      if (!dn.empty())
        part(br.empty(), [&] {
          std::vector<MV> d;
          for (int x : dn) d.push_back(Dv(x));
          trsm_dense(d, l);
        });
      if (!br.empty()) {
        std::vector<int> ch;
        for (int x : br)
          for (int i = 0; i < N(x).kr; ++i) ch.push_back(kid(x, i, 0));
        trsm(ch, l);
      }
      join(secs);
      ar.release(mk0);
      return;
    }
    if (!lr.empty())
      part(dn.empty() && br.empty(), [&] {
        compress(lr);
        std::vector<MV> vs;
        for (int x : lr) vs.push_back(Vv(x));
        solve_lower_multi(l, vs);
        if (ldl) {
          std::vector<CopyScaleItem> c;
          for (const MV& V : vs) c.push_back(cpy(V.p, V.ld, V, V.cols, 0, 1.0, dseg(rb(l)), 2));
          copy(c);
        }
      });
    if (!dn.empty())
      part(br.empty(), [&] {
        std::vector<MV> d;
        for (int x : dn) d.push_back(Dv(x));
        trsm_dense(d, l);
      });
    if (!br.empty()) {
      std::vector<int> l0, l1;
      std::vector<Trip> tr;
      for (int x : br)
        for (int i = 0; i < N(x).kr; ++i) {
          l0.push_back(kid(x, i, 0));
          l1.push_back(kid(x, i, 1));
          tr.push_back(Trip{kid(x, i, 1), kid(x, i, 0), kid(l, 1, 0)});
        }
      trsm(l0, kid(l, 0, 0));
      subprod(tr);
      trsm(l1, kid(l, 1, 1));
    }
    join(secs);
    ar.release(mk0);
  }

  // ------------------------------------------------------ add_low_rank ---
  struct Add {
    int c;
    MV p, q;  // p: rows at absolute row0, q: rows at absolute col0
    double alpha;
    int row0, col0;
  };
  // hblock.cpp:205-216: distribute an add over a branch target's stored leaves
  // (child order), keeping the P / Q rows that intersect each child.
  void expand_add(const Add& a, std::vector<Add>& out) {
    if (kind(a.c) != BRANCH) {
      out.push_back(a);
      return;
    }
    const HNode& nd = N(a.c);
    for (int pos = 0; pos < nd.kr * nd.kc; ++pos) {
      const int ch = nd.kids[pos];
      if (ch < 0) continue;
      const int r0 = std::max(a.row0, rb(ch)), r1 = std::min(a.row0 + a.p.rows, rb(ch) + nr(ch));
      const int c0 = std::max(a.col0, cb(ch)), c1 = std::min(a.col0 + a.q.rows, cb(ch) + nc(ch));
      if (r0 >= r1 || c0 >= c1) continue;
      expand_add(Add{ch, rows_of(a.p, r0 - a.row0, r1 - r0), rows_of(a.q, c0 - a.col0, c1 - c0),
                     a.alpha, r0, c0},
                 out);
    }
  }

  // add_low_rank for a list of terms IN REFERENCE ORDER; terms may share
  // targets.  Every term is expanded to leaf-level adds; each leaf receives its
  // adds in term order (the reference's sequence, so the watermark recompressions
  // happen at the same points), adds to different leaves run in parallel:
  // round r applies the r-th add of every leaf in one batched launch.
  void add_lr(const std::vector<Add>& terms) {
    if (terms.empty()) return;
    std::vector<Add> flat;
    for (const Add& a : terms) expand_add(a, flat);
    std::vector<std::vector<int>> seq;  // per target leaf: indices into flat
    std::vector<int> slot(F.nodes.size(), -1);
    for (int i = 0; i < (int)flat.size(); ++i) {
      int& s = slot[flat[i].c];
      if (s < 0) {
        s = (int)seq.size();
        seq.emplace_back();
      }
      seq[s].push_back(i);
    }
    // two launches in total: one CTA per dense target runs its GEMM updates in
    // order, one CTA per low-rank target runs its append / watermark
    // recompressions in order (same decisions as the reference, hblock.cpp:200)
    const size_t mk = ar.mark();
    std::vector<GemmItem> g;
    std::vector<int> goff{0};
    std::vector<TruncItem> t, tb, tp, td;
    std::vector<int> toff{0}, tboff{0}, tpoff{0}, tdoff{0};
    int sw = 0, smn = 0;
    std::array<int, 5> meta_t{}, meta_b{}, meta_p{}, meta_d{};  // stats: max m, max n, targets, longest seq
    auto meta = [](std::array<int, 5>& mt, int m, int n, int seq) {
      mt[0] = std::max(mt[0], m);
      mt[1] = std::max(mt[1], n);
      ++mt[2];
      mt[3] = std::max(mt[3], seq);
    };
    for (const auto& v : seq) {
      const int c = flat[v[0]].c;
      const LeafDev& l = LF(c);
      if (kind(c) == DENSE) {  // hblock.cpp:181-184
        for (int i : v) {
          const Add& a = flat[i];
          GemmItem gi{};
          gi.A = a.p.p;
          gi.lda = a.p.ld;
          gi.B = a.q.p;
          gi.ldb = a.q.ld;
          gi.tb = 1;
          gi.C = l.a + (size_t)(a.col0 - cb(c)) * l.m + (a.row0 - rb(c));
          gi.ldc = l.m;
          gi.M = dimv(a.p.rows);
          gi.N = dimv(a.q.rows);
          gi.K = a.p.cols;
          gi.alpha = a.alpha;
          g.push_back(gi);
        }
        goff.push_back((int)g.size());
      } else {  // hblock.cpp:185-203
        int rcap = 0;
        for (int i : v) rcap = std::max(rcap, l.cap + flat[i].p.cols.v);
        const int rt = trunc_route(l.m, l.n, rcap);
        double* ws = ar.dbl(trunc_ws_for(l.m, l.n, rcap));
        std::vector<TruncItem>& dst = rt == 2 ? tb : rt == 1 ? tp : rt == 3 ? td : t;
        for (int i : v) {
          const Add& a = flat[i];
          TruncItem ti = lritem(l.a, l.b, l.m, l.n, rankp(c), compp(c), 2, l.cap, &a.p, &a.q,
                                a.row0 - rb(c), a.col0 - cb(c), a.alpha, l.cap + a.p.cols.v);
          ti.ws = ws;
          dst.push_back(ti);
        }
        if (rt == 2) {
          tboff.push_back((int)tb.size());
          meta(meta_b, l.m, l.n, (int)v.size());
        } else if (rt == 1) {
          tpoff.push_back((int)tp.size());
          meta(meta_p, l.m, l.n, (int)v.size());
        } else if (rt == 3) {
          tdoff.push_back((int)td.size());
          meta(meta_d, l.m, l.n, (int)v.size());
        } else {
          toff.push_back((int)t.size());
          meta(meta_t, l.m, l.n, (int)v.size());
          trunc_smem_dims(l.m, l.n, &sw, &smn);
        }
      }
    }
    // the four groups touch disjoint targets: queue them as concurrent jobs
    const double e = eps;
    int* er = d_err;
    size_t ntr = 0;
    std::array<int, 5> mt{};
    if (!g.empty()) {
      const int ng = (int)goff.size() - 1;
      acc_all(g);
      add_job("gemm_seq", [=](cudaStream_t s) { launch_gemm_seq(sg.put(g), sg.put(goff), ng, s); });
      st_launch[S_GEMM]++;
      st_items[S_GEMM] += (long long)g.size();
    }
    if (!tb.empty()) {
      cluster_jobs(tb, tboff);
      ntr += tb.size();
      mt[0] = std::min(mt[0], -meta_b[0]);
      mt[1] = std::max(mt[1], meta_b[1]);
      mt[3] = std::max(mt[3], meta_b[3]);
    }
    for (int pass = 0; pass < 2; ++pass) {
      const std::vector<TruncItem>& tq = pass ? td : tp;
      const std::vector<int>& to = pass ? tdoff : tpoff;
      const std::array<int, 5>& mq = pass ? meta_d : meta_p;
      if (tq.empty()) continue;
      const int cnt = (int)to.size() - 1;
      int* dfr = pass == 1 ? ar.ints(cnt) : nullptr;
      acc_all(tq);
      A(dfr, 1);
      add_job(cls(dfr ? "pair-dfr" : "pair", tq, &to), [=, q = tq, o = to](cudaStream_t s) { launch_truncate_pair(sg.put(q), sg.put(o), cnt, e, er, s, dfr); });
      ntr += tq.size();
      mt[0] = std::min(mt[0], -mq[0]);
      mt[1] = std::max(mt[1], mq[1]);
      mt[3] = std::max(mt[3], mq[3]);
    }
    if (!t.empty()) {
      const int cnt = (int)toff.size() - 1;
      acc_all(t);
      add_job(cls("seq", t, &toff), [=](cudaStream_t s) { launch_truncate_seq(sg.put(t), sg.put(toff), cnt, e, er, s, sw, smn); });
      ntr += t.size();
      if (mt[0] >= 0) mt[0] = std::max(mt[0], meta_t[0]);
      mt[1] = std::max(mt[1], meta_t[1]);
      mt[3] = std::max(mt[3], meta_t[3]);
    }
    if (!jobs.empty()) {
      if (ntr) tslot();
      run_jobs();
      if (ntr) {
        mt[2] = (int)ntr;
        st_next = mt;
        stat(S_TRUNC, ntr);
        st_launch[S_TRUNC] += 0;
      } else {
        st_launch[S_GEMM]--;  // counted above; record the event against gemm
        st_items[S_GEMM] -= (long long)g.size();
        stat(S_GEMM, g.size());
      }
    }
    ar.release(mk);
  }

  // distinct leaf targets, one add each
  void add_leaves(const std::vector<Add>& its) {
    if (its.empty()) return;
    site = "add-leaves";
    std::vector<GemmItem> g;
    std::vector<TruncItem> t;
    std::vector<Add> br;
    const size_t mk = ar.mark();
    for (const Add& a : its) {
      const int k = kind(a.c);
      if (k == DENSE) {  // hblock.cpp:181-184
        const LeafDev& l = LF(a.c);
        GemmItem gi{};
        gi.A = a.p.p;
        gi.lda = a.p.ld;
        gi.B = a.q.p;
        gi.ldb = a.q.ld;
        gi.tb = 1;
        gi.C = l.a + (size_t)(a.col0 - cb(a.c)) * l.m + (a.row0 - rb(a.c));
        gi.ldc = l.m;
        gi.M = dimv(a.p.rows);
        gi.N = dimv(a.q.rows);
        gi.K = a.p.cols;
        gi.alpha = a.alpha;
        g.push_back(gi);
      } else if (k == LOWRANK) {  // hblock.cpp:185-203
        const LeafDev& l = LF(a.c);
        t.push_back(lritem(l.a, l.b, l.m, l.n, rankp(a.c), compp(a.c), 2, l.cap, &a.p, &a.q,
                           a.row0 - rb(a.c), a.col0 - cb(a.c), a.alpha, l.cap + a.p.cols.v));
      } else {
        br.push_back(a);
      }
    }
    gemm(g);
    site = "add-leaves";
    lrupd_ws(t);
    ar.release(mk);
  }

  // scaled copies: V (rows) * d over a column cluster
  MV scaled_copy_rows(MV src, int dbegin) {
    MV t = temp(src.rows, src.cols);
    std::vector<CopyScaleItem> c{cpy(src.p, src.ld, t, src.cols, 0, 1.0, dseg(dbegin), 1)};
    copy(c);
    return t;
  }

  // --------------------------------------------------- product_low_rank --
  struct Pair {
    MV p, q;
  };
  // Results are allocated on the arena BEFORE any internal temporary so the
  // caller can release them with its own mark.
  std::vector<Pair> product_lr(const std::vector<std::pair<int, int>>& abs) {
    const size_t n = abs.size();
    std::vector<Pair> out(n);
    std::vector<int> cls(n);  // 0 aLR, 1 bLR, 2 aDense, 3 bDense, 4 branch
    int nbr = 0;
    for (size_t i = 0; i < n; ++i) {
      const int a = abs[i].first, b = abs[i].second;
      nbr += !(kind(a) == LOWRANK || kind(b) == LOWRANK || kind(a) == DENSE || kind(b) == DENSE);
    }
    int* wcs = nbr ? ar.ints(nbr) : nullptr;
    if (nbr) {
      A(wcs, 1);
      run("memset", [&](cudaStream_t s) { HMGP_CUDA(cudaMemsetAsync(wcs, 0, 4ull * nbr, s)); });
    }
    int wci = 0;
    for (size_t i = 0; i < n; ++i) {
      const int a = abs[i].first, b = abs[i].second;
      cls[i] = kind(a) == LOWRANK ? 0 : kind(b) == LOWRANK ? 1 : kind(a) == DENSE ? 2
               : kind(b) == DENSE ? 3 : 4;
      switch (cls[i]) {
        case 0:
          out[i].p = Uv(a);
          out[i].q = temp(nr(b), Uv(a).cols);
          break;
        case 1:
          out[i].p = temp(nr(a), Uv(b).cols);
          out[i].q = Uv(b);
          break;
        case 2:
          out[i].p = temp(nr(a), dimv(nc(a)));
          out[i].q = kind(b) == DENSE ? Dv(b) : temp(nr(b), dimv(nc(b)));
          break;
        case 3:
          out[i].p = temp(nr(a), dimv(nr(b)));
          out[i].q = temp(nr(b), dimv(nr(b)));
          break;
        default: {
          int* wc = wcs + wci++;
          out[i].p = temp(nr(a), dimp(wc, TCAP));
          out[i].q = temp(nr(b), dimp(wc, TCAP));
        }
      }
    }
    const size_t mk = ar.mark();
    // simple cases; independent of the branch x branch products below, so they
    // run as a side-stream section when both kinds are present
    std::vector<Sec> psecs;
    bool any_simple = false, any_branch = false;
    for (size_t i = 0; i < n; ++i) (cls[i] == 4 ? any_branch : any_simple) = true;
    auto simple = [&] {
      std::vector<int> mb;
      std::vector<MV> mx, my;
      std::vector<CopyScaleItem> c;
      for (size_t i = 0; i < n; ++i) {
        const int a = abs[i].first, b = abs[i].second;
        switch (cls[i]) {
          case 0: {  // {U_a, B (V_a d)}
            MV va = Vv(a);
            if (ldl) {
              MV t = temp(va.rows, va.cols);
              c.push_back(cpy(va.p, va.ld, t, va.cols, 0, 1.0, dseg(cb(a)), 1));
              va = t;
            }
            mb.push_back(b);
            mx.push_back(va);
            my.push_back(out[i].q);
            break;
          }
          case 1: {  // {A (V_b d), U_b}
            MV vb = Vv(b);
            if (ldl) {
              MV t = temp(vb.rows, vb.cols);
              c.push_back(cpy(vb.p, vb.ld, t, vb.cols, 0, 1.0, dseg(cb(b)), 1));
              vb = t;
            }
            mb.push_back(a);
            mx.push_back(vb);
            my.push_back(out[i].p);
            break;
          }
          case 2: {  // {A.D diag(d), B materialised}
            c.push_back(cpy(LF(a).a, LF(a).m, out[i].p, dimv(nc(a)), 0, 1.0, dseg(cb(a)), 3));
            if (kind(b) != DENSE) {
              MV e = temp(nc(b), dimv(nc(b)));
              c.push_back(cpy(nullptr, 0, e, dimv(nc(b)), 0, 1.0, nullptr, 0));
              c.back().mode = 0;
              mb.push_back(b);
              mx.push_back(e);
              my.push_back(out[i].q);
            }
            break;
          }
          case 3: {  // {A (B.D^T d), I}
            MV x = temp(nc(b), dimv(nr(b)));
            c.push_back(cpy(LF(b).a, LF(b).m, x, dimv(nr(b)), 1, 1.0, dseg(cb(b)), 1));
            CopyScaleItem e = cpy(nullptr, 0, out[i].q, dimv(nr(b)), 0, 1.0, nullptr, 0);
            e.mode = 0;
            c.push_back(e);
            mb.push_back(a);
            mx.push_back(x);
            my.push_back(out[i].p);
            break;
          }
          default:
            break;
        }
      }
      copy(c);
      if (!mb.empty()) multiply_into(mb, mx, my);
    };
    if (any_simple) {
      if (any_branch)
        section(psecs, simple);
      else
        simple();
    }
    // branch x branch (hfactor.cpp:150-190)
    std::vector<size_t> bi;
    for (size_t i = 0; i < n; ++i)
      if (cls[i] == 4) bi.push_back(i);
    if (!bi.empty()) {
      struct Part {
        size_t item;
        int ii, jj, a0, b0;
        MV p, q;
        int* cols;
      };
      std::vector<Part> parts;
      size_t npart = 0;
      for (size_t i : bi) npart += (size_t)N(abs[i].first).kr * N(abs[i].second).kr;
      int* pcols = ar.ints(npart);
      A(pcols, 1);
      run("memset", [&](cudaStream_t s) { HMGP_CUDA(cudaMemsetAsync(pcols, 0, 4 * npart, s)); });
      for (size_t i : bi) {
        const int a = abs[i].first, b = abs[i].second;
        for (int ii = 0; ii < N(a).kr; ++ii)
          for (int jj = 0; jj < N(b).kr; ++jj) {
            Part pt;
            pt.item = i;
            pt.ii = ii;
            pt.jj = jj;
            pt.a0 = kid(a, ii, 0);
            pt.b0 = kid(b, jj, 0);
            pt.cols = pcols + parts.size();
            pt.p = temp(nr(pt.a0), dimp(pt.cols, TCAP));
            pt.q = temp(nr(pt.b0), dimp(pt.cols, TCAP));
            parts.push_back(pt);
          }
      }
      // All child products of every kk in ONE recursive call (they only read A, B);
      // the accumulation into each part then runs kk = 0, 1 in the reference's
      // order with the > 48 recompression rule (hfactor.cpp:164-172).
      std::vector<std::pair<int, int>> sub;
      std::vector<size_t> who;
      std::vector<int> whokk;
      for (int kk = 0; kk < 2; ++kk)
        for (size_t t = 0; t < parts.size(); ++t) {
          const int a = abs[parts[t].item].first, b = abs[parts[t].item].second;
          if (kk >= N(a).kc) continue;
          sub.push_back({kid(a, parts[t].ii, kk), kid(b, parts[t].jj, kk)});
          who.push_back(t);
          whokk.push_back(kk);
        }
      if (!sub.empty()) {
        const size_t mk2 = ar.mark();
        std::vector<Pair> tp = product_lr(sub);
        // per part: kk = 0 then kk = 1, one launch of ordered sequences
        std::vector<std::vector<TruncItem>> seqs(parts.size());
        for (int kk = 0; kk < 2; ++kk)
          for (size_t s = 0; s < sub.size(); ++s) {
            if (whokk[s] != kk) continue;
            Part& pt = parts[who[s]];
            seqs[who[s]].push_back(lritem(pt.p.p, pt.q.p, pt.p.rows, pt.q.rows, pt.cols, nullptr, 3, TCAP,
                                          &tp[s].p, &tp[s].q, 0, 0, 1.0, TCAP + tp[s].p.cols.v));
          }
        site = "plr-acc";
        lrupd_seq(seqs);
        ar.release(mk2);
      }
      // embed parts into out (pure appends; one launch per part index so the
      // same target is never appended to concurrently), then truncate once
      size_t maxparts = 0;
      std::vector<std::vector<size_t>> byitem(n);
      for (size_t t = 0; t < parts.size(); ++t) byitem[parts[t].item].push_back(t);
      for (size_t i : bi) maxparts = std::max(maxparts, byitem[i].size());
      {  // per item: its parts appended in order (one launch of sequences)
        std::vector<std::vector<TruncItem>> seqs;
        for (size_t i : bi) {
          seqs.emplace_back();
          for (size_t q = 0; q < byitem[i].size(); ++q) {
            const Part& pt = parts[byitem[i][q]];
            const int a = abs[i].first, b = abs[i].second;
            seqs.back().push_back(lritem(out[i].p.p, out[i].q.p, nr(a), nr(b),
                                         const_cast<int*>(out[i].p.cols.p), nullptr, 4, TCAP, &pt.p, &pt.q,
                                         rb(pt.a0) - rb(a), rb(pt.b0) - rb(b), 1.0, TCAP));
          }
        }
        site = "plr-embed";
        lrupd_seq(seqs);
      }
      (void)maxparts;
      std::vector<TruncItem> tr;
      for (size_t i : bi) {
        const int a = abs[i].first, b = abs[i].second;
        tr.push_back(lritem(out[i].p.p, out[i].q.p, nr(a), nr(b), const_cast<int*>(out[i].p.cols.p),
                            nullptr, 0, TCAP, nullptr, nullptr, 0, 0, 1.0, TCAP));
      }
      site = "plr-final";
      lrupd_ws(tr);
    }
    join(psecs);
    ar.release(mk);
    return out;
  }

  // --------------------------------------------------------- sub_product -
  // C -= A diag(d_K) B^T (hfactor.cpp:236-285)
  // Case 5 of the reference (C, A, B all branches) only recurses over
  // (kk, ii, jj); flatten it into the ordered list of terminal terms.
  void collect_terms(const Trip& t, std::vector<Trip>& out) {
    const int C = t.c, a = t.a, b = t.b;
    if (kind(a) == BRANCH && kind(b) == BRANCH && kind(C) == BRANCH) {
      for (int kk = 0; kk < N(a).kc; ++kk)
        for (int ii = 0; ii < N(a).kr; ++ii)
          for (int jj = 0; jj < N(b).kr; ++jj) {
            const int tg = kid(C, ii, jj);
            if (tg < 0) continue;  // implied upper mirror
            collect_terms(Trip{tg, kid(a, ii, kk), kid(b, jj, kk)}, out);
          }
      return;
    }
    out.push_back(t);
  }

  double term_bytes(const Trip& t) const {
    const int a = t.a, b = t.b;
    double d;
    if (kind(a) == LOWRANK)
      d = (double)(nr(b) + nc(a)) * LF(a).cap;
    else if (kind(b) == LOWRANK)
      d = (double)(nr(a) + nc(b)) * LF(b).cap;
    else if (kind(a) == DENSE)
      d = (double)nr(a) * nc(a) + (double)nr(b) * nc(b) + (double)nc(b) * nc(b);
    else if (kind(b) == DENSE)
      d = (double)nc(b) * nr(b) + (double)nr(a) * nr(b) + (double)nr(b) * nr(b);
    else
      d = 3.0 * (nr(a) + nr(b)) * TCAP;
    return 8.0 * d;
  }

  // sub_product for independent targets, two-phase: every product of the
  // flattened term list is computed in parallel (they only read A, B), then the
  // adds are applied per target leaf in the reference's order (add_lr rounds).
  void subprod(const std::vector<Trip>& ts) {
    if (ts.empty()) return;
    std::vector<Trip> terms;
    for (const Trip& t : ts) collect_terms(t, terms);
    const double budget = 6e9;
    size_t i0 = 0;
    while (i0 < terms.size()) {
      size_t i1 = i0;
      double bytes = 0;
      while (i1 < terms.size() && (i1 == i0 || (bytes + term_bytes(terms[i1]) < budget && i1 - i0 < 50000)))
        bytes += term_bytes(terms[i1++]);
      subprod_terms(std::vector<Trip>(terms.begin() + i0, terms.begin() + i1));
      i0 = i1;
    }
  }

  void subprod_terms(const std::vector<Trip>& ts) {
    if (ts.empty()) return;
    const size_t mk = ar.mark();
    std::vector<Add> adds;
    std::vector<int> mb;
    std::vector<MV> mx, my;
    std::vector<CopyScaleItem> c;
    std::vector<Trip> brc, leafc;
    for (const Trip& t : ts) {
      const int C = t.c, a = t.a, b = t.b;
      if (kind(a) == LOWRANK) {
        MV va = Vv(a);
        if (ldl) {
          MV s = temp(va.rows, va.cols);
          c.push_back(cpy(va.p, va.ld, s, va.cols, 0, 1.0, dseg(cb(a)), 1));
          va = s;
        }
        MV w = temp(nr(b), va.cols);
        mb.push_back(b);
        mx.push_back(va);
        my.push_back(w);
        adds.push_back(Add{C, Uv(a), w, -1.0, rb(a), rb(b)});
      } else if (kind(b) == LOWRANK) {
        MV vb = Vv(b);
        if (ldl) {
          MV s = temp(vb.rows, vb.cols);
          c.push_back(cpy(vb.p, vb.ld, s, vb.cols, 0, 1.0, dseg(cb(b)), 1));
          vb = s;
        }
        MV w = temp(nr(a), vb.cols);
        mb.push_back(a);
        mx.push_back(vb);
        my.push_back(w);
        adds.push_back(Add{C, w, Uv(b), -1.0, rb(a), rb(b)});
      } else if (kind(a) == DENSE) {
        MV p = temp(nr(a), dimv(nc(a)));
        c.push_back(cpy(LF(a).a, LF(a).m, p, dimv(nc(a)), 0, 1.0, dseg(cb(a)), 3));
        MV q;
        if (kind(b) == DENSE) {
          q = Dv(b);
        } else {
          q = temp(nr(b), dimv(nc(b)));
          MV e = temp(nc(b), dimv(nc(b)));
          CopyScaleItem ei = cpy(nullptr, 0, e, dimv(nc(b)), 0, 1.0, nullptr, 0);
          ei.mode = 0;
          c.push_back(ei);
          mb.push_back(b);
          mx.push_back(e);
          my.push_back(q);
        }
        adds.push_back(Add{C, p, q, -1.0, rb(a), rb(b)});
      } else if (kind(b) == DENSE) {
        MV x = temp(nc(b), dimv(nr(b)));
        c.push_back(cpy(LF(b).a, LF(b).m, x, dimv(nr(b)), 1, 1.0, dseg(cb(b)), 1));
        MV w = temp(nr(a), dimv(nr(b)));
        MV e = temp(nr(b), dimv(nr(b)));
        CopyScaleItem ei = cpy(nullptr, 0, e, dimv(nr(b)), 0, 1.0, nullptr, 0);
        ei.mode = 0;
        c.push_back(ei);
        mb.push_back(a);
        mx.push_back(x);
        my.push_back(w);
        adds.push_back(Add{C, w, e, -1.0, rb(a), rb(b)});
      } else if (kind(C) == BRANCH) {
        brc.push_back(t);
      } else {
        leafc.push_back(t);
      }
    }
    copy(c);
    // the block products (into fresh temporaries) and the leaf-level low-rank
    // products are independent: the former run as a side-stream section
    std::vector<Sec> secs;
    if (!mb.empty()) {
      if (!leafc.empty())
        section(secs, [&] { multiply_into(mb, mx, my); });
      else
        multiply_into(mb, mx, my);
    }
    if (!leafc.empty()) {
      std::vector<std::pair<int, int>> ab;
      for (const Trip& t : leafc) ab.push_back({t.a, t.b});
      std::vector<Pair> pr = product_lr(ab);
      for (size_t i = 0; i < leafc.size(); ++i)
        adds.push_back(Add{leafc[i].c, pr[i].p, pr[i].q, -1.0, rb(leafc[i].a), rb(leafc[i].b)});
    }
    join(secs);
    // restore the reference order of the terms (leafc terms were appended last)
    std::vector<Add> ordered;
    ordered.reserve(adds.size());
    {
      size_t ia = 0, il = adds.size() - leafc.size();
      for (const Trip& t : ts) {
        const bool is_leafc = !(kind(t.a) == LOWRANK || kind(t.b) == LOWRANK || kind(t.a) == DENSE ||
                                kind(t.b) == DENSE);
        ordered.push_back(is_leafc ? adds[il++] : adds[ia++]);
      }
    }
    (void)brc;
    site = "addlr";
    add_lr(ordered);
    ar.release(mk);
  }

  // --------------------------------------------------------- factor_diag -
  void factor_diag(int a) {
    if (kind(a) == DENSE) {
      const LeafDev& l = LF(a);
      A(l.a, 1);
      run("leaf", [&](cudaStream_t s) { launch_leaf_factor(l.a, l.m, rb(a), ldl ? 1 : 0, F.d_d, -1.0, F.d_status, s); });
      stat(S_LEAF, 1);
      return;
    }
    factor_diag(kid(a, 0, 0));
    trsm({kid(a, 1, 0)}, kid(a, 0, 0));
    subprod({Trip{kid(a, 1, 1), kid(a, 1, 0), kid(a, 1, 0)}});
    factor_diag(kid(a, 1, 1));
  }
};

// ------------------------------------------------------ solve schedules ---
// Diagonal-leaf triangular solve: the CTA stages L (b x b) and x in shared
// memory with coalesced loads, then one warp runs the substitution on-chip.
__global__ void k_trsv_leaf_smem(const double* __restrict__ Lg, int b, double* __restrict__ xg,
                                 int trans) {
  extern __shared__ double sm[];
  double* L = sm;
  double* x = sm + (size_t)b * b;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) L[e] = Lg[e];
  for (int e = threadIdx.x; e < b; e += blockDim.x) x[e] = xg[e];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (!trans) {
      for (int j = 0; j < b; ++j) {
        const double xj = x[j] / L[(size_t)j * b + j];
        __syncwarp();
        if (lane == 0) x[j] = xj;
        for (int i = j + 1 + lane; i < b; i += 32) x[i] -= L[(size_t)j * b + i] * xj;
        __syncwarp();
      }
    } else {
      for (int j = b - 1; j >= 0; --j) {
        double s = 0.0;
        for (int i = j + 1 + lane; i < b; i += 32) s += L[(size_t)j * b + i] * x[i];
        s = warp_sum(s);
        if (lane == 0) x[j] = (x[j] - s) / L[(size_t)j * b + j];
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b; e += blockDim.x) xg[e] = x[e];
}

__global__ void k_trsv_leaf(const double* __restrict__ L, int b, double* __restrict__ x, int trans) {
  // one warp; x has b entries (tree-order segment)
  const int lane = threadIdx.x;
  if (!trans) {
    for (int j = 0; j < b; ++j) {
      const double xj = x[j] / L[(size_t)j * b + j];
      __syncwarp();
      if (lane == 0) x[j] = xj;
      for (int i = j + 1 + lane; i < b; i += 32) x[i] -= L[(size_t)j * b + i] * xj;
      __syncwarp();
    }
  } else {
    for (int j = b - 1; j >= 0; --j) {
      double s = 0.0;
      for (int i = j + 1 + lane; i < b; i += 32) s += L[(size_t)j * b + i] * x[i];
      s = warp_sum(s);
      if (lane == 0) x[j] = (x[j] - s) / L[(size_t)j * b + j];
      __syncwarp();
    }
  }
}

struct CloneItem {
  const double* src;
  double* dst;
  size_t count;
};
__global__ void k_clone(const CloneItem* __restrict__ items) {
  const CloneItem it = items[blockIdx.x];
  for (size_t i = threadIdx.x; i < it.count; i += blockDim.x) it.dst[i] = it.src[i];
}

static void launch_trsv(const double* L, int b, double* x, int trans, cudaStream_t st) {
  const size_t bytes = ((size_t)b * b + b) * 8;
  if (bytes <= 200 * 1024) {
    static bool configured = false;
    if (!configured) {
      HMGP_CUDA(cudaFuncSetAttribute(k_trsv_leaf_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
      configured = true;
    }
    k_trsv_leaf_smem<<<1, 256, bytes, st>>>(L, b, x, trans);
  } else {
    k_trsv_leaf<<<1, 32, 0, st>>>(L, b, x, trans);
  }
  HMGP_LAUNCH_CHECK();
}

struct SolveBlk {
  int leaf;
  int r0, c0;
};

// y[rows] -= B x[cols]  (trans = 0)   or   y[cols] -= B^T x[rows]  (trans = 1)
__global__ void k_solve_apply(const SolveBlk* __restrict__ blks, const LeafDev* __restrict__ lf,
                              const int* __restrict__ rank, double* __restrict__ v, int trans) {
  const SolveBlk sb = blks[blockIdx.x];
  const LeafDev L = lf[sb.leaf];
  __shared__ double t[1024];
  const int in0 = trans ? sb.r0 : sb.c0, out0 = trans ? sb.c0 : sb.r0;
  if (L.kind == DENSE) {
    if (!trans) {
      for (int i = threadIdx.x; i < L.m; i += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < L.n; ++j) s += L.a[(size_t)j * L.m + i] * v[in0 + j];
        atomicAdd(&v[out0 + i], -s);
      }
    } else {
      for (int j = threadIdx.x; j < L.n; j += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < L.m; ++i) s += L.a[(size_t)j * L.m + i] * v[in0 + i];
        atomicAdd(&v[out0 + j], -s);
      }
    }
    return;
  }
  const int r = rank[sb.leaf];
  if (r <= 0) return;
  const double* A = trans ? L.a : L.b;  // contract over the input side
  const double* Bm = trans ? L.b : L.a;
  const int nin = trans ? L.m : L.n, nout = trans ? L.n : L.m;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int l = w; l < r; l += nw) {
    double s = 0.0;
    for (int j = lane; j < nin; j += 32) s += A[(size_t)l * nin + j] * v[in0 + j];
    s = warp_sum(s);
    if (lane == 0) t[l] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nout; i += blockDim.x) {
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += Bm[(size_t)l * nout + i] * t[l];
    atomicAdd(&v[out0 + i], -s);
  }
}

__global__ void k_gather(const double* __restrict__ src, const int* __restrict__ perm, int n,
                         double* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = src[perm[k]];
}
__global__ void k_scatter(const double* __restrict__ src, const int* __restrict__ perm, int n,
                          double* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[perm[k]] = src[k];
}
__global__ void k_div(double* __restrict__ v, const double* __restrict__ d, int n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) v[k] /= d[k];
}

// deterministic two-pass reductions: sum v^2/d (ldl) or v^2; sum log d
__global__ void k_reduce_partial(const double* __restrict__ v, const double* __restrict__ d, int n,
                                 int mode, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    if (mode == 0)
      s += v[k] * v[k];
    else if (mode == 1)
      s += v[k] * v[k] / d[k];
    else
      s += log(d[k]);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_reduce_final(const double* __restrict__ part, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += part[k];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}
__global__ void k_count_nonpos(const double* __restrict__ d, int n, int* out) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    if (!(d[k] > 0.0)) atomicAdd(out, 1);
}
// Cholesky: diag_ = L_ii of dense diagonal leaves (hfactor.cpp:302-310)
__global__ void k_collect_diag(const LeafDev* __restrict__ lf, const int* __restrict__ leaves,
                               const int* __restrict__ base, int count, double* __restrict__ d) {
  const int t = blockIdx.x;
  if (t >= count) return;
  const LeafDev L = lf[leaves[t]];
  for (int i = threadIdx.x; i < L.m; i += blockDim.x) d[base[t] + i] = L.a[(size_t)i * L.m + i];
}

// ------------------------------------------------- persistent H-solves ---
// One cooperative launch per sweep (K10).  Step t of the column sweep: CTA 0
// solves diagonal leaf t on-chip, grid barrier, then every block of the step
// (the blocks whose column range ends in leaf t for the forward sweep, whose
// row range starts in leaf t for the backward one) is applied by the whole
// grid: dense blocks and small low-rank blocks one CTA each, big low-rank
// blocks split into 2048-row chunks (phase A: V^T x partials per input chunk,
// barrier, phase B: y -= U (sum of partials, fixed order) per output chunk).
// Blocks of one step write disjoint rows (they share the column range's end /
// row range's start, so the lower-triangle partition makes their outputs
// disjoint), so no atomics are needed and the result is deterministic.
struct SUnit {
  int leaf;
  int kind;       // 0 dense, 1 small low-rank, 2 big phase A, 3 big phase B
  int in0, out0;  // v offsets of the block's input / output ranges
  int a0, a1;     // chunk of input (kind 2) or output (kind 3) rows, block-local
  int p0, p1;     // kind 2: partial slot p0; kind 3: slots [p0, p1)
};
struct SStep {
  int dleaf, base;
  int u2b, u2e, u3b, u3e;
};
constexpr int kSolveChunk = 512;  // low-rank blocks taller than this are cut over several CTAs
__device__ int d_solve_stats_on;
__device__ unsigned long long d_solve_cyc[2][6];
__device__ unsigned long long d_solve_sub[4];  // (stats) CTA 0: descriptor loads, prefetch wait, substitution, prefetch issue
constexpr int kSolveThreads = 256;

struct SolvePlan {
  std::vector<SUnit> units;
  std::vector<SStep> steps;
  int slots = 0, stride = 0;
};

static SolvePlan build_solve_plan(const Factor& F, const std::vector<SolveBlk>& flat,
                                  const std::vector<int>& off, bool trans) {
  SolvePlan P;
  const int nd = (int)F.diag_leaf.size();
  for (const SolveBlk& b : flat) {
    const LeafDev& l = F.leaf[b.leaf];
    if (l.kind != DENSE) P.stride = std::max(P.stride, l.cap);
  }
  P.stride = std::max(P.stride, 1);
  std::vector<SUnit> u3;
  for (int t = 0; t < nd; ++t) {
    SStep s{};
    s.dleaf = F.diag_leaf[t];
    s.base = F.diag_base[t];
    s.u2b = (int)P.units.size();
    u3.clear();
    for (int k = off[t]; k < off[t + 1]; ++k) {
      const SolveBlk& b = flat[k];
      const LeafDev& l = F.leaf[b.leaf];
      const int in0 = trans ? b.r0 : b.c0, out0 = trans ? b.c0 : b.r0;
      const int nin = trans ? l.m : l.n, nout = trans ? l.n : l.m;
      if (l.kind == DENSE) {
        P.units.push_back(SUnit{b.leaf, 0, in0, out0, 0, 0, 0, 0});
      } else if (std::max(nin, nout) <= kSolveChunk) {
        P.units.push_back(SUnit{b.leaf, 1, in0, out0, 0, 0, 0, 0});
      } else {
        const int p0 = P.slots;
        for (int a = 0; a < nin; a += kSolveChunk)
          P.units.push_back(SUnit{b.leaf, 2, in0, out0, a, std::min(nin, a + kSolveChunk), P.slots++, 0});
        for (int a = 0; a < nout; a += kSolveChunk)
          u3.push_back(SUnit{b.leaf, 3, in0, out0, a, std::min(nout, a + kSolveChunk), p0, P.slots});
      }
    }
    s.u2e = (int)P.units.size();
    s.u3b = s.u2e;
    P.units.insert(P.units.end(), u3.begin(), u3.end());
    s.u3e = (int)P.units.size();
    P.steps.push_back(s);
  }
  return P;
}

__device__ void solve_unit(const SUnit& u, const LeafDev* __restrict__ lf, const int* __restrict__ rank,
                           double* __restrict__ v, double* __restrict__ part, int stride, int trans,
                           double* sT) {
  const LeafDev L = lf[u.leaf];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (u.kind == 0) {
    if (!trans && L.n <= 1024 - (int)blockDim.x) {  // y[out0 + i] -= sum_j D(i, j) x[in0 + j]
      for (int j = threadIdx.x; j < L.n; j += blockDim.x) sT[j] = v[u.in0 + j];
      __syncthreads();
      const int split = (2 * L.m <= (int)blockDim.x) ? 2 : 1;
      const int half = (L.n + split - 1) / split;
      double* red = sT + 1024 - blockDim.x;  // scratch behind the x segment (n <= 1024 - blockDim)
      for (int i0 = 0; i0 < L.m; i0 += blockDim.x / split) {
        const int i = i0 + (int)threadIdx.x % (blockDim.x / split), h = (int)threadIdx.x / (blockDim.x / split);
        double s = 0.0;
        if (i < L.m) {
          const int j1 = min(L.n, (h + 1) * half);
#pragma unroll 8
          for (int j = h * half; j < j1; ++j) s += L.a[(size_t)j * L.m + i] * sT[j];
        }
        if (split == 2) {
          if (h == 1) red[threadIdx.x] = s;
          __syncthreads();
          if (h == 0 && i < L.m) v[u.out0 + i] -= s + red[threadIdx.x + blockDim.x / 2];
          __syncthreads();
        } else if (i < L.m) {
          v[u.out0 + i] -= s;
        }
      }
    } else if (!trans) {
      for (int i = threadIdx.x; i < L.m; i += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < L.n; ++j) s += L.a[(size_t)j * L.m + i] * v[u.in0 + j];
        v[u.out0 + i] -= s;
      }
    } else {  // y[out0 + j] -= sum_i D(i, j) x[in0 + i]
      for (int j = w; j < L.n; j += nw) {
        double s = 0.0;
        for (int i = lane; i < L.m; i += 32) s += L.a[(size_t)j * L.m + i] * v[u.in0 + i];
        s = warp_sum(s);
        if (lane == 0) v[u.out0 + j] -= s;
      }
    }
    return;
  }
  const int r = rank[u.leaf];
  if (r <= 0) return;
  const double* A = trans ? L.a : L.b;  // contracted with the input
  const double* Bm = trans ? L.b : L.a;
  const int nin = trans ? L.m : L.n, nout = trans ? L.n : L.m;
  if (u.kind == 1 || u.kind == 2) {
    const int j0 = u.kind == 1 ? 0 : u.a0, j1 = u.kind == 1 ? nin : u.a1;
    for (int l = w; l < r; l += nw) {
      double s = 0.0;
#pragma unroll 4
      for (int j = j0 + lane; j < j1; j += 32) s += A[(size_t)l * nin + j] * v[u.in0 + j];
      s = warp_sum(s);
      if (lane == 0) {
        if (u.kind == 1)
          sT[l] = s;
        else
          part[(size_t)u.p0 * stride + l] = s;
      }
    }
    if (u.kind == 2) return;
    __syncthreads();
    for (int i = threadIdx.x; i < nout; i += blockDim.x) {
      double s = 0.0;
#pragma unroll 4
      for (int l = 0; l < r; ++l) s += Bm[(size_t)l * nout + i] * sT[l];
      v[u.out0 + i] -= s;
    }
    return;
  }
  // kind 3: T = sum of the block's partials (fixed order), then its output chunk
  for (int l = threadIdx.x; l < r; l += blockDim.x) {
    double s = 0.0;
    for (int p = u.p0; p < u.p1; ++p) s += part[(size_t)p * stride + l];
    sT[l] = s;
  }
  __syncthreads();
  for (int i = u.a0 + threadIdx.x; i < u.a1; i += blockDim.x) {
    double s = 0.0;
    for (int l = 0; l < r; ++l) s += Bm[(size_t)l * nout + i] * sT[l];
    v[u.out0 + i] -= s;
  }
}

// Diagonal-leaf substitution by one CTA (L staged in shared memory when it
// fits).  Blocked by 32: warp 0 solves a 32-row diagonal block with the values
// in registers (one shuffle broadcast per column, reciprocal diagonal), then all
// threads apply the block to the remaining rows (a small mat-vec).
__device__ void solve_trsv_cta(const double* __restrict__ Lg, int b, double* __restrict__ xg, int trans,
                               double* sm, bool staged, int smem_b) {
  // L comes from shared memory when the leaf was prefetched there (cp.async issued
  // one step ahead, see k_solve_sweep: a single SM pulling 128 KB synchronously
  // from HBM was the 18 us that dominated a step), else straight from global
  // memory.  Warp 0 holds the 32 x 32 diagonal block of the current sub-step in
  // registers (lane = row) and runs the substitution on registers + shuffles; all
  // threads then apply the block column (forward) / block row (backward) to the
  // remaining unknowns, coalesced over rows.
  const double* Lsrc = staged ? sm : Lg;
  double* x = sm + (size_t)smem_b * smem_b;
  double* inv = x + smem_b;
  if (!staged) {
    x = sm;
    inv = x + b;
  }
  for (int e = threadIdx.x; e < b; e += blockDim.x) {
    x[e] = xg[e];
    inv[e] = 1.0 / Lsrc[(size_t)e * b + e];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (!trans) {
    for (int jb = 0; jb < b; jb += 32) {
      const int nb = min(32, b - jb);
      if (threadIdx.x < 32) {
        // row (jb + lane) of the diagonal block, pre-scaled by 1 / L(row, row): the
        // dependent chain of a step is then one shuffle and one FMA (an FP64 op costs
        // ~40 cycles of latency here), x_j = y_j / L_jj - sum_k (L_jk / L_jj) x_k
        const double li = lane < nb ? inv[jb + lane] : 0.0;
        double lr[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          lr[j] = (j < nb && lane < nb && lane > j) ? Lsrc[(size_t)(jb + j) * b + jb + lane] * li : 0.0;
        double xi = lane < nb ? x[jb + lane] * li : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < nb) {
            const double xj = __shfl_sync(0xffffffffu, xi, j);
            xi -= lr[j] * xj;  // lr[j] = 0 for lane <= j
          }
        }
        if (lane < nb) x[jb + lane] = xi;
      }
      __syncthreads();
      for (int i = jb + nb + threadIdx.x; i < b; i += blockDim.x) {
        double s4[4] = {0.0, 0.0, 0.0, 0.0};  // four independent chains
        for (int j = 0; j < nb; j += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j + u < nb) s4[u] += Lsrc[(size_t)(jb + j + u) * b + i] * x[jb + j + u];
        }
        x[i] -= (s4[0] + s4[1]) + (s4[2] + s4[3]);
      }
      __syncthreads();
    }
  } else {
    const int nblk = (b + 31) / 32;
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = nblk - 1; q >= 0; --q) {
      const int jb = q * 32, nb = min(32, b - jb);
      // x_J -= L(I, J)^T x_I for the rows I below the block (already solved):
      // a warp per column j of the block, lanes over the rows i (coalesced)
      for (int j = jb + w; j < jb + nb; j += nw) {
        double s = 0.0;
        for (int i = jb + nb + lane; i < b; i += 32) s += Lsrc[(size_t)j * b + i] * x[i];
        s = warp_sum(s);
        if (lane == 0) x[j] -= s;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        // column (jb + lane) of the diagonal block, pre-scaled by 1 / L(lane, lane)
        const double li = lane < nb ? inv[jb + lane] : 0.0;
        double lc[32];  // lc[i] = L(jb + i, jb + lane) / L(jb + lane, jb + lane)
#pragma unroll
        for (int i = 0; i < 32; ++i)
          lc[i] = (i < nb && lane < nb && i > lane) ? Lsrc[(size_t)(jb + lane) * b + jb + i] * li : 0.0;
        double xi = lane < nb ? x[jb + lane] * li : 0.0;
#pragma unroll
        for (int j = 31; j >= 0; --j) {
          if (j < nb) {
            const double xj = __shfl_sync(0xffffffffu, xi, j);
            xi -= lc[j] * xj;  // 0 unless j > lane
          }
        }
        if (lane < nb) x[jb + lane] = xi;
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < b; e += blockDim.x) xg[e] = x[e];
  __syncthreads();
}

// asynchronous copy of a diagonal leaf (b x b doubles) into shared memory: 8-byte
// cp.async per element (no alignment requirement beyond the double's), all threads
__device__ __forceinline__ void solve_prefetch_leaf(const double* __restrict__ Lg, int b, double* sm) {
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const int n = b * b;
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(base + 8u * (unsigned)e), "l"(Lg + e) : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void solve_prefetch_wait() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
}

__global__ void __launch_bounds__(kSolveThreads) k_solve_sweep(const SStep* __restrict__ steps, int nsteps,
                                                              const SUnit* __restrict__ units,
                                                              const LeafDev* __restrict__ lf,
                                                              const int* __restrict__ rank, double* v,
                                                              double* part, int stride, int trans,
                                                              int smem_b) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double ssm[];
  __shared__ double sT[1024];
  long long tc = clock64(), acc[6] = {0, 0, 0, 0, 0, 0};
  auto tick = [&](int i) {
    const long long now = clock64();
    acc[i] += now - tc;
    tc = now;
  };
  bool prefetched = false;
  // with more than one CTA, CTA 0 only runs the diagonal chain; the others share the blocks
  const bool solo = gridDim.x > 1;
  const int wid = solo ? (int)blockIdx.x - 1 : (int)blockIdx.x, nwk = solo ? (int)gridDim.x - 1 : (int)gridDim.x;
  for (int s = 0; s < nsteps; ++s) {
    const SStep st = steps[trans ? nsteps - 1 - s : s];
    if (blockIdx.x == 0) {
      long long ts = clock64();
      auto sub = [&](int i) {
        if (!d_solve_stats_on || threadIdx.x != 0) return;
        const long long now = clock64();
        atomicAdd(&d_solve_sub[i], (unsigned long long)(now - ts));
        ts = now;
      };
      const LeafDev d = lf[st.dleaf];
      const bool fits = d.m <= smem_b;
      sub(0);
      if (fits) {
        if (!prefetched) solve_prefetch_leaf(d.a, d.m, ssm);  // first step (or after a leaf that did not fit)
        solve_prefetch_wait();
      }
      sub(1);
      solve_trsv_cta(d.a, d.m, v + st.base, trans, ssm, fits, smem_b);
      sub(2);
      prefetched = false;
      if (!solo && s + 1 < nsteps) {  // (one-CTA grid: nobody else to wait for, issue right away)
        const LeafDev nx = lf[steps[trans ? nsteps - 2 - s : s + 1].dleaf];
        if (nx.m <= smem_b) {
          solve_prefetch_leaf(nx.a, nx.m, ssm);
          prefetched = true;
        }
      }
      sub(3);
    }
    if (!(solo && blockIdx.x == 0)) {
      // while CTA 0 runs the substitution, the other CTAs pull the payload of the
      // blocks they will apply in this step into L2 (their inputs are not ready yet)
      for (int k = st.u2b + wid; k < st.u2e; k += nwk) {
        const SUnit u = units[k];
        const LeafDev L = lf[u.leaf];
        const size_t ba = L.kind == DENSE ? (size_t)L.m * L.n * 8 : (size_t)L.m * max(rank[u.leaf], 0) * 8;
        const size_t bb = L.kind == DENSE ? 0 : (size_t)L.n * max(rank[u.leaf], 0) * 8;
        const char* pa = reinterpret_cast<const char*>(L.a);
        const char* pb = reinterpret_cast<const char*>(L.b);
        for (size_t o = (size_t)threadIdx.x * 128; o < ba; o += (size_t)blockDim.x * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + o));
        for (size_t o = (size_t)threadIdx.x * 128; o < bb; o += (size_t)blockDim.x * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + o));
      }
    }
    tick(0);
    grid.sync();
    tick(1);
    if (solo && blockIdx.x == 0) {
      // CTA 0 is the diagonal chain: while the other CTAs apply this step's blocks it
      // streams the next diagonal leaf into shared memory (16 K cp.async, ~3.6 us of
      // issue that used to sit between the substitution and the barrier)
      if (s + 1 < nsteps) {
        const LeafDev nx = lf[steps[trans ? nsteps - 2 - s : s + 1].dleaf];
        if (nx.m <= smem_b) {
          solve_prefetch_leaf(nx.a, nx.m, ssm);
          prefetched = true;
        }
      }
    } else {
      for (int k = st.u2b + wid; k < st.u2e; k += nwk) {
        solve_unit(units[k], lf, rank, v, part, stride, trans, sT);
        __syncthreads();
      }
    }
    tick(2);
    if (st.u3e > st.u3b) {
      grid.sync();
      tick(3);
      if (!(solo && blockIdx.x == 0))
        for (int k = st.u3b + wid; k < st.u3e; k += nwk) {
          solve_unit(units[k], lf, rank, v, part, stride, trans, sT);
          __syncthreads();
        }
      tick(4);
    }
    grid.sync();
    tick(5);
  }
  if (d_solve_stats_on && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 1))
    for (int i = 0; i < 6; ++i) atomicAdd(&d_solve_cyc[blockIdx.x][i], (unsigned long long)acc[i]);
}

static void solve_sweep(const Factor& F, double* v, bool trans, cudaStream_t st) {
  const int nsteps = (int)F.diag_leaf.size();
  if (nsteps == 0) return;
  static int grid = 0, smem_b = 0;
  static size_t smem = 0;
  if (!grid) {
    int dev = 0, sms = 0, optin = 0;
    HMGP_CUDA(cudaGetDevice(&dev));
    HMGP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HMGP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    smem = std::min<size_t>((size_t)optin - 8192 - 1024, (size_t)200 * 1024);
    int b = 1;
    while ((size_t)(b + 1) * (b + 1) * 8 + 2 * (size_t)(b + 1) * 8 <= smem) ++b;
    smem_b = b;
    HMGP_CUDA(cudaFuncSetAttribute(k_solve_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    HMGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_solve_sweep, kSolveThreads, smem));
    grid = std::max(1, per) * sms;
    // fewer CTAs make the grid-wide barriers cheaper; a step has few units
    if (const char* e = getenv("HMGP_SOLVE_GRID")) grid = std::max(1, std::min(grid, atoi(e)));
  }
  const SStep* d_steps = static_cast<const SStep*>(trans ? F.d_bsteps : F.d_fsteps);
  const SUnit* d_units = static_cast<const SUnit*>(trans ? F.d_bunits : F.d_funits);
  int ns = nsteps, tr = trans ? 1 : 0, stride = F.solve_stride, sb = smem_b;
  double* part = F.d_part;
  const LeafDev* lf = F.d_leaf;
  const int* rk = F.d_rank;
  void* args[] = {(void*)&d_steps, &ns, (void*)&d_units, (void*)&lf, (void*)&rk, &v, &part, &stride, &tr, &sb};
  const bool stats = getenv("HMGP_SOLVE_STATS") != nullptr;
  if (stats) {
    const int one = 1;
    static unsigned long long z[2][6] = {};
    HMGP_CUDA(cudaMemcpyToSymbol(d_solve_stats_on, &one, 4));
    HMGP_CUDA(cudaMemcpyToSymbol(d_solve_cyc, z, sizeof(z)));
  }
  HMGP_CUDA(cudaLaunchCooperativeKernel((const void*)k_solve_sweep, dim3(grid), dim3(kSolveThreads), args, smem, st));
  if (stats) {
    unsigned long long c[2][6];
    HMGP_CUDA(cudaStreamSynchronize(st));
    HMGP_CUDA(cudaMemcpyFromSymbol(c, d_solve_cyc, sizeof(c)));
    {
      unsigned long long sb[4], zz[4] = {0, 0, 0, 0};
      HMGP_CUDA(cudaMemcpyFromSymbol(sb, d_solve_sub, sizeof(sb)));
      HMGP_CUDA(cudaMemcpyToSymbol(d_solve_sub, zz, sizeof(zz)));
      fprintf(stderr, "[hmgp] solve sweep CTA 0 (ms): descriptor loads %.2f prefetch wait %.2f substitution %.2f prefetch issue %.2f\n",
              sb[0] / 1.965e6, sb[1] / 1.965e6, sb[2] / 1.965e6, sb[3] / 1.965e6);
    }
    for (int b = 0; b < 2; ++b)
      fprintf(stderr,
              "[hmgp] solve sweep (%s, CTA %d of %d, ms @1.965GHz): trsv %.2f sync %.2f units %.2f sync %.2f "
              "units-B %.2f sync %.2f\n",
              trans ? "bwd" : "fwd", b, grid, c[b][0] / 1.965e6, c[b][1] / 1.965e6, c[b][2] / 1.965e6,
              c[b][3] / 1.965e6, c[b][4] / 1.965e6, c[b][5] / 1.965e6);
  }
}

// ------------------------------------------------------------ Factor API --
Factor::~Factor() {
  if (!borrowed) {  // (a graph-replayed factor borrows these from the thread's graph cache)
    dev_free(pool);
    dev_free(d_leaf);
    dev_free(d_rank);
    dev_free(d_compact);
    dev_free(d_d);
    dev_free(d_status);
  }
  dev_free(d_fwd);
  dev_free(d_bwd);
  dev_free(d_work);
  dev_free(d_fsteps);
  dev_free(d_funits);
  dev_free(d_bsteps);
  dev_free(d_bunits);
  dev_free(d_part);
}

// Capacities (TCAP, low-rank column growth) of the last factorization that
// succeeded on this thread, keyed by the block structure: the next evaluation on
// the same structure (a θ-sweep, repeated L(θ)) starts there instead of repeating
// a failed attempt.  Capacities never change results, only memory and retries.
struct CapMemo {
  int n = -1, dim = 0, leaves = -1, tcap = 256, grow = 1;
};
// shared by the host threads (θ-batch workers start from what the caller's first
// θ found); read / written under g_memo_mu
static CapMemo g_cap_memo;
static std::mutex g_memo_mu;
static CapMemo memo_get() {
  std::lock_guard<std::mutex> lk(g_memo_mu);
  return g_cap_memo;
}
static void memo_set(const CapMemo& m) {
  std::lock_guard<std::mutex> lk(g_memo_mu);
  g_cap_memo = m;
}

// ------------------------------------------------ captured factorization ---
// The host walk of the factorization depends only on the block structure, the
// capacities and the configuration — never on θ (ranks stay on the device, the
// pivot clamp is read from the status block).  For the ephemeral factor of an
// L(θ) / predict call the walk is therefore captured ONCE per host thread into
// a CUDA graph over buffers the thread keeps (factor pool at fixed capacities,
// rank arrays, arena, descriptor store), and every later evaluation on the same
// structure clones its H-matrix into those buffers and replays the graph: one
// cudaGraphLaunch instead of ~85 000 launches + ~99 000 descriptor copies at C3.
// Same kernels, same arguments, same order => bit-identical results.  A θ whose
// assembled ranks outgrow the captured capacities re-captures with larger ones;
// a device-detected overflow falls back to the stream path with its redo loop.
thread_local bool t_graph_ok = false;

struct GraphCache {
  bool valid = false;
  uint64_t key = 0;
  int tcap = 0, grow = 0, L = 0, n = 0;
  bool ldl = false, one_stream = false;
  double eps = 0.0;
  std::vector<int> caps;
  std::vector<size_t> off;
  size_t total = 0;
  double* pool = nullptr;
  LeafDev* d_leaf = nullptr;
  int* d_rank = nullptr;
  int* d_compact = nullptr;
  double* d_d = nullptr;
  LeafFactorStatus* d_status = nullptr;
  CloneItem* d_ci = nullptr;
  size_t ci_cap = 0;
  std::vector<CloneItem> ci_host;
  LeafFactorStatus s0{};
  int* d_err = nullptr;
  char* arena_base = nullptr;
  size_t arena_cap = 0, arena_peak = 0;
  cudaGraphExec_t exec = nullptr;
  size_t nodes = 0;
  long long replays = 0;
  DescStore desc;
  size_t pool_alloc = 0;  // doubles allocated for pool (>= total: slack absorbs small regrowth)
  void drop_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    desc.rewind();
    valid = false;
  }
  void free_buffers() {
    drop_graph();
    desc.clear();
    pool_alloc = 0;
    cudaFree(pool);
    cudaFree(d_leaf);
    cudaFree(d_rank);
    cudaFree(d_compact);
    cudaFree(d_d);
    cudaFree(d_status);
    cudaFree(d_ci);
    pool = nullptr;
    d_leaf = nullptr;
    d_rank = d_compact = nullptr;
    d_d = nullptr;
    d_status = nullptr;
    d_ci = nullptr;
    ci_cap = 0;
    total = 0;
    L = n = 0;
    key = 0;
    caps.clear();
  }
  ~GraphCache() { free_buffers(); }
};
static thread_local GraphCache t_gc;
void drop_thread_graph() { t_gc.free_buffers(); }

// High-water capacities per block structure, shared by the host threads: a capture
// on any thread starts from the largest capacities any θ has needed so far, so a
// sweep over θ with different ranks settles after the first few captures instead
// of every worker re-capturing each time it meets a new record.
static std::mutex g_caps_mu;
static uint64_t g_caps_key = 0;
static std::vector<int> g_caps_high;
static void caps_merge(uint64_t key, std::vector<int>& caps) {  // caps <- max(caps, high); high <- caps
  std::lock_guard<std::mutex> lk(g_caps_mu);
  if (g_caps_key != key || g_caps_high.size() != caps.size()) {
    g_caps_key = key;
    g_caps_high = caps;
    return;
  }
  for (size_t k = 0; k < caps.size(); ++k) {
    caps[k] = std::max(caps[k], g_caps_high[k]);
    g_caps_high[k] = caps[k];
  }
}

static uint64_t structure_key(const HMat& H) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    h ^= v;
    h *= 1099511628211ull;
  };
  const Geometry& G = *H.g;
  mix((uint64_t)G.n);
  mix((uint64_t)G.dim);
  mix(H.leaf.size());
  for (const LeafDev& l : H.leaf) mix(((uint64_t)l.m << 34) ^ ((uint64_t)l.n << 4) ^ (uint64_t)l.kind);
  for (const HNode& nd : H.nodes) mix(((uint64_t)(uint32_t)nd.row << 32) ^ ((uint64_t)(uint32_t)nd.col << 2) ^ (uint64_t)nd.kind);
  return h;
}

// Returns 0 when the factorization ran (captured or replayed) without a capacity
// overflow; 1: could not capture (take the stream path at the same capacities);
// 2: overflow detected on device (take the stream path at doubled capacities).
static int factorize_graph(Factor& F, HMat& H, cudaStream_t st, size_t arena_bytes, int tcap, int grow) {
  GraphCache& gc = t_gc;
  const Geometry& G = *H.g;
  const int L = (int)H.leaf.size();
  const uint64_t key = structure_key(H);
  std::vector<int> need(L, 0);
  bool fits = gc.valid && gc.key == key && gc.tcap == tcap && gc.grow == grow && gc.ldl == F.ldl &&
              gc.eps == F.eps && gc.one_stream == t_one_stream && gc.arena_base == g_arena.base &&
              gc.arena_cap == g_arena.cap && (int)gc.caps.size() == L;
  for (int k = 0; k < L; ++k) {
    const LeafDev& l = H.leaf[k];
    if (l.kind == DENSE) continue;
    need[k] = std::min(std::min(l.m, l.n) + 16, l.cap * grow);
    if (fits && need[k] > gc.caps[k]) fits = false;
  }
  if (getenv("HMGP_TIMING")) {
    int over = 0;
    if ((int)gc.caps.size() == L)
      for (int k = 0; k < L; ++k) over += need[k] > gc.caps[k];
    fprintf(stderr, "[hmgp] graph %s (valid %d key %d caps-over %d arena %d one_stream %d/%d replays %lld)\n",
            fits ? "replay" : "capture", (int)gc.valid, (int)(gc.key == key), over,
            (int)(gc.arena_base == g_arena.base && gc.arena_cap == g_arena.cap), (int)gc.one_stream,
            (int)t_one_stream, gc.replays);
  }
  if (!fits) {
    // new layout: this θ's capacities with slack, never below the previous ones
    const bool same = gc.key == key && (int)gc.caps.size() == L;
    std::vector<int> caps(L, 0);
    for (int k = 0; k < L; ++k) {
      const LeafDev& l = H.leaf[k];
      if (l.kind == DENSE) continue;
      int c = need[k] + need[k] / 4 + 8;
      if (same) c = std::max(c, gc.caps[k]);
      caps[k] = std::min(std::min(l.m, l.n) + 16, c);
    }
    caps_merge(key ^ (uint64_t)grow, caps);
    std::vector<size_t> off(L);
    size_t total = 0;
    for (int k = 0; k < L; ++k) {
      const LeafDev& l = H.leaf[k];
      off[k] = total;
      total += l.kind == DENSE ? (size_t)l.m * l.n : (size_t)(l.m + l.n) * caps[k];
    }
    gc.drop_graph();
    if (total > gc.pool_alloc || !gc.pool) {
      cudaFree(gc.pool);
      gc.pool = nullptr;
      gc.total = gc.pool_alloc = 0;
      const size_t want = total + total / 8;  // slack: the next regrowth usually fits
      if (dev_malloc_plain((void**)&gc.pool, std::max<size_t>(1, want) * 8) == cudaSuccess) {
        gc.pool_alloc = want;
      } else if (dev_malloc_plain((void**)&gc.pool, std::max<size_t>(1, total) * 8) == cudaSuccess) {
        gc.pool_alloc = total;
      } else {
        cudaGetLastError();
        gc.pool = nullptr;
        return 1;
      }
    }
    gc.total = total;
    if (L != gc.L || G.n != gc.n || !gc.d_leaf) {
      cudaFree(gc.d_leaf);
      cudaFree(gc.d_rank);
      cudaFree(gc.d_compact);
      cudaFree(gc.d_d);
      cudaFree(gc.d_status);
      gc.d_leaf = nullptr;
      HMGP_CUDA(dev_malloc_plain((void**)&gc.d_leaf, sizeof(LeafDev) * std::max(L, 1)));
      HMGP_CUDA(dev_malloc_plain((void**)&gc.d_rank, 4 * std::max(L, 1)));
      HMGP_CUDA(dev_malloc_plain((void**)&gc.d_compact, 4 * std::max(L, 1)));
      HMGP_CUDA(dev_malloc_plain((void**)&gc.d_d, 8ull * G.n));
      HMGP_CUDA(dev_malloc_plain((void**)&gc.d_status, sizeof(LeafFactorStatus)));
      gc.L = L;
      gc.n = G.n;
    }
    gc.key = key;
    gc.caps = caps;
    gc.off = off;
    gc.tcap = tcap;
    gc.grow = grow;
    gc.ldl = F.ldl;
    gc.eps = F.eps;
    gc.one_stream = t_one_stream;
  }
  // the factor borrows the cache's buffers
  F.leaf = H.leaf;
  gc.ci_host.clear();
  for (int k = 0; k < L; ++k) {
    LeafDev& l = F.leaf[k];
    if (l.kind != DENSE) l.cap = gc.caps[k];
    l.a = gc.pool + gc.off[k];
    l.b = l.kind == DENSE ? nullptr : l.a + (size_t)l.m * l.cap;
    const LeafDev& sl = H.leaf[k];
    if (l.kind == DENSE) {
      gc.ci_host.push_back(CloneItem{sl.a, l.a, (size_t)l.m * l.n});
    } else if (H.rank_host[k] > 0) {
      gc.ci_host.push_back(CloneItem{sl.a, l.a, (size_t)l.m * H.rank_host[k]});
      gc.ci_host.push_back(CloneItem{sl.b, l.b, (size_t)l.n * H.rank_host[k]});
    }
  }
  F.pool = gc.pool;
  F.d_leaf = gc.d_leaf;
  F.d_rank = gc.d_rank;
  F.d_compact = gc.d_compact;
  F.d_d = gc.d_d;
  F.d_status = gc.d_status;
  F.borrowed = true;
  // per-evaluation state: payload clone (hblock.cpp:17-28, compact_cols = 0), ranks, status
  if (!fits) HMGP_CUDA(cudaMemcpyAsync(gc.d_leaf, F.leaf.data(), sizeof(LeafDev) * L, cudaMemcpyHostToDevice, st));
  if (!gc.ci_host.empty()) {
    if (gc.ci_host.size() > gc.ci_cap) {
      cudaFree(gc.d_ci);
      gc.ci_cap = gc.ci_host.size() + gc.ci_host.size() / 2;
      HMGP_CUDA(dev_malloc_plain((void**)&gc.d_ci, sizeof(CloneItem) * gc.ci_cap));
    }
    HMGP_CUDA(cudaMemcpyAsync(gc.d_ci, gc.ci_host.data(), sizeof(CloneItem) * gc.ci_host.size(),
                              cudaMemcpyHostToDevice, st));
    k_clone<<<(int)gc.ci_host.size(), 256, 0, st>>>(gc.d_ci);
    HMGP_LAUNCH_CHECK();
  }
  HMGP_CUDA(cudaMemcpyAsync(F.d_rank, H.d_rank, 4ull * L, cudaMemcpyDeviceToDevice, st));
  HMGP_CUDA(cudaMemsetAsync(F.d_compact, 0, 4ull * L, st));
  HMGP_CUDA(cudaMemsetAsync(F.d_d, 0, 8ull * G.n, st));
  gc.s0 = LeafFactorStatus{INT_MAX, 0, 0, 0, 0.0, INFINITY, F.clamp_tol};
  HMGP_CUDA(cudaMemcpyAsync(F.d_status, &gc.s0, sizeof(gc.s0), cudaMemcpyHostToDevice, st));
  int err = 0;
  if (fits) {
    HMGP_CUDA(cudaMemsetAsync(gc.d_err, 0, 4, st));
    HMGP_CUDA(cudaGraphLaunch(gc.exec, st));
    g_launches.fetch_add(gc.nodes);
    ++gc.replays;
  } else {
    std::vector<int> lr;
    for (int k = 0; k < L; ++k)
      if (F.leaf[k].kind == LOWRANK) lr.push_back(F.leaf_node[k]);
    cudaGraph_t graph = nullptr;
    bool ok = true;
    try {
      Engine E(F, st, arena_bytes, tcap, false);  // (re)sizes the arena, zeroes d_err on st
      gc.d_err = E.d_err;
      E.sg.store = &gc.desc;
      HMGP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
      try {
        E.factor_diag(0);
        E.compress(lr);  // compress_all (hfactor.cpp:321-328)
      } catch (const Error&) {
        ok = false;  // arena too small for this schedule: the stream path handles it
      }
      const cudaError_t ce = cudaStreamEndCapture(st, &graph);
      E.sg.store = nullptr;
      if (ce != cudaSuccess) {
        cudaGetLastError();
        ok = false;
      }
      gc.arena_peak = E.ar.peak;
    } catch (...) {
      g_stager.store = nullptr;
      if (graph) cudaGraphDestroy(graph);
      gc.drop_graph();
      throw;
    }
    if (ok) {
      gc.desc.finish_upload();
      ok = cudaGraphInstantiate(&gc.exec, graph, 0) == cudaSuccess;
      if (!ok) cudaGetLastError();
    }
    if (ok) {
      size_t nn = 0;
      cudaGraphGetNodes(graph, nullptr, &nn);
      gc.nodes = nn;
    }
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
      gc.drop_graph();
      HMGP_CUDA(cudaStreamSynchronize(st));
      return 1;
    }
    gc.arena_base = g_arena.base;
    gc.arena_cap = g_arena.cap;
    gc.valid = true;
    if (getenv("HMGP_TIMING"))
      fprintf(stderr, "[hmgp] captured factorization: %zu graph nodes, %.1f MB descriptors, arena peak %.2f GB\n",
              gc.nodes, gc.desc.bytes / 1e6, gc.arena_peak / 1e9);
    HMGP_CUDA(cudaGraphLaunch(gc.exec, st));
  }
  phase_mark(PH_FACTOR);
  HMGP_CUDA(cudaMemcpyAsync(&err, gc.d_err, 4, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  F.arena_peak = gc.arena_peak;
  t_last_arena_peak = gc.arena_peak;
  g_work.arena_peak = std::max(g_work.arena_peak, (double)gc.arena_peak);
  g_work.factor_attempts += 1;
  if (err) {  // capacity overflow detected on device: the stream path redoes it with larger capacities
    gc.drop_graph();
    return 2;
  }
  return 0;
}

void factorize(Factor& F, HMat& H, double eps_f, bool ldl, cudaStream_t st, size_t arena_bytes) {
  NvtxRange nvtx_range("hmgp:factorize(K6-K9)");
  const Geometry& G = *H.g;
  F.g = H.g;
  F.ldl = ldl;
  F.eps = eps_f;
  F.nodes = H.nodes;
  F.leaf_node = H.leaf_node;
  const int L = (int)H.leaf.size();
  t_last_pool_bytes = H.pool_doubles * 8;
  F.clamp_tol = 1e-14 * H.max_diag;  // hfactor.cpp:349

  // Temporaries are sized with a width capacity TCAP; a product wider than that
  // is detected on device (error flag) and the factorization is redone with a
  // doubled capacity — results never depend on the capacity that succeeded.
  // A low-rank block whose rank outgrows its column capacity, or a product wider
  // than TCAP, is detected on device; the factorization is then redone with
  // doubled capacities (results do not depend on the capacities that succeed).
  int grow = 1, tcap0 = 256;
  // 3-D admissible blocks carry ranks up to ~256 and their updates outgrow the
  // 2-D starting capacities (C5-shaped n = 262144: one full failed attempt)
  bool start_3d = false;  // heuristic start, dropped if its pool does not fit
  if (G.dim == 3) {
    grow = 2;
    tcap0 = 512;
    start_3d = true;
  }
  // (experiments: HMGP_TCAP / HMGP_GROW force the starting capacities)
  if (const char* e = getenv("HMGP_TCAP")) {
    tcap0 = std::max(64, atoi(e));
    start_3d = false;
  }
  if (const char* e = getenv("HMGP_GROW")) {
    grow = std::max(1, atoi(e));
    start_3d = false;
  }
  const CapMemo memo = memo_get();
  const bool memo_hit = memo.n == G.n && memo.dim == G.dim && memo.leaves == L;
  if (memo_hit) {
    start_3d = false;
    grow = std::max(grow, memo.grow);
    tcap0 = std::max(tcap0, memo.tcap);
  }
  size_t pool_doubles = 0;
  struct OneStreamScope {  // restores t_one_stream when factorize leaves
    bool on = false;
    void engage() {
      on = true;
      t_one_stream = true;
    }
    ~OneStreamScope() {
      if (on) t_one_stream = false;
    }
  } one_stream;
  // task flow (dag.h) on request (HMGP_DAG=1, or HMGP_DAG_DIAG for its critical-path
  // report).  Measured at C3 its DAG critical path is within 1.33x of the serial
  // sum and it does not beat the in-order stream + sections schedule, so it is
  // off by default.
  bool use_dag = getenv("HMGP_STATS") == nullptr && getenv("HMGP_SERIAL") == nullptr &&
                 ((getenv("HMGP_DAG") && atoi(getenv("HMGP_DAG")) != 0) || getenv("HMGP_DAG_DIAG"));
  // Ephemeral factors (L(θ), predict) on a structure whose capacities are known:
  // captured once per host thread, replayed afterwards (factorize_graph above).
  bool graph_done = false;
  {
    const char* ge = getenv("HMGP_GRAPH");
    // (small problems: a capture costs more than the few thousand launches it saves)
    int min_n = 32768;
    if (const char* e = getenv("HMGP_GRAPH_MIN_N")) min_n = atoi(e);
    // (a capture costs about as much as a stream evaluation, more when several θ-batch
    // workers capture at once: it pays from this thread's third evaluation on the
    // structure — a long sweep, an MLE fit, repeated L(θ) — not for a one-off batch)
    static thread_local uint64_t seen_key = 0;
    static thread_local int seen_count = 0;
    int after = 2;
    if (const char* e = getenv("HMGP_GRAPH_AFTER")) after = atoi(e);
    bool eligible = t_graph_ok && memo_hit && G.n >= min_n && !use_dag && !(ge && atoi(ge) == 0) &&
                    !getenv("HMGP_STATS") && !getenv("HMGP_SERIAL");
    if (eligible) {
      const uint64_t skey = ((uint64_t)G.n << 32) ^ (uint64_t)L;
      if (seen_key != skey) {
        seen_key = skey;
        seen_count = 0;
      }
      eligible = seen_count >= after || t_gc.valid;
      ++seen_count;
    }
    if (eligible) {
      const int rc = factorize_graph(F, H, st, arena_bytes, tcap0, grow);
      graph_done = rc == 0;
      if (!graph_done) {  // hand the borrowed buffers back; the stream path owns its own
        F.pool = nullptr;
        F.d_leaf = nullptr;
        F.d_rank = F.d_compact = nullptr;
        F.d_d = nullptr;
        F.d_status = nullptr;
        F.borrowed = false;
        if (rc == 2) {
          if (tcap0 >= 1024 && grow >= 16) throw Error(6, "factorize: low-rank capacity exceeded");
          tcap0 = std::min(1024, tcap0 * 2);
          grow *= 2;
        }
      }
    }
  }
  if (!graph_done) {
    F.d_leaf = static_cast<std::remove_reference_t<decltype(F.d_leaf)>>(dev_alloc(sizeof(LeafDev) * std::max(L, 1)));
    F.d_rank = static_cast<std::remove_reference_t<decltype(F.d_rank)>>(dev_alloc(4 * std::max(L, 1)));
    F.d_compact = static_cast<std::remove_reference_t<decltype(F.d_compact)>>(dev_alloc(4 * std::max(L, 1)));
    F.d_d = static_cast<std::remove_reference_t<decltype(F.d_d)>>(dev_alloc(8ull * G.n));
    F.d_status = static_cast<std::remove_reference_t<decltype(F.d_status)>>(dev_alloc(sizeof(LeafFactorStatus)));
  }
  for (int tcap = tcap0; !graph_done;) {
    // clone payload (hblock.cpp:17-28) into the factor's own layout; compact_cols = 0
    F.leaf = H.leaf;
    size_t total = 0;
    std::vector<size_t> off(L);
    for (int k = 0; k < L; ++k) {
      LeafDev& l = F.leaf[k];
      off[k] = total;
      if (l.kind == DENSE) {
        total += (size_t)l.m * l.n;
      } else {
        l.cap = std::min(std::min(l.m, l.n) + 16, H.leaf[k].cap * grow);
        total += (size_t)(l.m + l.n) * l.cap;
      }
    }
    if (total != pool_doubles) {
      dev_free(F.pool);
      F.pool = nullptr;
      if (try_alloc(&F.pool, std::max<size_t>(1, total) * 8)) {
        // a regrown pool (doubled capacities) may not fit next to the persistent
        // temporary arena: drop the arena (re-sized to what is left below) first
        cudaGetLastError();
        F.pool = nullptr;
        release_thread_workspace();
        if (start_3d && try_alloc(&F.pool, std::max<size_t>(1, total) * 8)) {
          // the doubled 3-D start does not fit: fall back to the 2-D start
          cudaGetLastError();
          F.pool = nullptr;
          start_3d = false;
          grow = 1;
          tcap = 256;
          pool_doubles = 0;
          continue;
        }
        if (!F.pool) F.pool = dev_alloc_n<double>(std::max<size_t>(1, total));
      }
      pool_doubles = total;
      start_3d = false;  // the fallback applies to the initial start only (not to a regrown pool)
    }
    std::vector<CloneItem> ci;
    for (int k = 0; k < L; ++k) {
      LeafDev& l = F.leaf[k];
      l.a = F.pool + off[k];
      l.b = l.kind == DENSE ? nullptr : l.a + (size_t)l.m * l.cap;
      const LeafDev& s = H.leaf[k];
      if (l.kind == DENSE) {
        ci.push_back(CloneItem{s.a, l.a, (size_t)l.m * l.n});
      } else if (H.rank_host[k] > 0) {  // U and V prefixes are contiguous (ld = m, n)
        ci.push_back(CloneItem{s.a, l.a, (size_t)l.m * H.rank_host[k]});
        ci.push_back(CloneItem{s.b, l.b, (size_t)l.n * H.rank_host[k]});
      }
    }
    HMGP_CUDA(cudaMemcpyAsync(F.d_leaf, F.leaf.data(), sizeof(LeafDev) * L, cudaMemcpyHostToDevice, st));
    if (!ci.empty()) {
      CloneItem* d_ci = nullptr;
      d_ci = static_cast<std::remove_reference_t<decltype(d_ci)>>(dev_alloc(sizeof(CloneItem) * ci.size()));
      HMGP_CUDA(cudaMemcpyAsync(d_ci, ci.data(), sizeof(CloneItem) * ci.size(), cudaMemcpyHostToDevice, st));
      k_clone<<<(int)ci.size(), 256, 0, st>>>(d_ci);
      HMGP_LAUNCH_CHECK();
      HMGP_CUDA(cudaStreamSynchronize(st));
      dev_free(d_ci);
    }
    HMGP_CUDA(cudaMemcpyAsync(F.d_rank, H.d_rank, 4ull * L, cudaMemcpyDeviceToDevice, st));
    HMGP_CUDA(cudaMemsetAsync(F.d_compact, 0, 4ull * L, st));
    HMGP_CUDA(cudaMemsetAsync(F.d_d, 0, 8ull * G.n, st));
    LeafFactorStatus s0{INT_MAX, 0, 0, 0, 0.0, INFINITY, F.clamp_tol};
    HMGP_CUDA(cudaMemcpyAsync(F.d_status, &s0, sizeof(s0), cudaMemcpyHostToDevice, st));
    int err = 0;
    bool redo_serial = false;
    try {
      Engine E(F, st, arena_bytes, tcap, use_dag);
      E.stats_begin();
      cudaEvent_t dg0 = nullptr;
      if (E.dag && E.dag->serial) {
        HMGP_CUDA(cudaEventCreate(&dg0));
        HMGP_CUDA(cudaEventRecord(dg0, E.dag->s[0]));
      }
      const auto h0 = std::chrono::steady_clock::now();
      E.factor_diag(0);
      // compress_all (hfactor.cpp:321-328): every LR leaf, independent
      std::vector<int> lr;
      for (int k = 0; k < L; ++k)
        if (F.leaf[k].kind == LOWRANK) lr.push_back(F.leaf_node[k]);
      E.compress(lr);
      if (E.dag) E.dag->join_into(st);
      if (dg0) {
        HMGP_CUDA(cudaStreamSynchronize(st));
        double ser = 0.0;
        const double cp = E.dag->critical_path_ms(dg0, &ser);
        fprintf(stderr, "[hmgp] task flow: %lld tasks, serial %.1f ms, DAG critical path %.1f ms (x%.2f)\n",
                E.dag->n_tasks, ser, cp, cp > 0 ? ser / cp : 0.0);
        cudaEventDestroy(dg0);
      }
      if (getenv("HMGP_STATS") || getenv("HMGP_TIMING")) {
        const auto h1 = std::chrono::steady_clock::now();
        cudaStreamSynchronize(st);
        const auto h2 = std::chrono::steady_clock::now();
        fprintf(stderr, "[hmgp] host enqueue %.1f ms (ring wraps %d, %.1f ms blocked; arena peak %.2f GB, "
                "allocated %.2f GB), then GPU drain %.1f ms\n",
                std::chrono::duration<double, std::milli>(h1 - h0).count(), E.sg.wraps, E.sg.wrap_ms,
                E.ar.peak / 1e9, E.ar.total / 1e9,
                std::chrono::duration<double, std::milli>(h2 - h1).count());
        if (E.dag)
          fprintf(stderr, "[hmgp] task flow: %lld tasks, %lld event waits, %zu objects\n", E.dag->n_tasks,
                  E.dag->n_waits, E.dag->objs.size());
        if (E.stats_on) E.print_stats();
      }
      phase_mark(PH_FACTOR);
      HMGP_CUDA(cudaMemcpyAsync(&err, E.d_err, 4, cudaMemcpyDeviceToHost, st));
      HMGP_CUDA(cudaStreamSynchronize(st));
      F.arena_peak = E.ar.peak;
      t_last_arena_peak = E.ar.peak;
      g_work.arena_peak = std::max(g_work.arena_peak, (double)E.ar.peak);
      g_work.factor_attempts += 1;
    } catch (const Error& e) {
      if (e.code == kArenaFull) {
        // side-stream sections hold their temporaries until the join; on one
        // stream the arena is reused step by step (lower peak).  Redo once there.
        if (t_one_stream) throw Error(6, e.what());
        HMGP_CUDA(cudaDeviceSynchronize());
        one_stream.engage();
        redo_serial = true;
      } else {
        if (e.code != kSubArenaFull) throw;
        HMGP_CUDA(cudaDeviceSynchronize());
        redo_serial = true;
      }
    }
    if (redo_serial) {  // task-flow sub-arenas too small: redo in program order
      use_dag = false;
      continue;
    }
    if (!err) {
      memo_set(CapMemo{G.n, G.dim, L, tcap, grow});
      break;
    }
    if (tcap >= 1024 && grow >= 16)
      throw Error(6, "factorize: low-rank capacity exceeded (code " + std::to_string(err) + ")");
    tcap = std::min(1024, tcap * 2);
    grow *= 2;
  }
  LeafFactorStatus s{};
  HMGP_CUDA(cudaMemcpyAsync(&s, F.d_status, sizeof(s), cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  F.clamped = s.clamped;
  F.negative = s.negative;
  F.min_pivot = s.min_pivot;
  F.fail_pos = s.fail_pos;
  F.fail_val = s.fail_val;

  // Cholesky diagonal
  std::vector<int> dl, db;
  for (int k = 0; k < L; ++k) {
    const HNode& nd = F.nodes[F.leaf_node[k]];
    if (nd.row == nd.col) {
      dl.push_back(k);
      db.push_back(G.nbeg[nd.row]);
    }
  }
  F.diag_leaf = dl;
  if (!ldl) {
    int *d1, *d2;
    d1 = static_cast<std::remove_reference_t<decltype(d1)>>(dev_alloc(4 * dl.size()));
    d2 = static_cast<std::remove_reference_t<decltype(d2)>>(dev_alloc(4 * dl.size()));
    HMGP_CUDA(cudaMemcpyAsync(d1, dl.data(), 4 * dl.size(), cudaMemcpyHostToDevice, st));
    HMGP_CUDA(cudaMemcpyAsync(d2, db.data(), 4 * db.size(), cudaMemcpyHostToDevice, st));
    k_collect_diag<<<(int)dl.size(), 128, 0, st>>>(F.d_leaf, d1, d2, (int)dl.size(), F.d_d);
    HMGP_LAUNCH_CHECK();
    HMGP_CUDA(cudaStreamSynchronize(st));
    dev_free(d1);
    dev_free(d2);
  }
  F.rank_host.resize(L);
  HMGP_CUDA(cudaMemcpyAsync(F.rank_host.data(), F.d_rank, 4ull * L, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));

  // ---- solve schedules (column sweep) ----
  // forward: block applied right after the diagonal leaf holding its last column
  // backward: block applied right after the diagonal leaf holding its first row
  const int nd = (int)dl.size();
  std::vector<int> leaf_of_pos(G.n);
  for (int t = 0; t < nd; ++t) {
    const LeafDev& l = F.leaf[dl[t]];
    for (int i = 0; i < l.m; ++i) leaf_of_pos[db[t] + i] = t;
  }
  std::vector<std::vector<SolveBlk>> fw(nd), bw(nd);
  for (int k = 0; k < L; ++k) {
    const HNode& nn = F.nodes[F.leaf_node[k]];
    if (nn.row == nn.col) continue;
    const int r0 = G.nbeg[nn.row], c0 = G.nbeg[nn.col], c1 = G.nend[nn.col];
    fw[leaf_of_pos[c1 - 1]].push_back(SolveBlk{k, r0, c0});
    bw[leaf_of_pos[r0]].push_back(SolveBlk{k, r0, c0});
  }
  std::vector<SolveBlk> flat_f, flat_b;
  F.fwd_off.assign(nd + 1, 0);
  F.bwd_off.assign(nd + 1, 0);
  for (int t = 0; t < nd; ++t) {
    F.fwd_off[t] = (int)flat_f.size();
    flat_f.insert(flat_f.end(), fw[t].begin(), fw[t].end());
    F.bwd_off[t] = (int)flat_b.size();
    flat_b.insert(flat_b.end(), bw[t].begin(), bw[t].end());
  }
  F.fwd_off[nd] = (int)flat_f.size();
  F.bwd_off[nd] = (int)flat_b.size();
  F.diag_base = db;
  F.d_fwd = static_cast<std::remove_reference_t<decltype(F.d_fwd)>>(dev_alloc(sizeof(SolveBlk) * std::max<size_t>(1, flat_f.size())));
  F.d_bwd = static_cast<std::remove_reference_t<decltype(F.d_bwd)>>(dev_alloc(sizeof(SolveBlk) * std::max<size_t>(1, flat_b.size())));
  HMGP_CUDA(cudaMemcpyAsync(F.d_fwd, flat_f.data(), sizeof(SolveBlk) * flat_f.size(), cudaMemcpyHostToDevice, st));
  HMGP_CUDA(cudaMemcpyAsync(F.d_bwd, flat_b.data(), sizeof(SolveBlk) * flat_b.size(), cudaMemcpyHostToDevice, st));
  F.d_work = static_cast<std::remove_reference_t<decltype(F.d_work)>>(dev_alloc(8ull * (2 * G.n + 1024)));
  {  // persistent-sweep plans (K10)
    const SolvePlan pf = build_solve_plan(F, flat_f, F.fwd_off, false);
    const SolvePlan pb = build_solve_plan(F, flat_b, F.bwd_off, true);
    auto up = [&](const void* src, size_t bytes) {
      void* d = nullptr;
      d = static_cast<std::remove_reference_t<decltype(d)>>(dev_alloc(std::max<size_t>(bytes, 16)));
      if (bytes) HMGP_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st));
      return d;
    };
    F.d_fsteps = up(pf.steps.data(), pf.steps.size() * sizeof(SStep));
    F.d_funits = up(pf.units.data(), pf.units.size() * sizeof(SUnit));
    F.d_bsteps = up(pb.steps.data(), pb.steps.size() * sizeof(SStep));
    F.d_bunits = up(pb.units.data(), pb.units.size() * sizeof(SUnit));
    F.solve_stride = std::max(pf.stride, pb.stride);
    const size_t pd = (size_t)std::max(pf.slots, pb.slots) * F.solve_stride;
    F.d_part = static_cast<std::remove_reference_t<decltype(F.d_part)>>(dev_alloc(std::max<size_t>(pd, 1) * 8));
  }
  phase_mark(PH_LAYOUT);
  HMGP_CUDA(cudaStreamSynchronize(st));
}

// v (tree order, device) <- L^{-1} v
void forward_solve(const Factor& F, double* v, cudaStream_t st) {
  if (F.d_fsteps && !getenv("HMGP_SOLVE_LEGACY")) {
    solve_sweep(F, v, false, st);
    return;
  }
  const int nd = (int)F.diag_leaf.size();
  for (int t = 0; t < nd; ++t) {
    const LeafDev& l = F.leaf[F.diag_leaf[t]];
    launch_trsv(l.a, l.m, v + F.diag_base[t], 0, st);
    HMGP_LAUNCH_CHECK();
    const int cnt = F.fwd_off[t + 1] - F.fwd_off[t];
    if (cnt > 0) {
      k_solve_apply<<<cnt, 128, 0, st>>>(static_cast<const SolveBlk*>(F.d_fwd) + F.fwd_off[t],
                                         F.d_leaf, F.d_rank, v, 0);
      HMGP_LAUNCH_CHECK();
    }
  }
}
// v <- L^{-T} v
void backward_solve(const Factor& F, double* v, cudaStream_t st) {
  if (F.d_bsteps && !getenv("HMGP_SOLVE_LEGACY")) {
    solve_sweep(F, v, true, st);
    return;
  }
  const int nd = (int)F.diag_leaf.size();
  for (int t = nd - 1; t >= 0; --t) {
    const LeafDev& l = F.leaf[F.diag_leaf[t]];
    launch_trsv(l.a, l.m, v + F.diag_base[t], 1, st);
    HMGP_LAUNCH_CHECK();
    const int cnt = F.bwd_off[t + 1] - F.bwd_off[t];
    if (cnt > 0) {
      k_solve_apply<<<cnt, 128, 0, st>>>(static_cast<const SolveBlk*>(F.d_bwd) + F.bwd_off[t],
                                         F.d_leaf, F.d_rank, v, 1);
      HMGP_LAUNCH_CHECK();
    }
  }
}

static double reduce(const Factor& F, const double* v, int mode, cudaStream_t st) {
  const int n = F.g->n;
  double* part = F.d_work + 2 * (size_t)n;
  const int nb = 148;
  k_reduce_partial<<<nb, 256, 0, st>>>(v, F.d_d, n, mode, part);
  HMGP_LAUNCH_CHECK();
  k_reduce_final<<<1, 256, 0, st>>>(part, nb, part + 512);
  HMGP_LAUNCH_CHECK();
  double out = 0;
  HMGP_CUDA(cudaMemcpyAsync(&out, part + 512, 8, cudaMemcpyDeviceToHost, st));
  HMGP_CUDA(cudaStreamSynchronize(st));
  return out;
}

// HFactor::log_det (hfactor.cpp:399-403)
double factor_log_det(const Factor& F, cudaStream_t st) {
  NvtxRange nvtx_range("hmgp:log_det(K11)");
  const int n = F.g->n;
  if (F.ldl) {
    int* cnt = reinterpret_cast<int*>(F.d_work + 2 * (size_t)n + 600);
    HMGP_CUDA(cudaMemsetAsync(cnt, 0, 4, st));
    k_count_nonpos<<<148, 256, 0, st>>>(F.d_d, n, cnt);
    HMGP_LAUNCH_CHECK();
    int h = 0;
    HMGP_CUDA(cudaMemcpyAsync(&h, cnt, 4, cudaMemcpyDeviceToHost, st));
    HMGP_CUDA(cudaStreamSynchronize(st));
    if (h) throw std::domain_error("indefinite factor");
    return reduce(F, F.d_d, 2, st);
  }
  return 2.0 * reduce(F, F.d_d, 2, st);
}

// HFactor::quad_form with b in original order on device (hfactor.cpp:389-397)
double factor_quad_form_dev(const Factor& F, const double* d_b, cudaStream_t st) {
  NvtxRange nvtx_range("hmgp:quad_form(K10)");
  const int n = F.g->n;
  double* v = F.d_work;
  k_gather<<<(n + 255) / 256, 256, 0, st>>>(d_b, F.g->d_perm, n, v);
  HMGP_LAUNCH_CHECK();
  forward_solve(F, v, st);
  return reduce(F, v, F.ldl ? 1 : 0, st);
}

// solve_factored / solve_lower with device b, x in original order
void factor_solve_dev(const Factor& F, const double* d_b, double* d_x, bool full, cudaStream_t st) {
  NvtxRange nvtx_range("hmgp:solve(K10)");
  const int n = F.g->n;
  double* v = F.d_work;
  k_gather<<<(n + 255) / 256, 256, 0, st>>>(d_b, F.g->d_perm, n, v);
  HMGP_LAUNCH_CHECK();
  forward_solve(F, v, st);
  if (full) {
    if (F.ldl) {
      k_div<<<(n + 255) / 256, 256, 0, st>>>(v, F.d_d, n);
      HMGP_LAUNCH_CHECK();
    }
    backward_solve(F, v, st);
  }
  k_scatter<<<(n + 255) / 256, 256, 0, st>>>(v, F.g->d_perm, n, d_x);
  HMGP_LAUNCH_CHECK();
}

double factor_storage_bytes(const Factor& F) {  // hfactor.cpp:412-419
  double b = 0;
  for (size_t k = 0; k < F.leaf.size(); ++k) {
    const LeafDev& l = F.leaf[k];
    b += l.kind == DENSE ? 8.0 * l.m * l.n : 8.0 * (l.m + l.n) * F.rank_host[k];
  }
  if (F.ldl) b += 8.0 * F.g->n;
  return b;
}

}  // namespace hmgp_gpu
