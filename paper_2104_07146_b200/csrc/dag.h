// Sequential task flow (STF) over CUDA streams for the H-factorization.
//
// The host walks the reference recursion (hfactor.cpp:287-319) and submits
// every batched launch as a TASK, in program order, together with the device
// memory the task reads and writes (objects: stored leaves, device-resident
// rank / compact counters, the D segments of diagonal leaves, arena
// temporaries).  A task waits only for the earlier tasks it conflicts with
// (read-after-write, write-after-read, write-after-write on the same object);
// the runtime picks a stream for it (the stream of its latest dependency when
// that dependency is the stream's tail, else the least recently used stream)
// and expresses the remaining dependencies as event waits.  Results are the
// ones of the program-order execution: every object sees exactly the same
// sequence of operations, only independent tasks overlap.  In the reference
// recursion the trsm / sub_product of a block-row can start as soon as the
// diagonal leaves it needs are factored, instead of after the whole
// preceding factor_diag call (the fork-join bound of the recursion).
//
// Arena temporaries are reused (stack discipline on the host); a new
// allocation that overlaps memory used by earlier tasks inherits those tasks
// as a fence, so reuse never races.  Hazard lists are compacted per stream
// (a later task on the same stream implies the earlier ones finished).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace hmgp_gpu {

struct Dag {
  static constexpr int kS = 32;   // streams
  static constexpr int kR = 256;  // event ring per stream
  cudaStream_t s[kS] = {};
  cudaEvent_t ev[kS][kR] = {};
  long long pos[kS] = {};  // tasks issued per stream
  long long lru[kS] = {};  // id of the latest task per stream (+1; 0 = none)
  bool serial = false;     // diagnostics: launch everything on stream 0 (timing)
  std::vector<cudaEvent_t> tev;  // serial mode: one event per task
  std::vector<int> tdeps_off, tdeps;  // serial mode: dependency lists
  const char* label = "";             // serial mode: label of the next task
  std::vector<const char*> tlabel;

  std::vector<int> tstream;
  std::vector<long long> tpos;

  struct Haz {
    std::vector<int> w, r;  // last writers (a fence may hold several), readers since
  };
  std::vector<Haz> objs;
  std::vector<int> freeo;
  int nfixed = 0;

  // fixed objects: stored leaves [0, nleaf)
  std::vector<uintptr_t> lbeg, lend;  // payload region per leaf (sorted by begin)
  std::vector<int> lorder;            // leaf index per sorted position
  uintptr_t rank_b = 0, comp_b = 0, d_b = 0;
  int nleaf = 0, npos = 0;
  std::vector<int> pos_obj;  // D position -> diagonal leaf object
  // arena temporaries: start -> (end, object)
  uintptr_t ar_b = 0, ar_e = 0;
  std::map<uintptr_t, std::pair<uintptr_t, int>> tmp;

  long long n_waits = 0, n_tasks = 0;

  ~Dag() {
    if (!s[0]) return;
    for (int i = 0; i < kS; ++i) {
      cudaStreamDestroy(s[i]);
      for (int j = 0; j < kR; ++j) cudaEventDestroy(ev[i][j]);
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  void init_streams() {
    if (s[0]) return;
    for (int i = 0; i < kS; ++i) {
      HMGP_CUDA(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
      for (int j = 0; j < kR; ++j) HMGP_CUDA(cudaEventCreateWithFlags(&ev[i][j], cudaEventDisableTiming));
    }
  }

  // start of one factorization: `fixed` leaf regions, counters, D
  void reset(const std::vector<uintptr_t>& beg, const std::vector<uintptr_t>& end, const int* d_rank,
             const int* d_comp, const double* d_d, const std::vector<int>& pobj, uintptr_t arena_b,
             uintptr_t arena_e) {
    init_streams();
    nleaf = (int)beg.size();
    lorder.resize(nleaf);
    for (int k = 0; k < nleaf; ++k) lorder[k] = k;
    std::sort(lorder.begin(), lorder.end(), [&](int a, int b) { return beg[a] < beg[b]; });
    lbeg.resize(nleaf);
    lend.resize(nleaf);
    for (int i = 0; i < nleaf; ++i) {
      lbeg[i] = beg[lorder[i]];
      lend[i] = end[lorder[i]];
    }
    rank_b = (uintptr_t)d_rank;
    comp_b = (uintptr_t)d_comp;
    d_b = (uintptr_t)d_d;
    pos_obj = pobj;
    npos = (int)pobj.size();
    ar_b = arena_b;
    ar_e = arena_e;
    tmp.clear();
    objs.assign(nleaf, Haz{});
    freeo.clear();
    nfixed = nleaf;
    tstream.clear();
    tpos.clear();
    for (int i = 0; i < kS; ++i) lru[i] = 0;
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
    tev.clear();
    tdeps_off.assign(1, 0);
    tdeps.clear();
    tlabel.clear();
    n_waits = n_tasks = 0;
  }

  int new_obj() {
    if (!freeo.empty()) {
      const int o = freeo.back();
      freeo.pop_back();
      objs[o].w.clear();
      objs[o].r.clear();
      return o;
    }
    objs.emplace_back();
    return (int)objs.size() - 1;
  }

  // add task t to a hazard list, keeping one (the latest) task per stream
  void add(std::vector<int>& v, int t) const {
    const int st = tstream[t];
    for (int& x : v)
      if (tstream[x] == st) {
        if (tpos[t] > tpos[x]) x = t;
        return;
      }
    v.push_back(t);
  }

  // arena allocation [a, b): fence it with the tasks that used overlapping memory
  void on_alloc(uintptr_t a, uintptr_t b) {
    const int o = new_obj();
    auto it = tmp.lower_bound(a);
    if (it != tmp.begin()) {
      auto pv = std::prev(it);
      if (pv->second.first > a) it = pv;
    }
    while (it != tmp.end() && it->first < b) {
      const uintptr_t s0 = it->first, e0 = it->second.first;
      const int oo = it->second.second;
      for (int x : objs[oo].w) add(objs[o].w, x);
      for (int x : objs[oo].r) add(objs[o].w, x);
      it = tmp.erase(it);
      const bool head = s0 < a, tail = e0 > b;
      if (head && tail) {
        const int oh = new_obj();
        objs[oh] = objs[oo];
        tmp[s0] = {a, oh};
        tmp[b] = {e0, oo};
      } else if (head) {
        tmp[s0] = {a, oo};
      } else if (tail) {
        tmp[b] = {e0, oo};
      } else {
        freeo.push_back(oo);
      }
    }
    tmp[a] = {b, o};
  }

  int lookup(const void* p) const {
    const uintptr_t x = (uintptr_t)p;
    if (!x) return -1;
    if (x >= ar_b && x < ar_e) {
      auto it = tmp.upper_bound(x);
      if (it == tmp.begin()) return -1;
      --it;
      return x < it->second.first ? it->second.second : -1;
    }
    if (x >= rank_b && x < rank_b + 4ull * nleaf) return (int)((x - rank_b) / 4);
    if (x >= comp_b && x < comp_b + 4ull * nleaf) return (int)((x - comp_b) / 4);
    if (x >= d_b && x < d_b + 8ull * npos) return pos_obj[(x - d_b) / 8];
    auto it = std::upper_bound(lbeg.begin(), lbeg.end(), x);
    if (it == lbeg.begin()) return -1;
    const size_t i = (it - lbeg.begin()) - 1;
    return x < lend[i] ? lorder[i] : -1;
  }

  // Launch one task: accs = (object, write) pairs; fn(stream) enqueues it.
  template <class Fn>
  cudaStream_t launch(const std::vector<std::pair<int, char>>& accs, Fn&& fn) {
    const int t = (int)tstream.size();
    long long need[kS];
    for (int i = 0; i < kS; ++i) need[i] = -1;
    std::vector<int>* dl = serial ? &tdeps : nullptr;
    auto dep = [&](int x) {
      if (x == t) return;
      const int st = tstream[x];
      need[st] = std::max(need[st], tpos[x]);
      if (dl) dl->push_back(x);
    };
    for (const auto& a : accs) {
      const Haz& h = objs[a.first];
      for (int x : h.w) dep(x);
      if (a.second)
        for (int x : h.r) dep(x);
    }
    // stream: the latest dependency that is its stream's tail, else the LRU stream
    int best = -1;
    long long bl = -1;
    for (int i = 0; i < kS; ++i)
      if (need[i] >= 0 && need[i] == pos[i] - 1 && lru[i] > bl) {
        best = i;
        bl = lru[i];
      }
    if (best < 0) {
      best = 0;
      for (int i = 1; i < kS; ++i)
        if (lru[i] < lru[best]) best = i;
    }
    cudaStream_t cs = serial ? s[0] : s[best];
    if (!serial)
      for (int i = 0; i < kS; ++i)
        if (i != best && need[i] >= 0) {
          HMGP_CUDA(cudaStreamWaitEvent(cs, ev[i][need[i] % kR], 0));
          ++n_waits;
        }
    tstream.push_back(best);
    tpos.push_back(pos[best]);
    for (const auto& a : accs) {
      Haz& h = objs[a.first];
      if (a.second) {
        h.w.assign(1, t);
        h.r.clear();
      } else {
        add(h.r, t);
      }
    }
    fn(cs);
    HMGP_CUDA(cudaEventRecord(ev[best][pos[best] % kR], cs));
    if (serial) {
      cudaEvent_t e;
      HMGP_CUDA(cudaEventCreate(&e));
      HMGP_CUDA(cudaEventRecord(e, cs));
      tev.push_back(e);
      tdeps_off.push_back((int)tdeps.size());
      tlabel.push_back(label);
    }
    ++pos[best];
    lru[best] = t + 1;
    ++n_tasks;
    return cs;
  }

  // make `main` wait for every stream (end of the factorization)
  void join_into(cudaStream_t main) {
    for (int i = 0; i < kS; ++i)
      if (pos[i] > 0) HMGP_CUDA(cudaStreamWaitEvent(main, ev[i][(pos[i] - 1) % kR], 0));
  }
  // every stream waits for `main` (start of the factorization)
  void fork_from(cudaStream_t main, cudaEvent_t e) {
    HMGP_CUDA(cudaEventRecord(e, main));
    for (int i = 0; i < kS; ++i) HMGP_CUDA(cudaStreamWaitEvent(s[i], e, 0));
  }

  // serial diagnostics: measured task durations -> DAG critical path (ms);
  // prints the path's time by task label
  double critical_path_ms(cudaEvent_t start, double* serial_ms) const {
    const int n = (int)tev.size();
    std::vector<double> fin(n, 0.0), dur(n, 0.0);
    std::vector<int> via(n, -1);
    double cp = 0.0, tot = 0.0;
    int last = -1;
    cudaEvent_t prev = start;
    for (int t = 0; t < n; ++t) {
      float d = 0.f;
      cudaEventElapsedTime(&d, prev, tev[t]);
      prev = tev[t];
      double st = 0.0;
      for (int k = tdeps_off[t]; k < tdeps_off[t + 1]; ++k)
        if (fin[tdeps[k]] > st) {
          st = fin[tdeps[k]];
          via[t] = tdeps[k];
        }
      dur[t] = d;
      fin[t] = st + d;
      if (fin[t] > cp) {
        cp = fin[t];
        last = t;
      }
      tot += d;
    }
    if (serial_ms) *serial_ms = tot;
    std::map<std::string, std::pair<double, int>> on, all;
    for (int t = 0; t < n; ++t) {
      auto& a = all[tlabel[t]];
      a.first += dur[t];
      a.second += 1;
    }
    int len = 0;
    for (int t = last; t >= 0; t = via[t]) {
      auto& a = on[tlabel[t]];
      a.first += dur[t];
      a.second += 1;
      ++len;
    }
    fprintf(stderr, "[hmgp] critical path: %d tasks\n", len);
    for (const auto& kv : all) {
      auto it = on.find(kv.first);
      fprintf(stderr, "[hmgp]   %-16s on path %9.1f ms (%6d tasks)   all %9.1f ms (%6d tasks)\n",
              kv.first.c_str(), it == on.end() ? 0.0 : it->second.first, it == on.end() ? 0 : it->second.second,
              kv.second.first, kv.second.second);
    }
    return cp;
  }
};

}  // namespace hmgp_gpu
