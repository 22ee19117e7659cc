"""Concurrency of a θ-batch under CUPTI (torch.profiler): sum of kernel time vs
the union of kernel intervals (how many kernels really overlap), per-stream busy
time, and the time-weighted number of resident CTAs' SMs (grid x cluster bound).

usage: python scripts/trace_batch.py g leaf eps ntheta
"""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import sweep as sw

g, leaf, eps, nth = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
x = hm.jittered_grid(g, 1); z = hm.normals(g * g, 7)
ctx = hm.default_context()
geo = hm.Geometry(x, leaf, 2.0, ctx=ctx)
dz = torch.from_numpy(z).cuda()
grid = sw.c4_theta_grid()
idx = list(range(200, 200 + nth))
cfg = hm.HConfig(leaf_size=leaf, rank=hm.RankControl.fixed_accuracy(eps))
n1 = int(sys.argv[4]); nth = int(sys.argv[5]); idx = list(range(200 + n1, 200 + n1 + nth))
sw.run_sweep(geo, dz.data_ptr(), grid, list(range(200, 200 + n1)), cfg, ctx)  # warm: workers capture
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t = time.time(); v = sw.run_sweep(geo, dz.data_ptr(), grid, idx, cfg, ctx); wall = time.time() - t
print(f"threads={os.environ.get('HMGP_BATCH_THREADS','8')} n={g*g} thetas={nth}: wall {wall:.2f}s {nth/wall:.3f} evals/s")
ev = prof.events()
kern = [(e.time_range.start, e.time_range.end, e.name) for e in ev
        if e.device_type == torch.autograd.DeviceType.CUDA and not e.name.startswith("Mem")]
cps = [(e.time_range.start, e.time_range.end) for e in ev
       if e.device_type == torch.autograd.DeviceType.CUDA and e.name.startswith("Memcpy")]
kern.sort()
tot = sum(e - s for s, e, _ in kern)
pts = []
for s, e, _ in kern:
    pts.append((s, 1)); pts.append((e, -1))
pts.sort()
busy = 0.0; depth = 0; last = None; hist = collections.Counter()
for t_, d in pts:
    if depth > 0:
        busy += t_ - last; hist[min(depth, 16)] += t_ - last
    depth += d; last = t_
span = kern[-1][1] - kern[0][0]
print(f"kernels {len(kern)}, span {span/1e3:.1f} ms, union busy {busy/1e3:.1f} ms, sum {tot/1e3:.1f} ms, "
      f"mean overlap {tot/max(busy,1):.2f}; memcpy ops {len(cps)} total {sum(e-s for s,e in cps)/1e3:.1f} ms")
for k in sorted(hist):
    print(f"   {k:2d} kernels running: {hist[k]/1e3:9.1f} ms")
by = collections.defaultdict(lambda: [0, 0.0])
for s, e, n in kern:
    by[n.split('(')[0][-40:]][0] += 1; by[n.split('(')[0][-40:]][1] += e - s
for n, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {t/1e3:10.1f} ms {c:7d}x avg {t/c:8.1f} us  {n}")
api = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
        a = api[e.name]; a[0] += 1; a[1] += e.time_range.end - e.time_range.start
for n, (c, t) in sorted(api.items(), key=lambda kv: -kv[1][1])[:6]:
    print(f"  API {n:28s} {c:8d}x {t/1e3:9.1f} ms (summed over threads)  {t/c:7.1f} us/call")
