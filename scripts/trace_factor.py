"""Timeline of one L(θ) under CUPTI (torch.profiler): GPU busy time (union of
kernel intervals) vs wall, and host time inside CUDA runtime calls — tells
whether the factorization is host-enqueue bound or device bound.

usage: python scripts/trace_factor.py g leaf eps s2,l,nu,tau2 [out.json]
"""
import collections, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2104_07146_b200 as hm

g, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
th = [float(v) for v in sys.argv[4].split(",")]
out = sys.argv[5] if len(sys.argv) > 5 else None
x = hm.jittered_grid(g, 1); z = hm.normals(g * g, 7)
cfg = hm.HConfig(leaf_size=leaf, rank=hm.RankControl.fixed_accuracy(eps), form="cholesky")
ctx = hm.default_context()
hm.evaluate_loglik(x, z, th, cfg, ctx=ctx)  # warm
torch.cuda.init()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t = time.time(); r = hm.evaluate_loglik(x, z, th, cfg, ctx=ctx); wall = time.time() - t
print(f"wall {wall*1e3:.1f} ms L={r.loglik:.10f}")
ev = prof.events()
kern = [(e.time_range.start, e.time_range.end, e.name) for e in ev if e.device_type == torch.autograd.DeviceType.CUDA]
kern.sort()
busy, cur_s, cur_e = 0.0, None, None
for s, e, _ in kern:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (kern[-1][1] - kern[0][0]) if kern else 0
print(f"device activities {len(kern)}, span {span/1e3:.1f} ms, busy (union) {busy/1e3:.1f} ms")
by = collections.defaultdict(lambda: [0, 0.0])
for s, e, n in kern:
    by[n][0] += 1; by[n][1] += e - s
for n, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {t/1e3:10.1f} ms {c:7d}x  {n[:110]}")
api = collections.defaultdict(lambda: [0, 0.0, 0.0])
for e in ev:
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
        d = e.time_range.end - e.time_range.start
        a = api[e.name]; a[0] += 1; a[1] += d; a[2] = max(a[2], d)
tot = 0
for n, (c, t, mx) in sorted(api.items(), key=lambda kv: -kv[1][1]):
    tot += t
    print(f"  API {n:32s} {c:7d}x {t/1e3:9.1f} ms  max {mx/1e3:8.2f} ms")
print(f"host time inside CUDA runtime calls: {tot/1e3:.1f} ms of {wall*1e3:.1f} ms wall")
if out:
    prof.export_chrome_trace(out)
