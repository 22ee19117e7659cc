"""Small-n θ-batch overhead: n = 256, batches of 8 through hmgp_loglik_sweep vs single evaluations."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import sweep as sw
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x = hm.random_locations(n, 8); z = hm.normals(n, 3)
cfg = hm.HConfig(rank=hm.RankControl.fixed_accuracy(1e-4))
ctx = hm.default_context()
geo = hm.Geometry(x, cfg.leaf_size, 2.0, ctx=ctx)
th = np.array([[1.0 + 0.01 * k, 0.1, 0.5, 0.001] for k in range(64)])
hm.evaluate_loglik(x, z, list(th[0]), cfg)
t = time.time()
for k in range(16): hm.evaluate_loglik(x, z, list(th[k]), cfg)
print(f"single: {1e3 * (time.time() - t) / 16:.2f} ms per eval", flush=True)
for nb in (1, 2, 8):
    sw.sweep_host(geo, z, th, list(range(nb)), cfg, ctx)
    t = time.time()
    reps = 20
    for r in range(reps): sw.sweep_host(geo, z, th, list(range(r, r + nb)), cfg, ctx)
    dt = (time.time() - t) / reps
    print(f"batch of {nb}: {1e3 * dt:.2f} ms per batch, {1e3 * dt / nb:.2f} ms per eval", flush=True)
