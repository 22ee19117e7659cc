"""θ-batch concurrency probe: hmgp_loglik_batch on a subset of the C4 grid with
HMGP_BATCH_THREADS workers; prints wall, evals/s and the L values."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
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
torch.cuda.synchronize()
t = time.time(); v = sw.run_sweep(geo, dz.data_ptr(), grid, idx, cfg, ctx); w = time.time() - t
print(f"threads={os.environ.get('HMGP_BATCH_THREADS','8')} n={g*g} thetas={nth}: {w:.2f}s {nth/w:.3f} evals/s")
print(" ".join(f"{a:.10e}" for a in v[:, 0]))
