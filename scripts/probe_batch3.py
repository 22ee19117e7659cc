"""θ-batch probe: two consecutive hmgp_loglik_sweep batches on one geometry (the
second finds the persistent workers warm: captured factorizations are replayed),
checked bit-for-bit against single evaluations of a few θ."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import sweep as sw

g, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
counts = [int(a) for a in sys.argv[4:]]
form = "cholesky" if g == 512 else "ldl"
x = hm.jittered_grid(g, 1); z = hm.normals(g * g, 7)
ctx = hm.default_context()
geo = hm.Geometry(x, leaf, 2.0, ctx=ctx)
grid = sw.c4_theta_grid()
if g == 512:
    grid = np.array([[1.5, 0.05 * (1 + 0.01 * k), 1.0, 0.01] for k in range(128)])
cfg = hm.HConfig(leaf_size=leaf, rank=hm.RankControl.fixed_accuracy(eps), form=form)
tag = f"T={os.environ.get('HMGP_BATCH_THREADS','16')} graph={os.environ.get('HMGP_GRAPH','1')} n={g*g}"
allv = {}
lo = 200 if g != 512 else 0
for rnd, cnt in enumerate(counts):
    idx = list(range(lo, lo + cnt)); lo += cnt
    t = time.time(); _, v = sw.sweep_host(geo, z, grid, idx, cfg, ctx); w = time.time() - t
    print(f"{tag} batch {rnd}: thetas={cnt}: {w:.2f}s {cnt/w:.3f} evals/s", flush=True)
    for i, r in zip(idx, v):
        allv[i] = r
chk = list(allv)[:: max(1, len(allv) // 3)][:3]
bad = 0
for i in chk:
    one = hm.evaluate_loglik(x, z, list(grid[i]), cfg, ctx=ctx)
    same = one.loglik == allv[i][0]
    bad += not same
    print(f"  theta {i}: batch {allv[i][0]!r} single {one.loglik!r} {'bit-identical' if same else 'DIFFERENT'}")
print("bitcheck", "ok" if not bad else "FAILED")
