"""3-D (C5-shaped) L(θ) probe: uniform points in [0,1]^3, theta=(1,0.08,0.5,0.005), leaf 128, eps 1e-5."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import _lib
_lib.hmgp_last_phases.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
n = int(sys.argv[1])
x = hm.random_locations(n, 1, dim=3); z = hm.normals(n, 1 ^ hm.Z_SEED_XOR)
cfg = hm.HConfig(leaf_size=128, rank=hm.RankControl.fixed_accuracy(1e-5), form="cholesky")
ctx = hm.default_context()
g = hm.Geometry(x, 128, 2.0, ctx=ctx); print("blocks", g.block_counts(), flush=True); del g
t = time.time(); r = hm.evaluate_loglik(x, z, [1.0, 0.08, 0.5, 0.005], cfg, ctx=ctx)
ph = (C.c_double * 10)(); _lib.hmgp_last_phases(ctx.h, ph, 10)
print(f"3D n={n}: wall {time.time()-t:.2f}s L={r.loglik:.8f} phases={[round(v,1) for v in ph]}", flush=True)
