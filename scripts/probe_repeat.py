"""Phase split of consecutive L(θ) evaluations in one process (steady state vs first)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import _lib

_lib.hmgp_last_phases.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
NAMES = ["start", "geometry", "dense_K3", "aca_K4K5", "layout", "factor", "logdet", "fwd_solve", "bwd", "cross"]
g = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = hm.jittered_grid(g, 1); z = hm.normals(g * g, 7)
cfg = hm.HConfig(leaf_size=128, rank=hm.RankControl.fixed_accuracy(1e-6), form="cholesky")
ctx = hm.default_context()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    t = time.time(); r = hm.evaluate_loglik(x, z, [1.5, 0.05, 1.0, 0.01], cfg, ctx=ctx); wall = time.time() - t
    ph = (C.c_double * 10)(); _lib.hmgp_last_phases(ctx.h, ph, 10)
    print(f"eval {it}: wall {wall:.3f}s", {k: round(v, 1) for k, v in zip(NAMES, ph)}, flush=True)
