"""Per-phase device time + work counters of one L(θ) evaluation."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import _lib

_lib.hmgp_last_phases.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
_lib.hmgp_work_counters.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int]
NAMES = ["start", "geometry", "dense_K3", "aca_K4K5", "layout", "factor", "logdet", "fwd_solve", "bwd", "cross"]
g, leaf, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
th = [float(v) for v in sys.argv[4].split(",")]
form = sys.argv[5] if len(sys.argv) > 5 else "cholesky"
x = hm.jittered_grid(g, 1); z = hm.normals(g * g, 7)
cfg = hm.HConfig(leaf_size=leaf, rank=hm.RankControl.fixed_accuracy(eps), form=form)
ctx = hm.default_context()
w = (C.c_double * 10)()
_lib.hmgp_work_counters(w, 10, 1)
t = time.time(); r = hm.evaluate_loglik(x, z, th, cfg, ctx=ctx); wall = time.time() - t
ph = (C.c_double * 10)(); _lib.hmgp_last_phases(ctx.h, ph, 10)
_lib.hmgp_work_counters(w, 10, 1)
print(f"n={g*g} leaf={leaf} th={th} {form}: wall {wall:.3f}s L={r.loglik:.10f}")
print("phases_ms", {k: round(v, 2) for k, v in zip(NAMES, ph)})
print("work", dict(zip(["dense_entries", "aca_entries", "kernel_flops", "gemm", "trsm", "leaf", "trunc_flops", "trunc_items", "arena_peak", "attempts"], [f"{v:.3g}" for v in w])))
