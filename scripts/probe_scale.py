"""Scale probe: L(θ) wall time on the GPU at growing n (C1 .. C3 shapes)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_07146_b200 as hm

cases = [
    ("C1", 64, 64, [1.0, 0.1, 0.5, 0.01], 1e-7),
    ("g128_l64_nu0.5", 128, 64, [1.0, 0.1, 0.5, 0.01], 1e-7),
    ("C2/C4_n65536_nu0.5", 256, 64, [1.0, 0.1, 0.5, 0.01], 1e-7),
    ("g256_l128_C3theta", 256, 128, [1.5, 0.05, 1.0, 0.01], 1e-6),
    ("C3_n262144", 512, 128, [1.5, 0.05, 1.0, 0.01], 1e-6),
]
only = sys.argv[1:] 
for name, g, leaf, th, eps in cases:
    if only and name not in only:
        continue
    x = hm.jittered_grid(g, 1)
    z = hm.normals(g * g, 7)
    for form in ("cholesky",):
        cfg = hm.HConfig(leaf_size=leaf, rank=hm.RankControl.fixed_accuracy(eps), form=form)
        ctx = hm.default_context()
        l0 = ctx.launches()
        t = time.time()
        try:
            r = hm.evaluate_loglik(x, z, th, cfg)
            msg = f"L={r.loglik:.10f} logdet={r.logdet:.6f} quad={r.quad_form:.6f}"
        except Exception as e:
            msg = f"ERROR {type(e).__name__}: {e}"
        print(f"{name} n={g*g} {form}: {time.time()-t:.3f}s launches={ctx.launches()-l0} {msg}", flush=True)
