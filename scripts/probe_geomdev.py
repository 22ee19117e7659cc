"""Bench-shaped step (device-built geometry + hmgp_loglik_geom) vs the host API:
per-phase split of consecutive evaluations, to locate the bench's 'layout' time."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import _lib

_lib.hmgp_last_phases.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
NAMES = ["start", "geometry", "dense_K3", "aca_K4K5", "layout", "factor", "logdet", "fwd_solve", "bwd", "cross"]
g = 512; n = g * g
x = hm.jittered_grid(g, 1); z = hm.normals(n, 7)
cfg = hm.HConfig(leaf_size=128, rank=hm.RankControl.fixed_accuracy(1e-6), form="cholesky").c()
th = hm.Matern(1.5, 0.05, 1.0, 0.01)
ctx = hm.default_context()
dx = torch.from_numpy(x).cuda(); dz = torch.from_numpy(z).cuda(); torch.cuda.synchronize()
res = hm._LogLik()
mode = sys.argv[1] if len(sys.argv) > 1 else "dev"
for it in range(3):
    t = time.time()
    gh = C.c_void_p()
    if mode == "dev":
        hm._chk(_lib.hmgp_geometry_build_device(ctx.h, C.c_void_p(dx.data_ptr()), n, 2, 128, 2.0, C.byref(gh)))
    else:
        hm._chk(_lib.hmgp_geometry_build(ctx.h, x.ctypes.data_as(hm._dp), n, 2, 128, 2.0, C.byref(gh)))
    t1 = time.time()
    hm._chk(_lib.hmgp_loglik_geom(ctx.h, gh, C.c_void_p(dz.data_ptr()), C.byref(th), C.byref(cfg), C.byref(res)))
    t2 = time.time()
    _lib.hmgp_geometry_destroy(gh)
    torch.cuda.synchronize()
    ph = (C.c_double * 10)(); _lib.hmgp_last_phases(ctx.h, ph, 10)
    print(f"{mode} eval {it}: build {1e3*(t1-t):.1f} ms, loglik {t2-t1:.3f}s, destroy {1e3*(time.time()-t2):.1f} ms",
          {k: round(v, 1) for k, v in zip(NAMES, ph)}, flush=True)
