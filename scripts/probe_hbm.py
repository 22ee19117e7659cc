"""C3 H-matvec and forward solve alone (for ncu --set full: DRAM traffic of the
HBM-bound kernels): assemble, 2 matvecs (device vectors), factorize, solve_lower."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2104_07146_b200 as hm
from paper_2104_07146_b200 import _chk, _lib

g = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = hm.jittered_grid(g, 1); z = hm.normals(g * g, 1 ^ hm.Z_SEED_XOR)
ctx = hm.default_context()
geo = hm.Geometry(x, 128, 2.0, ctx=ctx)
h = hm.assemble(geo, [1.5, 0.05, 1.0, 0.01], hm.RankControl.fixed_accuracy(1e-6))
print("H bytes", h.stats()["bytes"], flush=True)
dz = torch.from_numpy(z).cuda(); dy = torch.empty_like(dz)
for _ in range(2):
    _chk(_lib.hmgp_hmat_matvec_device(ctx.h, h.h, C.c_void_p(dz.data_ptr()), C.c_void_p(dy.data_ptr())))
torch.cuda.synchronize()
t = time.time()
for _ in range(5):
    _chk(_lib.hmgp_hmat_matvec_device(ctx.h, h.h, C.c_void_p(dz.data_ptr()), C.c_void_p(dy.data_ptr())))
torch.cuda.synchronize()
print(f"matvec {1e3 * (time.time() - t) / 5:.3f} ms", flush=True)
if len(sys.argv) > 2 and sys.argv[2] == "solve":
    f = hm.factorize(h, 1e-6, "cholesky")
    print("factor bytes", f.info["storage_bytes"], flush=True)
    f.solve_lower(z)
    t = time.time(); f.solve_lower(z); print(f"solve_lower {1e3 * (time.time() - t):.2f} ms")
