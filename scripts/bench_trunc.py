"""Time the batched recompression kernels on synthetic items (developer tool).

usage: python scripts/bench_trunc.py [route ...]   route: 0 single CTA, 1 pair, 2 cluster
Prints one line per (shape, route): ms per launch, us per item, kept rank.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2104_07146_b200", "libhmgp_cuda.so"))
f = lib.hmgp_debug_trunc_bench
f.argtypes = [ctypes.c_int] * 7 + [ctypes.c_double, ctypes.c_double,
                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]

# optional: route list, then "m,n,r0,add" shapes
routes = [int(a) for a in sys.argv[1:] if "," not in a] or [0, 1, 2]
user_shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:] if "," in a]
shapes = user_shapes or [(128, 128, 16, 16), (256, 256, 16, 16), (256, 256, 32, 16), (256, 256, 48, 16),
          (512, 512, 32, 16), (1024, 1024, 32, 16), (2048, 2048, 48, 16), (4096, 4096, 48, 16)]
for (m, n, r0, add) in shapes:
    for rt in routes:
        if rt == 1 and max(m, n) >= 512:
            continue
        for count in (1, 148):
            ms = ctypes.c_double()
            keep = ctypes.c_int()
            rc = f(m, n, r0, add, count, rt, 5, 1e-6, float(os.environ.get('DECAY', '0.7')), ctypes.byref(ms), ctypes.byref(keep))
            print(f"m={m:5d} n={n:5d} r={r0+add:3d} route={rt} count={count:3d}: "
                  f"{ms.value:8.3f} ms  {1e3*ms.value/count:8.1f} us/item  keep={keep.value} rc={rc}",
                  flush=True)
