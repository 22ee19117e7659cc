"""cudaMalloc / cudaMemset / cudaFree cost of the large per-evaluation buffers
(factor pool, ACA staging chunks) on this device."""
import time
from cuda.bindings import runtime as rt

rt.cudaSetDevice(0)
rt.cudaFree(0)
for gb in (0.5, 2, 4, 8, 16):
    n = int(gb * (1 << 30))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        err, p = rt.cudaMalloc(n)
        t1 = time.perf_counter()
        rt.cudaMemset(p, 0, n)
        rt.cudaDeviceSynchronize()
        t2 = time.perf_counter()
        rt.cudaFree(p)
        rt.cudaDeviceSynchronize()
        t3 = time.perf_counter()
        ts.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))
    print(f"{gb:5.1f} GB  malloc/memset/free ms: " + "  ".join(f"{a:.2f}/{b:.2f}/{c:.2f}" for a, b, c in ts))
