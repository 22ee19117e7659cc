"""sample_grf at C4 size (n = 65536) on the device: timing and a moment check."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2104_07146_b200 as hm
x = hm.jittered_grid(256, 1)
t = time.time()
z = hm.sample_grf(x, [1.0, 0.1, 0.5, 0.01], 1 ^ 0x517CC1B727220A95)
print(f"sample_grf n=65536: {time.time()-t:.2f} s, mean {z.mean():.4f} var {z.var():.4f} "
      f"finite {np.isfinite(z).all()}", flush=True)
