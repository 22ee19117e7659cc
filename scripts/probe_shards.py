"""C2 sharded assembly balance on one device: each of G shards' assembly timed
alone (what one GPU of a G-GPU job does), vs the full assembly.  Reports the
per-shard device ms, the max/mean imbalance and the leaf ranges."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2104_07146_b200 as hm

x = hm.jittered_grid(256, 1)
ctx = hm.default_context()
g = hm.Geometry(x, 64, 2.0, ctx=ctx)
rc = hm.RankControl.fixed_accuracy(1e-7)


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t) * 1e3


for nu in (0.5, 1.5, 0.325):
    th = [1.0, 0.1, nu, 0.01]
    timed(lambda: hm.assemble(g, th, rc))  # warm-up
    _, full_ms = timed(lambda: hm.assemble(g, th, rc))
    for G in (2, 4, 8):
        ms, ranges = [], []
        for s in range(G):
            h, t = timed(lambda: hm.assemble_shard(g, th, s, G, rc))
            ms.append(t)
            ranges.append(h.leaf_range)
            del h
        ms = np.array(ms)
        print(f"nu={nu} G={G}: full {full_ms:.1f} ms, shards max {ms.max():.1f} mean {ms.mean():.1f} "
              f"(imbalance {ms.max() / ms.mean():.2f}, projected speed-up {full_ms / ms.max():.2f}x) "
              f"ranges {ranges}", flush=True)
