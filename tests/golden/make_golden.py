"""Generate the committed golden fixtures from the UNMODIFIED reference build
(oracle/_ref/libhmgp_ref.so = /root/reference/proj/src/{geometry,covkernel}.cpp).

    python tests/golden/make_golden.py

geometry_c1.npz : C1 input (64x64 jittered grid, seed 1), leaf 64, eta 2 ->
                  reference perm and block list (DFS order)
kernel_ref.npz  : reference KernelEvaluator::at_distance over 4000 distances
                  for 8 orders (closed forms, half-integer, general nu)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, RefLib  # noqa: E402


def main():
    ref = RefLib()
    o = Oracle()
    x = o.jittered_grid(64, 1)
    perm = ref.cluster_perm(x, 64)
    blocks, na, nd = ref.block_leaves(x, 64, 2.0)
    np.savez_compressed(os.path.join(HERE, "geometry_c1.npz"), x=x, leaf=64, eta=2.0, perm=perm,
                        blocks=blocks, n_adm=na, n_dense=nd)
    rng = np.random.default_rng(12345)
    h = np.concatenate([10 ** rng.uniform(-11, 1.2, 3998), [0.0, 1e-12]])
    nus = np.array([0.5, 1.5, 2.5, 3.5, 0.325, 1.0, 0.82, 7.3])
    vals = np.stack([ref.at_distance([1.4, 0.07, nu, 0.3], h) for nu in nus])
    np.savez_compressed(os.path.join(HERE, "kernel_ref.npz"), h=h, nu=nus, sigma2=1.4, ell=0.07,
                        tau2=0.3, values=vals)
    print("wrote geometry_c1.npz, kernel_ref.npz", perm.shape, blocks.shape, vals.shape)


if __name__ == "__main__":
    main()
