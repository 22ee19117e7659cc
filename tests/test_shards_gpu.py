"""Sharded leaf assembly (SURVEY.md §8e, C2 on 1/2/4/8 GPUs) on one device:
every shard's leaves must be bit-identical to the full assembly's
(hmatrix.cpp:174-221 assembles each leaf independently), the shards' leaf
ranges must partition the stored-leaf list, and a shard must refuse the
whole-matrix operations."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check_shards(hm, x, leaf, eps, th, worlds, data=True):
    g = hm.Geometry(x, leaf, 2.0)
    rc = hm.RankControl.fixed_accuracy(eps)
    full = hm.assemble(g, th, rc)
    fl = full.leaves()
    L = len(fl)
    for world in worlds:
        covered = np.zeros(L, dtype=int)
        prev_end = 0
        for s in range(world):
            h = hm.assemble_shard(g, th, s, world, rc)
            lb, le = h.leaf_range
            assert lb == prev_end
            prev_end = le
            covered[lb:le] += 1
            sl = h.leaves()
            assert np.array_equal(sl[:, :4], fl[:, :4])            # same block structure
            # in range: same kind (incl. rank-driven coarsening to dense) and rank;
            # outside, the kind is the structural one (no rank, no coarsening)
            assert np.array_equal(sl[lb:le, 4:], fl[lb:le, 4:])
            assert np.all(sl[:lb, 5] == -2) and np.all(sl[le:, 5] == -2)
            if data:
                for k in range(lb, le):
                    d1, d2 = full.leaf_data(k, fl[k]), h.leaf_data(k, sl[k])
                    if isinstance(d1, tuple):
                        assert all(np.array_equal(p, q) for p, q in zip(d1, d2))
                    else:
                        assert np.array_equal(d1, d2)
            if world > 1 and le - lb < L:
                with pytest.raises(ValueError):
                    h.matvec(np.ones(len(x)))
        assert prev_end == L and np.all(covered == 1)


def test_assembly_shards_c1_bit_identical(hm):
    x = hm.jittered_grid(64, 1)
    _check_shards(hm, x, 64, 1e-7, [1.0, 0.1, 0.5, 0.01], (1, 2, 3, 4, 8))


def test_assembly_shards_general_nu_3d(hm):
    x = hm.random_locations(6000, 5, dim=3)
    _check_shards(hm, x, 64, 1e-6, [1.0, 0.15, 0.325, 0.01], (2, 8))


def test_assembly_shards_c2_ranks(hm):
    """C2 size (n = 65 536, leaf 64, ε = 1e-7, general ν): ranks of 8 shards."""
    x = hm.jittered_grid(256, 1)
    _check_shards(hm, x, 64, 1e-7, [1.0, 0.1, 0.325, 0.01], (8,), data=False)


def test_assembly_shard_refuses_factorize(hm):
    x = hm.jittered_grid(32, 1)
    g = hm.Geometry(x, 64, 2.0)
    h = hm.assemble_shard(g, [1.0, 0.1, 0.5, 0.01], 0, 2)
    with pytest.raises(ValueError):
        hm.h_cholesky(h, 1e-7)
    with pytest.raises(ValueError):
        hm.assemble_shard(g, [1.0, 0.1, 0.5, 0.01], 2, 2)
