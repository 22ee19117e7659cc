"""Dense diagnostics on the device: HMatrix::to_dense
(hmatrix.cpp:274-297), HFactor::lower_dense / reconstruct (hfactor.cpp:421-449).

Ports of /root/reference/proj/tests/test_hmatrix.cpp:41-106 and
test_hfactor.cpp:71-99; the dense covariance they compare against is built from
the CPU oracle's kernel entries (cov_dense semantics)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def cov_dense(oracle, x, th):
    n = len(x)
    ii, jj = np.meshgrid(np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32), indexing="ij")
    return oracle.kernel_pairs(x, th, ii.ravel(), jj.ravel()).reshape(n, n)


def test_to_dense_matches_dense_covariance(hm, oracle):
    """test_hmatrix.cpp:41-49"""
    x = oracle.random_locations(512, 17)
    th = [1.0, 0.2, 0.5, 0.0]
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, th, hm.RankControl.fixed_accuracy(1e-6))
    c = cov_dense(oracle, x, th)
    d = h.to_dense()
    assert np.linalg.norm(c - d) / np.linalg.norm(c) <= 1e-5
    assert np.array_equal(d, d.T)  # test_hmatrix.cpp:108-118: exactly symmetric
    # dense leaves hold the kernel entries themselves (≤ 1e-10 relative)
    leaves = g.blocks()
    perm = g.perm()
    for (r0, r1, c0, c1, tag) in leaves[:50]:
        if tag == 1 and c0 <= r0:  # dense, lower-stored
            ri, ci = perm[r0:r1], perm[c0:c1]
            assert np.allclose(d[np.ix_(ri, ci)], c[np.ix_(ri, ci)], rtol=1e-10, atol=0.0)


def test_to_dense_fixed_rank(hm, oracle):
    """test_hmatrix.cpp:51-60 and 100-106"""
    x = oracle.random_locations(512, 21)
    th = [1.0, 0.2, 0.5, 0.0]
    g = hm.Geometry(x, 32, 2.0)
    c = cov_dense(oracle, x, th)
    e4 = np.linalg.norm(c - hm.assemble(g, th, hm.RankControl.fixed_rank(4)).to_dense())
    e16 = np.linalg.norm(c - hm.assemble(g, th, hm.RankControl.fixed_rank(16)).to_dense())
    assert e16 <= e4
    x = oracle.random_locations(128, 9)
    th = [2.0, 0.3, 1.5, 0.1]
    g = hm.Geometry(x, 16, 2.0)
    c = cov_dense(oracle, x, th)
    d = hm.assemble(g, th, hm.RankControl.fixed_rank(128)).to_dense()
    assert np.linalg.norm(c - d) / np.linalg.norm(c) <= 1e-12


def test_to_dense_single_point_and_guard(hm):
    """test_hmatrix.cpp:91-98; the n <= 4096 guard (hmatrix.cpp:275-276)"""
    g = hm.Geometry(np.array([[0.4, 0.6]]), 32, 2.0)
    d = hm.assemble(g, [1.2, 0.1, 0.5, 0.3]).to_dense()
    assert abs(d[0, 0] - 1.5) <= 1.5e-14
    g = hm.Geometry(hm.random_locations(4097, 3), 64, 2.0)
    h = hm.assemble(g, [1.0, 0.1, 0.5, 0.01])
    with pytest.raises(ValueError):
        h.to_dense()


@pytest.mark.parametrize("form", ["cholesky", "ldl"])
def test_reconstruction_error_n512(hm, oracle, form):
    """test_hfactor.cpp:71-99: ||L D L^T - C|| / ||C|| <= 1e-4 at eps = 1e-6."""
    x = oracle.random_locations(512, 31)
    th = [1.0, 0.1, 0.5, 0.01]
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, th, hm.RankControl.fixed_accuracy(1e-6))
    f = hm.factorize(h, 1e-6, form)
    c = cov_dense(oracle, x, th)
    rec = f.reconstruct()
    assert np.linalg.norm(rec - c) / np.linalg.norm(c) <= 1e-4
    L = f.lower_dense()
    assert np.all(np.triu(L, 1) == 0.0)
    d = np.diag(L)
    if form == "ldl":
        assert np.all(d == 1.0)
    else:  # Cholesky: L_ii is the factor diagonal (tree order)
        assert np.all(d > 0.0)
    # the factor's own solve agrees with its reconstruction
    b = np.sin(np.arange(512.0))
    xs = f.solve_factored(b)
    assert np.linalg.norm(rec @ xs - b) <= 1e-8 * np.linalg.norm(b) * np.linalg.cond(rec)
