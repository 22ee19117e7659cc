"""Dense kriging variance and MLOE/MMOM.

kriging_variance_dense (krige.cpp:46-74) and mloe_mmom (metrics.cpp:17-69).
The CPU tests pin the oracle restatement (oracle/hmgp_oracle.cpp
orc_kriging_variance_dense / orc_mloe_mmom) on the reference's own cases from
/root/reference/proj/tests/test_krige_metrics.cpp; the GPU tests compare the
device path (hmgp_kriging_variance_dense / hmgp_mloe_mmom through the C ABI) with
that oracle on the same seeded inputs, and rerun the reference cases on it.
"""
import numpy as np
import pytest


def cov_dense(oracle, x, th):
    """cov_dense (covkernel.cpp:262-275) from the oracle's kernel entries."""
    n = len(x)
    ii, jj = np.meshgrid(np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32), indexing="ij")
    return oracle.kernel_pairs(x, th, ii.ravel(), jj.ravel()).reshape(n, n)


def cross(oracle, train, test, th):
    h = np.sqrt(((test[:, None, :] - train[None, :, :]) ** 2).sum(-1))
    return oracle.at_distance(th, h.ravel()).reshape(len(test), len(train))


# ------------------------------------------------------------- oracle pins (CPU)
def test_oracle_variance_coincident_far_bounds(oracle):
    """test_krige_metrics.cpp:80-91"""
    train = oracle.random_locations(256, 9)
    test = np.array([train[17], [123.0, -55.0]])
    v = oracle.kriging_variance_dense(train, test, [2.0, 0.1, 1.5, 0.0])
    assert abs(v[0]) <= 1e-10
    assert v[1] == pytest.approx(2.0, rel=1e-12)
    assert np.all(v >= 0.0) and np.all(v <= 2.0 + 1e-12)


def test_oracle_variance_explicit_inverse(oracle):
    """test_krige_metrics.cpp:93-109 (explicit-inverse oracle at n = 128)"""
    allp = oracle.random_locations(160, 13)
    train, test = allp[:128], allp[128:]
    th = [1.3, 0.12, 0.7, 0.05]
    got = oracle.kriging_variance_dense(train, test, th)
    cinv = np.linalg.inv(cov_dense(oracle, train, th))
    c = cross(oracle, train, test, th)
    want = (th[0] + th[3]) - np.einsum("ij,jk,ik->i", c, cinv, c)
    np.testing.assert_allclose(got, want, rtol=1e-10)


def test_oracle_mloe_special_cases(oracle):
    """test_krige_metrics.cpp:137-145, 212-233"""
    t = [1.5, 0.1, 0.5, 0.0]
    lo, mo = oracle.mloe_mmom(oracle.random_locations(64, 20), t, t, M=64)
    assert abs(lo) <= 1e-8 and abs(mo) <= 1e-8
    lo, mo = oracle.mloe_mmom(oracle.random_locations(64, 30), t, [0.6, 0.1, 0.5, 0.0], M=64)
    assert abs(lo) <= 1e-10 and abs(mo) > 0.1
    pts = oracle.random_locations(64, 40)
    for a in ([2.0, 0.3, 0.5, 0.0], [0.5, 0.02, 2.5, 1e-2], [1.5, 0.1, 1.0, 0.5]):
        assert oracle.mloe_mmom(pts, [1.5, 0.1, 1.0, 1e-4], a, M=64)[0] >= -1e-10


def test_oracle_mloe_monte_carlo(oracle):
    """test_krige_metrics.cpp:147-193: closed forms vs 1e5 common-random-number
    replicates at n = 32 (normals from mt19937_64(999) as the reference draws them)."""
    n, reps = 32, 100000
    pts = oracle.random_locations(n, 3)
    tt, ta = [1.5, 0.1, 0.5, 0.0], [1.0, 0.1, 0.5, 0.0]
    lo, mo = oracle.mloe_mmom(pts, tt, ta, M=n)
    ct, ca = cov_dense(oracle, pts, tt), cov_dense(oracle, pts, ta)
    it, ia = np.linalg.inv(ct), np.linalg.inv(ca)
    wt = -it / np.diag(it)[None, :]
    wa = -ia / np.diag(ia)[None, :]
    lt, la = np.linalg.cholesky(ct), np.linalg.cholesky(ca)
    g = oracle.normals(n * reps, 999).reshape(reps, n)
    zt, za = g @ lt.T, g @ la.T
    att = ((zt @ wt) ** 2).sum(0)
    ata = ((zt @ wa) ** 2).sum(0)
    aaa = ((za @ wa) ** 2).sum(0)
    assert abs(lo - np.mean(ata / att - 1.0)) <= 1e-3
    assert abs(mo - np.mean(aaa / ata - 1.0)) <= 1e-3


def test_oracle_guards(oracle):
    """test_krige_metrics.cpp:235-244 and krige.cpp:52-54"""
    from oracle.oracle import OracleError
    pts = oracle.random_locations(8, 1)
    t = [1, 0.1, 0.5, 0]
    with pytest.raises(OracleError):
        oracle.mloe_mmom(pts, t, t, M=0)
    with pytest.raises(OracleError):
        oracle.mloe_mmom(pts, t, t, M=4, dense_guard=4)
    with pytest.raises(OracleError):
        oracle.kriging_variance_dense(oracle.random_locations(4097, 1), pts, t)


# ---------------------------------------------------------------- GPU parity
@pytest.mark.gpu
@pytest.mark.parametrize("n,m,th,dim", [
    (256, 300, [2.0, 0.1, 1.5, 0.0], 2),
    (1000, 777, [1.3, 0.12, 0.7, 0.05], 2),      # general-ν Bessel path
    (4096, 300, [1.0, 0.1, 0.5, 0.01], 2),       # maximum n
    (300, 5000, [1.0, 0.1, 1.5, 0.01], 2),       # two column batches
    (800, 200, [1.0, 0.2, 2.5, 0.005], 3),
])
def test_gpu_variance_matches_oracle(hm, oracle, n, m, th, dim):
    train = oracle.random_locations(n, 100 + n, dim=dim)
    test = oracle.random_locations(m, 200 + m, dim=dim)
    test[:5] = train[:5]  # interpolation points
    got = hm.kriging_variance_dense(train, test, th)
    want = oracle.kriging_variance_dense(train, test, th)
    prior = th[0] + th[3]
    # dense FP64 solves, different summation order: absolute to the prior variance
    np.testing.assert_allclose(got, want, rtol=1e-8, atol=1e-9 * prior)
    assert np.all(got >= -1e-9)


@pytest.mark.gpu
def test_gpu_variance_reference_cases(hm, oracle):
    """test_krige_metrics.cpp:80-109 on the device"""
    train = oracle.random_locations(256, 9)
    v = hm.kriging_variance_dense(train, np.array([train[17], [123.0, -55.0]]), [2.0, 0.1, 1.5, 0.0])
    assert abs(v[0]) <= 1e-10 and v[1] == pytest.approx(2.0, rel=1e-12)
    allp = oracle.random_locations(160, 13)
    th = [1.3, 0.12, 0.7, 0.05]
    got = hm.kriging_variance_dense(allp[:128], allp[128:], th)
    cinv = np.linalg.inv(cov_dense(oracle, allp[:128], th))
    c = cross(oracle, allp[:128], allp[128:], th)
    np.testing.assert_allclose(got, (th[0] + th[3]) - np.einsum("ij,jk,ik->i", c, cinv, c), rtol=1e-10)
    assert hm.kriging_variance_dense(train, np.empty((0, 2)), th).size == 0


@pytest.mark.gpu
def test_gpu_variance_errors(hm):
    t = [1.0, 0.1, 0.5, 0.0]
    with pytest.raises(ValueError):
        hm.kriging_variance_dense(np.empty((0, 2)), np.zeros((1, 2)), t)
    with pytest.raises(ValueError):
        hm.kriging_variance_dense(np.random.rand(4097, 2), np.zeros((1, 2)), t)
    with pytest.raises(ValueError):
        hm.kriging_variance_dense(np.random.rand(8, 2), np.zeros((1, 2)), [1.0, -0.1, 0.5, 0.0])
    with pytest.raises(RuntimeError):  # duplicate points without nugget: C11 singular
        hm.kriging_variance_dense(np.array([[0.3, 0.3], [0.3, 0.3]]), np.zeros((1, 2)), t)


@pytest.mark.gpu
@pytest.mark.parametrize("n,M,seed,tt,ta,dim", [
    (64, 64, 0, [1.5, 0.1, 0.5, 0.0], [0.9, 0.15, 1.0, 1e-3], 2),
    (500, 100, 7, [1.0, 0.1, 0.5, 0.01], [1.2, 0.08, 0.5, 0.01], 2),
    (2048, 1000, 3, [1.5, 0.1, 1.0, 1e-4], [0.5, 0.02, 2.5, 1e-2], 2),
    (4096, 300, 11, [1.0, 0.1, 0.5, 0.01], [1.0, 0.12, 0.7, 0.02], 2),
    (400, 400, 5, [1.0, 0.2, 1.5, 0.01], [1.0, 0.1, 0.5, 0.01], 3),
])
def test_gpu_mloe_matches_oracle(hm, oracle, n, M, seed, tt, ta, dim):
    x = oracle.random_locations(n, 50 + n, dim=dim)
    got = hm.mloe_mmom(x, tt, ta, hm.MetricConfig(M=M, seed=seed))
    lo, mo = oracle.mloe_mmom(x, tt, ta, M=M, seed=seed)
    assert got.mloe == pytest.approx(lo, rel=1e-6, abs=1e-10)
    assert got.mmom == pytest.approx(mo, rel=1e-6, abs=1e-10)


@pytest.mark.gpu
def test_gpu_mloe_reference_cases(hm, oracle):
    """test_krige_metrics.cpp:137-244 on the device"""
    t = [1.5, 0.1, 0.5, 0.0]
    cfg = hm.MetricConfig(M=64)
    r = hm.mloe_mmom(oracle.random_locations(64, 20), t, t, cfg)
    assert abs(r.mloe) <= 1e-8 and abs(r.mmom) <= 1e-8
    r = hm.mloe_mmom(oracle.random_locations(64, 30), t, [0.6, 0.1, 0.5, 0.0], cfg)
    assert abs(r.mloe) <= 1e-10 and abs(r.mmom) > 0.1
    pts = oracle.random_locations(64, 12)
    sh = pts.copy()
    perm = np.random.default_rng(5).permutation(64)
    sh = sh[perm]
    a, b = [1.5, 0.08, 0.5, 0.0], [0.9, 0.15, 1.0, 1e-3]
    r1, r2 = hm.mloe_mmom(pts, a, b, cfg), hm.mloe_mmom(sh, a, b, cfg)
    assert r1.mloe == pytest.approx(r2.mloe, rel=1e-10)
    assert r1.mmom == pytest.approx(r2.mmom, rel=1e-10)
    pts = oracle.random_locations(64, 40)
    for b in ([2.0, 0.3, 0.5, 0.0], [0.5, 0.02, 2.5, 1e-2], [1.5, 0.1, 1.0, 0.5]):
        assert hm.mloe_mmom(pts, [1.5, 0.1, 1.0, 1e-4], b, cfg).mloe >= -1e-10
    small = oracle.random_locations(8, 1)
    with pytest.raises(ValueError):
        hm.mloe_mmom(small, t, t, hm.MetricConfig(M=0))
    with pytest.raises(ValueError):
        hm.mloe_mmom(small, t, t, hm.MetricConfig(M=4, dense_guard=4))
    with pytest.raises(ValueError):
        hm.mloe_mmom(small[:1], t, t, cfg)


def test_rmse_hand_values(hm):
    """test_krige_metrics.cpp:111-123 (host arithmetic)"""
    assert hm.rmse([1, 1], [1, 1]) == 0.0
    assert hm.rmse([1, 1], [0, 0]) == 1.0
    assert hm.rmse([1, 2, 3], [0, 0, 0]) == pytest.approx(2.1602468994692869, rel=1e-14)
    with pytest.raises(ValueError):
        hm.rmse([1, 1], [1, 2, 3])
    with pytest.raises(ValueError):
        hm.rmse([], [])


@pytest.mark.gpu
def test_gpu_mloe_beyond_4096_with_guard(hm, oracle):
    """dense_guard above the default (metrics.hpp:16): n = 6000, size-independent
    properties (matching models -> 0; pure σ² misspecification -> MLOE 0)."""
    x = oracle.random_locations(6000, 77)
    t = [1.0, 0.1, 0.5, 0.01]
    cfg = hm.MetricConfig(M=200, seed=1, dense_guard=8192)
    r = hm.mloe_mmom(x, t, t, cfg)
    assert abs(r.mloe) <= 1e-8 and abs(r.mmom) <= 1e-8
    r = hm.mloe_mmom(x, t, [0.5, 0.1, 0.5, 0.005], cfg)  # (σ², τ²) scaled together
    assert abs(r.mloe) <= 1e-8 and r.mmom == pytest.approx(-0.5, rel=1e-8)
    with pytest.raises(ValueError):
        hm.mloe_mmom(x, t, t, hm.MetricConfig(M=10))  # default guard 4096
