"""CPU tests: pin the oracle (restatement) against the reference's own golden
values and hand cases, and against the UNMODIFIED reference geometry.cpp /
covkernel.cpp build in oracle/_ref when present.  No GPU needed."""
import math

import numpy as np
import pytest

from tests.test_gpu_parity import BESSEL_TABLE


def rel(a, b):
    return abs(a - b) / abs(b)


def test_bessel_table(oracle):
    """test_covkernel.cpp:66-93"""
    for nu, x, v in BESSEL_TABLE:
        assert rel(oracle.bessel_k(nu, x), v) < 1e-12
        assert rel(oracle.bessel_k(nu, x, generic=True), v) < 1e-12


def test_half_integer_identities(oracle):
    """test_covkernel.cpp:54-64"""
    assert rel(oracle.bessel_k(0.5, 1.0), 0.46106850444789456) < 1e-14
    for x in (0.02, 0.7, 1.9, 3.5, 20.0, 300.0):
        kh = math.sqrt(math.pi / (2 * x)) * math.exp(-x)
        assert rel(oracle.bessel_k(0.5, x), kh) < 1e-14
        assert rel(oracle.bessel_k(1.5, x), kh * (1 + 1 / x)) < 1e-14
        assert rel(oracle.bessel_k(0.5, x, generic=True), kh) < 1e-12
        assert rel(oracle.bessel_k(1.5, x, generic=True), kh * (1 + 1 / x)) < 1e-12


def test_matern_golden(oracle):
    """test_covkernel.cpp:29-52"""
    assert oracle.matern(0.0, [2.0, 0.3, 0.7, 0.25]) == 2.25
    assert oracle.matern(0.0, [1.5, 0.1, 1.2, 0.0]) == 1.5
    assert rel(oracle.matern(1.0, [1.0, 1.0, 0.5, 0.0]), 0.36787944117144233) < 1e-13
    assert rel(oracle.matern(1.0, [1.0, 1.0, 1.5, 0.0]), 0.73575888234288464) < 1e-13
    assert rel(oracle.matern(1.0, [1.0, 1.0, 0.5, 0.0], generic=True), 0.36787944117144233) < 1e-12
    assert rel(oracle.matern(0.7, [1.3, 0.2, 0.6, 0.0]), 0.050105793549337933) < 1e-12
    assert rel(oracle.matern(0.05, [2.0, 0.1, 2.5, 0.0]), 1.9206804224233392) < 1e-13
    assert rel(oracle.matern(0.3, [1.0, 0.1, 1.5, 0.0]), 0.19914827347145577) < 1e-13


def test_generic_vs_closed_forms(oracle):
    """acceptance_main.cpp:70-82: generic path equals the closed forms to 1e-12."""
    t = 1e-6 * (50.0 / 1e-6) ** (np.arange(0, 10001, 7) / 10000.0)
    for nu in (0.5, 1.5, 2.5):
        closed = {0.5: np.exp(-t), 1.5: (1 + t) * np.exp(-t), 2.5: (1 + t + t * t / 3) * np.exp(-t)}[nu]
        got = np.array([oracle.matern(h, [1.7, 1.0, nu, 0.0], generic=True) for h in t])
        assert np.max(np.abs(got - 1.7 * closed) / (1.7 * closed)) < 1e-12


def test_domain_and_validation(oracle):
    from oracle.oracle import OracleError
    for nu, x in ((0.5, 0.0), (0.5, -1.0), (-1.0, 1.0)):
        with pytest.raises(OracleError) as e:
            oracle.bessel_k(nu, x)
        assert e.value.code == 2
    assert 0 <= oracle.bessel_k(0.5, 800.0) < 1e-300
    for th in ([0.0, 1, 0.5, 0], [1, -1, 0.5, 0], [1, 1, 0.0, 0], [1, 1, 0.5, -0.1]):
        with pytest.raises(OracleError):
            oracle.matern(1.0, th)


def test_normal_quantile(oracle):
    """test_simgen.cpp:10-29 (AS241)"""
    refs = [(0.975, 1.9599639845400542), (1e-10, -6.3613409024040562), (0.3, -0.52440051270804078),
            (1e-12, -7.0344838253011319), (0.0001, -3.7190164854556806), (0.6, 0.2533471031357998)]
    assert oracle.normal_quantile(0.5) == 0.0
    for p, x in refs:
        assert rel(oracle.normal_quantile(p), x) < 1e-13


def test_loglik_hand_cases(oracle):
    """test_loglik_mle.cpp:13-33"""
    from oracle.oracle import make_config
    r = oracle.loglik(np.array([[0.5, 0.5]]), np.zeros(1), [0.75, 0.1, 0.5, 0.25], make_config())
    assert abs(r.loglik - -0.9189385332046727) < 1e-14
    r2 = oracle.loglik(np.array([[0.0, 0.0], [1.0, 1.0]]), np.ones(2), [0.5, 1e-3, 0.5, 0.5],
                       make_config())
    assert rel(r2.loglik, -math.log(2 * math.pi) - 1.0) < 1e-10


def test_oracle_h_vs_dense_small(oracle):
    """test_loglik_mle.cpp:35-44: H vs dense within 1e-4 (the reference bar)."""
    from oracle.oracle import make_config
    x = oracle.random_locations(512, 4)
    th = [1.5, 0.1, 1.5, 1e-4]
    z = oracle.sample_grf(x, th, 99)
    for form in ("ldl", "cholesky"):
        got = oracle.loglik(x, z, th, make_config(eps=1e-6, form=form)).loglik
        want = oracle.dense_loglik(x, z, th)[0]
        assert rel(got, want) < 1e-4


def test_oracle_identical_points_fail(oracle):
    from oracle.oracle import OracleError, make_config
    with pytest.raises(OracleError) as e:
        oracle.loglik(np.tile([[0.25, 0.75]], (6, 1)), np.ones(6), [1.0, 0.1, 0.5, 0.0], make_config())
    assert e.value.code == 4 and "nugget" in str(e.value)


def test_oracle_predict_vs_dense(oracle):
    """test_krige_metrics.cpp:31-43"""
    from oracle.oracle import make_config
    allp = oracle.random_locations(576, 10)
    train, test = allp[:512], allp[512:]
    th = [1.5, 0.1, 1.5, 1e-4]
    z = oracle.sample_grf(allp, th, 44)[:512]
    got = oracle.predict(train, z, test, th, make_config(eps=1e-6))
    want = oracle.dense_predict(train, z, test, th)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-4


# ---------------------------------------------- pin against oracle/_ref ----
def _ref():
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref (reference build) not present")
    return RefLib()


def test_pin_geometry_against_reference_build(oracle):
    ref = _ref()
    rng = np.random.default_rng(1)
    cases = [(oracle.jittered_grid(64, 1), 64), (oracle.random_locations(2000, 3), 32),
             (np.array([[i / 8.0, j / 8.0] for i in range(8) for j in range(8)]), 16),
             (np.round(rng.random((777, 2)), 2), 8)]
    for x, leaf in cases:
        assert np.array_equal(oracle.cluster_perm(x, leaf), ref.cluster_perm(x, leaf))
        for eta in (0.5, 2.0, 100.0):
            a, na, nd = oracle.block_leaves(x, leaf, eta)
            b, nb, ne = ref.block_leaves(x, leaf, eta)
            assert (na, nd) == (nb, ne)
            assert np.array_equal(a, b)


def test_pin_kernel_against_reference_build(oracle):
    ref = _ref()
    rng = np.random.default_rng(2)
    h = np.concatenate([10 ** rng.uniform(-11, 1, 3000), [0.0, 1e-12]])
    for nu in (0.5, 1.5, 2.5, 3.5, 0.325, 1.0, 0.82, 7.3):
        th = [1.4, 0.07, nu, 0.3]
        a, b = oracle.at_distance(th, h), ref.at_distance(th, h)
        assert np.array_equal(a, b), nu  # same compiler, same operations -> bit-identical
    for nu, x, _ in BESSEL_TABLE:
        assert oracle.bessel_k(nu, x) == ref.bessel_k(nu, x)


def test_oracle_against_committed_reference_fixtures(oracle):
    """tests/golden/*.npz were produced by the reference build (make_golden.py)."""
    import os
    d = os.path.join(os.path.dirname(__file__), "golden")
    g = np.load(os.path.join(d, "geometry_c1.npz"))
    assert np.array_equal(oracle.cluster_perm(g["x"], int(g["leaf"])), g["perm"])
    b, na, nd = oracle.block_leaves(g["x"], int(g["leaf"]), float(g["eta"]))
    assert np.array_equal(b, g["blocks"]) and (na, nd) == (int(g["n_adm"]), int(g["n_dense"]))
    k = np.load(os.path.join(d, "kernel_ref.npz"))
    for nu, want in zip(k["nu"], k["values"]):
        got = oracle.at_distance([float(k["sigma2"]), float(k["ell"]), float(nu), float(k["tau2"])], k["h"])
        assert np.array_equal(got, want)
