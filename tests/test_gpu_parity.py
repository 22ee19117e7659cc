"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE north_star): bit-exact permutation and block partition;
relative 1e-10 on kernel entries; relative 1e-6 on L(θ) and predictions; L(θ)
also against the dense FP64 oracle at small n.  Reference test analogues are
cited per test (paths under /root/reference/proj/tests).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NU_SET = [0.5, 1.5, 2.5, 0.325, 1.0, 0.82, 3.5, 0.7]


def rel(a, b):
    return abs(a - b) / abs(b)


# --------------------------------------------------------------- geometry --
def point_sets(oracle):
    rng = np.random.default_rng(3)
    grid8 = np.array([[i / 8.0, j / 8.0] for i in range(8) for j in range(8)])
    signed0 = np.array([[0.0, 0.0], [-0.0, 0.5], [0.0, -0.0], [1.0, -0.0], [-0.0, 1.0],
                        [0.5, 0.5], [0.25, 0.75], [0.75, 0.25]] * 5)
    return {
        "C1_jittered_64x64_leaf64": (oracle.jittered_grid(64, 1), 64),
        "uniform_500_leaf32": (oracle.random_locations(500, 99), 32),
        "uniform_3001_leaf16": (oracle.random_locations(3001, 7), 16),
        "grid8_ties_leaf16": (grid8, 16),
        "signed_zero_ties_leaf4": (signed0, 4),
        "clustered_2000_leaf32": (np.concatenate([rng.random((1000, 2)) * 0.1,
                                                  10 + rng.random((1000, 2)) * 0.1]), 32),
        "single_point": (np.array([[0.3, 0.7]]), 32),
        "duplicates_leaf8": (np.repeat(oracle.random_locations(40, 5), 3, axis=0), 8),
    }


def test_geometry_bit_exact_vs_oracle(hm, oracle):
    for name, (x, leaf) in point_sets(oracle).items():
        for eta in (2.0, 0.5):
            g = hm.Geometry(x, leaf, eta)
            assert np.array_equal(g.perm(), oracle.cluster_perm(x, leaf)), name
            inv = g.inverse_perm()
            assert np.array_equal(g.perm()[inv], np.arange(len(x))), name
            ob, na, nd = oracle.block_leaves(x, leaf, eta)
            gb = g.blocks()
            cnt, gna, gnd = g.block_counts()
            assert (gna, gnd) == (na, nd), name
            assert np.array_equal(gb, ob), name


def test_geometry_bit_exact_vs_reference_build(hm, oracle):
    """Against the UNMODIFIED reference geometry.cpp (oracle/_ref), when built."""
    from oracle.oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    for name, (x, leaf) in point_sets(oracle).items():
        g = hm.Geometry(x, leaf, 2.0)
        assert np.array_equal(g.perm(), ref.cluster_perm(x, leaf)), name
        rb, na, nd = ref.block_leaves(x, leaf, 2.0)
        assert np.array_equal(g.blocks(), rb), name


def test_geometry_3d_vs_oracle(hm, oracle):
    x = oracle.random_locations(5000, 11, dim=3)
    g = hm.Geometry(x, 64, 2.0)
    assert np.array_equal(g.perm(), oracle.cluster_perm(x, 64))
    ob, na, nd = oracle.block_leaves(x, 64, 2.0)
    assert np.array_equal(g.blocks(), ob)


def test_geometry_golden_fixture(hm):
    """Committed fixture generated from the reference build (tests/golden/make_golden.py)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "geometry_c1.npz")
    if not os.path.exists(path):
        pytest.skip("fixture not generated")
    f = np.load(path)
    g = hm.Geometry(f["x"], int(f["leaf"]), float(f["eta"]))
    assert np.array_equal(g.perm(), f["perm"])
    assert np.array_equal(g.blocks(), f["blocks"])


def test_geometry_validation(hm):
    with pytest.raises(ValueError, match="empty dataset"):
        hm.Geometry(np.zeros((0, 2)), 32)
    with pytest.raises(ValueError, match="invalid location"):
        hm.Geometry(np.array([[0.1, np.nan]]), 32)
    with pytest.raises(ValueError):
        hm.Geometry(np.array([[0.1, 0.2]]), 0)
    with pytest.raises(ValueError, match="eta"):
        hm.Geometry(np.array([[0.1, 0.2]]), 32, 0.0)


# ----------------------------------------------------------------- kernel --
BESSEL_TABLE = [  # test_covkernel.cpp:70-86
    (1.0, 1.0, 0.60190723019723457), (0.3, 0.5, 0.97647412438178792),
    (0.6, 1.0, 0.47971569489286612), (1.0, 1e-6, 999999.99999278428),
    (2.7, 3.2, 0.072917852205606608), (5.5, 10.0, 7.3304530079850216e-5),
    (10.0, 0.01, 1.8579404390480640e+28), (25.0, 30.0, 3.7775319791336277e-10),
    (0.9, 650.0, 2.5140676518253439e-284), (7.3, 2.0, 543.63827738445926),
    (12.6, 0.37, 1.4985106123100319e+17), (3.0, 1e-8, 7.9999999999999999e+24),
    (0.01, 0.02, 4.0298381770492421), (24.5, 1e-8, 1.4946625757169951e+226),
    (1.9, 700.0, 4.6818247046354968e-306),
]


def test_bessel_golden_on_device(hm):
    nu = np.array([r[0] for r in BESSEL_TABLE])
    x = np.array([r[1] for r in BESSEL_TABLE])
    want = np.array([r[2] for r in BESSEL_TABLE])
    for generic in (False, True):
        got = hm.bessel_k(nu, x, generic=generic)
        assert np.all(np.abs(got - want) / want < 1e-12)
    with pytest.raises(hm.DomainError):
        hm.bessel_k([0.5], [0.0])


def test_kernel_entries_1e10(hm, oracle):
    x = oracle.jittered_grid(40, 2)
    rng = np.random.default_rng(0)
    ii = rng.integers(0, len(x), 20000).astype(np.int32)
    jj = rng.integers(0, len(x), 20000).astype(np.int32)
    ii[:50] = jj[:50]  # diagonal -> sigma2 + tau2
    worst = 0.0
    for nu in NU_SET:
        for ell in (0.05, 0.1, 0.3):
            th = [1.3, ell, nu, 0.01]
            got = hm.kernel_pairs(x, th, ii, jj)
            want = oracle.kernel_pairs(x, th, ii, jj)
            worst = max(worst, float(np.max(np.abs(got - want) / np.abs(want))))
    assert worst < 1e-10, worst


def test_at_distance_generic_vs_closed_1e12(hm, oracle):
    """acceptance_main.cpp:70-82 / test_covkernel.cpp:103-115 on the device path."""
    t = 1e-6 * (50.0 / 1e-6) ** (np.arange(2001) / 2000.0)
    for nu in (0.5, 1.5, 2.5):
        closed = {0.5: np.exp(-t), 1.5: (1 + t) * np.exp(-t), 2.5: (1 + t + t * t / 3) * np.exp(-t)}[nu]
        got = hm.at_distance([1.7, 1.0, nu, 0.0], t)
        assert np.max(np.abs(got - 1.7 * closed) / (1.7 * closed)) < 1e-12
        # same distances through the general-order path (nu nudged off the closed form is
        # not the same function; compare the device against the oracle instead)
        want = oracle.at_distance([1.7, 1.0, nu, 0.0], t)
        assert np.max(np.abs(got - want) / want) < 1e-13
    # t < 1e-10 returns sigma2
    assert hm.at_distance([2.0, 1.0, 0.7, 0.1], np.array([1e-12]))[0] == 2.0


def test_kernel_validation(hm):
    x = np.array([[0.1, 0.2], [0.3, 0.4]])
    with pytest.raises(ValueError):
        hm.kernel_pairs(x, [0.0, 1.0, 0.5, 0.0], [0], [1])
    with pytest.raises(IndexError):
        hm.kernel_pairs(x, [1.0, 1.0, 0.5, 0.0], [7], [1])


# --------------------------------------------------------------- assembly --
@pytest.mark.parametrize("nu", [0.5, 0.325, 1.0])
def test_assembly_vs_oracle(hm, oracle, nu):
    """the same partition after coarsening (leaf kinds), and per
    admissible block ||U V^T - U_o V_o^T||_F <= eps ||U_o V_o^T||_F.  Both sides run
    the reference's ACA pivot rules (hmatrix.cpp:13-102); the recompression keeps
    #{sigma_i > eps sigma_0} (hblock.cpp:151-153), so a rank can differ only by
    singular values within rounding of the cut — those are counted and must be
    +-1 with the error bar still met."""
    x = oracle.random_locations(1024, 17)
    th = [1.0, 0.1, nu, 0.01]
    eps = 1e-7
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, th, hm.RankControl.fixed_accuracy(eps))
    pr = oracle.problem(x, 32, 2.0)
    from oracle.oracle import make_config
    pr.assemble(th, make_config(leaf_size=32, eps=eps, threads=4))
    gl, ol = h.leaves(), pr.leaves()
    assert np.array_equal(gl[:, :5], ol[:, :5])  # same stored-leaf layout AND kinds
    ob = oracle.block_leaves(x, 32, 2.0)[0]
    dense_geom = {tuple(b[:4]) for b in ob if b[4] == 1}
    worst_dense, worst_lr, rank_diff = 0.0, 0.0, 0
    for k in range(len(gl)):
        if gl[k, 4] == 1:
            a, b = h.leaf_data(k, gl[k]), pr.leaf_data(k, ol[k])
            if tuple(gl[k, :4]) in dense_geom:  # kernel leaf: entries
                assert np.max(np.abs(a - b) / np.abs(b)) < 1e-10
            else:  # coarsened admissible block: U V^T product
                worst_dense = max(worst_dense, np.linalg.norm(a - b) / np.linalg.norm(b))
        else:
            u, v = h.leaf_data(k, gl[k])
            uo, vo = pr.leaf_data(k, ol[k])
            A, B = u @ v.T, uo @ vo.T
            nb = np.linalg.norm(B)
            if nb == 0.0:
                assert np.linalg.norm(A) == 0.0
                continue
            worst_lr = max(worst_lr, np.linalg.norm(A - B) / nb)
            if gl[k, 5] != ol[k, 5]:
                assert abs(int(gl[k, 5]) - int(ol[k, 5])) == 1, (k, gl[k], ol[k])
                rank_diff += 1
    print(f"nu={nu}: blocks {len(gl)}, worst LR {worst_lr:.2e} (eps {eps}), coarsened {worst_dense:.2e}, "
          f"rank +-1 in {rank_diff}")
    assert worst_lr <= eps, worst_lr
    assert worst_dense <= eps, worst_dense


def test_assembly_accuracy_vs_dense(hm, oracle):
    """test_hmatrix.cpp:41-49: ||C - C~||_F / ||C||_F <= 1e-5 at n = 512, eps = 1e-6."""
    x = oracle.random_locations(512, 17)
    th = [1.0, 0.2, 0.5, 0.0]
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, th, hm.RankControl.fixed_accuracy(1e-6))
    n = len(x)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    C = oracle.kernel_pairs(x, th, ii.ravel(), jj.ravel()).reshape(n, n)
    # matvec against dense (test_hmatrix.cpp:62-77)
    ones = np.ones(n)
    assert np.linalg.norm(h.matvec(ones) - C @ ones) / np.linalg.norm(C @ ones) <= 1e-5
    assert np.linalg.norm(h.matvec(np.zeros(n))) == 0.0
    assert h.stats()["bytes"] <= n * n * 8


def test_aca_constant_and_zero_blocks(hm):
    """test_hmatrix.cpp:27-39 analogue through assembly: far-apart identical clusters."""
    pts = np.concatenate([np.full((16, 2), 0.0), np.full((16, 2), 100.0)])
    g = hm.Geometry(pts, 16, 2.0)
    h = hm.assemble(g, [3.25, 1e4, 0.5, 0.0], hm.RankControl.fixed_accuracy(1e-8))
    lv = h.leaves()
    lr = lv[lv[:, 4] == 2]
    assert len(lr) == 1 and lr[0, 5] == 1  # numerically constant block -> rank 1
    h0 = hm.assemble(g, [1.0, 1e-3, 0.5, 0.0], hm.RankControl.fixed_accuracy(1e-8))
    lv0 = h0.leaves()
    assert lv0[lv0[:, 4] == 2][0, 5] == 0  # underflowed (zero) block -> rank 0


# ----------------------------------------------------------- factorization --
@pytest.mark.parametrize("form", ["ldl", "cholesky"])
def test_factor_vs_oracle_and_dense(hm, oracle, form):
    from oracle.oracle import make_config
    x = oracle.random_locations(1024, 13)
    th = [1.5, 0.08, 1.5, 1e-4]
    eps = 1e-6
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, th, hm.RankControl.fixed_accuracy(eps))
    f = hm.factorize(h, eps, form)
    pr = oracle.problem(x, 32, 2.0)
    pr.assemble(th, make_config(leaf_size=32, eps=eps, threads=4))
    pr.factorize(eps, form)
    z = oracle.normals(len(x), 5)
    assert rel(f.log_det(), pr.log_det()) < 1e-8
    assert rel(f.quad_form(z), pr.quad_form(z)) < 1e-7
    sx, so = f.solve_factored(z), pr.solve_factored(z)
    assert np.linalg.norm(sx - so) / np.linalg.norm(so) < 1e-6
    d_gpu, d_orc = f.diagonal(), pr.factor_diag()
    assert np.max(np.abs(d_gpu - d_orc) / np.abs(d_orc)) < 1e-6
    _, ld_dense, q_dense = oracle.dense_loglik(x, z, th)
    assert rel(f.log_det(), ld_dense) < 1e-4


def test_solve_inverts_matvec(hm, oracle):
    """test_hfactor.cpp:126-134: n = 700, theta = (1, 0.1, 1.5, 0.01), eps = 1e-6."""
    x = oracle.random_locations(700, 8)
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, [1.0, 0.1, 1.5, 0.01], hm.RankControl.fixed_accuracy(1e-6))
    f = hm.h_ldl(h, 1e-6)
    rhs = h.matvec(np.ones(700))
    assert np.linalg.norm(f.solve_factored(rhs) - 1) / math.sqrt(700) <= 1e-4


def test_factor_reports_failing_pivot(hm):
    """test_loglik_mle.cpp:89-94: identical points -> FactorError (nugget hint)."""
    pts = np.tile([[0.25, 0.75]], (6, 1))
    with pytest.raises(hm.FactorError, match="nugget") as e:
        hm.evaluate_loglik(pts, np.ones(6), [1.0, 0.1, 0.5, 0.0])
    assert 0 <= e.value.pivot_index < 6


# ---------------------------------------------------------------- L(θ) ----
def test_loglik_hand_cases(hm):
    """test_loglik_mle.cpp:13-33"""
    r = hm.evaluate_loglik(np.array([[0.5, 0.5]]), np.zeros(1), [0.75, 0.1, 0.5, 0.25])
    assert abs(r.loglik - -0.9189385332046727) <= 1e-14 * 0.92
    assert r.quad_form == 0.0
    r2 = hm.evaluate_loglik(np.array([[0.0, 0.0], [1.0, 1.0]]), np.ones(2), [0.5, 1e-3, 0.5, 0.5])
    assert rel(r2.loglik, -math.log(2 * math.pi) - 1.0) < 1e-10
    with pytest.raises(ValueError):
        hm.evaluate_loglik(np.array([[0.5, 0.5]]), np.zeros(2), [1, 0.1, 0.5, 0])
    with pytest.raises(ValueError):
        hm.evaluate_loglik(np.array([[0.5, 0.5]]), np.zeros(1), [1, -0.1, 0.5, 0])


@pytest.mark.parametrize("form", ["ldl", "cholesky"])
def test_loglik_C1_vs_oracle_and_dense(hm, oracle, form):
    """BASELINE config C1: 64x64 jittered grid, theta=(1,0.1,0.5,0.01), Z ~ N(0,C), leaf 64,
    eta 2, eps 1e-7; GPU vs oracle (1e-6) and vs the dense FP64 oracle (1e-6)."""
    from oracle.oracle import make_config
    x = oracle.jittered_grid(64, 1)
    th = [1.0, 0.1, 0.5, 0.01]
    z = oracle.sample_grf(x, th, 1 ^ 0x517CC1B727220A95)
    cfg = hm.HConfig(leaf_size=64, rank=hm.RankControl.fixed_accuracy(1e-7), form=form)
    got = hm.evaluate_loglik(x, z, th, cfg)
    want = oracle.loglik(x, z, th, make_config(leaf_size=64, eps=1e-7, form=form, threads=8))
    dense, _, _ = oracle.dense_loglik(x, z, th)
    assert rel(got.loglik, want.loglik) < 1e-6
    assert rel(got.loglik, dense) < 1e-6
    assert rel(got.logdet, want.logdet) < 1e-6


def test_loglik_general_nu_vs_oracle(hm, oracle):
    from oracle.oracle import make_config
    x = oracle.jittered_grid(48, 3)
    z = oracle.normals(len(x), 9)
    for th in ([1.5, 0.05, 1.0, 0.01], [1.0, 0.1, 0.325, 0.01], [2.0, 0.07, 0.7, 0.001]):
        cfg = hm.HConfig(leaf_size=64, rank=hm.RankControl.fixed_accuracy(1e-6))
        got = hm.evaluate_loglik(x, z, th, cfg).loglik
        want = oracle.loglik(x, z, th, make_config(leaf_size=64, eps=1e-6, threads=8)).loglik
        assert rel(got, want) < 1e-6, th


def test_loglik_translation_invariant(hm, oracle):
    """test_loglik_mle.cpp:75-87"""
    x = oracle.random_locations(300, 17)
    z = oracle.normals(300, 5)
    th = [1.2, 0.1, 0.8, 1e-4]
    a = hm.evaluate_loglik(x, z, th).loglik
    b = hm.evaluate_loglik(x + np.array([10.25, -4.75]), z, th).loglik
    assert abs(a - b) <= 1e-9 * abs(a)


def test_loglik_3d(hm, oracle):
    from oracle.oracle import make_config
    x = oracle.random_locations(3000, 21, dim=3)
    z = oracle.normals(3000, 2)
    th = [1.0, 0.08, 0.5, 0.005]
    cfg = hm.HConfig(leaf_size=64, rank=hm.RankControl.fixed_accuracy(1e-5))
    got = hm.evaluate_loglik(x, z, th, cfg).loglik
    want = oracle.loglik(x, z, th, make_config(leaf_size=64, eps=1e-5, threads=8)).loglik
    assert rel(got, want) < 1e-6


# --------------------------------------------------------------- predict --
def test_predict_vs_oracle_and_dense(hm, oracle):
    """test_krige_metrics.cpp:31-43 + 1e-6 GPU vs oracle."""
    from oracle.oracle import make_config
    allp = oracle.random_locations(576, 10)
    train, test = allp[:512], allp[512:]
    th = [1.5, 0.1, 1.5, 1e-4]
    z = oracle.sample_grf(allp, th, 44)[:512]
    cfg = hm.HConfig(rank=hm.RankControl.fixed_accuracy(1e-6))
    got = hm.predict(train, z, test, th, cfg).z2_hat
    want = oracle.predict(train, z, test, th, make_config(eps=1e-6, threads=8))
    dense = oracle.dense_predict(train, z, test, th)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-6
    assert np.linalg.norm(got - dense) / np.linalg.norm(dense) < 1e-4


def test_predict_edge_cases(hm, oracle):
    x = oracle.random_locations(32, 1)
    out = hm.predict(x, np.ones(32), np.zeros((0, 2)), [1.0, 0.1, 0.5, 0.0])
    assert out.z2_hat.size == 0
    with pytest.raises(ValueError):
        hm.predict(x, np.ones(31), x, [1.0, 0.1, 0.5, 0.0])
    # linearity (test_krige_metrics.cpp:62-78)
    allp = oracle.random_locations(300, 5)
    tr, te = allp[:256], allp[256:]
    th = [1.0, 0.1, 1.5, 1e-2]
    z1, z2 = oracle.normals(256, 7), oracle.normals(256, 8)
    a, b = 1.7, -0.4
    mixed = hm.predict(tr, a * z1 + b * z2, te, th).z2_hat
    combo = a * hm.predict(tr, z1, te, th).z2_hat + b * hm.predict(tr, z2, te, th).z2_hat
    assert np.max(np.abs(mixed - combo)) <= 1e-10


def test_kernel_vs_committed_reference_fixture(hm):
    """Device Matérn vs the reference build's at_distance (tests/golden/kernel_ref.npz)."""
    import os
    k = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernel_ref.npz"))
    for nu, want in zip(k["nu"], k["values"]):
        got = hm.at_distance([float(k["sigma2"]), float(k["ell"]), float(nu), float(k["tau2"])], k["h"])
        assert np.max(np.abs(got - want) / np.abs(want)) < 1e-10, nu
