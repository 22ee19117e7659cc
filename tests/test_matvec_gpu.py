"""H-matvec (csrc/matvec.cu): the HBM-oriented deterministic pass against the
oracle's matvec (hmatrix.cpp:244-272 restated) and the dense product, on layouts
that exercise every path — dense leaves, one-CTA low-rank leaves, chunked tall
low-rank leaves — plus bit-reproducibility (tests/test_hmatrix.cpp:165-171) and
the device-vector entry point."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dense(oracle, x, th):
    n = len(x)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    return oracle.kernel_pairs(x, th, ii.ravel(), jj.ravel()).reshape(n, n)


@pytest.mark.parametrize("n,leaf,dim", [(700, 32, 2), (3000, 64, 2), (1500, 32, 3)])
def test_matvec_vs_dense(hm, oracle, n, leaf, dim):
    x = hm.random_locations(n, 11, dim=dim) if dim == 3 else hm.random_locations(n, 11)
    th = [1.3, 0.09, 1.0, 0.01]
    g = hm.Geometry(x, leaf, 2.0)
    h = hm.assemble(g, th, hm.RankControl.fixed_accuracy(1e-8))
    rng = np.random.default_rng(3)
    Cd = _dense(oracle, x, th)
    for v in (np.ones(n), rng.standard_normal(n)):
        want = Cd @ v
        got = h.matvec(v)
        assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)
        assert np.array_equal(got, h.matvec(v))  # bit-reproducible
    assert np.linalg.norm(h.matvec(np.zeros(n))) == 0.0


def test_matvec_chunked_leaves_match_legacy_kernel(hm):
    """n = 16384, leaf 64: admissible blocks up to 4096 rows take the chunked path;
    the legacy one-CTA-per-leaf kernel (FP64 atomics) is the independent check."""
    x = hm.jittered_grid(128, 1)
    n = len(x)
    g = hm.Geometry(x, 64, 2.0)
    h = hm.assemble(g, [1.0, 0.1, 0.5, 0.01], hm.RankControl.fixed_accuracy(1e-7))
    v = hm.normals(n, 9)
    got = h.matvec(v)
    assert np.array_equal(got, h.matvec(v))
    os.environ["HMGP_MATVEC_LEGACY"] = "1"
    try:
        ref = h.matvec(v)
    finally:
        del os.environ["HMGP_MATVEC_LEGACY"]
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_matvec_device_entry_and_oracle_matvec(hm, oracle):
    import torch
    from paper_2104_07146_b200 import _chk, _lib
    x = hm.random_locations(900, 4)
    g = hm.Geometry(x, 32, 2.0)
    h = hm.assemble(g, [1.0, 0.1, 1.5, 0.0], hm.RankControl.fixed_accuracy(1e-7))
    v = hm.normals(900, 2)
    dv = torch.from_numpy(v).cuda()
    dy = torch.empty_like(dv)
    _chk(_lib.hmgp_hmat_matvec_device(h.ctx.h, h.h, C.c_void_p(dv.data_ptr()), C.c_void_p(dy.data_ptr())))
    torch.cuda.synchronize()
    assert np.array_equal(dy.cpu().numpy(), h.matvec(v))
    # oracle H-matvec (hmatrix.cpp:244-272 restated) on the same configuration
    from oracle.oracle import make_config
    prob = oracle.problem(x, 32, 2.0)
    prob.assemble([1.0, 0.1, 1.5, 0.0], make_config(leaf_size=32, eps=1e-7))
    want = prob.matvec(v)
    assert np.linalg.norm(h.matvec(v) - want) <= 1e-6 * np.linalg.norm(want)
