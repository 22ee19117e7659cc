"""The C-ABI θ-sweep / kriging-shard entry points (csrc/sweep.cu).

CPU: the host-only pieces (shard indices, predict ranges, world-1 gathers — no
NCCL, no device work) agree with the Python sharding logic.
GPU (-m gpu): hmgp_loglik_sweep against single evaluations (bit-identical), a
world-1 NCCL communicator, and a 2-process run of the REAL evaluator whose
gathered table equals the 1-process table (both ranks share cuda:0, so the
gather itself goes over gloo there; the ncclAllGather path needs two GPUs).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def test_shard_c_matches_python_shard(hm):
    from paper_2104_07146_b200 import sweep as sw
    g = sw.c4_theta_grid()
    for world in (1, 2, 3, 8):
        parts = []
        for r in range(world):
            a = sw.shard(len(g), r, world, nu=g[:, 2])
            b = sw.shard_c(g, r, world)
            assert np.array_equal(a, b)
            parts.append(b)
        assert np.array_equal(np.sort(np.concatenate(parts)), np.arange(len(g)))
    assert len(sw.shard_c(g[:0], 0, 1)) == 0  # empty θ list
    assert np.array_equal(sw.shard_c(g[:3], 2, 8), [2]) and len(sw.shard_c(g[:3], 5, 8)) == 0  # ragged


def test_predict_range_c_matches_python(hm):
    from paper_2104_07146_b200 import _lib
    from paper_2104_07146_b200 import sweep as sw
    for m in (0, 1, 7, 10000):
        for world in (1, 2, 8):
            want = sw.predict_ranges(m, world)
            for r in range(world):
                b, e = C.c_int(), C.c_int()
                assert _lib.hmgp_predict_range(m, r, world, C.byref(b), C.byref(e)) == 0
                assert (b.value, e.value) == want[r]
    b, e = C.c_int(), C.c_int()
    assert _lib.hmgp_predict_range(5, 2, 2, C.byref(b), C.byref(e)) != 0  # rank out of range


def test_world1_gathers_need_no_collective(hm):
    """comm == NULL: the gathers are local scatters (no NCCL, no device)."""
    from paper_2104_07146_b200 import _LogLik, _lib
    from paper_2104_07146_b200 import sweep as sw
    rows = (_LogLik * 2)()
    rows[0].loglik, rows[0].status = -1.5, 0
    rows[1].loglik, rows[1].status = -2.5, 1
    t = sw.gather_c(type("Ctx", (), {"h": None})(), None, np.array([3, 1], dtype=np.int32), rows, 4)
    assert t[3, 0] == -1.5 and t[1, 0] == -2.5 and t[1, 3] == 1
    assert np.isnan(t[0, 0]) and t[0, 3] == -2 and t[2, 3] == -2  # rows nobody evaluated
    loc = np.arange(5.0)
    out = sw.predict_gather_c(type("Ctx", (), {"h": None})(), None, loc, 5)
    assert np.array_equal(out, loc)
    assert len(sw.predict_gather_c(type("Ctx", (), {"h": None})(), None, np.empty(0), 0)) == 0


# -------------------------------------------------------------------- GPU --
def _problem(hm):
    x = hm.jittered_grid(48, 1)
    z = hm.normals(48 * 48, 5)
    cfg = hm.HConfig(leaf_size=64, rank=hm.RankControl.fixed_accuracy(1e-7))
    th = np.array([[1.0, 0.1, 0.5, 0.01], [1.2, 0.07, 1.1, 0.001], [0.8, 0.12, 1.5, 0.01],
                   [1.0, 0.05, 0.3, 0.01], [1.5, 0.1, 0.7, 0.001]])
    return x, z, cfg, th


@pytest.mark.gpu
def test_loglik_sweep_matches_single_evaluations(hm):
    from paper_2104_07146_b200 import sweep as sw
    x, z, cfg, th = _problem(hm)
    ctx = hm.default_context()
    geo = hm.Geometry(x, 64, 2.0, ctx=ctx)
    _, vals = sw.sweep_host(geo, z, th, list(range(len(th))), cfg, ctx)
    for k, t in enumerate(th):
        one = hm.evaluate_loglik(x, z, list(t), cfg)
        assert vals[k, 0] == one.loglik and vals[k, 1] == one.logdet and vals[k, 2] == one.quad_form
    # a θ that fails numerically scores -inf with status -1, the others are unaffected
    bad = np.vstack([th[:2], [[1.0, 0.5, 2.5, 0.0]]])
    xd = np.vstack([x, x[:1]])  # duplicated point, no nugget -> not SPD
    zd = np.append(z, z[0])
    geo2 = hm.Geometry(xd, 64, 2.0, ctx=ctx)
    _, v2 = sw.sweep_host(geo2, zd, bad, [0, 1, 2], cfg, ctx)
    assert v2[2, 3] == -1 and v2[2, 0] == -np.inf and np.isfinite(v2[0, 0]) and np.isfinite(v2[1, 0])


@pytest.mark.gpu
def test_world1_nccl_comm_and_gathers(hm):
    from paper_2104_07146_b200 import sweep as sw
    x, z, cfg, th = _problem(hm)
    ctx = hm.default_context()
    comm = sw.Comm(ctx, 0, 1)
    geo = hm.Geometry(x, 64, 2.0, ctx=ctx)
    idx = sw.shard_c(th, 0, 1)
    rows, vals = sw.sweep_host(geo, z, th, list(idx), cfg, ctx)
    table = sw.gather_c(ctx, comm, idx, rows, len(th))
    assert np.array_equal(table, vals)
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2104_07146_b200 as hm
    from paper_2104_07146_b200 import sweep as sw
    x, z, cfg, th = _problem(hm)
    ctx = hm.Context(0)  # both ranks share the one GPU of the test box
    geo = hm.Geometry(x, 64, 2.0, ctx=ctx)
    idx = sw.shard_c(th, rank, world)
    _, vals = sw.sweep_host(geo, z, th, list(idx), cfg, ctx)
    table = sw.gather_results(idx, vals, len(th), dist=dist)
    k, best, lb = sw.argmax_theta(th, table)
    te = hm.random_locations(301, 9)
    pred = sw.predict_sharded(x, z, te, list(best), cfg, dist=dist)
    if rank == 0:
        q.put((table, k, pred))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_real_evaluator_match_one_rank(hm):
    """2 processes, the real hmgp_loglik_sweep on each, gathered table == the
    1-process table bit for bit; sharded predictions == unsharded."""
    from paper_2104_07146_b200 import sweep as sw
    x, z, cfg, th = _problem(hm)
    ctx = hm.default_context()
    geo = hm.Geometry(x, 64, 2.0, ctx=ctx)
    _, want = sw.sweep_host(geo, z, th, list(range(len(th))), cfg, ctx)
    k1, best, _ = sw.argmax_theta(th, want)
    te = hm.random_locations(301, 9)
    pred1 = hm.predict(x, z, te, list(best), cfg).z2_hat
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    table, k2, pred2 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert np.array_equal(table, want)
    assert k1 == k2
    assert np.array_equal(pred2, pred1)
