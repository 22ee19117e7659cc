"""CPU tests of the multi-GPU θ-sweep host logic: grid literals, balanced
ν-major sharding, and the all-gather of per-θ results over a world-size-2
gloo process group (the NCCL path on GPUs runs the same code)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _import_sweep():
    import importlib.util
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2104_07146_b200", "sweep.py")
    spec = importlib.util.spec_from_file_location("sweep_mod", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_c4_grid_literals():
    sw = _import_sweep()
    g = sw.c4_theta_grid()
    assert g.shape == (512, 4)
    assert set(g[:, 2]) == {0.3, 0.7, 1.1, 1.5}  # exact literals, no 1.0999999999999999
    assert g[0].tolist() == [0.5, 0.02, 0.3, 0.001]
    assert g[-1].tolist() == [2.0, 0.2, 1.5, 0.01]
    np.testing.assert_allclose(np.unique(g[:, 0]), np.linspace(0.5, 2, 8), rtol=1e-15)
    np.testing.assert_allclose(np.unique(g[:, 1]), np.linspace(0.02, 0.2, 8), rtol=1e-15)


def test_shards_partition_and_balance():
    sw = _import_sweep()
    g = sw.c4_theta_grid()
    for world in (1, 2, 4, 8):
        parts = [sw.shard(len(g), r, world, nu=g[:, 2]) for r in range(world)]
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(len(g)))
        for p in parts:  # every rank gets the same number of ν = 1.5 (cheap) points
            assert np.sum(g[p, 2] == 1.5) == np.sum(g[:, 2] == 1.5) // world


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sw = _import_sweep()
    g = sw.c4_theta_grid()
    idx = sw.shard(len(g), rank, world, nu=g[:, 2])
    # stand-in evaluator (the GPU path calls hmgp_loglik_batch): a smooth function of θ
    vals = np.stack([-(g[idx, 0] - 1.1) ** 2 - (g[idx, 1] - 0.1) ** 2 - g[idx, 3],
                     g[idx, 0], g[idx, 1], np.where(g[idx, 2] == 0.3, -1, 0)], axis=1)
    table = sw.gather_results(idx, vals, len(g), dist=dist)
    if rank == 0:
        out.put(table)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gather_world2_gloo_matches_serial():
    sw = _import_sweep()
    g = sw.c4_theta_grid()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    table = q.get(timeout=150)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    serial = np.stack([-(g[:, 0] - 1.1) ** 2 - (g[:, 1] - 0.1) ** 2 - g[:, 3], g[:, 0], g[:, 1],
                       np.where(g[:, 2] == 0.3, -1, 0)], axis=1)
    assert np.array_equal(table, serial)
    k, th, L = sw.argmax_theta(g, table)
    assert th[2] != 0.3  # failed probes (status -1) never win
    assert L == np.max(np.where(serial[:, 3] >= 0, serial[:, 0], -np.inf))


def _predict_worker(rank, world, port, m, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sw = _import_sweep()
    x2 = np.random.default_rng(3).random((m, 2))
    # stand-in predictor (the GPU path calls hmgp_predict on this rank's slice)
    got = sw.predict_sharded(None, None, x2, None, dist=dist,
                             predictor=lambda te: np.sin(7 * te[:, 0]) + te[:, 1] ** 2)
    out.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("m", [10000, 3])
def test_predict_sharded_world2_gloo(m):
    """Kriging shards: contiguous m/G slices, one all-gather, every
    rank ends with all m predictions in order (m = 3: ragged slices)."""
    sw = _import_sweep()
    for world in (1, 2, 3, 8):
        r = sw.predict_ranges(m, world)
        assert r[0][0] == 0 and r[-1][1] == m and all(a[1] == b[0] for a, b in zip(r, r[1:]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_predict_worker, args=(rk, 2, port, m, q)) for rk in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=150) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x2 = np.random.default_rng(3).random((m, 2))
    want = np.sin(7 * x2[:, 0]) + x2[:, 1] ** 2
    for rk in range(2):
        assert np.array_equal(res[rk], want)


def test_balanced_leaf_ranges(hm):
    """Assembly shards: contiguous, covering, near-equal cost."""
    rng = np.random.default_rng(0)
    cost = np.where(rng.random(5000) < 0.25, 64.0 * 64, 16.0 * 128)  # dense / admissible mix
    for parts in (1, 2, 4, 8):
        b = hm.balanced_ranges(cost, parts)
        assert b[0] == 0 and b[-1] == cost.size and np.all(np.diff(b) >= 0)
        sums = np.array([cost[b[i]:b[i + 1]].sum() for i in range(parts)])
        assert sums.max() - sums.min() <= 2 * cost.max()
    b = hm.balanced_ranges(np.ones(3), 8)  # more parts than leaves: empty ranges allowed
    assert b[0] == 0 and b[-1] == 3 and np.all(np.diff(b) >= 0)
    assert hm.balanced_ranges(np.empty(0), 2).tolist() == [0, 0, 0]
