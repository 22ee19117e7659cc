"""θ-sweep sharding across GPUs (BASELINE config C4).

One L(θ) evaluation does not shard (its diagonal recursion is sequential), but
a sweep of independent θ does: every rank builds the θ-independent geometry
once, evaluates its share of the θ grid through ``hmgp_loglik_batch`` and the
per-θ results {L, logdet, quad, status} are gathered with one collective
(NCCL over NVLink on GPUs; gloo in the CPU tests).  Failed probes score -inf,
as the reference's ``fit`` does (mle.cpp:152-158).
"""
from __future__ import annotations

import numpy as np

# Exact decimal literals (computed grids like linspace(0.3,1.5,4)
# give 1.0999999999999999 and would miss the reference's closed-form branches).
C4_SIGMA2 = (0.5, 0.7142857142857143, 0.9285714285714286, 1.1428571428571428,
             1.3571428571428572, 1.5714285714285714, 1.7857142857142858, 2.0)
C4_ELL = (0.02, 0.045714285714285714, 0.07142857142857142, 0.09714285714285714,
          0.12285714285714286, 0.14857142857142858, 0.17428571428571427, 0.2)
C4_NU = (0.3, 0.7, 1.1, 1.5)
C4_TAU2 = (0.001, 0.01)


def c4_theta_grid():
    """512 θ flattened in (σ², ℓ, ν, τ²) row-major order."""
    return np.array([(s, l, v, t) for s in C4_SIGMA2 for l in C4_ELL for v in C4_NU for t in C4_TAU2],
                    dtype=np.float64)


def shard(n_theta, rank, world, nu=None):
    """Indices of the θ this rank evaluates: round-robin over the list sorted
    ν-major, so the ~40x cheaper closed-form ν = 1.5 points spread evenly."""
    order = np.arange(n_theta)
    if nu is not None:
        order = np.argsort(np.asarray(nu), kind="stable")
    return np.sort(order[rank::world])


def gather_results(local_idx, local_vals, n_theta, dist=None, device=None):
    """All-gather (index, L, logdet, quad, status) rows into one (n_theta, 4) table."""
    import torch
    rows = np.zeros((len(local_idx), 5))
    rows[:, 0] = local_idx
    rows[:, 1:] = local_vals
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        allrows = rows
    else:
        ws = dist.get_world_size()
        cap = (n_theta + ws - 1) // ws + 1
        buf = np.full((cap, 5), -1.0)
        buf[: len(rows)] = rows
        t = torch.from_numpy(buf).to(device or "cpu")
        outs = [torch.empty_like(t) for _ in range(ws)]
        dist.all_gather(outs, t)
        allrows = np.concatenate([o.cpu().numpy() for o in outs])
        allrows = allrows[allrows[:, 0] >= 0]
    table = np.full((n_theta, 4), np.nan)
    table[allrows[:, 0].astype(int)] = allrows[:, 1:]
    return table


def argmax_theta(thetas, table):
    L = np.where(table[:, 3] >= 0, table[:, 0], -np.inf)
    k = int(np.argmax(L))
    return k, thetas[k], L[k]


def run_sweep(geom, d_z_ptr, thetas, idx, cfg, ctx):
    """Evaluate θ[idx] on this rank's GPU (geometry built once)."""
    import ctypes as C

    from . import Matern, _LogLik, _chk, _lib
    arr = (Matern * len(idx))(*[Matern(*thetas[i]) for i in idx])
    res = (_LogLik * len(idx))()
    c = cfg.c()
    _chk(_lib.hmgp_loglik_batch(ctx.h, geom.h, C.c_void_p(d_z_ptr), arr, len(idx), C.byref(c), res))
    return np.array([[r.loglik, r.logdet, r.quad_form, r.status] for r in res])


# ------------------------------------------------ kriging and assembly shards
def predict_ranges(m, world):
    """Contiguous [begin, end) of the m new locations per rank (SURVEY.md §8e:
    every GPU factors C̃₁₁ itself — a replica — and predicts m/G points)."""
    b = [(m * r) // world for r in range(world + 1)]
    return [(b[r], b[r + 1]) for r in range(world)]


def predict_sharded(train, z1, new_locations, theta, cfg=None, dist=None, device=None, predictor=None):
    """Sharded predict (krige.cpp:9-44): this rank predicts its contiguous slice,
    one all-gather (NCCL on GPUs, gloo in the CPU tests) assembles the m values in
    order on every rank."""
    import torch
    x2 = np.ascontiguousarray(new_locations, dtype=np.float64)
    m = x2.shape[0]
    ws = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rk = dist.get_rank() if ws > 1 else 0
    if m == 0:
        return np.empty(0)
    lo, hi = predict_ranges(m, ws)[rk]
    run = predictor
    if run is None:
        from . import predict
        run = lambda te: predict(train, z1, te, theta, cfg).z2_hat  # noqa: E731
    local = np.asarray(run(x2[lo:hi]), dtype=np.float64) if hi > lo else np.empty(0)
    if ws == 1:
        return local
    cap = (m + ws - 1) // ws
    buf = np.zeros(cap)
    buf[: hi - lo] = local
    t = torch.from_numpy(buf).to(device or "cpu")
    outs = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(outs, t)
    parts = [o.cpu().numpy()[: e - b] for o, (b, e) in zip(outs, predict_ranges(m, ws))]
    return np.concatenate(parts)


def assemble_sharded(geom, theta, rc=None, dist=None):
    """Sharded assembly (C2): this rank assembles its cost-balanced contiguous
    range of the stored-leaf list (no data-path collective; payloads stay local)."""
    from . import assemble_shard
    ws = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rk = dist.get_rank() if ws > 1 else 0
    return assemble_shard(geom, theta, rk, ws, rc)


# ------------------------------------------------- the C-ABI path (no torch)
class Comm:
    """NCCL communicator of the C ABI (hmgp_comm_*): rank 0 makes the 128-byte
    unique id, the launcher hands it to the other ranks (here: any callable
    ``bcast(bytes_or_None) -> bytes``, e.g. torch.distributed / a file)."""

    def __init__(self, ctx, rank, world, bcast=None):
        import ctypes as C

        from . import _chk, _lib
        self.ctx, self.rank, self.world = ctx, rank, world
        self.h = C.c_void_p()
        ident = C.create_string_buffer(128)
        if world > 1:
            if rank == 0:
                _chk(_lib.hmgp_comm_unique_id(ident))
            raw = bcast(ident.raw if rank == 0 else None)
            ident = C.create_string_buffer(bytes(raw), 128)
        _chk(_lib.hmgp_comm_create(ctx.h, ident, rank, world, C.byref(self.h)))

    def close(self):
        from . import _lib
        if self.h:
            _lib.hmgp_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_c(thetas, rank, world):
    """hmgp_sweep_shard: the same ν-major round-robin as ``shard`` above."""
    import ctypes as C

    from . import Matern, _chk, _i, _lib
    th = np.asarray(thetas, dtype=np.float64).reshape(-1, 4)
    arr = (Matern * max(1, len(th)))(*[Matern(*t) for t in th])
    idx = np.empty(max(1, len(th)), dtype=np.int32)
    cnt = C.c_int()
    _chk(_lib.hmgp_sweep_shard(arr, len(th), rank, world, _i(idx), C.byref(cnt)))
    return idx[: cnt.value].copy()


def sweep_host(geom, z, thetas, idx, cfg, ctx):
    """hmgp_loglik_sweep: θ[idx] on this rank's GPU, z a HOST array (uploaded once).
    Returns the ctypes result rows (for hmgp_sweep_gather) and the value table."""
    import ctypes as C

    from . import Matern, _LogLik, _chk, _d, _lib
    z = np.ascontiguousarray(z, dtype=np.float64)
    k = len(idx)
    arr = (Matern * max(1, k))(*[Matern(*thetas[i]) for i in idx])
    res = (_LogLik * max(1, k))()
    c = cfg.c()
    _chk(_lib.hmgp_loglik_sweep(ctx.h, geom.h, _d(z), arr, k, C.byref(c), res))
    return res, np.array([[r.loglik, r.logdet, r.quad_form, r.status] for r in res[:k]]).reshape(k, 4)


def gather_c(ctx, comm, idx, res, n_theta):
    """hmgp_sweep_gather: ONE NCCL all-gather -> (n_theta, 4) table on every rank."""
    from . import _LogLik, _chk, _i, _lib
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    table = (_LogLik * max(1, n_theta))()
    _chk(_lib.hmgp_sweep_gather(ctx.h, comm.h if comm is not None else None, _i(idx), res, len(idx),
                                n_theta, table))
    return np.array([[r.loglik, r.logdet, r.quad_form, r.status] for r in table[:n_theta]]).reshape(n_theta, 4)


def predict_gather_c(ctx, comm, local, m):
    """hmgp_predict_gather: ONE NCCL all-gather of the contiguous prediction slices."""
    from . import _chk, _d, _lib
    local = np.ascontiguousarray(local, dtype=np.float64)
    out = np.empty(max(1, m))
    loc = local if local.size else np.zeros(1)
    _chk(_lib.hmgp_predict_gather(ctx.h, comm.h if comm is not None else None, _d(loc), m, _d(out)))
    return out[:m]
