"""hmgp on B200 — Python mirror of the reference's hmgp API over the C ABI.

The product is ``libhmgp_cuda.so`` (hand-written sm_100a CUDA + C++ host, built
in-tree by ``build.py``); this module binds its ``extern "C"`` boundary
(``include/hmgp_cuda.h``) with ctypes and mirrors the reference names
(``/root/reference/proj/include/hmgp/*.hpp``, ``python/bindings.cpp``):

    build_cluster_tree / ClusterTree      geometry.hpp:44-68
    build_block_tree / BlockClusterTree   geometry.hpp:72-109
    MaternParams, matern kernel entries   covkernel.hpp:11-69
    RankControl, HConfig                  hmatrix.hpp:17-36, pipeline.hpp:13-25
    assemble -> HMatrix                   hmatrix.hpp:44-90
    factorize / h_cholesky / h_ldl        hfactor.hpp:34-77
    evaluate_loglik -> LogLikResult       loglik.hpp:10-23
    predict -> PredictionResult           krige.hpp:10-21

Errors follow the reference: std::invalid_argument -> ValueError,
std::domain_error -> DomainError, std::out_of_range -> IndexError,
hmgp::FactorError -> FactorError (with pivot_index / pivot_value).  There is no
CPU fallback: importing fails loudly when the CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

# The task-flow factorization (csrc/dag.h) spreads independent launches over 32
# streams; the default 8 hardware work queues would serialise them again.  Must
# be set before the process creates its CUDA context.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhmgp_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_vp = C.c_void_p

HMGP_OK, HMGP_EINVAL, HMGP_EDOMAIN, HMGP_ERANGE, HMGP_ENOTSPD, HMGP_ECUDA, HMGP_ECAPACITY, HMGP_ERUNTIME = range(8)


class DomainError(ValueError):
    """std::domain_error (bessel_k domain, indefinite log_det)."""


class FactorError(RuntimeError):
    """hmgp::FactorError (hfactor.hpp:17-22): failing pivot, ORIGINAL index."""

    def __init__(self, msg, pivot_index, pivot_value):
        super().__init__(msg)
        self.pivot_index = pivot_index
        self.pivot_value = pivot_value


class CudaError(RuntimeError):
    pass


class CapacityError(RuntimeError):
    pass


class Matern(C.Structure):
    _fields_ = [("sigma2", C.c_double), ("ell", C.c_double), ("nu", C.c_double),
                ("tau2", C.c_double)]


class _RankControl(C.Structure):
    _fields_ = [("mode", C.c_int), ("eps", C.c_double), ("rank", C.c_int), ("max_rank", C.c_int)]


class _Config(C.Structure):
    _fields_ = [("eta", C.c_double), ("leaf_size", C.c_int), ("rank", _RankControl),
                ("eps_factor", C.c_double), ("form", C.c_int), ("threads", C.c_int)]


class _Block(C.Structure):
    _fields_ = [("row_begin", C.c_int32), ("row_end", C.c_int32), ("col_begin", C.c_int32),
                ("col_end", C.c_int32), ("tag", C.c_int32)]


class _FactorInfo(C.Structure):
    _fields_ = [("eps", C.c_double), ("clamped", C.c_int), ("negative", C.c_int),
                ("min_pivot", C.c_double), ("storage_bytes", C.c_double)]


class _LogLik(C.Structure):
    _fields_ = [("loglik", C.c_double), ("logdet", C.c_double), ("quad_form", C.c_double),
                ("n", C.c_int), ("seconds", C.c_double), ("status", C.c_int)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("hmgp_last_error", C.c_char_p, [])
_sig("hmgp_last_pivot_index", C.c_int, [])
_sig("hmgp_last_pivot_value", C.c_double, [])
_sig("hmgp_kernel_launches", C.c_uint64, [_vp])
_sig("hmgp_default_config", None, [C.POINTER(_Config)])
_sig("hmgp_ctx_create", C.c_int, [C.c_int, C.POINTER(_vp)])
_sig("hmgp_ctx_destroy", None, [_vp])
_sig("hmgp_geometry_build", C.c_int, [_vp, _dp, C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(_vp)])
_sig("hmgp_geometry_build_device", C.c_int, [_vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.POINTER(_vp)])
_sig("hmgp_geometry_perm", C.c_int, [_vp, _ip, _ip])
_sig("hmgp_geometry_clusters", C.c_int, [_vp, _ip, _dp, C.c_int, C.POINTER(C.c_int)])
_sig("hmgp_geometry_block_count", C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int),
                                            C.POINTER(C.c_int)])
_sig("hmgp_geometry_blocks", C.c_int, [_vp, C.POINTER(_Block), C.c_int64])
_sig("hmgp_geometry_destroy", None, [_vp])
_sig("hmgp_kernel_pairs", C.c_int, [_vp, _dp, C.c_int, C.c_int, C.POINTER(Matern), _ip, _ip,
                                    C.c_int64, _dp])
_sig("hmgp_at_distance", C.c_int, [_vp, C.POINTER(Matern), _dp, C.c_int64, _dp])
_sig("hmgp_bessel_k", C.c_int, [_vp, _dp, _dp, C.c_int64, C.c_int, _dp])
_sig("hmgp_assemble", C.c_int, [_vp, _vp, C.POINTER(Matern), C.POINTER(_RankControl), C.POINTER(_vp)])
_sig("hmgp_assemble_shard", C.c_int, [_vp, _vp, C.POINTER(Matern), C.POINTER(_RankControl), C.c_int, C.c_int,
                                     C.POINTER(_vp), C.POINTER(C.c_int), C.POINTER(C.c_int)])
_sig("hmgp_balanced_ranges", C.c_int, [_dp, C.c_int, C.c_int, _ip])
_sig("hmgp_hmat_stats", C.c_int, [_vp, _dp, C.POINTER(C.c_int), _dp])
_sig("hmgp_hmat_leaves", C.c_int, [_vp, _ip, C.c_int64, C.POINTER(C.c_int64)])
_sig("hmgp_hmat_leaf_data", C.c_int, [_vp, C.c_int64, _dp, _dp])
_sig("hmgp_hmat_matvec", C.c_int, [_vp, _vp, _dp, _dp])
_sig("hmgp_hmat_destroy", None, [_vp])
_sig("hmgp_factorize", C.c_int, [_vp, _vp, C.c_double, C.c_int, C.POINTER(_vp), C.POINTER(_FactorInfo)])
_sig("hmgp_log_det", C.c_int, [_vp, _vp, _dp])
_sig("hmgp_quad_form", C.c_int, [_vp, _vp, _dp, _dp])
_sig("hmgp_solve_factored", C.c_int, [_vp, _vp, _dp, _dp])
_sig("hmgp_solve_lower", C.c_int, [_vp, _vp, _dp, _dp])
_sig("hmgp_factor_diagonal", C.c_int, [_vp, _vp, _dp])
_sig("hmgp_factor_destroy", None, [_vp])
_sig("hmgp_hmat_to_dense", C.c_int, [_vp, _vp, _dp])
_sig("hmgp_factor_lower_dense", C.c_int, [_vp, _vp, _dp])
_sig("hmgp_factor_reconstruct", C.c_int, [_vp, _vp, _dp])
_sig("hmgp_loglik", C.c_int, [_vp, _dp, C.c_int, C.c_int, _dp, C.POINTER(Matern), C.POINTER(_Config),
                              C.POINTER(_LogLik)])
_sig("hmgp_loglik_geom", C.c_int, [_vp, _vp, C.c_void_p, C.POINTER(Matern), C.POINTER(_Config),
                                   C.POINTER(_LogLik)])
_sig("hmgp_loglik_batch", C.c_int, [_vp, _vp, C.c_void_p, C.POINTER(Matern), C.c_int, C.POINTER(_Config),
                                    C.POINTER(_LogLik)])
_sig("hmgp_loglik_sweep", C.c_int, [_vp, _vp, _dp, C.POINTER(Matern), C.c_int, C.POINTER(_Config),
                                    C.POINTER(_LogLik)])
_sig("hmgp_release_workspace", None, [])
_sig("hmgp_hmat_matvec_device", C.c_int, [_vp, _vp, C.c_void_p, C.c_void_p])
_sig("hmgp_sweep_shard", C.c_int, [C.POINTER(Matern), C.c_int, C.c_int, C.c_int, _ip, C.POINTER(C.c_int)])
_sig("hmgp_predict_range", C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)])
_sig("hmgp_comm_unique_id", C.c_int, [C.c_void_p])
_sig("hmgp_comm_create", C.c_int, [_vp, C.c_void_p, C.c_int, C.c_int, C.POINTER(_vp)])
_sig("hmgp_comm_destroy", None, [_vp])
_sig("hmgp_sweep_gather", C.c_int, [_vp, _vp, _ip, C.POINTER(_LogLik), C.c_int, C.c_int, C.POINTER(_LogLik)])
_sig("hmgp_predict_gather", C.c_int, [_vp, _vp, _dp, C.c_int, _dp])
_sig("hmgp_predict", C.c_int, [_vp, _dp, C.c_int, C.c_int, _dp, _dp, C.c_int, C.POINTER(Matern),
                               C.POINTER(_Config), _dp, _dp])
_sig("hmgp_cross_apply_device", C.c_int, [_vp, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_int, C.POINTER(Matern), C.c_void_p])
_sig("hmgp_kriging_variance_dense", C.c_int, [_vp, _dp, C.c_int, C.c_int, _dp, C.c_int, C.POINTER(Matern),
                                             _dp])
_sig("hmgp_mloe_mmom", C.c_int, [_vp, _dp, C.c_int, C.c_int, C.POINTER(Matern), C.POINTER(Matern), C.c_int,
                                 C.c_uint64, C.c_int, _dp, _dp])
_sig("hmgp_random_locations", C.c_int, [C.c_int, C.c_int, C.c_uint64, _dp])
_sig("hmgp_jittered_grid", C.c_int, [C.c_int, C.c_uint64, _dp])
_sig("hmgp_normals", C.c_int, [C.c_int, C.c_uint64, _dp])
_sig("hmgp_sample_grf", C.c_int, [_vp, _dp, C.c_int, C.c_int, C.POINTER(Matern), C.c_uint64, _dp])


def _chk(rc):
    if rc == HMGP_OK:
        return
    msg = _lib.hmgp_last_error().decode()
    if rc == HMGP_EINVAL:
        raise ValueError(msg)
    if rc == HMGP_EDOMAIN:
        raise DomainError(msg)
    if rc == HMGP_ERANGE:
        raise IndexError(msg)
    if rc == HMGP_ENOTSPD:
        raise FactorError(msg, _lib.hmgp_last_pivot_index(), _lib.hmgp_last_pivot_value())
    if rc == HMGP_ECAPACITY:
        raise CapacityError(msg)
    if rc == HMGP_ERUNTIME:
        raise RuntimeError(msg)
    raise CudaError(msg)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _pts(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] not in (2, 3):
        raise ValueError("locations must be an (n, 2) or (n, 3) array")
    return x


# ------------------------------------------------------------------ context
class Context:
    """One device + one stream (the C ABI's hmgp_ctx)."""

    def __init__(self, device=0):
        h = _vp()
        _chk(_lib.hmgp_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def __del__(self):
        try:
            _lib.hmgp_ctx_destroy(self.h)
        except Exception:
            pass

    def launches(self):
        return int(_lib.hmgp_kernel_launches(self.h))


def release_workspace():
    """hmgp_release_workspace: free the arenas / captured factorizations kept between calls."""
    _lib.hmgp_release_workspace()


_default_ctx = None


def default_context():
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------------------------- params
@dataclass
class MaternParams:
    """covkernel.hpp:11-19"""
    sigma2: float = 1.0
    ell: float = 0.1
    nu: float = 0.5
    tau2: float = 0.0

    def valid(self):  # covkernel.cpp:9-13
        v = (self.sigma2, self.ell, self.nu, self.tau2)
        return (all(np.isfinite(v)) and self.sigma2 > 0.0 and self.ell > 0.0 and self.nu > 0.0
                and self.tau2 >= 0.0)

    def c(self):
        return Matern(self.sigma2, self.ell, self.nu, self.tau2)


def _mp(p):
    if isinstance(p, MaternParams):
        return p.c()
    if isinstance(p, Matern):
        return p
    return Matern(*[float(v) for v in p])


@dataclass
class RankControl:
    """hmatrix.hpp:17-36"""
    mode: str = "accuracy"
    eps: float = 1e-6
    rank: int = 16
    max_rank: int = 256

    @staticmethod
    def fixed_accuracy(eps):
        return RankControl("accuracy", eps)

    @staticmethod
    def fixed_rank(k):
        return RankControl("rank", 1e-6, k)

    def c(self):
        return _RankControl(0 if self.mode == "accuracy" else 1, self.eps, self.rank, self.max_rank)


@dataclass
class HConfig:
    """pipeline.hpp:13-25"""
    eta: float = 2.0
    leaf_size: int = 32
    rank: RankControl = field(default_factory=lambda: RankControl.fixed_accuracy(1e-6))
    eps_factor: float = -1.0
    form: str = "ldl"
    threads: int = 1

    def factor_eps(self):
        if self.eps_factor > 0:
            return self.eps_factor
        return self.rank.eps if self.rank.mode == "accuracy" else 1e-6

    def c(self):
        return _Config(self.eta, self.leaf_size, self.rank.c(), self.eps_factor,
                       1 if self.form == "ldl" else 0, self.threads)


# ----------------------------------------------------------------- geometry
class Geometry:
    """ClusterTree + BlockClusterTree for one point set (built on the GPU)."""

    def __init__(self, locations, leaf_size=32, eta=2.0, ctx=None):
        self.ctx = ctx or default_context()
        self.x = _pts(locations)
        self.n, self.dim = self.x.shape
        self.leaf_size, self.eta = leaf_size, eta
        h = _vp()
        _chk(_lib.hmgp_geometry_build(self.ctx.h, _d(self.x), self.n, self.dim, leaf_size, eta,
                                      C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            _lib.hmgp_geometry_destroy(self.h)
        except Exception:
            pass

    def perm(self):
        p = np.empty(self.n, dtype=np.int32)
        _chk(_lib.hmgp_geometry_perm(self.h, _i(p), None))
        return p

    def inverse_perm(self):
        p = np.empty(self.n, dtype=np.int32)
        _chk(_lib.hmgp_geometry_perm(self.h, None, _i(p)))
        return p

    def clusters(self):
        cap = 4 * (self.n // max(1, self.leaf_size) + 2) + 16
        while True:
            out = np.empty((cap, 4), dtype=np.int32)
            box = np.empty((cap, 6))
            cnt = C.c_int()
            rc = _lib.hmgp_geometry_clusters(self.h, _i(out), _d(box), cap, C.byref(cnt))
            if rc == HMGP_ERANGE:
                cap = cnt.value
                continue
            _chk(rc)
            return out[: cnt.value], box[: cnt.value]

    def block_counts(self):
        cnt, na, nd = C.c_int64(), C.c_int(), C.c_int()
        _chk(_lib.hmgp_geometry_block_count(self.h, C.byref(cnt), C.byref(na), C.byref(nd)))
        return cnt.value, na.value, nd.value

    def blocks(self):
        """Leaves in the reference's DFS order: (row_begin,row_end,col_begin,col_end,tag)."""
        cnt, _, _ = self.block_counts()
        arr = (_Block * max(1, cnt))()
        _chk(_lib.hmgp_geometry_blocks(self.h, arr, cnt))
        out = np.frombuffer(arr, dtype=np.int32).reshape(-1, 5)[:cnt].copy()
        return out


def build_cluster_tree(locations, leaf_size=32, ctx=None):
    """geometry.hpp:68 (the block tree is built alongside; eta = 2)."""
    return Geometry(locations, leaf_size, 2.0, ctx)


# ------------------------------------------------------------------- kernel
def kernel_pairs(locations, params, ii, jj, ctx=None):
    """KernelEvaluator(i, j) (covkernel.hpp:45-48) evaluated on the GPU."""
    ctx = ctx or default_context()
    x = _pts(locations)
    ii = np.ascontiguousarray(ii, dtype=np.int32)
    jj = np.ascontiguousarray(jj, dtype=np.int32)
    out = np.empty(ii.size)
    m = _mp(params)
    _chk(_lib.hmgp_kernel_pairs(ctx.h, _d(x), x.shape[0], x.shape[1], C.byref(m), _i(ii), _i(jj),
                                ii.size, _d(out)))
    return out


def at_distance(params, h, ctx=None):
    ctx = ctx or default_context()
    h = np.ascontiguousarray(h, dtype=np.float64)
    out = np.empty_like(h)
    m = _mp(params)
    _chk(_lib.hmgp_at_distance(ctx.h, C.byref(m), _d(h), h.size, _d(out)))
    return out


def bessel_k(nu, x, generic=False, ctx=None):
    ctx = ctx or default_context()
    nu = np.ascontiguousarray(np.broadcast_to(nu, np.shape(x)), dtype=np.float64).ravel()
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    out = np.empty_like(x)
    _chk(_lib.hmgp_bessel_k(ctx.h, _d(nu), _d(x), x.size, int(generic), _d(out)))
    return out


# ----------------------------------------------------------------- H-matrix
class HMatrix:
    def __init__(self, geom: Geometry, params, rc: RankControl, shard=None):
        """shard=(i, n): assemble only the i-th of n cost-balanced contiguous ranges
        of the stored-leaf list (multi-GPU assembly); leaf_range is
        the [begin, end) this object holds payload for."""
        self.g = geom
        self.ctx = geom.ctx
        m = _mp(params)
        r = rc.c()
        h = _vp()
        if shard is None:
            _chk(_lib.hmgp_assemble(self.ctx.h, geom.h, C.byref(m), C.byref(r), C.byref(h)))
            self.leaf_range = None
        else:
            lb, le = C.c_int(), C.c_int()
            _chk(_lib.hmgp_assemble_shard(self.ctx.h, geom.h, C.byref(m), C.byref(r), int(shard[0]),
                                          int(shard[1]), C.byref(h), C.byref(lb), C.byref(le)))
            self.leaf_range = (lb.value, le.value)
        self.h = h

    def __del__(self):
        try:
            _lib.hmgp_hmat_destroy(self.h)
        except Exception:
            pass

    def stats(self):
        b, r, md = C.c_double(), C.c_int(), C.c_double()
        _chk(_lib.hmgp_hmat_stats(self.h, C.byref(b), C.byref(r), C.byref(md)))
        return {"bytes": b.value, "max_rank": r.value, "max_diagonal": md.value,
                "ratio": b.value / (8.0 * self.g.n * self.g.n)}

    def leaves(self):
        cap = 1 << 16
        while True:
            out = np.empty((cap, 6), dtype=np.int32)
            cnt = C.c_int64()
            rc = _lib.hmgp_hmat_leaves(self.h, _i(out), cap, C.byref(cnt))
            if rc == HMGP_ERANGE:
                cap = cnt.value
                continue
            _chk(rc)
            return out[: cnt.value].copy()

    def leaf_data(self, k, info):
        rb, re, cb, ce, kind, rank = (int(v) for v in info)
        m, n = re - rb, ce - cb
        if kind == 1:
            a = np.empty(m * n)
            _chk(_lib.hmgp_hmat_leaf_data(self.h, k, _d(a), None))
            return a.reshape(n, m).T
        u = np.empty(max(1, m * rank))
        v = np.empty(max(1, n * rank))
        _chk(_lib.hmgp_hmat_leaf_data(self.h, k, _d(u), _d(v)))
        return u[: m * rank].reshape(rank, m).T, v[: n * rank].reshape(rank, n).T

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.size != self.g.n:
            raise ValueError("matvec: dimension mismatch")
        y = np.empty(self.g.n)
        _chk(_lib.hmgp_hmat_matvec(self.ctx.h, self.h, _d(x), _d(y)))
        return y

    def to_dense(self):
        """hmatrix.cpp:274-297: entry-wise reconstruction, original order (n <= 4096)."""
        n = self.g.n
        out = np.empty((n, n), order="F")
        _chk(_lib.hmgp_hmat_to_dense(self.ctx.h, self.h, out.ctypes.data_as(_dp)))
        return out


def assemble(geom, params, rc=None):
    """hmatrix.hpp:88-89"""
    return HMatrix(geom, params, rc or RankControl.fixed_accuracy(1e-6))


def assemble_shard(geom, params, shard, n_shards, rc=None):
    """One GPU's share of a sharded assembly."""
    return HMatrix(geom, params, rc or RankControl.fixed_accuracy(1e-6), shard=(shard, n_shards))


def balanced_ranges(cost, parts):
    """Contiguous ranges of `cost` with near-equal sums: bounds[0..parts] (host, C ABI)."""
    c = np.ascontiguousarray(cost, dtype=np.float64)
    b = np.empty(parts + 1, dtype=np.int32)
    _chk(_lib.hmgp_balanced_ranges(_d(c), c.size, parts, _i(b)))
    return b


class HFactor:
    def __init__(self, hm: HMatrix, eps_f, form="ldl"):
        self.hm = hm  # keeps the geometry alive (factor lifetime <= tree lifetime)
        self.ctx = hm.ctx
        self.form = form
        info = _FactorInfo()
        h = _vp()
        _chk(_lib.hmgp_factorize(self.ctx.h, hm.h, eps_f, 1 if form == "ldl" else 0, C.byref(h),
                                 C.byref(info)))
        self.h = h
        self.info = {"eps": info.eps, "clamped": info.clamped, "negative": info.negative,
                     "min_pivot": info.min_pivot, "storage_bytes": info.storage_bytes}

    def __del__(self):
        try:
            _lib.hmgp_factor_destroy(self.h)
        except Exception:
            pass

    def log_det(self):
        o = C.c_double()
        _chk(_lib.hmgp_log_det(self.ctx.h, self.h, C.byref(o)))
        return o.value

    def quad_form(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.size != self.hm.g.n:
            raise ValueError("quad_form: dimension mismatch")
        o = C.c_double()
        _chk(_lib.hmgp_quad_form(self.ctx.h, self.h, _d(b), C.byref(o)))
        return o.value

    def solve_factored(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.size != self.hm.g.n:
            raise ValueError("solve_factored: dimension mismatch")
        x = np.empty_like(b)
        _chk(_lib.hmgp_solve_factored(self.ctx.h, self.h, _d(b), _d(x)))
        return x

    def solve_lower(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.size != self.hm.g.n:
            raise ValueError("solve_lower: dimension mismatch")
        x = np.empty_like(b)
        _chk(_lib.hmgp_solve_lower(self.ctx.h, self.h, _d(b), _d(x)))
        return x

    def diagonal(self):
        x = np.empty(self.hm.g.n)
        _chk(_lib.hmgp_factor_diagonal(self.ctx.h, self.h, _d(x)))
        return x

    def lower_dense(self):
        """hfactor.cpp:421-434: dense L in tree order (n <= 4096)."""
        n = self.hm.g.n
        out = np.empty((n, n), order="F")
        _chk(_lib.hmgp_factor_lower_dense(self.ctx.h, self.h, out.ctypes.data_as(_dp)))
        return out

    def reconstruct(self):
        """hfactor.cpp:436-449: L D L^T (or L L^T) in original order (n <= 4096)."""
        n = self.hm.g.n
        out = np.empty((n, n), order="F")
        _chk(_lib.hmgp_factor_reconstruct(self.ctx.h, self.h, out.ctypes.data_as(_dp)))
        return out


def factorize(hm, eps_f, form="ldl"):
    """hfactor.hpp:70"""
    if not eps_f > 0:
        raise ValueError("factorize: eps_f must be positive")
    return HFactor(hm, eps_f, form)


def h_cholesky(hm, eps_f):
    return factorize(hm, eps_f, "cholesky")


def h_ldl(hm, eps_f):
    return factorize(hm, eps_f, "ldl")


# ----------------------------------------------------------------- pipeline
@dataclass
class LogLikResult:
    """loglik.hpp:10-17"""
    loglik: float
    logdet: float
    quad_form: float
    n: int
    seconds: float
    clamped: bool


def evaluate_loglik(locations, z, params, cfg: HConfig = None, ctx=None):
    """evaluate_loglik (loglik.hpp:22-23) through the C ABI with host buffers."""
    ctx = ctx or default_context()
    cfg = cfg or HConfig()
    x = _pts(locations)
    z = np.ascontiguousarray(z, dtype=np.float64)
    if z.size != x.shape[0]:
        raise ValueError("evaluate_loglik: |z| != n")
    m = _mp(params)
    c = cfg.c()
    r = _LogLik()
    _chk(_lib.hmgp_loglik(ctx.h, _d(x), x.shape[0], x.shape[1], _d(z), C.byref(m), C.byref(c),
                          C.byref(r)))
    return LogLikResult(r.loglik, r.logdet, r.quad_form, r.n, r.seconds, r.status == 1)


@dataclass
class PredictionResult:
    """krige.hpp:10-13"""
    z2_hat: np.ndarray
    seconds: float


def predict(train, z1, new_locations, params, cfg: HConfig = None, ctx=None):
    """predict (krige.hpp:19-21) through the C ABI with host buffers."""
    ctx = ctx or default_context()
    cfg = cfg or HConfig()
    tr = _pts(train)
    z1 = np.ascontiguousarray(z1, dtype=np.float64)
    if z1.size != tr.shape[0]:
        raise ValueError("predict: |z1| != n")
    te = np.ascontiguousarray(new_locations, dtype=np.float64).reshape(-1, tr.shape[1])
    out = np.empty(te.shape[0])
    sec = C.c_double()
    m = _mp(params)
    c = cfg.c()
    _chk(_lib.hmgp_predict(ctx.h, _d(tr), tr.shape[0], tr.shape[1], _d(z1), _d(te), te.shape[0],
                           C.byref(m), C.byref(c), _d(out), C.byref(sec)))
    return PredictionResult(out, sec.value)


def kriging_variance_dense(train, new_locations, params, ctx=None):
    """kriging_variance_dense (krige.hpp / krige.cpp:46-74): σ²+τ² − cᵀC₁₁⁻¹c per new
    location, dense FP64 on the GPU, n <= 4096."""
    ctx = ctx or default_context()
    tr = _pts(train)
    te = np.ascontiguousarray(new_locations, dtype=np.float64).reshape(-1, tr.shape[1])
    out = np.empty(te.shape[0])
    m = _mp(params)
    _chk(_lib.hmgp_kriging_variance_dense(ctx.h, _d(tr), tr.shape[0], tr.shape[1], _d(te), te.shape[0],
                                          C.byref(m), _d(out)))
    return out


@dataclass
class MetricConfig:
    """metrics.hpp:13-17"""
    M: int = 1000
    seed: int = 0
    dense_guard: int = 4096


@dataclass
class MloeMmom:
    """metrics.hpp:19-22"""
    mloe: float
    mmom: float


def mloe_mmom(locations, theta_true, theta_approx, cfg: MetricConfig = None, ctx=None):
    """mloe_mmom (metrics.hpp:24-31 / metrics.cpp:17-69) on the GPU (dense FP64)."""
    ctx = ctx or default_context()
    cfg = cfg or MetricConfig()
    x = _pts(locations)
    mt, ma = _mp(theta_true), _mp(theta_approx)
    a, b = C.c_double(), C.c_double()
    _chk(_lib.hmgp_mloe_mmom(ctx.h, _d(x), x.shape[0], x.shape[1], C.byref(mt), C.byref(ma), cfg.M, cfg.seed,
                             cfg.dense_guard, C.byref(a), C.byref(b)))
    return MloeMmom(a.value, b.value)


def rmse(z_hat, z_true):
    """rmse (metrics.cpp:11-15): host arithmetic on two vectors, as in the reference."""
    a = np.asarray(z_hat, dtype=np.float64)
    b = np.asarray(z_true, dtype=np.float64)
    if a.size != b.size:
        raise ValueError("rmse: length mismatch")
    if a.size == 0:
        raise ValueError("rmse: empty input")
    return float(np.sqrt(np.sum((a - b) ** 2) / a.size))


# -------------------------------------------------------------- data utils
def random_locations(n, seed, dim=2):
    """simgen.cpp:114-123 (dim 3 extends the stream to x, y, z per point)."""
    out = np.empty((n, dim))
    _chk(_lib.hmgp_random_locations(n, dim, seed, _d(out)))
    return out


def jittered_grid(g, seed):
    out = np.empty((g * g, 2))
    _chk(_lib.hmgp_jittered_grid(g, seed, _d(out)))
    return out


def normals(n, seed):
    out = np.empty(n)
    _chk(_lib.hmgp_normals(n, seed, _d(out)))
    return out


def sample_grf(locations, params, seed, ctx=None):
    """sample_grf (simgen.cpp:125-141): exact Gaussian-field sample z = chol(C) w on
    the GPU (dense FP64 covariance + POTRF), w = AS241 normals of `seed`; n <= 65536."""
    ctx = ctx or default_context()
    x = _pts(locations)
    out = np.empty(x.shape[0])
    m = _mp(params)
    _chk(_lib.hmgp_sample_grf(ctx.h, _d(x), x.shape[0], x.shape[1], C.byref(m), seed, _d(out)))
    return out


Z_SEED_XOR = 0x517cc1b727220a95  # cmd_generate's field seed (tools/main.cpp:132)
