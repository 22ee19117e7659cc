"""ctypes loader for the CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(paper_2104_07146_b200) never imports it.

* ``Oracle``  -> oracle/build/libhmgp_oracle.so  (this repo's restatement)
* ``RefLib``  -> oracle/_ref/libhmgp_ref.so      (UNMODIFIED reference
  geometry.cpp + covkernel.cpp compiled from /root/reference)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libhmgp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhmgp_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def build():
    """Compile oracle/ (restatement always; _ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(RuntimeError):
    def __init__(self, code, msg, pivot_index=-1, pivot_value=0.0):
        super().__init__(msg)
        self.code = code
        self.pivot_index = pivot_index
        self.pivot_value = pivot_value


class Config(C.Structure):
    _fields_ = [("eta", C.c_double), ("leaf_size", C.c_int), ("eps", C.c_double),
                ("fixed_rank", C.c_int), ("max_rank", C.c_int), ("eps_factor", C.c_double),
                ("ldl", C.c_int), ("threads", C.c_int)]


class FactorInfo(C.Structure):
    _fields_ = [("clamped", C.c_int), ("negative", C.c_int), ("min_pivot", C.c_double),
                ("storage_bytes", C.c_double)]


class LogLikResult(C.Structure):
    _fields_ = [("loglik", C.c_double), ("logdet", C.c_double), ("quad_form", C.c_double),
                ("n", C.c_int), ("clamped", C.c_int), ("seconds", C.c_double),
                ("t_tree", C.c_double), ("t_assemble", C.c_double), ("t_factor", C.c_double)]


def make_config(eta=2.0, leaf_size=32, eps=1e-6, fixed_rank=0, max_rank=256, eps_factor=-1.0,
                form="ldl", threads=1):
    return Config(eta, leaf_size, eps, fixed_rank, max_rank, eps_factor,
                  1 if form == "ldl" else 0, threads)


def _xy(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.ndim == 2 and x.shape[1] in (2, 3)
    return x


class Oracle:
    """The C++ restatement of the reference hot path."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.L = C.CDLL(path)
        L = self.L
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_pivot_value.restype = C.c_double
        L.orc_problem_create.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.POINTER(C.c_void_p)]
        L.orc_problem_destroy.argtypes = [C.c_void_p]
        for name in ("orc_assemble", "orc_leaves", "orc_leaf_data", "orc_hmat_stats",
                     "orc_matvec", "orc_factorize", "orc_log_det", "orc_quad_form",
                     "orc_solve_factored", "orc_solve_lower", "orc_factor_diag"):
            getattr(L, name).argtypes = None
        L.orc_random_locations.argtypes = [C.c_int, C.c_int, C.c_uint64, _dp]
        L.orc_jittered_grid.argtypes = [C.c_int, C.c_uint64, _dp]
        L.orc_normals.argtypes = [C.c_int, C.c_uint64, _dp]
        L.orc_sample_grf.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_uint64, C.c_int, _dp]
        L.orc_bessel_k.argtypes = [C.c_double, C.c_double, C.c_int, _dp]
        L.orc_matern.argtypes = [C.c_double, _dp, C.c_int, _dp]
        L.orc_normal_quantile.argtypes = [C.c_double, _dp]
        L.orc_block_tree.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_double, _ip, C.c_int64,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_cluster_tree.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip, C.POINTER(C.c_int)]
        L.orc_at_distance.argtypes = [_dp, _dp, C.c_int64, _dp]
        L.orc_kernel_pairs.argtypes = [_dp, C.c_int, C.c_int, _dp, _ip, _ip, C.c_int64, _dp]
        L.orc_loglik.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.POINTER(Config),
                                 C.POINTER(LogLikResult)]
        L.orc_predict.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp,
                                  C.POINTER(Config), _dp, _dp]
        L.orc_cross_apply.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, C.c_int, _dp]
        L.orc_dense_loglik.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp]
        L.orc_dense_predict.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, _dp, C.c_int, _dp]
        L.orc_kriging_variance_dense.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, _dp, _dp]
        L.orc_mloe_mmom.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_uint64, C.c_int,
                                    _dp, _dp]

    def _chk(self, rc):
        if rc != 0:
            msg = self.L.orc_last_error().decode()
            raise OracleError(rc, msg, self.L.orc_last_pivot_index(), self.L.orc_last_pivot_value())

    # ---- inputs (simgen conventions) ----
    def random_locations(self, n, seed, dim=2):
        out = np.empty((n, dim))
        self._chk(self.L.orc_random_locations(n, dim, seed, _d(out)))
        return out

    def jittered_grid(self, g, seed):
        out = np.empty((g * g, 2))
        self._chk(self.L.orc_jittered_grid(g, seed, _d(out)))
        return out

    def normals(self, n, seed):
        out = np.empty(n)
        self._chk(self.L.orc_normals(n, seed, _d(out)))
        return out

    def sample_grf(self, x, theta, seed, threads=0):
        x = _xy(x)
        th = np.asarray(theta, dtype=np.float64)
        z = np.empty(x.shape[0])
        self._chk(self.L.orc_sample_grf(_d(x), x.shape[0], x.shape[1], _d(th), seed,
                                        threads or os.cpu_count(), _d(z)))
        return z

    def normal_quantile(self, p):
        o = C.c_double()
        self._chk(self.L.orc_normal_quantile(p, C.byref(o)))
        return o.value

    # ---- geometry ----
    def cluster_perm(self, x, leaf):
        x = _xy(x)
        perm = np.empty(x.shape[0], dtype=np.int32)
        nn = C.c_int()
        self._chk(self.L.orc_cluster_tree(_d(x), x.shape[0], x.shape[1], leaf, _i(perm),
                                          C.byref(nn)))
        return perm

    def block_leaves(self, x, leaf, eta):
        x = _xy(x)
        n = x.shape[0]
        cap = max(64, 64 * (n // max(1, leaf) + 1) * 8)
        while True:
            out = np.empty((cap, 5), dtype=np.int32)
            cnt, na, nd = C.c_int64(), C.c_int(), C.c_int()
            rc = self.L.orc_block_tree(_d(x), n, x.shape[1], leaf, eta, _i(out), cap,
                                       C.byref(cnt), C.byref(na), C.byref(nd))
            if rc == 3 and cnt.value > cap:
                cap = cnt.value
                continue
            self._chk(rc)
            return out[: cnt.value].copy(), na.value, nd.value

    # ---- kernel ----
    def bessel_k(self, nu, x, generic=False):
        o = C.c_double()
        self._chk(self.L.orc_bessel_k(nu, x, int(generic), C.byref(o)))
        return o.value

    def matern(self, h, theta, generic=False):
        o = C.c_double()
        th = np.asarray(theta, dtype=np.float64)
        self._chk(self.L.orc_matern(h, _d(th), int(generic), C.byref(o)))
        return o.value

    def at_distance(self, theta, h):
        th = np.asarray(theta, dtype=np.float64)
        h = np.ascontiguousarray(h, dtype=np.float64)
        out = np.empty_like(h)
        self._chk(self.L.orc_at_distance(_d(th), _d(h), h.size, _d(out)))
        return out

    def kernel_pairs(self, x, theta, ii, jj):
        x = _xy(x)
        th = np.asarray(theta, dtype=np.float64)
        ii = np.ascontiguousarray(ii, dtype=np.int32)
        jj = np.ascontiguousarray(jj, dtype=np.int32)
        out = np.empty(ii.size)
        self._chk(self.L.orc_kernel_pairs(_d(x), x.shape[0], x.shape[1], _d(th), _i(ii), _i(jj),
                                          ii.size, _d(out)))
        return out

    # ---- pipeline ----
    def loglik(self, x, z, theta, cfg):
        x = _xy(x)
        z = np.ascontiguousarray(z, dtype=np.float64)
        th = np.asarray(theta, dtype=np.float64)
        res = LogLikResult()
        self._chk(self.L.orc_loglik(_d(x), x.shape[0], x.shape[1], _d(z), _d(th),
                                    C.byref(cfg), C.byref(res)))
        return res

    def predict(self, train, z1, test, theta, cfg):
        train, test = _xy(train), _xy(test)
        z1 = np.ascontiguousarray(z1, dtype=np.float64)
        th = np.asarray(theta, dtype=np.float64)
        out = np.empty(test.shape[0])
        sec = C.c_double()
        self._chk(self.L.orc_predict(_d(train), train.shape[0], train.shape[1], _d(z1), _d(test),
                                     test.shape[0], _d(th), C.byref(cfg), _d(out), C.byref(sec)))
        return out

    def cross_apply(self, train, w, test, theta, threads=1):
        train, test = _xy(train), _xy(test)
        w = np.ascontiguousarray(w, dtype=np.float64)
        th = np.asarray(theta, dtype=np.float64)
        out = np.empty(test.shape[0])
        self._chk(self.L.orc_cross_apply(_d(train), train.shape[0], train.shape[1], _d(w),
                                         _d(test), test.shape[0], _d(th), threads, _d(out)))
        return out

    def dense_loglik(self, x, z, theta, threads=0):
        x = _xy(x)
        z = np.ascontiguousarray(z, dtype=np.float64)
        th = np.asarray(theta, dtype=np.float64)
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._chk(self.L.orc_dense_loglik(_d(x), x.shape[0], x.shape[1], _d(z), _d(th),
                                          threads or os.cpu_count(), C.byref(a), C.byref(b),
                                          C.byref(c)))
        return a.value, b.value, c.value

    def dense_predict(self, train, z1, test, theta, threads=0):
        train, test = _xy(train), _xy(test)
        z1 = np.ascontiguousarray(z1, dtype=np.float64)
        th = np.asarray(theta, dtype=np.float64)
        out = np.empty(test.shape[0])
        self._chk(self.L.orc_dense_predict(_d(train), train.shape[0], train.shape[1], _d(z1),
                                           _d(test), test.shape[0], _d(th),
                                           threads or os.cpu_count(), _d(out)))
        return out

    def kriging_variance_dense(self, train, test, theta):
        """krige.cpp:46-74 restated (hmgp_oracle.cpp orc_kriging_variance_dense)."""
        train, test = _xy(train), _xy(test)
        th = np.asarray(theta, dtype=np.float64)
        out = np.empty(test.shape[0])
        self._chk(self.L.orc_kriging_variance_dense(_d(train), train.shape[0], train.shape[1],
                                                    _d(test), test.shape[0], _d(th), _d(out)))
        return out

    def mloe_mmom(self, x, theta_true, theta_approx, M=1000, seed=0, dense_guard=4096):
        """metrics.cpp:17-69 restated (hmgp_oracle.cpp orc_mloe_mmom) -> (mloe, mmom)."""
        x = _xy(x)
        tt = np.asarray(theta_true, dtype=np.float64)
        ta = np.asarray(theta_approx, dtype=np.float64)
        a, b = C.c_double(), C.c_double()
        self._chk(self.L.orc_mloe_mmom(_d(x), x.shape[0], x.shape[1], _d(tt), _d(ta), M, seed,
                                       dense_guard, C.byref(a), C.byref(b)))
        return a.value, b.value

    def counters(self):
        out = np.zeros(11)
        self.L.orc_counters(_d(out))
        keys = ("entries_dense", "entries_aca", "fl_gemm", "fl_qr", "fl_svd", "fl_trsm",
                "fl_leaf", "n_truncate", "n_add", "n_gemm", "n_trsm")
        return dict(zip(keys, out.tolist()))

    def counters_reset(self):
        self.L.orc_counters_reset()

    def problem(self, x, leaf, eta):
        return Problem(self, x, leaf, eta)


class Problem:
    """Handle over one (tree, block tree, H-matrix, factor) in the oracle."""

    def __init__(self, orc: Oracle, x, leaf, eta):
        self.o = orc
        self.x = _xy(x)
        self.n = self.x.shape[0]
        h = C.c_void_p()
        orc._chk(orc.L.orc_problem_create(_d(self.x), self.n, self.x.shape[1], leaf, eta,
                                          C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.o.L.orc_problem_destroy(self.h)
        except Exception:
            pass

    def assemble(self, theta, cfg):
        th = np.asarray(theta, dtype=np.float64)
        sec = C.c_double()
        self.o._chk(self.o.L.orc_assemble(self.h, _d(th), C.byref(cfg), C.byref(sec)))
        return sec.value

    def leaves(self):
        cap = 1 << 16
        while True:
            out = np.empty((cap, 6), dtype=np.int32)
            cnt = C.c_int64()
            rc = self.o.L.orc_leaves(self.h, _i(out), C.c_int64(cap), C.byref(cnt))
            if rc == 3:
                cap = cnt.value
                continue
            self.o._chk(rc)
            return out[: cnt.value].copy()

    def leaf_data(self, k, info):
        rb, re, cb, ce, kind, rank = (int(v) for v in info)
        m, n = re - rb, ce - cb
        if kind == 1:
            a = np.empty(m * n)
            self.o._chk(self.o.L.orc_leaf_data(self.h, C.c_int64(k), _d(a), None))
            return a.reshape(n, m).T
        u = np.empty(max(1, m * rank))
        v = np.empty(max(1, n * rank))
        self.o._chk(self.o.L.orc_leaf_data(self.h, C.c_int64(k), _d(u), _d(v)))
        return u[: m * rank].reshape(rank, m).T, v[: n * rank].reshape(rank, n).T

    def stats(self):
        b, r, md = C.c_double(), C.c_int(), C.c_double()
        self.o._chk(self.o.L.orc_hmat_stats(self.h, C.byref(b), C.byref(r), C.byref(md)))
        return b.value, r.value, md.value

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        self.o._chk(self.o.L.orc_matvec(self.h, _d(x), _d(y)))
        return y

    def factorize(self, eps_f, form="ldl"):
        info = FactorInfo()
        sec = C.c_double()
        self.o._chk(self.o.L.orc_factorize(self.h, C.c_double(eps_f), 1 if form == "ldl" else 0,
                                           C.byref(info), C.byref(sec)))
        return info, sec.value

    def log_det(self):
        o = C.c_double()
        self.o._chk(self.o.L.orc_log_det(self.h, C.byref(o)))
        return o.value

    def quad_form(self, z):
        z = np.ascontiguousarray(z, dtype=np.float64)
        o = C.c_double()
        self.o._chk(self.o.L.orc_quad_form(self.h, _d(z), C.byref(o)))
        return o.value

    def solve_factored(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.n)
        self.o._chk(self.o.L.orc_solve_factored(self.h, _d(b), _d(x)))
        return x

    def factor_diag(self):
        x = np.empty(self.n)
        self.o._chk(self.o.L.orc_factor_diag(self.h, _d(x)))
        return x


class RefLib:
    """The unmodified reference geometry.cpp + covkernel.cpp (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.L = C.CDLL(path)
        L = self.L
        L.ref_last_error.restype = C.c_char_p
        L.ref_cluster_tree.argtypes = [_dp, C.c_int, C.c_int, _ip, _ip, C.POINTER(C.c_int)]
        L.ref_block_tree.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _ip, C.c_int64,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_bessel_k.argtypes = [C.c_double, C.c_double, _dp]
        L.ref_bessel_k_generic.argtypes = [C.c_double, C.c_double, _dp]
        L.ref_matern.argtypes = [C.c_double, _dp, _dp]
        L.ref_matern_generic.argtypes = [C.c_double, _dp, _dp]
        L.ref_kernel_pairs.argtypes = [_dp, C.c_int, _dp, _ip, _ip, C.c_int64, _dp]
        L.ref_at_distance.argtypes = [_dp, _dp, C.c_int64, _dp]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def cluster_perm(self, x, leaf):
        x = _xy(x)
        assert x.shape[1] == 2
        n = x.shape[0]
        perm = np.empty(n, dtype=np.int32)
        inv = np.empty(n, dtype=np.int32)
        nl = C.c_int()
        self._chk(self.L.ref_cluster_tree(_d(x), n, leaf, _i(perm), _i(inv), C.byref(nl)))
        return perm

    def block_leaves(self, x, leaf, eta):
        x = _xy(x)
        n = x.shape[0]
        cap = max(64, 64 * (n // max(1, leaf) + 1) * 8)
        while True:
            out = np.empty((cap, 5), dtype=np.int32)
            cnt, na, nd = C.c_int64(), C.c_int(), C.c_int()
            rc = self.L.ref_block_tree(_d(x), n, leaf, eta, _i(out), cap, C.byref(cnt),
                                       C.byref(na), C.byref(nd))
            if rc == 3 and cnt.value > cap:
                cap = cnt.value
                continue
            self._chk(rc)
            return out[: cnt.value].copy(), na.value, nd.value

    def bessel_k(self, nu, x, generic=False):
        o = C.c_double()
        f = self.L.ref_bessel_k_generic if generic else self.L.ref_bessel_k
        self._chk(f(nu, x, C.byref(o)))
        return o.value

    def matern(self, h, theta, generic=False):
        o = C.c_double()
        th = np.asarray(theta, dtype=np.float64)
        f = self.L.ref_matern_generic if generic else self.L.ref_matern
        self._chk(f(h, _d(th), C.byref(o)))
        return o.value

    def at_distance(self, theta, h):
        th = np.asarray(theta, dtype=np.float64)
        h = np.ascontiguousarray(h, dtype=np.float64)
        out = np.empty_like(h)
        self._chk(self.L.ref_at_distance(_d(th), _d(h), h.size, _d(out)))
        return out

    def kernel_pairs(self, x, theta, ii, jj):
        x = _xy(x)
        th = np.asarray(theta, dtype=np.float64)
        ii = np.ascontiguousarray(ii, dtype=np.int32)
        jj = np.ascontiguousarray(jj, dtype=np.int32)
        out = np.empty(ii.size)
        self._chk(self.L.ref_kernel_pairs(_d(x), x.shape[0], _d(th), _i(ii), _i(jj), ii.size,
                                          _d(out)))
        return out


def ref_available():
    return os.path.exists(REF_SO)
