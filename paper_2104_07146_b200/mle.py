"""Maximum-likelihood driver over the GPU L(θ).

Python mirror of include/hmgp/mle.hpp, itself the reference's
/root/reference/proj/include/hmgp/mle.hpp + src/mle.cpp: cyclic coordinate
ascent over the log-reparameterised θ, one bracketed Brent maximisation per
coordinate.  Every probe is one ``evaluate_loglik`` (GPU geometry, assembly,
H-factorization, logdet, forward solve); probes that raise score −inf, as in
the reference (mle.cpp:152-158).

``fit(..., evaluator=f)`` swaps the L(θ) evaluator (a callable
``f(MaternParams) -> float`` that may raise); the default is the GPU path.
Tests use it to run the identical driver over the CPU oracle.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from typing import Callable, List

import numpy as np

from . import HConfig, MaternParams, evaluate_loglik

_NINF = -math.inf


@dataclass
class ReparamPoint:
    """mle.hpp:12-27: sigma = 2/1.1^sigma0, ell = 1/1.5^ell0, nu = 1/1.2^nu0, tau = 1/2^tau0."""
    sigma0: float = 2.0
    ell0: float = 2.0
    nu0: float = 1.0
    tau0: float = 15.0

    _KEYS = ("sigma0", "ell0", "nu0", "tau0")

    def __getitem__(self, i):  # mle.cpp:9-24
        return getattr(self, self._KEYS[min(i, 3)])

    def __setitem__(self, i, v):
        setattr(self, self._KEYS[min(i, 3)], float(v))

    def copy(self):
        return replace(self)


def reparam_to_params(p: ReparamPoint) -> MaternParams:
    """mle.cpp:26-35."""
    s = 2.0 * math.pow(1.1, -p.sigma0)
    t = math.pow(2.0, -p.tau0)
    return MaternParams(s * s, math.pow(1.5, -p.ell0), math.pow(1.2, -p.nu0), t * t)


def params_to_reparam(p: MaternParams) -> ReparamPoint:
    """mle.cpp:37-46 (tau2 = 0 has no preimage: 50)."""
    if not p.valid():
        raise ValueError("invalid Matern parameters: need sigma2 > 0, ell > 0, nu > 0, tau2 >= 0")
    return ReparamPoint(
        -math.log(math.sqrt(p.sigma2) / 2.0) / math.log(1.1),
        -math.log(p.ell) / math.log(1.5),
        -math.log(p.nu) / math.log(1.2),
        -math.log(math.sqrt(p.tau2)) / math.log(2.0) if p.tau2 > 0.0 else 50.0)


@dataclass
class BrentResult:  # mle.hpp:29-33
    x: float = 0.0
    fx: float = 0.0
    evals: int = 0


class BracketInfeasible(RuntimeError):
    """brent_max_1d: every probe was non-finite (std::runtime_error in the reference)."""


def brent_max_1d(f: Callable[[float], float], lo: float, hi: float, xtol: float,
                 max_evals: int) -> BrentResult:
    """mle.cpp:49-150: parabolic interpolation with golden-section fallback;
    non-finite values are −inf; raises BracketInfeasible if all probes are."""
    if not lo < hi:
        raise ValueError("brent_max_1d: need lo < hi")
    if max_evals < 3:
        raise ValueError("brent_max_1d: max_evals too small")
    cg = 0.3819660112501051
    rt_eps = math.sqrt(np.finfo(np.float64).eps)
    st = {"evals": 0, "finite": False}

    def probe(t):
        st["evals"] += 1
        y = f(t)
        if not math.isfinite(y):
            return _NINF
        st["finite"] = True
        return y

    a, b = lo, hi
    x = a + cg * (b - a)
    w = v = x
    fx = probe(x)
    fw = fv = fx
    d = e = 0.0
    while st["evals"] < max_evals:
        mid = 0.5 * (a + b)
        tol = rt_eps * abs(x) + xtol
        if abs(x - mid) <= 2.0 * tol - 0.5 * (b - a):
            break
        step = 0.0
        golden = True
        if abs(e) > tol and math.isfinite(fx) and math.isfinite(fw) and math.isfinite(fv):
            r = (x - w) * (fx - fv)
            q = (x - v) * (fx - fw)
            p = (x - v) * q - (x - w) * r
            q = 2.0 * (q - r)
            if q > 0.0:
                p = -p
            q = abs(q)
            e_old, e = e, d
            if abs(p) < abs(0.5 * q * e_old) and p > q * (a - x) and p < q * (b - x):
                step = p / q
                u = x + step
                if u - a < 2.0 * tol or b - u < 2.0 * tol:
                    step = tol if x < mid else -tol
                golden = False
        if golden:
            e = (b if x < mid else a) - x
            step = cg * e
        d = step
        u = x + (step if abs(step) >= tol else (tol if step > 0.0 else -tol))
        fu = probe(u)
        if fu >= fx:
            if u < x:
                b = x
            else:
                a = x
            v, fv, w, fw, x, fx = w, fw, x, fx, u, fu
        else:
            if u < x:
                a = u
            else:
                b = u
            if fu >= fw or w == x:
                v, fv, w, fw = w, fw, u, fu
            elif fu >= fv or v == x or v == w:
                v, fv = u, fu
    if not st["finite"]:
        raise BracketInfeasible("brent_max_1d: likelihood undefined on bracket")
    return BrentResult(x, fx, st["evals"])


@dataclass
class OptimizerConfig:  # mle.hpp:40-49
    initial: ReparamPoint = field(default_factory=ReparamPoint)
    threshold: float = 1e-4
    max_iters: int = 400
    bracket_halfwidth: float = 8.0
    max_bracket_expansions: int = 3
    brent_xtol: float = 1e-3
    brent_max_evals: int = 32
    h: HConfig = field(default_factory=HConfig)


@dataclass
class FitTraceEntry:  # mle.hpp:51-56
    iteration: int
    coordinate: int
    point: ReparamPoint
    loglik: float


@dataclass
class FitReport:  # mle.hpp:58-67
    theta_hat: MaternParams = None
    reparam_hat: ReparamPoint = None
    loglik_at_opt: float = 0.0
    iterations: int = 0
    converged: bool = False
    final_sweep_delta: float = 0.0
    seconds: float = 0.0
    evaluations: int = 0
    trace: List[FitTraceEntry] = field(default_factory=list)


def fit(locations, z, cfg: OptimizerConfig = None, ctx=None, evaluator=None) -> FitReport:
    """mle.cpp:152-215 over the GPU L(θ)."""
    cfg = cfg or OptimizerConfig()
    x = np.asarray(locations, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    if x.size == 0:
        raise ValueError("fit: empty dataset")
    if z.size != x.shape[0]:
        raise ValueError("fit: |z| != n")
    if not cfg.threshold > 0.0:
        raise ValueError("fit: threshold must be > 0")
    if cfg.max_iters < 1:
        raise ValueError("fit: max_iters must be >= 1")
    if evaluator is None:
        def evaluator(th):
            return evaluate_loglik(x, z, th, cfg.h, ctx=ctx).loglik
    t0 = time.perf_counter()
    rep = FitReport()

    def L(p):
        rep.evaluations += 1
        try:
            return evaluator(reparam_to_params(p))
        except Exception:
            return _NINF

    pt = cfg.initial.copy()
    cur = L(pt)
    ok = math.isfinite(cur)
    while rep.iterations < cfg.max_iters:
        start = cur
        for c in range(4):
            if rep.iterations >= cfg.max_iters:
                break
            centre = pt[c]

            def slice_(t, c=c):
                q = pt.copy()
                q[c] = t
                return L(q)

            best = BrentResult(centre, cur, 0)
            half = cfg.bracket_halfwidth
            for _ in range(cfg.max_bracket_expansions + 1):
                lo, hi = centre - half, centre + half
                try:
                    r = brent_max_1d(slice_, lo, hi, cfg.brent_xtol, cfg.brent_max_evals)
                except BracketInfeasible:
                    break
                best = r
                edge = 4.0 * cfg.brent_xtol
                if r.x - lo > edge and hi - r.x > edge:
                    break
                half *= 2.0
            rep.iterations += 1
            if math.isfinite(best.fx) and best.fx > cur:
                pt[c] = best.x
                cur = best.fx
                ok = True
            rep.trace.append(FitTraceEntry(rep.iterations, c, pt.copy(), cur))
        rep.final_sweep_delta = cur - start
        if not math.isfinite(cur):
            break
        if rep.final_sweep_delta < cfg.threshold:
            rep.converged = True
            break
    if not ok:
        raise RuntimeError("fit: likelihood evaluation failed at every probed point")
    rep.reparam_hat = pt
    rep.theta_hat = reparam_to_params(pt)
    rep.loglik_at_opt = cur
    rep.seconds = time.perf_counter() - t0
    return rep
