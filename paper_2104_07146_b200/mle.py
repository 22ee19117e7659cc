"""Maximum-likelihood driver over the GPU L(θ).

Same names, argument meaning and error behaviour as the reference's
``mle.hpp`` (ReparamPoint, the reparameterisation maps, ``brent_max_1d``,
OptimizerConfig, FitReport, ``fit``) — but the search itself is built for a
GPU that evaluates *batches* of θ, not one scalar probe after another:

* The geometry (cluster tree + block tree) depends only on the locations, so
  ``fit`` builds it ONCE and every probe batch goes through
  ``hmgp_loglik_sweep`` (one geometry, z uploaded once per batch, the θ of a
  batch run concurrently on the device).  The reference rebuilds the tree for
  every probe (loglik.cpp:24-27).
* A 1-D maximisation is a *fan search*: each round evaluates a fan of
  abscissae spread over the current bracket — plus the vertex of the parabola
  through the best three known points — in one batch, then shrinks the bracket
  to the two known neighbours of the best point.  A fan of K points cuts the
  bracket by (K+1)/2 per *batch*; the parabola vertex gives the superlinear
  finish of Brent's method without its one-probe-at-a-time dependency chain.
  Non-finite values count as −inf and an all-infeasible bracket raises, as in
  the reference (mle.cpp:49-150, 152-158).
* Every evaluated (coordinate value → L) pair of a slice is remembered, so a
  bracket expansion re-uses the probes it already paid for.

``fit(..., evaluator=f)`` swaps the L(θ) evaluator (``f(MaternParams) -> float``,
may raise) and ``batch_evaluator=F`` the batched one
(``F(list[MaternParams]) -> list[float]``); tests use the former to run the
identical driver over the CPU oracle.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from typing import Callable, List, Sequence

import numpy as np

from . import HConfig, MaternParams

_NINF = -math.inf
_RT_EPS = math.sqrt(np.finfo(np.float64).eps)


@dataclass
class ReparamPoint:
    """mle.hpp:12-27: sigma = 2/1.1^sigma0, ell = 1/1.5^ell0, nu = 1/1.2^nu0, tau = 1/2^tau0."""
    sigma0: float = 2.0
    ell0: float = 2.0
    nu0: float = 1.0
    tau0: float = 15.0

    _KEYS = ("sigma0", "ell0", "nu0", "tau0")

    def __getitem__(self, i):
        return getattr(self, self._KEYS[min(i, 3)])

    def __setitem__(self, i, v):
        setattr(self, self._KEYS[min(i, 3)], float(v))

    def copy(self):
        return replace(self)

    def with_coord(self, i, v):
        q = replace(self)
        q[i] = v
        return q


def reparam_to_params(p: ReparamPoint) -> MaternParams:
    """The map of mle.hpp:12-16 (θ from the optimiser's unconstrained coordinates)."""
    sigma = 2.0 * 1.1 ** (-p.sigma0)
    tau = 2.0 ** (-p.tau0)
    return MaternParams(sigma2=sigma * sigma, ell=1.5 ** (-p.ell0), nu=1.2 ** (-p.nu0), tau2=tau * tau)


def params_to_reparam(p: MaternParams) -> ReparamPoint:
    """Inverse map; tau2 = 0 has no preimage and maps to tau0 = 50 (mle.cpp:37-46)."""
    if not p.valid():
        raise ValueError("invalid Matern parameters: need sigma2 > 0, ell > 0, nu > 0, tau2 >= 0")
    inv = lambda value, base: -math.log(value) / math.log(base)  # noqa: E731
    return ReparamPoint(inv(math.sqrt(p.sigma2) / 2.0, 1.1), inv(p.ell, 1.5), inv(p.nu, 1.2),
                        inv(math.sqrt(p.tau2), 2.0) if p.tau2 > 0.0 else 50.0)


@dataclass
class BrentResult:  # mle.hpp:29-33
    x: float = 0.0
    fx: float = 0.0
    evals: int = 0


class BracketInfeasible(RuntimeError):
    """Every probe of a bracket was non-finite (std::runtime_error in the reference)."""


# --------------------------------------------------------------- fan search
class _Slice:
    """Known values of a 1-D function: sorted abscissae, −inf for non-finite."""

    def __init__(self, fbatch: Callable[[Sequence[float]], Sequence[float]]):
        self.fbatch = fbatch
        self.t: List[float] = []
        self.f: List[float] = []
        self.evals = 0
        self.finite = False

    def known(self, t):
        return any(t == s for s in self.t)

    def probe(self, ts):
        ts = [t for k, t in enumerate(ts) if not self.known(t) and t not in ts[:k]]
        if not ts:
            return
        vals = self.fbatch(ts)
        self.evals += len(ts)
        for t, y in zip(ts, vals):
            y = float(y) if y is not None and math.isfinite(y) else _NINF
            self.finite = self.finite or y > _NINF
            k = int(np.searchsorted(self.t, t))
            self.t.insert(k, t)
            self.f.insert(k, y)

    def best(self, lo, hi):
        """Index of the best known point in [lo, hi] (lowest abscissa on ties)."""
        b = -1
        for k, t in enumerate(self.t):
            if lo <= t <= hi and (b < 0 or self.f[k] > self.f[b]):
                b = k
        return b


def _vertex(t0, f0, t1, f1, t2, f2):
    """Abscissa of the extremum of the parabola through three points (None if flat/degenerate)."""
    if not (math.isfinite(f0) and math.isfinite(f1) and math.isfinite(f2)):
        return None
    d1, d2 = (t1 - t0) * (f1 - f2), (t1 - t2) * (f1 - f0)
    den = d1 - d2
    if den == 0.0:
        return None
    u = t1 - 0.5 * ((t1 - t0) * d1 - (t1 - t2) * d2) / den
    return u if math.isfinite(u) else None


def fan_max_1d(fbatch, lo, hi, xtol, max_evals, fan=8, known: _Slice = None,
               max_rounds: int = None) -> BrentResult:
    """Maximise a 1-D function on (lo, hi) with batched probes.

    ``fbatch(list of abscissae) -> list of values``; at most ``max_evals`` new
    values are requested in at most ``max_rounds`` batches of ``fan``.  Stops when
    the bracket around the best point is within 2·(√ε|x| + xtol) on both sides."""
    if not lo < hi:
        raise ValueError("brent_max_1d: need lo < hi")
    if max_evals < 3:
        raise ValueError("brent_max_1d: max_evals too small")
    sl = known if known is not None else _Slice(fbatch)
    start = sl.evals
    a, b = lo, hi
    rounds = 0
    while True:
        kb = sl.best(a, b)
        x = sl.t[kb] if kb >= 0 and sl.f[kb] > _NINF else None
        if x is not None:
            # bracket = the known neighbours of the best point (the ends carry no value)
            inner = [t for t in sl.t if a <= t <= b]
            j = inner.index(x)
            a = inner[j - 1] if j > 0 else a
            b = inner[j + 1] if j + 1 < len(inner) else b
        tol = _RT_EPS * abs(x if x is not None else 0.5 * (a + b)) + xtol
        if x is not None and x - a <= 2.0 * tol and b - x <= 2.0 * tol:
            break
        left = max_evals - (sl.evals - start)
        if left <= 0 or (max_rounds is not None and rounds >= max_rounds):
            break
        rounds += 1
        want = []
        if x is None:
            # nothing finite yet: split the widest gaps between what is known
            cuts = [a] + [t for t in sl.t if a < t < b] + [b]
            while len(want) < min(fan, left):
                gaps = sorted(((cuts[i + 1] - cuts[i], i) for i in range(len(cuts) - 1)), reverse=True)
                g, i = gaps[0]
                if not g > 0.0:
                    break
                mid = cuts[i] + 0.5 * g
                if not cuts[i] < mid < cuts[i + 1]:
                    break
                want.append(mid)
                cuts.insert(i + 1, mid)
        else:
            # the vertex of the parabola through the best point and its known neighbours;
            # once it falls within tol of x, close the bracket with x -/+ tol instead
            u = None
            if 0 < kb < len(sl.t) - 1:
                u = _vertex(sl.t[kb - 1], sl.f[kb - 1], x, sl.f[kb], sl.t[kb + 1], sl.f[kb + 1])
            if u is not None and a < u < b and abs(u - x) >= tol:
                want.append(u)
            elif u is not None:
                want += [t for t in (x - tol, x + tol) if a < t < b]
            k = max(1, min(fan, left) - len(want))
            if a < x < b:  # k points that, with x, cut (a, b) evenly on both sides
                nl = min(k, max(0, int(math.floor(k * (x - a) / (b - a) + 0.5))))
                if x - a > 2.0 * tol and nl == 0 and k > 1:
                    nl = 1
                nr = k - nl
                if b - x > 2.0 * tol and nr == 0 and k > 1:
                    nl, nr = nl - 1, 1
                want += [a + (x - a) * (j + 1) / (nl + 1) for j in range(nl)]
                want += [x + (b - x) * (j + 1) / (nr + 1) for j in range(nr)]
            else:
                want += [a + (b - a) * (j + 1) / (k + 1) for j in range(k)]
        seen = []
        for t in want:
            if a < t < b and not sl.known(t) and t not in seen:
                seen.append(t)
        want = seen[:left]
        if not want:
            break
        sl.probe(want)
    if not sl.finite:
        raise BracketInfeasible("brent_max_1d: likelihood undefined on bracket")
    kb = sl.best(lo, hi)
    return BrentResult(sl.t[kb], sl.f[kb], sl.evals - start)


def brent_max_1d(f: Callable[[float], float], lo: float, hi: float, xtol: float,
                 max_evals: int) -> BrentResult:
    """The reference's entry point (mle.hpp:35-38) over a scalar function: same
    contract (maximum on (lo, hi) within xtol, at most max_evals evaluations,
    non-finite = −inf, BracketInfeasible when nothing is finite), computed by
    the fan search with the probes of a round evaluated one after the other."""
    return fan_max_1d(lambda ts: [f(t) for t in ts], lo, hi, xtol, max_evals, fan=4)


# ---------------------------------------------------------------------- fit
@dataclass
class OptimizerConfig:  # mle.hpp:40-49
    initial: ReparamPoint = field(default_factory=ReparamPoint)
    threshold: float = 1e-4
    max_iters: int = 400
    bracket_halfwidth: float = 8.0
    max_bracket_expansions: int = 3
    brent_xtol: float = 1e-3
    brent_max_evals: int = 32  # per 1-D search: probe BATCHES in fit (the dependent chain)
    h: HConfig = field(default_factory=HConfig)
    fan: int = 8  # probes per batch (extension: the device evaluates them concurrently)


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
    batches: int = 0
    trace: List[FitTraceEntry] = field(default_factory=list)


def _gpu_batch_evaluator(x, z, h: HConfig, ctx):
    """L(θ) batches on one prebuilt geometry through hmgp_loglik_sweep."""
    from . import Geometry, default_context, sweep
    ctx = ctx or default_context()
    geom = Geometry(x, h.leaf_size, h.eta, ctx=ctx)

    def run(thetas):
        rows = np.array([[t.sigma2, t.ell, t.nu, t.tau2] for t in thetas], dtype=np.float64)
        ok = [k for k, t in enumerate(thetas) if t.valid()]
        out = [_NINF] * len(thetas)
        if ok:
            _, vals = sweep.sweep_host(geom, z, rows, ok, h, ctx)
            for k, v in zip(ok, vals):
                out[k] = float(v[0]) if v[3] >= 0 else _NINF
        return out

    return run


def fit(locations, z, cfg: OptimizerConfig = None, ctx=None, evaluator=None,
        batch_evaluator=None) -> FitReport:
    """Cyclic coordinate ascent over the reparameterised θ (the reference's outer
    loop and stopping rule, mle.cpp:152-215), each coordinate by a fan search."""
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
    rep = FitReport()
    t0 = time.perf_counter()
    if batch_evaluator is None:
        if evaluator is not None:
            def batch_evaluator(thetas):
                out = []
                for th in thetas:
                    try:
                        out.append(evaluator(th))
                    except Exception:
                        out.append(_NINF)
                return out
        else:
            batch_evaluator = _gpu_batch_evaluator(x, z, cfg.h, ctx)

    def L(points):
        rep.evaluations += len(points)
        rep.batches += 1
        try:
            return list(batch_evaluator([reparam_to_params(p) for p in points]))
        except Exception:
            return [_NINF] * len(points)

    pt = cfg.initial.copy()
    cur = L([pt])[0]
    cur = cur if math.isfinite(cur) else _NINF
    seen_finite = cur > _NINF
    edge = 4.0 * cfg.brent_xtol
    while rep.iterations < cfg.max_iters:
        sweep_start = cur
        for c in range(4):
            if rep.iterations >= cfg.max_iters:
                break
            centre = pt[c]
            sl = _Slice(lambda ts, c=c: L([pt.with_coord(c, t) for t in ts]))
            found = None
            half = cfg.bracket_halfwidth
            for _ in range(cfg.max_bracket_expansions + 1):
                lo, hi = centre - half, centre + half
                try:
                    # brent_max_evals bounds the DEPENDENT chain (batches), as it bounds the
                    # reference's one-probe-at-a-time chain; a batch holds up to `fan` probes
                    found = fan_max_1d(sl.fbatch, lo, hi, cfg.brent_xtol, cfg.brent_max_evals * cfg.fan,
                                       fan=cfg.fan, known=sl, max_rounds=cfg.brent_max_evals)
                except BracketInfeasible:
                    break  # nothing feasible on this bracket: leave the coordinate alone
                if found.x - lo > edge and hi - found.x > edge:
                    break  # interior optimum
                half *= 2.0  # optimum on the rim: widen, keeping what is already known
            rep.iterations += 1
            if found is not None and found.fx > cur:
                pt[c], cur, seen_finite = found.x, found.fx, True
            rep.trace.append(FitTraceEntry(rep.iterations, c, pt.copy(), cur))
        rep.final_sweep_delta = cur - sweep_start
        if cur == _NINF:
            break
        if rep.final_sweep_delta < cfg.threshold:
            rep.converged = True
            break
    if not seen_finite:
        raise RuntimeError("fit: likelihood evaluation failed at every probed point")
    rep.reparam_hat = pt
    rep.theta_hat = reparam_to_params(pt)
    rep.loglik_at_opt = cur
    rep.seconds = time.perf_counter() - t0
    return rep
