"""Experiment drivers on the B200 backend.

Reference: `cmd_bench_dense` / `cmd_bench_action` (proj/core/src/cli.cpp:290-374), `cmd_theta`
(cli.cpp:136-167) and the acceptance suite's figure-trend / bound-compliance checks
(proj/tests/acceptance_main.cpp:150-252), which reproduce the paper's Fig. 2/3/4 trends.

Layout of a run:
* the methods under test are evaluated on the GPU -- every grid point of a dense sweep in ONE batched
  `pf_eval_dense_batched` launch (the partial-fraction methods), the Padé / Taylor comparators
  (dense.cpp:254-332) as batched DMMA GEMMs + batched LU solves on the same engine, the action
  methods through `pf_tridiag_action` / `pf_tridiag_matvec_batched`;
* the high-precision oracle stays on the host CPU (binary128 restatement of the reference's GMP
  oracles, cpp/src/hp_oracle.cpp), as does `two_norm_est`;
* output is the reference's CSV, byte for byte in format (`format_sig17` fields).

CLI: ``python -m paper_2210_03714_b200.drivers bench-dense --methods R4,R8,pade4 --dim 50``
(see ``--help``).
"""
from __future__ import annotations

import argparse
import ctypes as C
import math
import sys
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import methods as M
from . import workloads as W
from .errors import Errc, PfError
from .methods import format_sig17

DEFAULT_DIGITS = 40
K_INVERSE_PRODUCTS = 4.0 / 3.0  # dense inverse, in products (cli.cpp:161)
MATVEC_PER_D, SOLVE_PER_D = 5.0, 8.0  # CostModel::tridiagonal (action.hpp:91-92)


def _host():
    lib = W._host()
    if not getattr(lib, "_pf_drivers_bound", False):
        lib.pf_hp_dense_diff.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        lib.pf_hp_dense_diff.restype = C.c_int
        lib.pf_hp_action_error.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                           C.c_void_p, C.c_void_p]
        lib.pf_hp_action_error.restype = C.c_int
        lib.pf_two_norm_est_dense.argtypes = [C.c_int, C.c_void_p, C.c_int]
        lib.pf_two_norm_est_dense.restype = C.c_double
        lib.pf_two_norm_est_tridiag.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        lib.pf_two_norm_est_tridiag.restype = C.c_double
        lib._pf_drivers_bound = True
    return lib


def _c(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------------------------- inputs


@dataclass
class MatrixSpec:
    """MatrixSpec (cli.hpp): kind randn | cauchy | trid121, dimension, seed."""

    kind: str = "randn"
    dim: int = 50
    seed: int = 1

    def __post_init__(self):
        if self.kind not in ("randn", "cauchy", "trid121"):
            raise PfError(Errc.BadArgument, "unknown matrix kind: " + self.kind)


def make_dense_matrix(spec: MatrixSpec) -> np.ndarray:
    """make_dense_matrix (cli.cpp:35-56)."""
    if spec.dim < 1:
        raise PfError(Errc.BadArgument, "matrix dimension must be >= 1")
    if spec.kind == "randn":
        return W.randn_matrix(spec.dim, spec.seed)
    if spec.kind == "cauchy":
        return W.cauchy(spec.dim)
    return W.trid121_dense(spec.dim)


def trid121(d: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """TridiagMatrix::trid121 (action.cpp:27-33): sub / super -1, diagonal 2."""
    return -np.ones(d - 1), 2 * np.ones(d), -np.ones(d - 1)


def exact_decimal_string(x: float) -> str:
    """exact_decimal_string (rational.cpp:95-115): x = n / 2^k exactly, digits of n 5^k."""
    from fractions import Fraction

    if x == 0.0:
        return "0"
    if not math.isfinite(x):
        raise PfError(Errc.BadArgument, "non-finite value has no exact decimal")
    q = Fraction(x)
    neg = q < 0
    q = abs(q)
    num, den = q.numerator, q.denominator
    k = den.bit_length() - 1  # den is a power of two
    d = str(num * 5 ** k)
    exp10 = len(d) - 1 - k
    d = d.rstrip("0") or "0"
    out = ("-" if neg else "") + d[0]
    if len(d) > 1:
        out += "." + d[1:]
    if exp10 != 0:
        out += "e" + str(exp10)
    return out


def random_unit_vector(dim: int, seed: int) -> np.ndarray:
    """random_unit_vector (cli.cpp:65-78): NormalSampler draws, divided by their sequential 2-norm."""
    if dim < 1:
        raise PfError(Errc.BadArgument, "vector dimension must be >= 1")
    v = W.randn(seed, dim)
    n2 = 0.0
    for e in v:
        n2 += e * e
    n2 = math.sqrt(n2)
    return v / n2 if n2 > 0 else v


def log_grid(lo: float, hi: float, n: int) -> List[float]:
    """log_grid (cli.cpp:80-91)."""
    if n < 1 or lo <= 0 or hi < lo:
        raise PfError(Errc.BadArgument, "bad log grid")
    if n == 1:
        return [lo]
    ratio = math.log(hi / lo) / (n - 1)
    return [lo * math.exp(ratio * i) for i in range(n)]


def two_norm_est(m: np.ndarray, iterations: int = 120) -> float:
    """two_norm_est (dense.cpp:70-96; default 120 iterations, dense.hpp:42)."""
    m = _c(m)
    return _host().pf_two_norm_est_dense(m.shape[0], m.ctypes.data, iterations)


def two_norm_est_tridiag(sub, diag, sup, iterations: int = 200) -> float:
    """two_norm_est (action.cpp:67-94; default 200 iterations, action.hpp:27)."""
    sub, diag, sup = _c(sub), _c(diag), _c(sup)
    return _host().pf_two_norm_est_tridiag(len(diag), sub.ctypes.data, diag.ctypes.data, sup.ctypes.data, iterations)


# -------------------------------------------------------------------------------------- oracles


def dense_errors(kind: str, b: np.ndarray, approx: Sequence[np.ndarray], digits: int = DEFAULT_DIGITS) -> List[float]:
    """error_vs_oracle(expm_oracle(b) or phi1_oracle(b), approx_t) for each approximation
    (dense.cpp:460-499): one high-precision evaluation shared by all of them."""
    b = _c(b)
    d = b.shape[0]
    ap = _c(np.stack([np.asarray(a, dtype=np.float64) for a in approx]))
    diff = np.empty_like(ap)
    rc = _host().pf_hp_dense_diff(0 if kind == "exp" else 1, d, b.ctypes.data, digits, len(approx), ap.ctypes.data,
                                  diff.ctypes.data)
    if rc:
        raise PfError(Errc.BadArgument, "oracle digits must be >= 30")
    return [two_norm_est(diff[t]) for t in range(len(approx))]


def action_errors(sub, diag, sup, v, approx: Sequence[np.ndarray], digits: int = DEFAULT_DIGITS) -> List[float]:
    """error_vs_oracle(action_oracle(a, v), approx_t) (action.cpp:440-502)."""
    sub, diag, sup, v = _c(sub), _c(diag), _c(sup), _c(v)
    ap = _c(np.stack([np.asarray(a, dtype=np.float64) for a in approx]))
    err = np.empty(len(approx))
    rc = _host().pf_hp_action_error(len(diag), sub.ctypes.data, diag.ctypes.data, sup.ctypes.data, v.ctypes.data,
                                    digits, len(approx), ap.ctypes.data, err.ctypes.data)
    if rc:
        raise PfError(Errc.BadArgument, "oracle digits must be >= 30")
    return list(err)


# ---------------------------------------------------------------- comparators on the GPU engine


def _dev(Bs: np.ndarray):
    import torch

    return torch.from_numpy(_c(Bs)).cuda()


def _eye_like(t):
    import torch

    return torch.eye(t.shape[-1], dtype=t.dtype, device=t.device).expand_as(t).clone()


def _solve(den, num):
    from . import api

    return api.DenseLu(den).solve_matrix(num)


def pade4(Bs):
    """pade4 (dense.cpp:254-264): (I - B/2 + B^2/12)^{-1} (I + B/2 + B^2/12)."""
    from . import api

    b2 = api.gemm(Bs, Bs)
    num = _eye_like(Bs) + 0.5 * Bs + (1.0 / 12.0) * b2
    den = _eye_like(Bs) - 0.5 * Bs + (1.0 / 12.0) * b2
    return _solve(den, num)


def pade4_phi1(Bs):
    """pade4_phi1 (dense.cpp:266-276)."""
    from . import api

    b2 = api.gemm(Bs, Bs)
    num = _eye_like(Bs) + (1.0 / 10.0) * Bs + (1.0 / 60.0) * b2
    den = _eye_like(Bs) - (2.0 / 5.0) * Bs + (1.0 / 20.0) * b2
    return _solve(den, num)


def taylor8(Bs):
    """taylor8 (dense.cpp:278-307): degree-8 Taylor polynomial in three products."""
    from . import api

    s = math.sqrt(177.0)
    x3 = 2.0 / 3.0
    x1 = x3 * (1.0 + s) / 88.0
    x2 = x3 * (1.0 + s) / 352.0
    x4 = (-271.0 + 29.0 * s) / (315.0 * x3)
    x5 = 11.0 * (-1.0 + s) / (1260.0 * x3)
    x6 = 11.0 * (-9.0 + s) / (5040.0 * x3)
    x7 = (89.0 - s) / (5040.0 * x3 * x3)
    y2 = (857.0 - 58.0 * s) / 630.0
    b2 = api.gemm(Bs, Bs)
    t = x1 * Bs + x2 * b2
    b4 = api.gemm(b2, t)
    left = x3 * b2 + b4
    right = x4 * _eye_like(Bs) + x5 * Bs + x6 * b2 + x7 * b4
    b8 = api.gemm(left, right)
    return _eye_like(Bs) + Bs + y2 * b2 + b8


def pade10(Bs):
    """pade10 (dense.cpp:309-332)."""
    from . import api

    c0, c1, c2, c3, c4, c5 = 1.0, 0.5, 1.0 / 9.0, 1.0 / 72.0, 1.0 / 1008.0, 1.0 / 30240.0
    a2 = api.gemm(Bs, Bs)
    a4 = api.gemm(a2, a2)
    inner = c1 * _eye_like(Bs) + c3 * a2 + c5 * a4
    u = api.gemm(Bs, inner)
    v = c0 * _eye_like(Bs) + c2 * a2 + c4 * a4
    return _solve(v - u, v + u)


_COMPARATORS = {
    "pade4": ("exp", pade4, 1.0 + K_INVERSE_PRODUCTS),
    "pade4_phi1": ("phi1", pade4_phi1, 1.0 + K_INVERSE_PRODUCTS),
    "taylor8": ("exp", taylor8, 3.0),
    "pade10": ("exp", pade10, 3.0 + K_INVERSE_PRODUCTS),
}


def split_form(token: str) -> Tuple[str, Optional[int]]:
    """token = base[:plain|:residual] (cli.cpp:178-186)."""
    if ":" not in token:
        return token, None
    base, suffix = token.split(":", 1)
    if suffix == "plain":
        return base, M.PLAIN
    if suffix == "residual":
        return base, M.RESIDUAL
    raise PfError(Errc.BadArgument, "unknown form suffix in token: " + token)


@dataclass
class DenseEntry:
    token: str
    function: str  # "exp" | "phi1"
    evaluate: Callable  # (batch of B on the device) -> batch of f(B)
    serial_cost: float
    parallel_cost: float


def _function_name(fn) -> str:
    if fn == M.FunctionId.exp():
        return "exp"
    if fn == M.FunctionId.phi(1):
        return "phi1"
    return fn.name()


def dense_entry(token: str) -> DenseEntry:
    """dense_entry (cli.cpp:188-227)."""
    if token in _COMPARATORS:
        fn, ev, cost = _COMPARATORS[token]
        return DenseEntry(token, fn, ev, cost, cost)
    base, form = split_form(token)
    m = M.catalog(base)
    if form is not None:
        m = M.to_residual_form(m) if form == M.RESIDUAL else M.to_plain_form(m)
    poly_products = 1.0 if len(m.poly) == 3 else 0.0

    def ev(Bs, m=m):
        from . import _native as N, api

        # The plain form's round-off plateau decides the figure trends (acceptance_main.cpp:199-212):
        # evaluate it in the reference's exact operation order (bit-identical to dense.cpp).
        flags = N.PF_FLAG_REFERENCE_ORDER if m.form == M.PLAIN and Bs.shape[-1] <= N.PF_SMALL_N else 0
        return api.eval_dense(m, Bs, flags=flags)

    return DenseEntry(token, _function_name(m.function), ev, m.processors() * K_INVERSE_PRODUCTS + poly_products,
                      max(K_INVERSE_PRODUCTS, poly_products))


@dataclass
class ActionEntry:
    token: str
    evaluate: Callable  # (sub, diag, sup, V d x k) -> d x k
    serial_cost: float
    parallel_cost: float


def dense_action_taylor(degree: int, sub, diag, sup, V):
    """taylor_action (action.cpp:341-352) on a block of vectors: degree matvecs on the GPU."""
    from . import api

    t = api.TridiagMatrix(sub, diag, sup)
    acc = np.array(V, dtype=np.float64, copy=True)
    w = acc.copy()
    for k in range(1, degree + 1):
        w = api.tridiag_matvec(t, w) * (1.0 / k)
        acc = acc + w
    return acc


def action_entry(token: str) -> ActionEntry:
    """action_entry (cli.cpp:229-265)."""
    if token.startswith("taylor"):
        try:
            degree = int(token[6:])
        except ValueError:
            raise PfError(Errc.BadArgument, "bad taylor token: " + token) from None
        if degree < 1:
            raise PfError(Errc.BadArgument, "bad taylor token: " + token)
        return ActionEntry(token, lambda s, d, u, V, n=degree: dense_action_taylor(n, s, d, u, V), float(degree),
                           float(degree))
    base, form = split_form(token)
    m = M.catalog(base)
    if form is not None:
        m = M.to_residual_form(m) if form == M.RESIDUAL else M.to_plain_form(m)
    if m.function != M.FunctionId.exp():
        raise PfError(Errc.BadArgument, "action benchmark targets the exponential; token %s approximates %s"
                      % (token, m.function.name()))
    per_solve = SOLVE_PER_D + MATVEC_PER_D if m.form == M.RESIDUAL else SOLVE_PER_D
    poly = 2.0 * MATVEC_PER_D if len(m.poly) == 3 else 0.0

    def ev(s, d, u, V, m=m):
        from . import api

        return api.tridiag_action(m, api.TridiagMatrix(s, d, u), V, 1, m.form)

    return ActionEntry(token, ev, (m.processors() * per_solve + poly) / MATVEC_PER_D, max(per_solve, poly) / MATVEC_PER_D)


# -------------------------------------------------------------------------------------- commands


def _render(cost_unit: str, rows: Sequence[Tuple[str, float, float, float, float]]) -> str:
    out = ["method,h_norm,error_2norm,serial_cost_%s,parallel_cost_%s" % (cost_unit, cost_unit)]
    for r in rows:
        out.append("%s,%s,%s,%s,%s" % (r[0], format_sig17(r[1]), format_sig17(r[2]), format_sig17(r[3]),
                                       format_sig17(r[4])))
    return "\n".join(out) + "\n"


def _grid(grid: Optional[Sequence[float]]) -> List[float]:
    g = list(grid) if grid else log_grid(1e-2, 4.0, 40)
    if any(not (h > 0) for h in g):
        raise PfError(Errc.BadArgument, "h grid values must be positive")
    return g


def dense_sweep(entries: Sequence[DenseEntry], a: np.ndarray, grid: Sequence[float], digits: int = DEFAULT_DIGITS):
    """errors[method][grid point] of f(h A / ||A||_2) against the oracle; each method evaluates the
    whole grid in one batched GPU call."""
    scale = max(two_norm_est(a), 1e-300)
    Bs = np.stack([a * (h / scale) for h in grid])
    dB = _dev(Bs)
    vals = []
    for e in entries:
        out = e.evaluate(dB)
        vals.append(out.cpu().numpy() if hasattr(out, "cpu") else np.asarray(out))
    errs = [[0.0] * len(grid) for _ in entries]
    for gi in range(len(grid)):
        for fn in ("exp", "phi1"):
            idx = [mi for mi, e in enumerate(entries) if e.function == fn]
            if not idx:
                continue
            res = dense_errors(fn, Bs[gi], [vals[mi][gi] for mi in idx], digits)
            for mi, r in zip(idx, res):
                errs[mi][gi] = r
    return errs


def cmd_bench_dense(methods: Sequence[str], matrix: MatrixSpec = MatrixSpec(), grid: Optional[Sequence[float]] = None,
                    digits: int = DEFAULT_DIGITS) -> str:
    """cmd_bench_dense (cli.cpp:290-335)."""
    if not methods:
        raise PfError(Errc.BadArgument, "no methods given")
    if digits < 30:
        raise PfError(Errc.BadArgument, "oracle digits must be >= 30")
    g = _grid(grid)
    entries = [dense_entry(t) for t in methods]
    for e in entries:
        if e.function not in ("exp", "phi1"):
            raise PfError(Errc.BadArgument, "no dense oracle for function " + e.function)
    errs = dense_sweep(entries, make_dense_matrix(matrix), g, digits)
    rows = [(e.token, g[gi], errs[mi][gi], e.serial_cost, e.parallel_cost)
            for mi, e in enumerate(entries) for gi in range(len(g))]
    return _render("product_eq", rows)


def action_sweep(entries: Sequence[ActionEntry], d: int, seed: int, grid: Sequence[float],
                 digits: int = DEFAULT_DIGITS):
    sub, diag, sup = trid121(d)
    scale = max(two_norm_est_tridiag(sub, diag, sup), 1e-300)
    v = random_unit_vector(d, seed)
    errs = [[0.0] * len(grid) for _ in entries]
    for gi, hn in enumerate(grid):
        h = hn / scale
        s, dg, u = sub * h, diag * h, sup * h
        vals = [np.asarray(e.evaluate(s, dg, u, v.reshape(-1, 1))).reshape(-1) for e in entries]
        for mi, r in enumerate(action_errors(s, dg, u, v, vals, digits)):
            errs[mi][gi] = r
    return errs


def cmd_bench_action(methods: Sequence[str], matrix: MatrixSpec = MatrixSpec("trid121", 1000, 1),
                     grid: Optional[Sequence[float]] = None, digits: int = DEFAULT_DIGITS) -> str:
    """cmd_bench_action (cli.cpp:337-374)."""
    if not methods:
        raise PfError(Errc.BadArgument, "no methods given")
    if digits < 30:
        raise PfError(Errc.BadArgument, "oracle digits must be >= 30")
    if matrix.kind != "trid121":
        raise PfError(Errc.BadArgument, "action benchmarks need a tridiagonal matrix kind (trid121)")
    g = _grid(grid)
    entries = [action_entry(t) for t in methods]
    errs = action_sweep(entries, matrix.dim, matrix.seed, g, digits)
    rows = [(e.token, g[gi], errs[mi][gi], e.serial_cost, e.parallel_cost)
            for mi, e in enumerate(entries) for gi in range(len(g))]
    return _render("matvec_eq", rows)


def cmd_theta(methods: Sequence[str], tols: Sequence[float] = (), eps_grid: Sequence[float] = ()) -> str:
    """cmd_theta (cli.cpp:136-167) for catalog methods and taylorN."""
    if not methods:
        raise PfError(Errc.BadArgument, "no methods given")

    def profile(token):
        if token.startswith("taylor"):
            return M._Profile(None, M.FunctionId.exp(), int(token[6:]) + 1)
        m = M.catalog(token)
        return M._Profile(m, m.function, m.order + 1)

    out = []
    if eps_grid:
        out.append("method,x,epsilon")
        for t in methods:
            p = profile(t)
            hi = p.domain_limit()
            for x in eps_grid:
                if hi is not None and x >= float(hi):
                    continue
                out.append("%s,%s,%s" % (t, format_sig17(x), format_sig17(p.bound(x))))
        return "\n".join(out) + "\n"
    if not tols:
        raise PfError(Errc.BadArgument, "no tolerances given")
    out.append("method,tol,theta,theta_3dp,saturated")
    for t in methods:
        p = profile(t)
        for tol in tols:
            th = p.theta(tol)
            out.append("%s,%s,%s,%.3f,%d" % (t, exact_decimal_string(float(tol)), format_sig17(th), th,
                                             int(th >= p.domain_hi())))
    return "\n".join(out) + "\n"


# ------------------------------------------------------------------------------ acceptance trends


def _median(v: Sequence[float]) -> float:
    s = sorted(v)
    return s[len(s) // 2]


def figure_trends(d: int = 100, action_d: int = 1000, digits: int = DEFAULT_DIGITS) -> List[Tuple[bool, str]]:
    """figure_trends (acceptance_main.cpp:176-252): R4 <= pade4 and R8 <= taylor8 on >= 90% of the
    dominance window, R10star's round-off plateau >= 10x R10's, and the action's plain-form plateau
    >= 10x the residual form's."""
    a = make_dense_matrix(MatrixSpec("randn", d, 1))
    window = log_grid(0.3, 3.0, 12)
    low = log_grid(0.01, 0.2, 8)
    names = ["R4", "pade4", "R8", "taylor8", "R10star", "R10"]
    entries = [dense_entry(n) for n in names]
    rw = dense_sweep(entries, a, window, digits)
    r4_wins = sum(rw[0][g] <= rw[1][g] for g in range(len(window)))
    r8_wins = sum(rw[2][g] <= rw[3][g] for g in range(len(window)))
    res = [(r4_wins * 10 >= 12 * 9, "R4 <= pade4 on %d/12 grid points" % r4_wins),
           (r8_wins * 10 >= 12 * 9, "R8 <= taylor8 on %d/12 grid points" % r8_wins)]
    rl = dense_sweep(entries, a, low, digits)
    star, r10 = _median(rl[4]), _median(rl[5])
    res.append((star >= 10 * r10, "dense round-off plateaus: R10star %s vs R10 %s" % (format_sig17(star),
                                                                                    format_sig17(r10))))
    ae = [action_entry("R10"), action_entry("R10:residual")]
    errs = action_sweep(ae, action_d, 1, low, digits)
    p_plain, p_res = _median(errs[0]), _median(errs[1])
    res.append((p_plain >= 10 * p_res, "action round-off plateaus: plain %s vs residual %s" % (
        format_sig17(p_plain), format_sig17(p_res))))
    return res


def bound_compliance(d: int = 50, digits: int = DEFAULT_DIGITS, tol: float = 2.0 ** -24) -> List[Tuple[bool, str]]:
    """bound_compliance (acceptance_main.cpp:150-174): every catalog method at its theta(2^-24)
    stays within 10 x 2^-24 on 20 random matrices scaled up to theta."""
    import torch

    from . import api

    out = []
    for name in M.catalog_names():
        m = M.catalog(name)
        th = M.theta(m, m.function, tol)
        Bs = []
        for j in range(20):
            b = W.randn_matrix(d, 1000 + j)
            Bs.append(b * (th * (j + 1) / 20.0 / W.one_norm(b)))
        Bs = np.stack(Bs)
        vals = api.eval_dense(m, torch.from_numpy(Bs).cuda()).cpu().numpy()
        fn = _function_name(m.function)
        errs = [dense_errors(fn, Bs[j], [vals[j]], digits)[0] for j in range(20)]
        bad = sum(e > 10 * tol for e in errs)
        out.append((bad == 0, "%s exceeded 10*2^-24 on %d/20 matrices (worst %s)" % (name, bad,
                                                                                      format_sig17(max(errs)))))
    return out


# ------------------------------------------------------------------------------------------- CLI


def _floats(s: Optional[str]) -> List[float]:
    return [float(x) for x in s.split(",")] if s else []


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2210_03714_b200.drivers")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("bench-dense", "bench-action"):
        p = sub.add_parser(name)
        p.add_argument("--methods", required=True)
        p.add_argument("--kind", default="randn" if name == "bench-dense" else "trid121")
        p.add_argument("--dim", type=int, default=50 if name == "bench-dense" else 1000)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--grid", default=None, help="comma-separated h_norm values (default 40 log points in [1e-2, 4])")
        p.add_argument("--digits", type=int, default=DEFAULT_DIGITS)
    p = sub.add_parser("theta")
    p.add_argument("--methods", required=True)
    p.add_argument("--tols", default=None)
    p.add_argument("--eps-grid", default=None)
    sub.add_parser("acceptance")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "bench-dense":
            sys.stdout.write(cmd_bench_dense(args.methods.split(","), MatrixSpec(args.kind, args.dim, args.seed),
                                             _floats(args.grid), args.digits))
        elif args.cmd == "bench-action":
            sys.stdout.write(cmd_bench_action(args.methods.split(","), MatrixSpec(args.kind, args.dim, args.seed),
                                              _floats(args.grid), args.digits))
        elif args.cmd == "theta":
            sys.stdout.write(cmd_theta(args.methods.split(","), _floats(args.tols), _floats(args.eps_grid)))
        else:
            ok = True
            for passed, msg in bound_compliance() + figure_trends():
                ok = ok and passed
                print(("PASS " if passed else "FAIL ") + msg)
            return 0 if ok else 1
    except PfError as e:
        sys.stderr.write("error: %s\n" % e)
        return 3 if e.code not in (Errc.BadArgument,) else 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
