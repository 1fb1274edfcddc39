"""Exact partial-fraction method tables and theta thresholds (host side, no GPU work).

Restates the reference's method model so the kernels receive exactly the
doubles the reference would hand them:

* series coefficients a_k            -- proj/core/src/series.cpp:64-84
* moment system sum_i b_i c_i^k = a_k -- proj/core/src/methods.cpp:33-57, 95-111
* plain / hybrid builders            -- proj/core/src/methods.cpp:121-186
* frac4 / frac8 shift templates      -- proj/core/src/methods.cpp:213-231
* catalog entries                    -- proj/core/src/methods.cpp:298-369
* constant term a_0 = d_0 + sum b_i  -- proj/core/src/methods.cpp:75-80
* to_double_nearest (ties to even)   -- proj/core/src/rational.cpp:66-88
  (``float(Fraction)`` is correctly rounded with ties to even, identical doubles)
* forward bound / theta bisection    -- proj/core/src/bounds.cpp:97-201

GMP is replaced by ``fractions.Fraction`` (exact) and ``mpmath`` at 256 bits
(the reference's kSumPrecBits, bounds.cpp:16).

New derived weight sets the reference does not ship:
phi_1 weights on the R8 / R4 shifts (build_plain on the same shifts with
FunctionId::phi(1)), and the cos/sin real-pair sets obtained by merging the
complex-conjugate shifts +-i c of exp(iB).
"""
from __future__ import annotations

import functools
import math
import threading
from dataclasses import dataclass, field, replace
from fractions import Fraction
from typing import Dict, List, Optional, Sequence

from .errors import Errc, PfError, raise_error

# --------------------------------------------------------------------------------------
# series (series.cpp:64-84)
# --------------------------------------------------------------------------------------


@dataclass(frozen=True)
class FunctionId:
    tag: str  # "exp" | "phi" | "log1m" | "cos" | "sin"
    phi_order: int = 0

    @staticmethod
    def exp() -> "FunctionId":
        return FunctionId("exp")

    @staticmethod
    def phi(m: int) -> "FunctionId":
        return FunctionId("phi", m)

    @staticmethod
    def log_one_minus() -> "FunctionId":
        return FunctionId("log1m")

    @staticmethod
    def cosine() -> "FunctionId":
        return FunctionId("cos")

    @staticmethod
    def sine() -> "FunctionId":
        return FunctionId("sin")

    def name(self) -> str:
        return "phi%d" % self.phi_order if self.tag == "phi" else self.tag

    @staticmethod
    def parse(name: str) -> "FunctionId":
        """Inverse of name(); "phi" means phi1 and phi0 is exp (series.cpp:27-46)."""
        fixed = {"exp": FunctionId.exp(), "log1m": FunctionId.log_one_minus(), "cos": FunctionId.cosine(),
                 "sin": FunctionId.sine(), "phi": FunctionId.phi(1)}
        if name in fixed:
            return fixed[name]
        if name.startswith("phi") and len(name) > 3 and name[3:].isdigit():
            m = int(name[3:])
            return FunctionId.exp() if m == 0 else FunctionId.phi(m)
        raise_error(Errc.BadArgument, "unknown function: " + name)


@functools.lru_cache(maxsize=None)
def _factorial(k: int) -> int:
    return math.factorial(k)


def series_coeff(fn: FunctionId, k: int) -> Fraction:
    """a_k of the target function (series.cpp:64-84)."""
    if k < 0:
        raise_error(Errc.BadArgument, "negative series index")
    if fn.tag == "exp":
        return Fraction(1, _factorial(k))
    if fn.tag == "phi":
        return Fraction(1, _factorial(k + fn.phi_order))
    if fn.tag == "log1m":
        return Fraction(0) if k == 0 else Fraction(-1, k)
    if fn.tag == "cos":
        if k % 2:
            return Fraction(0)
        r = Fraction(1, _factorial(k))
        return r if (k // 2) % 2 == 0 else -r
    if fn.tag == "sin":
        if k % 2 == 0:
            return Fraction(0)
        r = Fraction(1, _factorial(k))
        return r if ((k - 1) // 2) % 2 == 0 else -r
    raise_error(Errc.BadArgument, "bad function tag")


def series_tail_bound(fn: FunctionId, K: int, x: Fraction) -> Fraction:
    """Analytic remainder sum_{k>K} |a_k| x^k majorant (series.cpp:142-167)."""
    if x < 0:
        raise_error(Errc.BadArgument, "tail bound needs x >= 0")
    if fn.tag in ("exp", "phi", "cos", "sin"):
        m = fn.phi_order if fn.tag == "phi" else 0
        ratio = x / (K + m + 2)
        if ratio >= 1:
            raise_error(Errc.OutOfConvergenceRadius, "tail bound needs K + 2 > x")
        lead = x ** (K + 1)
        return lead / _factorial(K + 1 + m) / (1 - ratio)
    if fn.tag == "log1m":
        if x >= 1:
            raise_error(Errc.OutOfConvergenceRadius, "log(1-x) series needs x < 1")
        return x ** (K + 1) / (K + 1) / (1 - x)
    raise_error(Errc.BadArgument, "bad function tag")


def series_radius(fn: FunctionId) -> Optional[Fraction]:
    return Fraction(1) if fn.tag == "log1m" else None


# --------------------------------------------------------------------------------------
# rational helpers (rational.cpp)
# --------------------------------------------------------------------------------------


def to_double_nearest(q: Fraction) -> float:
    """Nearest double, ties to even (rational.cpp:66-88). Fraction.__float__ is
    correctly rounded (integer true division), which gives the same double."""
    return float(Fraction(q))


def rational_from_string(s: str) -> Fraction:
    s = s.strip()
    try:
        return Fraction(s)
    except (ValueError, ZeroDivisionError):
        raise_error(Errc.BadArgument, "malformed rational literal: " + s)


def to_fraction_string(q: Fraction) -> str:
    q = Fraction(q)
    return str(q.numerator) if q.denominator == 1 else "%d/%d" % (q.numerator, q.denominator)


def format_sig17(x: float) -> str:
    return "%.17g" % x


# --------------------------------------------------------------------------------------
# method model (methods.hpp:23-48, methods.cpp)
# --------------------------------------------------------------------------------------

PLAIN = 0
RESIDUAL = 1


@dataclass
class FractionMethod:
    """r(x) = d_0 + d_1 x + d_2 x^2 + sum_i b_i / (1 - c_i x)  (methods.hpp:20-48)."""

    name: str
    function: FunctionId
    shifts: List[Fraction]
    weights: List[Fraction]
    poly: List[Fraction] = field(default_factory=list)
    order: int = 0
    form: int = PLAIN
    notes: List[str] = field(default_factory=list)

    def processors(self) -> int:
        return sum(1 for c in self.shifts if c != 0)

    def taylor_coeff(self, k: int) -> Fraction:
        acc = self.poly[k] if k < len(self.poly) else Fraction(0)
        for c, b in zip(self.shifts, self.weights):
            acc += b * (Fraction(1) if k == 0 else c ** k)
        return acc

    def constant_term(self) -> Fraction:
        return self.taylor_coeff(0)

    def max_coefficient(self) -> Fraction:
        return max([abs(b) for b in self.weights] + [abs(d) for d in self.poly] + [Fraction(0)])

    def max_abs_shift(self) -> Fraction:
        return max([abs(c) for c in self.shifts] + [Fraction(0)])

    # doubles exactly as eval_dense converts them (dense.cpp:203-204, 247-249)
    def shift_doubles(self) -> List[float]:
        return [to_double_nearest(c) for c in self.shifts]

    def weight_doubles(self) -> List[float]:
        return [to_double_nearest(b) for b in self.weights]


def _solve_linear(M: List[List[Fraction]], rhs: List[Fraction]) -> List[Fraction]:
    """Exact Gaussian elimination with partial pivoting on magnitude (methods.cpp:33-57)."""
    n = len(rhs)
    M = [row[:] for row in M]
    rhs = rhs[:]
    for col in range(n):
        piv = col
        for r in range(col + 1, n):
            if abs(M[r][col]) > abs(M[piv][col]):
                piv = r
        if M[piv][col] == 0:
            raise_error(Errc.DuplicateShift, "singular moment system")
        M[piv], M[col] = M[col], M[piv]
        rhs[piv], rhs[col] = rhs[col], rhs[piv]
        for r in range(col + 1, n):
            if M[r][col] == 0:
                continue
            f = M[r][col] / M[col][col]
            for j in range(col, n):
                M[r][j] -= f * M[col][j]
            rhs[r] -= f * rhs[col]
    x = [Fraction(0)] * n
    for i in range(n - 1, -1, -1):
        acc = rhs[i]
        for j in range(i + 1, n):
            acc -= M[i][j] * x[j]
        x[i] = acc / M[i][i]
    return x


def _shift_power(c: Fraction, k: int) -> Fraction:
    return Fraction(1) if k == 0 else c ** k


def _check_distinct(shifts: Sequence[Fraction]) -> None:
    for i in range(len(shifts)):
        for j in range(i + 1, len(shifts)):
            if shifts[i] == shifts[j]:
                raise_error(Errc.DuplicateShift, "duplicate shift c = %s at positions %d and %d"
                            % (to_fraction_string(shifts[i]), i + 1, j + 1))


def solve_weights(shifts: Sequence[Fraction], fn: FunctionId, order: int) -> List[Fraction]:
    """Moment system sum_i b_i c_i^k = a_k, k = 0..order (methods.cpp:95-111)."""
    if order < 0:
        raise_error(Errc.BadArgument, "order must be >= 0")
    if len(shifts) != order + 1:
        raise_error(Errc.LengthMismatch, "need order + 1 = %d shifts, got %d" % (order + 1, len(shifts)))
    shifts = [Fraction(c) for c in shifts]
    _check_distinct(shifts)
    n = len(shifts)
    M = [[_shift_power(shifts[i], k) for i in range(n)] for k in range(n)]
    rhs = [series_coeff(fn, k) for k in range(n)]
    return _solve_linear(M, rhs)


def verify_sum_rules(m: FractionMethod) -> None:
    for k in range(m.order + 1):
        if m.taylor_coeff(k) != series_coeff(m.function, k):
            raise_error(Errc.LengthMismatch, "sum rule violated at k = %d for method %s" % (k, m.name))


def build_plain(shifts: Sequence[Fraction], fn: FunctionId, order: int, name: str) -> FractionMethod:
    """methods.cpp:121-131."""
    shifts = [Fraction(c) for c in shifts]
    m = FractionMethod(name=name, function=fn, shifts=shifts,
                       weights=solve_weights(shifts, fn, order), order=order)
    verify_sum_rules(m)
    return m


def build_hybrid(shifts: Sequence[Fraction], free_weights: Dict[int, Fraction], fn: FunctionId,
                 order: int, name: str) -> FractionMethod:
    """methods.cpp:133-186: constrained b_i from k = 3..order, then d_0..d_2."""
    shifts = [Fraction(c) for c in shifts]
    _check_distinct(shifts)
    if any(c == 0 for c in shifts):
        raise_error(Errc.BadArgument, "hybrid methods need nonzero shifts")
    for idx in free_weights:
        if idx < 1 or idx > len(shifts):
            raise_error(Errc.UnderDetermined, "free weight index %d out of range" % idx)
    n_con = len(shifts) - len(free_weights)
    if n_con != order - 2:
        raise_error(Errc.UnderDetermined, "hybrid system needs order - 2 = %d constrained weights, got %d"
                    % (order - 2, n_con))
    constrained = [i for i in range(len(shifts)) if (i + 1) not in free_weights]
    M, rhs = [], []
    for row in range(len(constrained)):
        k = 3 + row
        r = series_coeff(fn, k)
        for idx, val in sorted(free_weights.items()):
            r -= Fraction(val) * _shift_power(shifts[idx - 1], k)
        rhs.append(r)
        M.append([_shift_power(shifts[j], k) for j in constrained])
    solved = _solve_linear(M, rhs)
    weights = [Fraction(0)] * len(shifts)
    for idx, val in free_weights.items():
        weights[idx - 1] = Fraction(val)
    for j, i in enumerate(constrained):
        weights[i] = solved[j]
    poly = []
    for k in range(3):
        acc = series_coeff(fn, k)
        for c, b in zip(shifts, weights):
            acc -= b * _shift_power(c, k)
        poly.append(acc)
    m = FractionMethod(name=name, function=fn, shifts=shifts, weights=weights, poly=poly, order=order)
    verify_sum_rules(m)
    return m


def to_residual_form(m: FractionMethod) -> FractionMethod:
    return replace(m, form=RESIDUAL)


def to_plain_form(m: FractionMethod) -> FractionMethod:
    return replace(m, form=PLAIN)


def frac4_shifts(a: Fraction) -> List[Fraction]:
    """(0, 1/a, -1/a, 1/(2a), -1/(2a)) -- methods.cpp:213-220."""
    a = Fraction(a)
    return [Fraction(0), 1 / a, -1 / a, 1 / (2 * a), -1 / (2 * a)]


def frac8_shifts(a: Fraction) -> List[Fraction]:
    """methods.cpp:222-231."""
    a = Fraction(a)
    return [Fraction(0), 1 / a, -1 / a, 2 / (3 * a), -2 / (3 * a), 1 / (2 * a), -1 / (2 * a),
            2 / (5 * a), -2 / (5 * a)]


def _rats(texts):
    return [rational_from_string(t) for t in texts]


def _cross_check(m: FractionMethod, weights: Sequence[str], poly: Sequence[str] = ()) -> None:
    """methods.cpp:279-290: published constants vs recomputed; recomputed wins."""
    for i, t in enumerate(weights):
        if i < len(m.weights) and m.weights[i] != rational_from_string(t):
            m.notes.append("published b%d = %s differs from recomputed %s; recomputed value is used"
                           % (i + 1, t, to_fraction_string(m.weights[i])))
    for k, t in enumerate(poly):
        if k < len(m.poly) and m.poly[k] != rational_from_string(t):
            m.notes.append("published d%d = %s differs from recomputed %s; recomputed value is used"
                           % (k, t, to_fraction_string(m.poly[k])))


def _make_catalog_entry(name: str) -> FractionMethod:
    """methods.cpp:298-357."""
    if name == "R4":
        m = build_plain(frac4_shifts(5), FunctionId.exp(), 4, "R4")
        _cross_check(m, ["128/3", "85/3", "20/9", "-515/9", "-15"])
        return m
    if name == "R4_phi1":
        m = build_plain(frac4_shifts(6), FunctionId.phi(1), 4, "R4_phi1")
        _cross_check(m, ["71/5", "117/10", "7/10", "-104/5", "-24/5"])
        return m
    if name == "R5":
        m = build_plain(_rats(["0", "1/3", "1/4", "1/5", "1/6", "1/7"]), FunctionId.exp(), 5, "R5")
        _cross_check(m, ["-43/12", "81/32", "-704/9", "23125/48", "-810", "117649/288"])
        return m
    if name == "R8":
        m = build_plain(frac8_shifts(5), FunctionId.exp(), 8, "R8")
        _cross_check(m, ["-9979069/32256", "-1995521/254016", "-392009/254016", "520866369/802816",
                         "48898161/802816", "-26686735/11907", "-3892615/11907",
                         "353067578125/195084288", "71873828125/195084288"])
        return m
    if name == "R10star":
        shifts = [Fraction(1, 6 + i) for i in range(1, 11)]
        m = build_hybrid(shifts, {9: Fraction(-50000), 10: Fraction(350000)}, FunctionId.exp(), 10, "R10star")
        _cross_check(m, ["-2385751622325187262153/1585084524134400000", "3752603696192081/82668600000",
                         "-87230538798639033213/187904819200000", "14789110319838821875/6934744793088",
                         "-10558563753676365149296981/2219118333788160000", "3520134037769971/716800000",
                         "-2263057299714115181019509/1585084524134400000",
                         "-2275831141003773874927/3095868211200000"],
                     ["-34244933704346617/14676708556800", "-18541933026870559/428070666240000",
                      "-6798371473106351/15410543984640000"])
        return m
    if name == "R10":
        shifts = []
        for i in range(1, 6):
            shifts += [Fraction(-1, 6 + 2 * i), Fraction(1, 6 + 2 * i)]
        m = build_hybrid(shifts, {9: Fraction(2000), 10: Fraction(-3500)}, FunctionId.exp(), 10, "R10")
        _cross_check(m, ["-57383239/760320", "-115498838729/239500800", "1648441938671875/1255673954304",
                         "56790060546875/4227858432", "-1476772203681/298188800",
                         "-31012455666807/656015360", "4891212112962371/1295536619520",
                         "171190903245297593/3886609858560"],
                     ["-781562376863/94371840", "-54849495983/330301440", "-8034429391/587202560"])
        return m
    raise_error(Errc.UnknownMethod, "unknown catalog method: " + name)


_catalog_lock = threading.Lock()
_catalog_cache: Dict[str, FractionMethod] = {}


def catalog(name: str) -> FractionMethod:
    """Process-lifetime cache guarded by a mutex (methods.cpp:361-369)."""
    with _catalog_lock:
        if name not in _catalog_cache:
            _catalog_cache[name] = _make_catalog_entry(name)
        return _catalog_cache[name]


def catalog_names() -> List[str]:
    return ["R4", "R4_phi1", "R5", "R8", "R10star", "R10"]


def taylor_expansion_of_method(m: FractionMethod, k_max: int) -> List[Fraction]:
    return [m.taylor_coeff(k) for k in range(k_max + 1)]


# --------------------------------------------------------------------------------------
# derived weight sets (Appendix A)
# --------------------------------------------------------------------------------------


def same_shift_method(base: FractionMethod, fn: FunctionId, name: Optional[str] = None) -> FractionMethod:
    """Weights for another function on the SAME shifts (build_plain on base.shifts);
    one LU per shift then feeds both weight sets."""
    if base.poly:
        raise_error(Errc.BadArgument, "same-shift weight sets need a pure fraction method")
    return build_plain(base.shifts, fn, base.order, name or "%s_%s" % (base.name, fn.name()))


@dataclass
class PairMethod:
    """cos/sin of B from exp(iB) with the conjugate shifts +-c merged into one real solve
    Y_c = (I + c^2 B^2)^{-1} (residual form: Z_c = Y_c c^2 B^2):
        cos B = a0 I - sum_c cw_c Z_c,   sin B = B (a1 I - sum_c sw_c Z_c)
    cw_c = b_c + b_{-c}, sw_c = c (b_c - b_{-c}); the zero shift adds b_0 to cos only."""

    name: str
    c2: List[Fraction]
    cw: List[Fraction]
    sw: List[Fraction]
    a0: Fraction
    a1: Fraction
    b0: Fraction


def pair_method(base: FractionMethod) -> PairMethod:
    shifts = list(base.shifts)
    w = dict(zip(shifts, base.weights))
    if base.poly:
        raise_error(Errc.BadArgument, "pair methods need a pure fraction method")
    seen = set()
    c2, cw, sw = [], [], []
    b0 = Fraction(0)
    for c in shifts:
        if c == 0:
            b0 = w[c]
            continue
        if abs(c) in seen:
            continue
        if -c not in w:
            raise_error(Errc.BadArgument, "pair methods need shifts symmetric about 0")
        seen.add(abs(c))
        cp = abs(c)
        c2.append(cp * cp)
        cw.append(w[cp] + w[-cp])
        sw.append(cp * (w[cp] - w[-cp]))
    order = sorted(range(len(c2)), key=lambda i: c2[i])
    c2 = [c2[i] for i in order]
    cw = [cw[i] for i in order]
    sw = [sw[i] for i in order]
    a0 = b0 + sum(cw, Fraction(0))
    a1 = sum(sw, Fraction(0))
    return PairMethod(name=base.name + "_cossin", c2=c2, cw=cw, sw=sw, a0=a0, a1=a1, b0=b0)


# --------------------------------------------------------------------------------------
# forward bound and theta (bounds.cpp:97-201)
# --------------------------------------------------------------------------------------

_K_MAX_TERMS = 1500
_DOMAIN_CAP = 500.0


class _Profile:
    def __init__(self, method: Optional[FractionMethod], fn: FunctionId, first_error_order: int):
        import mpmath

        self.mp = mpmath.mp.clone() if hasattr(mpmath.mp, "clone") else mpmath.mp
        self.method = method
        self.fn = fn
        self.s1 = first_error_order
        self._err: List[Fraction] = []  # |a_k - alpha_k| exact, k >= s1
        self._thetas: Dict[float, float] = {}

    def _err_coeff(self, idx: int) -> Fraction:
        while len(self._err) <= idx:
            k = self.s1 + len(self._err)
            alpha = self.method.taylor_coeff(k) if self.method is not None else Fraction(0)
            self._err.append(abs(series_coeff(self.fn, k) - alpha))
        return self._err[idx]

    def domain_limit(self) -> Optional[Fraction]:
        limit = None
        if self.method is not None:
            cmax = self.method.max_abs_shift()
            if cmax > 0:
                limit = 1 / cmax
        r = series_radius(self.fn)
        if r is not None and (limit is None or r < limit):
            limit = r
        return limit

    def bound(self, x: float) -> float:
        import mpmath

        if x < 0:
            raise_error(Errc.BadArgument, "forward bound needs x >= 0")
        if x == 0:
            return 0.0
        xq = Fraction(x)
        lim = self.domain_limit()
        if lim is not None and xq >= lim:
            raise_error(Errc.OutOfConvergenceRadius, "x = %r outside convergence domain" % x)
        with mpmath.workprec(256):
            s = mpmath.mpf(0)
            xf = mpmath.mpf(x)
            xpow = mpmath.mpf(xq.numerator) ** self.s1 / mpmath.mpf(xq.denominator) ** self.s1
            m_extra = self.fn.phi_order if self.fn.tag == "phi" else 0
            cutoff = mpmath.mpf("1e-40")
            k = self.s1
            while k < self.s1 + _K_MAX_TERMS:
                e = self._err_coeff(k - self.s1)
                term = mpmath.mpf(e.numerator) / e.denominator * xpow
                s += term
                if term != 0 and term < s * cutoff and k >= self.s1 + 4 and Fraction(k + m_extra) >= 2 * xq:
                    break
                xpow *= xf
                k += 1
            K = min(k, self.s1 + _K_MAX_TERMS - 1)
            tail = mpmath.mpf(0)
            if self.method is not None:
                for c, b in zip(self.method.shifts, self.method.weights):
                    if c == 0:
                        continue
                    cx = abs(c) * xq
                    cxf = mpmath.mpf(cx.numerator) / cx.denominator
                    tail += abs(mpmath.mpf(b.numerator) / b.denominator) * cxf ** (K + 1) / (1 - cxf)
            st = series_tail_bound(self.fn, K, xq)
            tail += mpmath.mpf(st.numerator) / st.denominator
            s += tail
            s *= 1 + mpmath.mpf("1e-25")
            out = float(s)
        return math.nextafter(out, math.inf)

    def domain_hi(self) -> float:
        lim = self.domain_limit()
        if lim is None:
            return _DOMAIN_CAP
        return min(_DOMAIN_CAP, to_double_nearest(lim) * (1 - 1e-9))

    def theta(self, tol: float) -> float:
        if tol <= 0:
            raise_error(Errc.BadArgument, "tolerance must be positive")
        if tol in self._thetas:
            return self._thetas[tol]
        hi = self.domain_hi()
        if self.bound(hi) <= tol:
            res = hi
        else:
            lo = 0.0
            for _ in range(200):
                mid = 0.5 * (lo + hi) if lo > 0 else hi / 2
                if self.bound(mid) <= tol:
                    lo = mid
                else:
                    hi = mid
                if lo > 0 and (hi - lo) <= 1e-6 * lo and self.bound(lo) >= tol * (1 - 1e-4):
                    break
            res = lo
        self._thetas[tol] = res
        return res


def forward_bound(m: FractionMethod, fn: FunctionId, x: float) -> float:
    return _Profile(m, fn, m.order + 1).bound(x)


def theta(m: FractionMethod, fn: Optional[FunctionId] = None, tol: float = 2.0 ** -53) -> float:
    """theta_m(tol): largest x with forward_bound(x) <= tol (bounds.cpp:175-201, 252-254)."""
    return _Profile(m, fn or m.function, m.order + 1).theta(tol)


def theta_taylor(degree: int, tol: float) -> float:
    if degree < 1:
        raise_error(Errc.BadArgument, "taylor degree must be >= 1")
    return _Profile(None, FunctionId.exp(), degree + 1).theta(tol)


# theta at u = 2^-53, regenerated by tools/gen_tables.py with the restated bound above and
# pinned by tests/test_methods.py (recomputation must reproduce every digit).
THETA_U53 = {
    "R4": 0.003078503065458018,
    "R4_phi1": 0.004910895596004059,
    "R5": 0.010800484557080145,
    "R8": 0.0973103939513804,
    "R10star": 0.31575259534731814,
    "R10": 0.2238531110432368,
    "R4_phi1set": 0.0029524299286583923,
    "R8_phi1set": 0.09290628125913689,
}


def squarings_for(norm1: float, theta_value: float) -> int:
    """j = smallest j >= 0 with ldexp(norm, -j) <= theta (exact; equals
    max(0, ceil(log2(norm/theta))) without libm rounding)."""
    if not (norm1 == norm1) or norm1 == math.inf:
        raise_error(Errc.BadArgument, "matrix norm is not finite")
    j = 0
    while math.ldexp(norm1, -j) > theta_value:
        j += 1
    return j


def substeps_for(norm1: float, theta_value: float) -> int:
    """N = ceil(norm/theta), at least 1 (action.cpp:398)."""
    if norm1 <= theta_value:
        return 1
    return int(math.ceil(norm1 / theta_value))
