"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of the CPU oracle (oracle/pf_oracle.c).

Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs as the
checker and the CPU baseline -- never by the product path. See pf_oracle.h for what it restates.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
_SO = HERE / "libpforacle.so"


class Status(C.Structure):
    _fields_ = [("code", C.c_int), ("batch_index", C.c_int), ("shift_index", C.c_int), ("column", C.c_int),
                ("pivot_magnitude", C.c_double), ("scale", C.c_double)]


DP = C.POINTER(C.c_double)


class Method(C.Structure):
    _fields_ = [("n_terms", C.c_int), ("shifts", DP), ("n_sets", C.c_int), ("weights", DP), ("has_poly", C.c_int),
                ("poly", DP), ("constant", DP), ("form", C.c_int)]


class PairMethod(C.Structure):
    _fields_ = [("n_pairs", C.c_int), ("c2", DP), ("cw", DP), ("sw", DP), ("a0", C.c_double), ("a1", C.c_double)]


class OracleError(RuntimeError):
    def __init__(self, st: Status):
        super().__init__("oracle error code %d (shift %d, column %d, pivot %r, scale %r, batch %d)" % (
            st.code, st.shift_index, st.column, st.pivot_magnitude, st.scale, st.batch_index))
        self.status = st
        self.code = st.code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            os.system("make -s -C %s" % HERE)
        _lib = C.CDLL(str(_SO))
        _lib.pfo_one_norm.restype = C.c_double
        _lib.pfo_max_abs.restype = C.c_double
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class OMethod:
    """Packs doubles for pfo_method: shifts, weight sets (rows), poly (3 per set), constants."""

    def __init__(self, shifts: Sequence[float], weights: Sequence[Sequence[float]], poly=None, constants=None,
                 form: int = 1):
        self.shifts = _f64(shifts)
        w = _f64(weights).reshape(len(weights), len(shifts))
        self.weights = np.ascontiguousarray(w)
        self.n_sets = w.shape[0]
        self.poly = _f64(poly).reshape(self.n_sets, 3) if poly is not None else np.zeros((self.n_sets, 3))
        self.constants = _f64(constants) if constants is not None else np.zeros(self.n_sets)
        self.c = Method(len(self.shifts), self.shifts.ctypes.data_as(DP), self.n_sets,
                        self.weights.ctypes.data_as(DP), 1 if poly is not None else 0,
                        self.poly.ctypes.data_as(DP), self.constants.ctypes.data_as(DP), int(form))

    @staticmethod
    def from_method(method, form: Optional[int] = None, extra=()):
        from paper_2210_03714_b200.methods import to_double_nearest

        form = method.form if form is None else form
        sets = [method] + list(extra)
        has_poly = any(len(s.poly) == 3 for s in sets)
        poly = None
        if has_poly:
            poly = [[to_double_nearest(d) for d in s.poly] if len(s.poly) == 3 else [0.0] * 3 for s in sets]
        return OMethod(method.shift_doubles(), [s.weight_doubles() for s in sets], poly,
                       [to_double_nearest(s.constant_term()) for s in sets], form)


def _check(rc, st):
    if rc:
        raise OracleError(st)


def one_norm(a) -> float:
    a = _f64(a)
    return lib().pfo_one_norm(a.shape[0], _p(a))


def squarings(norm: float, theta: float) -> int:
    return lib().pfo_squarings(C.c_double(norm), C.c_double(theta))


def mul(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    out = np.empty_like(a)
    lib().pfo_mul(a.shape[0], _p(a), _p(b), _p(out))
    return out


def mul_rows(a_rows, b) -> np.ndarray:
    """rows x n times n x n in pfo_mul's order (row i as in mul(a, b))."""
    a_rows, b = _f64(a_rows), _f64(b)
    out = np.empty((a_rows.shape[0], b.shape[1]))
    lib().pfo_mul_rows(a_rows.shape[0], b.shape[0], _p(a_rows), _p(b), _p(out))
    return out


def phi1_doubling(E, Phi, j: int):
    """pfo_expm_phi1's recurrence: Phi <- 0.5 ((E + I) Phi), E <- E E, j times."""
    E, Phi = _f64(E).copy(), _f64(Phi).copy()
    n = E.shape[0]
    for _ in range(j):
        T = E.copy()
        T[np.arange(n), np.arange(n)] += 1.0
        Phi = mul(T, Phi) * 0.5
        E = mul(E, E)
    return E, Phi


def mul_rect(a, b) -> np.ndarray:
    """(n x n)(n x k), i-k-j order with the zero skip (DenseMatrix::mul generalised)."""
    a, b = _f64(a), _f64(b)
    b2 = b.reshape(b.shape[0], -1)
    out = np.empty_like(b2)
    lib().pfo_mul_rect(a.shape[0], b2.shape[1], _p(a), _p(b2), _p(out))
    return out.reshape(b.shape)


def lu(a, rel_tol: float = 1e-14):
    lu_ = _f64(a).copy()
    n = lu_.shape[0]
    piv = np.zeros(n, dtype=np.int32)
    st = Status()
    rc = lib().pfo_lu(n, _p(lu_), _p(piv), C.c_double(rel_tol), C.byref(st))
    _check(rc, st)
    return lu_, piv


def lu_solve_matrix(lu_, piv, rhs) -> np.ndarray:
    lu_, rhs = _f64(lu_), _f64(rhs)
    out = np.empty_like(rhs)
    k = rhs.shape[1] if rhs.ndim == 2 else 1
    lib().pfo_lu_solve_matrix(lu_.shape[0], k, _p(lu_), _p(np.ascontiguousarray(piv, dtype=np.int32)), _p(rhs),
                              _p(out))
    return out


def solve_shifted(b, c: float) -> np.ndarray:
    b = _f64(b)
    out = np.empty_like(b)
    st = Status()
    rc = lib().pfo_solve_shifted(b.shape[0], _p(b), C.c_double(c), _p(out), C.byref(st))
    _check(rc, st)
    return out


def eval_dense(m: OMethod, b, workers: int = 1) -> np.ndarray:
    """All weight sets: returns (n_sets, n, n) (or (n, n) for one set)."""
    b = _f64(b)
    n = b.shape[0]
    outs = np.empty((m.n_sets, n, n))
    st = Status()
    rc = lib().pfo_eval_dense(n, _p(b), C.byref(m.c), workers, _p(outs), C.byref(st))
    _check(rc, st)
    return outs[0] if m.n_sets == 1 else outs


def expm(a, m: OMethod, theta: float, j_fixed: int = -1, workers: int = 1):
    a = _f64(a)
    out = np.empty_like(a)
    j = C.c_int()
    st = Status()
    rc = lib().pfo_expm(a.shape[0], _p(a), C.byref(m.c), C.c_double(theta), j_fixed, workers, _p(out), C.byref(j),
                        C.byref(st))
    _check(rc, st)
    return out, j.value


def expm_batched(a, m: OMethod, theta: float, threads: int = 1):
    a = _f64(a)
    bsz, n = a.shape[0], a.shape[1]
    out = np.empty_like(a)
    js = np.zeros(bsz, dtype=np.int32)
    st = Status()
    rc = lib().pfo_expm_batched(n, bsz, _p(a), C.byref(m.c), C.c_double(theta), threads, _p(out), _p(js),
                                C.byref(st))
    _check(rc, st)
    return out, js


def expm_phi1(a, m: OMethod, theta: float, j_fixed: int = -1, workers: int = 1):
    a = _f64(a)
    oe, op = np.empty_like(a), np.empty_like(a)
    j = C.c_int()
    st = Status()
    rc = lib().pfo_expm_phi1(a.shape[0], _p(a), C.byref(m.c), C.c_double(theta), j_fixed, workers, _p(oe), _p(op),
                             C.byref(j), C.byref(st))
    _check(rc, st)
    return oe, op, j.value


class OPair:
    def __init__(self, c2, cw, sw, a0, a1):
        self.c2, self.cw, self.sw = _f64(c2), _f64(cw), _f64(sw)
        self.c = PairMethod(len(self.c2), self.c2.ctypes.data_as(DP), self.cw.ctypes.data_as(DP),
                            self.sw.ctypes.data_as(DP), a0, a1)

    @staticmethod
    def from_pair(pm):
        from paper_2210_03714_b200.methods import to_double_nearest as d

        return OPair([d(x) for x in pm.c2], [d(x) for x in pm.cw], [d(x) for x in pm.sw], d(pm.a0), d(pm.a1))


def cossin(a, pm: OPair, theta: float, j_fixed: int = -1, workers: int = 1):
    a = _f64(a)
    oc, os_ = np.empty_like(a), np.empty_like(a)
    j = C.c_int()
    st = Status()
    rc = lib().pfo_cossin(a.shape[0], _p(a), C.byref(pm.c), C.c_double(theta), j_fixed, workers, _p(oc), _p(os_),
                          C.byref(j), C.byref(st))
    _check(rc, st)
    return oc, os_, j.value


def cossin_batched(a, pm: OPair, theta: float, threads: int = 1):
    a = _f64(a)
    bsz, n = a.shape[0], a.shape[1]
    oc, os_ = np.empty_like(a), np.empty_like(a)
    js = np.zeros(bsz, dtype=np.int32)
    st = Status()
    rc = lib().pfo_cossin_batched(n, bsz, _p(a), C.byref(pm.c), C.c_double(theta), threads, _p(oc), _p(os_), _p(js),
                                  C.byref(st))
    _check(rc, st)
    return oc, os_, js


def action(a, v, m: OMethod, substeps: int, workers: int = 1) -> np.ndarray:
    a, v = _f64(a), _f64(v)
    n = a.shape[0]
    k = v.shape[1] if v.ndim == 2 else 1
    out = np.empty_like(v)
    st = Status()
    rc = lib().pfo_action(n, k, _p(a), _p(v), C.byref(m.c), substeps, workers, _p(out), C.byref(st))
    _check(rc, st)
    return out


def rel_diff_1norm(a, b) -> float:
    """test_dense.cpp:24-28: ||a - b||_1 / max(||b||_1, 1e-300)."""
    a, b = _f64(a), _f64(b)
    if a.ndim == 3:
        return max(rel_diff_1norm(x, y) for x, y in zip(a, b))
    if a.ndim == 1:
        a, b = a[:, None], b[:, None]
    if a.shape[0] != a.shape[1]:  # rectangular blocks (action, multi-RHS solves): max column sum
        d = np.abs(a - b).sum(axis=0).max()
        return float(d / max(np.abs(b).sum(axis=0).max(), 1e-300))
    return one_norm(a - b) / max(one_norm(b), 1e-300)


# ---- f2: banded action (pf_oracle_band.c, restating proj/core/src/action.cpp)

class BandError(RuntimeError):
    """ZeroPivot from the banded solvers: row (and shift index for the action)."""

    def __init__(self, code: int, row: int, shift_index: int = 0):
        super().__init__("zero pivot at row %d%s" % (row, (" (shift %d)" % shift_index) if shift_index else ""))
        self.code, self.row, self.shift_index = code, row, shift_index


def _cols(x):
    x = _f64(x)
    return (x.reshape(-1, 1), True) if x.ndim == 1 else (x, False)


def tridiag_matvec(sub, diag, sup, v) -> np.ndarray:
    sub, diag, sup = _f64(sub), _f64(diag), _f64(sup)
    V, vec = _cols(v)
    d, k = V.shape
    out = np.empty_like(V)
    col, res = np.empty(d), np.empty(d)
    for c in range(k):
        col[:] = V[:, c]
        lib().pfo_tridiag_matvec(d, _p(sub), _p(diag), _p(sup), _p(col), _p(res))
        out[:, c] = res
    return out.reshape(-1) if vec else out


def tridiag_one_norm(sub, diag, sup) -> float:
    lib().pfo_tridiag_one_norm.restype = C.c_double
    return float(lib().pfo_tridiag_one_norm(len(diag), _p(_f64(sub)), _p(_f64(diag)), _p(_f64(sup))))


def thomas_solve(sub, diag, sup, rhs) -> np.ndarray:
    sub, diag, sup = _f64(sub), _f64(diag), _f64(sup)
    R, vec = _cols(rhs)
    d, k = R.shape
    out = np.empty_like(R)
    col, x = np.empty(d), np.empty(d)
    row = C.c_int(0)
    for c in range(k):
        col[:] = R[:, c]
        rc = lib().pfo_thomas_solve(d, _p(sub), _p(diag), _p(sup), _p(col), _p(x), C.byref(row))
        if rc:
            raise BandError(rc, row.value)
        out[:, c] = x
    return out.reshape(-1) if vec else out


def tridiag_factor(sub, diag, sup):
    """TridiagFactor: (mult, fdiag)."""
    sub, diag, sup = _f64(sub), _f64(diag), _f64(sup)
    d = len(diag)
    mult, fd = np.empty(max(d - 1, 1)), np.empty(d)
    row = C.c_int(0)
    rc = lib().pfo_tridiag_factor(d, _p(sub), _p(diag), _p(sup), _p(mult), _p(fd), C.byref(row))
    if rc:
        raise BandError(rc, row.value)
    return mult, fd


def tridiag_factor_solve(mult, fd, sup, rhs) -> np.ndarray:
    rhs = _f64(rhs)
    x = np.empty_like(rhs)
    lib().pfo_tridiag_factor_solve(len(fd), _p(_f64(mult)), _p(_f64(fd)), _p(_f64(sup)), _p(rhs), _p(x))
    return x


def pentadiag_solve(sub2, sub1, diag, super1, super2, rhs) -> np.ndarray:
    bands = [_f64(b) for b in (sub2, sub1, diag, super1, super2)]
    R, vec = _cols(rhs)
    d, k = R.shape
    out = np.empty_like(R)
    col, x = np.empty(d), np.empty(d)
    row = C.c_int(0)
    for c in range(k):
        col[:] = R[:, c]
        rc = lib().pfo_pentadiag_solve(d, *[_p(b) for b in bands], _p(col), _p(x), C.byref(row))
        if rc:
            raise BandError(rc, row.value)
        out[:, c] = x
    return out.reshape(-1) if vec else out


def tridiag_action(sub, diag, sup, v, m: OMethod, substeps: int = 1) -> np.ndarray:
    """substep_action (action_eval for substeps = 1) on every column of v (d x k or d)."""
    sub, diag, sup = _f64(sub), _f64(diag), _f64(sup)
    V, vec = _cols(v)
    V = np.ascontiguousarray(V)
    d, k = V.shape
    out = np.empty_like(V)
    st = Status()
    rc = lib().pfo_tridiag_action(d, k, _p(sub), _p(diag), _p(sup), _p(V), C.byref(m.c), substeps, _p(out),
                                  C.byref(st))
    if rc:
        raise BandError(rc, st.column, st.shift_index)
    return out.reshape(-1) if vec else out
