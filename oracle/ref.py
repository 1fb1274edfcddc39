"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of THE REFERENCE ITSELF (oracle/_ref/libparfrac_ref.so).

``oracle/Makefile`` compiles ``/root/reference/proj/core/src/*.cpp`` unmodified against the
GMP/gmpxx shims in ``oracle/shim/`` plus ``oracle/ref_capi.cpp``. This module is the checker that
pins ``oracle/pf_oracle.c`` (the fast restatement) bit for bit and the reference arm of
``bench.py``; the product path never loads it. ``available()`` is False where neither the sources
nor a prebuilt library exist.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
_SO = REF_DIR / "libparfrac_ref.so"
REF_SOURCES = Path("/root/reference/proj/core/src")

DP = C.POINTER(C.c_double)
_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__("reference error %d: %s" % (code, msg))
        self.code = code
        self.msg = msg


def build() -> bool:
    """Compile oracle/_ref when the reference sources are present (no-op on the GPU box)."""
    if REF_SOURCES.exists():
        subprocess.run(["make", "-s", "-j8", "-C", str(HERE), "ref"], check=True)
    return _SO.exists()


def available() -> bool:
    return _SO.exists() or REF_SOURCES.exists()


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = C.CDLL(str(_SO))
        L.pfr_catalog.restype = C.c_void_p
        L.pfr_build_plain.restype = C.c_void_p
        L.pfr_with_form.restype = C.c_void_p
        L.pfr_with_form.argtypes = [C.c_void_p, C.c_int]
        L.pfr_method_free.argtypes = [C.c_void_p]
        L.pfr_one_norm.restype = C.c_double
        L.pfr_solve_shifted.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_char_p, C.c_int]
        L.pfr_splitmix.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.pfr_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.pfr_normal.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        L.pfr_make_dense_matrix.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.c_char_p, C.c_int]
        L.pfr_random_unit_vector.argtypes = [C.c_int, C.c_uint64, C.c_void_p, C.c_char_p, C.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _err():
    return C.create_string_buffer(512)


def _check(rc: int, err):
    if rc:
        raise RefError(rc, err.value.decode(errors="replace"))


def _form(form: Optional[int]) -> int:
    return -1 if form is None else int(form)


class RefMethod:
    """A parfrac::FractionMethod owned by the reference library (catalog / build_plain)."""

    def __init__(self, handle: int):
        if not handle:
            raise RefError(-1, "method construction failed")
        self.h = C.c_void_p(handle)

    def __del__(self):
        if _lib is not None and getattr(self, "h", None):
            _lib.pfr_method_free(self.h)
            self.h = None

    @staticmethod
    def catalog(name: str) -> "RefMethod":
        err = _err()
        h = lib().pfr_catalog(name.encode(), err, len(err))
        if not h:
            raise RefError(-1, err.value.decode())
        return RefMethod(h)

    @staticmethod
    def build_plain(template: int, alpha: str, function: str, order: int) -> "RefMethod":
        err = _err()
        h = lib().pfr_build_plain(int(template), alpha.encode(), function.encode(), int(order), err, len(err))
        if not h:
            raise RefError(-1, err.value.decode())
        return RefMethod(h)

    def with_form(self, form: int) -> "RefMethod":
        return RefMethod(lib().pfr_with_form(self.h, int(form)))

    def doubles(self):
        sh, w, po = (C.c_double * 16)(), (C.c_double * 16)(), (C.c_double * 4)()
        n, npoly, form = C.c_int(), C.c_int(), C.c_int()
        a0 = C.c_double()
        lib().pfr_method_doubles(self.h, C.byref(n), sh, w, C.byref(npoly), po, C.byref(a0), C.byref(form))
        return dict(shifts=list(sh[: n.value]), weights=list(w[: n.value]), poly=list(po[: npoly.value]),
                    a0=a0.value, form=form.value)

    def text(self):
        buf = C.create_string_buffer(1 << 16)
        lib().pfr_method_text(self.h, buf, len(buf))
        return buf.value.decode().split("\n")[:-1]

    def theta(self, tol: float) -> Tuple[float, bool]:
        err, th, sat = _err(), C.c_double(), C.c_int()
        _check(lib().pfr_theta(self.h, C.c_double(tol), C.byref(th), C.byref(sat), err, len(err)), err)
        return th.value, bool(sat.value)


def theta_taylor(degree: int, tol: float) -> float:
    err, th = _err(), C.c_double()
    _check(lib().pfr_theta_taylor(int(degree), C.c_double(tol), C.byref(th), err, len(err)), err)
    return th.value


# ---------------------------------------------------------------- dense.cpp
def mul(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    out = np.empty_like(a)
    lib().pfr_mul(a.shape[0], _p(a), _p(b), _p(out))
    return out


def one_norm(a) -> float:
    a = _f64(a)
    return lib().pfr_one_norm(a.shape[0], _p(a))


def lu(a, rel_tol: float = 1e-14):
    a = _f64(a)
    n = a.shape[0]
    out, piv, err = np.empty_like(a), np.empty(n, dtype=np.int32), _err()
    _check(lib().pfr_lu(n, _p(a), C.c_double(rel_tol), _p(out), _p(piv), err, len(err)), err)
    return out, piv


def lu_solve_matrix(a, rhs) -> np.ndarray:
    a, rhs = _f64(a), _f64(rhs)
    out, err = np.empty_like(rhs), _err()
    _check(lib().pfr_lu_solve_matrix(a.shape[0], _p(a), _p(rhs), _p(out), err, len(err)), err)
    return out


def solve_shifted(b, c: float) -> np.ndarray:
    b = _f64(b)
    out, err = np.empty_like(b), _err()
    _check(lib().pfr_solve_shifted(b.shape[0], _p(b), c, _p(out), err, len(err)), err)
    return out


def eval_dense(m: RefMethod, b, form: Optional[int] = None, workers: int = 1) -> np.ndarray:
    b = _f64(b)
    out, err = np.empty_like(b), _err()
    _check(lib().pfr_eval_dense(m.h, _form(form), b.shape[0], _p(b), int(workers), _p(out), err, len(err)), err)
    return out


def baseline(which: str, b) -> np.ndarray:
    b = _f64(b)
    out, err = np.empty_like(b), _err()
    _check(lib().pfr_baseline(which.encode(), b.shape[0], _p(b), _p(out), err, len(err)), err)
    return out


def expm(m: RefMethod, a, theta: float, form: Optional[int] = None, j_fixed: int = -1, workers: int = 1):
    a = _f64(a)
    out, j, err = np.empty_like(a), C.c_int(), _err()
    _check(lib().pfr_expm(m.h, _form(form), a.shape[0], _p(a), C.c_double(theta), int(j_fixed), int(workers),
                          _p(out), C.byref(j), err, len(err)), err)
    return out, j.value


def expm_batched(m: RefMethod, a, theta: float, form: Optional[int] = None, threads: int = 1):
    a = _f64(a)
    batch, n = a.shape[0], a.shape[1]
    out, js = np.empty_like(a), np.empty(batch, dtype=np.int32)
    bad, err = C.c_int(-1), _err()
    _check(lib().pfr_expm_batched(m.h, _form(form), n, batch, _p(a), C.c_double(theta), int(threads), _p(out),
                                  _p(js), C.byref(bad), err, len(err)), err)
    return out, js


def expm_phi1(m_exp: RefMethod, m_phi: RefMethod, a, theta: float, form: Optional[int] = None, j_fixed: int = -1,
              workers: int = 1):
    a = _f64(a)
    oe, op, j, err = np.empty_like(a), np.empty_like(a), C.c_int(), _err()
    _check(lib().pfr_expm_phi1(m_exp.h, m_phi.h, _form(form), a.shape[0], _p(a), C.c_double(theta), int(j_fixed),
                               int(workers), _p(oe), _p(op), C.byref(j), err, len(err)), err)
    return oe, op, j.value


def dense_action(m: RefMethod, a, v, substeps: int, form: Optional[int] = None, workers: int = 1) -> np.ndarray:
    a, v = _f64(a), _f64(v)
    n, k = v.shape
    out, err = np.empty_like(v), _err()
    _check(lib().pfr_dense_action(m.h, _form(form), n, k, _p(a), _p(v), int(substeps), int(workers), _p(out), err,
                                  len(err)), err)
    return out


# ---------------------------------------------------------------- action.cpp (banded)
def thomas_solve(sub, diag, sup, rhs) -> np.ndarray:
    sub, diag, sup, rhs = map(_f64, (sub, diag, sup, rhs))
    out, err = np.empty_like(rhs), _err()
    _check(lib().pfr_thomas_solve(len(diag), _p(sub), _p(diag), _p(sup), _p(rhs), _p(out), err, len(err)), err)
    return out


def tridiag_factor_solve(sub, diag, sup, rhs) -> np.ndarray:
    sub, diag, sup, rhs = map(_f64, (sub, diag, sup, rhs))
    out, err = np.empty_like(rhs), _err()
    _check(lib().pfr_tridiag_factor_solve(len(diag), _p(sub), _p(diag), _p(sup), _p(rhs), _p(out), err, len(err)),
           err)
    return out


def pentadiag_solve(sub2, sub1, diag, super1, super2, rhs) -> np.ndarray:
    arrs = list(map(_f64, (sub2, sub1, diag, super1, super2, rhs)))
    out, err = np.empty_like(arrs[-1]), _err()
    _check(lib().pfr_pentadiag_solve(len(arrs[2]), *[_p(x) for x in arrs], _p(out), err, len(err)), err)
    return out


def tridiag_matvec(sub, diag, sup, v) -> np.ndarray:
    sub, diag, sup, v = map(_f64, (sub, diag, sup, v))
    out = np.empty_like(v)
    lib().pfr_tridiag_matvec(len(diag), _p(sub), _p(diag), _p(sup), _p(v), _p(out))
    return out


def tridiag_action(m: RefMethod, sub, diag, sup, v, mode: str = "eval", substeps: int = 1,
                   form: Optional[int] = None, workers: int = 1) -> np.ndarray:
    """mode 'eval' = action_eval, 'substep' = substep_action, 'operator' = ActionOperator::apply."""
    sub, diag, sup, v = map(_f64, (sub, diag, sup, v))
    out, err = np.empty_like(v), _err()
    md = {"eval": 0, "substep": 1, "operator": 2}[mode]
    _check(lib().pfr_tridiag_action(m.h, _form(form), md, len(diag), _p(sub), _p(diag), _p(sup), _p(v),
                                    int(substeps), int(workers), _p(out), err, len(err)), err)
    return out


# ---------------------------------------------------------------- generators
def splitmix(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().pfr_splitmix(seed, count, _p(out))
    return out


def uniform(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().pfr_uniform(seed, count, _p(out))
    return out


def normal(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().pfr_normal(seed, count, _p(out))
    return out


def make_dense_matrix(kind: str, dim: int, seed: int) -> np.ndarray:
    out, err = np.empty((dim, dim)), _err()
    k = {"randn": 0, "cauchy": 1, "trid121": 2}[kind]
    _check(lib().pfr_make_dense_matrix(k, dim, seed, _p(out), err, len(err)), err)
    return out


def random_unit_vector(dim: int, seed: int) -> np.ndarray:
    out, err = np.empty(dim), _err()
    _check(lib().pfr_random_unit_vector(dim, seed, _p(out), err, len(err)), err)
    return out


def run_unit_tests(suite: Optional[str] = None, timeout: float = 600) -> subprocess.CompletedProcess:
    """The reference's own doctest suites, built from proj/tests/*.cpp (oracle/_ref/unit_tests)."""
    cmd = [str(REF_DIR / "unit_tests")] + (["--test-suite=" + suite] if suite else [])
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)


def run_acceptance(timeout: float = 900) -> subprocess.CompletedProcess:
    """The reference's acceptance checklist (proj/tests/acceptance_main.cpp, oracle/_ref/acceptance)."""
    return subprocess.run([str(REF_DIR / "acceptance")], capture_output=True, text=True, timeout=timeout,
                          env=dict(os.environ))
