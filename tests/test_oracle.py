"""Pins the CPU oracle (oracle/pf_oracle.c) against the reference's own known-answer and property
tests for the dense path -- the reference itself cannot be built here (no gmpxx / vendor/), so
these KATs plus the committed golden fixtures are the oracle's pin (proj/tests/test_dense.cpp,
test_action.cpp, rng.hpp). An independent referee (scipy / mpmath) checks accuracy claims.
"""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2210_03714_b200 import methods as M
from paper_2210_03714_b200 import workloads as W

GOLD = Path(__file__).resolve().parent / "golden"


def rand(n, seed, norm):
    return W.scaled_to_one_norm(W.randn_matrix(n, seed), norm)


def om(name, form=M.RESIDUAL, oracle=None, extra=()):
    from oracle import oracle as O

    return O.OMethod.from_method(M.catalog(name) if isinstance(name, str) else name, form, extra)


# ------------------------------------------------------------------ generators (rng.hpp, rng.cpp)


def test_splitmix64_known_answer(oracle):
    import ctypes as C

    s = C.c_uint64(0)
    lib = oracle.lib()
    lib.pfo_splitmix_next.restype = C.c_uint64
    first = [lib.pfo_splitmix_next(C.byref(s)) for _ in range(3)]
    # the published SplitMix64 sequence from state 0
    assert first == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_host_and_oracle_generators_agree(oracle):
    a = W.randn(12345, 1001)
    b = np.empty(1001)
    oracle.lib().pfo_randn_fill(__import__("ctypes").c_uint64(12345), 1001, oracle._p(b))
    assert np.array_equal(a, b)
    assert np.all(W.uniform(7, 100) < 1.0) and np.all(W.uniform(7, 100) >= 0.0)


# ------------------------------------------------------------------ DenseLu (test_dense.cpp:34-83)


def test_lu_solve_and_singularity(oracle):
    a = np.array([[2.0, 1, 0], [0, 3, -1], [1, 0, 4]])
    lu, piv = oracle.lu(a)
    x = oracle.lu_solve_matrix(lu, piv, np.array([[3.0], [2.0], [5.0]]))[:, 0]
    np.testing.assert_allclose(a @ x, [3, 2, 5], rtol=1e-14)
    sing = np.array([[1.0, 0.0], [1.0, 0.0]])
    with pytest.raises(oracle.OracleError) as e:
        oracle.lu(sing)
    assert e.value.code == 7  # SingularShift + 1
    assert e.value.status.column == 1


def test_lu_pivot_rule_first_max_wins(oracle):
    """strict '>' in the column argmax: ties keep the earlier row (dense.cpp:107-115)."""
    a = np.array([[1.0, 2.0, 0.0], [-3.0, 1.0, 1.0], [3.0, 0.0, 2.0]])
    lu, piv = oracle.lu(a)
    assert list(piv[:1]) == [1]


def test_solve_shifted(oracle):
    z = np.zeros((4, 4))
    assert np.array_equal(oracle.solve_shifted(z, 0.3), np.eye(4))
    d = np.diag([1.0, -2.0, 0.5])
    di = oracle.solve_shifted(d, 0.25)
    for i in range(3):
        assert di[i, i] == pytest.approx(1.0 / (1.0 - 0.25 * d[i, i]), rel=1e-15)
    b = W.randn_matrix(8, 3)
    x = oracle.solve_shifted(b, 0.2)
    res = oracle.mul(np.eye(8) - 0.2 * b, x) - np.eye(8)
    assert oracle.one_norm(res) <= 1e-13 * oracle.one_norm(x)
    with pytest.raises(oracle.OracleError):
        oracle.solve_shifted(np.eye(5), 1.0)


# ------------------------------------------------------------------ eval_dense (test_dense.cpp:85-156)


def test_eval_dense_trivial_and_diagonal(oracle):
    z = np.zeros((5, 5))
    assert oracle.rel_diff_1norm(oracle.eval_dense(om("R4", M.PLAIN), z), np.eye(5)) <= 1e-12
    assert oracle.rel_diff_1norm(oracle.eval_dense(om("R10", M.PLAIN), z), np.eye(5)) <= 1e-9
    r4 = M.catalog("R4")
    v = oracle.eval_dense(om("R4", M.PLAIN), np.diag([0.1] * 3))
    scalar = 0.0
    for c, w in zip(r4.shift_doubles(), r4.weight_doubles()):
        scalar += w * (1.0 / (1 - c * 0.1))
    for i in range(3):
        assert abs(v[i, i] - scalar) <= 10 * abs(scalar) * 2.23e-16


def test_eval_dense_bit_identical_across_workers(oracle):
    b = rand(24, 5, 0.7)
    m = om("R8", M.PLAIN)
    w1 = oracle.eval_dense(m, b, workers=1)
    assert np.array_equal(w1, oracle.eval_dense(m, b, workers=2))
    assert np.array_equal(w1, oracle.eval_dense(m, b, workers=8))


def test_plain_and_residual_agree_and_singular_message(oracle):
    b = rand(24, 7, 1.0)
    plain = oracle.eval_dense(om("R10", M.PLAIN), b)
    resid = oracle.eval_dense(om("R10", M.RESIDUAL), b)
    assert np.linalg.norm(plain - resid, 2) <= 1e-8
    with pytest.raises(oracle.OracleError) as e:
        oracle.eval_dense(om("R10", M.PLAIN), 8.0 * np.eye(4))
    assert e.value.code == 7 and e.value.status.shift_index >= 1


def test_bound_compliance_at_single_precision_theta(oracle):
    """test_dense.cpp:142-156 with scipy.linalg.expm as the high-precision referee (its error,
    ~1e-15, is 8 orders below the 10 tol bar)."""
    sl = pytest.importorskip("scipy.linalg")
    tol = 5.9604644775390625e-8
    r8 = M.catalog("R8")
    th = M.theta(r8, tol=tol)
    b = rand(40, 11, th)
    err = np.linalg.norm(sl.expm(b) - oracle.eval_dense(om("R8", M.PLAIN), b), 2)
    assert err <= 10 * tol
    b1 = rand(100, 12, 1.0)
    err1 = np.linalg.norm(sl.expm(b1) - oracle.eval_dense(om("R8", M.PLAIN), b1), 2)
    assert err1 <= M.forward_bound(r8, r8.function, 1.0)


# ------------------------------------------------------------------ compositions


@pytest.mark.parametrize("name", ["R4", "R8"])
def test_expm_scaling_and_squaring_accuracy(oracle, name):
    sl = pytest.importorskip("scipy.linalg")
    a = W.cfg1()
    e, j = oracle.expm(a, om(name), M.THETA_U53[name])
    assert j == M.squarings_for(W.one_norm(a), M.THETA_U53[name])
    ref = sl.expm(a)
    assert oracle.rel_diff_1norm(e, ref) <= 1e-12


def test_expm_phi1_accuracy(oracle):
    sl = pytest.importorskip("scipy.linalg")
    r8 = M.catalog("R8")
    phi = M.same_shift_method(r8, M.FunctionId.phi(1))
    a = rand(60, 3, 5.0)
    th = min(M.THETA_U53["R8"], M.THETA_U53["R8_phi1set"])
    e, p, j = oracle.expm_phi1(a, om("R8", M.RESIDUAL, extra=[phi]), th)
    ee = sl.expm(a)
    assert oracle.rel_diff_1norm(e, ee) <= 1e-12
    # phi1(A) A = e^A - I
    assert oracle.rel_diff_1norm(p @ a, ee - np.eye(60)) <= 1e-11


def test_cossin_accuracy(oracle):
    from oracle import oracle as O

    pm = O.OPair.from_pair(M.pair_method(M.catalog("R8")))
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((48, 48)))
    lam = rng.uniform(0, 50, 48)
    a = (q * lam) @ q.T
    a = 0.5 * (a + a.T)
    c, s, j = oracle.cossin(a, pm, M.THETA_U53["R8"])
    w, v = np.linalg.eigh(a)
    assert np.abs(c - (v * np.cos(w)) @ v.T).max() <= 1e-10
    assert np.abs(s - (v * np.sin(w)) @ v.T).max() <= 1e-10


def test_action_matches_densified_evaluator(oracle):
    """test_action.cpp:124-147 on the dense block action: one substep of r(A)V equals
    eval_dense(A) V within max(1e-12, 100 max|coef| u)."""
    a = rand(50, 41, 1.2)
    v = W.randn(43, 50 * 3).reshape(50, 3)
    for name in ("R4", "R5", "R8", "R10", "R10star"):
        m = M.catalog(name)
        tol = max(1e-12, 100 * float(m.max_coefficient()) * 2.23e-16)
        for form in (M.PLAIN, M.RESIDUAL):
            by_action = oracle.action(a, v, om(name, form), 1)
            by_dense = oracle.eval_dense(om(name, form), a) @ v
            assert np.abs(by_action - by_dense).max() / np.abs(by_dense).max() <= tol


def test_action_determinism_and_substepping(oracle):
    sl = pytest.importorskip("scipy.linalg")
    a = W.trid121_dense(60)
    a *= 3.0 / W.one_norm(a)
    v = W.randn(61, 60 * 2).reshape(60, 2)
    n_sub = M.substeps_for(3.0, M.THETA_U53["R8"])
    w1 = oracle.action(a, v, om("R8"), n_sub, workers=1)
    w8 = oracle.action(a, v, om("R8"), n_sub, workers=8)
    assert np.array_equal(w1, w8)
    ref = sl.expm(a) @ v
    assert np.abs(w1 - ref).max() <= 1e-12 * np.abs(ref).max()


# ------------------------------------------------------------------ golden fixtures


def test_golden_fixtures_reproduce_bitwise(oracle):
    """The oracle reproduces the committed reference fixtures exactly (tests/golden/make_golden.py)."""
    meta = json.loads((GOLD / "golden.json").read_text())
    from tests.golden.make_golden import compute

    fresh = compute("oracle")
    for key, entry in meta["cases"].items():
        arr = np.load(GOLD / entry["file"])
        assert hashlib.sha256(arr.tobytes()).hexdigest() == entry["sha256"], key
        assert np.array_equal(fresh[key], arr), key
