"""CPU pinning of the banded oracle (oracle/pf_oracle_band.c) by the reference's own tests for
proj/core/src/action.cpp (test_action.cpp:49-188): thomas vs dense, factor reuse exactly equal,
pentadiagonal vs dense LU, ZeroPivot, action vs the densified evaluator, A = 0, determinism."""
import numpy as np
import pytest


def test_thomas_solve(oracle):
    d = 40
    eye = np.zeros(d - 1), np.ones(d), np.zeros(d - 1)
    v = np.random.default_rng(1).standard_normal(d)
    assert np.array_equal(oracle.thomas_solve(*eye, v), v)  # test_action.cpp:54
    rng = np.random.default_rng(2)
    sub, sup = rng.standard_normal(d - 1), rng.standard_normal(d - 1)
    diag = rng.standard_normal(d) + 4.0
    A = np.diag(diag) + np.diag(sub, -1) + np.diag(sup, 1)
    x = oracle.thomas_solve(sub, diag, sup, v)
    assert np.linalg.norm(x - np.linalg.solve(A, v)) / np.linalg.norm(x) <= 1e-13  # :62
    assert np.linalg.norm(A @ x - v) / np.linalg.norm(v) <= 1e-12  # :73
    mult, fd = oracle.tridiag_factor(sub, diag, sup)
    for s in range(5):  # :85-91 factorization reuse matches the one-shot solver exactly
        r = np.random.default_rng(10 + s).standard_normal(d)
        assert np.array_equal(oracle.tridiag_factor_solve(mult, fd, sup, r), oracle.thomas_solve(sub, diag, sup, r))
    z = np.zeros(d)
    with pytest.raises(oracle.BandError) as e:  # :75-82 ZeroPivot
        oracle.thomas_solve(np.ones(d - 1), z, np.ones(d - 1), v)
    assert e.value.code == 8 and e.value.row == 0


def test_pentadiag_solve(oracle):
    d = 30
    rng = np.random.default_rng(4)
    b = [rng.standard_normal(d - 2), rng.standard_normal(d - 1), rng.standard_normal(d) + 6.0,
         rng.standard_normal(d - 1), rng.standard_normal(d - 2)]
    A = np.diag(b[2]) + np.diag(b[1], -1) + np.diag(b[0], -2) + np.diag(b[3], 1) + np.diag(b[4], 2)
    rhs = rng.standard_normal(d)
    x = oracle.pentadiag_solve(*b, rhs)
    assert np.linalg.norm(x - np.linalg.solve(A, rhs)) / np.linalg.norm(x) <= 1e-12  # :95-114
    with pytest.raises(oracle.BandError):  # :117-121
        oracle.pentadiag_solve(np.zeros(0), np.zeros(1), np.zeros(2), np.zeros(1), np.zeros(0), np.ones(2))


@pytest.mark.parametrize("name,form", [("R4", 1), ("R8", 1), ("R8", 0), ("R10", 1), ("R10star", 0)])
def test_action_matches_densified_evaluator(oracle, name, form):
    from paper_2210_03714_b200 import methods as M

    m = M.catalog(name)
    d = 60
    sub, diag, sup = -0.2 * np.ones(d - 1), 0.4 * np.ones(d), -0.2 * np.ones(d - 1)
    A = np.diag(diag) + np.diag(sub, -1) + np.diag(sup, 1)
    v = np.random.default_rng(5).standard_normal((d, 3))
    om = oracle.OMethod.from_method(m, form)
    by_action = oracle.tridiag_action(sub, diag, sup, v, om, 2)
    by_dense = oracle.action(A, v, om, 2)
    amp = float(sum(abs(w) for w in m.weights) + sum(abs(x) for x in m.poly))
    assert oracle.rel_diff_1norm(by_action, by_dense) <= max(1e-11, 100 * amp * 2.23e-16)  # :124-147
    z = oracle.tridiag_action(np.zeros(d - 1), np.zeros(d), np.zeros(d - 1), v, om, 1)
    if form == 1:
        assert np.array_equal(z, v)  # :149-157 (a0 = 1 for exp)
    # determinism (:159-169): repeated evaluations identical
    assert np.array_equal(by_action, oracle.tridiag_action(sub, diag, sup, v, om, 2))


def test_matvec_and_norm(oracle):
    d = 9
    sub, diag, sup = -np.ones(d - 1), 2 * np.ones(d), -np.ones(d - 1)
    v = np.arange(d, dtype=float)
    A = np.diag(diag) + np.diag(sub, -1) + np.diag(sup, 1)
    assert np.array_equal(oracle.tridiag_matvec(sub, diag, sup, v), A @ v)
    assert oracle.tridiag_one_norm(sub, diag, sup) == 4.0
