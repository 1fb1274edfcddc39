"""Experiment drivers, host side: the binary128 oracles against independent
references, two_norm_est, the CSV formatting helpers and argument errors of cli.cpp."""
import math

import numpy as np
import pytest
import scipy.linalg as sl

from paper_2210_03714_b200 import drivers as D
from paper_2210_03714_b200.errors import Errc, PfError


def test_exact_decimal_string():
    # rational.cpp:95-115 (exact expansion, trailing zeros stripped, e-exponent)
    assert D.exact_decimal_string(2.0 ** -53) == "1.1102230246251565404236316680908203125e-16"
    assert D.exact_decimal_string(3.0) == "3"
    assert D.exact_decimal_string(1200.0) == "1.2e3"
    assert D.exact_decimal_string(-0.5) == "-5e-1"
    assert D.exact_decimal_string(0.0) == "0"


def test_log_grid_and_tokens():
    g = D.log_grid(1e-2, 4.0, 40)
    assert len(g) == 40 and g[0] == 1e-2 and abs(g[-1] - 4.0) < 1e-14
    assert D.log_grid(0.5, 1.0, 1) == [0.5]
    with pytest.raises(PfError):
        D.log_grid(0.0, 1.0, 3)
    assert D.split_form("R8:plain") == ("R8", 0) and D.split_form("R8:residual") == ("R8", 1)
    with pytest.raises(PfError) as e:
        D.split_form("R8:other")
    assert e.value.code == Errc.BadArgument


def test_two_norm_est():
    a = D.make_dense_matrix(D.MatrixSpec("randn", 40, 3))
    assert abs(D.two_norm_est(a) - np.linalg.norm(a, 2)) < 1e-6 * np.linalg.norm(a, 2)
    s, d, u = D.trid121(64)
    t = np.diag(d) + np.diag(s, -1) + np.diag(u, 1)
    # power iteration: a lower estimate, slow on trid121's clustered top singular values
    est, true = D.two_norm_est_tridiag(s, d, u), np.linalg.norm(t, 2)
    assert est <= true * (1 + 1e-12) and est > 0.99 * true


@pytest.mark.parametrize("h", [0.05, 0.7, 3.0])
def test_dense_oracle_matches_scipy(h):
    """the binary128 expm / phi1 oracles against scipy (double precision; the differences are
    scipy's own ~1e-16 errors)"""
    a = D.make_dense_matrix(D.MatrixSpec("randn", 24, 5))
    b = a * (h / D.two_norm_est(a))
    e_sc = sl.expm(b)
    err = D.dense_errors("exp", b, [e_sc])[0]
    assert err < 1e-13 * max(1.0, np.linalg.norm(e_sc, 2))
    # phi1(b) = top-right block of expm([[b, I], [0, 0]])
    n = b.shape[0]
    aug = np.zeros((2 * n, 2 * n))
    aug[:n, :n] = b
    aug[:n, n:] = np.eye(n)
    p_sc = sl.expm(aug)[:n, n:]
    err = D.dense_errors("phi1", b, [p_sc])[0]
    assert err < 1e-13 * max(1.0, np.linalg.norm(p_sc, 2))
    # a perturbed approximation is measured at its perturbation's size
    pert = e_sc.copy()
    pert[3, 4] += 1e-9
    assert abs(D.dense_errors("exp", b, [pert])[0] - 1e-9) < 1e-12


def _trid121_expm_v(n, h, v):
    """exp(h trid121) v from trid121's closed-form eigendecomposition (lambda_k = 2 - 2cos(k pi/(n+1)),
    q_jk = sqrt(2/(n+1)) sin(jk pi/(n+1))), in 40-digit mpmath"""
    import mpmath as mp

    with mp.workdps(40):
        hh = mp.mpf(h)
        res = [mp.mpf(0)] * n
        for k in range(1, n + 1):
            q = [mp.sqrt(mp.mpf(2) / (n + 1)) * mp.sin(j * k * mp.pi / (n + 1)) for j in range(1, n + 1)]
            c = mp.fsum(q[j] * mp.mpf(v[j]) for j in range(n)) * mp.exp(hh * (2 - 2 * mp.cos(k * mp.pi / (n + 1))))
            for j in range(n):
                res[j] += c * q[j]
        return res


def test_action_oracle_matches_closed_form():
    n = 40
    s, d, u = D.trid121(n)
    v = D.random_unit_vector(n, 1)
    assert abs(np.linalg.norm(v) - 1) < 1e-15
    scale = D.two_norm_est_tridiag(s, d, u)
    for hn in (0.01, 0.5, 4.0):
        h = hn / scale
        ex = _trid121_expm_v(n, h, v)
        ref = np.array([float(x) for x in ex])
        err = D.action_errors(s * h, d * h, u * h, v, [ref])[0]
        # only the rounding of the closed-form reference to doubles remains
        assert err <= 2 * np.sqrt(n) * np.finfo(float).eps * np.abs(ref).max()


def test_oracle_argument_errors():
    with pytest.raises(PfError):
        D.dense_errors("exp", np.eye(3), [np.eye(3)], digits=20)
    with pytest.raises(PfError):
        D.cmd_bench_dense([], D.MatrixSpec("randn", 4, 1))
    with pytest.raises(PfError):
        D.cmd_bench_action(["R8"], D.MatrixSpec("randn", 10, 1))
    with pytest.raises(PfError):
        D.MatrixSpec("bogus", 3, 1)


def test_theta_csv():
    out = D.cmd_theta(["R4", "R8"], [2.0 ** -53])
    lines = out.strip().split("\n")
    assert lines[0] == "method,tol,theta,theta_3dp,saturated"
    assert lines[1] == "R4,1.1102230246251565404236316680908203125e-16,0.0030785030654580181,0.003,0"
    assert lines[2].startswith("R8,1.1102230246251565404236316680908203125e-16,0.0973103939513804,0.097,")
    eps = D.cmd_theta(["R4"], eps_grid=[0.001, 0.01]).strip().split("\n")
    assert eps[0] == "method,x,epsilon" and len(eps) == 3
    assert float(eps[1].split(",")[2]) < float(eps[2].split(",")[2])
    with pytest.raises(PfError):
        D.cmd_theta(["R4"])


def test_costs():
    # cli.cpp:221-227 and 249-261
    e = D.dense_entry("R4")
    assert math.isclose(e.serial_cost, 4 * 4 / 3) and math.isclose(e.parallel_cost, 4 / 3)
    e = D.dense_entry("R10star")
    assert math.isclose(e.serial_cost, 10 * 4 / 3 + 1)
    assert D.dense_entry("taylor8").serial_cost == 3.0
    a = D.action_entry("R8:residual")
    assert math.isclose(a.serial_cost, 8 * 13 / 5) and math.isclose(a.parallel_cost, 13 / 5)
    a = D.action_entry("R8:plain")
    assert math.isclose(a.serial_cost, 8 * 8 / 5)
    assert D.action_entry("taylor20").serial_cost == 20.0
    with pytest.raises(PfError):
        D.action_entry("R4_phi1")
