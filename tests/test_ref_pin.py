"""Pins the fast CPU checker (oracle/pf_oracle.c, pf_oracle_band.c) and the method layer
(paper_2210_03714_b200/methods.py) against THE REFERENCE ITSELF, bit for bit.

oracle/_ref is /root/reference/proj/core/src/*.cpp compiled unmodified (oracle/Makefile, GMP/gmpxx
shims in oracle/shim/). Before it is trusted, the reference's own doctest suites
(proj/tests/test_*.cpp) and acceptance checklist (acceptance_main.cpp) run against the same build.
Every other comparison here is exact equality (np.array_equal on the raw doubles / pivots).
"""
import numpy as np
import pytest

from oracle import ref as R
from paper_2210_03714_b200 import methods as M
from paper_2210_03714_b200 import workloads as W

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built and reference sources absent")

METHODS = ["R4", "R4_phi1", "R5", "R8", "R10star", "R10"]


def rand(n, seed, norm):
    return W.scaled_to_one_norm(W.randn_matrix(n, seed), norm)


def om(name, form):
    from oracle import oracle as O

    return O.OMethod.from_method(M.catalog(name) if isinstance(name, str) else name, form)


@pytest.fixture(scope="module")
def ref():
    R.lib()
    return R


# ------------------------------------------------------------ the reference build is the reference


@pytest.mark.parametrize("suite", ["rational", "series", "methods", "bounds", "dense", "action", "cli"])
def test_reference_unit_suites_pass_on_this_build(ref, suite):
    r = ref.run_unit_tests(suite)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_reference_acceptance_passes_on_this_build(ref):
    """proj/tests/acceptance_main.cpp: all nine checks, incl. 'R8 <= taylor8 on >= 90 %' (:205-212)."""
    r = ref.run_acceptance()
    assert r.returncode == 0, r.stdout[-3000:]
    assert "all acceptance checks passed" in r.stdout
    assert r.stdout.count("[PASS]") == 9


# ------------------------------------------------------------ method layer (methods.cpp, bounds.cpp)


@pytest.mark.parametrize("name", METHODS)
def test_catalog_exact_and_doubles(ref, name):
    m, rm = M.catalog(name), ref.RefMethod.catalog(name)
    text = rm.text()
    ns = len(m.shifts)
    assert text[:ns] == [M.to_fraction_string(q) for q in m.shifts]
    assert text[ns:2 * ns] == [M.to_fraction_string(q) for q in m.weights]
    assert text[2 * ns:] == [M.to_fraction_string(q) for q in m.poly]
    d = rm.doubles()
    assert d["shifts"] == m.shift_doubles() and d["weights"] == m.weight_doubles()
    assert d["poly"] == [M.to_double_nearest(q) for q in m.poly]
    assert d["a0"] == M.to_double_nearest(m.constant_term())


@pytest.mark.parametrize("tmpl,alpha,fn,order", [(8, "5", "phi1", 8), (4, "10", "phi1", 4), (8, "5", "exp", 8),
                                                 (4, "7/2", "exp", 4), (8, "5", "cos", 8)])
def test_build_plain_matches(ref, tmpl, alpha, fn, order):
    a = M.rational_from_string(alpha)
    shifts = M.frac8_shifts(a) if tmpl == 8 else M.frac4_shifts(a)
    mine = M.build_plain(shifts, M.FunctionId.parse(fn), order, fn)
    theirs = ref.RefMethod.build_plain(tmpl, alpha, fn, order).text()
    assert theirs == [M.to_fraction_string(q) for q in list(mine.shifts) + list(mine.weights)]


@pytest.mark.parametrize("name", ["R4", "R5", "R8", "R10star", "R10", "R4_phi1"])
def test_theta_matches_reference(ref, name):
    """bounds.cpp:252 theta(): the reference bisects to 1e-6 relative width; THETA_U53 and the
    Python profile must agree with it to that width."""
    for tol in (2.0 ** -53, 2.0 ** -24, 1e-13):
        t_ref, _ = ref.RefMethod.catalog(name).theta(tol)
        t_py = M.theta(M.catalog(name), None, tol)
        assert abs(t_py - t_ref) <= 2e-6 * t_ref, (name, tol, t_py, t_ref)
    if name in M.THETA_U53:
        assert abs(M.THETA_U53[name] - ref.RefMethod.catalog(name).theta(2.0 ** -53)[0]) <= 2e-6 * M.THETA_U53[name]


def test_theta_phi1_on_r8_shifts(ref):
    t, _ = ref.RefMethod.build_plain(8, "5", "phi1", 8).theta(2.0 ** -53)
    assert abs(M.THETA_U53["R8_phi1set"] - t) <= 2e-6 * t


# ------------------------------------------------------------ dense.cpp, bit for bit


@pytest.mark.parametrize("n", [1, 2, 5, 17, 64, 128])
def test_lu_pivots_and_factors_bitwise(ref, oracle, n):
    for seed, shift in ((900, 0.2), (901, 1.3), (902, -0.7)):
        b = rand(n, seed + n, 40.0)
        a = np.eye(n) - shift * b
        lu_r, piv_r = ref.lu(a)
        lu_o, piv_o = oracle.lu(a)
        assert np.array_equal(piv_r, piv_o)
        assert np.array_equal(lu_r, lu_o)


@pytest.mark.parametrize("n", [300, 533])
def test_blocked_oracle_kernels_bitwise_multi_panel(ref, oracle, n):
    """pf_oracle.c tiles the LU (32-column panels), the multi-RHS solve (32-column blocks) and the
    products (32 x 512 tiles) without changing any element's operation order; sizes that span
    several ragged panels and tiles, with pivoting and exact zeros, must still match the reference."""
    b = rand(n, 7 + n, 50.0)
    a = np.eye(n) - 0.9 * b
    a[::7, ::5] = 0.0
    lu_r, piv_r = ref.lu(a)
    lu_o, piv_o = oracle.lu(a)
    assert np.array_equal(piv_r, piv_o) and np.array_equal(lu_r, lu_o)
    assert (piv_o != np.arange(n)).sum() > n // 2  # genuinely pivoting
    rhs = rand(n, 8 + n, 3.0)
    assert np.array_equal(ref.lu_solve_matrix(a, rhs), oracle.lu_solve_matrix(lu_o, piv_o, rhs))
    assert np.array_equal(ref.mul(a, rhs), oracle.mul(a, rhs))


def test_singular_detection_same_column(ref, oracle):
    a = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 6.0], [1.0, 0.0, 1.0]])
    with pytest.raises(ref.RefError) as er:
        ref.lu(a)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.lu(a)
    assert er.value.code == eo.value.code == 7
    assert "at column %d " % eo.value.status.column in er.value.msg


def test_mul_one_norm_solve_shifted_bitwise(ref, oracle):
    for n in (3, 40, 100):
        a, b = rand(n, 10 + n, 3.0), rand(n, 20 + n, 5.0)
        a[a < -0.01] = 0.0  # exercise the a_ik == 0 skip (dense.cpp:21)
        assert np.array_equal(ref.mul(a, b), oracle.mul(a, b))
        assert ref.one_norm(b) == oracle.one_norm(b)
        assert np.array_equal(ref.solve_shifted(b, 0.2), oracle.solve_shifted(b, 0.2))


@pytest.mark.parametrize("name", METHODS)
@pytest.mark.parametrize("form", [M.PLAIN, M.RESIDUAL])
def test_eval_dense_bitwise(ref, oracle, name, form):
    rm = ref.RefMethod.catalog(name)
    for n, seed, norm in ((5, 1, 0.3), (24, 5, 0.7), (64, 77, 0.05), (24, 900, 30.0)):
        b = rand(n, seed, norm)
        try:
            want = ref.eval_dense(rm, b, form, workers=1)
        except ref.RefError as e:  # pivoting input may be singular for some shift: same error
            with pytest.raises(oracle.OracleError) as eo:
                oracle.eval_dense(om(name, form), b)
            assert eo.value.code == e.code
            continue
        assert np.array_equal(want, oracle.eval_dense(om(name, form), b, workers=3))
        assert np.array_equal(want, ref.eval_dense(rm, b, form, workers=4))  # worker count is invisible
        assert np.array_equal(want, oracle.eval_dense(om(name, form), b, workers=20))  # threaded solves


@pytest.mark.parametrize("name", ["R4", "R8"])
def test_expm_cfg1_and_cfg2_bitwise(ref, oracle, name):
    rm = ref.RefMethod.catalog(name)
    th = M.THETA_U53[name]
    a = W.cfg1()
    e_r, j_r = ref.expm(rm, a, th, M.RESIDUAL)
    e_o, j_o = oracle.expm(a, om(name, M.RESIDUAL), th)
    assert j_r == j_o and np.array_equal(e_r, e_o)
    a2 = W.cfg2(batch=6)
    e_r, j_r = ref.expm_batched(rm, a2, th, M.RESIDUAL, threads=6)
    e_o, j_o = oracle.expm_batched(a2, om(name, M.RESIDUAL), th, threads=3)
    assert np.array_equal(j_r, j_o) and np.array_equal(e_r, e_o)


def test_expm_phi1_bitwise(ref, oracle):
    from oracle import oracle as O

    r8 = M.catalog("R8")
    phi = M.same_shift_method(r8, M.FunctionId.phi(1))
    a = rand(48, 31, 3.0)
    th = M.THETA_U53["R8_phi1set"]
    e_r, p_r, j_r = ref.expm_phi1(ref.RefMethod.catalog("R8"), ref.RefMethod.build_plain(8, "5", "phi1", 8), a, th,
                                  M.RESIDUAL)
    e_o, p_o, j_o = oracle.expm_phi1(a, O.OMethod.from_method(r8, M.RESIDUAL, extra=(phi,)), th, workers=19)
    assert j_r == j_o and np.array_equal(e_r, e_o) and np.array_equal(p_r, p_o)


@pytest.mark.parametrize("name,form", [("R8", M.RESIDUAL), ("R8", M.PLAIN), ("R10", M.RESIDUAL), ("R4", M.RESIDUAL)])
def test_dense_action_bitwise(ref, oracle, name, form):
    n, k = 40, 5
    a = rand(n, 41, 2.0)
    v = W.randn(42, n * k).reshape(n, k)
    want = ref.dense_action(ref.RefMethod.catalog(name), a, v, 3, form, workers=2)
    got = oracle.action(a, v, om(name, form), 3, workers=3)
    assert np.array_equal(want, got)
    v2 = W.randn(43, n * 40).reshape(n, 40)  # several 16-column solve blocks over threads
    assert np.array_equal(ref.dense_action(ref.RefMethod.catalog(name), a, v2, 2, form),
                          oracle.action(a, v2, om(name, form), 2, workers=29))


def test_golden_fixtures_are_reference_outputs(ref):
    """tests/golden/ (generated by make_golden.py from oracle/_ref) equal the reference bit for bit."""
    import json
    from pathlib import Path

    gold = Path(__file__).resolve().parent / "golden"
    cases = json.loads((gold / "golden.json").read_text())["cases"]
    from tests.golden.make_golden import compute

    fresh = compute("ref")
    for key, meta in cases.items():
        assert np.array_equal(np.load(gold / meta["file"]), fresh[key]), key


# ------------------------------------------------------------ action.cpp (banded), bit for bit


def _tri(d, seed, diag_shift=4.0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(d - 1), rng.standard_normal(d) + diag_shift, rng.standard_normal(d - 1)


def test_thomas_factor_pentadiag_bitwise(ref, oracle):
    for d in (1, 2, 7, 300):
        sub, diag, sup = _tri(d, d)
        rhs = np.random.default_rng(d + 1).standard_normal(d)
        assert np.array_equal(ref.thomas_solve(sub, diag, sup, rhs), oracle.thomas_solve(sub, diag, sup, rhs))
        mult, fd = oracle.tridiag_factor(sub, diag, sup)
        assert np.array_equal(ref.tridiag_factor_solve(sub, diag, sup, rhs),
                              oracle.tridiag_factor_solve(mult, fd, sup, rhs))
        assert np.array_equal(ref.tridiag_matvec(sub, diag, sup, rhs), oracle.tridiag_matvec(sub, diag, sup, rhs))
    for d in (3, 5, 64):
        rng = np.random.default_rng(d)
        b = [rng.standard_normal(d - 2), rng.standard_normal(d - 1), rng.standard_normal(d) + 6.0,
             rng.standard_normal(d - 1), rng.standard_normal(d - 2)]
        b[1][::3] = 0.0  # the f == 0 skip (action.cpp:187)
        rhs = rng.standard_normal(d)
        assert np.array_equal(ref.pentadiag_solve(*b, rhs), oracle.pentadiag_solve(*b, rhs))


def test_zero_pivot_rows_match(ref, oracle):
    d = 6
    sub, sup = np.ones(d - 1), np.ones(d - 1)
    diag = np.array([1.0, 1.0, 2.0, 1.0, 1.0, 1.0])  # row 1 pivot: 1 - 1*1/1 = 0
    with pytest.raises(ref.RefError) as er:
        ref.thomas_solve(sub, diag, sup, np.ones(d))
    with pytest.raises(oracle.BandError) as eo:
        oracle.thomas_solve(sub, diag, sup, np.ones(d))
    assert er.value.code == eo.value.code == 8
    assert er.value.msg.endswith("row %d" % eo.value.row)


@pytest.mark.parametrize("name", ["R5", "R8", "R10", "R10star"])
@pytest.mark.parametrize("form", [M.PLAIN, M.RESIDUAL])
def test_tridiag_action_bitwise(ref, oracle, name, form):
    d = 200
    t = W.trid121_dense(d)
    sub, diag, sup = np.diag(t, -1) * 0.5, np.diag(t) * 0.5, np.diag(t, 1) * 0.5
    v = ref.random_unit_vector(d, 17)
    rm = ref.RefMethod.catalog(name)
    m = om(name, form)
    want1 = ref.tridiag_action(rm, -sub, -diag, -sup, v, "eval", form=form)
    assert np.array_equal(want1, oracle.tridiag_action(-sub, -diag, -sup, v, m, 1))
    assert np.array_equal(want1, ref.tridiag_action(rm, -sub, -diag, -sup, v, "operator", form=form, workers=3))
    want4 = ref.tridiag_action(rm, -sub, -diag, -sup, v, "substep", substeps=4, form=form)
    assert np.array_equal(want4, oracle.tridiag_action(-sub, -diag, -sup, v, m, 4))


# ------------------------------------------------------------ generators (rng.hpp, rng.cpp, cli.cpp)


def test_generators_bitwise(ref, oracle):
    assert list(ref.splitmix(0, 3)) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert np.array_equal(ref.uniform(7, 1000), W.uniform(7, 1000))
    assert np.array_equal(ref.normal(12345, 1001), W.randn(12345, 1001))
    for n, seed in ((64, 1), (128, 1000), (33, 5)):
        assert np.array_equal(ref.make_dense_matrix("randn", n, seed), W.randn_matrix(n, seed))
    assert np.array_equal(ref.make_dense_matrix("cauchy", 30, 0), W.cauchy(30))
    assert np.array_equal(ref.make_dense_matrix("trid121", 30, 0), W.trid121_dense(30))
