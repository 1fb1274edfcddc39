"""GPU banded action against the CPU oracle's restatement of
proj/core/src/action.cpp: every column runs the reference's per-vector operation sequence, so the
results are compared bit for bit; ZeroPivot rows / shift indices as the reference reports them."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(pf):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need CUDA")
    from paper_2210_03714_b200 import api

    return api


def band(d, seed, dom=4.0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(d - 1), rng.standard_normal(d) + dom, rng.standard_normal(d - 1)


@pytest.mark.parametrize("d,k", [(1, 3), (2, 1), (257, 37), (4000, 130)])
def test_thomas_and_matvec_bitwise(dev, oracle, d, k):
    sub, diag, sup = band(d, d)
    rhs = np.random.default_rng(7).standard_normal((d, k))
    t = dev.TridiagMatrix(sub, diag, sup)
    assert np.array_equal(dev.thomas_solve(t, rhs), oracle.thomas_solve(sub, diag, sup, rhs))
    assert np.array_equal(dev.tridiag_matvec(t, rhs), oracle.tridiag_matvec(sub, diag, sup, rhs))
    # one vector
    assert np.array_equal(dev.thomas_solve(t, rhs[:, 0]), oracle.thomas_solve(sub, diag, sup, rhs[:, 0]))


def test_thomas_zero_pivot(dev, oracle):
    from paper_2210_03714_b200.errors import Errc, PfError

    sub, diag, sup = band(10, 3)
    diag[4] = 0.0
    sub[3] = sup[3] = 0.0  # the pivot of row 4 stays exactly 0
    with pytest.raises(oracle.BandError) as oe:
        oracle.thomas_solve(sub, diag, sup, np.ones(10))
    with pytest.raises(PfError) as ge:
        dev.thomas_solve(dev.TridiagMatrix(sub, diag, sup), np.ones(10))
    assert ge.value.code == Errc.ZeroPivot and "row %d" % oe.value.row in str(ge.value)


@pytest.mark.parametrize("d,k", [(1, 2), (3, 1), (600, 33)])
def test_pentadiag_bitwise(dev, oracle, d, k):
    rng = np.random.default_rng(d)
    b = [rng.standard_normal(max(d - 2, 0)), rng.standard_normal(max(d - 1, 0)), rng.standard_normal(d) + 6,
         rng.standard_normal(max(d - 1, 0)), rng.standard_normal(max(d - 2, 0))]
    if d > 5:
        b[0][2] = 0.0  # exercises the reference's f == 0 skip
    rhs = rng.standard_normal((d, k))
    assert np.array_equal(dev.pentadiag_solve(*b, rhs), oracle.pentadiag_solve(*b, rhs))


@pytest.mark.parametrize("name,form", [("R4", 1), ("R8", 1), ("R8", 0), ("R10", 1), ("R10star", 0), ("R5", 1)])
@pytest.mark.parametrize("substeps", [1, 4])
def test_tridiag_action_bitwise(dev, oracle, name, form, substeps):
    from paper_2210_03714_b200 import methods as M

    m = M.catalog(name)
    d, k = 3000, 70
    scale = 0.3
    sub, diag, sup = -scale * np.ones(d - 1), 2 * scale * np.ones(d), -scale * np.ones(d - 1)
    sub += 0.01 * np.random.default_rng(1).standard_normal(d - 1)
    v = np.random.default_rng(2).standard_normal((d, k))
    om = oracle.OMethod.from_method(m, form)
    ref = oracle.tridiag_action(sub, diag, sup, v, om, substeps)
    got = dev.tridiag_action(m, dev.TridiagMatrix(sub, diag, sup), v, substeps, form)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name,form", [("R8", 1), ("R8", 0), ("R10", 1), ("R4", 1), ("R5", 0)])
@pytest.mark.parametrize("d", [1, 2, 5, 203])
@pytest.mark.parametrize("k", [10240, 10241])
def test_tridiag_action_wide_bitwise(dev, oracle, name, form, d, k):
    """wide blocks: k = 10240 takes the bulk-copy kernel (>= 2 CTAs per SM, aligned rows), the odd
    k = 10241 the per-lane queue; ragged d (203 = 50 stages of 4 + 3) and the d <= 5 edges"""
    from paper_2210_03714_b200 import methods as M

    m = M.catalog(name)
    rng = np.random.default_rng(d + k)
    scale = 0.25
    sub = -scale * np.ones(max(d - 1, 0)) + 0.01 * rng.standard_normal(max(d - 1, 0))
    diag = 2 * scale * np.ones(d) + 0.01 * rng.standard_normal(d)
    sup = -scale * np.ones(max(d - 1, 0))
    v = rng.standard_normal((d, k))
    om = oracle.OMethod.from_method(m, form)
    ref = oracle.tridiag_action(sub, diag, sup, v, om, 2)
    got = dev.tridiag_action(m, dev.TridiagMatrix(sub, diag, sup), v, 2, form)
    assert np.array_equal(got, ref)


def test_tridiag_action_properties(dev, oracle):
    """the densified evaluator agrees (test_action.cpp:124-147); A = 0 gives a0 v (:149-157);
    trid121 heat step against scipy expm"""
    import scipy.linalg as sl

    from paper_2210_03714_b200 import methods as M

    m = M.catalog("R8")
    d = 200
    t = dev.TridiagMatrix.trid121(d)
    v = np.random.default_rng(3).standard_normal((d, 5))
    hs = 0.5
    a_sub, a_diag, a_sup = -hs * np.ones(d - 1), 2 * hs * np.ones(d), -hs * np.ones(d - 1)
    got = dev.tridiag_action(m, dev.TridiagMatrix(a_sub, a_diag, a_sup), v, 8, 1)
    dense = oracle.action(np.diag(a_diag) + np.diag(a_sub, -1) + np.diag(a_sup, 1), v,
                          oracle.OMethod.from_method(m, 1), 8)
    assert oracle.rel_diff_1norm(got, dense) <= 1e-11
    ex = sl.expm(-(np.diag(a_diag) + np.diag(a_sub, -1) + np.diag(a_sup, 1))) @ v
    neg = dev.tridiag_action(m, dev.TridiagMatrix(-a_sub, -a_diag, -a_sup), v, 8, 1)
    assert oracle.rel_diff_1norm(neg, ex) <= 1e-12
    z = dev.tridiag_action(m, dev.TridiagMatrix(np.zeros(d - 1), np.zeros(d), np.zeros(d - 1)), v, 1, 1)
    assert np.array_equal(z, v)  # residual r(0) v = a0 v, a0 = 1
    assert abs(t.one_norm() - 4.0) == 0.0


def test_tridiag_action_zero_pivot_shift(dev, oracle):
    from paper_2210_03714_b200 import methods as M
    from paper_2210_03714_b200.errors import Errc, PfError

    m = M.catalog("R4")
    c = m.shift_doubles()[1]
    d = 8
    diag = np.full(d, 2.0)
    diag[0] = 1.0 / c  # 1 - c a_00 = 0 for the second shift
    sub = np.zeros(d - 1)
    sup = np.zeros(d - 1)
    v = np.ones((d, 2))
    om = oracle.OMethod.from_method(m, 1)
    with pytest.raises(oracle.BandError) as oe:
        oracle.tridiag_action(sub, diag, sup, v, om, 1)
    with pytest.raises(PfError) as ge:
        dev.tridiag_action(m, dev.TridiagMatrix(sub, diag, sup), v, 1, 1)
    assert ge.value.code == Errc.ZeroPivot
    assert str(ge.value).startswith("shift %d: zero pivot at row %d" % (oe.value.shift_index, oe.value.row))


@pytest.mark.parametrize("form", [0, 1])
def test_tridiag_action_many_shifts_bitwise(dev, oracle, form):
    """a user-built method with 13 nonzero shifts (> the fused kernel's 12) and a zero shift takes
    the unfused chain (band_matvec / band_solve / band_accumulate): still the reference's bits"""
    from fractions import Fraction as Fr

    from paper_2210_03714_b200 import methods as M

    shifts = [Fr(0)] + [Fr(k + 1, 9) * (1 if k % 2 == 0 else -1) for k in range(13)]
    m = M.build_plain(shifts, M.FunctionId.exp(), 13, "P13")
    d, k = 257, 40
    rng = np.random.default_rng(11)
    sub = -0.2 * np.ones(d - 1) + 0.01 * rng.standard_normal(d - 1)
    diag = 0.4 * np.ones(d)
    sup = -0.2 * np.ones(d - 1)
    v = rng.standard_normal((d, k))
    om = oracle.OMethod.from_method(m, form)
    ref = oracle.tridiag_action(sub, diag, sup, v, om, 3)
    got = dev.tridiag_action(m, dev.TridiagMatrix(sub, diag, sup), v, 3, form)
    assert np.array_equal(got, ref)
