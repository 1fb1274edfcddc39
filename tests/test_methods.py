"""Host-side method tables and theta (CPU): the reference's exact known-answer tests.

Mirrors proj/tests/test_methods.cpp:26-183, test_bounds.cpp:59-71, test_rational.cpp:30-46 and the
correctly rounded doubles of SURVEY.md Appendix A.
"""
from fractions import Fraction as F

import pytest

from paper_2210_03714_b200 import methods as M
from paper_2210_03714_b200.errors import Errc, PfError


def rats(*xs):
    return [F(x) for x in xs]


def test_weight_system_for_shifts_half_to_sixth():
    """test_methods.cpp:26-37."""
    shifts = rats("1/2", "1/3", "1/4", "1/5", "1/6")
    assert M.solve_weights(shifts, M.FunctionId.exp(), 4) == rats("1/3", "-18", "128", "-625/3", "99")
    assert M.solve_weights(shifts, M.FunctionId.phi(1), 4) == rats("7/18", "-9", "128/3", "-500/9", "45/2")
    assert M.solve_weights(shifts, M.FunctionId.log_one_minus(), 4) == rats("-35/3", "153/2", "-160", "625/6", "-9")


def test_degenerate_and_invalid_weight_systems():
    """test_methods.cpp:39-48."""
    assert M.solve_weights([F(0)], M.FunctionId.exp(), 0) == [F(1)]
    with pytest.raises(PfError) as e:
        M.solve_weights(rats("1/2", "1/2", "1/4"), M.FunctionId.exp(), 2)
    assert e.value.code == Errc.DuplicateShift
    with pytest.raises(PfError) as e:
        M.solve_weights(rats("1/2", "1/3"), M.FunctionId.exp(), 2)
    assert e.value.code == Errc.LengthMismatch


def test_plain_builds_reproduce_published_sets():
    """test_methods.cpp:50-64."""
    m = M.build_plain(rats("0", "1/5", "-1/5", "1/10", "-1/10"), M.FunctionId.exp(), 4, "r4")
    assert m.weights == rats("128/3", "85/3", "20/9", "-515/9", "-15")
    assert m.processors() == 4 and m.poly == []
    p = M.build_plain(rats("0", "1/6", "-1/6", "1/12", "-1/12"), M.FunctionId.phi(1), 4, "r4p")
    assert p.weights == rats("71/5", "117/10", "7/10", "-104/5", "-24/5")
    r5 = M.build_plain(rats("0", "1/3", "1/4", "1/5", "1/6", "1/7"), M.FunctionId.exp(), 5, "r5")
    assert r5.weights == rats("-43/12", "81/32", "-704/9", "23125/48", "-810", "117649/288")


def test_hybrid_builds_reproduce_published_ten_processor_sets():
    """test_methods.cpp:66-92 (the R10 polynomial part is d0, d1, d2)."""
    shifts = [F(1, 6 + i) for i in range(1, 11)]
    m = M.build_hybrid(shifts, {9: F(-50000), 10: F(350000)}, M.FunctionId.exp(), 10, "r10star")
    assert m.weights[1] == F("3752603696192081/82668600000")
    assert m.weights[8] == -50000 and m.weights[9] == 350000
    assert len(m.poly) == 3
    assert m.poly[0] == F("-34244933704346617/14676708556800")
    alt = []
    for i in range(1, 6):
        alt += [F(-1, 6 + 2 * i), F(1, 6 + 2 * i)]
    r10 = M.build_hybrid(alt, {9: F(2000), 10: F(-3500)}, M.FunctionId.exp(), 10, "r10")
    assert r10.poly == rats("-781562376863/94371840", "-54849495983/330301440", "-8034429391/587202560")


def test_catalog_cross_checks_clean():
    """test_methods.cpp:94-110: every published constant matches the recomputation."""
    for name in M.catalog_names():
        m = M.catalog(name)
        assert m.notes == [], (name, m.notes)
        for k in range(m.order + 1):
            assert m.taylor_coeff(k) == M.series_coeff(m.function, k)
    with pytest.raises(PfError) as e:
        M.catalog("R99")
    assert e.value.code == Errc.UnknownMethod
    assert M.catalog("R4") is M.catalog("R4")  # process-lifetime cache


def test_coefficient_magnitudes():
    """test_methods.cpp:112-117: max coefficients 4.9e6 (R10star) and 4.7e4 (R10)."""
    assert 4.9e6 <= float(M.catalog("R10star").max_coefficient()) < 5.0e6
    assert 4.7e4 <= float(M.catalog("R10").max_coefficient()) < 4.8e4


def test_residual_form_is_the_same_function():
    """test_methods.cpp:161-183: a0 = d0 + sum b = 1 for exp; the residual rewrite keeps the Taylor
    coefficients."""
    for name in ("R4", "R5", "R8", "R10", "R10star"):
        m = M.catalog(name)
        r = M.to_residual_form(m)
        assert r.form == M.RESIDUAL and m.form == M.PLAIN
        assert r.constant_term() == 1
        assert M.taylor_expansion_of_method(r, 12) == M.taylor_expansion_of_method(m, 12)
        assert M.to_plain_form(r).form == M.PLAIN


def test_correctly_rounded_doubles_appendix_a():
    """SURVEY Appendix A hex table; to_double_nearest ties to even (rational.cpp:66-88)."""
    r4 = M.catalog("R4")
    assert [c.hex() for c in r4.shift_doubles()] == ["0x0.0p+0", "0x1.999999999999ap-3", "-0x1.999999999999ap-3",
                                                      "0x1.999999999999ap-4", "-0x1.999999999999ap-4"]
    assert [w.hex() for w in r4.weight_doubles()] == ["0x1.5555555555555p+5", "0x1.c555555555555p+4",
                                                       "0x1.1c71c71c71c72p+1", "-0x1.c9c71c71c71c7p+5",
                                                       "-0x1.e000000000000p+3"]
    r8 = M.catalog("R8")
    assert r8.shift_doubles()[3].hex() == "0x1.1111111111111p-3"
    assert r8.shift_doubles()[7].hex() == "0x1.47ae147ae147bp-4"
    assert r8.weight_doubles()[5].hex() == "-0x1.182875d1dc706p+11"
    # ties to even: (2^53 + 1) / 2^53 sits exactly between two doubles
    q = F(2 ** 53 + 1, 2 ** 53)
    assert M.to_double_nearest(q) == 1.0
    q = F(2 ** 53 + 3, 2 ** 53)
    assert M.to_double_nearest(q) == 1.0 + 2 * 2.0 ** -52
    # round trip of representable values (test_rational.cpp:30-38)
    import random

    rng = random.Random(7)
    for _ in range(200):
        x = (rng.random() - 0.5) * 2.0 ** rng.randint(-20, 20)
        assert M.to_double_nearest(F(x)) == x
    third = M.to_double_nearest(F(1, 3))
    import math

    assert abs(F(1, 3) - F(third)) <= abs(F(1, 3) - F(math.nextafter(third, 0)))
    assert abs(F(1, 3) - F(third)) <= abs(F(1, 3) - F(math.nextafter(third, 1)))


def test_phi1_and_pair_derived_sets_appendix_a():
    r8 = M.catalog("R8")
    phi = M.same_shift_method(r8, M.FunctionId.phi(1))
    assert phi.weights == rats("-85769/32256", "-208129/127008", "319/1323", "70838307/802816", "-5130297/802816",
                               "-1836295/7938", "606985/23814", "29585546875/195084288", "-1469921875/65028096")
    assert sum(phi.weights) == 1
    assert M.same_shift_method(M.catalog("R4"), M.FunctionId.phi(1)).weights == rats("1", "35/6", "-5/18", "-115/18",
                                                                                        "5/6")
    pm = M.pair_method(r8)
    assert pm.c2 == rats("4/625", "1/100", "4/225", "1/25")
    assert pm.cw == rats("212470703125/97542144", "-30579350/11907", "284882265/401408", "-1193765/127008")
    assert pm.sw == rats("78109375/677376", "-253268/1323", "9832671/125440", "-22271/17640")
    assert pm.a0 == 1 and pm.a1 == 1 and pm.b0 == F("-9979069/32256")
    p4 = M.pair_method(M.catalog("R4"))
    assert p4.c2 == rats("1/100", "1/25") and p4.cw == rats("-650/9", "275/9") and p4.sw == rats("-38/9", "47/9")


def test_pair_method_is_cos_sin_to_order_9():
    """Scalar check of the merged-pair formulas: |Re - cos|, |Im - sin| = O(x^9)."""
    import mpmath

    pm = M.pair_method(M.catalog("R8"))
    x = mpmath.mpf("0.01")
    with mpmath.workdps(60):
        z = [1 / (1 + mpmath.mpf(c.numerator) / c.denominator * x * x) for c in pm.c2]
        cosv = mpmath.mpf(pm.b0.numerator) / pm.b0.denominator + sum(
            mpmath.mpf(w.numerator) / w.denominator * zz for w, zz in zip(pm.cw, z))
        sinv = x * sum(mpmath.mpf(w.numerator) / w.denominator * zz for w, zz in zip(pm.sw, z))
        assert abs(cosv - mpmath.cos(x)) < 1e-24
        assert abs(sinv - mpmath.sin(x)) < 1e-23


def test_theta_reproduces_single_precision_tables():
    """test_bounds.cpp:59-71 (2^-24)."""
    t24 = 5.9604644775390625e-8
    assert abs(M.theta_taylor(5, t24) - 0.186) <= 0.002
    assert abs(M.theta_taylor(10, t24) - 1.073) <= 0.005
    assert abs(M.theta_taylor(15, t24) - 2.382) <= 0.01
    assert abs(M.theta(M.catalog("R5"), tol=t24) - 0.298) <= 0.002
    assert abs(M.theta(M.catalog("R10star"), tol=t24) - 1.734) <= 0.005
    assert M.theta(M.catalog("R10"), tol=t24) < 1.734


@pytest.mark.parametrize("name", ["R4", "R8"])
def test_theta_u53_table_is_pinned(name):
    """The shipped theta(2^-53) doubles are what the restated bound recomputes."""
    assert M.theta(M.catalog(name), tol=2.0 ** -53) == M.THETA_U53[name]
    # bisection invariants: bound(theta) <= tol < bound(theta * (1 + 1e-5))
    b = M.forward_bound(M.catalog(name), M.catalog(name).function, M.THETA_U53[name])
    assert b <= 2.0 ** -53


def test_squaring_and_substep_counts():
    assert M.squarings_for(2.0, M.THETA_U53["R4"]) == 10  # cfg1: ceil(log2(2 / 0.003079)) = 10
    assert M.squarings_for(16.0, M.THETA_U53["R8_phi1set"]) == 8  # cfg3
    assert M.substeps_for(4.0, M.THETA_U53["R8"]) == 42  # cfg4
    assert M.squarings_for(0.0, 0.1) == 0
    assert M.substeps_for(0.05, 0.1) == 1
