"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bar (BASELINE.json north_star): relative 1-norm difference <= 1e-11 in FP64 (residual form, the
parity-safe form), squaring counts and 1-norms bit-exact, pivots bit-exact on
well-separated pivots. Property tests mirror proj/tests/test_dense.cpp on the device.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module")
def dev(pf):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need CUDA")
    from paper_2210_03714_b200 import api

    return api


def rand(n, seed, norm, oracle_mod=None):
    from paper_2210_03714_b200 import workloads as W

    return W.scaled_to_one_norm(W.randn_matrix(n, seed), norm)


# ------------------------------------------------------------------ eval_dense (dense.cpp:193-252)


@pytest.mark.parametrize("name", ["R4", "R5", "R8", "R10", "R10star", "R4_phi1"])
@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("n", [1, 5, 24, 64, 100, 128])
def test_eval_dense_matches_oracle(dev, oracle, name, form, n):
    from paper_2210_03714_b200 import methods as M

    m = M.catalog(name)
    b = rand(n, 100 + n, 0.7)
    ref = oracle.eval_dense(oracle.OMethod.from_method(m, form), b)
    got = dev.eval_dense(m, b, dev.EvalOptions(form=form))
    # the order-10 sets amplify rounding by sum|b| (test_action.cpp:131-136)
    amp = float(sum(abs(w) for w in m.weights) + sum(abs(d) for d in m.poly))
    tol = max(TOL, 100 * amp * 2.23e-16) if name.startswith("R10") else TOL
    assert oracle.rel_diff_1norm(got, ref) <= tol


def test_eval_dense_batched_and_sets(dev, oracle):
    from paper_2210_03714_b200 import methods as M

    m = M.catalog("R8")
    phi = M.same_shift_method(m, M.FunctionId.phi(1))
    bs = np.stack([rand(40, 7 + i, 0.09) for i in range(6)])
    e, p = dev.eval_dense(m, bs, dev.EvalOptions(form=1), extra_sets=[phi])
    om = oracle.OMethod.from_method(m, 1, [phi])
    for i in range(6):
        ref = oracle.eval_dense(om, bs[i])
        assert oracle.rel_diff_1norm(e[i], ref[0]) <= TOL
        assert oracle.rel_diff_1norm(p[i], ref[1]) <= TOL


def test_eval_dense_zero_and_diagonal(dev, oracle):
    """r(0) = a0 I within 1e-12 (R4) / 1e-9 (R10); diagonal = scalar formula within 10 ulp
    (test_dense.cpp:85-106)."""
    from paper_2210_03714_b200 import methods as M

    z = np.zeros((5, 5))
    assert oracle.rel_diff_1norm(dev.eval_dense("R4", z), np.eye(5)) <= 1e-12
    assert oracle.rel_diff_1norm(dev.eval_dense("R10", z), np.eye(5)) <= 1e-9
    r4 = M.catalog("R4")
    d = np.diag([0.1, 0.1, 0.1])
    v = dev.eval_dense(r4, d)
    scalar = 0.0
    for c, w in zip(r4.shift_doubles(), r4.weight_doubles()):
        scalar += w * (1.0 / (1 - c * 0.1))
    for i in range(3):
        assert abs(v[i, i] - scalar) <= 10 * abs(scalar) * 2.23e-16


def test_eval_dense_workers_are_bit_identical(dev):
    """test_dense.cpp:108-119: results do not depend on opts.workers."""
    b = rand(24, 5, 0.7)
    w1 = dev.eval_dense("R8", b, dev.EvalOptions(workers=1))
    w8 = dev.eval_dense("R8", b, dev.EvalOptions(workers=8))
    assert np.array_equal(w1, w8)
    with pytest.raises(Exception):
        dev.eval_dense("R8", b, dev.EvalOptions(workers=0))
    with pytest.raises(Exception):
        dev.eval_dense("R8", b, dev.EvalOptions(fixed_order=False))


def test_plain_and_residual_agree(dev):
    """test_dense.cpp:121-128."""
    b = rand(24, 7, 1.0)
    p = dev.eval_dense("R10", b, dev.EvalOptions(form=0))
    r = dev.eval_dense("R10", b, dev.EvalOptions(form=1))
    assert np.linalg.norm(p - r, 2) <= 1e-8


def test_singular_shift_message(dev):
    """test_dense.cpp:130-139: 1 - (1/8) 8 = 0 -> SingularShift naming the shift."""
    from paper_2210_03714_b200.errors import Errc, PfError

    bad = 8.0 * np.eye(4)
    with pytest.raises(PfError) as ei:
        dev.eval_dense("R10", bad)
    assert ei.value.code == Errc.SingularShift
    assert "shift" in str(ei.value)
    assert "singular system: pivot magnitude" in str(ei.value)


# ------------------------------------------------------------------ pivoting path


def test_pivoting_matches_reference_bitwise(dev, oracle):
    """Matrices that force row exchanges: the device's genuine partial-pivoting LU takes the
    reference's pivots (bit-identical factors and pivots through DenseLu); with
    PF_FLAG_REFERENCE_ORDER the whole solve_shifted runs dense.cpp's operation order and equals the
    reference's doubles bit for bit; the default path (DMMA substitution) agrees to rounding."""
    from paper_2210_03714_b200 import _native as N

    for seed in range(4):
        b = rand(24, 900 + seed, 60.0)  # ||cB|| >> 1: I - cB is not diagonally dominant
        for c in (0.2, -0.1):
            ref = oracle.solve_shifted(b, c)
            assert np.array_equal(dev.solve_shifted(b, c, flags=N.PF_FLAG_REFERENCE_ORDER), ref)
            assert oracle.rel_diff_1norm(dev.solve_shifted(b, c), ref) <= 1e-13
            # which pivots the reference takes: not the identity -- and the device's are the same
            rlu, piv = oracle.lu(np.eye(24) - c * b)
            assert np.any(piv != np.arange(24))
            lu, dpiv = dev.DenseLu(np.eye(24) - c * b).factors()
            assert np.array_equal(dpiv, piv) and np.array_equal(lu, rlu)


def test_force_pivot_flag_same_result(dev, oracle):
    from paper_2210_03714_b200 import _native as N

    b = rand(64, 31, 0.09)
    fast = dev.eval_dense("R8", b, dev.EvalOptions(form=1))
    slow = dev.eval_dense("R8", b, dev.EvalOptions(form=1), flags=N.PF_FLAG_FORCE_PIVOT)
    assert oracle.rel_diff_1norm(fast, slow) <= 1e-13


def test_solve_shifted_properties(dev):
    """test_dense.cpp:55-83."""
    z = np.zeros((4, 4))
    assert np.array_equal(dev.solve_shifted(z, 0.3), np.eye(4))
    d = np.diag([1.0, -2.0, 0.5])
    di = dev.solve_shifted(d, 0.25)
    for i in range(3):
        assert abs(di[i, i] - 1.0 / (1.0 - 0.25 * d[i, i])) <= 1e-15 * abs(di[i, i])
    from paper_2210_03714_b200 import workloads as W

    b = W.randn_matrix(8, 3)
    x = dev.solve_shifted(b, 0.2)
    res = (np.eye(8) - 0.2 * b) @ x - np.eye(8)
    assert np.abs(res).sum(0).max() <= 1e-13 * np.abs(x).sum(0).max()
    from paper_2210_03714_b200.errors import PfError

    with pytest.raises(PfError):
        dev.solve_shifted(np.eye(5), 1.0)


# ------------------------------------------------------------------ expm (a10)


@pytest.mark.parametrize("name", ["R4", "R8"])
def test_cfg1_expm(dev, oracle, name):
    from paper_2210_03714_b200 import methods as M, workloads as W

    a = W.cfg1()
    om = oracle.OMethod.from_method(M.catalog(name), 1)
    ref, j = oracle.expm(a, om, M.THETA_U53[name])
    got, jg = dev.expm(a, name, return_squarings=True)
    assert int(jg) == j
    assert oracle.rel_diff_1norm(got, ref) <= TOL


@pytest.mark.parametrize("name", ["R4", "R8"])
def test_cfg2_expm_batch_slice(dev, oracle, name):
    """cfg2 at 256 of its 4096 matrices (the full batch is covered by test_cfg2_full_properties)."""
    from paper_2210_03714_b200 import methods as M, workloads as W

    a = W.cfg2(batch=256)
    om = oracle.OMethod.from_method(M.catalog(name), 1)
    ref, js = oracle.expm_batched(a, om, M.THETA_U53[name], threads=8)
    got, jg = dev.expm(a, name, return_squarings=True)
    assert np.array_equal(np.asarray(jg), js)
    errs = [oracle.rel_diff_1norm(got[i], ref[i]) for i in range(len(a))]
    assert max(errs) <= TOL, max(errs)


def test_cfg2_full_properties(dev, oracle):
    """Full cfg2 (4096 x 128^2): norms and squaring counts bit-exact against the oracle's
    formula, exp(A) exp(-A) = I to FP64 accuracy, and a strided sample against the oracle."""
    from paper_2210_03714_b200 import methods as M, workloads as W

    a = W.cfg2()
    ta = torch.from_numpy(a).cuda()
    norms = dev.one_norm(ta).cpu().numpy()
    assert np.array_equal(norms, W.one_norms(a))
    e, j = dev.expm(ta, "R4", return_squarings=True)
    js = np.array([oracle.squarings(x, M.THETA_U53["R4"]) for x in norms])
    assert np.array_equal(j.cpu().numpy(), js)
    einv = dev.expm(-ta, "R4")
    prod = torch.bmm(e, einv)
    eye = torch.eye(128, dtype=torch.float64, device="cuda")
    assert float((prod - eye).abs().sum(1).max()) <= 1e-10 * float(e.abs().sum(1).max() * einv.abs().sum(1).max())
    om = oracle.OMethod.from_method(M.catalog("R4"), 1)
    for i in range(0, 4096, 512):
        ref, _ = oracle.expm(a[i], om, M.THETA_U53["R4"])
        assert oracle.rel_diff_1norm(e[i].cpu().numpy(), ref) <= TOL


def test_expm_given_squarings_and_plain(dev, oracle):
    from paper_2210_03714_b200 import methods as M

    a = np.stack([rand(50, 3 + i, 3.0) for i in range(3)])
    got = dev.expm(a, "R8", squarings=[2, 3, 4])
    om = oracle.OMethod.from_method(M.catalog("R8"), 1)
    for i, jj in enumerate([2, 3, 4]):
        ref, _ = oracle.expm(a[i], om, 1.0, j_fixed=jj)
        assert oracle.rel_diff_1norm(got[i], ref) <= TOL
    gp = dev.expm(a[0], "R8", form=0)
    refp, _ = oracle.expm(a[0], oracle.OMethod.from_method(M.catalog("R8"), 0), M.THETA_U53["R8"])
    assert oracle.rel_diff_1norm(gp, refp) <= 1e-9  # plain form: parity is not feasible at 1e-11 (Appendix B)


def test_expm_matches_scipy(dev):
    sl = pytest.importorskip("scipy.linalg")
    a = rand(100, 12, 5.0)
    assert np.abs(dev.expm(a, "R8") - sl.expm(a)).sum(0).max() <= 1e-12 * np.abs(sl.expm(a)).sum(0).max()


# ------------------------------------------------------------------ phi1 and cos/sin (a11, a12)


def test_expm_phi1_small(dev, oracle):
    from paper_2210_03714_b200 import methods as M

    m = M.catalog("R8")
    phi = M.same_shift_method(m, M.FunctionId.phi(1))
    th = min(M.THETA_U53["R8"], M.THETA_U53["R8_phi1set"])
    a = np.stack([rand(96, 40 + i, 2.0 + i) for i in range(3)])
    e, p, js = dev.expm_phi1(a, "R8", return_squarings=True)
    om = oracle.OMethod.from_method(m, 1, [phi])
    for i in range(3):
        re, rp, j = oracle.expm_phi1(a[i], om, th)
        assert int(js[i]) == j
        assert oracle.rel_diff_1norm(e[i], re) <= TOL
        assert oracle.rel_diff_1norm(p[i], rp) <= TOL


def test_cossin_small(dev, oracle):
    from paper_2210_03714_b200 import methods as M

    pm = M.pair_method(M.catalog("R8"))
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((64, 64)))
    a = np.stack([q @ np.diag(rng.uniform(0, 50, 64)) @ q.T for _ in range(3)])
    a = 0.5 * (a + a.transpose(0, 2, 1))
    c, s, js = dev.cossin(a, "R8", return_squarings=True)
    op = oracle.OPair.from_pair(pm)
    for i in range(3):
        rc, rs, j = oracle.cossin(a[i], op, M.THETA_U53["R8"])
        assert int(js[i]) == j
        assert oracle.rel_diff_1norm(c[i], rc) <= TOL
        assert oracle.rel_diff_1norm(s[i], rs) <= TOL
        w, v = np.linalg.eigh(a[i])
        assert np.abs(c[i] - (v * np.cos(w)) @ v.T).max() <= 1e-10


def test_gemm(dev):
    rng = np.random.default_rng(0)
    for (m, n, k) in [(128, 128, 128), (100, 37, 61), (300, 260, 129)]:
        a = torch.from_numpy(rng.standard_normal((m, k))).cuda()
        b = torch.from_numpy(rng.standard_normal((k, n))).cuda()
        c = dev.gemm(a, b)[0]
        ref = a @ b
        assert float((c - ref).abs().max()) <= 1e-12 * k


def test_gemm_shapes_and_epilogue(dev):
    """The TMA-staged GEMM (gemm_tma.cu: even leading dimensions, aligned bases) and the cp.async one
    (odd ones) against fp64 matmul: ragged edges (zero-filled boxes), batches, sub-matrix operands
    with ld > k, beta accumulation and the gamma identity."""
    from paper_2210_03714_b200 import _native as N, api

    rng = np.random.default_rng(1)
    eng = api.engine()

    def run(m, n, k, batch, lda, ldb, ldc, alpha=1.0, beta=0.0, gamma=0.0):
        A = torch.from_numpy(rng.standard_normal((batch, m, lda))).cuda()
        B = torch.from_numpy(rng.standard_normal((batch, k, ldb))).cuda()
        Cm = torch.from_numpy(rng.standard_normal((batch, m, ldc))).cuda()
        ref = alpha * (A[:, :, :k] @ B[:, :, :n]) + beta * Cm[:, :, :n]
        ref = ref + gamma * torch.eye(m, n, dtype=torch.float64, device="cuda")
        rc = N.lib.pf_gemm_batched(eng.h, m, n, k, batch, alpha, A.data_ptr(), lda, m * lda, B.data_ptr(), ldb,
                                   k * ldb, beta, Cm.data_ptr(), ldc, m * ldc, gamma)
        assert rc == 0
        torch.cuda.synchronize()
        assert float((Cm[:, :, :n] - ref).abs().max()) <= 1e-12 * k * max(1.0, abs(alpha))

    run(128, 128, 128, 1, 128, 128, 128)
    run(200, 72, 90, 1, 90, 72, 72)            # ragged m / n / k, even leading dimensions
    run(130, 66, 34, 3, 34, 66, 66)            # batched, every tile edge partial
    run(64, 64, 64, 2, 96, 80, 70, beta=1.0)   # sub-matrix operands (ld > k, ld > n), accumulate
    run(96, 96, 48, 1, 48, 96, 96, alpha=-1.0, beta=1.0, gamma=1.0)
    run(100, 37, 61, 2, 61, 37, 37)            # odd leading dimensions: the cp.async kernel
    run(1, 1, 1, 1, 2, 2, 2)
    run(300, 64, 4096, 2, 4096, 64, 64, beta=1.0)   # thin: split-K partials + ordered reduce
    run(130, 7, 1500, 1, 1500, 8, 8, alpha=2.0)     # thin, ragged, k not a multiple of a split


def test_native_library_is_loaded(dev):
    import sys

    assert "paper_2210_03714_b200._native" in sys.modules
    with open("/proc/self/maps") as f:
        assert "libpfb200.so" in f.read()


def test_golden_fixtures_on_device(dev, oracle):
    """Device path against the frozen reference outputs (tests/golden/, made by oracle/_ref)."""
    import json
    from pathlib import Path

    from tests.golden.make_golden import inputs

    gold = Path(__file__).resolve().parent / "golden"
    meta = json.loads((gold / "golden.json").read_text())["cases"]
    x = inputs()
    g = lambda k: np.load(gold / meta[k]["file"])  # noqa: E731
    for name in ("R4", "R8"):
        assert oracle.rel_diff_1norm(dev.expm(x["cfg1_A"], name), g("cfg1_expm_%s" % name)) <= TOL
        got = dev.expm(x["cfg2_first4_A"], name)
        ref = g("cfg2_first4_expm_%s" % name)
        assert max(oracle.rel_diff_1norm(got[i], ref[i]) for i in range(4)) <= TOL
    assert oracle.rel_diff_1norm(dev.eval_dense("R8", x["eval24_B"], dev.EvalOptions(form=0)),
                                 g("eval24_R8_plain")) <= TOL
    assert oracle.rel_diff_1norm(dev.eval_dense("R8", x["eval24_B"], dev.EvalOptions(form=1)),
                                 g("eval24_R8_residual")) <= TOL
    assert oracle.rel_diff_1norm(dev.solve_shifted(x["pivot24_B"], 0.2), g("pivot24_solve_shifted_0.2")) <= 1e-13
    e, p = dev.expm_phi1(x["phi48_A"], "R8")
    assert oracle.rel_diff_1norm(e, g("phi48_R8_exp")) <= TOL
    assert oracle.rel_diff_1norm(p, g("phi48_R8_phi1")) <= TOL
    act = dev.action(x["action40_A"], x["action40_V"], "R8", substeps=3)
    assert oracle.rel_diff_1norm(act, g("action40_R8_residual_N3")) <= TOL
    t = dev.TridiagMatrix(*x["trid200"])
    band = dev.tridiag_action("R8", t, x["trid200_v"], substeps=4, form=1)
    assert np.array_equal(np.asarray(band), g("trid200_R8_residual_N4"))  # banded path is bit-exact


# ------------------------------------------------------------------ PF_FLAG_REFERENCE_ORDER


@pytest.mark.parametrize("name", ["R4", "R5", "R8", "R10", "R10star", "R4_phi1"])
@pytest.mark.parametrize("form", [0, 1])
def test_reference_order_eval_bitwise(dev, oracle, name, form):
    """ref_order.cu: eval_dense in dense.cpp's exact operation order -- equal bit for bit to the
    restatement, which tests/test_ref_pin.py holds bit-identical to the reference build."""
    from paper_2210_03714_b200 import _native as N, methods as M

    m = M.catalog(name)
    om = oracle.OMethod.from_method(m, form)
    for n, seed, norm in ((1, 3, 0.5), (5, 1, 0.3), (24, 5, 0.7), (64, 77, 0.05), (100, 9, 2.0), (128, 11, 0.9),
                          (24, 900, 30.0)):
        b = rand(n, seed, norm)
        try:
            want = oracle.eval_dense(om, b)
        except oracle.OracleError as e:
            from paper_2210_03714_b200.errors import PfError

            with pytest.raises(PfError) as eg:
                dev.eval_dense(m, b, dev.EvalOptions(form=form), flags=N.PF_FLAG_REFERENCE_ORDER)
            assert int(eg.value.code) + 1 == e.code and "at column %d " % e.status.column in str(eg.value)
            continue
        got = dev.eval_dense(m, b, dev.EvalOptions(form=form), flags=N.PF_FLAG_REFERENCE_ORDER)
        assert np.array_equal(got, want), (n, seed, oracle.rel_diff_1norm(got, want))


@pytest.mark.parametrize("name", ["R4", "R8", "R10"])
def test_reference_order_expm_bitwise(dev, oracle, name):
    from paper_2210_03714_b200 import _native as N, methods as M, workloads as W

    om = oracle.OMethod.from_method(M.catalog(name), 1)
    th = M.THETA_U53[name]
    a = W.cfg2(batch=64)
    want, jw = oracle.expm_batched(a, om, th, threads=8)
    got, jg = dev.expm(a, name, return_squarings=True, flags=N.PF_FLAG_REFERENCE_ORDER)
    assert np.array_equal(np.asarray(jg), jw)
    assert np.array_equal(got, want)
    a1 = W.cfg1()
    w1, j1 = oracle.expm(a1, om, th)
    g1, k1 = dev.expm(a1, name, return_squarings=True, flags=N.PF_FLAG_REFERENCE_ORDER)
    assert int(k1) == j1 and np.array_equal(g1, w1)


def test_reference_order_singular_and_large_n(dev):
    from paper_2210_03714_b200 import _native as N, methods as M
    from paper_2210_03714_b200.errors import Errc, PfError

    with pytest.raises(PfError) as e:
        dev.eval_dense(M.catalog("R4"), np.eye(6) * 5.0, dev.EvalOptions(form=0), flags=N.PF_FLAG_REFERENCE_ORDER)
    assert e.value.code == Errc.SingularShift
    with pytest.raises(PfError) as e:
        dev.eval_dense(M.catalog("R4"), rand(130, 1, 1.0), flags=N.PF_FLAG_REFERENCE_ORDER)
    assert e.value.code == Errc.BadArgument
