"""GPU parity at the full BASELINE configs (BASELINE.json configs[1..4]) against the CPU checker.

* cfg2 (4096 x 128^2, R4 and R8): every matrix against THE REFERENCE BUILD (oracle/_ref:
  eval_dense + DenseMatrix::mul from /root/reference compiled unmodified) when present, else the
  restatement pinned to it bit for bit (tests/test_ref_pin.py); squaring counts exact.
* cfg3 (exp and phi1 of one 4096^2, R8 shifts, j = 8): the full matrix against the restatement's
  exp+phi1 (threaded over shifts / solve columns / product rows; no element's operation order
  changes), both outputs.
* cfg4: n = 4096, k = 64, N = 42 substeps against the dense block action restatement (factor once,
  assemble_action order); the full 16384^2 x 64 action against torch.linalg.matrix_exp(tA) V.
* cfg5 (cos/sin of 256 x 512^2): 32 matrices spread over the batch against the restatement's
  C^2 - S^2 / 2SC composition; squaring counts exact for the whole batch.
Bar: relative 1-norm difference <= 1e-11 (north_star), rel_diff_1norm of test_dense.cpp:24-28.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


def threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


@pytest.fixture(scope="module")
def dev(pf):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need CUDA")
    from paper_2210_03714_b200 import api

    return api


def rel_rows(got, ref):
    """rel_diff_1norm per matrix of a batch (max column sum of |diff| / of |ref|)."""
    d = np.abs(got - ref).sum(axis=-2).max(axis=-1)
    r = np.abs(ref).sum(axis=-2).max(axis=-1)
    return d / r


@pytest.mark.parametrize("name", ["R4", "R8"])
def test_cfg2_full_batch_vs_reference(dev, oracle, name):
    from oracle import ref as R
    from paper_2210_03714_b200 import methods as M, workloads as W

    a = W.cfg2()
    th = M.THETA_U53[name]
    got, jg = dev.expm(torch.from_numpy(a).cuda(), name, return_squarings=True)
    got, jg = got.cpu().numpy(), jg.cpu().numpy()
    if R.available():
        want, jw = R.expm_batched(R.RefMethod.catalog(name), a, th, M.RESIDUAL, threads=threads())
    else:
        want, jw = oracle.expm_batched(a, oracle.OMethod.from_method(M.catalog(name), 1), th, threads=threads())
    assert np.array_equal(jg, jw)
    errs = rel_rows(got, want)
    assert errs.shape == (4096,)
    assert errs.max() <= TOL, (int(errs.argmax()), float(errs.max()))


def test_cfg3_full_vs_oracle(dev, oracle):
    from paper_2210_03714_b200 import methods as M, workloads as W

    a = W.cfg3()
    r8 = M.catalog("R8")
    phi = M.same_shift_method(r8, M.FunctionId.phi(1))
    th = min(M.THETA_U53["R8"], M.THETA_U53["R8_phi1set"])
    e, p, j = dev.expm_phi1(torch.from_numpy(a).cuda(), "R8", return_squarings=True)
    e, p = e.cpu().numpy(), p.cpu().numpy()
    re, rp, rj = oracle.expm_phi1(a, oracle.OMethod.from_method(r8, 1, [phi]), th, workers=max(threads(), 8))
    assert int(j) == rj == 8
    assert oracle.rel_diff_1norm(e, re) <= TOL
    assert oracle.rel_diff_1norm(p, rp) <= TOL


def test_cfg4_reduced_vs_oracle(dev, oracle):
    """cfg4's construction at n = 4096, k = 64 with the full-size substep count N = 42."""
    from paper_2210_03714_b200 import methods as M, workloads as W

    a, v = W.cfg4(n=4096, k=64)
    n_sub = M.substeps_for(W.one_norm(a), M.THETA_U53["R8"])
    assert n_sub == 42
    got = dev.action(torch.from_numpy(a).cuda(), torch.from_numpy(v).cuda(), "R8", substeps=n_sub).cpu().numpy()
    want = oracle.action(a, v, oracle.OMethod.from_method(M.catalog("R8"), 1), n_sub, workers=max(threads(), 8))
    assert oracle.rel_diff_1norm(got, want) <= TOL


def test_cfg4_full_vs_referee(dev):
    """Full cfg4 (16384^2, k = 64, N = 42): exp(tA) V against torch.linalg.matrix_exp(tA) @ V."""
    from paper_2210_03714_b200 import methods as M, workloads as W

    a, v = W.cfg4()
    n_sub = M.substeps_for(W.one_norm(a), M.THETA_U53["R8"])
    dA, dV = torch.from_numpy(a).cuda(), torch.from_numpy(v).cuda()
    del a
    got = dev.action(dA, dV, "R8", substeps=n_sub)
    ref = torch.linalg.matrix_exp(dA) @ dV
    rel = float((got - ref).abs().sum(0).max() / ref.abs().sum(0).max())
    assert n_sub == 42 and rel <= 1e-12, rel


def test_cfg5_vs_oracle(dev, oracle):
    from paper_2210_03714_b200 import methods as M, workloads as W

    a = W.cfg5()
    c, s, j = dev.cossin(torch.from_numpy(a).cuda(), "R8", return_squarings=True)
    j = j.cpu().numpy()
    pm = oracle.OPair.from_pair(M.pair_method(M.catalog("R8")))
    th = M.THETA_U53["R8"]
    norms = W.one_norms(a)
    assert np.array_equal(j, [oracle.squarings(x, th) for x in norms])
    idx = np.arange(0, 256, 8)
    rc, rs, rj = oracle.cossin_batched(a[idx], pm, th, threads=threads())
    assert np.array_equal(j[idx], rj)
    c, s = c[idx].cpu().numpy(), s[idx].cpu().numpy()
    ec, es = rel_rows(c, rc), rel_rows(s, rs)
    assert ec.max() <= TOL and es.max() <= TOL, (float(ec.max()), float(es.max()))
