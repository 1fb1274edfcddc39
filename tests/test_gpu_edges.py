"""Edge cases of the evaluators on the B200: empty batches, the 128 / 129 boundary between the fused
kernel and the large engine, leading dimensions larger than n through the C ABI, and the small
kernel's pair mode declining (non-dominant shifted systems) -- which must then be the per-shift
path bit for bit."""
import ctypes as C

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


def _mat(n, seed, norm):
    from paper_2210_03714_b200 import workloads as W

    return W.scaled_to_one_norm(W.randn_matrix(n, seed), norm)


def test_empty_batch(dev):
    a = torch.zeros((0, 128, 128), dtype=torch.float64, device="cuda")
    assert dev.expm(a, "R4").shape == (0, 128, 128)
    b = torch.zeros((0, 200, 200), dtype=torch.float64, device="cuda")
    assert dev.expm(b, "R8").shape == (0, 200, 200)


@pytest.mark.parametrize("n", [127, 128, 129])
@pytest.mark.parametrize("name", ["R4", "R8"])
def test_expm_around_the_engine_boundary(dev, oracle, n, name):
    from paper_2210_03714_b200 import methods as M

    a = _mat(n, 40 + n, 5.0)
    om = oracle.OMethod.from_method(M.catalog(name), 1)
    ref, j_ref = oracle.expm(a, om, M.THETA_U53[name])
    got, j = dev.expm(a, name, return_squarings=True)
    assert oracle.rel_diff_1norm(got, ref) <= TOL
    assert int(np.asarray(j).reshape(-1)[0]) == int(np.asarray(j_ref).reshape(-1)[0])


def test_leading_dimension_larger_than_n(dev, oracle):
    """pf_expm_batched on the top-left n x n of an (n + 8)-wide buffer, output with ldo = n + 3."""
    from paper_2210_03714_b200 import _native as N, methods as M

    n, lda, ldo = 128, 136, 131
    a = _mat(n, 7, 3.0)
    buf = torch.zeros((n, lda), dtype=torch.float64)
    buf[:, :n] = torch.from_numpy(a)
    dA = buf.cuda()
    dO = torch.full((n, ldo), np.nan, dtype=torch.float64, device="cuda")
    pk = dev.PackedMethod(M.catalog("R4"), 1)
    st = N.PfStatus()
    rc = N.lib.pf_expm_batched(dev.engine().h, pk.ptr(), M.THETA_U53["R4"], n, 1, dA.data_ptr(), lda, n * lda,
                               None, None, dO.data_ptr(), ldo, n * ldo, 0, C.byref(st))
    assert rc == 0
    ref, _ = oracle.expm(a, oracle.OMethod.from_method(M.catalog("R4"), 1), M.THETA_U53["R4"])
    got = dO[:, :n].cpu().numpy()
    assert oracle.rel_diff_1norm(got, ref) <= TOL
    assert torch.isnan(dO[:, n:]).all()  # nothing written past the n columns


def test_small_pair_mode_declines_to_the_per_shift_path(dev, oracle):
    """n = 128, no scaling, ||B||_1 large: the I -/+ cB are not dominant, the fused kernel declines
    the pair and runs the reference's per-shift (pivoting) path: identical bits to PF_FLAG_PER_SHIFT."""
    from paper_2210_03714_b200 import _native as N, methods as M

    m = M.catalog("R8")
    b = _mat(128, 77, 60.0)
    opts = dev.EvalOptions(form=1)
    got = dev.eval_dense(m, b, opts)
    per_shift = dev.eval_dense(m, b, opts, flags=N.PF_FLAG_PER_SHIFT)
    assert np.array_equal(np.asarray(got), np.asarray(per_shift))
    ref = oracle.eval_dense(oracle.OMethod.from_method(m, 1), b)
    assert oracle.rel_diff_1norm(got, ref) <= 1e-9  # a large-norm direct evaluation: conditioning-limited
    # a mixed batch: the small matrix takes the pair path, the large one declines; each equals its own call
    small = _mat(128, 78, 0.05)
    both = dev.eval_dense(m, np.stack([small, b]), opts)
    assert np.array_equal(np.asarray(both[1]), np.asarray(got))
    assert np.array_equal(np.asarray(both[0]), np.asarray(dev.eval_dense(m, small, opts)))
