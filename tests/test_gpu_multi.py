"""pf_context_create_multi / pf_eval_multi_gpu: one matrix, its shifts
partitioned over the devices of ONE process, one NCCL exchange before the recurrence.

Only one GPU is available here. [0] runs the real NCCL path as a one-rank communicator
(ncclCommInitAll, ncclBroadcast / ncclReduce / ncclSend+ncclRecv); repeated ids [0, 0, ...] run the
same partition, per-device threads and reduction order with peer copies. Deterministic mode must be
bit-identical for every device count (the reference's bit-identical-workers contract,
test_dense.cpp:108-119), fast mode equal to rounding; both against the oracle at 1e-11."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11
GROUPS = [[0], [0, 0], [0, 0, 0], [0, 0, 0, 0], [0] * 8]


@pytest.fixture(scope="module")
def dev(pf):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need CUDA")
    from paper_2210_03714_b200 import api

    return api


@pytest.fixture(scope="module")
def groups(dev):
    gs = {len(g): dev.MultiDevice(g) for g in GROUPS}
    yield gs
    for g in gs.values():
        g.close()


def rand(n, seed, norm):
    from paper_2210_03714_b200 import workloads as W

    return W.scaled_to_one_norm(W.randn_matrix(n, seed), norm)


def test_one_rank_group_uses_nccl(groups):
    assert groups[1].uses_nccl
    assert not groups[2].uses_nccl  # repeated ids: peer copies


@pytest.mark.parametrize("n", [64, 128, 200])
@pytest.mark.parametrize("name,form", [("R8", 1), ("R4", 1), ("R8", 0), ("R10", 1), ("R10star", 0)])
def test_eval_dense_partitioned(dev, oracle, groups, n, name, form):
    from paper_2210_03714_b200 import methods as M

    m = M.catalog(name)
    b = rand(n, 500 + n, 0.08 if form == 0 else 0.5)
    ref = oracle.eval_dense(oracle.OMethod.from_method(m, form), b)
    amp = float(sum(abs(w) for w in m.weights) + sum(abs(d) for d in m.poly))
    tol = max(TOL, 100 * amp * 2.23e-16) if (name.startswith("R10") or form == 0) else TOL
    det = [groups[g].eval_dense(m, b, form=form, deterministic=True) for g in sorted(groups)]
    for d in det[1:]:
        assert np.array_equal(d, det[0])  # any device count, same bits
    assert oracle.rel_diff_1norm(det[0], ref) <= tol
    for g in sorted(groups):
        fast = groups[g].eval_dense(m, b, form=form, deterministic=False)
        assert oracle.rel_diff_1norm(fast, ref) <= tol
    # one device: the fast path is the single-device evaluator itself
    one = dev.eval_dense(m, b, dev.EvalOptions(form=form))
    assert np.array_equal(groups[1].eval_dense(m, b, form=form, deterministic=False), one)


@pytest.mark.parametrize("name", ["R4", "R8"])
@pytest.mark.parametrize("n", [96, 256])
def test_expm_partitioned(dev, oracle, groups, name, n):
    from paper_2210_03714_b200 import methods as M

    a = rand(n, 900 + n, 3.0)
    ref, j = oracle.expm(a, oracle.OMethod.from_method(M.catalog(name), 1), M.THETA_U53[name])
    det = [groups[g].expm(name, a, return_squarings=True) for g in sorted(groups)]
    for e, jj in det:
        assert jj == j
        assert np.array_equal(e, det[0][0])
    assert oracle.rel_diff_1norm(det[0][0], ref) <= TOL
    for g in sorted(groups):
        assert oracle.rel_diff_1norm(groups[g].expm(name, a, deterministic=False), ref) <= TOL


def test_expm_phi1_partitioned(dev, oracle, groups):
    from paper_2210_03714_b200 import methods as M

    r8 = M.catalog("R8")
    phi = M.same_shift_method(r8, M.FunctionId.phi(1))
    a = rand(160, 77, 5.0)
    th = min(M.THETA_U53["R8"], M.THETA_U53["R8_phi1set"])
    re, rp, rj = oracle.expm_phi1(a, oracle.OMethod.from_method(r8, 1, [phi]), th)
    outs = [groups[g].expm_phi1("R8", a, return_squarings=True) for g in sorted(groups)]
    for e, p, j in outs:
        assert j == rj
        assert np.array_equal(e, outs[0][0]) and np.array_equal(p, outs[0][1])
    assert oracle.rel_diff_1norm(outs[0][0], re) <= TOL and oracle.rel_diff_1norm(outs[0][1], rp) <= TOL


def test_singular_shift_reports_global_index(dev, groups):
    from paper_2210_03714_b200 import methods as M
    from paper_2210_03714_b200.errors import Errc, PfError

    b = np.eye(8) * 5.0  # 1 - c 5 = 0 at c = 1/5, shift index 2 of R4 (0, 1/5, -1/5, 1/10, -1/10)
    for g in sorted(groups):
        for det in (True, False):
            with pytest.raises(PfError) as e:
                groups[g].eval_dense(M.catalog("R4"), b, form=0, deterministic=det)
            assert e.value.code == Errc.SingularShift
            assert str(e.value).startswith("shift 2: singular system")
