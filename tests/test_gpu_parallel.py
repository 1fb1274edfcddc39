"""Multi-GPU building blocks on one B200. The rank partition is emulated sequentially in one process
(no concurrently waiting kernels): the deterministic mode's ordered reduction of every rank's terms
must equal the single-GPU evaluation bit for bit, for the small (n <= 128) and large engines."""
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


def _a(n, seed, norm):
    from paper_2210_03714_b200 import workloads as W

    return torch.from_numpy(W.scaled_to_one_norm(W.randn_matrix(n, seed), norm)).cuda()


@pytest.mark.parametrize("n", [100, 128, 200])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_emulated_shift_partition_is_bit_identical(dev, n, world):
    from paper_2210_03714_b200 import methods as M, parallel as P

    m = M.catalog("R8")
    phi = M.same_shift_method(m, M.FunctionId.phi(1))
    A = _a(n, 9, 6.0)
    be = P.CudaBackend()
    j = be.squarings(A, M.THETA_U53["R8_phi1set"])
    # single GPU, all shifts in one call, per-shift evaluation (the deterministic mode's reference;
    # the default merges (c, -c) pairs into one solve)
    from paper_2210_03714_b200 import _native as N

    full = dev.eval_dense_raw(A, m.shift_doubles(), [m.weight_doubles(), phi.weight_doubles()],
                              [1.0, 1.0], M.RESIDUAL, squarings=j, flags=N.PF_FLAG_PER_SHIFT)
    paired = dev.eval_dense_raw(A, m.shift_doubles(), [m.weight_doubles(), phi.weight_doubles()],
                                [1.0, 1.0], M.RESIDUAL, squarings=j)
    for s in range(2):  # the pair path agrees to rounding
        assert float((paired[s] - full[s]).abs().sum(0).max()) <= 1e-12 * float(full[s].abs().sum(0).max())
    # every rank's terms, gathered and summed in ascending shift order
    terms = {}
    for r in range(world):
        for i in P.owned_terms(m, M.RESIDUAL, r, world):
            res = be.eval(A, j, [m.shift_doubles()[i]], [[m.weight_doubles()[i]], [phi.weight_doubles()[i]]],
                          [0.0, 0.0], M.RESIDUAL)
            terms[i] = res
    for s in range(2):
        ts = [terms[i][s] for i in sorted(terms)]
        ts += be.eval(A, j, [], [[]], [1.0], M.RESIDUAL)
        got = be.ordered_sum(ts)
        assert torch.equal(got, full[s])


def test_sharded_world1_matches_expm_phi1(dev):
    from paper_2210_03714_b200 import parallel as P

    from paper_2210_03714_b200 import _native as N

    A = _a(96, 4, 5.0)
    E, Phi = P.expm_phi1_sharded(A, "R8", deterministic=True)
    E2, Phi2 = dev.expm_phi1(A, "R8", flags=N.PF_FLAG_PER_SHIFT)
    assert torch.equal(E, E2) and torch.equal(Phi, Phi2)
    Ef, Phif = P.expm_phi1_sharded(A, "R8", deterministic=False)
    assert float((Ef - E2).abs().max()) <= 1e-13 * float(E2.abs().max())


@pytest.mark.parametrize("n", [96, 200])
def test_action_operator_and_partition(dev, n):
    from paper_2210_03714_b200 import methods as M, parallel as P, workloads as W

    a = W.randn_matrix(n, 40) / np.sqrt(n) - 2.0 * np.eye(n)
    a *= 1.5 / W.one_norm(a)
    A = torch.from_numpy(a).cuda()
    V = torch.from_numpy(W.randn(41, n * 4).reshape(n, 4)).cuda()
    nsub = 5
    from paper_2210_03714_b200 import _native as N

    # the deterministic partition reproduces the per-shift evaluation; the default pf_action_block
    # merges (c, -c) pairs (equal to rounding)
    ref = dev.action(A, V, "R8", substeps=nsub, flags=N.PF_FLAG_PER_SHIFT)
    paired = dev.action(A, V, "R8", substeps=nsub)
    assert float((paired - ref).abs().sum(0).max()) <= 1e-12 * float(ref.abs().sum(0).max())
    # one operator owning everything == pf_action_block
    X = P.action_sharded(A, V, "R8", nsub, M.RESIDUAL, deterministic=True)
    assert torch.equal(X, ref)
    # emulated 2-rank deterministic substeps
    m = M.catalog("R8")
    ops = [dev.ActionOperator(A, m, nsub, M.RESIDUAL, owned=P.owned_terms(m, M.RESIDUAL, r, 2)) for r in range(2)]
    X = V.clone()
    for _ in range(nsub):
        parts = []
        poly = None
        for r, op in enumerate(ops):
            _, terms = op.apply(X, include_poly=True, with_terms=True)
            for q, i in enumerate(P.owned_terms(m, M.RESIDUAL, r, 2)):
                parts.append((i, terms[q]))
            poly = [terms[op.terms + q] for q in range(op.poly_terms)]
        parts.sort(key=lambda p: p[0])
        X = dev.ordered_sum([p[1] for p in parts] + poly)
    assert torch.equal(X, ref)
    for op in ops:
        op.close()


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_distributed_doubling_is_bit_identical(dev, world):
    """f1 on one B200: every rank's row block of each doubling step (the all-gather emulated by a
    concatenation in rank order) reproduces pf_phi1_doubling bit for bit."""
    from paper_2210_03714_b200 import parallel as P

    n = 300
    g = torch.Generator().manual_seed(5)
    E0 = (torch.eye(n, dtype=torch.float64) + 0.02 * torch.randn(n, n, generator=g, dtype=torch.float64)).cuda()
    P0 = (torch.eye(n, dtype=torch.float64) + 0.01 * torch.randn(n, n, generator=g, dtype=torch.float64)).cuda()
    j = 4
    E_ref, P_ref = dev.phi1_doubling(E0.clone(), P0.clone(), torch.tensor([j], dtype=torch.int32, device="cuda"))
    be = P.CudaBackend()
    rows = -(-n // world)
    E, Phi = E0.clone(), P0.clone()
    for _ in range(j):
        blocks = [be.phi1_step_rows(E, Phi, min(n, r * rows), min(n, (r + 1) * rows)) for r in range(world)]
        E = torch.cat([b[0] for b in blocks], 0)
        Phi = torch.cat([b[1] for b in blocks], 0)
    assert torch.equal(E, E_ref) and torch.equal(Phi, P_ref)


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_distributed_square_and_cossin(dev, world):
    """f1 for expm's squaring chain and the cos/sin double angle: the row split reproduces
    pf_square_chain and pf_cossin_doubling bit for bit."""
    from paper_2210_03714_b200 import parallel as P

    n = 256
    g = torch.Generator().manual_seed(9)
    E0 = (torch.eye(n, dtype=torch.float64) + 0.02 * torch.randn(n, n, generator=g, dtype=torch.float64)).cuda()
    S0 = (0.05 * torch.randn(n, n, generator=g, dtype=torch.float64)).cuda()
    j = 3
    jt = torch.tensor([j], dtype=torch.int32, device="cuda")
    be = P.CudaBackend()
    rows = -(-n // world)
    ref = dev.square_chain(E0.clone(), jt)
    E = E0.clone()
    for _ in range(j):
        E = torch.cat([be.square_rows(E, min(n, r * rows), min(n, (r + 1) * rows)) for r in range(world)], 0)
    assert torch.equal(E, ref)
    from paper_2210_03714_b200 import _native as N

    C_ref, S_ref = E0.clone(), S0.clone()
    rc = N.lib.pf_cossin_doubling(dev.engine().h, n, 1, jt.data_ptr(), C_ref.data_ptr(), S_ref.data_ptr())
    assert rc == 0
    Cm, S = E0.clone(), S0.clone()
    for _ in range(j):
        blocks = [be.cossin_step_rows(Cm, S, min(n, r * rows), min(n, (r + 1) * rows)) for r in range(world)]
        Cm = torch.cat([b[0] for b in blocks], 0)
        S = torch.cat([b[1] for b in blocks], 0)
    assert torch.equal(Cm, C_ref) and torch.equal(S, S_ref)
