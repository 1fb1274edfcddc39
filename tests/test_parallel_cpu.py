"""The multi-GPU partition logic (paper_2210_03714_b200/parallel.py) on CPU: world_size 2 over gloo,
with an oracle backend standing in for the device. Deterministic mode must reproduce the
single-process evaluation bit for bit (the reference's bit-identical-across-workers contract,
dense.hpp:64-68); fast mode agrees to rounding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_03714_b200 import methods as M
from paper_2210_03714_b200 import parallel as P


class OracleBackend:
    def __init__(self):
        from oracle import oracle as O

        self.O = O

    def squarings(self, A, theta):
        return torch.tensor([self.O.squarings(self.O.one_norm(A.numpy()), theta)], dtype=torch.int32)

    def eval(self, A, j, shifts, weights, constants, form, poly=None):
        B = np.ldexp(A.numpy(), -int(j[0]))
        om = self.O.OMethod(shifts, weights if shifts else [[] for _ in constants], poly, constants, form)
        if not shifts:
            om = self.O.OMethod([], [[]] * len(constants), poly, constants, form)
        out = self.O.eval_dense(om, B)
        out = out if out.ndim == 3 else out[None]
        return [torch.from_numpy(np.ascontiguousarray(o)) for o in out]

    def ordered_sum(self, terms):
        acc = terms[0].clone()
        for t in terms[1:]:
            acc = acc + t
        return acc

    def phi1_doubling(self, E, Phi, j):
        return E, Phi

    def square_rows(self, E, r0, r1, **kw):
        e = E.numpy()
        return torch.from_numpy(self.O.mul_rows(e[r0:r1], e))

    def phi1_step_rows(self, E, Phi, r0, r1, **kw):
        O = self.O
        e, ph = E.numpy(), Phi.numpy()
        T = e[r0:r1].copy()
        T[np.arange(r1 - r0), r0 + np.arange(r1 - r0)] += 1.0
        return torch.from_numpy(O.mul_rows(e[r0:r1], e)), torch.from_numpy(O.mul_rows(T, ph) * 0.5)


class OracleActionOperator:
    """Restates the oracle's block action per owned shift (oracle/pf_oracle.c pfo_action)."""

    def __init__(self, A, m, substeps, form, owned):
        from oracle import oracle as O

        self.O = O
        self.m = m
        self.form = form
        a = A.numpy()
        self.B = a * (1.0 / substeps)
        n = a.shape[0]
        self.own = [i for i in owned]
        self.facs = {}
        for i in self.own:
            c = m.shift_doubles()[i]
            if c != 0.0:
                mm = self.B * (-c)
                mm[np.arange(n), np.arange(n)] += 1.0
                self.facs[i] = O.lu(mm)
        self.terms = len(self.own)
        hybrid = len(m.poly) == 3
        self.poly_terms = (1 if (form == M.RESIDUAL or hybrid) else 0) + (1 if hybrid else 0)

    def apply(self, X, include_poly=True, with_terms=False):
        O, m = self.O, self.m
        x = X.numpy()
        hybrid = len(m.poly) == 3
        bv = O.mul_rect(self.B, x) if (self.form == M.RESIDUAL or hybrid) else None
        ts = []
        for i in self.own:
            c, w = m.shift_doubles()[i], m.weight_doubles()[i]
            if self.form == M.PLAIN:
                xi = x.copy() if c == 0.0 else O.lu_solve_matrix(*self.facs[i], x)
            else:
                xi = O.lu_solve_matrix(*self.facs[i], c * bv)
            ts.append(xi * w)
        if include_poly and (self.form == M.RESIDUAL or hybrid):
            cst = M.to_double_nearest(m.constant_term()) if self.form == M.RESIDUAL else M.to_double_nearest(m.poly[0])
            ts.append(cst * x)
            if hybrid:
                d1, d2 = M.to_double_nearest(m.poly[1]), M.to_double_nearest(m.poly[2])
                b2v = O.mul_rect(self.B, bv)
                ts.append(d1 * bv + d2 * b2v)
        terms = torch.from_numpy(np.stack(ts)) if ts else torch.zeros((0,) + x.shape)
        out = terms[0].clone()
        for t in terms[1:]:
            out = out + t
        return (out, terms) if with_terms else out

    def close(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_03714_b200 import workloads as W

        if case == "square":
            rng = np.random.default_rng(12)
            E = torch.from_numpy(np.eye(19) + 0.1 * rng.standard_normal((19, 19)))
            e2 = P.square_chain_distributed(E, 4, None, OracleBackend())
            if rank == 0:
                q.put([e2.numpy()])
        elif case == "doubling":
            rng = np.random.default_rng(11)
            E = torch.from_numpy(np.eye(21) + 0.1 * rng.standard_normal((21, 21)))
            Phi = torch.from_numpy(np.eye(21) + 0.05 * rng.standard_normal((21, 21)))
            e2, p2 = P.phi1_doubling_distributed(E, Phi, 3, None, OracleBackend())
            if rank == 0:
                q.put([e2.numpy(), p2.numpy()])
        elif case.startswith("eval"):
            det = case.endswith("det")
            m = M.catalog("R8")
            phi = M.same_shift_method(m, M.FunctionId.phi(1))
            A = torch.from_numpy(W.scaled_to_one_norm(W.randn_matrix(24, 3), 3.0))
            be = OracleBackend()
            j = be.squarings(A, M.THETA_U53["R8_phi1set"])
            res = P.eval_sets_sharded(A, j, m, [phi], M.RESIDUAL, det, None, be)
            if rank == 0:
                q.put([r.numpy() for r in res])
        else:
            det = case.endswith("det")
            name = "R10" if "hybrid" in case else "R8"
            form = M.PLAIN if "plain" in case else M.RESIDUAL
            a = W.randn_matrix(30, 40) / np.sqrt(30) - 2.0 * np.eye(30)
            a *= 1.5 / W.one_norm(a)
            V = torch.from_numpy(W.randn(41, 30 * 3).reshape(30, 3))
            out = P.action_sharded(torch.from_numpy(a), V, name, 4, form, det, None, OracleActionOperator,
                                   OracleBackend().ordered_sum)
            if rank == 0:
                q.put([out.numpy()])
    finally:
        dist.destroy_process_group()


def _run(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    return res


def test_term_partition():
    m = M.catalog("R8")
    assert P.term_indices(m, M.RESIDUAL) == list(range(1, 9))
    assert P.term_indices(m, M.PLAIN) == list(range(9))
    # residual R8: the units are the (c, -c) pairs (1,2) (3,4) (5,6) (7,8), pair u -> rank u mod G
    assert P.term_units(m, M.RESIDUAL) == [[1, 2], [3, 4], [5, 6], [7, 8]]
    parts = [P.owned_terms(m, M.RESIDUAL, r, 3) for r in range(3)]
    assert sorted(sum(parts, [])) == list(range(1, 9))
    assert parts == [[1, 2, 7, 8], [3, 4], [5, 6]]
    # plain form: single terms (the zero shift is a term)
    assert P.term_units(m, M.PLAIN) == [[i] for i in range(9)]
    assert P.owned_terms(m, M.PLAIN, 0, 3) == [0, 3, 6]
    # more ranks than pairs: single shifts, so R8 keeps 8 GPUs busy (one shift each); 4 ranks: pairs
    assert P.term_units(m, M.RESIDUAL, 8) == [[i] for i in range(1, 9)]
    assert [P.owned_terms(m, M.RESIDUAL, r, 8) for r in range(8)] == [[i] for i in range(1, 9)]
    assert [P.owned_terms(m, M.RESIDUAL, r, 4) for r in range(4)] == [[1, 2], [3, 4], [5, 6], [7, 8]]
    # deterministic mode: one shift per unit regardless of the pairing
    assert P.owned_terms(m, M.RESIDUAL, 0, 3, per_shift=True) == [1, 4, 7]


@pytest.mark.parametrize("world", [2, 5])
def test_sharded_eval_deterministic_is_bit_identical(world):
    """world 5 > 4 pairs: single shifts per rank; the root-only gather + ascending sum still equals
    the single-process evaluation bit for bit."""
    from oracle import oracle as O
    from paper_2210_03714_b200 import workloads as W

    e2 = _run("eval_det", world)
    m = M.catalog("R8")
    phi = M.same_shift_method(m, M.FunctionId.phi(1))
    a = W.scaled_to_one_norm(W.randn_matrix(24, 3), 3.0)
    j = O.squarings(O.one_norm(a), M.THETA_U53["R8_phi1set"])
    ref = O.eval_dense(O.OMethod.from_method(m, M.RESIDUAL, [phi]), np.ldexp(a, -j))
    assert np.array_equal(e2[0], ref[0]) and np.array_equal(e2[1], ref[1])


@pytest.mark.parametrize("world", [2, 5])
def test_sharded_eval_fast_agrees(world):
    from oracle import oracle as O
    from paper_2210_03714_b200 import workloads as W

    e2 = _run("eval_fast", world)
    m = M.catalog("R8")
    phi = M.same_shift_method(m, M.FunctionId.phi(1))
    a = W.scaled_to_one_norm(W.randn_matrix(24, 3), 3.0)
    j = O.squarings(O.one_norm(a), M.THETA_U53["R8_phi1set"])
    ref = O.eval_dense(O.OMethod.from_method(m, M.RESIDUAL, [phi]), np.ldexp(a, -j))
    assert O.rel_diff_1norm(e2[0], ref[0]) <= 1e-13 and O.rel_diff_1norm(e2[1], ref[1]) <= 1e-13


@pytest.mark.parametrize("case", ["action_det", "action_plain_det", "action_hybrid_det"])
def test_sharded_action_deterministic_is_bit_identical(case):
    from oracle import oracle as O
    from paper_2210_03714_b200 import workloads as W

    out = _run(case, 2)[0]
    name = "R10" if "hybrid" in case else "R8"
    form = M.PLAIN if "plain" in case else M.RESIDUAL
    a = W.randn_matrix(30, 40) / np.sqrt(30) - 2.0 * np.eye(30)
    a *= 1.5 / W.one_norm(a)
    v = W.randn(41, 30 * 3).reshape(30, 3)
    ref = O.action(a, v, O.OMethod.from_method(M.catalog(name), form), 4)
    assert np.array_equal(out, ref)


def test_sharded_action_fast_agrees():
    from oracle import oracle as O
    from paper_2210_03714_b200 import workloads as W

    out = _run("action_fast", 2)[0]
    a = W.randn_matrix(30, 40) / np.sqrt(30) - 2.0 * np.eye(30)
    a *= 1.5 / W.one_norm(a)
    v = W.randn(41, 30 * 3).reshape(30, 3)
    ref = O.action(a, v, O.OMethod.from_method(M.catalog("R8"), M.RESIDUAL), 4)
    assert O.rel_diff_1norm(out, ref) <= 1e-13


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_doubling_is_bit_identical(world):
    """f1: the row-split phi1 doubling (all-gather per step) equals the single-process recurrence."""
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    E = np.eye(21) + 0.1 * rng.standard_normal((21, 21))
    Phi = np.eye(21) + 0.05 * rng.standard_normal((21, 21))
    e_ref, p_ref = O.phi1_doubling(E, Phi, 3)
    e2, p2 = _run("doubling", world)
    assert np.array_equal(e2, e_ref) and np.array_equal(p2, p_ref)


def test_distributed_square_chain_is_bit_identical():
    """f1 for expm: the row-split squaring chain over gloo (world 2) equals repeated E E."""
    from oracle import oracle as O

    rng = np.random.default_rng(12)
    E = np.eye(19) + 0.1 * rng.standard_normal((19, 19))
    ref = E
    for _ in range(4):
        ref = O.mul(ref, ref)
    (e2,) = _run("square", 2)
    assert np.array_equal(e2, ref)
