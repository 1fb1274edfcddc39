"""Multi-GPU partition of the hot path: one process per GPU, torch.distributed
(NCCL over NVLink on GPUs, gloo in the CPU tests) for the plumbing.

* Single-matrix configs (cfg3 exp+phi1, cfg4 action): the s independent resolvents are the units.
  Term t (every nonzero shift; plus the zero shift in plain form) belongs to rank t mod G -- the
  B200 analogue of the reference's one-thread-per-shift parallel_for_index (worker_pool.hpp:16-44).
  There is exactly one exchange per evaluation (cfg3) or per substep (cfg4):
    fast           each rank sums its own weighted terms; NCCL reduce / all-reduce (sum) -- the
                   addition order depends on G, like any NCCL sum;
    deterministic  each rank ships its weighted terms; every term is then added in ascending shift
                   index (pf_ordered_sum), which reproduces the single-GPU per-shift evaluation
                   (PF_FLAG_PER_SHIFT) bit for bit for any G -- the reference's "bit-identical for
                   any worker count" contract (dense.hpp:64-68). The default single-GPU evaluation
                   merges (c, -c) shift pairs into one solve (faster, equal up to rounding), so it
                   is not the deterministic mode's bit-level reference.
  Units are (c, -c) pairs when the method's nonzero shifts pair up (every frac4/frac8 set), single
  terms otherwise, so that a rank evaluates whole pairs in the fast mode.
  The polynomial / constant part is added once. The doubling recurrence runs on the root after the
  reduce ("NCCL-reduce the weighted results over NVLink before squaring"), or, with
  distributed_doubling=True, on every rank: each product of the recurrence is
  split by rows (rank r computes rows [r R, (r + 1) R) of (E + I) Phi / 2 and E E) and the row
  blocks are all-gathered after each step. A row of a product depends on that row of the left
  factor only, so every element is computed exactly as the single-GPU product computes it: the
  result is bit-identical to the root-only doubling for any G.
* Batched configs (cfg2, cfg5): independent matrices, sharded by batch with no data-path collective
  (bench.py runs one batch per rank: weak scaling).

The partition logic is backend-agnostic: `CudaBackend` drives the C ABI on the local GPU,
tests/test_parallel_cpu.py runs the same code with an oracle backend over gloo.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from .methods import (PLAIN, RESIDUAL, THETA_U53, FractionMethod, FunctionId, catalog, same_shift_method,
                      to_double_nearest)


def term_indices(method: FractionMethod, form: int) -> List[int]:
    """Shift indices that produce a term (eval_dense: residual zero shifts fold into a_0)."""
    return [i for i, c in enumerate(method.shifts) if c != 0 or form == PLAIN]


def term_units(method: FractionMethod, form: int, world: int = 1) -> List[List[int]]:
    """Partition units: (c, -c) shift pairs (residual form, every nonzero shift paired) while there
    are at least as many pairs as ranks, else single terms -- R8 (4 pairs) keeps 8 GPUs busy with one
    shift each, the north_star's "one shift per GPU"."""
    terms = term_indices(method, form)
    sh = method.shift_doubles()
    if form == RESIDUAL and terms:
        units, used = [], set()
        for i in terms:
            if i in used:
                continue
            j = next((k for k in terms if k > i and k not in used and sh[k] == -sh[i]), None)
            if j is None:
                break
            used.update((i, j))
            units.append([i, j])
        else:
            if len(units) >= world:
                return units
    return [[i] for i in terms]


def owned_terms(method: FractionMethod, form: int, rank: int, world: int, per_shift: bool = False) -> List[int]:
    units = [[i] for i in term_indices(method, form)] if per_shift else term_units(method, form, world)
    return sorted(i for u, unit in enumerate(units) if u % world == rank for i in unit)


class CudaBackend:
    """The C-ABI operations the partition needs, on the local GPU. `j` is the device int32 tensor of
    squaring counts: every evaluation is of r(2^-j A)."""

    def __init__(self):
        from . import api

        self.api = api

    def squarings(self, A, theta):
        return self.api.squarings(A, theta)

    def eval(self, A, j, shifts, weights, constants, form, poly=None) -> List[torch.Tensor]:
        return self.api.eval_dense_raw(A, list(shifts), weights, list(constants), form, poly, squarings=j)

    def ordered_sum(self, terms: Sequence[torch.Tensor]) -> torch.Tensor:
        return self.api.ordered_sum(list(terms))

    def phi1_doubling(self, E, Phi, j):
        return self.api.phi1_doubling(E, Phi, j)

    def square_rows(self, E, r0: int, r1: int, out=None):
        """Rows [r0, r1) of E E (pf_square_chain's product), into `out` when given."""
        return self.api.gemm(E[r0:r1], E, Cm=out)[0]

    def cossin_step_rows(self, Cm, S, r0: int, r1: int, out_c=None, out_s=None, scratch=None):
        """Rows [r0, r1) of one cos/sin double-angle step as pf_cossin_doubling forms it:
        (C - S)(C + S) and 2 S C, the differences / sums by pf_sum_diff (no eager tensor math)."""
        if scratch is None:
            scratch = (torch.empty_like(Cm[r0:r1]), torch.empty_like(Cm))
        D, E = scratch
        self.api.sum_diff(Cm[r0:r1], S[r0:r1], diff=D)
        self.api.sum_diff(Cm, S, total=E)
        return self.api.gemm(D, E, Cm=out_c)[0], self.api.gemm(S[r0:r1], Cm, alpha=2.0, Cm=out_s)[0]

    def phi1_step_rows(self, E, Phi, r0: int, r1: int, out_e=None, out_p=None, scratch=None):
        """Rows [r0, r1) of one doubling step, as pf_phi1_doubling computes them: T = E + I (the
        diagonal by a rounded add, pf_add_identity_rows), 0.5 (T Phi) and E E on the DMMA GEMM."""
        T = scratch if scratch is not None else torch.empty_like(E[r0:r1])
        self.api.add_identity_rows(E[r0:r1], r0, T)
        return self.api.gemm(E[r0:r1], E, Cm=out_e)[0], self.api.gemm(T, Phi, alpha=0.5, Cm=out_p)[0]


def _gather_terms_to_root(method: FractionMethod, form: int, local_terms: torch.Tensor, group, world: int, rank: int,
                          root: int, per_shift: bool = True) -> Tuple[List[int], List[torch.Tensor]]:
    """Every rank's weighted terms to `root` only (torch.distributed.gather: NCCL send/recv on GPUs):
    the partition is known on every rank, so the root knows whose stack holds which shift index.
    Returns (shift indices, terms) in ascending index on the root, ([], []) elsewhere."""
    owners = [owned_terms(method, form, r, world, per_shift) for r in range(world)]
    mx = max(len(o) for o in owners)
    shape = tuple(local_terms.shape[1:])
    pad = local_terms
    if local_terms.shape[0] < mx:
        pad = torch.empty((mx,) + shape, dtype=local_terms.dtype, device=local_terms.device)
        pad[: local_terms.shape[0]] = local_terms
    gathered = [torch.empty_like(pad) for _ in range(world)] if rank == root else None
    dist.gather(pad.contiguous(), gathered, dst=root, group=group)
    if rank != root:
        return [], []
    pairs = [(owners[r][q], gathered[r][q]) for r in range(world) for q in range(len(owners[r]))]
    pairs.sort(key=lambda p: p[0])
    return [p[0] for p in pairs], [p[1] for p in pairs]


def _constants(sets, form):
    return [to_double_nearest(s.constant_term()) if form == RESIDUAL
            else (to_double_nearest(s.poly[0]) if len(s.poly) == 3 else 0.0) for s in sets]


def _poly(sets):
    if not any(len(s.poly) == 3 for s in sets):
        return None
    return [[to_double_nearest(d) for d in s.poly] if len(s.poly) == 3 else [0.0, 0.0, 0.0] for s in sets]


def eval_sets_sharded(A: torch.Tensor, j, method: FractionMethod, extra_sets: Sequence[FractionMethod] = (),
                      form: int = RESIDUAL, deterministic: bool = True, group=None, backend=None,
                      root: int = 0) -> Optional[List[torch.Tensor]]:
    """r_s(2^-j A) for the method's weight set and every extra set on the same shifts, the terms
    partitioned over the ranks of `group`. Returns the list of results on `root`, None elsewhere."""
    backend = backend or CudaBackend()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sets = [method] + list(extra_sets)
    mine = owned_terms(method, form, rank, world, per_shift=deterministic)
    sh = method.shift_doubles()
    constants = _constants(sets, form)
    poly = _poly(sets)
    has_poly_part = form == RESIDUAL or poly is not None
    if deterministic:
        # each owned term on its own (a one-term method with constant 0 returns exactly w X, or
        # w I for a plain-form zero shift), every term to every rank, then the ascending-shift sum
        local = [[] for _ in sets]
        for i in mine:
            res = backend.eval(A, j, [sh[i]], [[s.weight_doubles()[i]] for s in sets], [0.0] * len(sets),
                               form if sh[i] != 0 else PLAIN)
            for s_i in range(len(sets)):
                local[s_i].append(res[s_i])
        results = []
        for s_i in range(len(sets)):
            lt = torch.stack(local[s_i]) if local[s_i] else torch.zeros((0,) + tuple(A.shape), dtype=A.dtype,
                                                                         device=A.device)
            if world > 1:
                idx, terms = _gather_terms_to_root(method, form, lt, group, world, rank, root)
            else:
                idx, terms = mine, list(lt)
            if rank != root:
                continue
            if has_poly_part:
                terms = list(terms) + backend.eval(A, j, [], [[] for _ in range(1)], [constants[s_i]], form,
                                                   [poly[s_i]] if poly else None)
            results.append(backend.ordered_sum(terms) if len(terms) > 1 else terms[0].clone())
        return results if rank == root else None
    # fast: local partial sums (the root also adds the constant / poly part) + reduce
    cst = constants if rank == root else [0.0] * len(sets)
    pl = poly if rank == root else None
    if mine or rank == root:
        parts = backend.eval(A, j, [sh[i] for i in mine], [[s.weight_doubles()[i] for i in mine] for s in sets],
                             cst, form, pl)
    else:
        parts = [torch.zeros_like(A) for _ in sets]
    out = []
    for p in parts:
        if world > 1:
            dist.reduce(p, dst=root, op=dist.ReduceOp.SUM, group=group)
        out.append(p)
    return out if rank == root else None


def _allgather_rows(block: torch.Tensor, n: int, rows: int, group, world: int, buf: torch.Tensor) -> torch.Tensor:
    """Every rank's row block (the last one padded to `rows`) gathered into the preallocated
    (world * rows) x n buffer `buf` (one all_gather_into_tensor); returns its first n rows."""
    if block.shape[0] < rows:
        pad = torch.zeros((rows,) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
        pad[: block.shape[0]] = block
        block = pad
    dist.all_gather_into_tensor(buf, block.contiguous(), group=group)
    return buf[:n]


def _row_range(n: int, group):
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    rows = -(-n // world)
    return world, rows, min(n, rank * rows), min(n, (rank + 1) * rows)


def phi1_doubling_distributed(E: torch.Tensor, Phi: torch.Tensor, j: int, group=None, backend=None):
    """f1: Phi <- 0.5 (E + I) Phi, E <- E E, j times, every product split by rows over the ranks of
    `group` with one all-gather of each row block per step into preallocated buffers. E and Phi must
    be replicated on entry; they are replicated on exit, bit-identical to the single-process recurrence."""
    backend = backend or CudaBackend()
    n = E.shape[0]
    world, rows, r0, r1 = _row_range(n, group)
    if world == 1:
        for _ in range(int(j)):
            E, Phi = backend.phi1_step_rows(E, Phi, 0, n)
        return E, Phi
    # double-buffered full matrices and the local row blocks, allocated once
    bufs_e = [torch.empty((world * rows, n), dtype=E.dtype, device=E.device) for _ in range(2)]
    bufs_p = [torch.empty_like(bufs_e[0]) for _ in range(2)]
    e_r, p_r, t_r = (torch.empty((r1 - r0, n), dtype=E.dtype, device=E.device) for _ in range(3))
    for s in range(int(j)):
        e_b, p_b = backend.phi1_step_rows(E, Phi, r0, r1, out_e=e_r, out_p=p_r, scratch=t_r)
        E = _allgather_rows(e_b, n, rows, group, world, bufs_e[s % 2])
        Phi = _allgather_rows(p_b, n, rows, group, world, bufs_p[s % 2])
    return E.contiguous(), Phi.contiguous()


def square_chain_distributed(E: torch.Tensor, j: int, group=None, backend=None):
    """f1 for expm: E <- E E, j times, each product split by rows over the ranks of `group` with an
    all-gather per step; bit-identical to the single-process chain (pf_square_chain)."""
    backend = backend or CudaBackend()
    n = E.shape[0]
    world, rows, r0, r1 = _row_range(n, group)
    if world == 1:
        for _ in range(int(j)):
            E = backend.square_rows(E, 0, n)
        return E
    bufs = [torch.empty((world * rows, n), dtype=E.dtype, device=E.device) for _ in range(2)]
    e_r = torch.empty((r1 - r0, n), dtype=E.dtype, device=E.device)
    for s in range(int(j)):
        e_b = backend.square_rows(E, r0, r1, out=e_r)
        E = _allgather_rows(e_b, n, rows, group, world, bufs[s % 2])
    return E.contiguous()


def cossin_doubling_distributed(Cm: torch.Tensor, S: torch.Tensor, j: int, group=None, backend=None):
    """f1 for cos/sin: C <- (C - S)(C + S), S <- 2 S C, j times, split by rows with an all-gather of
    both per step; bit-identical to pf_cossin_doubling."""
    backend = backend or CudaBackend()
    n = Cm.shape[0]
    world, rows, r0, r1 = _row_range(n, group)
    if world == 1:
        for _ in range(int(j)):
            Cm, S = backend.cossin_step_rows(Cm, S, 0, n)
        return Cm, S
    bufs_c = [torch.empty((world * rows, n), dtype=Cm.dtype, device=Cm.device) for _ in range(2)]
    bufs_s = [torch.empty_like(bufs_c[0]) for _ in range(2)]
    c_r, s_r, d_r = (torch.empty((r1 - r0, n), dtype=Cm.dtype, device=Cm.device) for _ in range(3))
    e_full = torch.empty_like(Cm)
    for s in range(int(j)):
        c_b, s_b = backend.cossin_step_rows(Cm, S, r0, r1, out_c=c_r, out_s=s_r, scratch=(d_r, e_full))
        Cm = _allgather_rows(c_b, n, rows, group, world, bufs_c[s % 2])
        S = _allgather_rows(s_b, n, rows, group, world, bufs_s[s % 2])
    return Cm.contiguous(), S.contiguous()


def expm_phi1_sharded(A: torch.Tensor, method="R8", deterministic: bool = True, group=None, root: int = 0,
                      backend=None, distributed_doubling: bool = False):
    """cfg3: exp(A) and phi1(A) with the shifts split across the ranks, one reduce before the
    doubling recurrence -- on the root, or split by rows over all ranks (f1, distributed_doubling).
    Returns (E, Phi) on the root, None elsewhere."""
    backend = backend or CudaBackend()
    m = catalog(method) if isinstance(method, str) else method
    phi = same_shift_method(m, FunctionId.phi(1))
    theta = min(THETA_U53[m.name], THETA_U53.get(m.name + "_phi1set", THETA_U53[m.name]))
    j = backend.squarings(A, theta)
    res = eval_sets_sharded(A, j, m, [phi], RESIDUAL, deterministic, group, backend, root)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if distributed_doubling and world > 1:
        rank = dist.get_rank(group)
        E, Phi = res if res is not None else (torch.empty_like(A), torch.empty_like(A))
        dist.broadcast(E, src=root, group=group)
        dist.broadcast(Phi, src=root, group=group)
        E, Phi = phi1_doubling_distributed(E, Phi, int(j.max()), group, backend)
        return (E, Phi) if rank == root else None
    if res is None:
        return None
    E, Phi = res
    backend.phi1_doubling(E, Phi, j)
    return E, Phi


def action_sharded(A: torch.Tensor, V: torch.Tensor, method="R8", substeps: int = 1, form: int = RESIDUAL,
                   deterministic: bool = True, group=None, operator_factory=None, ordered_sum=None):
    """cfg4: exp(A) V by N substeps; every rank factors its shifts once (ActionOperator) and each
    substep ends with one all-reduce (fast) or all-gather + ordered sum (deterministic) of n x k."""
    if operator_factory is None:
        from . import api

        operator_factory = api.ActionOperator
        ordered_sum = api.ordered_sum
    m = catalog(method) if isinstance(method, str) else method
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mine = owned_terms(m, form, rank, world, per_shift=deterministic)
    op = operator_factory(A, m, substeps, form, owned=mine)
    X = V.reshape(V.shape[0], -1).contiguous()
    for _ in range(substeps):
        if deterministic:
            # every weighted term to rank 0 only, the ascending-shift sum there, the next iterate to all
            _, terms = op.apply(X, include_poly=True, with_terms=True)
            nloc = op.terms
            local = terms[:nloc]
            if world > 1:
                _, gathered = _gather_terms_to_root(m, form, local, group, world, rank, 0)
            else:
                gathered = list(local)
            if rank == 0:
                ts = list(gathered) + [terms[nloc + q] for q in range(op.poly_terms)]
                X = ordered_sum(ts) if len(ts) > 1 else ts[0].clone()
            if world > 1:
                dist.broadcast(X, src=0, group=group)
        else:
            part = op.apply(X, include_poly=(rank == 0))
            if world > 1:
                dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
            X = part
    op.close()
    return X.reshape(V.shape)
