"""Python mirror of the reference's public surface for the hot path, over the C ABI.

Reference surface (proj/core/include/parfrac/):
  eval_dense(method, B, opts)     dense.hpp:74-75      -> eval_dense()
  solve_shifted(B, c)             dense.hpp:62         -> solve_shifted()
  EvalOptions{workers, fixed_order, form}  dense.hpp:64-68 -> EvalOptions
  catalog / to_residual_form      methods.hpp:73-77    -> methods.catalog / methods.to_residual_form
  theta                           bounds.hpp:62        -> methods.theta / THETA_U53
New entry points: expm (scaling and squaring), expm_phi1, cossin, action_block,
all batched.

Arrays: torch float64 CUDA tensors are used in place (device pointers, the caller's current
stream); numpy arrays / host tensors are copied to the device and the result copied back. Shapes
(n, n) or (batch, n, n), row-major contiguous. Errors raise PfError with the reference's
message text (dense.cpp:117-119, 219-221).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from . import _native as N
from .errors import Errc, PfError
from .methods import (PLAIN, RESIDUAL, THETA_U53, FractionMethod, FunctionId, PairMethod, catalog,
                      format_sig17, pair_method, same_shift_method, to_double_nearest)

ArrayLike = Union[torch.Tensor, np.ndarray]


@dataclass
class EvalOptions:
    """dense.hpp:64-68. `workers` is accepted for source compatibility; the device evaluates all
    shifts concurrently and the reduction is always in ascending shift order, so results do not
    depend on it (the reference's bit-identical-across-workers contract)."""

    workers: int = 1
    fixed_order: bool = True
    form: Optional[int] = None


# ------------------------------------------------------------------------------------------ packing


class PackedMethod:
    """pf_method with its arrays kept alive. Sets: weights of `method` first, then the extra
    weight sets (same shifts; e.g. phi1 via methods.same_shift_method)."""

    def __init__(self, method: FractionMethod, form: Optional[int] = None, extra: Sequence[FractionMethod] = ()):
        form = method.form if form is None else form
        sets = [method] + list(extra)
        for s in sets[1:]:
            if [Fraction_(c) for c in s.shifts] != [Fraction_(c) for c in method.shifts]:
                raise PfError(Errc.BadArgument, "weight sets must share the shifts")
        n = len(method.shifts)
        if n > N.PF_MAX_TERMS:
            raise PfError(Errc.BadArgument, "at most %d shifts" % N.PF_MAX_TERMS)
        self.shifts = (C.c_double * max(n, 1))(*method.shift_doubles())
        w = []
        for s in sets:
            w += s.weight_doubles()
        self.weights = (C.c_double * max(len(w), 1))(*w)
        has_poly = any(len(s.poly) == 3 for s in sets)
        poly = []
        for s in sets:
            poly += [to_double_nearest(d) for d in s.poly] if len(s.poly) == 3 else [0.0, 0.0, 0.0]
        self.poly = (C.c_double * len(poly))(*poly)
        self.constant = (C.c_double * len(sets))(*[to_double_nearest(s.constant_term()) for s in sets])
        self.c = N.PfMethod(n, self.shifts, len(sets), self.weights, 1 if has_poly else 0, self.poly, self.constant,
                            int(form))
        self.method = method

    def ptr(self):
        return C.byref(self.c)


def Fraction_(x):
    from fractions import Fraction

    return Fraction(x)


class PackedPair:
    def __init__(self, pm: PairMethod):
        n = len(pm.c2)
        self.c2 = (C.c_double * n)(*[to_double_nearest(x) for x in pm.c2])
        self.cw = (C.c_double * n)(*[to_double_nearest(x) for x in pm.cw])
        self.sw = (C.c_double * n)(*[to_double_nearest(x) for x in pm.sw])
        self.c = N.PfPairMethod(n, self.c2, self.cw, self.sw, to_double_nearest(pm.a0), to_double_nearest(pm.a1))

    def ptr(self):
        return C.byref(self.c)


# ------------------------------------------------------------------------------------------ engine


class Engine:
    """One pf_context (device, stream, workspace). Not thread-safe (one host thread at a time)."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise PfError(Errc.CudaError, "paper_2210_03714_b200 needs a CUDA device (there is no CPU path)")
        self.device = device
        torch.cuda.set_device(device)
        h = C.c_void_p()
        rc = N.lib.pf_context_create(device, C.byref(h))
        if rc:
            raise PfError(Errc.CudaError, "pf_context_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            N.lib.pf_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bind_stream(self):
        N.lib.pf_context_set_stream(self.h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))

    def launch_count(self) -> int:
        return int(N.lib.pf_context_launch_count(self.h))


_engines: dict = {}


def engine(device: Optional[int] = None) -> Engine:
    """The context of `device` (default: torch's current CUDA device), one per device per process,
    bound to torch's current stream on that device."""
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    eng = _engines.get(device)
    if eng is None:
        eng = _engines[device] = Engine(device)
    eng.bind_stream()
    return eng


# ------------------------------------------------------------------------------------------ helpers


def _raise(rc: int, st: N.PfStatus, batched: bool):
    code = Errc(rc - 1) if 0 < rc <= len(Errc) else Errc.CudaError
    if code == Errc.SingularShift:
        msg = "singular system: pivot magnitude %s at column %d (scale %s)" % (
            format_sig17(st.pivot_magnitude), st.column, format_sig17(st.scale))
        if st.shift_index > 0:
            msg = "shift %d: %s" % (st.shift_index, msg)
        if batched:
            msg = "matrix %d: %s" % (st.batch_index, msg)
        raise PfError(code, msg)
    if code == Errc.ZeroPivot:  # thomas_solve / pentadiag_solve (action.cpp:104,113,185)
        msg = "zero pivot at row %d" % st.column
        if st.shift_index > 0:
            msg = "shift %d: %s" % (st.shift_index, msg)
        raise PfError(code, msg)
    if code == Errc.CudaError:
        raise PfError(code, "CUDA failure in the B200 engine")
    raise PfError(code, "bad argument")


def _to_device(x: ArrayLike) -> Tuple[torch.Tensor, bool]:
    """Returns (contiguous float64 cuda tensor, was_host)."""
    if isinstance(x, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        return t.cuda(non_blocking=False), True
    if not isinstance(x, torch.Tensor):
        raise PfError(Errc.BadArgument, "expected a numpy array or torch tensor")
    if x.dtype != torch.float64:
        raise PfError(Errc.BadArgument, "FP64 only")
    if x.is_cuda:
        if torch.cuda.is_available() and x.device.index != torch.cuda.current_device():
            raise PfError(Errc.BadArgument, "tensor on cuda:%d but the current device (engine) is cuda:%d; use "
                                            "torch.cuda.device(...)" % (x.device.index, torch.cuda.current_device()))
        return x.contiguous(), False
    return x.contiguous().cuda(), True


def _as_batch(t: torch.Tensor) -> Tuple[torch.Tensor, bool]:
    if t.dim() == 2:
        if t.shape[0] != t.shape[1]:
            raise PfError(Errc.BadArgument, "matrix must be square")
        return t.unsqueeze(0), False
    if t.dim() == 3 and t.shape[1] == t.shape[2]:
        return t, True
    raise PfError(Errc.BadArgument, "expected (n, n) or (batch, n, n)")


def _back(t: torch.Tensor, host: bool, squeeze: bool, like: ArrayLike):
    if squeeze:
        t = t[0]
    if host:
        return t.cpu().numpy() if isinstance(like, np.ndarray) else t.cpu()
    return t


def _resolve_method(method) -> FractionMethod:
    return catalog(method) if isinstance(method, str) else method


def _theta_for(method: FractionMethod, theta: Optional[float]) -> float:
    if theta is not None:
        return float(theta)
    if method.name in THETA_U53:
        return THETA_U53[method.name]
    from .methods import theta as theta_fn

    return theta_fn(method, tol=2.0 ** -53)


# ------------------------------------------------------------------------------------------ entry points


def eval_dense(method, B: ArrayLike, opts: Optional[EvalOptions] = None, extra_sets: Sequence[FractionMethod] = (),
               flags: int = 0):
    """r(B) (dense.cpp:193-252) for one matrix or a batch. With `extra_sets`, returns a list
    [r_0(B), r_1(B), ...] computed from the same solves."""
    opts = opts or EvalOptions()
    if opts.workers < 1:
        raise PfError(Errc.BadArgument, "workers must be >= 1")
    if not opts.fixed_order:
        raise PfError(Errc.BadArgument, "only fixed-order reduction is supported")
    m = _resolve_method(method)
    pk = PackedMethod(m, opts.form, extra_sets)
    eng = engine()
    dB, host = _to_device(B)
    dB3, batched = _as_batch(dB)
    bsz, n = dB3.shape[0], dB3.shape[1]
    outs = [torch.empty_like(dB3) for _ in range(1 + len(extra_sets))]
    ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    st = N.PfStatus()
    rc = N.lib.pf_eval_dense_batched(eng.h, pk.ptr(), n, bsz, dB3.data_ptr(), n, n * n, ptrs, n, n * n, flags,
                                     C.byref(st))
    if rc:
        _raise(rc, st, batched)
    res = [_back(o, host, not batched, B) for o in outs]
    return res if extra_sets else res[0]


def eval_dense_raw(B: torch.Tensor, shifts: Sequence[float], weights: Sequence[Sequence[float]],
                   constants: Sequence[float], form: int = RESIDUAL, poly: Optional[Sequence[Sequence[float]]] = None,
                   flags: int = 0, squarings: Optional[torch.Tensor] = None) -> List[torch.Tensor]:
    """eval_dense on explicit doubles (device tensors in and out): one output per weight set, of
    B itself or -- with `squarings` (device int32, one per matrix) -- of 2^-j B. Used by the shift
    partition (parallel.py) to evaluate a rank's subset of the terms."""
    eng = engine()
    dB3, batched = _as_batch(B.contiguous())
    bsz, n = dB3.shape[0], dB3.shape[1]
    nt = len(shifts)
    sets = len(weights)
    sh = (C.c_double * max(nt, 1))(*shifts)
    w = (C.c_double * max(nt * sets, 1))(*[x for row in weights for x in row])
    cst = (C.c_double * sets)(*constants)
    pl = (C.c_double * (3 * sets))(*([x for row in poly for x in row] if poly else [0.0] * (3 * sets)))
    m = N.PfMethod(nt, sh, sets, w, 1 if poly else 0, pl, cst, int(form))
    outs = [torch.empty_like(dB3) for _ in range(sets)]
    ptrs = (C.c_void_p * sets)(*[o.data_ptr() for o in outs])
    st = N.PfStatus()
    if squarings is not None:
        jin = squarings.to(dtype=torch.int32, device=dB3.device).contiguous()
        rc = N.lib.pf_eval_scaled_batched(eng.h, C.byref(m), 0.0, n, bsz, dB3.data_ptr(), n, n * n, jin.data_ptr(),
                                          None, ptrs, n, n * n, flags, C.byref(st))
    else:
        rc = N.lib.pf_eval_dense_batched(eng.h, C.byref(m), n, bsz, dB3.data_ptr(), n, n * n, ptrs, n, n * n, flags,
                                         C.byref(st))
    if rc:
        _raise(rc, st, batched)
    return [o if batched else o[0] for o in outs]


def ordered_sum(terms: Sequence[torch.Tensor]) -> torch.Tensor:
    """((t0 + t1) + t2) + ... on the device (pf_ordered_sum): the reference's fixed reduction order."""
    eng = engine()
    ts = [t.contiguous() for t in terms]
    out = torch.empty_like(ts[0])
    ptrs = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    rc = N.lib.pf_ordered_sum(eng.h, len(ts), ptrs, ts[0].numel(), out.data_ptr())
    if rc:
        _raise(rc, N.PfStatus(), False)
    return out


def squarings(A: torch.Tensor, theta: float) -> torch.Tensor:
    eng = engine()
    a3, _ = _as_batch(A.contiguous())
    bsz, n = a3.shape[0], a3.shape[1]
    j = torch.empty(bsz, dtype=torch.int32, device=a3.device)
    rc = N.lib.pf_squarings_batched(eng.h, n, bsz, a3.data_ptr(), n, n * n, float(theta), j.data_ptr())
    if rc:
        _raise(rc, N.PfStatus(), True)
    return j


def phi1_doubling(E: torch.Tensor, Phi: torch.Tensor, j: torch.Tensor):
    eng = engine()
    e3, _ = _as_batch(E)
    p3, _ = _as_batch(Phi)
    rc = N.lib.pf_phi1_doubling(eng.h, e3.shape[1], e3.shape[0], j.data_ptr(), e3.data_ptr(), p3.data_ptr())
    if rc:
        _raise(rc, N.PfStatus(), True)
    return E, Phi


def square_chain(E: torch.Tensor, j: torch.Tensor):
    eng = engine()
    e3, _ = _as_batch(E)
    rc = N.lib.pf_square_chain(eng.h, e3.shape[1], e3.shape[0], j.data_ptr(), e3.data_ptr())
    if rc:
        _raise(rc, N.PfStatus(), True)
    return E


class ActionOperator:
    """ActionOperator on a dense A (action.hpp:68-82): B = A (1/N), LU of every owned shift computed
    once; apply() = one substep r(B) V over the owned terms (optionally with the poly part)."""

    def __init__(self, A: torch.Tensor, method="R8", substeps: int = 1, form: int = RESIDUAL,
                 owned: Optional[Sequence[int]] = None, flags: int = 0):
        self.method = _resolve_method(method)
        self.pk = PackedMethod(self.method, form)
        eng = engine()
        self.A = A.contiguous()
        n = self.A.shape[0]
        own = None
        if owned is not None:
            own = (C.c_int * len(self.method.shifts))(*[1 if i in set(owned) else 0
                                                        for i in range(len(self.method.shifts))])
        h = C.c_void_p()
        st = N.PfStatus()
        rc = N.lib.pf_action_create(eng.h, self.pk.ptr(), n, self.A.data_ptr(), n, int(substeps), own, flags,
                                    C.byref(st), C.byref(h))
        if rc:
            _raise(rc, st, False)
        self.h = h
        self.n = n
        self.terms = int(N.lib.pf_action_term_count(h))
        hybrid = len(self.method.poly) == 3
        self.poly_terms = (1 if (form == RESIDUAL or hybrid) else 0) + (1 if hybrid else 0)

    def apply(self, V: torch.Tensor, include_poly: bool = True, with_terms: bool = False):
        V2 = V.reshape(self.n, -1).contiguous()
        k = V2.shape[1]
        out = torch.empty_like(V2)
        nterm = self.terms + (self.poly_terms if include_poly else 0)
        terms = torch.empty((nterm, self.n, k), dtype=torch.float64, device=V2.device) if with_terms else None
        st = N.PfStatus()
        rc = N.lib.pf_action_apply(self.h, V2.data_ptr(), k, k, out.data_ptr(), k, 1 if include_poly else 0,
                                   terms.data_ptr() if terms is not None else None, C.byref(st))
        if rc:
            _raise(rc, st, False)
        return (out, terms) if with_terms else out

    def close(self):
        if getattr(self, "h", None):
            N.lib.pf_action_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_shifted(B: ArrayLike, c: float, flags: int = 0):
    """(I - cB)^{-1} (dense.cpp:165-171)."""
    eng = engine()
    dB, host = _to_device(B)
    dB3, batched = _as_batch(dB)
    bsz, n = dB3.shape[0], dB3.shape[1]
    out = torch.empty_like(dB3)
    st = N.PfStatus()
    rc = N.lib.pf_solve_shifted_batched(eng.h, n, bsz, dB3.data_ptr(), n, n * n, float(c), out.data_ptr(), n, n * n,
                                        flags, C.byref(st))
    if rc:
        _raise(rc, st, batched)
    return _back(out, host, not batched, B)


def expm(A: ArrayLike, method="R4", theta: Optional[float] = None, squarings: Optional[ArrayLike] = None,
         form: int = RESIDUAL, return_squarings: bool = False, flags: int = 0, out: Optional[torch.Tensor] = None):
    """exp(A) by r(2^-j A)^(2^j), j = smallest j >= 0 with ||A||_1 2^-j <= theta_m.
    Residual form by default (the parity-safe form)."""
    m = _resolve_method(method)
    th = _theta_for(m, theta)
    pk = PackedMethod(m, form)
    eng = engine()
    dA, host = _to_device(A)
    dA3, batched = _as_batch(dA)
    bsz, n = dA3.shape[0], dA3.shape[1]
    o = out if out is not None else torch.empty_like(dA3)
    j_in = None
    if squarings is not None:
        j_in = torch.as_tensor(squarings, dtype=torch.int32).reshape(-1).to(dA3.device).contiguous()
    j_out = torch.empty(bsz, dtype=torch.int32, device=dA3.device)
    st = N.PfStatus()
    rc = N.lib.pf_expm_batched(eng.h, pk.ptr(), th, n, bsz, dA3.data_ptr(), n, n * n,
                               j_in.data_ptr() if j_in is not None else None, j_out.data_ptr(), o.data_ptr(), n, n * n,
                               flags, C.byref(st))
    if rc:
        _raise(rc, st, batched)
    res = _back(o, host, not batched, A)
    if return_squarings:
        js = j_out.cpu().numpy() if host else j_out
        return res, (js[0] if not batched else js)
    return res


class MultiDevice:
    """pf_context_create_multi + pf_eval_multi_gpu: ONE matrix with its shifts partitioned over
    several GPUs of this process (the C ABI's own NCCL communicator), the single-process counterpart
    of parallel.py's one-process-per-GPU path. ``deterministic=True`` gives results bit-identical
    for any device count (the reference's workers contract, dense.cpp:202/245-246); repeated device
    ids emulate several shares on one GPU (tests)."""

    def __init__(self, device_ids: Sequence[int]):
        ids = (C.c_int * len(device_ids))(*device_ids)
        h = C.c_void_p()
        rc = N.lib.pf_context_create_multi(len(device_ids), ids, C.byref(h))
        if rc:
            raise PfError(Errc.CudaError, "pf_context_create_multi failed (%d)" % rc)
        self.h = h
        self.device_ids = list(device_ids)
        self.root = device_ids[0]

    @property
    def uses_nccl(self) -> bool:
        return bool(N.lib.pf_context_uses_nccl(self.h))

    def close(self):
        if getattr(self, "h", None):
            N.lib.pf_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run(self, method, A: ArrayLike, recurrence: int, theta: Optional[float], form: int, deterministic: bool,
             extra: Sequence[FractionMethod] = (), flags: int = 0):
        m = _resolve_method(method)
        pk = PackedMethod(m, form, extra)
        with torch.cuda.device(self.root):
            dA, host = _to_device(A)
            n = dA.shape[0]
            if dA.dim() != 2 or dA.shape[1] != n:
                raise PfError(Errc.BadArgument, "expected one square matrix")
            outs = [torch.empty_like(dA) for _ in range(1 + len(extra))]
            torch.cuda.synchronize()
            st = N.PfStatus()
            j = C.c_int(0)
            rc = N.lib.pf_eval_multi_gpu(self.h, pk.ptr(), float(theta or 0.0), recurrence, n, dA.data_ptr(), n,
                                         outs[0].data_ptr(), outs[1].data_ptr() if len(outs) > 1 else None, n,
                                         1 if deterministic else 0, flags, C.byref(j), C.byref(st))
            if rc:
                _raise(rc, st, False)
            torch.cuda.synchronize()
        res = [_back(o.unsqueeze(0), host, True, A) for o in outs]
        return res, j.value

    def eval_dense(self, method, B: ArrayLike, form: int = RESIDUAL, deterministic: bool = True):
        return self._run(method, B, N.PF_REC_NONE, None, form, deterministic)[0][0]

    def expm(self, method, A: ArrayLike, theta: Optional[float] = None, form: int = RESIDUAL,
             deterministic: bool = True, return_squarings: bool = False):
        m = _resolve_method(method)
        (e,), j = self._run(m, A, N.PF_REC_EXP, _theta_for(m, theta), form, deterministic)
        return (e, j) if return_squarings else e

    def expm_phi1(self, method, A: ArrayLike, theta: Optional[float] = None, deterministic: bool = True,
                  return_squarings: bool = False):
        m = _resolve_method(method)
        phi = same_shift_method(m, FunctionId.phi(1))
        th = theta if theta is not None else min(_theta_for(m, None), THETA_U53.get(m.name + "_phi1set")
                                                 or _theta_for(phi, None))
        (e, p), j = self._run(m, A, N.PF_REC_EXP_PHI1, th, RESIDUAL, deterministic, extra=[phi])
        return (e, p, j) if return_squarings else (e, p)


class HostPipeline:
    """Batched expm of HOST matrices with the host->device copy, the evaluation and the
    device->host copy overlapped across chunks: `streams` CUDA streams, one pf_context each (so
    every stream has its own status buffers), chunk c on stream c mod streams. Inputs/outputs
    should be pinned for the copies to be asynchronous."""

    def __init__(self, n: int, batch: int, chunk: int = 512, streams: int = 3, device: Optional[int] = None):
        if not torch.cuda.is_available():
            raise PfError(Errc.CudaError, "paper_2210_03714_b200 needs a CUDA device (there is no CPU path)")
        self.device = torch.cuda.current_device() if device is None else device
        self.n, self.batch, self.chunk = n, batch, min(chunk, batch)
        self.streams = [torch.cuda.Stream(self.device) for _ in range(streams)]
        self.engines = [Engine(self.device) for _ in range(streams)]
        for e, s in zip(self.engines, self.streams):
            N.lib.pf_context_set_stream(e.h, C.c_void_p(s.cuda_stream))
        shape = (self.chunk, n, n)
        self.dA = [torch.empty(shape, dtype=torch.float64, device=self.device) for _ in range(streams)]
        self.dO = [torch.empty(shape, dtype=torch.float64, device=self.device) for _ in range(streams)]
        self._pending = []
        self._armed = False

    def launch_count(self) -> int:
        return sum(e.launch_count() for e in self.engines)

    def submit(self, host_in: torch.Tensor, host_out: torch.Tensor, method="R4", theta: Optional[float] = None,
               form: int = RESIDUAL):
        """Enqueue host_in -> expm -> host_out without synchronising: chunk c on stream c mod streams,
        each stream ordered (its buffers are reused only after its own previous chunk), so
        successive submissions overlap -- the next batch's first copies run under the previous
        batch's last kernels. Device status is sticky across submissions; finish() checks it."""
        m = _resolve_method(method)
        th = _theta_for(m, theta)
        pk = PackedMethod(m, form)
        self._pending.append((host_in, m, th, form))
        n, S = self.n, len(self.streams)
        if not self._armed:
            for e in self.engines:
                N.lib.pf_context_set_sticky_status(e.h, 1)
            self._armed = True
        st = N.PfStatus()
        for c, start in enumerate(range(0, self.batch, self.chunk)):
            k = c % S
            mb = min(self.chunk, self.batch - start)
            with torch.cuda.stream(self.streams[k]):
                self.dA[k][:mb].copy_(host_in[start:start + mb], non_blocking=True)
                rc = N.lib.pf_expm_batched(self.engines[k].h, pk.ptr(), th, n, mb, self.dA[k].data_ptr(), n, n * n,
                                           None, None, self.dO[k].data_ptr(), n, n * n, N.PF_FLAG_ASYNC, C.byref(st))
                if rc:
                    _raise(rc, st, True)
                host_out[start:start + mb].copy_(self.dO[k][:mb], non_blocking=True)
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams:  # the caller's stream (and its events) sees the submitted work
            cur.wait_stream(s)
        return host_out

    def finish(self):
        """Synchronise every submission and raise the first error (recomputed synchronously on the
        offending batch for the exact status)."""
        failed = [N.lib.pf_context_pending_error(e.h) for e in self.engines]
        for e in self.engines:
            N.lib.pf_context_set_sticky_status(e.h, 0)
        self._armed = False
        pending, self._pending = self._pending, []
        if any(failed):
            for host_in, m, th, form in pending:
                expm(host_in.cuda(), m, th, form=form)

    def expm(self, host_in: torch.Tensor, host_out: torch.Tensor, method="R4", theta: Optional[float] = None,
             form: int = RESIDUAL):
        self.submit(host_in, host_out, method, theta, form)
        self.finish()
        return host_out


def expm_phi1(A: ArrayLike, method="R8", theta: Optional[float] = None, form: int = RESIDUAL, flags: int = 0,
              return_squarings: bool = False):
    """(exp(A), phi1(A)) from one solve per shift (weight sets exp and phi1 on the method's
    shifts), then j doublings Phi <- 0.5 (E + I) Phi, E <- E E."""
    m = _resolve_method(method)
    phi = same_shift_method(m, FunctionId.phi(1))
    th = theta if theta is not None else min(_theta_for(m, None), THETA_U53.get(m.name + "_phi1set")
                                             or _theta_for(phi, None))
    pk = PackedMethod(m, form, [phi])
    eng = engine()
    dA, host = _to_device(A)
    dA3, batched = _as_batch(dA)
    bsz, n = dA3.shape[0], dA3.shape[1]
    oE, oP = torch.empty_like(dA3), torch.empty_like(dA3)
    j_out = torch.empty(bsz, dtype=torch.int32, device=dA3.device)
    st = N.PfStatus()
    rc = N.lib.pf_expm_phi1_batched(eng.h, pk.ptr(), float(th), n, bsz, dA3.data_ptr(), n, n * n, None,
                                    j_out.data_ptr(), oE.data_ptr(), oP.data_ptr(), n, n * n, flags, C.byref(st))
    if rc:
        _raise(rc, st, batched)
    res = (_back(oE, host, not batched, A), _back(oP, host, not batched, A))
    if return_squarings:
        js = j_out.cpu().numpy() if host else j_out
        return res + ((js[0] if not batched else js),)
    return res


def cossin(A: ArrayLike, method="R8", theta: Optional[float] = None, flags: int = 0, return_squarings: bool = False):
    """(cos A, sin A) through exp(iB) with merged conjugate shifts and the C^2 - S^2 / 2SC
    double-angle recurrence."""
    m = _resolve_method(method)
    pm = pair_method(m)
    th = _theta_for(m, theta)
    pk = PackedPair(pm)
    eng = engine()
    dA, host = _to_device(A)
    dA3, batched = _as_batch(dA)
    bsz, n = dA3.shape[0], dA3.shape[1]
    oC, oS = torch.empty_like(dA3), torch.empty_like(dA3)
    j_out = torch.empty(bsz, dtype=torch.int32, device=dA3.device)
    st = N.PfStatus()
    rc = N.lib.pf_cossin_batched(eng.h, pk.ptr(), float(th), n, bsz, dA3.data_ptr(), n, n * n, None,
                                 j_out.data_ptr(), oC.data_ptr(), oS.data_ptr(), n, n * n, flags, C.byref(st))
    if rc:
        _raise(rc, st, batched)
    res = (_back(oC, host, not batched, A), _back(oS, host, not batched, A))
    if return_squarings:
        js = j_out.cpu().numpy() if host else j_out
        return res + ((js[0] if not batched else js),)
    return res


def action(A: ArrayLike, V: ArrayLike, method="R8", substeps: Optional[int] = None, theta: Optional[float] = None,
           form: int = RESIDUAL, flags: int = 0):
    """exp(A) V by N-fold substepping V <- r(A/N) V with one LU per shift reused across substeps
    (dense analogue of substep_action / ActionOperator, action.cpp:300-339). N defaults to
    ceil(||A||_1 / theta_m) (select_method, action.cpp:398)."""
    m = _resolve_method(method)
    pk = PackedMethod(m, form)
    eng = engine()
    dA, host = _to_device(A)
    dV, _ = _to_device(V)
    if dA.dim() != 2 or dA.shape[0] != dA.shape[1] or dV.dim() not in (1, 2) or dV.shape[0] != dA.shape[0]:
        raise PfError(Errc.LengthMismatch, "vector length mismatch")
    vec = dV.dim() == 1
    dV2 = dV.reshape(dV.shape[0], -1).contiguous()
    n, k = dV2.shape
    if substeps is None:
        from .methods import substeps_for

        substeps = substeps_for(one_norm(dA), _theta_for(m, theta))
    out = torch.empty_like(dV2)
    st = N.PfStatus()
    rc = N.lib.pf_action_block(eng.h, pk.ptr(), n, k, dA.data_ptr(), n, dV2.data_ptr(), k, int(substeps),
                               out.data_ptr(), k, flags, C.byref(st))
    if rc:
        _raise(rc, st, False)
    res = out.reshape(-1) if vec else out
    return _back(res.unsqueeze(0), host, True, A)


class DenseLu:
    """DenseLu (dense.hpp:46-59): PA = LU with partial pivoting, reusable across right-hand sides.
    `piv` is the LAPACK-style 0-based swap sequence (the reference keeps it private, piv_)."""

    def __init__(self, A: ArrayLike, pivot_rel_tol: float = 1e-14, flags: int = 0):
        eng = engine()
        dA, self._host = _to_device(A)
        dA3, self._batched = _as_batch(dA)
        self.lu = dA3.clone()
        bsz, n = self.lu.shape[0], self.lu.shape[1]
        self.piv = torch.empty(bsz, n, dtype=torch.int32, device=self.lu.device)
        st = N.PfStatus()
        rc = N.lib.pf_lu_factor_batched(eng.h, n, bsz, self.lu.data_ptr(), n, n * n, self.piv.data_ptr(),
                                        float(pivot_rel_tol), flags, C.byref(st))
        if rc:
            _raise(rc, st, self._batched)

    def solve_matrix(self, rhs: ArrayLike):
        eng = engine()
        dR, host = _to_device(rhs)
        if dR.dim() == 1:
            dR = dR.reshape(-1, 1)
        r3 = dR if dR.dim() == 3 else dR.unsqueeze(0)
        r3 = r3.clone()
        bsz, n, k = r3.shape
        rc = N.lib.pf_lu_solve_batched(eng.h, n, k, bsz, self.lu.data_ptr(), n, n * n, self.piv.data_ptr(),
                                       r3.data_ptr(), k, n * k)
        if rc:
            _raise(rc, N.PfStatus(), self._batched)
        out = r3 if dR.dim() == 3 else r3[0]
        return out.cpu().numpy() if host and isinstance(rhs, np.ndarray) else (out.cpu() if host else out)

    def solve(self, rhs: ArrayLike):
        res = self.solve_matrix(rhs)
        return res.reshape(-1) if hasattr(res, "reshape") else res

    def factors(self):
        lu = self.lu if self._batched else self.lu[0]
        piv = self.piv if self._batched else self.piv[0]
        if self._host:
            return lu.cpu().numpy(), piv.cpu().numpy()
        return lu, piv


def one_norm(A: ArrayLike):
    eng = engine()
    dA, host = _to_device(A)
    dA3, batched = _as_batch(dA)
    bsz, n = dA3.shape[0], dA3.shape[1]
    out = torch.empty(bsz, dtype=torch.float64, device=dA3.device)
    rc = N.lib.pf_one_norm_batched(eng.h, n, bsz, dA3.data_ptr(), n, n * n, out.data_ptr())
    if rc:
        _raise(rc, N.PfStatus(), batched)
    if host:
        out = out.cpu().numpy()
    return out if batched else float(out[0])


def gemm(A: torch.Tensor, B: torch.Tensor, alpha: float = 1.0, beta: float = 0.0, Cm: Optional[torch.Tensor] = None,
         gamma: float = 0.0) -> torch.Tensor:
    """C = alpha A B + beta C + gamma I on the FP64 DMMA GEMM (device tensors, (m,k)x(k,n) or batched)."""
    eng = engine()
    a3 = A if A.dim() == 3 else A.unsqueeze(0)
    b3 = B if B.dim() == 3 else B.unsqueeze(0)
    bsz, m, k = a3.shape
    n = b3.shape[2]
    if Cm is None:  # beta == 0: the output is not read
        Cm = (torch.empty if beta == 0.0 else torch.zeros)(bsz, m, n, dtype=torch.float64, device=a3.device)
    c3 = Cm if Cm.dim() == 3 else Cm.unsqueeze(0)
    rc = N.lib.pf_gemm_batched(eng.h, m, n, k, bsz, alpha, a3.data_ptr(), k, m * k, b3.data_ptr(), n, k * n, beta,
                               c3.data_ptr(), n, m * n, gamma)
    if rc:
        _raise(rc, N.PfStatus(), True)
    return Cm


def add_identity_rows(X_rows: torch.Tensor, r0: int, out: torch.Tensor) -> torch.Tensor:
    """out = rows [r0, r0 + R) of X + I, given those rows of X (pf_add_identity_rows)."""
    eng = engine()
    rows, n = X_rows.shape
    rc = N.lib.pf_add_identity_rows(eng.h, rows, n, r0, X_rows.data_ptr(), X_rows.stride(0), out.data_ptr(),
                                    out.stride(0))
    if rc:
        _raise(rc, N.PfStatus(), False)
    return out


def sum_diff(Cm: torch.Tensor, S: torch.Tensor, diff: Optional[torch.Tensor] = None,
             total: Optional[torch.Tensor] = None):
    """diff = C - S and/or total = C + S elementwise on the device (pf_sum_diff)."""
    eng = engine()
    rc = N.lib.pf_sum_diff(eng.h, Cm.numel(), Cm.data_ptr(), S.data_ptr(), diff.data_ptr() if diff is not None else None,
                           total.data_ptr() if total is not None else None)
    if rc:
        _raise(rc, N.PfStatus(), False)
    return diff, total


# ---- f2: banded action (proj/core/src/action.cpp). A tridiagonal matrix is (sub, diag, super) with
# lengths d-1, d, d-1 (TridiagMatrix); vectors are columns of a d x k block, each processed exactly as
# the reference processes one vector.


class TridiagMatrix:
    """Compact three-diagonal matrix (action.hpp:13-24), device arrays."""

    def __init__(self, sub: ArrayLike, diag: ArrayLike, sup: ArrayLike):
        self.sub = _to_device(sub)[0].reshape(-1)
        self.diag = _to_device(diag)[0].reshape(-1)
        self.sup = _to_device(sup)[0].reshape(-1)
        self.d = int(self.diag.numel())
        if self.sub.numel() != max(self.d - 1, 0) or self.sup.numel() != max(self.d - 1, 0):
            raise PfError(Errc.LengthMismatch, "band length mismatch")

    @staticmethod
    def trid121(d: int) -> "TridiagMatrix":
        """trid{-1, 2, -1} (action.cpp:27-33)."""
        o = torch.full((max(d - 1, 0),), -1.0, dtype=torch.float64)
        return TridiagMatrix(o, torch.full((d,), 2.0, dtype=torch.float64), o.clone())

    def _ptrs(self):
        # d = 1: the off-diagonal arrays are empty; hand the kernels a valid pointer
        sp = self.sub.data_ptr() if self.sub.numel() else self.diag.data_ptr()
        up = self.sup.data_ptr() if self.sup.numel() else self.diag.data_ptr()
        return sp, self.diag.data_ptr(), up

    def one_norm(self) -> float:
        s, dg, u = self.sub.abs(), self.diag.abs(), self.sup.abs()
        col = dg.clone()
        col[1:] += u
        col[:-1] += s
        return float(col.max()) if self.d else 0.0


def _block(V: ArrayLike, d: int):
    dV, host = _to_device(V)
    vec = dV.dim() == 1
    V2 = (dV.reshape(d, 1) if vec else dV).contiguous()
    if V2.shape[0] != d:
        raise PfError(Errc.LengthMismatch, "vector length mismatch")
    return V2, host, vec


def _unblock(out: torch.Tensor, host: bool, vec: bool):
    out = out.reshape(-1) if vec else out
    return out.cpu().numpy() if host else out


def tridiag_matvec(t: TridiagMatrix, V: ArrayLike):
    eng = engine()
    V2, host, vec = _block(V, t.d)
    out = torch.empty_like(V2)
    s, dg, u = t._ptrs()
    rc = N.lib.pf_tridiag_matvec_batched(eng.h, t.d, V2.shape[1], s, dg, u, V2.data_ptr(), V2.shape[1],
                                         out.data_ptr(), V2.shape[1])
    if rc:
        _raise(rc, N.PfStatus(), False)
    return _unblock(out, host, vec)


def thomas_solve(t: TridiagMatrix, rhs: ArrayLike):
    """thomas_solve (action.cpp:100-118) for every column of rhs."""
    eng = engine()
    R, host, vec = _block(rhs, t.d)
    out = torch.empty_like(R)
    st = N.PfStatus()
    s, dg, u = t._ptrs()
    rc = N.lib.pf_thomas_solve_batched(eng.h, t.d, R.shape[1], s, dg, u, R.data_ptr(), R.shape[1], out.data_ptr(),
                                       R.shape[1], C.byref(st))
    if rc:
        _raise(rc, st, False)
    return _unblock(out, host, vec)


def pentadiag_solve(sub2: ArrayLike, sub1: ArrayLike, diag: ArrayLike, super1: ArrayLike, super2: ArrayLike,
                    rhs: ArrayLike):
    """pentadiag_solve (action.cpp:170-202): banded LU without pivoting, every column of rhs."""
    eng = engine()
    bands = [_to_device(b)[0].reshape(-1) for b in (sub2, sub1, diag, super1, super2)]
    d = int(bands[2].numel())
    R, host, vec = _block(rhs, d)
    out = torch.empty_like(R)
    st = N.PfStatus()
    ptrs = [b.data_ptr() if b.numel() else bands[2].data_ptr() for b in bands]
    rc = N.lib.pf_pentadiag_solve_batched(eng.h, d, R.shape[1], *ptrs, R.data_ptr(), R.shape[1], out.data_ptr(),
                                          R.shape[1], C.byref(st))
    if rc:
        _raise(rc, st, False)
    return _unblock(out, host, vec)


def tridiag_action(method, t: TridiagMatrix, V: ArrayLike, substeps: int = 1, form: Optional[int] = None,
                   flags: int = 0):
    """substep_action (action.cpp:327-339) -- action_eval for substeps = 1 -- on every column of V:
    v <- r(A / N) v, N = substeps, with one factorization per shift reused (ActionOperator)."""
    m = _resolve_method(method)
    pk = PackedMethod(m, form)
    eng = engine()
    V2, host, vec = _block(V, t.d)
    out = torch.empty_like(V2)
    st = N.PfStatus()
    s, dg, u = t._ptrs()
    rc = N.lib.pf_tridiag_action(eng.h, pk.ptr(), t.d, V2.shape[1], s, dg, u, V2.data_ptr(), V2.shape[1],
                                 int(substeps), out.data_ptr(), V2.shape[1], flags, C.byref(st))
    if rc:
        _raise(rc, st, False)
    return _unblock(out, host, vec)
