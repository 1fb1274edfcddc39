#!/usr/bin/env python
"""Headline benchmark: BASELINE.json configs[1] -- batched expm of 4096 independent 128x128 FP64
matrices (entries iid N(0,1), 1-norm uniform in [0.5, 8]), s = 4 (R4, headline) and s = 8 (R8)
partial-fraction methods with scaling and squaring, residual form.

A "step" = one pf_expm_batched call over the whole batch (norm -> j_b -> s shifted LU + solves ->
weighted sum -> j_b squarings, all inside one fused kernel per matrix). The K timed steps run back
to back on the device (PF_FLAG_ASYNC); every step's device status is kept (sticky) and checked once
after the region, so a failing step still fails the run. `e2e` times the same through the public
host-buffer API (api.HostPipeline: pinned H2D of the batch, the evaluation, D2H of the result,
every step). `roofline` divides the algorithmic FLOPs of one launch by that launch's median CUDA-event
time (executed FLOPs beside them) against the FP64 DMMA peak probed live on this GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--method R4|R8]

--gpus N > 1 without a torchrun environment re-launches this script under torch.distributed.run
with N ranks (one per GPU); batch-sharded weak scaling: every rank evaluates its own 4096-matrix
batch, no collective on the data path (the matrices are independent); time = max over ranks.

Parity: the timed run's outputs are compared, matrix by matrix, with THE REFERENCE BUILD
(oracle/_ref: /root/reference/proj/core/src compiled unmodified; eval_dense + DenseMatrix::mul)
over the whole batch; the same run is the cpu_baseline (kind "reference").
`--impl reference` times that reference build on the host cores over the whole batch per step
(all host threads, parallel over the batch as cli.cpp:314), on rank 0 only.
Secondary lines (N = 1): the R8 variant of the headline, and clocked single-GPU lines for
configs[2..4] (cfg3 exp+phi1 4096^2, cfg4 action 16384^2 x 64, cfg5 cos/sin 256 x 512^2) with a
reduced-unit reference CPU timing extrapolated by the SURVEY §8(d) FLOP model.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_MAT = 128
BATCH = 4096


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--method", default="R4")
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-secondary", action="store_true", help="skip the R8 and cfg3/4/5 secondary lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference legs (cpu_baseline, parity)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: start N ranks on this node (one per GPU) and wait."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def host_cpu():
    """(threads usable by this process, CPU model string)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


def reference_backend():
    """THE REFERENCE BUILD (oracle/_ref) when present, else the restatement pinned to it bit for bit."""
    from oracle import ref as R

    if R.available():
        try:
            R.lib()
            return "reference"
        except Exception:
            pass
    return "port"


def cpu_expm_batched(a, method_name, threads):
    """expm over a batch on the host: reference build (eval_dense + DenseMatrix::mul) or the port."""
    from paper_2210_03714_b200 import methods as M

    th = M.THETA_U53[method_name]
    if reference_backend() == "reference":
        from oracle import ref as R

        return R.expm_batched(R.RefMethod.catalog(method_name), a, th, M.RESIDUAL, threads=threads)
    from oracle import oracle as O

    return O.expm_batched(a, O.OMethod.from_method(M.catalog(method_name), M.RESIDUAL), th, threads=threads)


def parity_vs_reference(got, js_got, a, method_name, threads):
    """Whole-batch comparison with the reference build; returns (parity dict, cpu seconds, kind)."""
    t0 = time.perf_counter()
    want, js = cpu_expm_batched(a, method_name, threads)
    dt = time.perf_counter() - t0
    num = np.abs(got - want).sum(axis=1).max(axis=1)
    den = np.abs(want).sum(axis=1).max(axis=1)
    rel = num / den
    kind = reference_backend()
    return ({"vs": "oracle/_ref (reference build)" if kind == "reference" else "oracle restatement (pinned)",
             "max_rel_1norm": float(rel.max()), "mean_rel_1norm": float(rel.mean()),
             "squarings_equal": bool(np.array_equal(np.asarray(js_got), js)), "n_compared": int(len(rel)),
             "tol": 1e-11, "pass": bool(rel.max() <= 1e-11 and np.array_equal(np.asarray(js_got), js))},
            dt, kind)


def algorithmic_flops(js: np.ndarray, n_shifts: int, n: int = N_MAT) -> float:
    """per matrix (P * 8/3 + 2 j_b) n^3 (residual LU+TRSM per shift, one GEMM per squaring)."""
    return float(np.sum(n_shifts * (8.0 / 3.0) + 2.0 * js.astype(np.float64)) * n ** 3)


def executed_flops(js: np.ndarray, n_shifts: int, n: int = N_MAT) -> float:
    """What the kernel performs in pair mode (every cfg2 matrix is certified, since
    ||2^-j A||_1 <= theta): B^2 (2n^3), per (c, -c) pair one LU of I - c^2 B^2 and one TRSM with a
    dense RHS (8/3 n^3), the final A.V product (2n^3), then 2 j_b n^3 of squaring."""
    pairs = n_shifts // 2
    return float(np.sum(2.0 + pairs * (8.0 / 3.0) + 2.0 + 2.0 * js.astype(np.float64)) * n ** 3)


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in names.items():
                    if mask & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.01)  # ~10 samples over a 100 ms timed region

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def load_profile_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary, if any."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("small_eval_kernel_bytes_per_launch"), d
        except Exception:
            pass
    return None, None


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) of the headline workload on the host
    cores: every step evaluates the whole batch (all host threads, parallel over the batch)."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2210_03714_b200 import workloads as W

    cores, model = host_cpu()
    kind = reference_backend()
    a = W.cfg2(batch=args.batch)
    for _ in range(args.warmup):
        cpu_expm_batched(a, args.method, cores)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        cpu_expm_batched(a, args.method, cores)
        times.append(time.perf_counter() - t)
    per = float(np.mean(times))
    value = args.batch / per
    what = ("reference build oracle/_ref (/root/reference/proj/core/src compiled unmodified, -O3 -DNDEBUG): "
            "eval_dense + DenseMatrix::mul" if kind == "reference" else "oracle restatement of dense.cpp (pinned)")
    line = {"impl": "reference", "metric": "f(A) evals/sec (FP64)", "value": value, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2_batched_expm_%dx128x128_%s" % (args.batch, args.method), "batch": args.batch,
                       "n": N_MAT, "method": args.method, "form": "residual"},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": kind, "cpu_model": model,
                             "sample": "the whole %d-matrix batch per step, %d host threads (affinity), %s" % (
                                 args.batch, cores, what)},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def time_ours(args, method_name, A, rank, world, local, dist, eng):
    import torch
    from paper_2210_03714_b200 import _native as N, api, methods as M

    m = M.catalog(method_name)
    pk = api.PackedMethod(m, M.RESIDUAL)
    th = M.THETA_U53[method_name]
    bsz = A.shape[0]
    out = torch.empty_like(A)
    j_out = torch.empty(bsz, dtype=torch.int32, device=A.device)
    st = N.PfStatus()
    import ctypes as C

    def step(flags=0, a=A, o=out):
        rc = N.lib.pf_expm_batched(eng.h, pk.ptr(), th, N_MAT, bsz, a.data_ptr(), N_MAT, N_MAT * N_MAT, None,
                                   j_out.data_ptr(), o.data_ptr(), N_MAT, N_MAT * N_MAT, flags, C.byref(st))
        if rc:
            raise RuntimeError("pf_expm_batched failed: %d" % rc)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    js = j_out.cpu().numpy()
    flops = algorithmic_flops(js, m.processors())
    exe_flops = executed_flops(js, m.processors())

    # --- timed region: K steps, barrier + sync both sides, CUDA events on the context stream
    stream = torch.cuda.current_stream()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = eng.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # steps back to back (PF_FLAG_ASYNC: no host round trip per step); the device status of every step
    # is kept (sticky) and checked once after the region -- a failed step still fails the run
    N.lib.pf_context_set_sticky_status(eng.h, 1)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step(N.PF_FLAG_ASYNC)
        e1.record(stream)
        torch.cuda.synchronize()
    pending = N.lib.pf_context_pending_error(eng.h)
    N.lib.pf_context_set_sticky_status(eng.h, 0)
    if pending:
        raise RuntimeError("a timed pf_expm_batched step reported a device error (%d)" % pending)
    launches = eng.launch_count() - l0
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # --- dominant-kernel duration (single launch per step; PF_FLAG_ASYNC = no status read)
    kt = []
    for _ in range(max(3, args.steps)):
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        step(N.PF_FLAG_ASYNC)
        k1.record(stream)
        torch.cuda.synchronize()
        kt.append(k0.elapsed_time(k1))
    kernel_ms = float(np.median(kt))  # median of the individually timed launches (robust to one slow launch)
    return {"ms": ms, "flops": flops, "exe_flops": exe_flops, "kernel_ms": kernel_ms, "launches": launches,
            "clocks": clk.summary(), "js": js, "out": out}


def time_e2e(args, method_name, A_host_pinned, eng):
    """Public-API path with host buffers: H2D of the inputs, expm, D2H of the result, every step."""
    import torch
    from paper_2210_03714_b200 import api

    hO = torch.empty(A_host_pinned.shape, dtype=torch.float64, pin_memory=True)
    stream = torch.cuda.current_stream()
    # public API for host-resident batches: H2D / evaluation / D2H overlapped across chunks
    pipe = api.HostPipeline(A_host_pinned.shape[1], A_host_pinned.shape[0], chunk=256, streams=4)

    def step():
        # every step: pinned H2D of the batch, the evaluation, D2H of the result (public API); the
        # device status of all steps is checked by finish() (one synchronisation)
        pipe.submit(A_host_pinned, hO, method_name)

    for _ in range(max(1, args.warmup)):
        step()
    pipe.finish()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    pipe.finish()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    nbytes = A_host_pinned.numel() * 8
    return ms, nbytes, nbytes


def timed_region(fn, steps, local, stream):
    """K calls bracketed by synchronisation, CUDA events on the launching stream, clocks sampled."""
    import torch

    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, clk.summary()


def large_config_lines(peak, local, cores):
    """Clocked single-GPU lines for BASELINE configs[2..4] plus a reduced-unit reference CPU timing
    extrapolated by the SURVEY §8(d) FLOP model (the full CPU runs take hours)."""
    import torch
    from paper_2210_03714_b200 import api, methods as M, workloads as W

    stream = torch.cuda.current_stream()
    eng = api.engine()
    lines = []
    kind = reference_backend()

    def ref_unit(n, fn, reps=1):
        t = time.perf_counter()
        for _ in range(reps):
            fn(n)
        return (time.perf_counter() - t) / reps

    def mk(name, workload, unit_s, ms, clocks, alg, exe, launches, cpu, extra):
        tf = alg / (ms * 1e-3) / 1e12
        te = exe / (ms * 1e-3) / 1e12
        d = {"config": name, "workload": workload, "value": 1e3 / ms * unit_s, "unit": "evals/s",
             "ms_per_eval": ms / unit_s if unit_s > 1 else ms, "ms_per_step": ms, "clocks": clocks,
             "algorithmic_tflops": tf, "frac_algorithmic": tf / peak, "executed_tflops": te,
             "frac_executed": te / peak, "flops_algorithmic": alg, "flops_executed": exe,
             "gpu_launches_per_step": launches, "cpu_baseline": cpu}
        d.update(extra)
        return d

    # ---- cfg3: exp and phi1 of one 4096^2, R8 shifts, j = 8
    from oracle import ref as R

    A = torch.from_numpy(W.cfg3()).cuda()
    n = 4096
    fn = lambda: api.expm_phi1(A, "R8")  # noqa: E731
    fn()
    l0 = eng.launch_count()
    fn()
    torch.cuda.synchronize()
    launches = eng.launch_count() - l0
    ms, clk = timed_region(fn, 3, local, stream)
    alg = 8 * (8 / 3) * n ** 3 + 8 * 2 * 2 * n ** 3
    exe = (2 + 4 * (8 / 3) + 2 * 2 + 8 * 2 * 2) * n ** 3
    cpu = None
    if kind == "reference":
        nu = 1024
        b = W.scaled_to_one_norm(W.randn_matrix(nu, 3), 0.2)
        mm = np.eye(nu) - 0.2 * b
        t_shift = ref_unit(nu, lambda _: R.lu_solve_matrix(mm, b))
        t_mul = ref_unit(nu, lambda _: R.mul(b, b))
        scale = (n / nu) ** 3
        waves = math.ceil(8 / min(8, cores))
        est = waves * t_shift * scale + 16 * t_mul * scale
        cpu = {"value": 1.0 / est, "unit": "evals/s", "cores": min(8, cores), "kind": "reference",
               "sample": "reduced unit, extrapolated: reference DenseLu + solve_matrix (one residual shift) and "
                         "DenseMatrix::mul at n = 1024 (%.2f s, %.2f s), x (4096/1024)^3; 8 shifts over "
                         "workers = min(8, cores) (dense.cpp:202), 16 single-threaded products" % (t_shift, t_mul)}
    lines.append(mk("cfg3", "exp+phi1 of one 4096^2, R8 shifts, j = 8, residual", 1, ms, clk, alg, exe, launches, cpu,
                    {"executed_basis": "pair mode: B^2, 4 pair LU+TRSM, 2 combine products, 16 doubling GEMMs"}))
    del A

    # ---- cfg5: cos/sin of 256 x 512^2, R8 pairs, j = 12
    A = torch.from_numpy(W.cfg5()).cuda()
    n, bsz = 512, 256
    fn = lambda: api.cossin(A, "R8")  # noqa: E731
    fn()
    l0 = eng.launch_count()
    fn()
    torch.cuda.synchronize()
    launches = eng.launch_count() - l0
    ms, clk = timed_region(fn, 3, local, stream)
    _, _, js = api.cossin(A, "R8", return_squarings=True)
    jm = float(js.double().mean())
    alg = bsz * (1 + 4 * 4 / 3 + 1 + 3 * jm) * 2 * n ** 3
    exe = bsz * (1 + 4 * 4 / 3 + 1 + 2 * jm) * 2 * n ** 3
    cpu = None
    if kind == "reference":
        from oracle import oracle as O

        nu = 256
        a1 = W.cfg5(batch=1, n=nu)
        pm = O.OPair.from_pair(M.pair_method(M.catalog("R8")))
        t_unit = ref_unit(nu, lambda _: O.cossin(a1[0], pm, M.THETA_U53["R8"], j_fixed=int(jm + 0.5)))
        per_mat = t_unit * (n / nu) ** 3
        est = per_mat * math.ceil(bsz / cores)
        cpu = {"value": bsz / est, "unit": "evals/s", "cores": cores, "kind": "port",
               "sample": "reduced unit, extrapolated: one cos/sin evaluation at n = 256 with j = %d on the "
                         "restatement (the reference has no cos/sin composition; its LU/solve/mul are pinned bit for "
                         "bit), x (512/256)^3, batch of 256 over %d threads" % (int(jm + 0.5), cores)}
    lines.append(mk("cfg5", "cos/sin of 256 x 512^2 symmetric, R8 pairs, C^2-S^2 / 2SC", bsz, ms, clk, alg, exe,
                    launches, cpu, {"mean_squarings": jm,
                                    "executed_basis": "C^2 - S^2 formed as (C - S)(C + S): 2 GEMMs per doubling"}))
    del A

    # ---- cfg4: exp(tA) V, 16384^2, k = 64, N = 42
    a, v = W.cfg4()
    nsub = M.substeps_for(W.one_norm(a), M.THETA_U53["R8"])
    A = torch.from_numpy(a).cuda()
    V = torch.from_numpy(v).cuda()
    del a
    n, k = 16384, 64
    fn = lambda: api.action(A, V, "R8", substeps=nsub)  # noqa: E731
    fn()
    l0 = eng.launch_count()
    fn()
    torch.cuda.synchronize()
    launches = eng.launch_count() - l0
    ms, clk = timed_region(fn, 2, local, stream)
    alg = 8 * (2 / 3) * n ** 3 + nsub * 8 * 2 * n * n * k + nsub * 2 * n * n * k
    exe = 2 * n ** 3 + 4 * (2 / 3) * n ** 3 + nsub * 6 * 2 * n * n * k
    cpu = None
    if kind == "reference":
        nu = 1024
        au = W.randn_matrix(nu, 4) / np.sqrt(nu) - 2.0 * np.eye(nu)
        au *= 4.0 / W.one_norm(au) / nsub
        vu = W.randn(5, nu * k).reshape(nu, k)
        rm = R.RefMethod.catalog("R8")
        w = min(8, cores)
        t1 = ref_unit(nu, lambda _: R.dense_action(rm, au, vu, 1, M.RESIDUAL, workers=w))
        t2 = ref_unit(nu, lambda _: R.dense_action(rm, au, vu, 2, M.RESIDUAL, workers=w))
        t_step = max(t2 - t1, 1e-9)
        t_fac = max(t1 - t_step, 1e-9)
        est = t_fac * (n / nu) ** 3 + nsub * t_step * (n / nu) ** 2
        cpu = {"value": 1.0 / est, "unit": "evals/s", "cores": w, "kind": "reference",
               "sample": "reduced unit, extrapolated: the dense block action (reference DenseLu per shift factored "
                         "once, assemble_action order per column) at n = 1024, k = 64 with 1 and 2 substeps "
                         "(factor %.2f s, substep %.3f s), x (16384/1024)^3 for the LUs and ^2 per substep, "
                         "%d substeps, workers = %d" % (t_fac, t_step, nsub, w)}
    lines.append(mk("cfg4", "exp(tA)V, 16384^2 x 64, R8, N = %d substeps, factor once" % nsub, 1, ms, clk, alg, exe,
                    launches, cpu, {"substeps": nsub,
                                    "executed_basis": "pair mode: B^2, 4 pair LUs, per substep BX + 4 pair solves "
                                                      "+ B.V (6 x 2n^2k)"}))
    del A, V
    torch.cuda.empty_cache()
    return lines


def time_cfg3_sharded(local, dist, steps: int = 3):
    """cfg3 (exp + phi1 of one 4096^2, R8 shifts) with the s resolvents partitioned over the ranks
    (parallel.expm_phi1_sharded: one NCCL reduce before the doubling, the doubling split by rows
    with an all-gather per step -- f1). Every rank times the same evaluation; max over ranks."""
    import torch
    from paper_2210_03714_b200 import parallel as P, workloads as W

    A = torch.from_numpy(W.cfg3()).cuda()
    fn = lambda: P.expm_phi1_sharded(A, "R8", deterministic=False, distributed_doubling=True)  # noqa: E731
    fn()
    if dist:
        dist.barrier()
    stream = torch.cuda.current_stream()
    ms, clk = timed_region(fn, steps, local, stream)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del A
    n = 4096
    flops = 8 * (8 / 3) * n ** 3 + 8 * 2 * 2 * n ** 3
    return {"config": "cfg3", "workload": "exp+phi1 of one 4096^2, R8 shifts partitioned over the ranks "
                                          "(pairs, or single shifts when ranks > pairs), NCCL reduce, row-split "
                                          "doubling with all-gathers", "value": 1e3 / ms, "unit": "evals/s",
            "ms_per_eval": ms, "algorithmic_tflops": flops / (ms * 1e-3) / 1e12, "steps": steps, "clocks": clk,
            "scaling": "strong"}


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d" % (world, args.gpus))
    dist = None
    if world > 1:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    torch.cuda.set_device(local)
    from paper_2210_03714_b200 import _native as N, api, workloads as W

    eng = api.engine()
    peak_probe = float(N.lib.pf_probe_dmma_tflops(local))
    cores, model = host_cpu()
    # inputs: each rank evaluates its own cfg2-distributed batch (weak scaling; seeds offset by rank)
    a_np = W.cfg2(batch=args.batch, seed0=1000 + rank * args.batch)
    A = torch.from_numpy(a_np).cuda()
    main = time_ours(args, args.method, A, rank, world, local, dist, eng)
    secondary = None
    if not args.no_secondary:
        other = "R8" if args.method != "R8" else "R4"
        secondary = time_ours(args, other, A, rank, world, local, dist, eng)
        secondary["name"] = other
    hostA = torch.from_numpy(a_np).pin_memory()
    e2e_ms, h2d, d2h = time_e2e(args, args.method, hostA, eng)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # parity of the timed outputs against the reference build, whole batch (rank 0's shard at N > 1);
    # at N = 1 the same reference run is the cpu_baseline
    cpu, parity, parity2 = None, None, None
    if rank == 0 and not args.no_cpu:
        parity, dt, kind = parity_vs_reference(main["out"].cpu().numpy(), main["js"], a_np, args.method, cores)
        if world == 1:
            cpu = {"value": args.batch / dt, "unit": "evals/s", "cores": cores, "kind": kind, "cpu_model": model,
                   "sample": "the whole %d-matrix batch (%s, residual, scaling+squaring) once, %d host threads "
                             "(affinity), parallel over the batch (cli.cpp:314); %s" % (
                                 args.batch, args.method, cores,
                                 "reference build oracle/_ref: eval_dense + DenseMatrix::mul from "
                                 "/root/reference compiled unmodified" if kind == "reference"
                                 else "restatement pinned bit for bit to the reference")}
        if secondary is not None:
            parity2, _, _ = parity_vs_reference(secondary["out"].cpu().numpy(), secondary["js"], a_np,
                                                secondary["name"], cores)
    del main["out"]
    if secondary is not None:
        del secondary["out"]
    sharded = None
    if not args.no_secondary:
        sharded = time_cfg3_sharded(local, dist)
    large = None
    if rank == 0 and world == 1 and not args.no_secondary:
        del A
        torch.cuda.empty_cache()
        large = large_config_lines(peak_probe, local, cores)
    if dist:
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    traffic, _ = load_profile_traffic()

    def roof(res):
        achieved = res["flops"] / (res["kernel_ms"] * 1e-3) / 1e12
        executed = res["exe_flops"] / (res["kernel_ms"] * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": peak_probe, "unit": "TFLOP/s",
                "frac": achieved / peak_probe, "traffic": traffic,
                "flops_basis": "algorithmic (SURVEY §8(d): per matrix P*8/3 n^3 + 2 j_b n^3); pair mode executes "
                               "fewer -- see executed_*",
                "executed_achieved": executed, "executed_frac": executed / peak_probe,
                "executed_flops_per_launch": res["exe_flops"],
                "kernel": "small_eval_kernel (fused norm+LU+solve+accumulate+squaring)",
                "kernel_ms": res["kernel_ms"],
                "flops_per_launch": res["flops"],
                "peak_source": "FP64 DMMA.8x8x4 probe measured live on this GPU (MEASURED_PEAKS.json has no FP64 "
                               "figure); cuBLAS DGEMM 8192^3 on this pool: 35.5 TFLOP/s"}

    value = args.batch * world / (main["ms"] * 1e-3)
    line = {
        "metric": "f(A) evals/sec (FP64)",
        "value": value,
        "unit": "evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": main["ms"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "cfg2_batched_expm_%dx128x128_%s" % (args.batch, args.method), "batch": args.batch,
                   "n": N_MAT, "method": args.method, "form": "residual", "parallelism": "batch-sharded dp%d" % world,
                   "mean_squarings": float(main["js"].mean()),
                   "l2": "inputs %d MiB per rank > 126 MB L2" % (args.batch * N_MAT * N_MAT * 8 >> 20)},
        "roofline": roof(main),
        "parity": parity,
        "cpu_baseline": cpu,
        "e2e": {"value": args.batch * world / (e2e_ms * 1e-3), "unit": "evals/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": main["launches"],
        "clocks": main["clocks"],
        "fp64_peak_tflops_probe": peak_probe,
        "host": {"cpu_model": model, "threads": cores},
    }
    if secondary is not None:
        line["secondary"] = {"method": secondary["name"], "value": args.batch * world / (secondary["ms"] * 1e-3),
                             "unit": "evals/s", "ms_per_step": secondary["ms"], "roofline": roof(secondary),
                             "mean_squarings": float(secondary["js"].mean()), "parity": parity2,
                             "clocks": secondary["clocks"]}
    if large is not None:
        line["large_configs"] = large
    if sharded is not None:
        line["cfg3_shift_partitioned"] = sharded
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
