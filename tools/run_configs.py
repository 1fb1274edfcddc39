"""Full-size BASELINE configs 3-5 on one GPU: time (CUDA events) + size-independent checks against
an independent referee (torch.linalg.matrix_exp / eigh, fp64 on the device)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_03714_b200 import api, methods as M, workloads as W  # noqa: E402

which = sys.argv[1:] or ["cfg3", "cfg4", "cfg5"]
res = {}
dev = torch.device("cuda")


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


def rel1(a, b):
    return float((a - b).abs().sum(0).max() / b.abs().sum(0).max())


if "cfg3" in which:
    t0 = time.time()
    A = torch.from_numpy(W.cfg3()).to(dev)
    (E, P), ms = timed(lambda: api.expm_phi1(A, "R8"))
    ref = torch.linalg.matrix_exp(A)
    I = torch.eye(A.shape[0], dtype=torch.float64, device=dev)
    flops = 8 * (8 / 3) * 4096 ** 3 + 8 * 2 * 2 * 4096 ** 3
    res["cfg3"] = {"ms": ms, "evals_per_s": 1e3 / ms, "tflops": flops / ms / 1e9,
                   "rel_vs_torch_matrix_exp": rel1(E, ref),
                   "phi1_identity_rel": rel1(P @ A, E - I), "setup_s": time.time() - t0}
    print(json.dumps({"cfg3": res["cfg3"]}), flush=True)
    del A, E, P, ref

if "cfg5" in which:
    A = torch.from_numpy(W.cfg5()).to(dev)
    (Cm, S), ms = timed(lambda: api.cossin(A, "R8"))
    w, v = torch.linalg.eigh(A)
    Cref = (v * torch.cos(w)[:, None, :]) @ v.transpose(1, 2)
    Sref = (v * torch.sin(w)[:, None, :]) @ v.transpose(1, 2)
    I = torch.eye(512, dtype=torch.float64, device=dev)
    flops = 256 * (1 + 4 * 4 / 3 + 1 + 36) * 2 * 512 ** 3
    res["cfg5"] = {"ms": ms, "evals_per_s": 256e3 / ms, "tflops": flops / ms / 1e9,
                   "cos_max_abs_err_vs_eigh": float((Cm - Cref).abs().max()),
                   "sin_max_abs_err_vs_eigh": float((S - Sref).abs().max()),
                   "pythagoras_max": float((Cm @ Cm + S @ S - I).abs().max())}
    print(json.dumps({"cfg5": res["cfg5"]}), flush=True)
    del A, Cm, S, w, v, Cref, Sref

if "cfg4" in which:
    a_np, v_np = W.cfg4()
    A = torch.from_numpy(a_np).to(dev)
    V = torch.from_numpy(v_np).to(dev)
    del a_np
    nsub = M.substeps_for(4.0, M.THETA_U53["R8"])
    out, ms = timed(lambda: api.action(A, V, "R8", substeps=nsub))
    ref = torch.linalg.matrix_exp(A) @ V
    n, k = V.shape
    flops = 8 * (2 / 3) * n ** 3 + nsub * 8 * 2 * n * n * k + nsub * 2 * n * n * k
    res["cfg4"] = {"ms": ms, "evals_per_s": 1e3 / ms, "tflops": flops / ms / 1e9, "substeps": nsub,
                   "rel_vs_matrix_exp_V": rel1(out, ref)}
    print(json.dumps({"cfg4": res["cfg4"]}), flush=True)
