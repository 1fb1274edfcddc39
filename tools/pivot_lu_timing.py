"""Blocked partial-pivoting LU (pivot_lu.cu + pf_large.cu rlu_pivot) throughput: 8 non-dominant systems
I - 3 G / sqrt(n) (G seeded Gaussian; the certificate rejects them, so every system pivots), timed with
CUDA events (DenseLu = copy + factor); fraction of the live FP64 DMMA probe at (2/3) n^3 flops per
system. PF_PIVOT_UNBLOCKED=1 times the previous one-CTA unblocked kernel instead (small n only)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, _native as N  # noqa: E402

peak = float(N.lib.pf_probe_dmma_tflops(0))
for n in [int(x) for x in (sys.argv[1:] or ["512", "1024", "2048", "4096"])]:
    g = torch.Generator(device="cuda").manual_seed(n)
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    Ms = torch.stack([I - 3.0 * torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
                      for _ in range(8)])
    api.DenseLu(Ms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        lu = api.DenseLu(Ms)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    piv = lu.piv.cpu()
    swaps = int((piv != torch.arange(n, dtype=piv.dtype)).sum())
    tf = 8 * (2.0 / 3.0) * n ** 3 / (ms * 1e-3) / 1e12
    print(json.dumps({"n": n, "systems": 8, "pivoted": True, "row_exchanges": swaps, "ms": ms, "tflops": tf,
                      "frac_of_dmma_peak": tf / peak}), flush=True)
