"""Large batched LU throughput: 8 shifted systems I - c B (certified, no exchanges) of order n,
timed with CUDA events; fraction of the measured FP64 DMMA peak at (2/3) n^3 flops per system."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, _native as N, workloads as W  # noqa: E402

peak = float(N.lib.pf_probe_dmma_tflops(0))
full = torch.from_numpy(W.cfg3()).cuda()
for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096"])]:
    if n <= full.shape[0]:
        B = full[:n, :n].contiguous() * (2.0 ** -8)
    else:  # larger than cfg3: a seeded Gaussian of the same scale
        g = torch.Generator(device="cuda").manual_seed(n)
        B = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) * (2.0 / n)
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    Ms = torch.stack([I - c * B for c in (0.1, -0.1, 0.2, -0.2, 0.3, -0.3, 0.4, -0.4)])
    for _ in range(2):  # warm-up: the second call captures the recursion's launch graph
        api.DenseLu(Ms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        api.DenseLu(Ms)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 8 * (2.0 / 3.0) * n ** 3 / (ms * 1e-3) / 1e12
    print(json.dumps({"n": n, "systems": 8, "ms": ms, "tflops": tf, "frac_of_dmma_peak": tf / peak}))
