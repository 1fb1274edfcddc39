"""ncu targets outside the headline: one 4096^3 DMMA GEMM ("gemm") or one banded action (d 8192,
k 16384, R8 residual, 1 substep: "band"), each after a warm-up; profile the second launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_03714_b200 import api, methods as M  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "gemm"
if what == "gemm":
    a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    api.gemm(a, a, Cm=c)
    torch.cuda.synchronize()
    api.gemm(a, a, Cm=c)
else:
    d, k = 8192, 16384
    t = api.TridiagMatrix(-0.25 * np.ones(d - 1), 0.5 * np.ones(d), -0.25 * np.ones(d - 1))
    V = torch.randn(d, k, dtype=torch.float64, device="cuda")
    api.tridiag_action(M.catalog("R8"), t, V, 1, M.RESIDUAL)
    torch.cuda.synchronize()
    api.tridiag_action(M.catalog("R8"), t, V, 1, M.RESIDUAL)
torch.cuda.synchronize()
print("done", what)
