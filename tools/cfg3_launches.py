"""ncu target: one cfg3 exp + phi1 evaluation (4096^2, R8, residual, pair mode) after a warm-up."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, workloads as W  # noqa: E402

A = torch.from_numpy(W.cfg3()).cuda()
api.expm_phi1(A, "R8")
torch.cuda.synchronize()
api.expm_phi1(A, "R8")
torch.cuda.synchronize()
print("done")
