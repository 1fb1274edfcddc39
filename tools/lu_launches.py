"""Target for an ncu launch list of the large LU: one batched DenseLu of 8 shifted systems of order n."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
A = torch.from_numpy(W.cfg3()).cuda()[:n, :n].contiguous()
B = A * (2.0 ** -8)
I = torch.eye(n, dtype=torch.float64, device="cuda")
Ms = torch.stack([I - c * B for c in (0.1, -0.1, 0.2, -0.2, 0.3, -0.3, 0.4, -0.4)])
torch.cuda.synchronize()
lu = api.DenseLu(Ms)
torch.cuda.synchronize()
print("done", n)
