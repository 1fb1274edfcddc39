"""ncu target: one cfg5 cos/sin evaluation (256 x 512^2, R8 conjugate pairs) after a warm-up."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, workloads as W  # noqa: E402

A = torch.from_numpy(W.cfg5()).cuda()
api.cossin(A, "R8")
torch.cuda.synchronize()
torch.cuda.profiler.start()
api.cossin(A, "R8")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
