"""Minimal target for `ncu --set full`: one cfg2 batched expm call (R4 or R8) after a warm-up."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, workloads as W  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "R4"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
a = torch.from_numpy(W.cfg2(batch=batch)).cuda()
out = torch.empty_like(a)
api.expm(a, method, out=out)  # warm-up
torch.cuda.synchronize()
api.expm(a, method, out=out)  # profiled
torch.cuda.synchronize()
print("done", method, batch)
