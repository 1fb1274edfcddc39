"""ncu target: build the cfg4 action operator (16384^2, R8, 8 shifted LUs), then profile one substep
only (cudaProfilerStart/Stop around op.apply; run ncu with --profile-from-start off)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, methods as M, workloads as W  # noqa: E402

a_np, v_np = W.cfg4()
A = torch.from_numpy(a_np).cuda()
V = torch.from_numpy(v_np).cuda()
del a_np
op = api.ActionOperator(A, "R8", 42, M.RESIDUAL)
op.apply(V)
torch.cuda.synchronize()
torch.cuda.profiler.start()
op.apply(V)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
