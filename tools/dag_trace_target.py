"""ncu / PF_DAG_TRACE target: one certified batched DenseLu of `systems` shifted cfg3 slices of order n (argv: n systems)."""
import sys; sys.path.insert(0, '.')
import torch
from paper_2210_03714_b200 import api, workloads as W
full = torch.from_numpy(W.cfg3()).cuda()
n = int(sys.argv[1]); ns = int(sys.argv[2])
B = full[:n, :n].contiguous() * (2.0 ** -8)
I = torch.eye(n, dtype=torch.float64, device="cuda")
Ms = torch.stack([I - (0.1 * (1 + q // 2)) * (1 if q % 2 == 0 else -1) * B for q in range(ns)])
api.DenseLu(Ms); torch.cuda.synchronize()
print("done")
