"""Certified batched LU time vs the number of systems (same n): latency floor vs work (DAG at 1024 / 2048)."""
import sys, json
sys.path.insert(0, '.')
import torch
from paper_2210_03714_b200 import api, workloads as W
full = torch.from_numpy(W.cfg3()).cuda()
for n in (1024, 2048):
    B = full[:n, :n].contiguous() * (2.0 ** -8)
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    for ns in (1, 2, 4, 8, 16, 32):
        cs = [0.1 * (1 + q // 2) * (1 if q % 2 == 0 else -1) for q in range(ns)]
        Ms = torch.stack([I - c * B for c in cs])
        for _ in range(2): api.DenseLu(Ms)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): api.DenseLu(Ms)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"n": n, "systems": ns, "ms": ms, "tflops": ns * 2 / 3 * n ** 3 / ms / 1e9}))
