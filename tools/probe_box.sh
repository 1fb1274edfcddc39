#!/bin/bash
# One-shot box probe: FP64 DMMA/DFMA rates, cuBLAS DGEMM peak (probe only), host cores.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu >> gpurun_out/nproc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_fp64 tools/probe_fp64.cu && /tmp/probe_fp64 > gpurun_out/probe_fp64.jsonl 2>&1
python - <<'PY' > gpurun_out/probe_dgemm.jsonl 2>&1
import torch, json
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"probe": "cublas_dgemm", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
# batched 128x128 dgemm
a = torch.randn(4096, 128, 128, dtype=torch.float64, device='cuda'); b = torch.randn_like(a)
for _ in range(3): torch.bmm(a, b)
torch.cuda.synchronize(); best = 1e9
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); c = torch.bmm(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"probe": "cublas_dgemm_batched_128", "batch": 4096, "ms": best, "tflops": 2 * 4096 * 128**3 / best / 1e9}))
PY
cat gpurun_out/probe_fp64.jsonl gpurun_out/probe_dgemm.jsonl
