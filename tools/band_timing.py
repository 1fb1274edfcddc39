"""f2 banded action throughput: R8 residual substep_action on a block of k vectors of a tridiagonal
A (heat operator trid121 * h scaled), d rows, on the GPU (CUDA events) vs the CPU oracle on a column
sample. Prints one JSON line.

Traffic model (HBM bytes per substep) of the fused step (band.cu band_action_*_kernel): V is read
by the forward sweep and again by the backward sums, each shift's forward result Y_t is written
once and read back once, the next iterate is written once: 8 (2 P + 3) d k bytes. min_traffic
is the same less the second V read (a kernel that kept V's rows on chip): 8 (2 P + 2) d k."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_03714_b200 import api, methods as M  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
k = int(sys.argv[2]) if len(sys.argv) > 2 else 256
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
m = M.catalog("R8")
P = sum(1 for c in m.shift_doubles() if c != 0.0)
h = 0.25
t = api.TridiagMatrix(-h * np.ones(d - 1), 2 * h * np.ones(d), -h * np.ones(d - 1))
V = torch.from_numpy(np.random.default_rng(0).standard_normal((d, k))).cuda()
api.tridiag_action(m, t, V, steps, M.RESIDUAL)  # warm-up
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record()
for _ in range(reps):
    out = api.tridiag_action(m, t, V, steps, M.RESIDUAL)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
bytes_model = steps * 8.0 * d * k * (2 * P + 3)
min_bytes = steps * 8.0 * d * k * (2 * P + 2)  # per column: write+read one sweep per shift, read/write the vector
# CPU oracle on a column sample
from oracle import oracle as O  # noqa: E402

ks = 4
vs = V[:, :ks].cpu().numpy()
om = O.OMethod.from_method(m, 1)
t0 = time.perf_counter()
ref = O.tridiag_action(-h * np.ones(d - 1), 2 * h * np.ones(d), -h * np.ones(d - 1), vs, om, steps)
cpu_s = time.perf_counter() - t0
exact = bool(np.array_equal(out[:, :ks].cpu().numpy(), ref))
print(json.dumps({"workload": "tridiag action R8 residual", "d": d, "k": k, "substeps": steps, "ms": ms,
                  "vectors_per_s": k / (ms * 1e-3), "model_GBps": bytes_model / (ms * 1e-3) / 1e9,
                  "min_traffic_GBps": min_bytes / (ms * 1e-3) / 1e9,
                  "cpu_vectors_per_s_1thread": ks / cpu_s, "bitwise_equal_to_oracle_sample": exact}))
