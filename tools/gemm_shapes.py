"""CUDA-event timing of the batched DMMA GEMM at the small shapes the large LU recursion issues."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api  # noqa: E402


def tm(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (m, n, k) in [(64, 64, 64), (64, 128, 64), (128, 128, 128), (256, 256, 256), (64, 2048, 64), (2048, 64, 64),
                  (512, 512, 512), (1024, 1024, 1024)]:
    a = torch.randn(8, m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(8, k, n, dtype=torch.float64, device="cuda")
    c = torch.zeros(8, m, n, dtype=torch.float64, device="cuda")
    us = tm(lambda: api.gemm(a, b, Cm=c))
    print("batch 8 gemm %4dx%4dx%4d: %8.1f us  %6.2f TF/s" % (m, n, k, us, 8 * 2 * m * n * k / us / 1e6))
