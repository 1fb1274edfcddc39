"""Small inputs through the round-2 kernels, for compute-sanitizer (memcheck / racecheck / synccheck):
TMA GEMM (ragged, batched, split-K) and its cp.async fallback, the blocked pivoting LU (one CTA and a
2-CTA cluster), the device-scheduled LU, the large-n 1-norm, cos/sin (GEMM sum/diff epilogue), the
fused small kernel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_03714_b200 import api, _native as N  # noqa: E402

rng = np.random.default_rng(0)
dev = "cuda"
eng = api.engine()
for (m, n, k, b, lda, ldb) in [(130, 66, 34, 3, 34, 66), (300, 64, 2048, 1, 2048, 64), (100, 37, 61, 1, 61, 37)]:
    A = torch.from_numpy(rng.standard_normal((b, m, lda))).to(dev)
    B = torch.from_numpy(rng.standard_normal((b, k, ldb))).to(dev)
    C = torch.zeros(b, m, n, dtype=torch.float64, device=dev)
    assert N.lib.pf_gemm_batched(eng.h, m, n, k, b, 1.0, A.data_ptr(), lda, m * lda, B.data_ptr(), ldb, k * ldb, 1.0,
                                 C.data_ptr(), n, m * n, 0.0) == 0
for n in (200, 300):
    mm = np.eye(n) - 3.0 * rng.standard_normal((n, n)) / np.sqrt(n)
    api.DenseLu(mm).factors()
n = 1024
Bm = rng.standard_normal((n, n)) * (0.5 / n)
api.DenseLu(np.stack([np.eye(n) - c * Bm for c in (0.5, -0.5)])).factors()
api.expm(torch.from_numpy(rng.standard_normal((1, 600, 600)) * 0.01).to(dev), "R8")
S = rng.standard_normal((2, 256, 256)) * 0.05
api.cossin(torch.from_numpy(S + S.transpose(0, 2, 1)).to(dev), "R8")
api.expm(torch.from_numpy(rng.standard_normal((4, 128, 128))).to(dev), "R4")
torch.cuda.synchronize()
print("sanitize target done")
