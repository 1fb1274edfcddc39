"""Per-grid-point errors of the acceptance dominance window (acceptance_main.cpp:176-204) for R8 in
pair mode (default), R8 per shift (the reference's operation order), R8 residual, and taylor8."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_03714_b200 import api, drivers as D, methods as M, _native as N  # noqa: E402

a = D.make_dense_matrix(D.MatrixSpec("randn", 100, 1))
scale = D.two_norm_est(a)
for name, grid in (("window", D.log_grid(0.3, 3.0, 12)), ("low", D.log_grid(0.01, 0.2, 8))):
    Bs = np.stack([a * (h / scale) for h in grid])
    dB = torch.from_numpy(Bs).cuda()
    m8 = M.catalog("R8")
    vals = {
        "R8 pair": api.eval_dense(m8, dB).cpu().numpy(),
        "R8 per-shift": api.eval_dense(m8, dB, flags=N.PF_FLAG_PER_SHIFT).cpu().numpy(),
        "R8 residual": api.eval_dense(M.to_residual_form(m8), dB).cpu().numpy(),
        "R4": api.eval_dense(M.catalog("R4"), dB).cpu().numpy(),
        "taylor8": D.taylor8(dB).cpu().numpy(),
        "pade4": D.pade4(dB).cpu().numpy(),
    }
    print(name, "form R8 =", m8.form)
    for gi, h in enumerate(grid):
        errs = D.dense_errors("exp", Bs[gi], [v[gi] for v in vals.values()])
        print("h %.4f " % h + " ".join("%s %.3e" % (k, e) for k, e in zip(vals, errs)))
