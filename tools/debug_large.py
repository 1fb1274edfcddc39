import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from oracle import oracle as O
from paper_2210_03714_b200 import api, methods as M, workloads as W

for n, norm in [(40, 50.0), (100, 0.1), (200, 60.0)]:
    b = W.scaled_to_one_norm(W.randn_matrix(n, 77 + n), norm)
    mm = np.eye(n) - 0.2 * b
    lu = api.DenseLu(mm)
    LU, piv = lu.factors()
    for k in (1, 7, 64, 70):
        rhs = W.randn(5, n * k).reshape(n, k)
        x = lu.solve_matrix(rhs)
        res = mm @ x - rhs
        print(n, norm, k, "nan", np.isnan(x).sum(), "resid", np.abs(res).max(), "piv_id", np.array_equal(piv, np.arange(n)))
a = W.randn_matrix(96, 40) / np.sqrt(96) - 2.0 * np.eye(96)
a *= 1.5 / W.one_norm(a)
v = W.randn(41, 96 * 4).reshape(96, 4)
for nsub in (1, 2, 16):
    got = api.action(a, v, "R8", substeps=nsub)
    ref = O.action(a, v, O.OMethod.from_method(M.catalog("R8"), 1), nsub)
    print("action", nsub, np.abs(got - ref).max(), np.isnan(got).sum(), np.abs(ref).max())
