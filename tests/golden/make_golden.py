"""Generates the golden fixtures of tests/golden/ from the oracle (oracle/pf_oracle.c).

    python tests/golden/make_golden.py

Each fixture is a small .npy array plus its sha256 in golden.json. The inputs come from the
reference's generators (SplitMix64 / NormalSampler); the GPU parity tests compare the device path
against these frozen outputs at 1e-11, and tests/test_oracle.py checks the oracle still reproduces
them bit for bit.
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))


def inputs():
    from paper_2210_03714_b200 import workloads as W

    return {
        "cfg1_A": W.cfg1(),
        "eval24_B": W.scaled_to_one_norm(W.randn_matrix(24, 5), 0.7),
        "pivot24_B": W.scaled_to_one_norm(W.randn_matrix(24, 900), 60.0),
        "cfg2_first4_A": W.cfg2(batch=4),
    }


def compute():
    from oracle import oracle as O
    from paper_2210_03714_b200 import methods as M

    x = inputs()
    out = {}
    for name in ("R4", "R8"):
        om = O.OMethod.from_method(M.catalog(name), M.RESIDUAL)
        out["cfg1_expm_%s" % name] = O.expm(x["cfg1_A"], om, M.THETA_U53[name])[0]
        out["cfg2_first4_expm_%s" % name] = O.expm_batched(x["cfg2_first4_A"], om, M.THETA_U53[name], 1)[0]
    out["eval24_R8_plain"] = O.eval_dense(O.OMethod.from_method(M.catalog("R8"), M.PLAIN), x["eval24_B"])
    out["eval24_R8_residual"] = O.eval_dense(O.OMethod.from_method(M.catalog("R8"), M.RESIDUAL), x["eval24_B"])
    out["pivot24_solve_shifted_0.2"] = O.solve_shifted(x["pivot24_B"], 0.2)
    out["pivot24_lu_piv"] = O.lu(np.eye(24) - 0.2 * x["pivot24_B"])[1].astype(np.int32)
    return out


def main():
    cases = {}
    for key, arr in compute().items():
        fn = key.replace(".", "_") + ".npy"
        np.save(HERE / fn, arr)
        cases[key] = {"file": fn, "sha256": hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest(),
                      "shape": list(arr.shape)}
    (HERE / "golden.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py", "cases": cases},
                                                 indent=1))
    print("wrote", len(cases), "fixtures")


if __name__ == "__main__":
    main()
