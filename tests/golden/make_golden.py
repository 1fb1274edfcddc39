"""Generates the golden fixtures of tests/golden/ from THE REFERENCE ITSELF (oracle/_ref, i.e.
/root/reference/proj/core/src compiled unmodified; see oracle/Makefile).

    python tests/golden/make_golden.py

Each fixture is a small .npy array plus its sha256 in golden.json. The inputs come from the
reference's generators (SplitMix64 / NormalSampler). ``compute("ref")`` is the generator (needs
oracle/_ref); ``compute("oracle")`` recomputes the same cases with the fast restatement
(oracle/pf_oracle.c), which tests/test_oracle.py requires to reproduce every fixture bit for bit.
The GPU parity tests compare the device path against these frozen reference outputs.
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

    t = W.trid121_dense(200) * 0.5
    return {
        "cfg1_A": W.cfg1(),
        "eval24_B": W.scaled_to_one_norm(W.randn_matrix(24, 5), 0.7),
        "pivot24_B": W.scaled_to_one_norm(W.randn_matrix(24, 900), 60.0),
        "cfg2_first4_A": W.cfg2(batch=4),
        "phi48_A": W.scaled_to_one_norm(W.randn_matrix(48, 31), 3.0),
        "action40_A": W.scaled_to_one_norm(W.randn_matrix(40, 41), 2.0),
        "action40_V": W.randn(42, 40 * 5).reshape(40, 5),
        "trid200": (-np.diag(t, -1).copy(), -np.diag(t).copy(), -np.diag(t, 1).copy()),
        "trid200_v": W.randn(17, 200),
    }


def compute(backend: str = "ref"):
    from paper_2210_03714_b200 import methods as M

    x = inputs()
    out = {}
    r8 = M.catalog("R8")
    th_phi = M.THETA_U53["R8_phi1set"]
    if backend == "ref":
        from oracle import ref as R

        for name in ("R4", "R8"):
            rm = R.RefMethod.catalog(name)
            out["cfg1_expm_%s" % name] = R.expm(rm, x["cfg1_A"], M.THETA_U53[name], M.RESIDUAL)[0]
            out["cfg2_first4_expm_%s" % name] = R.expm_batched(rm, x["cfg2_first4_A"], M.THETA_U53[name], M.RESIDUAL,
                                                              threads=4)[0]
        rm8 = R.RefMethod.catalog("R8")
        out["eval24_R8_plain"] = R.eval_dense(rm8, x["eval24_B"], M.PLAIN)
        out["eval24_R8_residual"] = R.eval_dense(rm8, x["eval24_B"], M.RESIDUAL)
        out["pivot24_solve_shifted_0.2"] = R.solve_shifted(x["pivot24_B"], 0.2)
        out["pivot24_lu_piv"] = R.lu(np.eye(24) - 0.2 * x["pivot24_B"])[1].astype(np.int32)
        e, p, _ = R.expm_phi1(rm8, R.RefMethod.build_plain(8, "5", "phi1", 8), x["phi48_A"], th_phi, M.RESIDUAL)
        out["phi48_R8_exp"], out["phi48_R8_phi1"] = e, p
        out["action40_R8_residual_N3"] = R.dense_action(rm8, x["action40_A"], x["action40_V"], 3, M.RESIDUAL)
        out["trid200_R8_residual_N4"] = R.tridiag_action(rm8, *x["trid200"], x["trid200_v"], "substep", 4,
                                                         M.RESIDUAL)
        return out
    from oracle import oracle as O

    for name in ("R4", "R8"):
        om = O.OMethod.from_method(M.catalog(name), M.RESIDUAL)
        out["cfg1_expm_%s" % name] = O.expm(x["cfg1_A"], om, M.THETA_U53[name])[0]
        out["cfg2_first4_expm_%s" % name] = O.expm_batched(x["cfg2_first4_A"], om, M.THETA_U53[name], 1)[0]
    om8 = O.OMethod.from_method(r8, M.RESIDUAL)
    out["eval24_R8_plain"] = O.eval_dense(O.OMethod.from_method(r8, M.PLAIN), x["eval24_B"])
    out["eval24_R8_residual"] = O.eval_dense(om8, x["eval24_B"])
    out["pivot24_solve_shifted_0.2"] = O.solve_shifted(x["pivot24_B"], 0.2)
    out["pivot24_lu_piv"] = O.lu(np.eye(24) - 0.2 * x["pivot24_B"])[1].astype(np.int32)
    phi = M.same_shift_method(r8, M.FunctionId.phi(1))
    e, p, _ = O.expm_phi1(x["phi48_A"], O.OMethod.from_method(r8, M.RESIDUAL, extra=(phi,)), th_phi)
    out["phi48_R8_exp"], out["phi48_R8_phi1"] = e, p
    out["action40_R8_residual_N3"] = O.action(x["action40_A"], x["action40_V"], om8, 3)
    out["trid200_R8_residual_N4"] = O.tridiag_action(*x["trid200"], x["trid200_v"], om8, 4)
    return out


def main():
    cases = {}
    for key, arr in compute("ref").items():
        fn = key.replace(".", "_") + ".npy"
        np.save(HERE / fn, arr)
        cases[key] = {"file": fn, "sha256": hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest(),
                      "shape": list(arr.shape)}
    (HERE / "golden.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py", "cases": cases},
                                                 indent=1))
    print("wrote", len(cases), "fixtures")


if __name__ == "__main__":
    main()
