"""Large-engine phase timing: cfg4 operator build (8 LUs of 16384^2) vs one substep, cfg3 eval vs
doubling, and the DMMA GEMM at the shapes the recursion uses."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, methods as M, workloads as W  # noqa: E402


def tm(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


which = sys.argv[1] if len(sys.argv) > 1 else "all"
eng = api.engine()
if which in ("all", "gemm"):
    for (m, n, k) in [(4096, 4096, 4096), (8192, 8192, 8192), (16384, 64, 16384), (2048, 2048, 2048), (512, 512, 512)]:
        a = torch.randn(m, k, dtype=torch.float64, device="cuda")
        b = torch.randn(k, n, dtype=torch.float64, device="cuda")
        c = torch.empty(m, n, dtype=torch.float64, device="cuda")
        ms, _ = tm(lambda: api.gemm(a, b, Cm=c), 3)
        print("gemm %dx%dx%d: %.3f ms %.1f TF/s" % (m, n, k, ms, 2 * m * n * k / ms / 1e9))
        del a, b, c
if which in ("all", "cfg4"):
    a_np, v_np = W.cfg4()
    A = torch.from_numpy(a_np).cuda()
    V = torch.from_numpy(v_np).cuda()
    del a_np
    n = A.shape[0]
    l0 = eng.launch_count()
    ms_build, op = tm(lambda: api.ActionOperator(A, "R8", 42, M.RESIDUAL))
    print("cfg4 operator build (8 LU of 16384^2): %.1f ms, %.1f TF/s, launches %d" % (
        ms_build, 8 * (2 / 3) * n ** 3 / ms_build / 1e9, eng.launch_count() - l0))
    l0 = eng.launch_count()
    ms_step, _ = tm(lambda: op.apply(V), 3)
    print("cfg4 one substep: %.2f ms, %.1f TF/s, launches/step %d" % (
        ms_step, (8 * 2 * n * n * 64 + 2 * n * n * 64) / ms_step / 1e9, (eng.launch_count() - l0) // 4))
if which in ("all", "cfg3"):
    A = torch.from_numpy(W.cfg3()).cuda()
    n = A.shape[0]
    m = M.catalog("R8")
    rm = M.to_residual_form(m) if hasattr(M, "to_residual_form") else None
    j = api.squarings(A, api._theta_for(api._resolve_method("R8"), None))
    jj = int(j.max())
    B = A * (2.0 ** -jj)
    ms_lu, _ = tm(lambda: api.DenseLu(torch.eye(n, dtype=torch.float64, device="cuda") - 0.5 * B))
    lu = api.DenseLu(torch.eye(n, dtype=torch.float64, device="cuda") - 0.5 * B)
    R = B.clone()
    ms_solve, _ = tm(lambda: lu.solve_matrix(R))
    print("cfg3 j=%d; one shifted LU 4096^2: %.2f ms (%.1f TF/s); solve with 4096 RHS: %.2f ms (%.1f TF/s)" % (
        jj, ms_lu, (2 / 3) * n ** 3 / ms_lu / 1e9, ms_solve, 2 * n ** 3 / ms_solve / 1e9))
    ms_all, (E, P) = tm(lambda: api.expm_phi1(A, "R8"))
    ms_dbl, _ = tm(lambda: api.phi1_doubling(E.clone(), P.clone(), j))
    print("cfg3 total %.1f ms; phi1 doubling (%d steps, 2 GEMMs each) %.1f ms (%.1f TF/s)" % (
        ms_all, jj, ms_dbl, jj * 2 * 2 * n ** 3 / ms_dbl / 1e9))
if which in ("all", "lu8"):
    # the cfg3 eval shape: 8 shifted 4096^2 systems per launch, factor then solve with 4096 RHS
    A = torch.from_numpy(W.cfg3()).cuda()
    n = A.shape[0]
    B = A * (2.0 ** -8)
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    Ms = torch.stack([I - c * B for c in (0.1, -0.1, 0.2, -0.2, 0.3, -0.3, 0.4, -0.4)])
    del A
    lus = [None]

    def fac():
        lus[0] = api.DenseLu(Ms)
    ms_f, _ = tm(fac)
    R = torch.stack([B] * 8)
    ms_s, _ = tm(lambda: lus[0].solve_matrix(R))
    print("batched 8 x LU 4096^2: %.1f ms (%.1f TF/s); 8 x solve with 4096 RHS: %.1f ms (%.1f TF/s)" % (
        ms_f, 8 * (2 / 3) * n ** 3 / ms_f / 1e9, ms_s, 8 * 2 * n ** 3 / ms_s / 1e9))
    for nn in (1024, 2048):
        Ms2 = Ms[:, :nn, :nn].contiguous()
        R2 = R[:, :nn, :nn].contiguous()
        ms_f, _ = tm(lambda: lus.__setitem__(0, api.DenseLu(Ms2)))
        ms_s, _ = tm(lambda: lus[0].solve_matrix(R2))
        print("batched 8 x LU %d^2: %.2f ms (%.1f TF/s); solve %d RHS: %.2f ms (%.1f TF/s)" % (
            nn, ms_f, 8 * (2 / 3) * nn ** 3 / ms_f / 1e9, nn, ms_s, 8 * 2 * nn ** 3 / ms_s / 1e9))
