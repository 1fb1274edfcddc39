"""Phase breakdown of the fused small kernel: time with forced squaring counts (j = 0 isolates
the shifted-solve part; j = 10 vs 0 gives the cost per squaring)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, workloads as W  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


B = 4096
a = torch.from_numpy(W.cfg2(batch=B)).cuda()
out = torch.empty_like(a)
res = {}
for m in ("R4", "R8"):
    for j in (0, 1, 10):
        js = torch.full((B,), j, dtype=torch.int32)
        res["%s_j%d" % (m, j)] = t(lambda: api.expm(a, m, squarings=js, out=out))
    res["%s_auto" % m] = t(lambda: api.expm(a, m, out=out))
res["gemm_128_batched_x10"] = t(lambda: [api.gemm(a, a, Cm=out) for _ in range(10)])
print(json.dumps(res, indent=1))

# per-phase SM cycles (sum over CTAs, thread 0 clock64), R4 and R8 automatic j
from paper_2210_03714_b200 import _native as N  # noqa: E402

# per-shift path: load_M, lu (lu.* sub-phases), certificate, solve_acc; pair path: solve_acc holds the
# whole pair work, with pair.* sub-phases in the slots the per-shift path leaves unused
names = ["norm", "load_M", "lu", "certificate", "pair.B2+stats", "solve_acc", "shift_start+E_form", "squaring",
         "output", "pair.cert+M2", "lu.factor|pair.lu", "lu.inverse|pair.solve", "lu.panels|pair.UV",
         "lu.trailing|pair.finish_AV"]
eng = api.engine()
for m in ("R4", "R8"):
    prof = torch.zeros(16, dtype=torch.int64, device="cuda")
    N.lib.pf_context_set_profile(eng.h, prof.data_ptr())
    api.expm(a, m, out=out)
    torch.cuda.synchronize()
    N.lib.pf_context_set_profile(eng.h, None)
    cyc = prof.cpu().numpy().astype(float)[:14] / B
    print(m, "cycles per matrix:", json.dumps({k: round(v) for k, v in zip(names, cyc)}), "total", round(cyc[:10].sum()))
