"""HostPipeline correctness (equals the device-resident call bit for bit) and timing."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_03714_b200 import api, workloads as W  # noqa: E402

a = W.cfg2()
hA = torch.from_numpy(a).pin_memory()
hO = torch.empty_like(hA).pin_memory()
pipe = api.HostPipeline(128, 4096, chunk=512, streams=3)
pipe.expm(hA, hO, "R4")
torch.cuda.synchronize()
ref = api.expm(torch.from_numpy(a).cuda(), "R4").cpu()
print("bit-identical:", torch.equal(ref, hO))
for chunk, ns in ((512, 3), (256, 4), (1024, 2)):
    pipe = api.HostPipeline(128, 4096, chunk=chunk, streams=ns)
    pipe.expm(hA, hO, "R4")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pipe.expm(hA, hO, "R4")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print("chunk", chunk, "streams", ns, "ms", ms, "evals/s", 4096 / ms * 1e3)
