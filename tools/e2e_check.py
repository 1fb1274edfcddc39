"""HostPipeline: correctness (equals the device-resident call bit for bit), a chunk / stream sweep of
the submit loop the bench times, and the raw PCIe ceiling (pinned H2D and D2H of the same bytes,
alone and concurrently on two streams)."""
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


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dA = torch.empty(hA.shape, dtype=torch.float64, device="cuda")
gb = hA.numel() * 8 / 1e9
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2d = timed(lambda: dA.copy_(hA, non_blocking=True))
d2h = timed(lambda: hO.copy_(dA, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        dA.copy_(hA, non_blocking=True)
    with torch.cuda.stream(s2):
        hO.copy_(dA, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


duplex = timed(both)
print("PCIe: H2D %.2f ms (%.1f GB/s), D2H %.2f ms (%.1f GB/s), both at once %.2f ms" % (
    h2d, gb / h2d * 1e3, d2h, gb / d2h * 1e3, duplex))
kernel = timed(lambda: api.expm(dA, "R4", out=dA.new_empty(dA.shape)))
print("device-resident expm %.2f ms" % kernel)
for chunk, ns in ((256, 4), (128, 4), (128, 8), (512, 3), (64, 8)):
    pipe = api.HostPipeline(128, 4096, chunk=chunk, streams=ns)

    def loop():
        for _ in range(4):
            pipe.submit(hA, hO, "R4")
        pipe.finish()
    ms = timed(loop, 2) / 4
    print("chunk", chunk, "streams", ns, "ms/batch %.2f" % ms, "evals/s %.0f" % (4096 / ms * 1e3))
