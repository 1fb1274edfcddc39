"""The host-buffer pipeline (api.HostPipeline, the bench's e2e path): chunks over several streams,
H2D / evaluation / D2H overlapped, successive submissions overlapped; results equal the
device-resident evaluation bit for bit, errors surface at finish()."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(pf):
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need CUDA")
    from paper_2210_03714_b200 import api

    return api


def test_pipeline_matches_device_call(dev):
    from paper_2210_03714_b200 import workloads as W

    a = torch.from_numpy(W.cfg2(batch=300)).pin_memory()
    ref = dev.expm(a.cuda(), "R4").cpu()
    pipe = dev.HostPipeline(128, 300, chunk=64, streams=3)
    out = torch.empty_like(a).pin_memory()
    pipe.expm(a, out, "R4")
    assert torch.equal(out, ref)
    # several submissions before one finish (the e2e bench loop)
    outs = [torch.empty_like(a).pin_memory() for _ in range(3)]
    for o in outs:
        pipe.submit(a, o, "R4")
    pipe.finish()
    for o in outs:
        assert torch.equal(o, ref)


def test_pipeline_error_surfaces_at_finish(dev):
    from paper_2210_03714_b200.errors import Errc, PfError

    n = 128
    a = np.zeros((4, n, n))
    for b in range(4):
        a[b] = np.eye(n) * 0.1
    # matrix 2: I - cB singular for the first shift of R4 (c b = 1 on a diagonal entry)
    from paper_2210_03714_b200 import methods as M

    c = M.catalog("R4").shift_doubles()[1]
    a[2, 5, 5] = 1.0 / c
    ta = torch.from_numpy(a).pin_memory()
    pipe = dev.HostPipeline(n, 4, chunk=2, streams=2)
    out = torch.empty_like(ta).pin_memory()
    pipe.submit(ta, out, "R4", theta=1e9)  # no scaling: the singular system is evaluated as given
    with pytest.raises(PfError) as e:
        pipe.finish()
    assert e.value.code == Errc.SingularShift
