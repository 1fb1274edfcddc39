"""The C-ABI library loads and exports every symbol include/pf_b200.h declares (no GPU needed,
no compute calls); the host library exports its generators."""
import ctypes as C
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", text)))


def test_engine_exports_every_declared_symbol():
    from paper_2210_03714_b200 import _native as N

    names = declared("pf_b200.h")
    assert len(names) >= 15
    for name in names:
        assert hasattr(N.lib, name), name
    bound = {n for n, _, _ in N.SIGNATURES}
    assert set(names) <= bound, set(names) - bound
    assert N.lib.pf_version() >= 1
    assert N.lib.pf_error_string(7) == b"SingularShift"


def test_error_ordinals_match_reference_errc():
    """pf_err = parfrac::Errc ordinal + 1 (error.hpp:8-19)."""
    from paper_2210_03714_b200.errors import Errc

    text = (ROOT / "include" / "pf_b200.h").read_text()
    for e in Errc:
        if e == Errc.CudaError:
            continue
        snake = re.sub(r"(?<!^)(?=[A-Z])", "_", e.name).upper()
        m = re.search(r"PF_ERR_%s\s*=\s*(\d+)" % snake, text)
        assert m and int(m.group(1)) == int(e) + 1, e


def test_context_create_fails_cleanly_without_gpu():
    import torch

    from paper_2210_03714_b200 import _native as N

    if torch.cuda.is_available():
        return
    h = C.c_void_p()
    rc = N.lib.pf_context_create(0, C.byref(h))
    assert rc == 11 and not h.value  # PF_ERR_CUDA, nothing allocated


def test_generator_library_is_host_only():
    """The input generators (used by the CPU reference arm) live in libparfrac_gen.so, which does not
    link the CUDA engine; libparfrac_host.so (the C++ drop-in layer) exports them too."""
    import subprocess

    lib_dir = ROOT / "paper_2210_03714_b200" / "_lib"
    for so in ("libparfrac_gen.so", "libparfrac_host.so"):
        lib = C.CDLL(str(lib_dir / so))
        for name in ("pf_gen_randn", "pf_gen_uniform", "pf_gen_randn_batch"):
            assert hasattr(lib, name)
    deps = subprocess.run(["ldd", str(lib_dir / "libparfrac_gen.so")], capture_output=True, text=True).stdout
    assert "libpfb200" not in deps and "libcuda" not in deps and "libcudart" not in deps


def test_api_fails_loudly_without_device():
    import pytest
    import torch

    from paper_2210_03714_b200 import api
    from paper_2210_03714_b200.errors import PfError

    if torch.cuda.is_available():
        return
    with pytest.raises(PfError):
        api.Engine(0)
