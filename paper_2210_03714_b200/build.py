"""In-tree build of the native libraries (no JIT cache: the .so files travel with the repo).

* ``_lib/libpfb200.so``  -- the CUDA engine behind include/pf_b200.h (nvcc, sm_100a only)
* ``_lib/libparfrac_host.so`` -- the C++ host layer (namespace parfrac, the reference's API)
* ``_lib/libparfrac_gen.so``  -- host-only input generators and binary128 error oracles (no CUDA:
  the CPU reference arm loads it without touching the engine)

``python -m paper_2210_03714_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
CPP = PKG / "cpp"
LIB = PKG / "_lib"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
              "--expt-relaxed-constexpr", "-I" + str(INCLUDE), "-I" + str(CSRC)]
# the exact method layer (Rational, moment solve, theta) runs on the GMP runtime, as the reference's
# does; the image has libgmp.so.10 but no development symlink, so link it by soname
GMP_LINK = "-l:libgmp.so.10"
CXX_FLAGS = ["-O3", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-I" + str(INCLUDE), "-I" + str(CPP / "include")]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA engine cannot be built")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: %s\n%s" % (" ".join(cmd), r.stdout))
    return r.stdout


def build_engine(verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libpfb200.so"
    sources = sorted(CSRC.glob("*.cu"))
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [INCLUDE / "pf_b200.h"]
    objdir = LIB / "obj"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        if _stale(obj, [src] + headers):
            log = _run([nvcc, *ARCH, *NVCC_FLAGS, "-Xptxas", "-v", "-c", str(src), "-o", str(obj)])
            (objdir / (src.stem + ".ptxas.txt")).write_text(log)
            if verbose:
                print(log)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources))
    if _stale(out, objs):
        _run([nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(out), *map(str, objs), "-cudart", "static"])
    return out


def build_host(verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libparfrac_host.so"
    srcs = sorted((CPP / "src").glob("*.cpp")) if (CPP / "src").exists() else []
    srcs = [p for p in srcs if p.name not in GEN_SOURCES or p.name == "generators.cpp"]
    if not srcs:
        return out
    hdrs = list((CPP / "include").rglob("*.hpp")) + list((CPP / "src").glob("*.h*")) + \
        list((CPP / "src").glob("*.inc")) + [INCLUDE / "pf_b200.h"]
    if _stale(out, srcs + hdrs + [LIB / "libpfb200.so"]):
        cxx = shutil.which("g++") or "g++"
        _run([cxx, *CXX_FLAGS, "-shared", "-o", str(out), *map(str, srcs), "-L" + str(LIB), "-lpfb200",
              "-Wl,-rpath,$ORIGIN", GMP_LINK, "-lpthread"])
    return out


GEN_SOURCES = ("generators.cpp", "hp_oracle.cpp")


def build_gen(verbose: bool = False) -> Path:
    """Seeded generators + binary128 oracles, host only (not linked to the CUDA engine)."""
    LIB.mkdir(exist_ok=True)
    out = LIB / "libparfrac_gen.so"
    srcs = [CPP / "src" / f for f in GEN_SOURCES]
    hdrs = list((CPP / "include").rglob("*.hpp"))
    if _stale(out, srcs + hdrs):
        cxx = shutil.which("g++") or "g++"
        _run([cxx, *CXX_FLAGS, "-shared", "-o", str(out), *map(str, srcs), "-lpthread"])
    return out


def build_cpp_tests(verbose: bool = False) -> Path:
    """The C++ parity test binary over the host layer (tests/cpp/test_parfrac.cpp)."""
    src = ROOT / "tests" / "cpp" / "test_parfrac.cpp"
    out = LIB / "test_parfrac"
    if not src.exists():
        return out
    deps = [src, LIB / "libparfrac_host.so"] + list((CPP / "include").rglob("*.hpp"))
    if _stale(out, deps):
        cxx = shutil.which("g++") or "g++"
        _run([cxx, *CXX_FLAGS, "-o", str(out), str(src), "-L" + str(LIB), "-lparfrac_host", "-lpfb200",
              "-Wl,-rpath,$ORIGIN", GMP_LINK, "-lpthread"])
    return out


def build_oracle() -> Path:
    """The CPU checker (test infrastructure; never loaded by the product path)."""
    _run(["make", "-s", "-j8", "-C", str(ROOT / "oracle")])
    return ROOT / "oracle" / "libpforacle.so"


def build_all(verbose: bool = False):
    eng = build_engine(verbose)
    build_gen(verbose)
    host = build_host(verbose)
    tst = build_cpp_tests(verbose)
    orc = build_oracle()
    return eng, host, tst, orc


if __name__ == "__main__":
    for p in build_all(verbose="-v" in sys.argv):
        print(p)
