"""The C++ host layer's generated catalog table equals a fresh exact derivation (CPU)."""
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_catalog_table_is_current():
    import importlib.util

    spec = importlib.util.spec_from_file_location("gen_tables", ROOT / "tools" / "gen_tables.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.OUT.read_text() == mod.render()


def test_cpp_binary_and_host_library_built():
    lib = ROOT / "paper_2210_03714_b200" / "_lib"
    assert (lib / "libparfrac_host.so").exists()
    assert (lib / "test_parfrac").exists()
