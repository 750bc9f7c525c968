"""libpslr.so loads and exports every symbol include/pslr.h declares (no device calls)."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pslr.h")
LIB = os.path.join(ROOT, "paper_2002_00917_b200", "lib", "libpslr.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pslr_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for needed in ("pslr_apply", "pslr_solve_B", "pslr_solve_C0", "pslr_apply_Es",
                   "pslr_apply_neumann", "pslr_apply_Err", "pslr_arnoldi", "pslr_gmres",
                   "pslr_spmv", "pslr_ilut_blocks", "pslr_partition_bisect", "pslr_cg",
                   "pslr_cgs_pass", "pslr_comm_init", "pslr_ctx_set_halo", "pslr_ctx_create",
                   "pslr_ctx_set_correction", "pslr_ctx_destroy", "pslr_last_error"):
        assert needed in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_2002_00917_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True)
    if out.returncode != 0:
        import pytest
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_abi_version_and_error_string():
    from paper_2002_00917_b200 import _lib
    assert _lib.fns["pslr_abi_version"]() >= 1
    assert isinstance(_lib.fns["pslr_last_error"](), bytes)
