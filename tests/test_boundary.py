"""The drop-in boundary: libsem.so loads here (no GPU needed), exports every
symbol include/sem.h declares, the ctypes table matches the header, and the
product package never touches the oracle."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sem.h")
PKG = os.path.join(ROOT, "paper_2005_13425_b200")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sem_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2005_13425_b200.build import build
    build()
    from paper_2005_13425_b200 import _lib
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_ctypes_table_matches_header(lib):
    from paper_2005_13425_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == declared_functions()


def test_abi_metadata(lib):
    assert lib.sem_abi_version() == 1
    assert (lib.sem_min_points(), lib.sem_max_points()) == (2, 16)
    assert lib.sem_reduce_scratch_bytes() > 0
    assert lib.sem_ax_num_variants(10) >= 1 and lib.sem_ax_num_variants(17) == 0


def test_invalid_arguments_rejected_without_gpu(lib):
    # argument validation happens before any CUDA call
    assert lib.sem_ax(None, None, None, None, None, 1, 10, None) == 1001
    assert b"null" in lib.sem_last_error()
    assert lib.sem_dssum_box(None, None, 1, 1, 1, 17, 0, None) == 1001
    assert lib.sem_mask_box(None, None, 0, 1, 1, 4, None) == 1001


def test_state_struct_layout():
    from paper_2005_13425_b200._lib import sem_cg_state
    assert ctypes.sizeof(sem_cg_state) == 7 * 8 + 6 * 4


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), f
                assert "sem_oracle" not in text and "libsem_oracle" not in text, f


def test_so_has_sm100a_code(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(PKG, "libsem.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_alignment_contract_rejected_before_any_launch():
    """Misaligned metric / field pointers are argument errors, reported before
    any CUDA call (so this runs without a GPU) instead of device faults."""
    from paper_2005_13425_b200._lib import load
    lib = load()
    dx = (ctypes.c_double * 100)()
    base = 1 << 20  # never dereferenced: the check precedes every launch
    rc = lib.sem_ax(base, base + 8, dx, dx, base + 4096, 4, 10, None)
    assert rc == 1001 and b"16-byte" in lib.sem_last_error()
    rc = lib.sem_ax(base + 8, base, dx, dx, base + 4096, 4, 10, None)
    assert rc == 1001 and b"field pointers" in lib.sem_last_error()
    rc = lib.sem_dssum_box(base + 8, base + 4096, 2, 2, 2, 4, 1, None)
    assert rc == 1001
