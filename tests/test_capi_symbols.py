"""The C-ABI library loads without a GPU and exports exactly what include/vgicp.h declares."""

import re
import subprocess

import pytest

from paper_2202_00242_b200 import _lib

HEADER = _lib.LIB_PATH.parents[2] / "include" / "vgicp.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(vg_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert "vg_batch_linearize" in names and "vg_map_build" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vg_\w+)", out))
    assert set(declared()) <= exported


def test_binding_covers_header():
    assert set(declared()) == set(_lib.EXPORTED_SYMBOLS)


def test_abi_version_and_error_string():
    lib = _lib.load_library()
    assert lib.vg_abi_version() == 1
    assert isinstance(lib.vg_last_error(), bytes)


def test_no_gpu_fails_loudly():
    """Without a device the product path raises instead of falling back to the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(_lib.VgicpUnavailable):
        _lib.Context(0)


def test_sm100a_cubin_present():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_null_handles_return_status_codes():
    """The C-ABI validates its arguments before touching a device: null handles and bad
    modes come back as VG_ERR_INVALID with a message, never as a crash (no GPU needed)."""
    import ctypes

    lib = _lib.load_library()
    VG_ERR_INVALID = 1
    null = ctypes.c_void_p(0)
    dptr = ctypes.POINTER(ctypes.c_double)()
    assert lib.vg_batch_linearize(null, dptr, 0, dptr) == VG_ERR_INVALID
    assert b"null" in lib.vg_last_error().lower() or lib.vg_last_error()
    assert lib.vg_batch_linearize_poses(null, dptr, 1, 0, dptr) == VG_ERR_INVALID
    assert lib.vg_batch_assemble_setup(null, 4, None, None) == VG_ERR_INVALID
    assert lib.vg_batch_info(null, None, None, None) == VG_ERR_INVALID
    assert lib.vg_map_info(null, None, None, None) == VG_ERR_INVALID
    out = ctypes.c_void_p()
    assert lib.vg_cloud_create(null, dptr, dptr, 3, ctypes.byref(out)) == VG_ERR_INVALID
    assert lib.vg_batch_destroy(null) == 0 and lib.vg_map_destroy(null) == 0
