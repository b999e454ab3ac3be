"""The C-ABI library builds for sm_100a, loads, and exports every symbol of include/uhmv.h."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT, ensure_built


def header_symbols():
    text = open(os.path.join(ROOT, "include", "uhmv.h")).read()
    return sorted(set(re.findall(r"\b(uhmv_[a-z_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for s in ("uhmv_plan_create", "uhmv_execute", "uhmv_matvec_host", "uhmv_plan_destroy", "uhmv_last_error"):
        assert s in syms


def test_library_exports_all_header_symbols():
    L = ensure_built()
    for s in header_symbols():
        assert hasattr(L, s), s
    from paper_2405_15573_b200 import _lib

    assert L.uhmv_abi_version() == _lib.ABI_VERSION == 13
    assert L.uhmv_last_error() == b""


def test_library_is_sm100a():
    from paper_2405_15573_b200 import _lib

    ensure_built()
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        import pytest

        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_plan_create_rejects_bad_descriptor():
    from paper_2405_15573_b200 import _lib

    L = ensure_built()
    d = _lib.UhmvDesc()
    d.abi_version = 99
    h = ctypes.c_void_p()
    rc = L.uhmv_plan_create(ctypes.byref(d), ctypes.byref(h))
    assert rc == -1 and b"ABI" in L.uhmv_last_error()
    assert L.uhmv_plan_create(None, ctypes.byref(h)) == -1
    assert L.uhmv_execute(None, None, None, 0, 0, None) == -1
    assert L.uhmv_plan_destroy(None) == 0


def test_execute_peer_rejects_bad_arguments():
    from paper_2405_15573_b200 import _lib

    L = ensure_built()
    ranks = (_lib.UhmvPeerRank * 2)()
    plans = (ctypes.c_void_p * 1)(None)
    ws = (ctypes.c_void_p * 1)(None)
    assert L.uhmv_execute_peer(None, 1, 0, 2, ranks, None, ws, 0, 1, None) == -1
    assert L.uhmv_execute_peer(plans, 1, 0, 9, ranks, ctypes.c_void_p(16), ws, 0, 1, None) == -1
    assert b"rank range" in L.uhmv_last_error()
    assert L.uhmv_execute_peer(plans, 1, 0, 2, ranks, ctypes.c_void_p(16), ws, 0, 0, None) == -1
    assert b"epoch" in L.uhmv_last_error()


def test_diagnostic_and_io_entries_reject_null_plan():
    L = ensure_built()
    assert L.uhmv_plan_set_io(None, None, None, None) == -1
    assert b"null plan" in L.uhmv_last_error()
    assert L.uhmv_plan_set_trace(None, None) == -1
    assert L.uhmv_plan_set_profile(None, None) == -1
    assert L.uhmv_peer_set_diag(None, 28) == 0  # process-wide diagnostics switch, always accepted
    assert L.uhmv_plan_set_host_path(None, 0, 1) == -1
    assert L.uhmv_plan_last_host_path(None, 0) == -1
    assert L.uhmv_host_pinned(None) == 0  # no CUDA context needed for a null pointer
