"""The C-ABI library loads without a GPU and exports every entry point the public
header declares (no compute calls are made here)."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2211_00391_b200 import _native

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "obtree_b200.h"


def declared_functions() -> list:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(obt_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib_path = _native.library_path()
    if not lib_path.exists():
        pytest.fail(f"{lib_path} was not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (obt_[a-z0-9_]+)$", out, flags=re.M))
    missing = set(declared_functions()) - exported
    assert not missing, missing


def test_library_loads_and_reports_abi_without_gpu():
    lib = _native.load_library()
    assert lib.obt_abi_version() == 1
    assert isinstance(lib.obt_last_error(), bytes)
    # argument errors come back as codes + messages, no GPU needed to reject them
    rc = lib.obt_model_create(None, 0, ctypes.byref(ctypes.c_void_p()))
    assert rc == _native.OBT_E_INVALID
    assert b"null" in lib.obt_last_error()


def test_sm100a_code_present():
    """The library carries sm_100a SASS (not only PTX for another target)."""
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.library_path())], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout[:500]


def test_path_options_roundtrip_without_gpu():
    """Every planner choice a test forces is a named path option: automatic (-1) by
    default, settable, restorable; unknown names are refused with the name in the error."""
    for name in _native.PATH_OPTIONS:
        assert _native.get_path_option(name) == -1, name
    with _native.path_options(wide=1, tpw=2):
        assert _native.get_path_option("wide") == 1 and _native.get_path_option("tpw") == 2
    assert _native.get_path_option("wide") == -1 and _native.get_path_option("tpw") == -1
    with pytest.raises(_native.NativeError, match="no_such_path"):
        _native.set_path_option("no_such_path", 1)


def test_no_environment_switches_in_the_library():
    """Kernel selection never reads the environment per call (the path options above are
    the one, explicit way to force a path)."""
    import glob

    for src in glob.glob(str(ROOT / "paper_2211_00391_b200" / "csrc" / "*")):
        assert "getenv(" not in Path(src).read_text(), src


def test_sharded_entry_rejects_bad_arguments_without_gpu():
    """obt_predict_sharded validates its arguments before touching a device."""
    lib = _native.load_library()
    none = (ctypes.c_void_p * 2)(None, None)
    assert lib.obt_predict_sharded(none, 0, 0, None, 0, 0, 1.0, 0.0, None) == _native.OBT_E_INVALID
    assert b"shard count" in lib.obt_last_error()
    assert lib.obt_predict_sharded(none, 2, 7, None, 0, 0, 1.0, 0.0, None) == _native.OBT_E_INVALID
    assert b"shard mode" in lib.obt_last_error()
    assert lib.obt_predict_sharded(none, 2, _native.SHARD_TREES, None, 0, 0, 1.0, 0.0, None) == _native.OBT_E_INVALID
    assert b"null model" in lib.obt_last_error()
