"""The C-ABI library loads on a CPU-only host and exports every entry point that
include/photon.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "photon.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(photon_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(F):
    from paper_2411_02908_b200 import _capi

    lib = _capi.lib()
    names = declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding declares exactly the header's surface
    assert sorted(_capi.EXPORTED) == names
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (photon_[a-z0-9_]+)", out))
    assert set(names) <= exported


def test_abi_version_and_status_names(F):
    from paper_2411_02908_b200 import _capi

    lib = _capi.lib()
    assert lib.photon_abi_version() == 2
    for code, name in ((0, b"OK"), (1, b"ConfigError"), (8, b"DivergenceError"),
                       (11, b"RoundFailureError")):
        assert lib.photon_status_name(code) == name


def test_no_cpu_fallback_symbols(F):
    """The product library never links or embeds the oracle."""
    from paper_2411_02908_b200 import _capi

    out = subprocess.run(["nm", "-D", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out and "ref_" not in out
    deps = subprocess.run(["ldd", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "liboracle" not in deps and "libfedsim_ref" not in deps


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2411_02908_b200 import _capi

    monkeypatch.setattr(_capi, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_capi, "_lib", None)
    try:
        _capi.lib()
        raise AssertionError("expected ImportError")
    except ImportError as e:
        assert "no CPU fallback" in str(e)
