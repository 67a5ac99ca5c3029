"""The reference-side adapter (include/photon_fedsim.hpp) compiles against the
reference's own headers (when /root/reference is present)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/core/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_adapter_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "use.cpp"
    src.write_text('#include "photon_fedsim.hpp"\n'
                   "int main() { return photon_abi_version() == PHOTON_ABI_VERSION ? 0 : 1; }\n")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{REF_INC}",
                        f"-I{os.path.join(ROOT, 'include')}", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_c_header_is_plain_c(tmp_path):
    src = tmp_path / "use.c"
    src.write_text('#include "photon.h"\nint main(void) { photon_err e; (void)e; return 0; }\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only",
                        f"-I{os.path.join(ROOT, 'include')}", str(src)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
