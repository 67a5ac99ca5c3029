"""The reference's acceptance criteria c3 and c4 (acceptance_main.cpp:237-337)
with the photon drop-in substituted, as a C++ program linked against the
reference's own objects and libphoton.so (tests/cpp/acceptance_photon.cpp,
built by oracle/Makefile into oracle/_ref/acceptance_photon).  Stated bounds:
c3 <= 1e-9 through the f64 entry points (as the reference), <= 2e-6 through the
fp32 device round; c4 bitwise through the f64 entry points and device runner vs
device centralized, <= 5e-3 device runner (fp32 AdamW, 200 steps) vs the f64
reference."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_photon")


@pytest.mark.skipif(not os.path.exists(BIN), reason="built only where /root/reference exists")
def test_reference_acceptance_c3_c4_with_photon_substituted():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("[c")]
    assert {l.split("]")[0][1:] for l in lines} >= {"c3a", "c3b", "c3c", "c4a", "c4b", "c4c", "c4d"}
    assert all(" PASS " in l for l in lines), lines
    assert r.stdout.strip().endswith("ALL PASS")
