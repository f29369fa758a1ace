"""Markstein division (a shared correctly rounded reciprocal plus one FMA
correction) against IEEE '/': the identity behind the EXACT K1's LDLT column
divisions (dbag_exact.cu ldlt_col). This fuzz checks bit-identity
with '/' on random (the whole guarded exponent band and beyond), adversarial
and LDLT-like operands, compiled with hardware FMA; operands outside the band
take '/' as on the device."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_markstein_division_is_ieee_division(tmp_path):
    exe = str(tmp_path / "mfuzz")
    r = subprocess.run(["g++", "-O2", "-mfma", "-ffp-contract=off", "-std=c++17",
                        os.path.join(HERE, "native", "markstein_fuzz.cpp"), "-o", exe],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("no FMA-capable g++: " + r.stderr[-200:])
    out = subprocess.run([exe, "5000000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout
