"""The C ABI from plain C (tools/mmtest.c: the paper's test program, with
cudaMalloc'd buffers and libmm_b200.so only -- no Python on the call path): it runs, prints a row
per method with the printed-band deviation at n = 200, and the ABI's error paths answer from C."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_mmtest_c_client():
    from paper_1106_1347_b200 import build

    exe = build.build_tools()
    r = subprocess.run([exe, "-O", "200", "-R", "3"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = {}
    for line in r.stdout.splitlines():
        parts = [p.strip() for p in line.strip().strip("|").split("|")]
        if len(parts) == 3 and parts[2] and parts[0] not in ("method",):
            rows[parts[0]] = float(parts[2])
    for name in ("NaivStandard", "StrassenNaiv", "StrassenWinograd", "WinogradOriginal", "WinogradScaled"):
        assert name in rows, r.stdout
        assert 0.0 <= rows[name] < 1.875e-10, (name, rows[name])  # the n = 200 printed bands
    assert "C overlaps A or B" in r.stdout
    # the host-buffer entry point (mm_methods_host) from C: Kahan's product is the device call's
    assert "NaivKahan product bitwise the device call's: yes" in r.stdout, r.stdout
