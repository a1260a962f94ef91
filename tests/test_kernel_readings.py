"""CPU pins for arithmetic readings the CUDA kernels rely on,
independent of both the oracle and the CUDA path."""
import os

import pytest


def test_markstein_division_reading(tmp_path):
    """DESIGN.md 6.1 reading: the sweep kernel divides by the degree d as
    fma(e, r, q) with r = RN(1/d), q = RN(x r), e = fma(-q, d, x) -- equal to
    the correctly rounded x / d (Markstein) in the kernel's operand window.
    Brute force with midpoint-adjacent operands, in C (IEEE double, no
    contraction)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    src = os.path.join(os.path.dirname(__file__), "c", "markstein_check.c")
    exe = str(tmp_path / "markstein_check")
    subprocess.run([cc, "-O2", "-ffp-contract=off", "-o", exe, src, "-lm"], check=True)
    out = subprocess.run([exe, "200000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "mismatches 0" in out.stdout
