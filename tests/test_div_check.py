"""The EIM solver's fast quotient (csrc/eim.cu div_rn_pre: RN(1/b), then two FMA remainder
corrections) equals the IEEE division on random and adversarial operand pairs whose exponents
stay in [-500, 500) -- the range the kernel takes that path in (scripts/div_check.c, host C)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_fast_quotient_is_the_ieee_quotient(tmp_path):
    exe = tmp_path / "div_check"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), os.path.join(ROOT, "scripts", "div_check.c"), "-lm"],
                   check=True)
    out = subprocess.run([str(exe), "30000000"], check=True, capture_output=True, text=True).stdout
    assert out.strip().endswith("mismatches=0"), out
