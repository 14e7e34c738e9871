"""Static checks of the built sm_100a code (no GPU needed): cuobjdump of libbmc.so.

* no predicated FP64 MMA: mma.sync.aligned must be executed by every lane of the warp;
  a lane-dependent select feeding an MMA operand can make the compiler split one MMA
  into predicated copies, and the warp then deadlocks (seen once);
* the hot kernel uses the FP64 tensor-core MMA and the fast MUFU paths it is built around.
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2109_13030_b200", "libbmc.so")


@pytest.fixture(scope="module")
def sass():
    if not os.path.exists(LIB):
        pytest.skip("libbmc.so not built")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    return subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, check=True).stdout


def test_no_predicated_mma(sass):
    bad = re.findall(r"@!?U?P\w+\s+(?:DMMA|HMMA|IMMA)\S*", sass)
    assert not bad, bad[:5]


def test_hot_kernel_uses_fp64_mma_and_mufu(sass):
    assert "DMMA.8x8x4" in sass
    assert "MUFU.RSQ" in sass
    assert "REDUX" in sass or "CREDUX" in sass
