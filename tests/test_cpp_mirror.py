"""The reference-shaped C++ mirror (include/pba_b200.hpp) passes restated reference tests on the GPU."""
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
BIN = REPO / "tests" / "cpp" / "_build" / "test_mirror"


def test_mirror_builds():
    subprocess.run(["make", "-C", str(REPO / "oracle"), "mirror"], check=True, capture_output=True)
    assert BIN.exists()


@pytest.mark.gpu
def test_cpp_mirror_cases():
    if not BIN.exists():
        subprocess.run(["make", "-C", str(REPO / "oracle"), "mirror"], check=True)
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 6 and "FAIL" not in out.stdout, out.stdout
