"""The C++ drop-in API (include/spct/*.hpp) compiled and run like a reference test binary.

build/dropin_test is built by `make dropin` (part of __graft_entry__.build()): it
includes the reference include paths spct/{imagecore,integral,likelihood}.hpp, calls the
unchanged spct:: signatures and links libspct_b200.so.  Compiling it is a CPU check;
running it needs the GPU.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin_test")


def test_dropin_compiles():
    r = subprocess.run(["make", "-C", ROOT, "dropin"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "dropin"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "checks passed" in r.stdout


ACC = os.path.join(ROOT, "build", "acceptance_test")


@pytest.mark.gpu
def test_acceptance_criteria_on_gpu():
    """proj/tests/acceptance.cpp:64-137 at the stated counts: 50 images x every schedule x
    threads {1,2,4,8}; 1000 exhaustive 6x6 images + 200 rects at 256x256/32."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(ACC):
        subprocess.run(["make", "-C", ROOT, "acceptance"], check=True)
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "criterion 1: PASS" in r.stdout and "criterion 2: PASS" in r.stdout
