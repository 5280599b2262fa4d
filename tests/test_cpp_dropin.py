"""The C++ drop-in header (include/lf_gpu.hpp) used like the reference API.

CPU: the programs compile and link against liblfg.so (and, where the
reference exists, against the reference's own headers + oracle/_ref).
GPU: they run and cross-check lf::gpu against the reference CPU functions.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")


def _build():
    from paper_1204_5072_b200 import build

    build.build()
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if os.path.isdir("/root/reference") or not os.path.exists(os.path.join(BUILD, "dropin_standalone")):
        subprocess.run(["bash", os.path.join(ROOT, "tests", "cpp", "build.sh")], check=True)


def test_dropin_programs_build():
    _build()
    assert os.path.exists(os.path.join(BUILD, "dropin_standalone"))
    if os.path.isdir("/root/reference/proj/include"):
        assert os.path.exists(os.path.join(BUILD, "dropin_reference"))


@pytest.mark.gpu
@pytest.mark.parametrize("prog", ["dropin_standalone", "dropin_reference"])
def test_dropin_programs_run(prog):
    exe = os.path.join(BUILD, prog)
    if not os.path.exists(exe):
        if prog == "dropin_reference":
            pytest.skip("reference variant is built where /root/reference exists")
        _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin OK" in r.stdout, r.stdout
