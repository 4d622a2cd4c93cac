"""GPU: the C++ drop-in (include/moesim_b200.hpp) driven by a host program that
replays the reference's own test assertions (tests/cpp/compat_main.cpp, built
by paper_2205_10034_b200/csrc/Makefile next to libmoe_b200.so)."""
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

EXE = os.path.join(os.path.dirname(__file__), "..", "paper_2205_10034_b200", "build",
                   "compat_main")


def test_cpp_drop_in_cases():
    assert os.path.exists(EXE), "build it: make -C paper_2205_10034_b200/csrc"
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "FAIL" not in r.stdout
