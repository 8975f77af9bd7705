"""The reference's seqpar unit tests restated in C++ against include/spl_seqpar.hpp (the
drop-in facade with the reference signatures), run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_reference_suite():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = os.path.join(ROOT, "build", "test_facade")
    if not os.path.exists(exe):
        subprocess.run(["make", "build/test_facade"], cwd=ROOT, check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
