"""CPU-side checks of the product library: it loads without a GPU, exports every symbol
include/spl.h declares, fails loudly (not silently) when no device exists, and its host-side
accountant equals the oracle on the BASELINE table."""
import subprocess

import pytest

import paper_2205_05198_b200 as spl
from paper_2205_05198_b200 import _lib


def test_library_loads_and_exports_header():
    L = spl.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 31
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(syms) <= exported


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(spl.SplError):
        spl.SeqparLayer(spl.BlockConfig(8, 256, 128, 2), 1, dtype="f32")


@pytest.mark.parametrize("shape,t", [((8, 256, 128, 2), 1), ((64, 6144, 2048, 4), 8), ((96, 12288, 2048, 1), 1),
                                     ((96, 12288, 2048, 1), 2), ((96, 12288, 2048, 1), 4), ((96, 12288, 2048, 1), 8),
                                     ((128, 20480, 2048, 1), 8), ((160, 25600, 2048, 1), 8)])
def test_accountant_matches_oracle(orc, shape, t):
    a, h, s, b = shape
    for kind in ("none", "selective", "full"):
        for sp in (False, True):
            assert spl.per_layer_bytes(a, h, s, b, t, kind, sp) == orc.per_layer_bytes(a, h, s, b, t, kind, sp)
            assert spl.per_layer_bytes_exact(a, h, s, b, t, kind, sp) == orc.per_layer_bytes_exact(a, h, s, b, t, kind, sp)
    assert spl.per_layer_bytes(2, 8, 4, 1, 1, "none", False, act=4) == 66 * 32 + 9 * 32


def test_accountant_pins():
    # test_activation_memory.cpp:42-57, test_cli.cpp:118-125
    assert spl.per_layer_bytes(64, 6144, 2048, 4, 1, "none", False) == 7_079_985_152
    assert spl.per_layer_bytes(64, 6144, 2048, 4, 8, "none", True) == 884_998_144
    assert spl.per_layer_bytes(64, 6144, 2048, 4, 8, "selective", True) == 213_909_504
    assert spl.per_layer_bytes(64, 6144, 2048, 4, 8, "full", True) == 100_663_296
    assert spl.per_layer_bytes(128, 20480, 2048, 1, 8, "selective", True) == 178_257_920
    with pytest.raises(ValueError):
        spl.per_layer_bytes(4, 100, 2048, 1, 8, "none", False)
