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


def test_accountant_extras_match_oracle(orc):
    """layer_component_breakdown, percent_of_baseline and total_first_stage_bytes of the product
    library (host code behind the C ABI) equal the oracle restatement and the reference pins."""
    import random
    assert spl.layer_component_breakdown(2, 8, 4, 1) == dict(attention=512, mlp=608, layer_norms=128, total=1248)
    assert spl.percent_of_baseline(128, 20480, 2048, 1, 8, "selective", True) == (17, 84)
    assert spl.percent_of_baseline(128, 20480, 2048, 1, 8, "full", False) == (2, 21)
    assert spl.total_first_stage_bytes(128, 20480, 2048, 1, 8, "selective", True, 105, 35, 3) == 24_777_850_880
    rng = random.Random(7)
    for _ in range(500):
        a = rng.randint(1, 16)
        h = a * rng.randint(1, 32)
        t = rng.choice([1, 2, 4, 8])
        if a % t or h % t:
            continue
        s = t * rng.randint(1, 64)
        b = rng.randint(1, 8)
        act, mask = rng.choice([(2, 1), (4, 1), (2, 2)])
        kind = rng.choice(["none", "selective", "full"])
        sp = rng.random() < 0.5
        L = rng.choice([1, 2, 6, 12])
        p = rng.choice([1, 2, 3])
        m = rng.choice([1, 2])
        assert spl.layer_component_breakdown(a, h, s, b, act, mask) == orc.layer_component_breakdown(a, h, s, b, act, mask)
        assert spl.percent_of_baseline(a, h, s, b, t, kind, sp, act, mask) == \
            orc.percent_of_baseline(a, h, s, b, t, kind, sp, act, mask)
        if L % (p * m):
            with pytest.raises(ValueError):
                spl.total_first_stage_bytes(a, h, s, b, t, kind, sp, L, p, m, act, mask)
        else:
            assert spl.total_first_stage_bytes(a, h, s, b, t, kind, sp, L, p, m, act, mask) == \
                orc.total_first_stage_bytes(a, h, s, b, t, kind, sp, L, p, m, act, mask)


def test_layer_comm_bytes_match_oracle(orc):
    """collectives.cpp:75-87 through the C ABI: SP and TP move the same volume (verify.cpp:285-321)."""
    for (s, b, h) in ((2048, 4, 6144), (2048, 1, 12288), (128, 2, 256), (2048, 1, 25600)):
        for t in (1, 2, 4, 8):
            sp = spl.layer_comm_bytes(s, b, h, t, 2, True)
            tp = spl.layer_comm_bytes(s, b, h, t, 2, False)
            assert sp == orc.layer_comm_bytes_sp(s, b, h, t) and tp == orc.layer_comm_bytes_tp(s, b, h, t)
            assert sp == tp == (0 if t == 1 else 8 * (2 * s * b * h // t) * (t - 1))
