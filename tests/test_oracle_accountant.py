"""Oracle accountant vs the reference tests' known answers
(/root/reference/proj/tests/test_activation_memory.cpp, test_seqpar.cpp:120-137,
test_cli.cpp:118-125) and BASELINE.md §2."""
import random

import pytest

S22 = (64, 6144, 2048)
S175 = (96, 12288, 2048)
S530 = (128, 20480, 2048)
S1T = (160, 25600, 2048)


def test_22b_regimes(orc):  # test_activation_memory.cpp:42-57
    a, h, s = S22
    assert orc.per_layer_bytes(a, h, s, 4, 1, "none", False) == 7_079_985_152
    assert orc.per_layer_bytes(a, h, s, 4, 8, "none", True) == 884_998_144
    assert orc.per_layer_bytes(a, h, s, 4, 8, "selective", True) == 213_909_504
    assert orc.per_layer_bytes(a, h, s, 4, 1, "full", False) == 2 * 2048 * 4 * 6144
    assert orc.per_layer_bytes(a, h, s, 4, 8, "full", True) == 2 * 2048 * 4 * 6144


def test_toy_breakdown(orc):  # test_activation_memory.cpp:59-66
    b = orc.layer_component_breakdown(2, 8, 4, 1)
    assert b == dict(attention=512, mlp=608, layer_norms=128, total=1248)


def test_530b_sel_seq(orc):  # test_cli.cpp:118-125 / BASELINE.md §2
    a, h, s = S530
    assert orc.per_layer_bytes(a, h, s, 1, 8, "selective", True) == 178_257_920


def test_percent_of_baseline_530b(orc):  # test_activation_memory.cpp:198-206
    a, h, s = S530
    assert orc.percent_of_baseline(a, h, s, 1, 8, "selective", True) == (17, 84)
    assert orc.percent_of_baseline(a, h, s, 1, 8, "full", False) == (2, 21)
    assert orc.percent_of_baseline(a, h, s, 1, 8, "none", False) == (1, 1)


def test_selective_kept_fraction(orc):  # test_activation_memory.cpp:208-228
    for shape, saving in ((S175, 0.7018), (S530, 0.6531)):
        a, h, s = shape
        ns, ds = orc.per_layer_bytes_exact(a, h, s, 1, 8, "selective", True)
        nn, dn = orc.per_layer_bytes_exact(a, h, s, 1, 8, "none", True)
        kept = (ns * dn) / (ds * nn)
        assert 1 - kept == pytest.approx(saving, rel=1e-3)
    a, h, s = S175
    ns, ds = orc.per_layer_bytes_exact(a, h, s, 1, 8, "selective", True)
    nn, dn = orc.per_layer_bytes_exact(a, h, s, 1, 8, "none", True)
    from fractions import Fraction
    assert Fraction(ns, ds) / Fraction(nn, dn) == Fraction(34, 114)


def test_sp_divides_by_t(orc):  # test_activation_memory.cpp:230-245
    from fractions import Fraction
    for a in (2, 4, 8):
        for hd in (2, 5):
            for t in (2, 4):
                if a % t:
                    continue
                s = 8 * t
                n1, d1 = orc.per_layer_bytes_exact(a, a * hd, s, 3, t, "none", True)
                n0, d0 = orc.per_layer_bytes_exact(a, a * hd, s, 3, 1, "none", False)
                assert Fraction(n1, d1) == Fraction(n0, d0) / t


def test_breakdown_equals_formula_random(orc):  # test_activation_memory.cpp:247-261
    rng = random.Random(12345)
    for _ in range(1000):
        a = rng.randint(1, 12)
        h = a * rng.randint(1, 16)
        s = rng.randint(1, 64)
        b = rng.randint(1, 8)
        assert orc.layer_component_breakdown(a, h, s, b)["total"] == orc.per_layer_bytes(a, h, s, b, 1, "none", False)


def test_regime_ordering(orc):  # test_activation_memory.cpp:263-288
    from fractions import Fraction as F
    for t in (2, 4, 8, 16):
        for a in (16, 32):
            for hd in (64, 128):
                h, s = a * hd, 16 * t
                v = lambda k, sp, tt=t: F(*orc.per_layer_bytes_exact(a, h, s, 1, tt, k, sp))
                assert v("full", False) <= v("selective", True) <= v("selective", False)
                assert v("selective", True) <= v("none", True) <= v("none", False) <= v("none", False, 1)


def test_monotone_in_t(orc):  # test_activation_memory.cpp:290-304
    for k, sp in (("none", False), ("none", True), ("selective", False), ("selective", True), ("full", False)):
        prev = None
        for t in (1, 2, 4, 8, 16):
            v = orc.per_layer_bytes(16, 1024, 64, 1, t, k, sp)
            assert prev is None or v <= prev
            prev = v


def test_fp32_convention(orc):  # test_activation_memory.cpp:306-314
    assert orc.per_layer_bytes(2, 8, 4, 1, 1, "none", False, act=4, mask=1) == 66 * 32 + 9 * 32
    assert orc.layer_component_breakdown(2, 8, 4, 1, act=4)["total"] == 66 * 32 + 9 * 32


def test_invalid_rejected(orc):  # test_activation_memory.cpp:329-338
    with pytest.raises(ValueError):
        orc.per_layer_bytes(4, 100, 2048, 1, 8, "none", False)
    with pytest.raises(ValueError):
        orc.per_layer_bytes(64, 6144, 2048, 1, 1, "none", False, act=0)


BASELINE_TABLE = {  # BASELINE.md §2 (none TP, none+SP, sel TP, sel+SP, full)
    ("tiny", 1): (3_538_944, 3_538_944, 2_228_224, 2_228_224, 131_072),
    ("22B", 8): (1_325_400_064, 884_998_144, 654_311_424, 213_909_504, 100_663_296),
    ("175B", 1): (2_868_903_936, 2_868_903_936, 855_638_016, 855_638_016, 50_331_648),
    ("175B", 2): (1_560_281_088, 1_434_451_968, 553_648_128, 427_819_008, 50_331_648),
    ("175B", 4): (905_969_664, 717_225_984, 402_653_184, 213_909_504, 50_331_648),
    ("175B", 8): (578_813_952, 358_612_992, 327_155_712, 106_954_752, 50_331_648),
    ("530B", 8): (880_803_840, 513_802_240, 545_259_520, 178_257_920, 83_886_080),
    ("1T", 8): (1_101_004_800, 642_252_800, 681_574_400, 222_822_400, 104_857_600),
}
SHAPES = {"tiny": (8, 256, 128, 2), "22B": (64, 6144, 2048, 4), "175B": (96, 12288, 2048, 1),
          "530B": (128, 20480, 2048, 1), "1T": (160, 25600, 2048, 1)}


@pytest.mark.parametrize("key", list(BASELINE_TABLE))
def test_baseline_table(orc, key):
    a, h, s, b = SHAPES[key[0]]
    t = key[1]
    got = (orc.per_layer_bytes(a, h, s, b, t, "none", False), orc.per_layer_bytes(a, h, s, b, t, "none", True),
           orc.per_layer_bytes(a, h, s, b, t, "selective", False), orc.per_layer_bytes(a, h, s, b, t, "selective", True),
           orc.per_layer_bytes(a, h, s, b, t, "full", True))
    assert got == BASELINE_TABLE[key]
    # the paper's SP formulas: sbh(34/t + 5as/(ht)) and 34 sbh / t
    from fractions import Fraction as F
    sbh = s * b * h
    assert F(*orc.per_layer_bytes_exact(a, h, s, b, t, "none", True)) == sbh * (F(34, t) + F(5 * a * s, h * t))
    assert F(*orc.per_layer_bytes_exact(a, h, s, b, t, "selective", True)) == F(34 * sbh, t)


def test_comm_models(orc):  # collectives.cpp:75-87; verify.cpp:285-321
    for t in (2, 4, 8):
        assert orc.layer_comm_bytes_sp(2048, 4, 6144, t) == orc.layer_comm_bytes_tp(2048, 4, 6144, t)


def test_total_first_stage(orc):  # test_activation_memory.cpp:76-99
    a, h, s = S22
    assert orc.total_first_stage_bytes(a, h, s, 4, 8, "none", False, 48) == \
        orc.per_layer_bytes(a, h, s, 4, 8, "none", False) * 48
    a, h, s = S530  # ParallelLayout{t=8, p=35, m=3, d=1, b=1, n_mb=280}
    assert orc.total_first_stage_bytes(a, h, s, 1, 8, "selective", True, 105, 35, 3) == 24_777_850_880
    # interleave factors 31/24 (175B, p=8 m=3) and 139/105 (530B, p=35 m=3): 96 L -> 124 L
    a, h, s = S175
    one = orc.per_layer_bytes(a, h, s, 1, 8, "selective", True)
    assert orc.total_first_stage_bytes(a, h, s, 1, 8, "selective", True, 96, 8, 3) == one * 124
    with pytest.raises(ValueError):  # L % (p*m) != 0 (config.cpp:114-117)
        orc.total_first_stage_bytes(a, h, s, 1, 8, "selective", True, 96, 7, 3)
