"""FLOP / MFU reporting (paper_2205_05198_b200/report.py) against the reference's own known
answers (/root/reference/proj/tests/test_flops.cpp)."""
from fractions import Fraction

import pytest

from paper_2205_05198_b200 import report as R

K175 = R.ModelShape(96, 12288, 96, 2048, 51200)
K530 = R.ModelShape(128, 20480, 105, 2048, 51200)
K22 = R.ModelShape(64, 6144, 48, 2048, 51200)
K1T = R.ModelShape(160, 25600, 128, 2048, 51200)


def test_model_flops_pins():  # test_flops.cpp:30-50
    assert R.model_flops(K175, 64) == 141091531099471872
    assert R.model_flops(K530, 560) == 2 * R.model_flops(K530, 280)
    s = R.ModelShape(96, 12288, 96, 2048, 1)
    assert R.model_flops(s, 64) == 72 * 64 * 96 * 2048 * 12288 ** 2 + 12 * 64 * 96 * 2048 ** 2 * 12288 + 6 * 64 * 2048 * 12288


def test_hardware_flops():  # test_flops.cpp:52-86
    B = 64
    m = R.model_flops(K175, B)
    assert R.hardware_flops(K175, B, "none") == m
    assert R.hardware_flops(K175, B, "selective") == 144891443285065728
    assert R.hardware_flops(K175, B, "full") == m + 24 * B * 96 * 2048 * 12288 ** 2 + 4 * B * 96 * 2048 ** 2 * 12288
    m8 = R.model_flops(K530, 8)
    assert R.hardware_flops(K530, 8, "selective", "equation") - m8 == 12 * 8 * 105 * 2048 ** 2 * 20480
    assert R.hardware_flops(K530, 8, "selective", "text") - m8 == 4 * 8 * 105 * 2048 ** 2 * 20480
    for sh in (K22, K175, K530, K1T):
        d = R.hardware_flops(sh, 17, "selective") - R.model_flops(sh, 17)
        assert Fraction(d) == Fraction(72 * 17 * sh.layers * sh.seq_len * sh.hidden ** 2) * Fraction(sh.seq_len, 6 * sh.hidden)


def test_ratios():  # test_flops.cpp:88-99
    assert float(R.hw_model_ratio_exact(K175)) - 1 == pytest.approx(0.0269, rel=0.01)
    assert float(R.hw_model_ratio_exact(K530)) - 1 == pytest.approx(0.0164, rel=0.01)
    assert R.hw_model_ratio_approx(K175) == 1 + Fraction(2048, 6 * 12288)


def test_mfu_hfu_reference_points():  # test_flops.cpp:101-116 (Table 5 of the paper)
    mfu, hfu = R.mfu_hfu(K175, 64, "selective", "13.75", 64)
    assert float(mfu) * 100 == pytest.approx(51.4, rel=0.004)
    assert float(hfu) * 100 == pytest.approx(52.8, rel=0.004)
    mfu, _ = R.mfu_hfu(K530, 2240, "selective", "39.15", 2240)
    assert float(mfu) * 100 == pytest.approx(54.2, rel=0.004)
    mfu, hfu = R.mfu_hfu(K1T, 512, "selective", "71.49", 512)
    assert float(mfu) * 100 == pytest.approx(56.3, rel=0.004)
    assert float(hfu) * 100 == pytest.approx(57.0, rel=0.004)
    a, b = R.mfu_hfu(K22, 4, "selective", "1.10", 8)
    c, d = R.mfu_hfu(K22, 4, "selective", "2.20", 8)
    assert a == 2 * c and b == 2 * d


def test_microbatch_level_and_ordering():  # test_flops.cpp:131-154
    for k in ("none", "selective", "full"):
        hw, m = R.hardware_flops(K530, 280, k), R.model_flops(K530, 280)
        assert hw >= m and (hw == m) == (k == "none")
    m = R.model_flops(K175, 64)
    extra = R.hardware_flops(K175, 64, "selective") - m
    assert R.hardware_flops(K175, 64, "selective", "equation", Fraction(1, 2), True) == m + extra // 2
    assert R.hardware_flops(K175, 64, "selective", "equation", Fraction(0), True) == m


def test_report_json():  # test_flops.cpp:156-168
    bare = R.flops_report(K175, 64, "selective", None, 64)
    assert "mfu_percent" not in bare and bare["hw_model_ratio_value"] > 1
    doc = R.flops_report(K175, 64, "selective", "13.75", 64)
    assert doc["mfu_percent"] == "51.4" and doc["hfu_percent"] == "52.8"
    assert doc["model_flops_per_iter"] == "141091531099471872"


def test_invalid():  # test_flops.cpp:170-181
    with pytest.raises(ValueError):
        R.model_flops(K175, 0)
    with pytest.raises(ValueError):
        R.mfu_hfu(K175, 64, "none", 0, 64)
    with pytest.raises(ValueError):
        R.mfu_hfu(K175, 64, "none", -1, 64)
    with pytest.raises(ValueError):
        R.hardware_flops(K175, 64, "selective", "equation", Fraction(2))
    with pytest.raises(ValueError):
        R.rational_from_decimal("1.2.3")


def test_table4_rows():
    meas = {("none", False): (1.0, 2.0), ("none", True): (0.9, 1.9), ("full", False): (1.0, 3.0),
            ("selective", False): (1.0, 2.2), ("selective", True): (0.9, 2.1)}
    rows = R.table4(meas)
    assert [r["experiment"] for r in rows][0] == "Baseline no recompute"
    assert rows[0]["overhead_percent"] == 0.0
    assert rows[2]["overhead_percent"] == pytest.approx(100.0 / 3.0)
    assert rows[4]["a100_published_ms"]["combined"] == 20.3
