"""FLOPs / MFU / HFU reporting over measured layer times.

Restates the reference's FLOP model so that measured B200 layer times can be reported in its
own terms (Table 4/5 rows of the paper, flops_report.schema.json):

  model_flops      flops.cpp:49-58    72·B·L·s·h² + 12·B·L·s²·h + 6·B·s·h·v
  hardware_flops   flops.cpp:60-84    + selective extra (Equation 12·B·L·s²·h | Text 4·B·L·s²·h,
                                      flops.cpp:38-47) or one transformer forward (full,
                                      flops.cpp:28-35); microbatch-level strategies scale the
                                      extra by the recomputed fraction (floor)
  hw_model_ratio   flops.cpp:86-96
  mfu_hfu          flops.cpp:98-113   FLOPs / (iteration_time · devices · peak)
  flops_report     flops.cpp:115-144  JSON: exact integers as decimal strings, ratios num/den,
                                      percents with one decimal (config.cpp:355-359)

Exact integers are Python ints and ratios fractions.Fraction (the reference uses Boost
cpp_int / rational). Errors follow the reference: std::invalid_argument -> ValueError.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

A100_PEAK = 312_000_000_000_000  # Hardware{} default (config.hpp:82-86)
B200_NOMINAL_BF16 = 2_250_000_000_000_000


@dataclass(frozen=True)
class ModelShape:  # config.hpp:27-35
    attention_heads: int
    hidden: int
    layers: int
    seq_len: int
    vocab: int


def rational_from_decimal(text: str) -> Fraction:
    """config.cpp:321-346: exact decimal string -> rational."""
    t = text.strip()
    neg = t.startswith("-")
    if t[:1] in "+-":
        t = t[1:]
    if not t or t.count(".") > 1 or not t.replace(".", "").isdigit():
        raise ValueError(f"bad decimal: {text}")
    whole, _, frac = t.partition(".")
    v = Fraction(int(whole or "0") * 10 ** len(frac) + int(frac or "0"), 10 ** len(frac))
    return -v if neg else v


def percent_string(fraction: Fraction, decimals: int = 1) -> str:
    return f"{float(fraction) * 100.0:.{decimals}f}"


def _check_batch(b_total: int):
    if b_total < 1:
        raise ValueError("b_total must be >= 1")


def transformer_forward_flops(shape: ModelShape, b_total: int) -> int:
    B, s, h = b_total, shape.seq_len, shape.hidden
    return shape.layers * (24 * B * s * h * h + 4 * B * s * s * h)


def model_flops(shape: ModelShape, b_total: int) -> int:
    _check_batch(b_total)
    B, L, s, h, v = b_total, shape.layers, shape.seq_len, shape.hidden, shape.vocab
    return 72 * B * L * s * h * h + 12 * B * L * s * s * h + 6 * B * s * h * v


def hardware_flops(shape: ModelShape, b_total: int, kind: str = "none",
                   selective_model: str = "equation", recompute_fraction: Fraction = Fraction(1),
                   microbatch_level: bool = False) -> int:
    _check_batch(b_total)
    f = Fraction(recompute_fraction)
    if f < 0 or f > 1:
        raise ValueError("recompute_fraction must lie in [0, 1]")
    model = model_flops(shape, b_total)
    B, s, h = b_total, shape.seq_len, shape.hidden
    if kind == "none":
        return model
    if kind == "selective":
        per = 12 * B * s * s * h if selective_model == "equation" else 4 * B * s * s * h
        extra = shape.layers * per
    elif kind == "full":
        extra = transformer_forward_flops(shape, b_total)
    else:
        raise ValueError(f"unknown recompute kind {kind!r}")
    if microbatch_level:
        return model + (Fraction(extra) * f).numerator // (Fraction(extra) * f).denominator
    return model + extra


def hw_model_ratio_exact(shape: ModelShape) -> Fraction:
    return Fraction(hardware_flops(shape, 1, "selective"), model_flops(shape, 1))


def hw_model_ratio_approx(shape: ModelShape) -> Fraction:
    return 1 + Fraction(shape.seq_len, 6 * shape.hidden)


def mfu_hfu(shape: ModelShape, b_total: int, kind: str, iteration_time, devices: int,
            peak_flops_per_device: int = A100_PEAK, selective_model: str = "equation",
            recompute_fraction: Fraction = Fraction(1), microbatch_level: bool = False):
    it = rational_from_decimal(iteration_time) if isinstance(iteration_time, str) else Fraction(iteration_time)
    if it <= 0:
        raise ValueError("iteration_time must be positive")
    denom = it * devices * peak_flops_per_device
    mfu = Fraction(model_flops(shape, b_total)) / denom
    hfu = Fraction(hardware_flops(shape, b_total, kind, selective_model, recompute_fraction,
                                  microbatch_level)) / denom
    return mfu, hfu


def flops_report(shape: ModelShape, b_total: int, kind: str, iteration_time=None, devices: int = 1,
                 peak_flops_per_device: int = A100_PEAK, selective_model: str = "equation") -> dict:
    """flops_report + to_json (flops.cpp:115-144), schemas/flops_report.schema.json."""
    mf = model_flops(shape, b_total)
    hf = hardware_flops(shape, b_total, kind, selective_model)
    ratio = Fraction(hf, mf)
    doc = {"model_flops_per_iter": str(mf), "hardware_flops_per_iter": str(hf),
           "hw_model_ratio": {"num": str(ratio.numerator), "den": str(ratio.denominator)},
           "hw_model_ratio_value": float(ratio),
           "hw_model_ratio_approx": float(hw_model_ratio_approx(shape))}
    if iteration_time is not None:
        mfu, hfu = mfu_hfu(shape, b_total, kind, iteration_time, devices, peak_flops_per_device,
                           selective_model)
        doc["mfu_percent"] = percent_string(mfu)
        doc["hfu_percent"] = percent_string(hfu)
    return doc


# ---------------------------------------------------------------- Table 4 of the paper
# "Time to execute the forward and backward passes of one transformer layer of the 22B model"
# (t = 8 A100s): rows and the published numbers (ms).
TABLE4_ROWS = [  # (label, recompute, sequence_parallel, published fwd, bwd)
    ("Baseline no recompute", "none", False, 7.7, 11.9),
    ("Sequence Parallelism", "none", True, 7.2, 11.8),
    ("Baseline with recompute", "full", False, 7.7, 19.5),
    ("Selective Recompute", "selective", False, 7.7, 13.2),
    ("Selective + Sequence", "selective", True, 7.2, 13.1),
]


def table4(measured: dict) -> list[dict]:
    """Rows of Table 4 from measured {(recompute, sp): (fwd_ms, bwd_ms)}; overhead is the
    combined time over the no-recompute tensor-parallel baseline, minus one."""
    base = sum(measured[("none", False)])
    rows = []
    for label, rc, sp, pf, pb in TABLE4_ROWS:
        f, b = measured[(rc, sp)]
        rows.append({"experiment": label, "recompute": rc, "sequence_parallel": sp,
                     "forward_ms": f, "backward_ms": b, "combined_ms": f + b,
                     "overhead_percent": (f + b) / base * 100.0 - 100.0,
                     "a100_published_ms": {"forward": pf, "backward": pb, "combined": round(pf + pb, 1)}})
    return rows
