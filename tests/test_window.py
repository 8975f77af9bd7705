"""Microbatch-level recompute window planner: the oracle restatement pinned
to the reference's known answers (test_pipeline_sim.cpp:257-362, acceptance_test.cpp:205-240),
and the libspl planner (C ABI) checked against the oracle. CPU only."""
import random
from fractions import Fraction

import pytest

import paper_2205_05198_b200 as spl
from oracle import window as W
from paper_2205_05198_b200 import report as R

TOY = dict(heads=2, hidden=8, layers=8, seq=4, vocab=16)  # kToy (test_pipeline_sim.cpp:48)


def both(**kw):
    return spl.ModelShape(**kw), W.Model(**kw)


def scenario_budget(m):
    # one fully stored microbatch next to the checkpointed steady state on rank 0
    # (test_pipeline_sim.cpp:262-269: per_layer·L/p + floor(first-stage extras))
    lps = m.layers // m.pipeline
    extras = m.mask_bytes * m.seq * m.microbatch * m.hidden // m.tensor
    full = spl.per_layer_bytes(m.heads, m.hidden, m.seq, m.microbatch, m.tensor, "none",
                               m.sequence_parallel) * lps + extras
    ckpt = spl.per_layer_bytes(m.heads, m.hidden, m.seq, m.microbatch, m.tensor, m.recompute,
                               m.sequence_parallel) * lps + extras
    return full + 3 * ckpt


@pytest.mark.parametrize("impl", ["oracle", "libspl"])
def test_moving_window_scenario(impl):
    m, om = both(**TOY, pipeline=4, microbatches=9, recompute="full", sequence_parallel=False)
    budget = scenario_budget(m)
    plan = W.window_plan(om, budget) if impl == "oracle" else spl.window_plan(m, budget)
    stored = [mb for mb in range(1, 10) if plan["modes"][0][mb - 1]]
    assert stored == [1, 5, 9]
    assert plan["stage_counts"][0] == (3, 6)
    ck = [c for _, c in plan["stage_counts"]]
    assert all(ck[s] <= ck[s - 1] for s in range(1, 4)) and ck[-1] == 0
    assert plan["recomputed_fraction"] == Fraction(6 + 6 + 4 + 0, 4 * 9)
    tl = W.stage_timeline if impl == "oracle" else spl.stage_timeline
    _, peak = tl(om if impl == "oracle" else m, 0, plan["modes"][0], True)
    assert peak <= budget


@pytest.mark.parametrize("impl", ["oracle", "libspl"])
def test_window_boundary_budgets(impl):
    m, om = both(**TOY, pipeline=4, microbatches=9, recompute="selective", sequence_parallel=False)
    plan_fn = W.window_plan if impl == "oracle" else spl.window_plan
    mm = om if impl == "oracle" else m
    big = plan_fn(mm, 2**63 - 1)
    assert all(c == 0 for _, c in big["stage_counts"])
    assert big["recomputed_fraction"] == 0
    tight = plan_fn(mm, big["min_feasible_budget"])
    assert tight["stage_counts"][0] == (0, 9)
    s1, os1 = both(**TOY, pipeline=1, microbatches=3, recompute="selective", sequence_parallel=False)
    one = s1 if impl == "libspl" else os1
    probe = plan_fn(one, 2**63 - 1)
    plan = plan_fn(one, probe["min_feasible_budget"])
    assert plan["stage_counts"][0][0] == 0 and plan["recomputed_fraction"] == 1
    exc = spl.InfeasibleBudget if impl == "libspl" else W.InfeasibleBudget
    with pytest.raises(exc) as e:
        plan_fn(mm, 16)
    assert e.value.min_feasible_budget > 16
    plan_fn(mm, e.value.min_feasible_budget)


def test_window_flops_uplift_175b():
    # test_pipeline_sim.cpp:339-362 on the 175b preset (config.cpp:297)
    kw = dict(heads=96, hidden=12288, layers=96, seq=2048, vocab=51200, tensor=8, pipeline=8,
              interleave=3, microbatch=1, microbatches=64, recompute="selective",
              sequence_parallel=True)
    m, om = both(**kw)
    probe = spl.window_plan(m, 2**63 - 1)
    budget = probe["min_feasible_budget"] + probe["min_feasible_budget"] // 4
    plan = spl.window_plan(m, budget)
    assert plan == W.window_plan(om, budget)
    f = plan["recomputed_fraction"]
    assert 0 < f < 1
    shape = R.ModelShape(96, 12288, 96, 2048, 51200)
    b_total = 1 * 64
    hw = R.hardware_flops(shape, b_total, "selective", recompute_fraction=f, microbatch_level=True)
    ratio = Fraction(hw, R.model_flops(shape, b_total))
    assert 1 < ratio and ratio - 1 <= R.hw_model_ratio_exact(shape) - 1


def test_window_errors():
    m, om = both(**TOY, pipeline=4, microbatches=3)  # n_mb < p
    with pytest.raises(ValueError):
        spl.window_plan(m, 10**9)
    with pytest.raises(ValueError):
        W.window_plan(om, 10**9)
    m, om = both(**TOY, pipeline=2, microbatches=4, recompute="none")
    with pytest.raises(ValueError, match="full or selective"):
        spl.window_plan(m, 10**9)
    with pytest.raises(ValueError):
        W.window_plan(om, 10**9)
    m, _ = both(**{**TOY, "layers": 6}, pipeline=4, microbatches=4)  # L % p
    with pytest.raises(ValueError):
        spl.microbatch_bytes(m, 0)
    with pytest.raises(ValueError):
        spl.microbatch_bytes(spl.ModelShape(**TOY, pipeline=2, microbatches=2), 2)  # stage >= p


def test_in_flight():
    assert spl.in_flight(35, 0) == 35 and spl.in_flight(4, 3) == 1 and spl.in_flight(4, 9) == 0
    with pytest.raises(ValueError):
        spl.in_flight(4, -1)


def test_window_matches_oracle_random():
    rng = random.Random(7)
    for _ in range(300):
        a = rng.choice([1, 2, 4, 8])
        t = rng.choice([1, 2, 4])
        h = a * t * rng.choice([1, 2, 4])
        p = rng.choice([1, 2, 3, 4, 8])
        kw = dict(heads=a, hidden=h, layers=p * rng.choice([1, 2, 3]), seq=t * rng.choice([1, 2, 8]),
                  vocab=rng.choice([1, 16, 50]), tensor=t, pipeline=p,
                  microbatch=rng.choice([1, 2, 4]), microbatches=p + rng.choice([0, 1, 5]),
                  recompute=rng.choice(["full", "selective"]),
                  sequence_parallel=rng.choice([True, False]))
        m, om = both(**kw)
        for s in range(p):
            assert spl.microbatch_bytes(m, s) == W.microbatch_bytes(om, s)
        probe = W.window_plan(om, 2**63 - 1)
        lo = probe["min_feasible_budget"]
        full0 = W.microbatch_bytes(om, 0)[0]
        for budget in (lo, lo + 1, lo + full0 // 2, lo + full0, lo + 3 * full0, 2**63 - 1,
                       rng.randint(lo, lo + 4 * full0)):
            plan = spl.window_plan(m, budget)
            assert plan == W.window_plan(om, budget), kw
            for s in range(p):
                for dealloc in (True, False):
                    assert spl.stage_timeline(m, s, plan["modes"][s], dealloc) == \
                        W.stage_timeline(om, s, plan["modes"][s], dealloc)
                if budget != 2**63 - 1:
                    assert W.stage_timeline(om, s, plan["modes"][s], True)[1] <= budget
        if lo > 0:
            with pytest.raises(spl.InfeasibleBudget) as e:
                spl.window_plan(m, lo - 1)
            assert e.value.min_feasible_budget == lo


def test_cpp_pipeline_facade():
    """The reference's window cases restated in C++ against include/spl_pipeline.hpp (the
    actplan::pipeline signatures over the C ABI); host-only."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "test_window_facade")
    subprocess.run(["make", "build/test_window_facade"], cwd=root, check=True,
                   capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
