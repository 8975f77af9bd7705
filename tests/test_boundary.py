"""Host-side pieces of the drop-in boundary (no GPU): RecomputeStrategy::parse / name
(config.cpp:36-84, test_config.cpp:92-106) and RankShardedTensor (tensor.cpp:227-259,
test_seqpar.cpp:109-120) in the Python mirror, and the C-ABI symbols of the free-standing
reference functions."""
import numpy as np
import pytest

import paper_2205_05198_b200 as spl


def test_strategy_round_trip():
    S = spl.RecomputeStrategy
    for n in ("none", "full", "selective", "none+seq", "full+seq", "selective+seq",
              "full+mblevel", "selective+seq+mblevel"):
        assert S.parse(n).name() == n
    assert S.parse("full+seq").sequence_parallel
    assert S.parse("selective+mblevel").microbatch_level
    assert S.parse("seq+selective") == S.parse("selective+seq")
    for bad in ("none+mblevel", "bogus", "full+bogus", "full+selective", "seq", ""):
        with pytest.raises(ValueError):
            S.parse(bad)


def test_rank_sharded_tensor(orc):
    full = orc.random_uniform(1, (4, 2, 6), -1, 1)
    sh = spl.RankShardedTensor.from_full(full, "sequence", 0, 2)
    assert len(sh.shards) == 2 and np.array_equal(sh.to_full(0), full)
    sh.check()
    rep = spl.RankShardedTensor.from_full(full, "replicated", 0, 2)
    rep.check()
    rep.shards[1][0, 0, 0] += 1.0
    with pytest.raises(ValueError):
        rep.check()
    with pytest.raises(ValueError):
        spl.RankShardedTensor.from_full(full, "sequence", 0, 3)


def test_boundary_symbols_exported():
    lib = spl.lib()
    for name in ("spl_attention_interior_qk", "spl_all_gather", "spl_reduce_scatter",
                 "spl_all_reduce"):
        assert hasattr(lib, name)
        assert name in spl.header_symbols()
