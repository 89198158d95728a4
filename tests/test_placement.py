"""Placement planners against the SPEC's examples — CPU only."""
import itertools

import numpy as np
import pytest

from paper_2210_08803_b200 import HpsError
from paper_2210_08803_b200 import placement as P
from tests import oracle_lib as O

UNIT = 4  # one "unit" = a 1-row dim-1 slot (4 bytes)


def test_localized_examples():
    assert P.plan_localized([P.SlotSpec(10, 1)], [1000]) == [0]
    assert sorted(P.plan_localized([P.SlotSpec(10, 1), P.SlotSpec(10, 1)], [1000, 1000])) == [0, 1]
    # sizes 5,3,3 units on 2 devices of 8 units -> {5} + {3,3}
    plan = P.plan_localized([P.SlotSpec(5, 1), P.SlotSpec(3, 1), P.SlotSpec(3, 1)], [8 * UNIT, 8 * UNIT])
    assert plan[1] == plan[2] != plan[0]
    with pytest.raises(HpsError) as e:
        P.plan_localized([P.SlotSpec(9, 1)], [8 * UNIT, 8 * UNIT])
    assert e.value.code == 16  # Infeasible


def test_localized_is_lpt_and_matches_brute_force_on_small_cases():
    rs = np.random.default_rng(1)
    for _ in range(30):
        sizes = rs.integers(1, 20, rs.integers(1, 7))
        budgets = [int(s) for s in rs.integers(20, 60, 3)]
        slots = [P.SlotSpec(int(s), 1) for s in sizes]
        try:
            plan = P.plan_localized(slots, [b * UNIT for b in budgets])
        except HpsError:
            continue
        # restate LPT: descending size (ties by index), device with most remaining budget (ties lowest)
        rem = list(budgets)
        want = [0] * len(sizes)
        for s in sorted(range(len(sizes)), key=lambda i: (-sizes[i], i)):
            d = max(range(len(rem)), key=lambda j: (rem[j], -j))
            want[s] = d
            rem[d] -= sizes[s]
        assert plan == want


def test_distributed_examples():
    slots = [P.SlotSpec(1000, 4)]
    P.plan_distributed(slots, [4000 * 4])
    with pytest.raises(HpsError):
        P.plan_distributed(slots, [1000, 1000])  # 16 KB over 2 x 1 KB
    keys = np.random.default_rng(2).integers(0, 2**63, 1_000_000, dtype=np.int64).astype(np.uint64)
    assert not P.shard_of(keys, 1).any()
    c = np.bincount(P.shard_of(keys, 8), minlength=8)
    assert c.max() / c.mean() <= 1.05
    want = np.empty(len(keys), dtype=np.uint32)
    O.lib().orc_partition_of_n(O.P(keys), len(keys), 8, O.P(want))
    assert np.array_equal(P.shard_of(keys, 8), want)


def test_estimate_comm_examples():
    fwd, bwd = P.estimate_comm(P.DISTRIBUTED, 1024, [P.SlotSpec(100, 16)], 8)
    assert fwd == 57344 and bwd == 57344
    assert P.estimate_comm(P.LOCALIZED, 1024, [P.SlotSpec(100, 16)], 1) == (0.0, 0.0)
    assert P.estimate_comm(P.HYBRID, 1024, [P.SlotSpec(100, 16, 3)], 8, p_cold=[0.0]) == (0.0, 0.0)
    f1, _ = P.estimate_comm(P.HYBRID, 1024, [P.SlotSpec(100, 16, 3)], 8, p_cold=[0.5])
    assert f1 == 1024 * 3 * 0.5 * 16 * 4 * 7 / 8


def test_hybrid_hot_set():
    keys = np.array([5, 3, 9, 1, 7], dtype=np.uint64)
    counts = np.array([10, 10, 2, 50, 0], dtype=np.uint64)
    assert list(P.plan_hybrid(keys, counts, 4, 3 * 16)) == [1, 3, 5]  # count desc, key asc
    assert len(P.plan_hybrid(keys, counts, 4, 0)) == 0                 # budget 0 == distributed
    assert len(P.plan_hybrid(keys, counts, 4, 10**9)) == 5            # all hot
