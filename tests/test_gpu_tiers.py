"""The orchestrator's three-tier lookup on the GPU (csrc/tiered.cu): L1 = the
HPS GPU cache, L2 = the VDB, L3 = the PDB (host tiers, csrc/tiers.cpp). Spec examples plus a
randomized batch with duplicates against the tiers' own contents (the expected row of a key
is the first tier holding it, else the PDB table's default vector)."""
import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import HotCache
from paper_2210_08803_b200 import tiers as T

pytestmark = pytest.mark.gpu
DIM = 24


def setup(ctx, tmp_path, default=None, cap=1 << 12):
    cache = HotCache(ctx, cap, DIM, ways=8, max_batch=4096)
    vdb = T.Vdb(4, 1 << 12, DIM)
    pdb = T.Pdb(str(tmp_path / "pdb"))
    pdb.create_table("emb", DIM, default=default)
    return cache, vdb, pdb, T.TieredLookup(cache, vdb, pdb, "emb", 4096)


def dev(keys):
    return torch.from_numpy(np.asarray(keys, np.uint64).view(np.int64)).cuda()


def rows(rs, n):
    return rs.standard_normal((n, DIM)).astype(np.float32)


def test_all_keys_in_l1(ctx, tmp_path):
    rs = np.random.default_rng(1)
    cache, vdb, pdb, tl = setup(ctx, tmp_path)
    keys = np.arange(1, 201, dtype=np.uint64) * 7919
    x = rows(rs, 200)
    cache.insert(dev(keys), torch.from_numpy(x).cuda(), dev(np.ones(200, np.uint64)))
    out = tl.lookup(dev(keys)).cpu().numpy()
    assert tl.sources() == {"L1": 200, "L2": 0, "L3": 0, "Default": 0}
    assert np.array_equal(out, x)


def test_cold_start_from_pdb_then_l1(ctx, tmp_path):
    rs = np.random.default_rng(2)
    cache, vdb, pdb, tl = setup(ctx, tmp_path)
    keys = np.arange(1, 301, dtype=np.uint64) * 104729
    x = rows(rs, 300)
    pdb.put_batch("emb", keys, x, np.full(300, 3, np.uint64))
    batch = np.concatenate([keys, keys[:50]])  # duplicates: one tier probe per distinct key
    cache.reset_stats()
    out = tl.lookup(dev(batch)).cpu().numpy()
    assert tl.sources() == {"L1": 0, "L2": 0, "L3": 350, "Default": 0}
    assert np.array_equal(out, np.concatenate([x, x[:50]]))
    assert cache.stats()["queries"] == 300
    tl.await_migrations()
    f, got, ver = vdb.get_batch(keys)  # L3 -> L2 migration at the PDB version
    assert f.all() and (ver == 3).all() and np.array_equal(got, x)
    out = tl.lookup(dev(batch)).cpu().numpy()
    assert tl.sources() == {"L1": 350, "L2": 0, "L3": 0, "Default": 0}
    assert np.array_equal(out, np.concatenate([x, x[:50]]))


def test_l2_hits_migrate_to_l1_only(ctx, tmp_path):
    rs = np.random.default_rng(3)
    cache, vdb, pdb, tl = setup(ctx, tmp_path)
    keys = np.arange(1, 101, dtype=np.uint64) * 15485863
    x = rows(rs, 100)
    vdb.put_batch(keys, x, np.full(100, 9, np.uint64))
    out = tl.lookup(dev(keys)).cpu().numpy()
    assert tl.sources()["L2"] == 100 and np.array_equal(out, x)
    tl.await_migrations()
    assert not pdb.get_batch("emb", keys)[0].any()  # nothing flows down
    out = tl.lookup(dev(keys)).cpu().numpy()
    assert tl.sources()["L1"] == 100 and np.array_equal(out, x)


def test_absent_keys_default_and_no_pollution(ctx, tmp_path):
    cache, vdb, pdb, tl = setup(ctx, tmp_path, default=np.full(DIM, 0.25, np.float32))
    keys = np.array([5, 6, 5, 7], np.uint64)
    for _ in range(2):
        out = tl.lookup(dev(keys)).cpu().numpy()
        assert tl.sources() == {"L1": 0, "L2": 0, "L3": 0, "Default": 4}
        assert (out == 0.25).all()
        tl.await_migrations()
    assert vdb.size() == 0 and cache.size() == 0


def test_randomized_mixed_tiers(ctx, tmp_path):
    rs = np.random.default_rng(4)
    cache, vdb, pdb, tl = setup(ctx, tmp_path, cap=1 << 15)
    universe = np.unique(rs.integers(1, 2**63, 3000).astype(np.uint64))[:2000]
    x = rows(rs, len(universe))
    tier = rs.integers(0, 4, len(universe))  # 0 L1 (+L2+L3), 1 L2 (+L3), 2 L3, 3 nowhere
    ones = np.ones(len(universe), np.uint64)
    m = tier <= 2
    pdb.put_batch("emb", universe[m], x[m], ones[m] * 2)
    m = tier <= 1
    vdb.put_batch(universe[m], x[m], ones[m] * 2)
    m = tier == 0
    cache.insert(dev(universe[m]), torch.from_numpy(x[m]).cuda(), dev(ones[m] * 2))
    for step in range(3):
        pick = rs.integers(0, len(universe), 3000)  # duplicates included
        out = tl.lookup(dev(universe[pick])).cpu().numpy()
        want = np.where((tier[pick] == 3)[:, None], 0.0, x[pick])
        assert np.array_equal(out, want), f"step {step}"
        t = tier[pick]
        assert tl.sources() == {"L1": int((t == 0).sum()), "L2": int((t == 1).sum()), "L3": int((t == 2).sum()),
                                "Default": int((t == 3).sum())}, f"step {step}"
        tl.await_migrations()
        hit = pick[tier[pick] <= 2]
        tier[hit] = 0  # every present key looked up is in L1 now (the cache holds them all)
