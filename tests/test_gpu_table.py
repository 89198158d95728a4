"""GPU parity for K2-K5 (index insert/find, fused lookup, dedup + reduction + optimizers)
against the CPU oracle, through the C-ABI. Bit-exact for indices/rows/dedup; fp32 values
are compared bitwise as well (both sides follow DESIGN.md §4's operation order) and, as the
documented contract, within 1e-5 relative."""
import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import EmbeddingTableGroup, HpsError, opt_params
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def t64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def close(gpu, cpu):
    gpu = np.asarray(gpu, dtype=np.float32)
    cpu = np.asarray(cpu, dtype=np.float32)
    tol = RTOL * np.maximum(np.abs(cpu), 1e-6)
    bad = np.abs(gpu - cpu) > tol
    assert not bad.any(), f"{bad.sum()} elements out of tolerance; max abs err {np.abs(gpu - cpu).max()}"
    return np.array_equal(gpu.view(np.uint32), cpu.view(np.uint32))


def make_pair(ctx, caps, dim, slot_table, optimizer="sgd", seed=11, a0=0.0, max_keys=1 << 16, max_bags=1 << 16):
    g = EmbeddingTableGroup(ctx, caps, dim, slot_table, optimizer, max_keys, max_bags, seed, a0)
    o = O.OracleTable(caps, dim, slot_table, optimizer, seed, a0)
    return g, o


def test_init_value_matches_oracle(ctx):
    L = O.lib()
    for seed in [0, 1, 2**63 + 5]:
        for key in [0, 1, 2**64 - 1, 123456789]:
            for j in [0, 1, 15, 127]:
                a = ctx.lib.hps_gpu_init_value(seed, key, j)
                b = L.orc_init_value(seed, key, j)
                assert np.float32(a).view(np.uint32) == np.float32(b).view(np.uint32)


def test_insert_find_rows_first_occurrence(ctx):
    g, o = make_pair(ctx, [1000, 50], 16, [0, 1])
    rs = np.random.default_rng(0)
    for rnd in range(4):
        keys = rs.integers(0, 300, 500).astype(np.uint64)  # lots of duplicates, incl. key 0
        keys[:3] = [0, 2**64 - 1, 0]
        got = g.insert(0, t64(keys)).cpu().numpy().view(np.uint64)
        st, want = o.insert(0, keys)
        ctx.sync()
        assert st == 0
        np.testing.assert_array_equal(got, want)
        assert g.size(0) == o.size(0)
    n = g.size(0)
    w, _, _ = g.export(0, 0, n)
    ow, _, _ = o.export(0, 0, n)
    np.testing.assert_array_equal(w.cpu().numpy().view(np.uint32), ow.view(np.uint32))
    np.testing.assert_array_equal(g.row_keys(0, 0, n).cpu().numpy().view(np.uint64), o.row_keys(0, 0, n))
    probe = rs.integers(0, 400, 1000).astype(np.uint64)
    np.testing.assert_array_equal(g.find(0, t64(probe)).cpu().numpy().view(np.uint64), o.find(0, probe))
    # table 1 is an independent namespace
    np.testing.assert_array_equal(g.find(1, t64(probe)).cpu().numpy().view(np.uint64), o.find(1, probe))


def test_insert_with_rows_first_occurrence_wins(ctx):
    g, o = make_pair(ctx, [100], 8, [0])
    keys = np.array([5, 6, 5, 7, 6], dtype=np.uint64)
    rows = np.arange(40, dtype=np.float32).reshape(5, 8)
    g.insert(0, t64(keys), torch.from_numpy(rows).cuda())
    o.insert(0, keys, rows)
    keys2 = np.array([7, 9, 7], dtype=np.uint64)  # existing 7 updated by its first occurrence
    rows2 = -np.arange(24, dtype=np.float32).reshape(3, 8)
    g.insert(0, t64(keys2), torch.from_numpy(rows2).cuda())
    o.insert(0, keys2, rows2)
    ctx.sync()
    n = g.size(0)
    assert n == o.size(0) == 4
    np.testing.assert_array_equal(g.export(0, 0, n)[0].cpu().numpy(), o.export(0, 0, n)[0])


def test_insert_non_finite_rejected_whole_call(ctx):
    g, o = make_pair(ctx, [100], 8, [0])
    rows = np.ones((3, 8), dtype=np.float32)
    rows[2, 5] = np.nan
    g.insert(0, t64(np.array([1, 2, 3], dtype=np.uint64)), torch.from_numpy(rows).cuda())
    with pytest.raises(HpsError) as e:
        ctx.sync()
    assert e.value.code == 10
    assert g.size(0) == 0
    assert (g.find(0, t64(np.array([1, 2, 3], dtype=np.uint64))).cpu().numpy() == -1).all()


def test_insert_capacity_infeasible_rolls_back(ctx):
    g, o = make_pair(ctx, [10], 8, [0])
    g.insert(0, t64(np.arange(6, dtype=np.uint64)))
    ctx.sync()
    g.insert(0, t64(np.arange(3, 12, dtype=np.uint64)))  # 6 new keys > 4 free rows
    with pytest.raises(HpsError) as e:
        ctx.sync()
    assert e.value.code == 16
    assert g.size(0) == 6
    found = g.find(0, t64(np.arange(12, dtype=np.uint64))).cpu().numpy()
    assert (found[:6] == np.arange(6)).all() and (found[6:] == -1).all()
    g.insert(0, t64(np.arange(3, 10, dtype=np.uint64)))  # 4 new keys fit exactly
    ctx.sync()
    assert g.size(0) == 10


def _one_hot_round(ctx, g, o, keys, n_samples, rs, opt="sgd", steps=3, dim=16, lr=0.05, **kw):
    for step in range(1, steps + 1):
        out = g.lookup(t64(keys), n_samples, train=True)
        ref = o.lookup(keys, n_samples, train=True)
        close(out.cpu().numpy(), ref)
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(opt, lr, step=step, **kw)
        g.backward_update(torch.from_numpy(dout).cuda(), lr, params=p)
        o.backward_update(dout, p)
        ctx.sync()
        np.testing.assert_array_equal(g.last_unique().cpu().numpy().view(np.uint32), o.last_unique())


@pytest.mark.parametrize("opt", ["sgd", "adagrad", "adam"])
def test_one_hot_train_step_parity(ctx, opt):
    rs = np.random.default_rng(5)
    caps = [3000, 17, 500]
    slots = [0, 1, 2, 1]
    g, o = make_pair(ctx, caps, 32, slots, opt, a0=0.1 if opt == "adagrad" else 0.0)
    for t, c in enumerate(caps):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks))
        o.insert(t, ks)
        if t == 0:
            pool0 = ks
        if t == 1:
            pool1 = ks
        if t == 2:
            pool2 = ks
    B = 700
    keys = np.stack([rs.choice(pool0, B), rs.choice(pool1, B), rs.choice(pool2, B), rs.choice(pool1, B)], 1).ravel()
    keys[::97] = 12345678901  # absent keys -> default vector, no update
    g.set_default_vector(2, np.full(32, 0.25, np.float32))
    o.set_default(2, np.full(32, 0.25, np.float32))
    _one_hot_round(ctx, g, o, keys, B, rs, opt, eps=1e-7 if opt == "adagrad" else 1e-8)
    for t, c in enumerate(caps):
        w, s0, s1 = g.export(t, 0, c)
        ow, os0, os1 = o.export(t, 0, c)
        assert close(w.cpu().numpy(), ow), "weights not bitwise equal"
        if s0 is not None:
            assert close(s0.cpu().numpy(), os0)
        if s1 is not None:
            assert close(s1.cpu().numpy(), os1)


@pytest.mark.parametrize("combiner", ["sum", "mean"])
def test_multi_hot_train_step_parity(ctx, combiner):
    rs = np.random.default_rng(9)
    caps = [4000, 40]
    slots = [0, 1, 0]
    g, o = make_pair(ctx, caps, 64, slots, "adagrad", a0=0.0)
    pools = []
    for t, c in enumerate(caps):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks))
        o.insert(t, ks)
        pools.append(ks)
    B = 500
    lens = rs.integers(0, 20, B * 3)  # includes empty bags
    lens[5] = 300  # one long bag
    offsets = np.zeros(B * 3 + 1, dtype=np.uint32)
    offsets[1:] = np.cumsum(lens)
    keys = []
    for b in range(B * 3):
        pool = pools[slots[b % 3]]
        # zipf-ish skew: a few hot keys take most occurrences (multi-chunk segments)
        hot = rs.random(lens[b]) < 0.5
        keys.append(np.where(hot, pool[rs.integers(0, 3, lens[b])], rs.choice(pool, lens[b])))
    keys = np.concatenate(keys).astype(np.uint64)
    for step in range(1, 4):
        out = g.lookup(t64(keys), B, offsets=torch.from_numpy(offsets.view(np.int32)).cuda(), combiner=combiner,
                       train=True)
        ref = o.lookup(keys, B, offsets=offsets, combiner=combiner, train=True)
        close(out.cpu().numpy(), ref)
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params("adagrad", 0.01, eps=1e-7)
        g.backward_update(torch.from_numpy(dout).cuda(), 0.01, params=p)
        o.backward_update(dout, p)
        ctx.sync()
    for t, c in enumerate(caps):
        w, s0, _ = g.export(t, 0, c)
        ow, os0, _ = o.export(t, 0, c)
        assert close(w.cpu().numpy(), ow)
        assert close(s0.cpu().numpy(), os0)
    np.testing.assert_array_equal(g.last_unique().cpu().numpy().view(np.uint32), o.last_unique())


def test_lookup_from_host_buffers(ctx):
    rs = np.random.default_rng(2)
    g, o = make_pair(ctx, [1000], 16, [0, 0])
    ks = rs.integers(0, 2**63, 1000).astype(np.uint64)
    g.insert(0, t64(ks))
    o.insert(0, ks)
    keys = rs.choice(ks, 2 * 300)
    pinned = torch.from_numpy(keys.view(np.int64)).pin_memory()
    out = g.lookup(pinned, 300, keys_on_host=True)
    close(out.cpu().numpy(), o.lookup(keys, 300))


def test_config1_full_size_parity(ctx):
    """BASELINE config 1 in full: 1M keys, dim 16, 26 slots x 1 hot, batch 2048, SGD."""
    from paper_2210_08803_b200 import workload as W
    cfg = W.config1()
    g, o = make_pair(ctx, cfg.cards, cfg.dim, cfg.slots(), "sgd", seed=cfg.seed, max_keys=2048 * 26,
                     max_bags=2048 * 26)
    all_keys = W.table_keys(cfg.seed, 0, np.arange(cfg.cards[0]))
    g.insert(0, t64(all_keys))
    o.insert(0, all_keys)
    gen = W.BatchGen(cfg)
    rs = np.random.default_rng(4)
    for step in range(3):
        keys, _, idx, _ = gen.batch(step)
        np.testing.assert_array_equal(g.find(0, t64(keys[:1000])).cpu().numpy(), idx[:1000])
        _one_hot_round(ctx, g, o, keys, cfg.batch, rs, "sgd", steps=1, lr=cfg.lr)
    w = g.export(0, 0, cfg.cards[0])[0].cpu().numpy()
    assert close(w, o.export(0, 0, cfg.cards[0])[0])


@pytest.mark.parametrize("opt", ["sgd", "adam"])
def test_skewed_segments_all_paths(ctx, opt):
    """Segment lengths 1, 2, 3..32 (warp bitonic), 33..4096 (CTA smem sort) and > 4096
    (bitmap walk), in one batch, one key per bag, through every backward kernel."""
    rs = np.random.default_rng(21)
    g, o = make_pair(ctx, [100000], 16, [0], opt, max_keys=1 << 17, max_bags=1 << 17)
    pool = rs.integers(0, 2**63, 100000).astype(np.uint64)
    g.insert(0, t64(pool))
    o.insert(0, pool)
    parts = [np.repeat(pool[0], 20000), np.repeat(pool[1], 4097), np.repeat(pool[2], 4096), np.repeat(pool[3], 33),
             np.repeat(pool[4:40], 32), np.repeat(pool[40:90], 3), np.repeat(pool[90:300], 2), pool[300:20000]]
    keys = np.concatenate(parts)
    keys = keys[rs.permutation(len(keys))]
    for step in range(1, 3):
        out = g.lookup(t64(keys), len(keys), train=True)
        ref = o.lookup(keys, len(keys), train=True)
        close(out.cpu().numpy(), ref)
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(opt, 0.01, step=step)
        g.backward_update(torch.from_numpy(dout).cuda(), 0.01, params=p)
        o.backward_update(dout, p)
        ctx.sync()
        np.testing.assert_array_equal(g.last_unique().cpu().numpy().view(np.uint32), o.last_unique())
    w = g.export(0, 0, 100000)[0].cpu().numpy()
    assert close(w, o.export(0, 0, 100000)[0])


def test_train_lookup_twice_without_backward(ctx):
    """A training lookup whose gradients are never applied must not leak into the next step."""
    rs = np.random.default_rng(8)
    g, o = make_pair(ctx, [500], 16, [0])
    pool = rs.integers(0, 2**63, 500).astype(np.uint64)
    g.insert(0, t64(pool))
    o.insert(0, pool)
    k1 = rs.choice(pool, 300)
    g.lookup(t64(k1), 300, train=True)
    k2 = rs.choice(pool, 400)
    g.lookup(t64(k2), 400, train=True)
    o.lookup(k2, 400, train=True)
    d = rs.standard_normal((400, 16)).astype(np.float32)
    p = opt_params("sgd", 0.1)
    g.backward_update(torch.from_numpy(d).cuda(), 0.1, params=p)
    o.backward_update(d, p)
    ctx.sync()
    assert close(g.export(0, 0, 500)[0].cpu().numpy(), o.export(0, 0, 500)[0])


@pytest.mark.parametrize("multi", [False, True])
def test_insert_on_miss_train_parity(ctx, multi):
    """Config-5 shape at small scale: one hashed table, rows materialise on first touch
    (HPS_LOOKUP_INSERT), Adam. The oracle inserts the batch (first-occurrence rows) then
    looks up: same rows, same init, same updates."""
    from paper_2210_08803_b200 import workload as W
    cfg = W.config5(batch_per_gpu=128, capacity=40_000)
    cfg.dim, cfg.keyspace = 64, 2_000_000
    if multi:
        cfg.hot = 3
    gen = W.BatchGen(cfg)
    g, o = make_pair(ctx, cfg.cards, cfg.dim, cfg.slots(), "adam", max_keys=1 << 15, max_bags=1 << 13)
    rs = np.random.default_rng(3)
    for step in range(1, 5):
        keys, offs, _, _ = gen.batch(step)
        if multi:
            kh = torch.from_numpy(keys.view(np.int64)).pin_memory()
            oh = torch.from_numpy(offs.view(np.int32)).pin_memory()
            out = g.lookup(kh, cfg.batch, offsets=oh, train=True, keys_on_host=True, insert_missing=True)
        else:
            out = g.lookup(t64(keys), cfg.batch, train=True, insert_missing=True)
        st, _ = o.insert(0, keys)
        assert st == 0
        ref = o.lookup(keys, cfg.batch, offsets=offs, train=True)
        assert close(out.cpu().numpy(), ref)
        dout = (rs.standard_normal(ref.shape) * 0.1).astype(np.float32)
        p = opt_params("adam", 0.01, step=step)
        g.backward_update(torch.from_numpy(dout).cuda(), 0.01, params=p)
        o.backward_update(dout, p)
        ctx.sync()
        assert g.size(0) == o.size(0)
    n = g.size(0)
    assert n > cfg.batch  # rows really materialised on first touch
    np.testing.assert_array_equal(g.row_keys(0, 0, n).cpu().numpy().view(np.uint64), o.row_keys(0, 0, n))
    w, s0, s1 = g.export(0, 0, n)
    ow, os0, os1 = o.export(0, 0, n)
    assert close(w.cpu().numpy(), ow) and close(s0.cpu().numpy(), os0) and close(s1.cpu().numpy(), os1)


def test_insert_on_miss_rejects_multi_table(ctx):
    g, _ = make_pair(ctx, [100, 100], 8, [0, 1])
    with pytest.raises(HpsError) as e:
        g.lookup(t64(np.arange(8, dtype=np.uint64)), 4, insert_missing=True)
    assert e.value.code == 1


def test_keys_only_insert_matches_oracle(ctx):
    """The keys-only insert (no rows, no rows_out: read-only probe for keys committed
    earlier) assigns the same first-occurrence rows as the oracle."""
    g, o = make_pair(ctx, [5000], 16, [0])
    rs = np.random.default_rng(12)
    for rnd in range(5):
        keys = rs.integers(0, 6000, 1500).astype(np.uint64)  # mix of present, new and repeated keys
        assert g.insert(0, t64(keys), return_rows=False) is None
        o.insert(0, keys)
        ctx.sync()
        assert g.size(0) == o.size(0)
    n = g.size(0)
    np.testing.assert_array_equal(g.row_keys(0, 0, n).cpu().numpy().view(np.uint64), o.row_keys(0, 0, n))
    np.testing.assert_array_equal(g.export(0, 0, n)[0].cpu().numpy().view(np.uint32), o.export(0, 0, n)[0].view(np.uint32))


def _bt_used(ctx, g):
    import ctypes
    v = ctypes.c_uint64(0)
    assert ctx.lib.hps_gpu_debug_batch_table_used(g.h, ctypes.byref(v)) == 0
    return v.value


@pytest.mark.parametrize("multi", [False, True])
def test_batch_table_self_cleaning(ctx, multi):
    """The per-batch dedup table returns to empty after every backward, after a training
    lookup whose backward never came (reset by the next record), over many steps with
    skewed keys (long segments, hot rows shared by every counting CTA)."""
    rs = np.random.default_rng(21)
    caps = [3, 50, 20000]
    g, o = make_pair(ctx, caps, 32, [0, 1, 2, 2], optimizer="adagrad")
    pools = []
    for t, c in enumerate(caps):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks))
        o.insert(t, ks)
        pools.append(ks)
    B = 3000
    for step in range(6):
        if multi:
            lens = rs.integers(0, 6, B * 4).astype(np.uint32)
            offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
            keys = np.concatenate([rs.choice(pools[[0, 1, 2, 2][b % 4]], l) for b, l in enumerate(lens)]).astype(np.uint64)
            ot = torch.from_numpy(offs.view(np.int32)).cuda()
        else:
            keys = np.stack([rs.choice(pools[s], B) for s in [0, 1, 2, 2]], 1).ravel()
            offs, ot = None, None
        out = g.lookup(t64(keys), B, offsets=ot, train=True)
        ref = o.lookup(keys, B, offsets=offs, train=True)
        assert np.array_equal(out.cpu().numpy(), ref)
        if step == 2:
            continue  # no backward: the next record must clean up
        d = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params("adagrad", 0.05)
        g.backward_update(torch.from_numpy(d).cuda(), 0.05, params=p)
        o.backward_update(d, p)
        assert _bt_used(ctx, g) == 0
    for t, c in enumerate(caps):
        assert close(g.export(t, 0, c)[0].cpu().numpy(), o.export(t, 0, c)[0])


@pytest.mark.parametrize("dedup", ["persistent", "flat"])
def test_unconsumed_record_between_graph_replays(ctx, dedup, monkeypatch):
    """A captured [training lookup + backward] graph replayed after an EAGER training lookup
    whose backward never came: the graph's dedup must first return that record's batch-table
    entries to empty (k_dedup checks counts[5] itself; the flat dedup's reset kernel is in the
    graph). Both dedup variants, against the oracle."""
    monkeypatch.setenv("HPS_GPU_DEDUP", dedup)
    rs = np.random.default_rng(17)
    caps = [3, 800]
    g, o = make_pair(ctx, caps, 32, [0, 1, 1])
    pools = []
    for t, c in enumerate(caps):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks))
        o.insert(t, ks)
        pools.append(ks)
    B = 500
    kbuf = torch.zeros(B * 3, dtype=torch.int64, device="cuda")
    dbuf = torch.zeros(B * 3, 32, dtype=torch.float32, device="cuda")
    obuf = torch.zeros(B * 3, 32, dtype=torch.float32, device="cuda")
    p = opt_params("sgd", 0.05)

    def batch():
        return np.stack([rs.choice(pools[t], B) for t in [0, 1, 1]], 1).ravel()

    def step():
        g.lookup(kbuf, B, train=True, out=obuf)
        g.backward_update(dbuf, 0.05, params=p)

    stream = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    stream.wait_stream(main)
    gr = None
    with torch.cuda.stream(stream):
        ctx.set_stream(stream)
        try:
            for it in range(6):
                keys = batch()
                d = rs.standard_normal((B * 3, 32)).astype(np.float32)
                kbuf.copy_(t64(keys))
                dbuf.copy_(torch.from_numpy(d))
                ref = o.lookup(keys, B, train=True)
                o.backward_update(d, p)
                if gr is None:
                    step()  # warm-up, then capture
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gr, stream=stream):
                        step()
                else:
                    gr.replay()
                stream.synchronize()
                if it > 0:
                    assert close(obuf.cpu().numpy(), ref), f"replay {it}"
                # an eager training lookup (different keys) whose backward never comes
                junk = batch()
                g.lookup(t64(junk), B, train=True)
                o.lookup(junk, B, train=True)
            gr.replay()  # (the oracle's pending record is the junk one: replay without a check)
            stream.synchronize()
        finally:
            main.wait_stream(stream)
            ctx.set_stream(main)
    ctx.sync()
    # the last replay used kbuf/dbuf of iteration 5 again: apply it to the oracle too
    o.lookup(keys, B, train=True)
    o.backward_update(d, p)
    assert _bt_used(ctx, g) == 0
    for t, c in enumerate(caps):
        assert close(g.export(t, 0, c)[0].cpu().numpy(), o.export(t, 0, c)[0]), f"table {t}"


@pytest.mark.parametrize("multi", [False, True])
def test_f16_inference_table_matches_oracle(ctx, multi):
    """binary16 table rows: bulk load (init values and given rows,
    rounded to nearest even), pooled inference lookups (sum / mean, absent keys -> default
    vector), export (exact widening) — bit-identical to the oracle; training calls on the
    inference table are DtypeMismatch; a row beyond binary16 range is F16Range."""
    rs = np.random.default_rng(31)
    caps, dim, slots = [3000, 500], 24, [0, 1, 1]
    g = EmbeddingTableGroup(ctx, caps, dim, slots, "sgd", 1 << 15, 1 << 15, 5, dtype="f16")
    o = O.OracleTable(caps, dim, slots, "sgd", 5, dtype="f16")
    pools = []
    for t, c in enumerate(caps):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        if t == 0:
            g.insert(t, t64(ks))
            o.insert(t, ks)
        else:  # given rows: a wide dynamic range (binary16 subnormals, ties, near 65504)
            rows = (rs.standard_normal((c, dim)) * np.exp2(rs.integers(-26, 15, (c, dim)))).astype(np.float32)
            g.insert(t, t64(ks), torch.from_numpy(rows).cuda())
            o.insert(t, ks, rows)
        pools.append(ks)
    dvec = rs.standard_normal(dim).astype(np.float32)
    g.set_default_vector(1, dvec)
    o.set_default(1, dvec)
    B = 700
    if multi:
        lens = rs.integers(0, 5, B * len(slots)).astype(np.uint32)
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
        keys = np.concatenate([np.where(rs.random(l) < 0.1, rs.integers(0, 2**63, l).astype(np.uint64),
                                        rs.choice(pools[slots[b % len(slots)]], l)) for b, l in enumerate(lens)]).astype(np.uint64)
        ot = torch.from_numpy(offs.view(np.int32)).cuda()
        for comb in ("sum", "mean"):
            out = g.lookup(t64(keys), B, offsets=ot, combiner=comb)
            ref = o.lookup(keys, B, offsets=offs, combiner=comb)
            assert np.array_equal(out.cpu().numpy(), ref), comb
    else:
        keys = np.stack([rs.choice(pools[s], B) for s in slots], 1).ravel()
        keys[::17] = rs.integers(0, 2**63, len(keys[::17])).astype(np.uint64)  # absent keys
        out = g.lookup(t64(keys), B)
        ref = o.lookup(keys, B)
        assert np.array_equal(out.cpu().numpy(), ref)
    for t, c in enumerate(caps):
        assert np.array_equal(g.export(t, 0, c)[0].cpu().numpy(), o.export(t, 0, c)[0])
    with pytest.raises(HpsError) as e:
        g.lookup(t64(pools[0][:3].repeat(3)), 3, train=True)
    assert e.value.code == 8  # DtypeMismatch
    bad = np.zeros((2, dim), np.float32)
    bad[1, 3] = 1e6
    with pytest.raises(HpsError) as e:
        g.insert(0, t64(rs.integers(0, 2**63, 2).astype(np.uint64)), torch.from_numpy(bad).cuda())
        ctx.sync()
    assert e.value.code == 9  # F16Range


def test_adam_graph_step_matches_eager(ctx):
    """Adam inside a captured CUDA graph: the per-step bias-corrected lr_t reaches the
    kernels through hps_opt_params.lr_t_device (a device scalar written before each replay),
    so replayed steps (device keys, and pinned host keys through run_host_async) produce
    bitwise the same table as eager steps (host lr_t, checked against the oracle above)."""
    from paper_2210_08803_b200 import workload as W
    from paper_2210_08803_b200.sharded import TrainStep, build_tables
    cfg = W.config5(batch_per_gpu=256, capacity=60_000)
    cfg.dim, cfg.keyspace = 64, 2_000_000
    gen = W.BatchGen(cfg)
    rs = np.random.default_rng(5)
    batches = [gen.batch(s)[:2] for s in range(1, 4)]
    douts = [torch.from_numpy((rs.standard_normal((cfg.batch * cfg.n_slots, cfg.dim)) * 0.1).astype(np.float32)).cuda()
             for _ in range(2)]
    res = []
    for mode in ("eager", "graph", "host"):
        tab = build_tables(ctx, cfg)
        ts = TrainStep(ctx, tab, cfg, use_graph=mode != "eager")
        staged = [ts.stage_host(k, None) if mode == "host" else ts.stage_batch(k, None) for k, _ in batches]
        for step in range(1, 9):
            b, d = staged[step % 3], douts[step % 2]
            if mode == "host":
                ts.run_host_async(b, d, step, step % 2)
                ts.read_host_result(step % 2)
            else:
                ts.run(b, d, step=step)
        ctx.sync()
        n = tab.size(0)
        res.append([x.cpu().numpy() for x in tab.export(0, 0, n)])
    for mode, other in zip(("graph", "host"), res[1:]):
        for k, (a, b) in enumerate(zip(res[0], other)):
            np.testing.assert_array_equal(a, b, err_msg=f"{mode} vs eager, state {k}")


def test_multi_hot_pipelined_host_steps_match_eager(ctx):
    """Multi-hot (config-3 shape, small tables): the pipelined end-to-end path (keys AND bag
    offsets H2D on a copy stream into device slots, then one graph per slot) produces
    bitwise the table of eager device steps."""
    from paper_2210_08803_b200 import workload as W
    from paper_2210_08803_b200.sharded import TrainStep, build_tables
    cfg = W.config3(batch_per_gpu=128)
    cfg.cards = [4000 + 37 * t for t in range(26)]
    gen = W.BatchGen(cfg)
    rs = np.random.default_rng(9)
    batches = [gen.batch(s)[:2] for s in range(1, 4)]
    douts = [torch.from_numpy((rs.standard_normal((cfg.batch * cfg.n_slots, cfg.dim)) * 0.1).astype(np.float32)).cuda()
             for _ in range(2)]
    res = []
    for mode in ("eager", "host"):
        tab = build_tables(ctx, cfg)
        ts = TrainStep(ctx, tab, cfg, use_graph=mode != "eager")
        staged = [ts.stage_host(k, o) if mode == "host" else ts.stage_batch(k, o) for k, o in batches]
        for step in range(1, 8):
            b, d = staged[step % 3], douts[step % 2]
            if mode == "host":
                ts.run_host_async(b, d, step, step % 2)
                ts.read_host_result(step % 2)
            else:
                ts.run(b, d, step=step)
        ctx.sync()
        res.append([np.concatenate([x.cpu().numpy().ravel() for x in tab.export(t, 0, c) if x is not None])
                    for t, c in enumerate(cfg.cards)])
    for a, b in zip(res[0], res[1]):
        np.testing.assert_array_equal(a, b)
