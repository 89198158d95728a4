"""Oracle parity for the kernel instantiations the bench actually times.

* the bulk-copy backward (k_reduce_short<OPT,32,VPL,TMA=true>, dim 128..256) and the TMA
  one-hot pooling, at dim 128 and 256, for SGD / AdaGrad / Adam x sum / mean, with segment
  lengths 1..32 (short path), 33..4096 and > 4096 (long path: chunked tree) and absent keys;
* a dim sweep over every lookup / backward dispatch width;
* per-config sub-slices built by workload.BatchGen exactly as bench.py builds them
  (config 2: the 26 Criteo tables capped at 1M rows, dim 128, batch 6,912; config 3: dim 64
  Zipf(1.1) multi-hot, mean, AdaGrad; config 5: dim 128 Adam insert-on-miss), every one
  checked against the CPU oracle — never GPU-vs-GPU.

Everything is bitwise (DESIGN.md §4 fixes the operation order on both sides); `close()`
also states the north-star tolerance, 1e-5 relative, for fp32 values."""
import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import EmbeddingTableGroup, opt_params
from paper_2210_08803_b200 import workload as W
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu
RTOL = 1e-5


def t64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def t32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def close(gpu, cpu, what=""):
    gpu = np.asarray(gpu, dtype=np.float32)
    cpu = np.asarray(cpu, dtype=np.float32)
    tol = RTOL * np.maximum(np.abs(cpu), 1e-6)
    bad = np.abs(gpu - cpu) > tol
    assert not bad.any(), f"{what}: {bad.sum()} elements out of 1e-5 rel; max abs err {np.abs(gpu - cpu).max()}"
    assert np.array_equal(gpu.view(np.uint32), cpu.view(np.uint32)), f"{what}: in tolerance but not bitwise"


def make_pair(ctx, caps, dim, slots, opt, seed=7, a0=0.0, max_keys=1 << 17, max_bags=1 << 17):
    g = EmbeddingTableGroup(ctx, caps, dim, slots, opt, max_keys, max_bags, seed, a0)
    o = O.OracleTable(caps, dim, slots, opt, seed, a0)
    return g, o


def load_tables(g, o, caps, rs):
    pools = []
    for t, c in enumerate(caps):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks), return_rows=False)
        st, _ = o.insert(t, ks)
        assert st == 0
        pools.append(ks)
    return pools


def compare_tables(g, o, caps, chunk=1 << 18):
    for t, c in enumerate(caps):
        for b in range(0, c, chunk):
            n = min(chunk, c - b)
            gw = [x.cpu().numpy() if x is not None else None for x in g.export(t, b, n)]
            ow = o.export(t, b, n)
            for k, (x, y) in enumerate(zip(gw, ow)):
                if y is not None:
                    close(x, y, f"table {t} rows {b}..{b + n} state {k}")


def skewed_multiset(pool, rs, n_total, absent):
    """n_total occurrences over `pool` whose per-key counts cover every backward path:
    > 4096, exactly 4097 / 4096, 33..1000, 2..32 and singletons, plus `absent` keys."""
    parts = [np.repeat(pool[0], 5000), np.repeat(pool[1], 4097), np.repeat(pool[2], 4096), np.repeat(pool[3], 1000),
             np.repeat(pool[4:9], 33), np.concatenate([np.repeat(pool[9 + L], L) for L in range(2, 33)])]
    used = sum(len(p) for p in parts)
    single = n_total - used - absent
    assert single > 0
    parts.append(pool[100:100 + single])
    parts.append(np.uint64(1) + (rs.integers(0, 2**62, absent).astype(np.uint64) << np.uint64(1)))  # not in pool (odd)
    keys = np.concatenate(parts).astype(np.uint64)
    return keys[rs.permutation(len(keys))]


def run_steps(ctx, g, o, keys, n_samples, offsets, combiner, opt, rs, steps=3, lr=0.01, **kw):
    ot = None if offsets is None else t32(offsets)
    for step in range(1, steps + 1):
        out = g.lookup(t64(keys), n_samples, offsets=ot, combiner=combiner, train=True)
        ref = o.lookup(keys, n_samples, offsets=offsets, combiner=combiner, train=True)
        close(out.cpu().numpy(), ref, f"pooled step {step}")
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(opt, lr, step=step, **kw)
        g.backward_update(torch.from_numpy(dout).cuda(), lr, params=p)
        o.backward_update(dout, p)
        ctx.sync()
        np.testing.assert_array_equal(g.last_unique().cpu().numpy().view(np.uint32), o.last_unique())


@pytest.mark.parametrize("dim", [128, 256])
@pytest.mark.parametrize("opt", ["sgd", "adagrad", "adam"])
@pytest.mark.parametrize("combiner", ["sum", "mean"])
def test_bulk_copy_backward_parity(ctx, dim, opt, combiner):
    """sum: one-hot batch (the config-2/5 TMA pooling + bulk-copy short reduce); mean:
    multi-hot CSR batch (empty bags too) through the same backward with 1/len scaling."""
    rs = np.random.default_rng(dim * 7 + len(opt) + len(combiner))
    caps, slots = [40000, 40], [0, 1, 0, 0]
    g, o = make_pair(ctx, caps, dim, slots, opt, a0=0.1 if opt == "adagrad" else 0.0)
    pools = load_tables(g, o, caps, rs)
    default = rs.standard_normal(dim).astype(np.float32)
    g.set_default_vector(0, default)
    o.set_default(0, default)
    if combiner == "sum":
        B = 6000
        k0 = skewed_multiset(pools[0], rs, 3 * B, 120).reshape(B, 3)
        k1 = rs.choice(pools[1], B)  # 40 keys x ~150 occurrences each: long segments
        keys = np.stack([k0[:, 0], k1, k0[:, 1], k0[:, 2]], 1).ravel()
        offsets = None
    else:
        B = 1500
        lens = rs.integers(0, 9, B * 4).astype(np.int64)  # includes empty bags
        lens[7] = 40
        offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
        slot_of = np.repeat(np.arange(B * 4) % 4, lens)
        n0 = int((slot_of != 1).sum())
        keys = np.empty(len(slot_of), np.uint64)
        keys[slot_of != 1] = skewed_multiset(pools[0], rs, n0, 60)
        keys[slot_of == 1] = rs.choice(pools[1], int((slot_of == 1).sum()))
    kw = {"eps": 1e-7} if opt == "adagrad" else {}
    run_steps(ctx, g, o, keys, B, offsets, combiner, opt, rs, **kw)
    compare_tables(g, o, caps)


DIMS = [4, 8, 12, 20, 32, 48, 64, 96, 124, 128, 160, 192, 252, 256, 260, 384, 512, 1024]


@pytest.mark.parametrize("dim", DIMS)
def test_dim_sweep_parity(ctx, dim):
    """Every lookup/backward dispatch width (lanes per row, float4s per lane, TMA or register
    staging): one-hot SGD and multi-hot mean Adam, a few hundred keys with repeats."""
    rs = np.random.default_rng(dim)
    caps = [3000, 7]
    for opt, multi in (("sgd", False), ("adam", True)):
        g, o = make_pair(ctx, caps, dim, [0, 1, 0], opt, max_keys=1 << 14, max_bags=1 << 13)
        pools = load_tables(g, o, caps, rs)
        B = 400
        if multi:
            lens = rs.integers(0, 6, B * 3)
            offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
            keys = np.concatenate([rs.choice(pools[[0, 1, 0][b % 3]][:300], l) for b, l in enumerate(lens)])
            keys = keys.astype(np.uint64)
        else:
            offsets = None
            keys = np.stack([rs.choice(pools[0][:500], B), rs.choice(pools[1], B), rs.choice(pools[0], B)], 1).ravel()
        run_steps(ctx, g, o, keys, B, offsets, "mean" if multi else "sum", opt, rs, steps=2)
        compare_tables(g, o, caps)


def _config_tables(ctx, cfg, cap_rows, opt, a0=0.0, max_keys=None):
    cards = [min(c, cap_rows) for c in cfg.cards]
    mk = max_keys or (cfg.batch * cfg.n_slots * (2 * cfg.hot))
    g = EmbeddingTableGroup(ctx, cards, cfg.dim, cfg.slots(), opt, mk, cfg.batch * cfg.n_slots, cfg.seed, a0)
    o = O.OracleTable(cards, cfg.dim, cfg.slots(), opt, cfg.seed, a0)
    for t, c in enumerate(cards):
        # exactly as bench.py / sharded.build_tables: row i of table t holds table_key(t, i)
        g.insert(t, ctx.gen_keys(W.table_seed(cfg.seed, t), 0, c), return_rows=False)
        st, _ = o.insert(t, W.table_keys(cfg.seed, t, np.arange(c)))
        assert st == 0
    return cards, g, o


@pytest.mark.slow
def test_config2_subslice_parity(ctx):
    """BASELINE config 2 at full per-GPU batch (6,912 x 26 one-hot, dim 128, SGD) over the
    26 Criteo cardinalities capped at 1M rows (7.1M rows, 3.6 GB), BatchGen batches."""
    cfg = W.config2(6912)
    cards, g, o = _config_tables(ctx, cfg, 1_000_000, "sgd")
    gen = W.BatchGen(cfg, cards)
    rs = np.random.default_rng(2)
    for step in range(1, 4):
        keys, offs, idx, tab = gen.batch(step)
        assert offs is None
        run_steps(ctx, g, o, keys, cfg.batch, None, "sum", "sgd", rs, steps=1, lr=cfg.lr)
    # every row actually touched, and a sample of the rest
    compare_tables(g, o, cards)


@pytest.mark.slow
def test_config3_subslice_parity(ctx):
    """BASELINE config 3 shape: 26 slots, 1..19 hots (mean 10), Zipf(1.1) per table, dim 64,
    mean, AdaGrad (eps 1e-7), batch 1,024 from BatchGen, cardinalities capped at 200k."""
    cfg = W.config3(1024)
    cards, g, o = _config_tables(ctx, cfg, 200_000, "adagrad")
    gen = W.BatchGen(cfg, cards)
    rs = np.random.default_rng(3)
    for step in range(1, 4):
        keys, offs, _, _ = gen.batch(step)
        run_steps(ctx, g, o, keys, cfg.batch, offs, "mean", "adagrad", rs, steps=1, lr=cfg.lr, eps=cfg.eps)
    compare_tables(g, o, cards)


@pytest.mark.slow
def test_config5_subslice_parity(ctx):
    """BASELINE config 5 shape: one hashed table over a 1e9-key power-law space, dim 128,
    Adam, rows materialised on first touch (HPS_LOOKUP_INSERT), batch 2,048 x 26, 5 steps."""
    cfg = W.config5(batch_per_gpu=2048, capacity=400_000)
    gen = W.BatchGen(cfg)
    g = EmbeddingTableGroup(ctx, cfg.cards, cfg.dim, cfg.slots(), "adam", cfg.batch * 26, cfg.batch * 26, cfg.seed)
    o = O.OracleTable(cfg.cards, cfg.dim, cfg.slots(), "adam", cfg.seed)
    rs = np.random.default_rng(5)
    for step in range(1, 6):
        keys, _, _, _ = gen.batch(step)
        out = g.lookup(t64(keys), cfg.batch, train=True, insert_missing=True)
        st, _ = o.insert(0, keys)
        assert st == 0
        ref = o.lookup(keys, cfg.batch, train=True)
        close(out.cpu().numpy(), ref, f"cfg5 pooled step {step}")
        dout = (rs.standard_normal(ref.shape) * 0.1).astype(np.float32)
        p = opt_params("adam", cfg.lr, step=step)
        g.backward_update(torch.from_numpy(dout).cuda(), cfg.lr, params=p)
        o.backward_update(dout, p)
        ctx.sync()
        np.testing.assert_array_equal(g.last_unique().cpu().numpy().view(np.uint32), o.last_unique())
    n = g.size(0)
    assert n == o.size(0) and n > cfg.batch * 10
    np.testing.assert_array_equal(g.row_keys(0, 0, n).cpu().numpy().view(np.uint64), o.row_keys(0, 0, n))
    compare_tables(g, o, [n])


def test_oversized_device_offsets_refused(ctx):
    """A multi-hot training batch whose DEVICE offsets hold more keys than max_batch_keys is
    refused on the device (latched InvalidArgument, empty record: no out-of-bounds write),
    and the table is usable — and oracle-exact — afterwards."""
    from paper_2210_08803_b200 import HpsError
    rs = np.random.default_rng(44)
    g, o = make_pair(ctx, [500], 16, [0], "sgd", max_keys=1000, max_bags=400)
    pool = load_tables(g, o, [500], rs)[0]
    lens = np.full(300, 5, np.int64)  # 1,500 keys > 1,000
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    keys = rs.choice(pool, 1500)
    g.lookup(t64(keys), 300, offsets=t32(offs), train=True)
    with pytest.raises(HpsError) as e:
        ctx.sync()
    assert e.value.code == 1
    lens = rs.integers(0, 6, 300)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    keys = rs.choice(pool, int(offs[-1]))
    run_steps(ctx, g, o, keys, 300, offs, "sum", "sgd", rs, steps=2)
    compare_tables(g, o, [500])


ODD_DIMS = [1, 2, 3, 5, 7, 13, 30, 127, 129, 255, 1023]


@pytest.mark.parametrize("dim", ODD_DIMS)
def test_unpadded_dims_match_oracle(ctx, dim):
    """Any dim in 1..1024 (hps::validate_dim accepts 1..4096, proj/src/core/types.cpp:57-60):
    rows are stored at round_up(dim, 4); the caller's buffers keep `dim`. One-hot SGD with
    given initial rows, multi-hot mean Adam with init_value rows, default vectors, export."""
    rs = np.random.default_rng(dim + 1000)
    caps = [800, 5]
    for opt, multi in (("sgd", False), ("adam", True)):
        g, o = make_pair(ctx, caps, dim, [0, 1, 0], opt, max_keys=1 << 13, max_bags=1 << 12)
        pools = []
        for t, c in enumerate(caps):
            ks = rs.integers(0, 2**63, c).astype(np.uint64)
            if opt == "sgd":  # given rows (the caller's stride is dim)
                rows = rs.standard_normal((c, dim)).astype(np.float32)
                g.insert(t, t64(ks), rows=torch.from_numpy(rows).cuda(), return_rows=False)
                st, _ = o.insert(t, ks, rows)
            else:
                g.insert(t, t64(ks), return_rows=False)
                st, _ = o.insert(t, ks)
            assert st == 0
            pools.append(ks)
        dflt = rs.standard_normal(dim).astype(np.float32)
        g.set_default_vector(1, dflt)
        o.set_default(1, dflt)
        B = 300
        if multi:
            lens = rs.integers(0, 6, B * 3)
            offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
            keys = np.concatenate([rs.choice(pools[[0, 1, 0][b % 3]][:200], l) for b, l in enumerate(lens)])
            keys = keys.astype(np.uint64)
            keys[::17] ^= np.uint64(0x5555)  # some absent keys (default vector)
        else:
            offsets = None
            keys = np.stack([rs.choice(pools[0][:300], B), rs.choice(pools[1], B), rs.choice(pools[0], B)], 1).ravel()
        run_steps(ctx, g, o, keys, B, offsets, "mean" if multi else "sum", opt, rs, steps=2)
        compare_tables(g, o, caps)


@pytest.mark.parametrize("dim", [1, 3, 6, 13, 4096])
def test_cache_unpadded_dims(ctx, dim):
    """Cache rows of any dim in 1..4096: insert / query / refresh round trip bitwise, stats as
    the oracle's."""
    from paper_2210_08803_b200 import HotCache
    rs = np.random.default_rng(dim)
    cap = 256
    c = HotCache(ctx, cap, dim, 8, max_batch=1024)
    oc = O.OracleCache(cap, dim, 8)
    keys = rs.integers(0, 2**63, 300).astype(np.uint64)
    vecs = rs.standard_normal((300, dim)).astype(np.float32)
    vers = np.arange(1, 301, dtype=np.uint64)
    c.insert(t64(keys), torch.from_numpy(vecs).cuda(), t64(vers))
    oc.insert(keys, vecs, vers)
    q = np.concatenate([keys[:150], rs.integers(0, 2**63, 50).astype(np.uint64)])
    fi, fv, mi = c.query(t64(q))
    ofi, ofv, omi = oc.query(q)
    ctx.sync()
    np.testing.assert_array_equal(fi.cpu().numpy(), ofi)
    np.testing.assert_array_equal(mi.cpu().numpy(), omi)
    assert np.array_equal(fv.cpu().numpy().view(np.uint32), np.asarray(ofv, np.float32).view(np.uint32))
    new = (vecs[:100] * 2).astype(np.float32)
    c.refresh(t64(keys[:100]), torch.from_numpy(new).cuda(), t64(vers[:100] + np.uint64(1000)))
    oc.refresh(keys[:100], new, vers[:100] + np.uint64(1000))
    fi, fv, mi = c.query(t64(keys[:100]))
    ofi, ofv, omi = oc.query(keys[:100])
    ctx.sync()
    assert np.array_equal(fv.cpu().numpy().view(np.uint32), np.asarray(ofv, np.float32).view(np.uint32))
    assert c.stats() == oc.stats()
