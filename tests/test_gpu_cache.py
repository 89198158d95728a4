"""GPU parity for the HPS cache (K6-K8) against the CPU restatement of SPEC.md:112-190.
Hit/miss sets, found order, vectors, stats and the per-set LFU metadata must be identical."""
import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import HotCache, HpsError
from paper_2210_08803_b200 import workload as W
from tests import oracle_lib as O

pytestmark = pytest.mark.gpu


def t64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def tf(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def pair(ctx, capacity, dim, ways=8, aging=0, max_batch=4096):
    return HotCache(ctx, capacity, dim, ways, aging, max_batch), O.OracleCache(capacity, dim, ways, aging)


def q_both(g, o, keys):
    gi, gv, gm = g.query(t64(keys))
    oi, ov, om = o.query(keys)
    np.testing.assert_array_equal(gi.cpu().numpy().view(np.uint32), oi)
    np.testing.assert_array_equal(gm.cpu().numpy().view(np.uint32), om)
    np.testing.assert_array_equal(gv.cpu().numpy().view(np.uint32), ov.view(np.uint32))
    return oi, om


def ins_both(ctx, g, o, keys, vecs, vers):
    n = g.insert(t64(keys), tf(vecs), t64(vers))
    on, st = o.insert(keys, vecs, vers)
    try:
        ctx.sync()
        gst = 0
    except HpsError as e:
        gst = e.code
    assert gst == st
    assert int(n.item()) == on
    return on


def assert_same_state(g, o, cap):
    """White-box: every way of every set identical — key, version, freq, last_touch, the
    row — and every set's aging counter (hps_gpu_cache_debug_export vs the oracle)."""
    gs, os_ = g.export_state(), o.export(cap)
    for name, x, y in zip(["keys", "versions", "freq", "last_touch", "set_access", "vecs"], gs, os_):
        if name in ("keys", "versions", "last_touch", "vecs"):  # an empty way's payload is unspecified
            live = os_[2] != 0
            x, y = x[live], y[live]
        if name == "vecs":
            x, y = x.view(np.uint32), y.view(np.uint32)
        np.testing.assert_array_equal(x, y, err_msg=name)


def test_spec_examples(ctx):
    g, o = pair(ctx, 64, 4)
    fi, fv, mi = g.query(t64(np.array([1, 2, 3], dtype=np.uint64)))  # empty cache: all missing
    assert len(fi) == 0 and mi.cpu().tolist() == [0, 1, 2]
    fi, fv, mi = g.query(t64(np.zeros(0, dtype=np.uint64)))
    assert len(fi) == 0 and len(mi) == 0
    v = np.arange(4, dtype=np.float32)[None]
    assert int(g.insert(t64(np.array([7], dtype=np.uint64)), tf(v), t64(np.array([3], dtype=np.uint64))).item()) == 1
    fi, fv, mi = g.query(t64(np.array([7], dtype=np.uint64)))
    assert fi.cpu().tolist() == [0] and fv.cpu().numpy().tolist() == v.tolist()
    # refresh: newer replaces, older is ignored, non-resident never inserts
    assert int(g.refresh(t64(np.array([7], dtype=np.uint64)), tf(v + 1), t64(np.array([5], dtype=np.uint64))).item()) == 1
    assert int(g.refresh(t64(np.array([7], dtype=np.uint64)), tf(v + 9), t64(np.array([4], dtype=np.uint64))).item()) == 0
    assert int(g.refresh(t64(np.array([8], dtype=np.uint64)), tf(v), t64(np.array([9], dtype=np.uint64))).item()) == 0
    fi, fv, mi = g.query(t64(np.array([7, 8], dtype=np.uint64)))
    assert fv.cpu().numpy().tolist() == (v + 1).tolist() and mi.cpu().tolist() == [1]
    s = g.stats()
    assert s["hits"] + s["misses"] == s["queries"] == 6
    assert g.size() == 1
    g.reset_stats()
    assert all(v == 0 for v in g.stats().values())


def test_eviction_victim_spec(ctx):
    # fill one set (8 colliding keys), touch them, insert one more: LFU/last-touch victim
    cap, ways, dim = 64, 8, 4
    g, o = pair(ctx, cap, dim, ways)
    sets = cap // ways
    from tests.oracle_lib import lib
    L = lib()
    coll = [k for k in range(20000) if L.orc_key_hash(k) % sets == 3][:9]
    keys = np.array(coll[:8], dtype=np.uint64)
    vecs = np.arange(8 * dim, dtype=np.float32).reshape(8, dim)
    ins_both(ctx, g, o, keys, vecs, np.ones(8, dtype=np.uint64))
    q_both(g, o, keys[[0, 1, 2, 3, 4, 5, 6, 0, 1, 2]])
    assert ins_both(ctx, g, o, np.array([coll[8]], np.uint64), np.full((1, dim), 9, np.float32),
                    np.ones(1, np.uint64)) == 1
    assert g.stats() == o.stats()
    assert g.stats()["evictions"] == 1
    q_both(g, o, np.array(coll, dtype=np.uint64))  # key coll[7] (freq 1, oldest) was evicted


def test_non_finite_entry_skipped(ctx):
    g, o = pair(ctx, 64, 4)
    vecs = np.ones((3, 4), dtype=np.float32)
    vecs[1, 2] = np.inf
    ins_both(ctx, g, o, np.array([1, 2, 3], np.uint64), vecs, np.ones(3, np.uint64))
    q_both(g, o, np.array([1, 2, 3], np.uint64))
    assert g.stats() == o.stats()


@pytest.mark.parametrize("small_sort", [True, False])
@pytest.mark.parametrize("cap,ways,aging", [(256, 8, 0), (96, 4, 40), (512, 8, 700), (32, 1, 0), (1024, 32, 0)])
def test_randomized_sequences_match_oracle(ctx, cap, ways, aging, small_sort, monkeypatch):
    """small_sort=False: batches <= 2048 keys also take the multi-kernel set sort (histogram +
    onesweep passes + segment scan) instead of the single-CTA sort + segment kernel."""
    dim = 8
    if not small_sort:
        monkeypatch.setenv("HPS_GPU_NO_SMALL_SORT", "1")  # read when the cache is created
    g, o = pair(ctx, cap, dim, ways, aging)
    rs = np.random.default_rng(cap + ways + aging)
    zipf = W.Zipf(3 * cap, 1.05)
    version = 1
    for rnd in range(25):
        keys = zipf.ranks(W.rng(rnd * 7 + 1, np.arange(int(rs.integers(1, 700)), dtype=np.uint64))).astype(np.uint64)
        keys = W.mix64(keys)  # spread ranks over the key space
        oi, om = q_both(g, o, keys)
        miss = keys[om]
        if len(miss):
            vecs = rs.standard_normal((len(miss), dim)).astype(np.float32)
            vers = (version + rs.integers(0, 3, len(miss))).astype(np.uint64)
            ins_both(ctx, g, o, miss, vecs, vers)
        if rnd % 3 == 0:
            rk = keys[: min(50, len(keys))]
            vecs = rs.standard_normal((len(rk), dim)).astype(np.float32)
            vers = (version + rs.integers(-1, 3, len(rk))).clip(0).astype(np.uint64)
            gn = g.refresh(t64(rk), tf(vecs), t64(vers))
            on, _ = o.refresh(rk, vecs, vers)
            assert int(gn.item()) == on
        version += 2
        assert g.stats() == o.stats(), rnd
    assert g.size() == o.size()
    assert_same_state(g, o, cap)
    q_both(g, o, W.mix64(np.arange(3 * cap, dtype=np.uint64)))


def test_zipf_hit_rate_bound(ctx):
    """Zipf(1.2), 100k keys, capacity 10k: hit rate >= 0.9 * top-10k mass."""
    n, cap = 100_000, 10_000
    g = HotCache(ctx, cap, 8, 8, 0, 1 << 15)
    z = W.Zipf(n, 1.2)
    M = float(z.cdf[cap - 1] / z.H)
    vecs = torch.ones(1 << 15, 8, device="cuda")
    vers = torch.ones(1 << 15, dtype=torch.int64, device="cuda")
    def run(first, total):
        for b in range(first, first + total, 1 << 14):
            keys = W.mix64(z.ranks(W.rng(99, np.arange(b, b + (1 << 14), dtype=np.uint64))).astype(np.uint64))
            fv, fi, mi, cnt = g.query_async(t64(keys))
            nm = int(cnt[1].item())
            if nm:
                miss = t64(keys)[mi[:nm].long()]
                g.insert(miss, vecs[:nm], vers[:nm])
    run(0, 200_000)
    g.reset_stats()
    run(200_000, 200_000)
    s = g.stats()
    assert s["hits"] / s["queries"] >= 0.9 * M, (s, M)


def first_occurrence_unique(q):
    """Distinct keys in order of first occurrence and the inverse map."""
    _, first, inv_sorted = np.unique(q, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    return q[first[order]], rank[inv_sorted]


def oracle_read_through(ocache, truth, default, q, dim):
    """The orchestrator lookup restated on the oracle cache + a dict table: one probe per
    distinct key (first-occurrence order), distinct present misses inserted once (version 0
    = bulk load), rows expanded to input order, per-key source counts {L1, L2, L3, Default}."""
    u, inv = first_occurrence_unique(q)
    fi, fv, mi = ocache.query(u)
    rows = np.empty((len(u), dim), np.float32)
    src = np.empty(len(u), np.int64)
    rows[fi] = fv
    src[fi] = 0
    miss = u[mi]
    present = np.array([int(k) in truth for k in miss], dtype=bool)
    mrows = np.stack([truth.get(int(k), default) for k in miss]) if len(mi) else np.zeros((0, dim), np.float32)
    rows[mi] = mrows
    src[mi] = np.where(present, 1, 3)
    if present.any():
        ocache.insert(miss[present], mrows[present], np.zeros(int(present.sum()), np.uint64))
    return rows[inv], np.bincount(src[inv], minlength=4), len(u)


@pytest.mark.parametrize("graphed,cap,group", [(False, 512, None), (True, 512, None), (False, 4096, None),
                                               (False, 4096, "1"), (True, 4096, "1")])
def test_read_through_matches_oracle(ctx, graphed, cap, group, monkeypatch):
    """Orchestrator lookup (cache + backing table): rows in input order, duplicate keys served
    from one probe per distinct key (so cache stats count distinct keys), distinct misses
    migrated once (absent keys never cached), source counts per input key — bit-exact with
    the oracle cache + a dict table. Batches span the one-CTA dedup (<= 2,048 keys) and the
    claim-table dedup. graphed: lookup_graphed (one CUDA graph per batch size). The migration
    groups its inserts by set from the query's sorted list (cache_insert_after_query): cap 512
    (64 sets) sorts in one radix pass, cap 4096 (512 sets) in two, which leaves the query's
    list in the buffers the insert's entry prep would otherwise overwrite. group="1": the
    query groups its distinct keys by set with counters instead of the radix sort (the
    default only when sets >= 8 x max_batch; forced here, so ranges hold several keys)."""
    if group is not None:
        monkeypatch.setenv("HPS_GPU_COUNT_GROUP", group)
    from paper_2210_08803_b200 import EmbeddingTableGroup
    from paper_2210_08803_b200.api import CachedLookup
    dim, n_keys = 8, 5000
    rs = np.random.default_rng(17)
    keys_all = W.mix64(np.arange(n_keys, dtype=np.uint64))
    table = EmbeddingTableGroup(ctx, [n_keys], dim, [0], "sgd", 8192, 8192, 3)
    table.insert(0, t64(keys_all))
    default = np.full(dim, 0.5, np.float32)
    table.set_default_vector(0, default)
    rows = table.export(0, 0, n_keys)[0].cpu().numpy()
    truth = {int(k): rows[i] for i, k in enumerate(keys_all)}
    cache = HotCache(ctx, cap, dim, 8, 0, 8192)
    rt = CachedLookup(cache, table)
    ocache = O.OracleCache(cap, dim, 8, 0)
    z = W.Zipf(n_keys + 200, 1.1)
    for rnd in range(24):
        m = int(rs.integers(1, 7000)) if not graphed else [1, 37, 2048, 5000][rnd % 4]
        ranks = z.ranks(W.rng(rnd, np.arange(m, dtype=np.uint64)))
        q = W.mix64(ranks.astype(np.uint64))  # ranks >= n_keys are absent from the table
        got = (rt.lookup_graphed(t64(q)) if graphed else rt.lookup(t64(q))).cpu().numpy()
        want, want_src, n_u = oracle_read_through(ocache, truth, default, q, dim)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
        assert rt.source_counts.tolist() == want_src.tolist(), rnd
        assert int(rt.n_unique.item()) == n_u
        assert cache.stats() == ocache.stats(), rnd
    assert cache.size() == ocache.size()
    assert_same_state(cache, ocache, cap)


@pytest.mark.parametrize("f16", [False, True])
def test_apply_update_frame_matches_oracle_refresh(ctx, f16):
    """UpdateBatch frame -> host validation -> one H2D of the entry bytes -> device decode
    -> K8 refresh at version = seq, against the oracle cache's
    refresh of the same (key, vector, version) entries."""
    from paper_2210_08803_b200 import updates as U
    rs = np.random.default_rng(41)
    dim = 32
    g, o = pair(ctx, 512, dim, ways=4)
    keys = np.unique(rs.integers(0, 2**63 - 1, 400, dtype=np.int64)).astype(np.uint64)[:300]
    vers = rs.integers(1, 6, len(keys)).astype(np.uint64)
    ins_both(ctx, g, o, keys, rs.standard_normal((len(keys), dim)).astype(np.float32), vers)
    # frame: half resident keys (mixed older/newer versions than seq 4) + non-resident keys
    fk = np.concatenate([keys[::2], np.arange(10**6, 10**6 + 50, dtype=np.uint64)])
    rs.shuffle(fk)
    vals = rs.standard_normal((len(fk), dim)).astype(np.float32)
    if f16:
        bits = vals.astype(np.float16).view(np.uint16)
        frame = U.encode_update_batch("emb", 4, fk, bits)
        widened = bits.view(np.float16).astype(np.float32)  # exact widening
    else:
        frame = U.encode_update_batch("emb", 4, fk, vals)
        widened = vals
    replaced = g.apply_update(frame)
    o_replaced, st = o.refresh(fk, widened, np.full(len(fk), 4, np.uint64))
    assert st == 0 and replaced == o_replaced and replaced > 0
    q_both(g, o, np.concatenate([keys, fk]))
    assert g.stats() == o.stats()


def test_apply_update_rejects_malformed_and_dim_mismatch(ctx):
    from paper_2210_08803_b200 import updates as U
    g, _ = pair(ctx, 64, 8)
    frame = U.encode_update_batch("emb", 1, np.array([1, 2], np.uint64), np.ones((2, 8), np.float32))
    with pytest.raises(HpsError) as e:
        g.apply_update(frame[:-1])
    assert e.value.code == 4
    with pytest.raises(HpsError) as e:
        g.apply_update(U.encode_update_batch("emb", 1, np.array([1], np.uint64), np.ones((1, 4), np.float32)))
    assert e.value.code == 7


def pair16(ctx, capacity, dim, ways=8, aging=0, max_batch=4096):
    return (HotCache(ctx, capacity, dim, ways, aging, max_batch, dtype="f16"),
            O.OracleCache(capacity, dim, ways, aging, dtype="f16"))


@pytest.mark.parametrize("cap,ways,aging", [(256, 8, 0), (96, 4, 40), (1024, 32, 0)])
def test_f16_storage_sequences_match_oracle(ctx, cap, ways, aging):
    """binary16 cache rows: the same randomized
    query/insert/refresh sequences; found vectors are the exact widening of the RNE-rounded
    inserted values, bit-identical to the oracle (whose binary16 is pinned to the reference)."""
    dim = 12
    g, o = pair16(ctx, cap, dim, ways, aging)
    rs = np.random.default_rng(cap * 3 + ways)
    zipf = W.Zipf(3 * cap, 1.05)
    version = 1
    for rnd in range(15):
        keys = W.mix64(zipf.ranks(W.rng(rnd * 5 + 3, np.arange(int(rs.integers(1, 500)), dtype=np.uint64))).astype(np.uint64))
        oi, om = q_both(g, o, keys)
        miss = keys[om]
        if len(miss):
            # wide dynamic range: subnormal binary16, ties, values near the 65504 limit
            vecs = (rs.standard_normal((len(miss), dim)) * np.exp2(rs.integers(-26, 15, (len(miss), dim)))).astype(np.float32)
            vers = (version + rs.integers(0, 3, len(miss))).astype(np.uint64)
            ins_both(ctx, g, o, miss, vecs, vers)
        if rnd % 3 == 0:
            rk = keys[: min(40, len(keys))]
            vecs = rs.standard_normal((len(rk), dim)).astype(np.float32)
            vers = (version + rs.integers(-1, 3, len(rk))).clip(0).astype(np.uint64)
            gn = g.refresh(t64(rk), tf(vecs), t64(vers))
            on, _ = o.refresh(rk, vecs, vers)
            assert int(gn.item()) == on
        version += 2
        assert g.stats() == o.stats(), rnd
    assert_same_state(g, o, cap)
    q_both(g, o, W.mix64(np.arange(3 * cap, dtype=np.uint64)))


@pytest.mark.parametrize("aging_p", [0, 16])
def test_config4_shape_large_batches(ctx, aging_p):
    """BASELINE config 4 shape at reduced capacity: dim 128 rows, 8 ways, Zipf(1.05) query
    batches of 131,072 keys (Zipf-head sets see thousands of accesses per batch: the huge-set
    replay), misses inserted after each batch; found order, rows, missing order, stats and
    the whole set state identical to the oracle. aging_p: accesses per set-aging period
    (0 = the 10 x capacity default, i.e. 80; 16 exercises the per-32-access closed form)."""
    cap, dim, ways, n = 1 << 16, 128, 8, 131072
    sets = cap // ways
    g = HotCache(ctx, cap, dim, ways, aging_p * sets, n)
    o = O.OracleCache(cap, dim, ways, aging_p * sets)
    zipf = W.Zipf(2_000_000, 1.05)
    rs = np.random.default_rng(aging_p)
    for rnd in range(4):
        keys = W.mix64(zipf.ranks(W.rng(1000 + rnd, np.arange(n, dtype=np.uint64))).astype(np.uint64))
        oi, om = q_both(g, o, keys)
        miss = keys[om]
        vecs = rs.standard_normal((len(miss), dim)).astype(np.float32)
        ins_both(ctx, g, o, miss, vecs, np.full(len(miss), rnd + 1, np.uint64))
        assert g.stats() == o.stats(), rnd
    s = g.stats()
    assert s["hits"] > 0 and s["evictions"] > 0
    assert_same_state(g, o, cap)


def test_f16_storage_range_and_spec_examples(ctx):
    """{0, 1, -1} exact; 1/3 within 2^-11; 1e6 is a saturation error
    (F16Range, the entry skipped — rejected, not clamped). 65504 is the largest accepted."""
    g, o = pair16(ctx, 64, 4)
    vecs = np.array([[0.0, 1.0, -1.0, 1.0 / 3.0], [1e6, 0, 0, 0], [65504.0, -65519.0, 0, 0]], dtype=np.float32)
    ins_both(ctx, g, o, np.array([1, 2, 3], np.uint64), vecs, np.ones(3, np.uint64))
    fi, fv, mi = g.query(t64(np.array([1, 2, 3], np.uint64)))
    assert fi.cpu().tolist() == [0, 2] and mi.cpu().tolist() == [1]
    row = fv.cpu().numpy()[0]
    assert row[:3].tolist() == [0.0, 1.0, -1.0] and abs(row[3] - 1.0 / 3.0) <= 2.0 ** -11
    assert fv.cpu().numpy()[1][:2].tolist() == [65504.0, -65504.0]
    oi, ov, om = o.query(np.array([1, 2, 3], np.uint64))
    np.testing.assert_array_equal(fv.cpu().numpy().view(np.uint32), ov.view(np.uint32))
    assert g.stats() == o.stats()
