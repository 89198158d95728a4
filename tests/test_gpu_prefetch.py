"""Batch pipelining (hps_gpu_table_set_pipeline / _prefetch / _join_prefetch): the record +
dedup of batch i+1 run on their slot's stream while batch i pools and updates. Every case is
checked against the CPU oracle running the plain sequence (insert -> lookup -> backward per
batch), bitwise — pipelining must not change a single bit — in eager mode, from host keys,
with insert-on-miss (rows created in prefetch order = batch order), and replayed as the CUDA
graphs bench.py uses (one per slot parity, the prefetch joined inside each graph)."""
import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import EmbeddingTableGroup, HpsError, opt_params
from paper_2210_08803_b200 import workload as W
from tests import oracle_lib as O
from tests.test_gpu_paths import close, compare_tables, load_tables, make_pair, skewed_multiset, t32, t64

pytestmark = pytest.mark.gpu


def onehot_batches(pools, rs, B, n):
    out = []
    for _ in range(n):
        if 3 * B >= 16000:
            k0 = skewed_multiset(pools[0], rs, 3 * B, 50).reshape(B, 3)
        else:  # small batches: a few hot keys (long segments) over a uniform background
            k0 = np.where(rs.random(3 * B) < 0.3, rs.choice(pools[0][:8], 3 * B),
                          rs.choice(pools[0], 3 * B)).reshape(B, 3)
        k1 = rs.choice(pools[1], B)
        out.append(np.stack([k0[:, 0], k1, k0[:, 1], k0[:, 2]], 1).ravel().astype(np.uint64))
    return out


def multihot_batches(pools, rs, B, n, slots):
    out = []
    for _ in range(n):
        lens = rs.integers(0, 12, B * len(slots)).astype(np.int64)
        offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
        keys = np.concatenate([rs.choice(pools[slots[b % len(slots)]][:2000], l) for b, l in enumerate(lens)])
        out.append((keys.astype(np.uint64), offs))
    return out


def oracle_step(o, keys, B, offs, combiner, dout, p):
    ref = o.lookup(keys, B, offsets=offs, combiner=combiner, train=True)
    o.backward_update(dout, p)
    return ref


@pytest.mark.parametrize("dim,opt", [(128, "sgd"), (128, "adam"), (32, "adagrad")])
def test_prefetch_onehot_eager(ctx, dim, opt):
    rs = np.random.default_rng(dim + len(opt))
    caps, slots = [30000, 40], [0, 1, 0, 0]
    g, o = make_pair(ctx, caps, dim, slots, opt, a0=0.1 if opt == "adagrad" else 0.0)
    pools = load_tables(g, o, caps, rs)
    g.set_pipeline(2)
    B, S = 6000, 5
    batches = onehot_batches(pools, rs, B, S)
    dev = [t64(k) for k in batches]
    kw = {"eps": 1e-7} if opt == "adagrad" else {}
    g.prefetch(0, dev[0], B)
    for s in range(S):
        if s + 1 < S:
            g.prefetch((s + 1) % 2, dev[s + 1], B)  # concurrent with this batch's pooling + update
        out = g.lookup_prefetched(s % 2, B)
        dout = rs.standard_normal((B * 4, dim)).astype(np.float32)
        p = opt_params(opt, 0.01, step=s + 1, **kw)
        g.backward_update(torch.from_numpy(dout).cuda(), 0.01, params=p)
        ref = oracle_step(o, batches[s], B, None, "sum", dout, p)
        close(out.cpu().numpy(), ref, f"pooled step {s}")
        np.testing.assert_array_equal(g.last_unique().cpu().numpy().view(np.uint32), o.last_unique())
    g.join_prefetch()
    ctx.sync()
    compare_tables(g, o, caps)
    assert g.batch_table_used() == 0  # every slot's batch table is clean after its backward


def test_prefetch_multihot_host_keys(ctx):
    """Multi-hot mean AdaGrad, keys + offsets from pinned host memory (staged per slot)."""
    rs = np.random.default_rng(31)
    caps, slots, dim = [20000, 500, 3000], [0, 1, 2, 0], 64
    g, o = make_pair(ctx, caps, dim, slots, "adagrad", a0=0.1)
    pools = load_tables(g, o, caps, rs)
    g.set_pipeline(2)
    B, S = 700, 4
    batches = multihot_batches(pools, rs, B, S, slots)
    host = [(torch.from_numpy(k.view(np.int64)).pin_memory(), torch.from_numpy(f.view(np.int32)).pin_memory())
            for k, f in batches]
    g.prefetch(0, host[0][0], B, offsets=host[0][1], combiner="mean", keys_on_host=True)
    for s in range(S):
        if s + 1 < S:
            g.prefetch((s + 1) % 2, host[s + 1][0], B, offsets=host[s + 1][1], combiner="mean", keys_on_host=True)
        out = g.lookup_prefetched(s % 2, B, offsets=None, combiner="mean")
        dout = rs.standard_normal((B * 4, dim)).astype(np.float32)
        p = opt_params("adagrad", 0.01, eps=1e-7)
        g.backward_update(torch.from_numpy(dout).cuda(), 0.01, params=p)
        ref = oracle_step(o, batches[s][0], B, batches[s][1], "mean", dout, p)
        close(out.cpu().numpy(), ref, f"pooled step {s}")
    g.join_prefetch()
    ctx.sync()
    compare_tables(g, o, caps)


def test_prefetch_insert_on_miss_adam(ctx):
    """Config-5 shape: hashed table, rows materialise in the prefetch (batch order)."""
    cfg = W.config5(batch_per_gpu=1024, capacity=200_000)
    gen = W.BatchGen(cfg)
    g = EmbeddingTableGroup(ctx, cfg.cards, cfg.dim, cfg.slots(), "adam", cfg.batch * 26, cfg.batch * 26, cfg.seed)
    o = O.OracleTable(cfg.cards, cfg.dim, cfg.slots(), "adam", cfg.seed)
    g.set_pipeline(2)
    rs = np.random.default_rng(55)
    S = 5
    batches = [gen.batch(s + 1)[0] for s in range(S)]
    dev = [t64(k) for k in batches]
    g.prefetch(0, dev[0], cfg.batch, insert_missing=True)
    for s in range(S):
        if s + 1 < S:
            g.prefetch((s + 1) % 2, dev[s + 1], cfg.batch, insert_missing=True)
        out = g.lookup_prefetched(s % 2, cfg.batch)
        st, _ = o.insert(0, batches[s])
        assert st == 0
        dout = (rs.standard_normal((cfg.batch * 26, cfg.dim)) * 0.1).astype(np.float32)
        p = opt_params("adam", cfg.lr, step=s + 1)
        g.backward_update(torch.from_numpy(dout).cuda(), cfg.lr, params=p)
        ref = oracle_step(o, batches[s], cfg.batch, None, "sum", dout, p)
        close(out.cpu().numpy(), ref, f"cfg5 pooled step {s}")
    g.join_prefetch()
    ctx.sync()
    n = g.size(0)
    assert n == o.size(0)
    np.testing.assert_array_equal(g.row_keys(0, 0, n).cpu().numpy().view(np.uint64), o.row_keys(0, 0, n))
    compare_tables(g, o, [n])


@pytest.mark.parametrize("multi", [False, True])
def test_prefetch_graph_replay(ctx, multi):
    """The bench's pattern: graph k (k = step parity) = prefetch(batch s+1 -> slot (s+1)%2)
    + lookup(slot s%2) + backward + join_prefetch, captured once and replayed; device key /
    offset / d_out buffers refilled between replays."""
    rs = np.random.default_rng(77 + multi)
    dim = 64 if multi else 128
    opt = "adagrad" if multi else "sgd"
    caps, slots = [20000, 60, 3000], ([0, 1, 2, 0] if multi else [0, 1, 0, 0])
    g, o = make_pair(ctx, caps, dim, slots, opt, a0=0.1 if multi else 0.0)
    pools = load_tables(g, o, caps, rs)
    g.set_pipeline(2)
    B, S = 800, 8
    if multi:
        batches = multihot_batches(pools, rs, B, S, slots)
    else:
        batches = [(k, None) for k in onehot_batches([pools[0], pools[1]], rs, B, S)]
    nmax = max(len(k) for k, _ in batches)
    kbuf = [torch.zeros(nmax, dtype=torch.int64, device="cuda") for _ in range(2)]
    obuf = [torch.zeros(B * 4 + 1, dtype=torch.int32, device="cuda") for _ in range(2)]
    dbuf = torch.zeros(B * 4, dim, dtype=torch.float32, device="cuda")
    outbuf = torch.zeros(B * 4, dim, dtype=torch.float32, device="cuda")
    comb = "mean" if multi else "sum"
    p = opt_params(opt, 0.01, eps=1e-7) if multi else opt_params(opt, 0.01)

    def fill(slot, s):
        k, f = batches[s]
        kbuf[slot].zero_()
        kbuf[slot][:len(k)].copy_(t64(k))
        if multi:
            obuf[slot].copy_(t32(f))

    def keys_of(slot, s):
        return kbuf[slot][:len(batches[s][0])]

    stream = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    stream.wait_stream(main)
    graphs = {}
    with torch.cuda.stream(stream):
        ctx.set_stream(stream)
        try:
            fill(0, 0)
            g.prefetch(0, keys_of(0, 0), B, offsets=obuf[0] if multi else None, combiner=comb)
            g.join_prefetch()
            for s in range(S):
                nxt = min(s + 1, S - 1)  # the last step prefetches a dummy repeat (never consumed)
                fill((s + 1) % 2, nxt)
                dout = rs.standard_normal((B * 4, dim)).astype(np.float32)
                dbuf.copy_(torch.from_numpy(dout))
                par = s % 2
                if par not in graphs:
                    # the key-count of a one-hot batch is fixed by B; multi-hot reads it from the offsets
                    cg = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(cg, stream=stream):
                        g.prefetch((s + 1) % 2, kbuf[(s + 1) % 2][:len(batches[nxt][0])] if not multi else kbuf[(s + 1) % 2],
                                   B, offsets=obuf[(s + 1) % 2] if multi else None, combiner=comb)
                        g.lookup_prefetched(par, B, offsets=obuf[par] if multi else None, combiner=comb, out=outbuf)
                        g.backward_update(dbuf, 0.01, params=p)
                        g.join_prefetch()
                    graphs[par] = cg
                graphs[par].replay()
                ref = oracle_step(o, batches[s][0], B, batches[s][1], comb, dout, p)
                stream.synchronize()
                close(outbuf.cpu().numpy(), ref, f"graph step {s}")
        finally:
            main.wait_stream(stream)
            ctx.set_stream(main)  # (torch's current stream inside this block is `stream`)
    ctx.sync()
    compare_tables(g, o, caps)


def test_prefetch_refusals_and_mixing(ctx):
    rs = np.random.default_rng(9)
    caps, dim = [5000], 32
    g, o = make_pair(ctx, caps, dim, [0, 0], "sgd")
    pools = load_tables(g, o, caps, rs)
    B = 300
    k = [rs.choice(pools[0], 2 * B).astype(np.uint64) for _ in range(4)]
    with pytest.raises(HpsError):
        g.prefetch(1, t64(k[0]), B)  # depth 1: slot 1 does not exist
    g.set_pipeline(2)
    with pytest.raises(HpsError):
        g.lookup_prefetched(1, B)  # nothing prefetched there
    # plain lookup (slot 0) awaiting its backward: that slot cannot be prefetched into
    out = g.lookup(t64(k[0]), B, train=True)
    with pytest.raises(HpsError):
        g.prefetch(0, t64(k[1]), B)
    g.prefetch(1, t64(k[1]), B)  # the other slot is fine, concurrent with this backward
    d0 = rs.standard_normal((2 * B, dim)).astype(np.float32)
    g.backward_update(torch.from_numpy(d0).cuda(), 0.01)
    close(out.cpu().numpy(), oracle_step(o, k[0], B, None, "sum", d0, opt_params("sgd", 0.01)), "mixed 0")
    with pytest.raises(HpsError):
        g.lookup_prefetched(1, B + 1)  # bag count differs from the prefetch
    out = g.lookup_prefetched(1, B)
    d1 = rs.standard_normal((2 * B, dim)).astype(np.float32)
    g.backward_update(torch.from_numpy(d1).cuda(), 0.01)
    close(out.cpu().numpy(), oracle_step(o, k[1], B, None, "sum", d1, opt_params("sgd", 0.01)), "mixed 1")
    # a prefetched slot overwritten by a plain training lookup before it was consumed
    g.prefetch(0, t64(k[2]), B)
    out = g.lookup(t64(k[3]), B, train=True)  # current slot is 1 (the last consumed)
    d3 = rs.standard_normal((2 * B, dim)).astype(np.float32)
    g.backward_update(torch.from_numpy(d3).cuda(), 0.01)
    close(out.cpu().numpy(), oracle_step(o, k[3], B, None, "sum", d3, opt_params("sgd", 0.01)), "mixed 3")
    out = g.lookup_prefetched(0, B)  # the prefetch of k[2] is still intact
    d2 = rs.standard_normal((2 * B, dim)).astype(np.float32)
    g.backward_update(torch.from_numpy(d2).cuda(), 0.01)
    close(out.cpu().numpy(), oracle_step(o, k[2], B, None, "sum", d2, opt_params("sgd", 0.01)), "mixed 2")
    ctx.sync()
    compare_tables(g, o, caps)
    assert g.batch_table_used() == 0
