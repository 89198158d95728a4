"""The sharded C-ABI step (hps_gpu_dist_*, csrc/sharded.cu) against the oracle.

World of one (the NCCL-free aliasing path) and loopback worlds of 2 and 4 ranks on the one
B200: each rank is a context (own stream) + its shard table (the keys with
partition_of(key, G) == rank) + a dist handle, its calls on its own host thread; the
all-to-alls are device copies between the ranks' fixed-capacity regions
(hps_gpu_dist_create_loopback) — the same kernels, regions and ordering as over NCCL.
Pooled outputs and every owned row (weights and optimizer state) must be bit-identical to
ONE oracle table driven with the concatenated global batch (rank-major), as SPEC.md:487-491
placement promises. Graph capture of a world-1 step is checked too."""
import ctypes as C
import threading

import numpy as np
import pytest
import torch

from paper_2210_08803_b200 import Context, DistTable, EmbeddingTableGroup, opt_params
from paper_2210_08803_b200 import _lib as L
from tests import oracle_lib as O
from tests.test_gpu_paths import close, t32, t64

pytestmark = pytest.mark.gpu


def owners(keys, world):
    own = np.empty(len(keys), dtype=np.uint32)
    O.lib().orc_partition_of_n(O.P(keys), len(keys), world, O.P(own))
    return own


def global_batch(rs, pools, slot_table, n_samples, multi):
    S = len(slot_table)
    lens = rs.integers(0, 6, n_samples * S) if multi else np.ones(n_samples * S, dtype=np.int64)
    offs = np.zeros(n_samples * S + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    keys = []
    for b in range(n_samples * S):
        pool = pools[slot_table[b % S]]
        hot = rs.random(lens[b]) < 0.3
        keys.append(np.where(hot, pool[rs.integers(0, 3, lens[b])], rs.choice(pool, lens[b])))
    return np.concatenate(keys).astype(np.uint64), offs


def compare_owned(shards, single, pools, world):
    for r, sh in enumerate(shards):
        for t, ks in enumerate(pools):
            mine = ks[owners(ks, world) == r]
            n = sh.size(t)
            if n == 0:
                assert len(mine) == 0
                continue
            rk_t, ex = sh.row_keys(t, 0, n), sh.export(t, 0, n)
            torch.cuda.synchronize()  # (the copies ran on the rank's context stream)
            rk = rk_t.cpu().numpy().view(np.uint64)
            assert set(rk.tolist()) == set(mine.tolist()), f"rank {r} table {t}: owned key set"
            gw = [x.cpu().numpy() if x is not None else None for x in ex]
            orow = single.find(t, rk).astype(np.int64)
            ow = single.export(t, 0, single.size(t))
            for k, (g, o) in enumerate(zip(gw, ow)):
                if o is not None:
                    close(g, o[orow], f"rank {r} table {t} state {k}")


def run_world(world, multi, optimizer, steps=3, insert=False, transport="nccl"):
    rs = np.random.default_rng(100 * world + 10 * multi + len(optimizer))
    cards, slot_table, dim = [3000, 9, 600], [0, 1, 2, 1], 32 if multi else 128
    comb = "mean" if multi else "sum"
    B, S = 96, len(slot_table)
    pools = [rs.integers(0, 2**63, c).astype(np.uint64) for c in cards]
    a0 = 0.1 if optimizer == "adagrad" else 0.0
    single = O.OracleTable(cards, dim, slot_table, optimizer, seed=5, a0=a0)
    max_keys = B * S * (6 if multi else 1)
    ctxs = [Context(0, torch.cuda.Stream()) for _ in range(world)]
    cfg_probe = L.DistConfig(S, (C.c_uint32 * S)(*slot_table), dim, max_keys, B * S, 0.0)
    cap = max_keys if world == 1 else min(max_keys, int(np.ceil(1.25 * max_keys / world)) + 1024)
    shards = [EmbeddingTableGroup(ctxs[r], cards, dim, list(range(len(cards))), optimizer, world * cap,
                                  world * cap, 5, a0) for r in range(world)]
    for t, ks in enumerate(pools):
        single.insert(t, ks)
        if not insert:
            own = owners(ks, world)
            for r in range(world):
                shards[r].insert(t, t64(ks[own == r]), return_rows=False)
    for c in ctxs:
        c.sync()
    if world == 1:
        dists = [DistTable(ctxs[0], shards[0], slot_table, max_keys, B * S)]
    else:
        outs = (C.c_void_p * world)()
        L.check(ctxs[0].lib.hps_gpu_dist_create_loopback((C.c_void_p * world)(*[c.h for c in ctxs]),
                                                         (C.c_void_p * world)(*[s.h for s in shards]),
                                                         C.byref(cfg_probe), world, outs), "dist_create_loopback")
        dists = []
        for r in range(world):
            d = DistTable.__new__(DistTable)
            d.ctx, d.shard, d.lib, d.n_slots, d.dim, d.h = ctxs[r], shards[r], ctxs[r].lib, S, dim, C.c_void_p(outs[r])
            cp = C.c_uint64(0)
            L.check(d.lib.hps_gpu_dist_capacity(d.h, C.byref(cp)), "capacity")
            d.capacity = int(cp.value)
            dists.append(d)
    assert dists[0].capacity == cap
    if transport != "nccl":
        for d in dists:
            d.set_transport(transport)

    def on_ranks(fn):
        errs = [None] * world
        def body(r):
            try:
                with torch.cuda.stream(ctxs[r].stream):
                    fn(r)
                ctxs[r].sync()
            except BaseException as e:  # noqa: BLE001
                errs[r] = e
        th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        for e in errs:
            if e is not None:
                raise e

    for step in range(1, steps + 1):
        keys, offs = global_batch(rs, pools, slot_table, B * world, multi)
        ref = single.lookup(keys, B * world, offsets=offs.astype(np.uint32) if multi else None, combiner=comb,
                            train=True)
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(optimizer, 0.05, step=step, eps=1e-7)
        outs_l = [None] * world
        loc = []
        for r in range(world):
            lo, hi = offs[r * B * S], offs[(r + 1) * B * S]
            k = t64(keys[lo:hi])
            o = t32(offs[r * B * S:(r + 1) * B * S + 1] - lo) if multi else None
            d = torch.from_numpy(dout[r * B * S:(r + 1) * B * S].copy()).cuda()
            loc.append((k, o, d))
        torch.cuda.synchronize()

        # outputs allocated here, not inside the rank threads: loopback ranks share one device,
        # and an allocation that synchronises the device while a peer's wait kernel spins on
        # this rank's (not yet enqueued) signal would deadlock the peer transport
        outs_pre = [torch.empty(B * S, dim, dtype=torch.float32, device="cuda") for _ in range(world)]
        torch.cuda.synchronize()

        def fwd(r):
            k, o, _ = loc[r]
            outs_l[r] = dists[r].forward(k, B, offsets=o, combiner=comb, train=True, insert_missing=insert,
                                         out=outs_pre[r])

        served0 = [d.unique_rows_served() for d in dists] if transport == "peer" else None
        on_ranks(fwd)
        if transport == "peer":
            # per-destination unique rows: every requester fetched exactly one row per distinct
            # (table, key) of its own batch (each key has one owner), summed over the owners
            served = sum(d.unique_rows_served() for d in dists) - sum(served0)
            want = 0
            for r in range(world if world > 1 else 0):  # (a world of one pools its own rows)
                lo, hi = offs[r * B * S], offs[(r + 1) * B * S]
                bag = np.repeat(np.arange(B * S), np.diff(offs[r * B * S:(r + 1) * B * S + 1])) if multi \
                    else np.arange(B * S)
                tab = np.asarray(slot_table, dtype=np.uint64)[bag % S]
                want += len(set(zip(tab.tolist(), keys[lo:hi].tolist())))
            assert served == want, f"world {world} step {step}: {served} unique rows served, want {want}"
        for r in range(world):
            close(outs_l[r].cpu().numpy(), ref[r * B * S:(r + 1) * B * S], f"world {world} rank {r} step {step}")
        on_ranks(lambda r: dists[r].backward(loc[r][2], p))
        single.backward_update(dout, p)
    compare_owned(shards, single, pools, world)
    for d in dists:
        d.close()


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("multi,optimizer", [(False, "sgd"), (True, "adagrad"), (False, "adam")])
def test_dist_step_matches_single_table(ctx, world, multi, optimizer):
    run_world(world, multi, optimizer)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("multi,optimizer", [(False, "sgd"), (True, "adagrad")])
def test_dist_peer_transport_matches_single_table(ctx, world, multi, optimizer):
    """The peer-memory transport (hps_gpu_dist_set_transport(HPS_DIST_PEER)): the region
    kernel stores into the owners' buffers, the pooling loads the owners' rows, the gradient
    scatter stores into the owners' regions, epochs in flag words order the phases — on the
    loopback ranks the peers' memory is this device's, the same code that runs over NVLink."""
    run_world(world, multi, optimizer, transport="peer")


def test_dist_graph_step_world1(ctx):
    """A world-1 dist step (bucketize, regions, gather, pool, scatter, backward) captured as
    one CUDA graph and replayed: identical to the oracle sequence."""
    rs = np.random.default_rng(7)
    cards, slot_table, dim = [5000, 20], [0, 1, 0], 64
    B, S = 200, 3
    pools = [rs.integers(0, 2**63, c).astype(np.uint64) for c in cards]
    single = O.OracleTable(cards, dim, slot_table, "sgd", seed=5)
    sh = EmbeddingTableGroup(ctx, cards, dim, list(range(2)), "sgd", B * S, B * S, 5)
    for t, ks in enumerate(pools):
        single.insert(t, ks)
        sh.insert(t, t64(ks), return_rows=False)
    dt = DistTable(ctx, sh, slot_table, B * S, B * S)
    kbuf = torch.zeros(B * S, dtype=torch.int64, device="cuda")
    dbuf = torch.zeros(B * S, dim, dtype=torch.float32, device="cuda")
    obuf = torch.zeros(B * S, dim, dtype=torch.float32, device="cuda")
    p = opt_params("sgd", 0.05)
    stream = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    stream.wait_stream(main)
    g = None
    with torch.cuda.stream(stream):
        ctx.set_stream(stream)
        try:
            for step in range(4):
                keys, _ = global_batch(rs, pools, slot_table, B, False)
                kbuf.copy_(t64(keys))
                dout = rs.standard_normal((B * S, dim)).astype(np.float32)
                dbuf.copy_(torch.from_numpy(dout))
                if g is None:
                    dt.forward(kbuf, B, out=obuf)  # warm-up (module loading), then capture
                    dt.backward(dbuf, p)
                    single.lookup(keys, B, train=True)
                    single.backward_update(dout, p)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        dt.forward(kbuf, B, out=obuf)
                        dt.backward(dbuf, p)
                    continue
                g.replay()
                ref = single.lookup(keys, B, train=True)
                single.backward_update(dout, p)
                stream.synchronize()
                close(obuf.cpu().numpy(), ref, f"graph step {step}")
        finally:
            main.wait_stream(stream)
            ctx.set_stream(main)
    ctx.sync()
    for t in range(2):
        n = sh.size(t)
        rk = sh.row_keys(t, 0, n).cpu().numpy().view(np.uint64)
        close(sh.export(t, 0, n)[0].cpu().numpy(), single.export(t, 0, single.size(t))[0][single.find(t, rk).astype(np.int64)],
              f"table {t}")
