"""GPU parity for the exchange kernels (exchange.cu) and the distributed step on one rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2210_08803_b200 import EmbeddingTableGroup, opt_params
from paper_2210_08803_b200.exchange import DistributedExchange, GpuEngine
from tests import oracle_lib as O
from tests.cpu_engine import CpuEngine, pool_sequential

pytestmark = pytest.mark.gpu


def t64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


@pytest.mark.parametrize("G", [1, 2, 8, 5])
def test_bucketize_matches_stable_partition(ctx, G):
    rs = np.random.default_rng(G)
    g = EmbeddingTableGroup(ctx, [100, 100, 100], 8, [0, 1, 2], "sgd", 1 << 15, 1 << 15)
    eng = GpuEngine(ctx, g, [0, 1, 2], 1 << 15, G)
    cpu = CpuEngine(None, [0, 1, 2], G, 8)
    keys = rs.integers(-2**63, 2**63 - 1, 20000, dtype=np.int64)
    sk, st, perm, counts = eng.bucketize(torch.from_numpy(keys).cuda(), None)
    rk, rt, rp, rc = cpu.bucketize(torch.from_numpy(keys), None)
    assert np.array_equal(sk.cpu().numpy(), rk.numpy())
    assert np.array_equal(st.cpu().numpy(), rt.numpy())
    assert np.array_equal(perm.cpu().numpy(), rp.numpy())
    assert np.array_equal(counts.cpu().numpy(), rc.numpy())
    offs = np.zeros(6001, dtype=np.int32)
    offs[1:] = np.cumsum(rs.integers(0, 7, 6000))
    ob = eng.occurrence_bags(torch.from_numpy(offs).cuda(), 6000)[: offs[-1]].cpu().numpy()
    assert np.array_equal(ob, np.repeat(np.arange(6000), np.diff(offs)))


@pytest.mark.parametrize("dim,mean", [(128, False), (64, True), (16, True)])
def test_pool_and_scatter(ctx, dim, mean):
    rs = np.random.default_rng(dim)
    g = EmbeddingTableGroup(ctx, [10], dim, [0], "sgd", 1 << 15, 1 << 15)
    eng = GpuEngine(ctx, g, [0], 1 << 15, 1)
    n_bags = 3000
    offs = np.zeros(n_bags + 1, dtype=np.int32)
    offs[1:] = np.cumsum(rs.integers(0, 9, n_bags))
    n = int(offs[-1])
    perm = rs.permutation(n).astype(np.int32)
    rows = rs.standard_normal((n, dim)).astype(np.float32)
    got = eng.pool_rows(torch.from_numpy(rows).cuda(), torch.from_numpy(perm).cuda(), torch.from_numpy(offs).cuda(),
                        n_bags, 1 if mean else 0).cpu().numpy()
    want = pool_sequential(rows, perm.astype(np.int64), offs, n_bags, mean)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    dout = rs.standard_normal((n_bags, dim)).astype(np.float32)
    got = eng.scatter_grads(torch.from_numpy(dout).cuda(), torch.from_numpy(perm).cuda(),
                            torch.from_numpy(offs).cuda(), n_bags, n, 1 if mean else 0).cpu().numpy()
    want = CpuEngine(None, [0], 1, dim).scatter_grads(torch.from_numpy(dout), torch.from_numpy(perm),
                                                       torch.from_numpy(offs), n_bags, n, 1 if mean else 0).numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.fixture(scope="module")
def nccl1(ctx):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def test_distributed_step_single_rank_nccl(ctx, nccl1):
    """The full exchange path (bucketize -> NCCL all-to-all -> gather -> pool -> grads ->
    all-to-all -> dedup/reduce/update) on a world of one, bit-exact with the oracle table."""
    rs = np.random.default_rng(3)
    cards, slots, dim = [3000, 12], [0, 1, 0], 32
    g = EmbeddingTableGroup(ctx, cards, dim, list(range(len(cards))), "adagrad", 1 << 16, 1 << 16, 9, 0.1)
    o = O.OracleTable(cards, dim, slots, "adagrad", 9, 0.1)
    pools = []
    for t, c in enumerate(cards):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks))
        o.insert(t, ks)
        pools.append(ks)
    ex = DistributedExchange(GpuEngine(ctx, g, slots, 1 << 16, 1), "mean", 0, 1)
    B = 400
    for step in range(3):
        lens = rs.integers(0, 8, B * 3)
        offs = np.zeros(B * 3 + 1, dtype=np.uint32)
        offs[1:] = np.cumsum(lens)
        keys = np.concatenate([rs.choice(pools[slots[b % 3]], lens[b]) for b in range(B * 3)]).astype(np.uint64)
        out = ex.forward(t64(keys), torch.from_numpy(offs.view(np.int32)).cuda(), B * 3).cpu().numpy()
        ref = o.lookup(keys, B, offsets=offs, combiner="mean", train=True)
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params("adagrad", 0.05, eps=1e-7)
        ex.backward(torch.from_numpy(dout).cuda(), p)
        o.backward_update(dout, p)
        ctx.sync()
    for t, c in enumerate(cards):
        assert np.array_equal(g.export(t, 0, c)[0].cpu().numpy(), o.export(t, 0, c)[0])
    ex.e.close()


@pytest.mark.parametrize("multi", [False, True])
def test_localized_engine_ops_match_cpu(ctx, multi):
    """regroup_bags / lengths_to_offsets / place_pooled (both directions) for a 3-owner plan
    against the numpy engine, bit-exact."""
    from paper_2210_08803_b200.exchange import LocalizedGpuEngine
    from tests.cpu_engine import LocalizedCpuEngine
    rs = np.random.default_rng(7)
    S, b, dim = 6, 300, 16
    owned = [[0, 4], [1, 2, 5], [3]]
    lens = rs.integers(0, 7, b * S) if multi else np.ones(b * S, dtype=np.int64)
    offs = np.zeros(b * S + 1, dtype=np.int32)
    offs[1:] = np.cumsum(lens)
    keys = rs.integers(-2**63, 2**63 - 1, int(offs[-1]), dtype=np.int64)
    eng = LocalizedGpuEngine(ctx, None, S, owned, b, int(offs[-1]), dim)
    cpu = LocalizedCpuEngine(None, S, owned, dim)
    ko, oo = torch.from_numpy(keys), torch.from_numpy(offs) if multi else None
    kd, od = ko.cuda(), (oo.cuda() if multi else None)
    full = torch.from_numpy(rs.standard_normal((b * S, dim)).astype(np.float32))
    out_g = torch.zeros(b * S, dim, device="cuda")
    out_c = torch.zeros(b * S, dim)
    for g in range(3):
        gk, gl, go = eng.regroup(kd, od, b, g)
        ck, cl, co = cpu.regroup(ko, oo, b, g)
        n = int(go[-1].item())
        assert n == int(co[-1])
        assert np.array_equal(gk[:n].cpu().numpy(), ck.numpy())
        assert np.array_equal(gl.cpu().numpy(), cl.numpy())
        assert np.array_equal(go.cpu().numpy(), co.numpy())
        assert np.array_equal(eng.offsets_from_lengths(gl).cpu().numpy(), co.numpy())
        blk_g = torch.empty(b * len(owned[g]), dim, device="cuda")
        blk_c = torch.empty(b * len(owned[g]), dim)
        eng.place(full.cuda(), g, b, blk_g, 1)
        cpu.place(full, g, b, blk_c, 1)
        assert torch.equal(blk_g.cpu(), blk_c)
        eng.place(blk_g, g, b, out_g, 0)
        cpu.place(blk_c, g, b, out_c, 0)
    assert torch.equal(out_g.cpu(), full) and torch.equal(out_c, full)


@pytest.mark.parametrize("multi,opt", [(False, "sgd"), (True, "adagrad")])
def test_localized_step_single_rank_nccl(ctx, nccl1, multi, opt):
    """Localized exchange over NCCL on a world of one: regroup -> all-to-all -> owner lookup
    -> all-to-all -> place; backward the reverse. Bit-exact with the oracle table."""
    from paper_2210_08803_b200.exchange import LocalizedExchange, LocalizedGpuEngine
    rs = np.random.default_rng(11)
    cards, slots, dim = [3000, 12, 700], [2, 0, 1, 0], 32
    S, B = len(slots), 500
    owned = [[0, 1, 2, 3]]
    g = EmbeddingTableGroup(ctx, cards, dim, slots, opt, 1 << 16, 1 << 16, 9, 0.1)
    o = O.OracleTable(cards, dim, slots, opt, 9, 0.1)
    pools = []
    for t, c in enumerate(cards):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        g.insert(t, t64(ks))
        o.insert(t, ks)
        pools.append(ks)
    comb = "mean" if multi else "sum"
    ex = LocalizedExchange(LocalizedGpuEngine(ctx, g, S, owned, B, 1 << 16, dim), comb, 0, 1, S, owned)
    for step in range(3):
        lens = rs.integers(0, 8, B * S) if multi else np.ones(B * S, dtype=np.int64)
        offs = np.zeros(B * S + 1, dtype=np.uint32)
        offs[1:] = np.cumsum(lens)
        keys = np.concatenate([rs.choice(pools[slots[k % S]], lens[k]) for k in range(B * S)]).astype(np.uint64)
        od = torch.from_numpy(offs.view(np.int32)).cuda() if multi else None
        out = ex.forward(t64(keys), od, B).cpu().numpy()
        ref = o.lookup(keys, B, offsets=offs if multi else None, combiner=comb, train=True)
        assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(opt, 0.05, eps=1e-7)
        ex.backward(torch.from_numpy(dout).cuda(), p)
        o.backward_update(dout, p)
        ctx.sync()
    for t, c in enumerate(cards):
        assert np.array_equal(g.export(t, 0, c)[0].cpu().numpy(), o.export(t, 0, c)[0])


def test_sum_partials_matches_numpy(ctx):
    from paper_2210_08803_b200.exchange import _ptr
    from paper_2210_08803_b200 import _lib as L
    from tests.cpu_engine import sum_partials_np
    rs = np.random.default_rng(5)
    G, R, D = 3, 500, 16
    parts = rs.standard_normal((G, R, D)).astype(np.float32)
    parts[1, 7] = -0.0
    touched = (rs.random((G, R)) < 0.5).astype(np.int32)
    out = torch.empty(R, D, device="cuda")
    t = torch.empty(R, dtype=torch.int32, device="cuda")
    pg, tg = torch.from_numpy(parts).cuda(), torch.from_numpy(touched).cuda()
    L.check(ctx.lib.hps_gpu_sum_partials(ctx.h, _ptr(pg), _ptr(tg), G, R, D, _ptr(out), _ptr(t)), "sum_partials")
    ro, rt = sum_partials_np(parts, touched, G, R)
    np.testing.assert_array_equal(t.cpu().numpy(), rt.numpy())
    m = rt.numpy() != 0
    assert np.array_equal(out.cpu().numpy()[m].view(np.uint32), ro.numpy()[m].view(np.uint32))


@pytest.mark.parametrize("multi,opt", [(False, "sgd"), (True, "adam")])
def test_hybrid_step_single_rank_nccl(ctx, nccl1, multi, opt):
    """Hybrid exchange on a world of one over NCCL: hot replica + cold shard, every kernel of
    the path (probe, cold bucketize/gather, pool, cold grads, backward_reduce, sum_partials,
    apply_grads), against the single-table oracle with the hybrid reduction order."""
    from paper_2210_08803_b200.exchange import HybridExchange, HybridGpuEngine
    from tests.test_multiproc_exchange import _hybrid_reference_step
    rs = np.random.default_rng(13)
    cards, slots, dim = [3000, 12, 700], [2, 0, 1, 0], 32
    S, B = len(slots), 400
    n_hot = [30, 4, 50]
    comb = "mean" if multi else "sum"
    ref = O.OracleTable(cards, dim, slots, opt, 9, 0.1)
    hot = EmbeddingTableGroup(ctx, n_hot, dim, slots, opt, 1 << 16, 1 << 16, 9, 0.1)
    cold = EmbeddingTableGroup(ctx, cards, dim, list(range(3)), opt, 1 << 16, 1 << 16, 9, 0.1)
    pools, hot_rows = [], []
    for t, c in enumerate(cards):
        ks = rs.integers(0, 2**63, c).astype(np.uint64)
        ref.insert(t, ks)
        hot.insert(t, t64(ks[:n_hot[t]]))
        cold.insert(t, t64(ks[n_hot[t]:]))
        hot_rows.extend((int(sum(cards[:t])) + ref.find(t, ks[:n_hot[t]]).astype(np.int64)).tolist())
        pools.append(ks)
    hot_rows = np.array(hot_rows, dtype=np.int64)
    eng = HybridGpuEngine(ctx, hot, GpuEngine(ctx, cold, slots, 1 << 16, 1), 1 << 16)
    ex = HybridExchange(eng, comb, 0, 1, S)
    for step in range(1, 4):
        lens = rs.integers(0, 8, B * S) if multi else np.ones(B * S, dtype=np.int64)
        offs = np.zeros(B * S + 1, dtype=np.int64)
        offs[1:] = np.cumsum(lens)
        keys = np.concatenate([np.where(rs.random(lens[k]) < 0.5, pools[slots[k % S]][rs.integers(0, 3, lens[k])],
                                        rs.choice(pools[slots[k % S]], lens[k])) for k in range(B * S)]).astype(np.uint64)
        od = torch.from_numpy(offs.astype(np.int32)).cuda() if multi else None
        ref_out = ref.lookup(keys, B, offsets=offs.astype(np.uint32) if multi else None, combiner=comb)
        out = ex.forward(t64(keys), od, B).cpu().numpy()
        assert np.array_equal(out.view(np.uint32), ref_out.view(np.uint32))
        dout = rs.standard_normal(ref_out.shape).astype(np.float32)
        p = opt_params(opt, 0.05, step=step)
        ex.backward(torch.from_numpy(dout).cuda(), p)
        _hybrid_reference_step(ref, keys, offs, B, 1, S, multi, comb, dout, p, hot_rows)
        ctx.sync()
    for t, c in enumerate(cards):
        rw = ref.export(t, 0, c)[0]
        hr = ref.find(t, pools[t][:n_hot[t]]).astype(np.int64)
        assert np.array_equal(hot.export(t, 0, n_hot[t])[0].cpu().numpy(), rw[hr])
        cr = ref.find(t, pools[t][n_hot[t]:]).astype(np.int64)
        assert np.array_equal(cold.export(t, 0, c - n_hot[t])[0].cpu().numpy(), rw[cr])
    eng.cold.close()
