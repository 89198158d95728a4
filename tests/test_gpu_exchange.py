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


def test_distributed_step_single_rank_nccl(ctx):
    """The full exchange path (bucketize -> NCCL all-to-all -> gather -> pool -> grads ->
    all-to-all -> dedup/reduce/update) on a world of one, bit-exact with the oracle table."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
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
    dist.destroy_process_group()
