"""World-size-2 gloo test of the distributed-slot exchange orchestration (exchange.py).

Each rank owns the keys with partition_of(key, 2) == rank; the SAME DistributedExchange
host code that runs over NCCL on B200s runs here over gloo with the CPU engine
(tests/cpu_engine.py, oracle-backed). Pooled outputs and every updated row must be
bit-identical to one unsharded oracle table driven with the concatenated global batch.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_batch(rs, pools, slot_table, n_samples, multi):
    S = len(slot_table)
    lens = rs.integers(0, 6, n_samples * S) if multi else np.ones(n_samples * S, dtype=np.int64)
    offs = np.zeros(n_samples * S + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens)
    keys = []
    for b in range(n_samples * S):
        pool = pools[slot_table[b % S]]
        hot = rs.random(lens[b]) < 0.4
        keys.append(np.where(hot, pool[rs.integers(0, 2, lens[b])], rs.choice(pool, lens[b])))
    return np.concatenate(keys).astype(np.uint64), offs


def _worker(rank, world, port, out_dir, multi, optimizer):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2210_08803_b200.api import opt_params
    from paper_2210_08803_b200.exchange import DistributedExchange
    from tests import oracle_lib as O
    from tests.cpu_engine import CpuEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rs = np.random.default_rng(123)
    cards, slot_table, dim = [400, 9, 60], [0, 1, 2, 1], 8
    combiner = "mean" if multi else "sum"
    pools = [rs.integers(0, 2**63, c).astype(np.uint64) for c in cards]
    single = O.OracleTable(cards, dim, slot_table, optimizer, seed=5, a0=0.1)
    shard = O.OracleTable(cards, dim, slot_table, optimizer, seed=5, a0=0.1)
    for t, ks in enumerate(pools):
        single.insert(t, ks)
        own = np.empty(len(ks), dtype=np.uint32)
        O.lib().orc_partition_of_n(O.P(ks), len(ks), world, O.P(own))
        shard.insert(t, ks[own == rank])
    ex = DistributedExchange(CpuEngine(shard, slot_table, world, dim), combiner, rank, world)
    B, S = 24, len(slot_table)
    for step in range(1, 4):
        keys, offs = _global_batch(rs, pools, slot_table, B * world, multi)
        ref = single.lookup(keys, B * world, offsets=offs.astype(np.uint32) if multi else None, combiner=combiner,
                            train=True)
        lo, hi = offs[rank * B * S], offs[(rank + 1) * B * S]
        k_local = torch.from_numpy(keys[lo:hi].view(np.int64).copy())
        o_local = torch.from_numpy((offs[rank * B * S:(rank + 1) * B * S + 1] - lo).astype(np.int32)) if multi else None
        out = ex.forward(k_local, o_local, B * S).numpy()
        assert np.array_equal(out.view(np.uint32), ref[rank * B * S:(rank + 1) * B * S].view(np.uint32)), "forward"
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(optimizer, 0.05, step=step, eps=1e-7)
        ex.backward(torch.from_numpy(dout[rank * B * S:(rank + 1) * B * S].copy()), p)
        single.backward_update(dout, p)
    # every key this rank owns: same row values (and optimizer state) as the single table
    mism = 0
    for t, ks in enumerate(pools):
        own = np.empty(len(ks), dtype=np.uint32)
        O.lib().orc_partition_of_n(O.P(ks), len(ks), world, O.P(own))
        mine = ks[own == rank]
        rs_rows, rg_rows = shard.find(t, mine), single.find(t, ks[own == rank])
        ws, s0s, _ = shard.export(t, 0, shard.size(t))
        wg, s0g, _ = single.export(t, 0, single.size(t))
        mism += int((ws[rs_rows.astype(np.int64)].view(np.uint32) != wg[rg_rows.astype(np.int64)].view(np.uint32)).sum())
        if s0s is not None:
            mism += int((s0s[rs_rows.astype(np.int64)] != s0g[rg_rows.astype(np.int64)]).sum())
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(str(mism))
    dist.destroy_process_group()


@pytest.mark.parametrize("multi,optimizer", [(False, "sgd"), (True, "adagrad"), (False, "adam")])
def test_distributed_exchange_world2_bit_exact(multi, optimizer):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d, multi, optimizer), nprocs=2, join=True)
        for r in range(2):
            assert open(os.path.join(d, f"rank{r}.txt")).read() == "0"


def _local_worker(rank, world, port, out_dir, multi, optimizer, owned):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2210_08803_b200.api import opt_params
    from paper_2210_08803_b200.exchange import LocalizedExchange
    from tests import oracle_lib as O
    from tests.cpu_engine import LocalizedCpuEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rs = np.random.default_rng(321)
    cards, slot_table, dim = [400, 9, 60], [0, 1, 2, 1], 8
    combiner = "mean" if multi else "sum"
    pools = [rs.integers(0, 2**63, c).astype(np.uint64) for c in cards]
    single = O.OracleTable(cards, dim, slot_table, optimizer, seed=5, a0=0.1)
    for t, ks in enumerate(pools):
        single.insert(t, ks)
    # the owner holds whole tables: local table j = my_tables[j]; local slot table follows owned[rank]
    mine = owned[rank]
    my_tables = sorted({slot_table[s] for s in mine})
    shard = None
    if mine:
        shard = O.OracleTable([cards[t] for t in my_tables], dim, [my_tables.index(slot_table[s]) for s in mine],
                              optimizer, seed=5, a0=0.1)
        for j, t in enumerate(my_tables):
            shard.insert(j, pools[t])
    S = len(slot_table)
    ex = LocalizedExchange(LocalizedCpuEngine(shard, S, owned, dim), combiner, rank, world, S, owned)
    B = 24
    for step in range(1, 4):
        keys, offs = _global_batch(rs, pools, slot_table, B * world, multi)
        ref = single.lookup(keys, B * world, offsets=offs.astype(np.uint32) if multi else None, combiner=combiner,
                            train=True)
        lo, hi = offs[rank * B * S], offs[(rank + 1) * B * S]
        k_local = torch.from_numpy(keys[lo:hi].view(np.int64).copy())
        o_local = torch.from_numpy((offs[rank * B * S:(rank + 1) * B * S + 1] - lo).astype(np.int32)) if multi else None
        out = ex.forward(k_local, o_local, B).numpy()
        assert np.array_equal(out.view(np.uint32), ref[rank * B * S:(rank + 1) * B * S].view(np.uint32)), "forward"
        dout = rs.standard_normal(ref.shape).astype(np.float32)
        p = opt_params(optimizer, 0.05, step=step, eps=1e-7)
        ex.backward(torch.from_numpy(dout[rank * B * S:(rank + 1) * B * S].copy()), p)
        single.backward_update(dout, p)
    mism = 0
    for j, t in enumerate(my_tables):
        a, b = shard.export(j, 0, cards[t]), single.export(t, 0, cards[t])
        for x, y in zip(a, b):
            if x is not None:
                mism += int((x.view(np.uint32) != y.view(np.uint32)).sum())
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(str(mism))
    dist.destroy_process_group()


@pytest.mark.parametrize("multi,optimizer,owned", [
    (False, "sgd", [[0, 2], [1, 3]]),
    (True, "adagrad", [[1, 3], [0, 2]]),
    (True, "adam", [[0, 1, 2, 3], []]),
])
def test_localized_exchange_world2_bit_exact(multi, optimizer, owned):
    """Localized slots (config 3): keys of each slot go to its owner, which pools every
    rank's samples; pooled blocks and gradients travel back along the batch dimension.
    Outputs and every owned table's rows + state must equal one unsharded oracle table."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_local_worker, args=(2, _free_port(), d, multi, optimizer, owned), nprocs=2, join=True)
        for r in range(2):
            assert open(os.path.join(d, f"rank{r}.txt")).read() == "0"


def _hybrid_reference_step(ref, keys, offs, B, world, S, multi, combiner, dout, p, hot_rows):
    """Single-table oracle semantics of the hybrid step: cold rows canonical over the global
    batch; a hot row's gradient = rank-ordered sum of each rank's canonical partial."""
    from tests.cpu_engine import sum_partials_np
    ref.lookup(keys, B * world, offsets=offs.astype(np.uint32) if multi else None, combiner=combiner, train=True)
    gc, tc = ref.reduce_only(dout)
    parts, touched = [], []
    for r in range(world):
        lo, hi = offs[r * B * S], offs[(r + 1) * B * S]
        o = (offs[r * B * S:(r + 1) * B * S + 1] - lo).astype(np.uint32) if multi else None
        ref.lookup(keys[lo:hi], B, offsets=o, combiner=combiner, train=True)
        g, t = ref.reduce_only(dout[r * B * S:(r + 1) * B * S])
        parts.append(g)
        touched.append(t)
    hs, ht = sum_partials_np(np.stack(parts), np.stack(touched), world, gc.shape[0])
    hs, ht = hs.numpy(), ht.numpy()
    gc[hot_rows] = hs[hot_rows]
    ref.apply_grads(gc, tc, p)


def _hybrid_worker(rank, world, port, out_dir, multi, optimizer):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2210_08803_b200.api import opt_params
    from paper_2210_08803_b200.exchange import HybridExchange
    from tests import oracle_lib as O
    from tests.cpu_engine import CpuEngine, HybridCpuEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rs = np.random.default_rng(77)
    cards, slot_table, dim = [400, 9, 60], [0, 1, 2, 1], 8
    combiner = "mean" if multi else "sum"
    pools = [rs.integers(0, 2**63, c).astype(np.uint64) for c in cards]
    n_hot = [20, 3, 8]
    hot_keys = [pools[t][:n_hot[t]] for t in range(3)]
    ref = O.OracleTable(cards, dim, slot_table, optimizer, seed=5, a0=0.1)
    hot = O.OracleTable(n_hot, dim, slot_table, optimizer, seed=5, a0=0.1)
    cold = O.OracleTable(cards, dim, slot_table, optimizer, seed=5, a0=0.1)
    hot_rows = []
    for t, ks in enumerate(pools):
        ref.insert(t, ks)
        hot.insert(t, hot_keys[t])
        hot_rows.extend((int(sum(cards[:t])) + ref.find(t, hot_keys[t]).astype(np.int64)).tolist())
        rest = ks[n_hot[t]:]
        own = np.empty(len(rest), dtype=np.uint32)
        O.lib().orc_partition_of_n(O.P(rest), len(rest), world, O.P(own))
        cold.insert(t, rest[own == rank])
    hot_rows = np.array(hot_rows, dtype=np.int64)
    S = len(slot_table)
    eng = HybridCpuEngine(hot, CpuEngine(cold, slot_table, world, dim), slot_table, dim)
    ex = HybridExchange(eng, combiner, rank, world, S)
    B = 24
    for step in range(1, 4):
        keys, offs = _global_batch(rs, pools, slot_table, B * world, multi)
        ref_out = ref.lookup(keys, B * world, offsets=offs.astype(np.uint32) if multi else None, combiner=combiner)
        lo, hi = offs[rank * B * S], offs[(rank + 1) * B * S]
        k_local = torch.from_numpy(keys[lo:hi].view(np.int64).copy())
        o_local = torch.from_numpy((offs[rank * B * S:(rank + 1) * B * S + 1] - lo).astype(np.int32)) if multi else None
        out = ex.forward(k_local, o_local, B).numpy()
        assert np.array_equal(out.view(np.uint32), ref_out[rank * B * S:(rank + 1) * B * S].view(np.uint32)), "fwd"
        dout = rs.standard_normal(ref_out.shape).astype(np.float32)
        p = opt_params(optimizer, 0.05, step=step, eps=1e-7)
        ex.backward(torch.from_numpy(dout[rank * B * S:(rank + 1) * B * S].copy()), p)
        _hybrid_reference_step(ref, keys, offs, B, world, S, multi, combiner, dout, p, hot_rows)
    mism = 0
    for t, ks in enumerate(pools):
        rw = ref.export(t, 0, cards[t])
        hw = hot.export(t, 0, n_hot[t])
        hr = ref.find(t, hot_keys[t]).astype(np.int64)
        for x, y in zip(hw, rw):
            if x is not None:
                mism += int((x.view(np.uint32) != y[hr].view(np.uint32)).sum())
        rest = ks[n_hot[t]:]
        own = np.empty(len(rest), dtype=np.uint32)
        O.lib().orc_partition_of_n(O.P(rest), len(rest), world, O.P(own))
        mine = rest[own == rank]
        cw = cold.export(t, 0, cold.size(t))
        cr = cold.find(t, mine).astype(np.int64)
        rr = ref.find(t, mine).astype(np.int64)
        for x, y in zip(cw, rw):
            if x is not None:
                mism += int((x[cr].view(np.uint32) != y[rr].view(np.uint32)).sum())
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(str(mism))
    dist.destroy_process_group()


@pytest.mark.parametrize("multi,optimizer", [(False, "sgd"), (True, "adagrad"), (True, "adam")])
def test_hybrid_exchange_world2(multi, optimizer):
    """Hybrid sparse embedding: hot keys replicated (deterministic rank-ordered all-reduce of
    per-rank partial gradients), cold keys sharded by partition_of. Forward outputs are
    bit-identical to one unsharded table; every hot replica and cold shard row equals the
    single-table oracle with the hybrid reduction order for hot rows."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_hybrid_worker, args=(2, _free_port(), d, multi, optimizer), nprocs=2, join=True)
        for r in range(2):
            assert open(os.path.join(d, f"rank{r}.txt")).read() == "0"
