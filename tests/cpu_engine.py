"""CPU engine for paper_2210_08803_b200.exchange — TEST INFRASTRUCTURE ONLY.

Implements the device-side ops of the distributed exchange with the oracle (numpy +
oracle/liboracle.so) so that the SAME host orchestration (DistributedExchange) runs over
torch.distributed gloo on CPU. The product engine is exchange.GpuEngine.
"""
import numpy as np
import torch

from tests import oracle_lib as O


def pool_sequential(rows, perm, offsets, n_bags, mean):
    """fp32 bag sums in bag order from +0.0, numpy-vectorised over bags."""
    dim = rows.shape[1]
    offs = np.arange(n_bags + 1, dtype=np.int64) if offsets is None else offsets.astype(np.int64)
    lens = offs[1:] - offs[:-1]
    acc = np.zeros((n_bags, dim), dtype=np.float32)
    for k in range(int(lens.max()) if n_bags else 0):
        m = lens > k
        acc[m] = acc[m] + rows[perm[offs[:-1][m] + k]]
    if mean:
        nz = lens > 0
        acc[nz] = acc[nz] / lens[nz, None].astype(np.float32)
    return acc


class CpuEngine:
    def __init__(self, oracle_table, slot_table, n_shards, dim):
        self.t, self.slot_table, self.G, self.dim = oracle_table, np.asarray(slot_table, np.int64), n_shards, dim

    def occurrence_bags(self, offsets, n_bags):
        o = offsets.numpy().astype(np.int64)
        return torch.from_numpy(np.repeat(np.arange(n_bags, dtype=np.int32), o[1:] - o[:-1]))

    def bucketize(self, keys, occ_bag):
        k = keys.numpy().view(np.uint64)
        owners = np.empty(len(k), dtype=np.uint32)
        O.lib().orc_partition_of_n(O.P(k), len(k), self.G, O.P(owners))
        order = np.argsort(owners, kind="stable")
        bag = np.arange(len(k)) if occ_bag is None else occ_bag.numpy().astype(np.int64)
        tables = self.slot_table[bag % len(self.slot_table)].astype(np.int32)
        perm = np.empty(len(k), dtype=np.int32)
        perm[order] = np.arange(len(k), dtype=np.int32)
        counts = np.bincount(owners, minlength=self.G).astype(np.int32)
        return (torch.from_numpy(k[order].view(np.int64).copy()), torch.from_numpy(tables[order].copy()),
                torch.from_numpy(perm), torch.from_numpy(counts))

    def gather_rows(self, keys, tables, train):
        return torch.from_numpy(O.gather_rows(self.t, keys.numpy().view(np.uint64), tables.numpy().view(np.uint32),
                                              train))

    def pool_rows(self, rows, perm, offsets, n_bags, combiner):
        return torch.from_numpy(pool_sequential(rows.numpy(), perm.numpy().astype(np.int64),
                                                None if offsets is None else offsets.numpy(), n_bags, combiner == 1))

    def scatter_grads(self, dout, perm, offsets, n_bags, n_occ, combiner):
        d = dout.numpy()
        offs = np.arange(n_bags + 1) if offsets is None else offsets.numpy().astype(np.int64)
        lens = offs[1:] - offs[:-1]
        bag = np.repeat(np.arange(n_bags), lens)
        g = d[bag]
        if combiner == 1:
            g = g / lens[bag, None].astype(np.float32)
        out = np.empty((n_occ, self.dim), dtype=np.float32)
        out[perm.numpy().astype(np.int64)] = g
        return torch.from_numpy(out)

    def backward(self, grads, params):
        self.t.backward_update(grads.numpy(), params)

    def to_host(self, t):
        return [int(x) for x in t.tolist()]


class LocalizedCpuEngine:
    """Oracle-backed engine for exchange.LocalizedExchange (test infrastructure only)."""

    def __init__(self, oracle_table, n_slots, owned, dim):
        self.t, self.n_slots, self.owned, self.dim = oracle_table, n_slots, owned, dim

    def regroup(self, keys, offsets, n_samples, g):
        sel = np.asarray(self.owned[g], dtype=np.int64)
        k = keys.numpy()
        S = self.n_slots
        offs = np.arange(n_samples * S + 1) if offsets is None else offsets.numpy().astype(np.int64)
        bags = (np.arange(n_samples)[:, None] * S + sel[None, :]).ravel()
        lens = (offs[bags + 1] - offs[bags]).astype(np.int32)
        out = np.concatenate([k[offs[b]:offs[b + 1]] for b in bags]) if len(bags) else k[:0]
        o = np.zeros(len(bags) + 1, dtype=np.int32)
        o[1:] = np.cumsum(lens)
        return torch.from_numpy(out.copy()), torch.from_numpy(lens), torch.from_numpy(o)

    def offsets_from_lengths(self, lens):
        o = np.zeros(lens.numel() + 1, dtype=np.int32)
        o[1:] = np.cumsum(lens.numpy())
        return torch.from_numpy(o)

    def lookup(self, keys, offsets, n_samples, combiner, train):
        k = keys.numpy().view(np.uint64)
        o = None if offsets is None else offsets.numpy().view(np.uint32)
        return torch.from_numpy(self.t.lookup(k, n_samples, offsets=o, combiner="mean" if combiner == 1 else "sum",
                                              train=train))

    def place(self, src, g, n_samples, dst, direction):
        sel = np.asarray(self.owned[g], dtype=np.int64)
        if len(sel) == 0:
            return
        full = torch.from_numpy((np.arange(n_samples)[:, None] * self.n_slots + sel[None, :]).ravel())
        if direction == 0:
            dst[full] = src
        else:
            dst.copy_(src[full])

    def backward(self, grads, params):
        self.t.backward_update(grads.numpy(), params)

    def to_host(self, t):
        return [int(x) for x in t.tolist()]


class HybridCpuEngine:
    """Oracle-backed engine for exchange.HybridExchange (test infrastructure only).
    hot: OracleTable replica of the hot keys; cold: a CpuEngine over this rank's shard."""

    def __init__(self, hot_table, cold_engine, slot_table, dim):
        self.hot, self.cold, self.dim = hot_table, cold_engine, dim
        self.slot_table = np.asarray(slot_table, np.int64)
        self.hot_rows = hot_table.caps_total
        self._hot_occ = None

    def probe(self, keys, offsets, n_samples, combiner):
        k = keys.numpy().view(np.uint64)
        S = len(self.slot_table)
        n_bags = n_samples * S
        offs = np.arange(n_bags + 1) if offsets is None else offsets.numpy().astype(np.int64)
        bag = np.repeat(np.arange(n_bags), offs[1:] - offs[:-1])
        tables = self.slot_table[bag % S]
        # training state of the hot replica (pooled output unused) + hot rows per occurrence
        self.hot.lookup(k, n_samples, offsets=None if offsets is None else offsets.numpy().view(np.uint32),
                        combiner="mean" if combiner == 1 else "sum", train=True)
        rows = np.full(len(k), np.iinfo(np.uint64).max, dtype=np.uint64)
        for t in np.unique(tables):
            m = tables == t
            rows[m] = self.hot.find(int(t), k[m])
        cold = rows == np.iinfo(np.uint64).max
        cold_pos = (np.cumsum(cold) - 1).astype(np.int32)
        self._hot_occ = (k, tables, cold)
        return (torch.from_numpy(k[cold].view(np.int64).copy()), torch.from_numpy(bag[cold].astype(np.int32)),
                torch.from_numpy(cold_pos), int(cold.sum()))

    def pool(self, cold_pos, perm, back, offsets, n_bags, combiner):
        from tests import oracle_lib as O
        k, tables, cold = self._hot_occ
        rows = O.gather_rows(self.hot, k, tables.astype(np.uint32), False)
        cp = cold_pos.numpy().astype(np.int64)
        if cold.any():
            rows[cold] = back.numpy()[perm.numpy().astype(np.int64)[cp[cold]]]
        offs = None if offsets is None else offsets.numpy()
        return torch.from_numpy(pool_sequential(rows, np.arange(len(k)), offs, n_bags, combiner == 1))

    def cold_grads(self, dout, bags, perm, offsets, n, combiner):
        d = dout.numpy()
        b = bags.numpy().astype(np.int64)
        g = d[b]
        if combiner == 1 and offsets is not None:
            o = offsets.numpy().astype(np.int64)
            g = g / (o[b + 1] - o[b])[:, None].astype(np.float32)
        out = np.empty((n, self.dim), dtype=np.float32)
        out[perm.numpy().astype(np.int64)] = g
        return torch.from_numpy(out)

    def hot_reduce(self, dout):
        g, t = self.hot.reduce_only(dout.numpy())
        return torch.from_numpy(g), torch.from_numpy(t.astype(np.int32))

    def sum_partials(self, parts, touched, n_parts, rows):
        return sum_partials_np(parts.numpy(), touched.numpy(), n_parts, rows)

    def hot_apply(self, grads, touched, params):
        self.hot.apply_grads(grads.numpy(), touched.numpy().astype(np.uint32), params)

    def to_host(self, t):
        return [int(x) for x in t.tolist()]


def sum_partials_np(parts, touched, n_parts, rows):
    """Rank-ordered sum of the parts that touched a row (the first starts the sum)."""
    p = parts.reshape(n_parts, rows, -1)
    t = touched.reshape(n_parts, rows) != 0
    out = np.zeros((rows, p.shape[2]), dtype=np.float32)
    any_ = np.zeros(rows, dtype=bool)
    for q in range(n_parts):
        m = t[q]
        first = m & ~any_
        out[first] = p[q][first]
        later = m & any_
        out[later] = out[later] + p[q][later]
        any_ |= m
    return torch.from_numpy(out), torch.from_numpy(any_.astype(np.int32))
