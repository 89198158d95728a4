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
