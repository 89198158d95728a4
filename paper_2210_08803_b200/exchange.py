"""Model-parallel embedding exchange over torch.distributed (NCCL on B200 / NVLink 5).

Distributed slot placement: every key is owned by rank
partition_of(key, G) (proj/include/hps/hash.hpp:52-54); each rank holds that shard of
every table. One training step:

  requester  bucketize its key occurrences by owner (stable)       hps_gpu_xplan_bucketize
  all-to-all counts, keys, table ids
  owner      gather rows of the received keys (training state)    hps_gpu_gather_rows
  all-to-all rows back
  requester  pool bags from the received rows                      hps_gpu_pool_rows
  ... dense model (out of scope) ...
  requester  per-occurrence gradients in send order                hps_gpu_scatter_grads
  all-to-all gradients
  owner      dedup + blocked reduction + optimizer                 hps_gpu_backward_update

Every step is stable, so each key's occurrences reach its owner in global canonical
order (rank 0's batch, then rank 1's, ...): the sharded step is bit-identical to the
single-table step on the concatenated global batch (tests/test_multiproc_exchange.py).

The orchestration below is backend-neutral host logic; the device work is done by an
*engine*. The product engine is GpuEngine (libhps_gpu.so); tests inject a CPU engine
built on the oracle to run the same orchestration over gloo without a GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from . import workload as W


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class GpuEngine:
    """Device side of the exchange on one rank: a table-group shard + an exchange plan."""

    def __init__(self, ctx, table, slot_table: List[int], max_keys: int, n_shards: int,
                 insert_missing: bool = False):
        self.ctx, self.table, self.lib = ctx, table, ctx.lib
        self.insert_flag = L.LOOKUP_INSERT if insert_missing else 0
        self.dim = table.dim
        self.device = table.device
        self.slot_table = torch.tensor(slot_table, dtype=torch.int32, device=self.device)
        self.n_slots = len(slot_table)
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_xplan_create(ctx.h, max_keys, n_shards, C.byref(h)), "xplan_create")
        self.plan = h
        self.max_keys = max_keys
        self.n_shards = n_shards
        d = self.device
        self.send_keys = torch.empty(max_keys, dtype=torch.int64, device=d)
        self.send_tables = torch.empty(max_keys, dtype=torch.int32, device=d)
        self.perm = torch.empty(max_keys, dtype=torch.int32, device=d)
        self.occ_bag = torch.empty(max_keys, dtype=torch.int32, device=d)
        self.counts = torch.empty(n_shards, dtype=torch.int32, device=d)

    def occurrence_bags(self, offsets: torch.Tensor, n_bags: int) -> torch.Tensor:
        L.check(self.lib.hps_gpu_occurrence_bags(self.ctx.h, _ptr(offsets), n_bags, _ptr(self.occ_bag)), "occ_bags")
        return self.occ_bag

    def bucketize(self, keys: torch.Tensor, occ_bag: Optional[torch.Tensor]):
        n = keys.numel()
        L.check(self.lib.hps_gpu_xplan_bucketize(self.plan, _ptr(keys), n, _ptr(occ_bag), self.n_slots,
                                                 _ptr(self.slot_table), _ptr(self.send_keys),
                                                 _ptr(self.send_tables), _ptr(self.perm), _ptr(self.counts)),
                "bucketize")
        return self.send_keys[:n], self.send_tables[:n], self.perm[:n], self.counts

    def gather_rows(self, keys: torch.Tensor, tables: torch.Tensor, train: bool) -> torch.Tensor:
        n = keys.numel()
        rows = torch.empty(n, self.dim, dtype=torch.float32, device=self.device)
        L.check(self.lib.hps_gpu_gather_rows(self.table.h, _ptr(keys), _ptr(tables), n, _ptr(rows),
                                             (L.LOOKUP_TRAIN if train else 0) | self.insert_flag), "gather_rows")
        return rows

    def pool_rows(self, rows, perm, offsets, n_bags: int, combiner: int) -> torch.Tensor:
        out = torch.empty(n_bags, self.dim, dtype=torch.float32, device=self.device)
        L.check(self.lib.hps_gpu_pool_rows(self.ctx.h, _ptr(rows), _ptr(perm), _ptr(offsets), n_bags, self.dim,
                                           combiner, _ptr(out)), "pool_rows")
        return out

    def scatter_grads(self, dout, perm, offsets, n_bags: int, n_occ: int, combiner: int) -> torch.Tensor:
        grads = torch.empty(n_occ, self.dim, dtype=torch.float32, device=self.device)
        L.check(self.lib.hps_gpu_scatter_grads(self.ctx.h, _ptr(dout), _ptr(perm), _ptr(offsets), n_bags, self.dim,
                                               combiner, _ptr(grads)), "scatter_grads")
        return grads

    def backward(self, grads: torch.Tensor, params: L.OptParams) -> None:
        L.check(self.lib.hps_gpu_backward_update(self.table.h, _ptr(grads), C.byref(params)), "backward_update")

    def to_host(self, t: torch.Tensor) -> List[int]:
        return [int(x) for x in t.tolist()]

    def close(self):
        if getattr(self, "plan", None):
            self.lib.hps_gpu_xplan_destroy(self.plan)
            self.plan = None


class DistributedExchange:
    """Distributed-slot forward/backward for one rank (host orchestration)."""

    def __init__(self, engine, combiner: str, rank: int, world: int, group=None):
        self.e, self.rank, self.world, self.group = engine, rank, world, group
        self.combiner = 1 if combiner == "mean" else 0
        self._saved = None
        self.last_recv = 0

    def _a2a(self, x: torch.Tensor, out_split: List[int], in_split: List[int]) -> torch.Tensor:
        out = torch.empty((sum(out_split),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x, out_split, in_split, group=self.group)
        return out

    def forward(self, keys: torch.Tensor, offsets: Optional[torch.Tensor], n_bags: int, train: bool = True):
        occ_bag = self.e.occurrence_bags(offsets, n_bags) if offsets is not None else None
        send_keys, send_tables, perm, counts = self.e.bucketize(keys, occ_bag)
        in_counts = torch.empty_like(counts)
        dist.all_to_all_single(in_counts, counts, group=self.group)
        sc, rc = self.e.to_host(counts), self.e.to_host(in_counts)
        recv_keys = self._a2a(send_keys, rc, sc)
        recv_tables = self._a2a(send_tables, rc, sc)
        rows = self.e.gather_rows(recv_keys, recv_tables, train)
        back = self._a2a(rows, sc, rc)
        out = self.e.pool_rows(back, perm, offsets, n_bags, self.combiner)
        self._saved = (perm, offsets, n_bags, keys.numel(), sc, rc)
        self.last_recv = sum(rc)
        return out

    def backward(self, dout: torch.Tensor, params: L.OptParams) -> None:
        perm, offsets, n_bags, n_occ, sc, rc = self._saved
        grads = self.e.scatter_grads(dout, perm, offsets, n_bags, n_occ, self.combiner)
        recv = self._a2a(grads, rc, sc)
        self.e.backward(recv, params)

    def exchanged_bytes(self, dim: int) -> int:
        """Bytes this rank sent off-rank in the last step (keys + tables + rows + grads)."""
        perm, offsets, n_bags, n_occ, sc, rc = self._saved
        off_send = sum(c for g, c in enumerate(sc) if g != self.rank)
        off_recv = sum(c for g, c in enumerate(rc) if g != self.rank)
        return off_send * (8 + 4 + dim * 4) + off_recv * dim * 4
