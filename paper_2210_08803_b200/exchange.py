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


# ---------------------------------------------------------------------------------------
# Localized slot placement (config 3)
# ---------------------------------------------------------------------------------------
#
#   requester  regroup its bags by owner of the slot (sample-major CSR)  hps_gpu_regroup_bags
#   all-to-all keys (+ bag lengths for multi-hot)
#   owner      offsets over the received lengths                          hps_gpu_lengths_to_offsets
#              pooled lookup over every rank's samples of its slots       hps_gpu_lookup_pooled
#   all-to-all pooled [b x S_owned x D] blocks back (batch dimension)
#   requester  place the blocks into [b x S x D]                          hps_gpu_place_pooled
#   ... dense model ...
#   requester  gather d_out per owner                                     hps_gpu_place_pooled(1)
#   all-to-all gradients
#   owner      dedup + blocked reduction + optimizer                      hps_gpu_backward_update
#
# The owner's bags arrive rank-major (rank 0's samples, then rank 1's, ...), which is the
# global sample order, so the owner's lookup and backward are the single-GPU kernels on the
# global batch restricted to its slots: bit-identical to one unsharded table group.


class LocalizedGpuEngine:
    """Device side of localized slot placement on one rank. `table` is the group of the
    tables this rank owns, with slot_table = the local table of each owned slot, in
    owned[rank] order (None when the rank owns no slot)."""

    def __init__(self, ctx, table, n_slots: int, owned: List[List[int]], max_samples: int, max_keys: int, dim: int):
        self.ctx, self.table, self.lib = ctx, table, ctx.lib
        self.dim, self.n_slots, self.owned = dim, n_slots, owned
        d = torch.device("cuda", torch.cuda.current_device())
        self.device = d
        self.sel = [torch.tensor(s if s else [0], dtype=torch.int32, device=d) for s in owned]
        n_sel_max = max(len(s) for s in owned)
        self.lens = [torch.empty(max(1, max_samples * len(s)), dtype=torch.int32, device=d) for s in owned]
        self.keys = [torch.empty(max(1, max_keys), dtype=torch.int64, device=d) for _ in owned]
        self.offs = [torch.zeros(max_samples * len(s) + 1, dtype=torch.int32, device=d) for s in owned]
        world = len(owned)
        tiles = (max_samples * max(n_sel_max, 1) * world) // 2048 + 2
        self.scan = torch.empty(tiles + 2, dtype=torch.int64, device=d)
        self.own_offs = torch.empty(max_samples * world * max(n_sel_max, 1) + 1, dtype=torch.int32, device=d)

    def regroup(self, keys: torch.Tensor, offsets: Optional[torch.Tensor], n_samples: int, g: int):
        """-> (keys of owner g's slots, their bag lengths, device CSR offsets)."""
        n_sel = len(self.owned[g])
        if n_sel == 0:
            return self.keys[g][:0], self.lens[g][:0], self.offs[g][:1]
        L.check(self.lib.hps_gpu_regroup_bags(self.ctx.h, _ptr(keys), _ptr(offsets), n_samples, self.n_slots,
                                              _ptr(self.sel[g]), n_sel, _ptr(self.lens[g]), _ptr(self.keys[g]),
                                              _ptr(self.offs[g]), _ptr(self.scan)), "regroup_bags")
        return self.keys[g], self.lens[g][:n_samples * n_sel], self.offs[g][:n_samples * n_sel + 1]

    def offsets_from_lengths(self, lens: torch.Tensor) -> torch.Tensor:
        n = lens.numel()
        out = self.own_offs[:n + 1]
        L.check(self.lib.hps_gpu_lengths_to_offsets(self.ctx.h, _ptr(lens), n, _ptr(out), _ptr(self.scan)),
                "lengths_to_offsets")
        return out

    def lookup(self, keys, offsets, n_samples: int, combiner: int, train: bool) -> torch.Tensor:
        return self.table.lookup(keys, n_samples, offsets=offsets, combiner="mean" if combiner == 1 else "sum",
                                 train=train)

    def place(self, src: torch.Tensor, g: int, n_samples: int, dst: torch.Tensor, direction: int) -> None:
        n_sel = len(self.owned[g])
        if n_sel == 0:
            return
        L.check(self.lib.hps_gpu_place_pooled(self.ctx.h, _ptr(src), _ptr(self.sel[g]), n_sel, n_samples,
                                              self.n_slots, self.dim, direction, _ptr(dst)), "place_pooled")

    def backward(self, grads: torch.Tensor, params: L.OptParams) -> None:
        L.check(self.lib.hps_gpu_backward_update(self.table.h, _ptr(grads), C.byref(params)), "backward_update")

    def to_host(self, t: torch.Tensor) -> List[int]:
        return [int(x) for x in t.tolist()]


class LocalizedExchange:
    """Localized-slot forward/backward for one rank (host orchestration). owned[g] = the
    slots rank g owns (e.g. placement.plan_localized); every rank has n_samples samples."""

    def __init__(self, engine, combiner: str, rank: int, world: int, n_slots: int, owned: List[List[int]],
                 group=None):
        self.e, self.rank, self.world, self.group = engine, rank, world, group
        self.combiner = 1 if combiner == "mean" else 0
        self.n_slots, self.owned = n_slots, owned
        self._saved = None

    def _a2a(self, x: torch.Tensor, out_split: List[int], in_split: List[int]) -> torch.Tensor:
        out = torch.empty((sum(out_split),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x, out_split, in_split, group=self.group)
        return out

    def forward(self, keys: torch.Tensor, offsets: Optional[torch.Tensor], n_samples: int, train: bool = True):
        G, b, me = self.world, n_samples, self.rank
        n_sel = [len(s) for s in self.owned]
        parts = [self.e.regroup(keys, offsets, b, g) for g in range(G)]
        dim = self.e.dim
        if offsets is None:  # one key per bag: sizes are known on every rank
            sc = [b * n_sel[g] for g in range(G)]
            rc = [b * n_sel[me]] * G
            send_keys = torch.cat([p[0][:sc[g]] for g, p in enumerate(parts)])
            recv_keys = self._a2a(send_keys, rc, sc)
            own_offs = None
        else:
            ends = torch.stack([p[2][-1] for p in parts]).to(torch.int32)
            in_counts = torch.empty_like(ends)
            dist.all_to_all_single(in_counts, ends, group=self.group)
            sc, rc = self.e.to_host(ends), self.e.to_host(in_counts)
            send_keys = torch.cat([p[0][:sc[g]] for g, p in enumerate(parts)])
            recv_keys = self._a2a(send_keys, rc, sc)
            send_lens = torch.cat([p[1] for p in parts])
            recv_lens = self._a2a(send_lens, [b * n_sel[me]] * G, [b * n_sel[g] for g in range(G)])
            own_offs = self.e.offsets_from_lengths(recv_lens)
        if n_sel[me]:
            pooled = self.e.lookup(recv_keys, own_offs, G * b, self.combiner, train)
        else:
            pooled = torch.empty(0, dim, dtype=torch.float32, device=keys.device)
        back = self._a2a(pooled, [b * n_sel[g] for g in range(G)], [b * n_sel[me]] * G)
        out = torch.empty(b * self.n_slots, dim, dtype=torch.float32, device=keys.device)
        base = 0
        for g in range(G):
            self.e.place(back[base:base + b * n_sel[g]], g, b, out, 0)
            base += b * n_sel[g]
        self._saved = (b, sc, rc, offsets is not None)
        return out

    def backward(self, dout: torch.Tensor, params: L.OptParams) -> None:
        G, me = self.world, self.rank
        b = self._saved[0]
        n_sel = [len(s) for s in self.owned]
        send = torch.empty(b * self.n_slots, self.e.dim, dtype=torch.float32, device=dout.device)
        base = 0
        for g in range(G):
            self.e.place(dout, g, b, send[base:base + b * n_sel[g]], 1)
            base += b * n_sel[g]
        recv = self._a2a(send, [b * n_sel[me]] * G, [b * n_sel[g] for g in range(G)])
        if n_sel[me]:
            self.e.backward(recv, params)

    def exchanged_bytes(self, dim: int) -> int:
        """Bytes this rank sent off-rank in the last step (keys [+ lengths] + pooled + grads)."""
        b, sc, rc, multi = self._saved
        n_sel = [len(s) for s in self.owned]
        keys_off = sum(c for g, c in enumerate(sc) if g != self.rank) * 8
        lens_off = sum(b * n_sel[g] for g in range(self.world) if g != self.rank) * 4 if multi else 0
        pooled_off = b * n_sel[self.rank] * (self.world - 1) * dim * 4
        grads_off = sum(b * n_sel[g] for g in range(self.world) if g != self.rank) * dim * 4
        return keys_off + lens_off + pooled_off + grads_off


# ---------------------------------------------------------------------------------------
# Hybrid sparse embedding
# ---------------------------------------------------------------------------------------
#
# Hot keys (placement.plan_hybrid) are replicated on every rank in a "hot" table group
# (data parallel); every other key lives on its owner partition_of(key, G) exactly as in
# the distributed exchange (model parallel). One step on rank r:
#
#   hps_gpu_hybrid_probe     hot-index probe of every occurrence (records the hot group's
#                            training state) + compaction of the cold occurrences
#   cold occurrences         bucketize -> all-to-all -> owner gather -> all-to-all back
#   hps_gpu_hybrid_pool      bag sums in occurrence order (hot replica rows | cold rows)
#   ... dense model ...
#   hps_gpu_cold_grads       -> all-to-all -> owner dedup/reduce/optimizer
#   hps_gpu_backward_reduce  per-hot-row gradient sums of rank r's batch (canonical tree)
#   deterministic all-reduce: all-to-all of row slices, hps_gpu_sum_partials (ranks in
#                            order), all-gather of the summed slices
#   hps_gpu_apply_grads      the same optimizer step on every replica
#
# Only cold rows and the dense hot-gradient all-reduce travel. Numerics: cold keys are
# bit-identical to one unsharded table; a hot key's gradient is the rank-ordered sum of
# each rank's canonical partial (the data-parallel reduction; identical on every rank).


class HybridGpuEngine:
    def __init__(self, ctx, hot_table, cold_engine: GpuEngine, max_keys: int):
        self.ctx, self.hot, self.cold, self.lib = ctx, hot_table, cold_engine, ctx.lib
        self.dim = hot_table.dim
        d = hot_table.device
        self.device = d
        self.hot_rows = int(sum(hot_table.row_capacity))
        self.cold_pos = torch.empty(max(1, max_keys), dtype=torch.int32, device=d)
        self.cold_keys = torch.empty(max(1, max_keys), dtype=torch.int64, device=d)
        self.cold_bags = torch.empty(max(1, max_keys), dtype=torch.int32, device=d)
        self.cold_count = torch.zeros(1, dtype=torch.int64, device=d)
        self.grads = torch.empty(self.hot_rows, self.dim, dtype=torch.float32, device=d)
        self.touched = torch.zeros(self.hot_rows, dtype=torch.int32, device=d)

    def probe(self, keys, offsets, n_samples: int, combiner: int):
        L.check(self.lib.hps_gpu_hybrid_probe(self.hot.h, _ptr(keys), _ptr(offsets), n_samples, combiner, keys.numel(),
                                              _ptr(self.cold_pos), _ptr(self.cold_keys), _ptr(self.cold_bags),
                                              _ptr(self.cold_count)), "hybrid_probe")
        nc = int(self.cold_count.item())
        return self.cold_keys[:nc], self.cold_bags[:nc], self.cold_pos, nc

    def pool(self, cold_pos, perm, back, offsets, n_bags: int, combiner: int):
        out = torch.empty(n_bags, self.dim, dtype=torch.float32, device=self.device)
        L.check(self.lib.hps_gpu_hybrid_pool(self.hot.h, _ptr(cold_pos), _ptr(perm), _ptr(back), _ptr(offsets), n_bags,
                                             combiner, _ptr(out)), "hybrid_pool")
        return out

    def cold_grads(self, dout, bags, perm, offsets, n: int, combiner: int):
        g = torch.empty(n, self.dim, dtype=torch.float32, device=self.device)
        L.check(self.lib.hps_gpu_cold_grads(self.ctx.h, _ptr(dout), _ptr(bags), _ptr(perm), _ptr(offsets), n, self.dim,
                                            combiner, _ptr(g)), "cold_grads")
        return g

    def hot_reduce(self, dout):
        self.touched.zero_()
        L.check(self.lib.hps_gpu_backward_reduce(self.hot.h, _ptr(dout), _ptr(self.grads), _ptr(self.touched)),
                "backward_reduce")
        return self.grads, self.touched

    def sum_partials(self, parts, touched, n_parts: int, rows: int):
        out = torch.empty(rows, self.dim, dtype=torch.float32, device=self.device)
        t = torch.empty(rows, dtype=torch.int32, device=self.device)
        L.check(self.lib.hps_gpu_sum_partials(self.ctx.h, _ptr(parts), _ptr(touched), n_parts, rows, self.dim,
                                              _ptr(out), _ptr(t)), "sum_partials")
        return out, t

    def hot_apply(self, grads, touched, params):
        L.check(self.lib.hps_gpu_apply_grads(self.hot.h, _ptr(grads), _ptr(touched), C.byref(params)), "apply_grads")

    def to_host(self, t: torch.Tensor) -> List[int]:
        return [int(x) for x in t.tolist()]


class HybridExchange:
    """Hybrid forward/backward for one rank (host orchestration over an engine)."""

    def __init__(self, engine, combiner: str, rank: int, world: int, n_slots: int, group=None):
        self.e, self.rank, self.world, self.group = engine, rank, world, group
        self.combiner = 1 if combiner == "mean" else 0
        self.n_slots = n_slots
        self._saved = None

    def _a2a(self, x: torch.Tensor, out_split: List[int], in_split: List[int]) -> torch.Tensor:
        out = torch.empty((sum(out_split),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(out, x, out_split, in_split, group=self.group)
        return out

    def forward(self, keys: torch.Tensor, offsets: Optional[torch.Tensor], n_samples: int, train: bool = True):
        n_bags = n_samples * self.n_slots
        cold_keys, cold_bags, cold_pos, nc = self.e.probe(keys, offsets, n_samples, self.combiner)
        send_keys, send_tables, perm, counts = self.e.cold.bucketize(cold_keys, cold_bags)
        in_counts = torch.empty_like(counts)
        dist.all_to_all_single(in_counts, counts, group=self.group)
        sc, rc = self.e.to_host(counts), self.e.to_host(in_counts)
        recv_keys = self._a2a(send_keys, rc, sc)
        recv_tables = self._a2a(send_tables, rc, sc)
        rows = self.e.cold.gather_rows(recv_keys, recv_tables, train)
        back = self._a2a(rows, sc, rc)
        out = self.e.pool(cold_pos, perm, back, offsets, n_bags, self.combiner)
        self._saved = (perm, cold_bags, nc, offsets, sc, rc)
        return out

    def backward(self, dout: torch.Tensor, params: L.OptParams) -> None:
        perm, cold_bags, nc, offsets, sc, rc = self._saved
        grads = self.e.cold_grads(dout, cold_bags, perm, offsets, nc, self.combiner)
        recv = self._a2a(grads, rc, sc)
        self.e.cold.backward(recv, params)
        # hot rows: deterministic all-reduce of the per-rank partial sums, then every
        # replica takes the same optimizer step
        g, t = self.e.hot_reduce(dout)
        G, R = self.world, g.shape[0]
        sl = (R + G - 1) // G
        if G * sl != R:
            g = torch.cat([g, torch.zeros(G * sl - R, g.shape[1], dtype=g.dtype, device=g.device)])
            t = torch.cat([t, torch.zeros(G * sl - R, dtype=t.dtype, device=t.device)])
        parts = self._a2a(g, [sl] * G, [sl] * G)   # [G x sl x D]: every rank's partial of my slice
        tparts = self._a2a(t, [sl] * G, [sl] * G)
        s, ts = self.e.sum_partials(parts, tparts, G, sl)
        fs = [torch.empty_like(s) for _ in range(G)]
        ft = [torch.empty_like(ts) for _ in range(G)]
        dist.all_gather(fs, s, group=self.group)
        dist.all_gather(ft, ts, group=self.group)
        self.e.hot_apply(torch.cat(fs)[:R].contiguous(), torch.cat(ft)[:R].contiguous(), params)

    def exchanged_bytes(self, dim: int) -> int:
        perm, cold_bags, nc, offsets, sc, rc = self._saved
        off_send = sum(c for g, c in enumerate(sc) if g != self.rank)
        off_recv = sum(c for g, c in enumerate(rc) if g != self.rank)
        G = self.world
        R = self.e.hot_rows
        sl = (R + G - 1) // G
        allreduce = 2 * (G - 1) * sl * (dim * 4 + 4)
        return off_send * (8 + 4 + dim * 4) + off_recv * dim * 4 + allreduce
