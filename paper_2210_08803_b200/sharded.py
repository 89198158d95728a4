"""Table construction and the training step used by bench.py (1..8 GPUs).

Single GPU: one table group holds every table. Multi-GPU (distributed slot sharding,
SPEC.md:487-491): rank r owns the keys with partition_of(key, G) == r;
the exchange lives in paper_2210_08803_b200.exchange.
"""
from __future__ import annotations

import os

import math
from typing import List, Optional

import numpy as np
import torch

from . import workload as W
from . import _lib as L
from .api import Context, EmbeddingTableGroup, _ptr, opt_params


def _owned_keys(ctx: Context, cfg: W.Config, t: int, rank: int, world: int, first: int, n: int) -> torch.Tensor:
    keys = ctx.gen_keys(W.table_seed(cfg.seed, t), first, n)
    if world > 1:
        keys = keys[ctx.partition_of(keys, world) == rank]
    return keys


def long_sort_passes(max_keys: int) -> int:
    """Radix passes of the long-segment list sort (table_internal.cuh bwd_long_passes)."""
    m = max_keys // 33 + 2
    b = m.bit_length()
    return 1 if b <= 8 else (b + 7) // 8


def table_max_keys(cfg: W.Config, world: int) -> int:
    """Key occurrences one rank may have to hold in a step (an owner can receive every
    rank's keys in the worst case)."""
    n_bags = cfg.batch * cfg.n_slots
    return n_bags * (2 * cfg.hot - 1 if cfg.hot > 1 else 1) * world


def build_tables(ctx: Context, cfg: W.Config, rank: int = 0, world: int = 1,
                 chunk: int = 1 << 24, batch_cap: int = 0) -> EmbeddingTableGroup:
    """Create the (shard of the) table group and bulk-insert every key of every table,
    in index order, so that on one GPU row i of table t holds table_key(t, i). batch_cap:
    size the per-batch workspaces for up to that many samples (default cfg.batch)."""
    if batch_cap > cfg.batch:
        cfg = W.Config(**{**cfg.__dict__, "batch": batch_cap})
    n_bags = cfg.batch * cfg.n_slots
    max_keys = table_max_keys(cfg, world)
    n_bags_cap = n_bags if world == 1 else max(n_bags * world, max_keys)
    caps = []
    for c in cfg.cards:
        # a hashed table's card is already the per-GPU row pool
        caps.append(c if world == 1 or cfg.keyspace else int(c / world * 1.02 + 64 * math.sqrt(c / world + 1) + 64))
    g = EmbeddingTableGroup(ctx, caps, cfg.dim, cfg.slots() if world == 1 else list(range(len(cfg.cards))),
                            cfg.optimizer, max_batch_keys=max_keys, max_batch_bags=n_bags_cap, init_seed=cfg.seed)
    if cfg.keyspace:  # hashed table: rows materialise on first touch (HPS_LOOKUP_INSERT)
        return g
    for t, c in enumerate(cfg.cards):
        for first in range(0, c, chunk):
            n = min(chunk, c - first)
            g.insert(t, _owned_keys(ctx, cfg, t, rank, world, first, n), return_rows=False)
    ctx.sync()
    return g


def localized_plan(cfg: W.Config, world: int, budget_bytes: int = 170 * 10**9) -> List[List[int]]:
    """Owner of every slot under localized placement: LPT over whole tables by bytes
    (hps_plan_localized), so slots sharing a table share its owner.
    Returns owned[g] = the slots rank g serves, ascending."""
    from .placement import SlotSpec, plan_localized
    n_state = {"sgd": 0, "adagrad": 1, "adam": 2}[cfg.optimizer]
    # the planner sizes vocab x dim x 4 B; optimizer state scales the effective dim
    specs = [SlotSpec(c, cfg.dim * (1 + n_state), cfg.hot) for c in cfg.cards]
    owner_of_table = plan_localized(specs, [budget_bytes] * world)
    slots = cfg.slots()
    return [[s for s in range(len(slots)) if owner_of_table[slots[s]] == g] for g in range(world)]


def build_tables_localized(ctx: Context, cfg: W.Config, owned: List[List[int]], rank: int, world: int,
                           chunk: int = 1 << 24) -> Optional[EmbeddingTableGroup]:
    """The whole tables this rank owns (local table j = my_tables[j]); None if it owns none."""
    slots = cfg.slots()
    mine = owned[rank]
    if not mine:
        return None
    my_tables = sorted({slots[s] for s in mine})
    local_slot_table = [my_tables.index(slots[s]) for s in mine]
    n_local = table_max_keys(cfg, 1)
    g = EmbeddingTableGroup(ctx, [cfg.cards[t] for t in my_tables], cfg.dim, local_slot_table, cfg.optimizer,
                            max_batch_keys=n_local * world, max_batch_bags=cfg.batch * len(mine) * world,
                            init_seed=cfg.seed)
    for j, t in enumerate(my_tables):
        c = cfg.cards[t]
        for first in range(0, c, chunk):
            g.insert(j, ctx.gen_keys(W.table_seed(cfg.seed, t), first, min(chunk, c - first)), return_rows=False)
    ctx.sync()
    return g


def hybrid_hot_set(cfg: W.Config, hot_budget_bytes: int, sample_steps: int = 4) -> List[np.ndarray]:
    """Hot keys per table (SPEC.md:492-496 plan_hybrid): keys ranked by frequency over
    `sample_steps` synthetic batches (count desc; ties by table then key asc), taken while
    the replicated rows (weights + optimizer state) fit hot_budget_bytes per device."""
    gen = W.BatchGen(cfg)
    n_state = {"sgd": 0, "adagrad": 1, "adam": 2}[cfg.optimizer]
    row_bytes = cfg.dim * 4 * (1 + n_state)
    ks, ts = [], []
    for s in range(sample_steps):
        k, _, _, tab = gen.batch(10_000 + s)
        ks.append(k)
        ts.append(tab.astype(np.int64))
    k, t = np.concatenate(ks), np.concatenate(ts)
    pair = np.stack([t.astype(np.uint64), k]).T
    uniq, counts = np.unique(pair, axis=0, return_counts=True)
    order = np.lexsort((uniq[:, 1], uniq[:, 0], -counts))  # count desc, then (table, key) asc
    take = order[: max(0, hot_budget_bytes // row_bytes)]
    hot = uniq[take]
    return [np.sort(hot[hot[:, 0] == i, 1]) for i in range(len(cfg.cards))]


def build_tables_hybrid(ctx: Context, cfg: W.Config, rank: int, world: int, hot_keys: List[np.ndarray],
                        chunk: int = 1 << 24):
    """(hot replica group, cold shard group): the hot keys of every table on every rank;
    every other key on its owner partition_of(key, G)."""
    n_bags = cfg.batch * cfg.n_slots
    max_keys = table_max_keys(cfg, world)
    hot_caps = [max(1, len(h)) for h in hot_keys]
    hot = EmbeddingTableGroup(ctx, hot_caps, cfg.dim, cfg.slots(), cfg.optimizer, max_batch_keys=table_max_keys(cfg, 1),
                              max_batch_bags=n_bags, init_seed=cfg.seed)
    caps = [int(c / world * 1.02 + 64 * math.sqrt(c / world + 1) + 64) for c in cfg.cards]
    cold = EmbeddingTableGroup(ctx, caps, cfg.dim, list(range(len(cfg.cards))), cfg.optimizer,
                               max_batch_keys=max_keys, max_batch_bags=max(n_bags * world, max_keys),
                               init_seed=cfg.seed)
    for t, c in enumerate(cfg.cards):
        hk = torch.from_numpy(hot_keys[t].view(np.int64)).cuda()
        if hk.numel():
            hot.insert(t, hk, return_rows=False)
        for first in range(0, c, chunk):
            keys = _owned_keys(ctx, cfg, t, rank, world, first, min(chunk, c - first))
            if hk.numel():
                keys = keys[~torch.isin(keys, hk)]
            cold.insert(t, keys, return_rows=False)
    ctx.sync()
    return hot, cold


class CabiDistExchange:
    """Distributed-slot exchange through the C-ABI (hps_gpu_dist_*, sharded.cu): the
    NCCL communicator lives in the context (rank 0's id broadcast over torch.distributed)."""

    def __init__(self, ctx: Context, table: EmbeddingTableGroup, cfg: W.Config, rank: int, world: int,
                 insert_missing: bool = False):
        from .api import DistTable
        if world > 1:
            import torch.distributed as dist
            obj = [Context.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            ctx.comm_init(obj[0], rank, world)
        self.world, self.cfg, self.insert_missing = world, cfg, insert_missing
        self.combiner = cfg.combiner
        self.dt = DistTable(ctx, table, cfg.slots(), table_max_keys(cfg, 1), cfg.batch * cfg.n_slots)
        self.out = torch.empty(cfg.batch * cfg.n_slots, cfg.dim, dtype=torch.float32, device="cuda")
        self.last_recv = 0

    def forward(self, keys, offs, n_bags, train=True):
        self.dt.forward(keys, n_bags // self.dt.n_slots, offsets=offs, combiner=self.combiner, train=train,
                        insert_missing=self.insert_missing, out=self.out)
        return self.out

    def backward(self, dout, params):
        self.dt.backward(dout, params)

    def exchanged_bytes(self, dim: int) -> int:
        """Bytes this rank sends to its peers per step: keys + table ids, rows, gradients
        (fixed-capacity regions, so independent of the batch)."""
        C_ = self.dt.capacity
        return (self.world - 1) * C_ * (8 + 4 + 2 * dim * 4)


class TrainStep:
    """One fwd+bwd+update step over a staged batch. world == 1 runs the fused path
    (2 C-ABI calls, optionally replayed as one CUDA graph); world > 1 runs the
    distributed or localized exchange (paper_2210_08803_b200.exchange)."""

    def __init__(self, ctx: Context, table: Optional[EmbeddingTableGroup], cfg: W.Config, rank: int = 0,
                 world: int = 1, use_graph: bool = True, owned: Optional[List[List[int]]] = None,
                 hybrid_hot: Optional[EmbeddingTableGroup] = None, force_exchange: bool = False,
                 pipeline: bool = False, cabi: bool = True, transport: str = "nccl"):
        """owned (world > 1): localized placement, owned[g] = slots of rank g (localized_plan);
        None = distributed placement."""
        self.ctx, self.table, self.cfg, self.rank, self.world = ctx, table, cfg, rank, world
        multi = world > 1 or force_exchange  # force_exchange: the exchange path on a world of one
        self.placement = ("single" if not multi else "localized" if owned is not None
                          else "hybrid" if hybrid_hot is not None else "distributed")
        self.n_bags = cfg.batch * cfg.n_slots
        self.out = torch.empty(self.n_bags, cfg.dim, dtype=torch.float32, device="cuda")
        self.params = opt_params(cfg.optimizer, cfg.lr, eps=cfg.eps)
        self.insert_missing = bool(cfg.keyspace)
        self.graph_mode = bool(use_graph and world == 1)
        # Adam in a graph: the bias-corrected lr_t of each step (host fp32, as the oracle) is
        # copied into a device scalar the kernels read (hps_opt_params.lr_t_device)
        self._lr_dev = torch.zeros(1, dtype=torch.float32, device="cuda")
        self._lr_ring = torch.zeros(64, dtype=torch.float32).pin_memory()
        self._lr_ev = [None] * 64
        self._graphs = {}
        # training record + dedup (backward.cu launch_dedup): probe, dedup, long-list histogram,
        # its radix passes, long registration, long tasks; backward: short + long reduce
        rec = 2 + long_sort_passes(table_max_keys(cfg, 1))  # probe, dedup (persistent kernel), sort passes
        self.kernels_per_step = rec + 1 + 2  # + pooling
        self._cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        self._cnt_host = torch.zeros(1, dtype=torch.int64).pin_memory()
        # pipelined e2e (run_host_async): one pinned result slot + event per step in flight
        self._cnt_slots = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(2)]
        self._slot_ev = [torch.cuda.Event() for _ in range(2)]
        self.exchange = None
        if multi and owned is not None:
            from .exchange import LocalizedExchange, LocalizedGpuEngine
            self.engine = LocalizedGpuEngine(ctx, table, cfg.n_slots, owned, cfg.batch, table_max_keys(cfg, 1), cfg.dim)
            self.exchange = LocalizedExchange(self.engine, cfg.combiner, rank, world, cfg.n_slots, owned)
            multi = cfg.hot > 1
            # regroup (lengths + scan + keys) per owner [+ owner offsets] + training lookup
            # (record + dedup + pooling) + place per owner + place(1) per owner + backward (2)
            self.kernels_per_step = 3 * world + (1 if multi else 0) + rec + 1 + 2 * world + 2
        elif multi and hybrid_hot is not None:
            from .exchange import GpuEngine, HybridExchange, HybridGpuEngine
            cold_engine = GpuEngine(ctx, table, cfg.slots(), table_max_keys(cfg, 1), world)
            self.engine = HybridGpuEngine(ctx, hybrid_hot, cold_engine, table_max_keys(cfg, 1))
            self.exchange = HybridExchange(self.engine, cfg.combiner, rank, world, cfg.n_slots)
            # hot record + dedup + cold scan + bucketize(5) + cold gather (record + dedup + pooling)
            # + pool + cold grads + cold backward(2) + hot reduce(2) + sum_partials + apply
            self.kernels_per_step = rec + 1 + 5 + rec + 1 + 1 + 1 + 2 + 2 + 2
        elif multi and cabi:
            # distributed slot through the C-ABI (sharded.cu): NCCL inside libhps_gpu, fixed
            # per-peer regions, no host sync, so the step is replayed as one CUDA graph
            self.exchange = CabiDistExchange(ctx, table, cfg, rank, world, self.insert_missing)
            self.exchange.dt.set_transport(transport)
            self.placement = "distributed"
            self.graph_mode = bool(use_graph)
            self.kernels_per_step = 5 + 1 + rec + 1 + 1 + 1 + 2 + (1 if cfg.hot > 1 else 0)
        elif multi:
            from .exchange import DistributedExchange, GpuEngine
            max_keys = table_max_keys(cfg, 1)
            self.engine = GpuEngine(ctx, table, cfg.slots(), max_keys, world, insert_missing=self.insert_missing)
            self.exchange = DistributedExchange(self.engine, cfg.combiner, rank, world)
            # bucketize (owner + hist + 1 radix pass + pack + counts) + owner gather (record +
            # dedup + pooling) + pool + scatter + backward (2) [+ occ_bags]
            self.kernels_per_step = 5 + rec + 1 + 1 + 1 + 2 + (1 if cfg.hot > 1 else 0)
        if self.insert_missing:  # claim + scan + commit + finish
            self.kernels_per_step += 4
        # Batch pipelining (single path): the record + dedup of batch i+1 (prefetch, on the
        # table's slot stream) overlap batch i's pooling + backward; run(..., next_b=) names
        # batch i+1. +1 kernel: the step's unique-row count (k_unique_count) into self._cnt.
        import os
        if os.environ.get("HPS_PIPELINE") == "0":  # A/B knob
            pipeline = False
        self.pipeline = bool(pipeline and self.exchange is None and table is not None)
        if self.pipeline:
            table.set_pipeline(2)
            self.kernels_per_step += 1
        self._pre = None        # (batch dict, slot) prefetched and not yet consumed
        self._free_slot = 0     # slot the next eager prefetch goes to
        self._warmed = False    # the first pipelined step runs eagerly (module loading)
        self._pipe_stage = None

    # -- inputs -------------------------------------------------------------------------
    def stage_batch(self, keys: np.ndarray, offs: Optional[np.ndarray]):
        k = torch.from_numpy(np.ascontiguousarray(keys).view(np.int64)).cuda()
        o = None if offs is None else torch.from_numpy(np.ascontiguousarray(offs).view(np.int32)).cuda()
        return {"keys": k, "offs": o, "n_keys": int(len(keys))}

    def stage_host(self, keys: np.ndarray, offs: Optional[np.ndarray]):
        k = torch.from_numpy(np.ascontiguousarray(keys).view(np.int64)).pin_memory()
        o = None if offs is None else torch.from_numpy(np.ascontiguousarray(offs).view(np.int32)).pin_memory()
        return {"keys": k, "offs": o, "n_keys": int(len(keys))}

    # -- the step --------------------------------------------------------------------------
    def _prep_step(self, step: int) -> None:
        """Adam: this step's lr_t into the device scalar (a pinned ring slot -> async copy,
        stream-ordered before the step's kernels)."""
        if self.cfg.optimizer != "adam":
            return
        k = step % self._lr_ring.numel()
        if self._lr_ev[k] is not None:
            self._lr_ev[k].synchronize()  # the copy that last read this pinned slot has run
        self._lr_ring[k] = float(opt_params("adam", self.cfg.lr, eps=self.cfg.eps, step=step).lr_t)
        self._lr_dev.copy_(self._lr_ring[k:k + 1], non_blocking=True)
        self._lr_ev[k] = torch.cuda.Event()
        self._lr_ev[k].record()

    def _eager(self, b, dout, step, keys_on_host=False):
        if self.cfg.optimizer == "adam":
            self.params = opt_params("adam", self.cfg.lr, eps=self.cfg.eps, step=step)
            if self.graph_mode:
                self.params.lr_t_device = self._lr_dev.data_ptr()
        self.table.lookup(b["keys"], self.cfg.batch, offsets=b["offs"], combiner=self.cfg.combiner, train=True,
                          out=self.out, keys_on_host=keys_on_host, insert_missing=self.insert_missing)
        self.table.backward_update(dout, self.cfg.lr, params=self.params)

    def _exchange_step(self, keys, offs, dout, step, graph=True):
        if isinstance(self.exchange, CabiDistExchange):
            self._prep_step(step)
            self._adam_params(step)

            def body():
                self.out = self.exchange.forward(keys, offs, self.n_bags, train=True)
                self.exchange.backward(dout, self.params)
            if self.graph_mode and graph:
                return self._graph(("dist", id(keys), id(offs), id(dout)), body)
            return body()
        if self.cfg.optimizer == "adam":
            self.params = opt_params("adam", self.cfg.lr, eps=self.cfg.eps, step=step)
        n = self.cfg.batch if self.placement in ("localized", "hybrid") else self.n_bags
        self.out = self.exchange.forward(keys, offs, n, train=True)
        self.exchange.backward(dout, self.params)

    def _graph(self, key, fn):
        """Capture fn() once per key as a CUDA graph (warm-up run outside the capture for lazy
        module loading) and replay it."""
        g = self._graphs.get(key)
        if g is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.ctx.set_stream(s)
                fn()  # this call's step (capture below records without executing)
                dump = os.environ.get("HPS_GRAPH_DUMP")  # debug: the captured graph as DOT
                g = torch.cuda.CUDAGraph(keep_graph=bool(dump))
                if dump:
                    g.enable_debug_mode()
                with torch.cuda.graph(g, stream=s):
                    fn()
                if dump:
                    g.debug_dump(f"{dump}_{len(self._graphs)}.dot")
            torch.cuda.current_stream().wait_stream(s)
            self.ctx.set_stream(torch.cuda.current_stream())
            self._graphs[key] = g
            return
        g.replay()

    # -- pipelined step (hps_gpu_table_prefetch) ----------------------------------------------
    def _adam_params(self, step):
        if self.cfg.optimizer == "adam":
            self.params = opt_params("adam", self.cfg.lr, eps=self.cfg.eps, step=step)
            if self.graph_mode:
                self.params.lr_t_device = self._lr_dev.data_ptr()

    def _prefetch(self, slot, nb, keys_on_host):
        self.table.prefetch(slot, nb["keys"], self.cfg.batch, offsets=nb["offs"], combiner=self.cfg.combiner,
                            keys_on_host=keys_on_host, insert_missing=self.insert_missing)

    def _pipe_body(self, b, nb, dout, slot, keys_on_host=False, result=None):
        """prefetch(nb -> other slot) ; lookup(slot) ; backward ; unique count ; join."""
        if nb is not None:
            self._prefetch(1 - slot, nb, keys_on_host)
        offs = None if (keys_on_host or b["offs"] is None) else b["offs"]
        self.table.lookup_prefetched(slot, self.cfg.batch, offsets=offs, combiner=self.cfg.combiner, out=self.out)
        self.table.backward_update(dout, self.cfg.lr, params=self.params)
        L.check(self.ctx.lib.hps_gpu_table_last_unique(self.table.h, _ptr(self._cnt), None), "last_unique")
        if result is not None:
            result.copy_(self._cnt, non_blocking=True)
        if nb is not None:
            self.table.join_prefetch()

    def _run_pipe(self, b, dout, step, nb, keys_on_host=False, result=None, tag="dev"):
        """One pipelined step. Host state advances exactly once per call: eagerly, or by the
        capture of a graph that is then replayed (replays of captured graphs leave it alone)."""
        self._adam_params(step)
        if self._pre is None or self._pre[0] is not b:  # b was not prefetched by the previous step
            self._prefetch(self._free_slot, b, keys_on_host)
            self.table.join_prefetch()
            self._pre = (b, self._free_slot)
        slot = self._pre[1]
        if self.insert_missing and nb is not None and not keys_on_host:
            # a dynamic table streams fresh batches: the next batch's keys go to a per-slot
            # device staging buffer (D2D before the replay), one graph per slot parity
            if self._pipe_stage is None:
                self._pipe_stage = [torch.empty(table_max_keys(self.cfg, 1), dtype=torch.int64, device="cuda")
                                    for _ in range(2)]
            buf = self._pipe_stage[1 - slot][:nb["keys"].numel()]
            buf.copy_(nb["keys"], non_blocking=True)
            nb_g = {"keys": buf, "offs": nb["offs"], "n_keys": nb["n_keys"]}
            key = (tag, "stage", slot, nb["keys"].numel(), id(dout), id(result))
        else:
            nb_g = nb
            key = (tag, id(b["keys"]), None if nb is None else id(nb["keys"]), id(dout), slot, id(result))
        if not self.graph_mode or not self._warmed or nb is None:
            self._pipe_body(b, nb_g, dout, slot, keys_on_host, result)
            self._warmed = True
        else:
            g = self._graphs.get(key)
            if g is None:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    self.ctx.set_stream(s)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s):
                        self._pipe_body(b, nb_g, dout, slot, keys_on_host, result)
                torch.cuda.current_stream().wait_stream(s)
                self.ctx.set_stream(torch.cuda.current_stream())
                self._graphs[key] = g
            g.replay()
        if nb is None:
            self._pre, self._free_slot = None, 1 - slot
        else:
            self._pre, self._free_slot = (nb, 1 - slot), slot

    def run(self, b, dout, step: int = 1, next_b=None):
        self._last_n = b["n_keys"]
        if self.exchange is None:
            self._prep_step(step)
        if self.exchange is not None:
            return self._exchange_step(b["keys"], b["offs"], dout, step)
        if self.pipeline:
            return self._run_pipe(b, dout, step, next_b)
        if not self.graph_mode:
            return self._eager(b, dout, step)
        if self.insert_missing and b["offs"] is None:
            # a dynamic table streams fresh batches: one graph over a device staging buffer
            # (a D2D copy of the keys precedes each replay) instead of one capture per batch
            if not hasattr(self, "_stage_keys"):
                self._stage_keys = torch.empty(self.n_bags, dtype=torch.int64, device="cuda")
            self._stage_keys[:b["keys"].numel()].copy_(b["keys"], non_blocking=True)
            sb = {"keys": self._stage_keys[:b["keys"].numel()], "offs": None, "n_keys": b["n_keys"]}
            self._graph(("stage", sb["keys"].numel(), id(dout)), lambda: self._eager(sb, dout, step))
            return
        self._graph((id(b["keys"]), id(dout)), lambda: self._eager(b, dout, step))

    def _host_step(self, b, dout, step, out=None):
        self._eager(b, dout, step, keys_on_host=True)
        L.check(self.ctx.lib.hps_gpu_table_last_unique(self.table.h, _ptr(self._cnt), None), "last_unique")
        (self._cnt_host if out is None else out).copy_(self._cnt, non_blocking=True)

    def run_host_async(self, b, dout, step: int, slot: int, next_b=None):
        """End-to-end step from pinned HOST keys, pipelined one step deep: the keys go H2D on a
        copy stream into device staging slot `slot` (while the previous step computes), the
        step (kernels + the D2H of its result into pinned slot `slot`) follows on the main
        stream; read_host_result(slot) waits for it. Every step moves its inputs H2D and its
        result D2H inside the timed region; the copies overlap the previous step's kernels."""
        h2d = b["keys"].numel() * 8 + (0 if b["offs"] is None else b["offs"].numel() * 4)
        multi = b["offs"] is not None
        if self.pipeline and next_b is not None:
            # pipelined: the NEXT batch's pinned keys (+ offsets) go H2D inside its prefetch, on
            # the slot stream, overlapping this batch's pooling + update; the step's result (unique
            # rows, 8 B) goes D2H into pinned slot `slot`
            self._prep_step(step)
            self._last_n = b["n_keys"]
            self._run_pipe(b, dout, step, next_b, keys_on_host=True, result=self._cnt_slots[slot], tag="host")
            self._slot_ev[slot].record()
            nb = next_b
            return nb["keys"].numel() * 8 + (0 if nb["offs"] is None else nb["offs"].numel() * 4), 8
        if self.exchange is not None or not self.graph_mode or (multi and self.insert_missing):
            self.run_host(b, dout, step)
            self._cnt_slots[slot].copy_(self._cnt_host)
            self._slot_ev[slot].record()
            return h2d, 8
        self._prep_step(step)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream()
            nk = max(self.n_bags, table_max_keys(self.cfg, 1))
            self._dev_keys = [torch.empty(nk, dtype=torch.int64, device="cuda") for _ in range(2)]
            # multi-hot: the bag offsets travel too; the graph's kernels read sizes from them
            self._dev_offs = [torch.empty(self.n_bags + 1, dtype=torch.int32, device="cuda") for _ in range(2)]
            self._copy_ev = [torch.cuda.Event() for _ in range(2)]
        main = torch.cuda.current_stream()
        with torch.cuda.stream(self._copy_stream):
            self._copy_stream.wait_event(self._slot_ev[slot])  # the slot's previous step is done with it
            self._dev_keys[slot][:b["keys"].numel()].copy_(b["keys"], non_blocking=True)
            if multi:
                self._dev_offs[slot].copy_(b["offs"], non_blocking=True)
            self._copy_ev[slot].record()
        main.wait_event(self._copy_ev[slot])
        dk = {"keys": self._dev_keys[slot], "offs": self._dev_offs[slot] if multi else None, "n_keys": b["n_keys"]}
        out = self._cnt_slots[slot]

        def dev_step():
            self._eager(dk, dout, step)
            L.check(self.ctx.lib.hps_gpu_table_last_unique(self.table.h, _ptr(self._cnt), None), "last_unique")
            out.copy_(self._cnt, non_blocking=True)

        self._graph(("dev", slot, id(dout)), dev_step)
        self._slot_ev[slot].record()
        return h2d, 8

    def read_host_result(self, slot: int) -> int:
        self._slot_ev[slot].synchronize()
        return int(self._cnt_slots[slot][0])

    def run_host(self, b, dout, step: int = 1):
        """End-to-end through the C-ABI: keys from pinned host memory (H2D inside the call),
        and a D2H read of the step's result (the number of rows updated). One-hot steps replay
        the whole thing (H2D copy node -> kernels -> D2H copy node) as one CUDA graph per
        pinned input buffer; the caller refills that buffer between steps."""
        h2d = b["keys"].numel() * 8 + (0 if b["offs"] is None else b["offs"].numel() * 4)
        if self.exchange is None:
            self._prep_step(step)
        if self.exchange is not None:
            keys = b["keys"].to("cuda", non_blocking=True)
            offs = None if b["offs"] is None else b["offs"].to("cuda", non_blocking=True)
            self._exchange_step(keys, offs, dout, step, graph=False)
            _ = self._unique_count()
            return h2d, 8
        if self.graph_mode and b["offs"] is None:
            self._graph(("host", id(b["keys"]), id(dout)), lambda: self._host_step(b, dout, step))
        else:
            self._host_step(b, dout, step)
        torch.cuda.current_stream().synchronize()
        _ = int(self._cnt_host[0])
        return h2d, 8

    def _unique_count(self) -> int:
        """Rows the last backward updated on this rank (D2H read of the step's result)."""
        if self.table is None:  # localized rank that owns no slot
            torch.cuda.current_stream().synchronize()
            return 0
        if self.pipeline:  # every pipelined step writes its count into self._cnt
            return int(self._cnt.item())
        self.ctx.lib.hps_gpu_table_last_unique(self.table.h, self._cnt.data_ptr(), None)
        return int(self._cnt.item())

    def last_counts(self):
        return self._last_n, self._unique_count()

    def lookup_only(self, b):
        if self.exchange is not None:
            n = self.cfg.batch if self.placement in ("localized", "hybrid") else self.n_bags
            self.exchange.forward(b["keys"], b["offs"], n, train=False)
            return
        self.table.lookup(b["keys"], self.cfg.batch, offsets=b["offs"], combiner=self.cfg.combiner, train=False,
                          out=self.out)  # roofline leg: batches were materialised by the timed steps
