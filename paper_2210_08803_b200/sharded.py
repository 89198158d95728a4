"""Table construction and the training step used by bench.py (1..8 GPUs).

Single GPU: one table group holds every table. Multi-GPU (distributed slot sharding,
SPEC.md:487-491): rank r owns the keys with partition_of(key, G) == r;
the exchange lives in paper_2210_08803_b200.exchange.
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np
import torch

from . import workload as W
from .api import Context, EmbeddingTableGroup, opt_params


def _owned_keys(ctx: Context, cfg: W.Config, t: int, rank: int, world: int, first: int, n: int) -> torch.Tensor:
    keys = ctx.gen_keys(W.table_seed(cfg.seed, t), first, n)
    if world > 1:
        keys = keys[ctx.partition_of(keys, world) == rank]
    return keys


def table_max_keys(cfg: W.Config, world: int) -> int:
    """Key occurrences one rank may have to hold in a step (an owner can receive every
    rank's keys in the worst case)."""
    n_bags = cfg.batch * cfg.n_slots
    return n_bags * (2 * cfg.hot - 1 if cfg.hot > 1 else 1) * world


def build_tables(ctx: Context, cfg: W.Config, rank: int = 0, world: int = 1,
                 chunk: int = 1 << 24) -> EmbeddingTableGroup:
    """Create the (shard of the) table group and bulk-insert every key of every table,
    in index order, so that on one GPU row i of table t holds table_key(t, i)."""
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
            g.insert(t, _owned_keys(ctx, cfg, t, rank, world, first, n))
    ctx.sync()
    return g


class TrainStep:
    """One fwd+bwd+update step over a staged batch. world == 1 runs the fused path
    (2 C-ABI calls, optionally replayed as one CUDA graph); world > 1 runs the
    distributed exchange (paper_2210_08803_b200.exchange)."""

    def __init__(self, ctx: Context, table: EmbeddingTableGroup, cfg: W.Config, rank: int = 0, world: int = 1,
                 use_graph: bool = True):
        self.ctx, self.table, self.cfg, self.rank, self.world = ctx, table, cfg, rank, world
        self.n_bags = cfg.batch * cfg.n_slots
        self.out = torch.empty(self.n_bags, cfg.dim, dtype=torch.float32, device="cuda")
        self.params = opt_params(cfg.optimizer, cfg.lr, eps=cfg.eps)
        self.insert_missing = bool(cfg.keyspace)
        self.graph_mode = bool(use_graph and world == 1 and cfg.optimizer != "adam")
        self._graphs = {}
        # lookup + dedup scan + scatter + short reduce + long sort/chunks/combine
        self.kernels_per_step = 7
        self._cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.exchange = None
        if world > 1:
            from .exchange import DistributedExchange, GpuEngine
            max_keys = table_max_keys(cfg, 1)
            self.engine = GpuEngine(ctx, table, cfg.slots(), max_keys, world, insert_missing=self.insert_missing)
            self.exchange = DistributedExchange(self.engine, cfg.combiner, rank, world)
            # bucketize (owner + hist + 1 radix pass + pack + counts) + gather + pool
            # + scatter + backward (hist + passes + scan + 3 reduce kernels) [+ occ_bags]
            self.kernels_per_step = 5 + 1 + 1 + 1 + 7 + (1 if cfg.hot > 1 else 0)
        if self.insert_missing:  # claim + scan + commit + finish
            self.kernels_per_step += 4

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
    def _eager(self, b, dout, step, keys_on_host=False):
        if self.cfg.optimizer == "adam":
            self.params = opt_params("adam", self.cfg.lr, eps=self.cfg.eps, step=step)
        self.table.lookup(b["keys"], self.cfg.batch, offsets=b["offs"], combiner=self.cfg.combiner, train=True,
                          out=self.out, keys_on_host=keys_on_host, insert_missing=self.insert_missing)
        self.table.backward_update(dout, self.cfg.lr, params=self.params)

    def _exchange_step(self, keys, offs, dout, step):
        if self.cfg.optimizer == "adam":
            self.params = opt_params("adam", self.cfg.lr, eps=self.cfg.eps, step=step)
        self.out = self.exchange.forward(keys, offs, self.n_bags, train=True)
        self.exchange.backward(dout, self.params)

    def run(self, b, dout, step: int = 1):
        self._last_n = b["n_keys"]
        if self.exchange is not None:
            return self._exchange_step(b["keys"], b["offs"], dout, step)
        if not self.graph_mode:
            return self._eager(b, dout, step)
        key = (id(b["keys"]), id(dout))
        g = self._graphs.get(key)
        if g is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.ctx.set_stream(s)
                self._eager(b, dout, step)  # warm: lazy module loading outside capture
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self._eager(b, dout, step)
            torch.cuda.current_stream().wait_stream(s)
            self.ctx.set_stream(torch.cuda.current_stream())
            self._graphs[key] = g
        g.replay()

    def run_host(self, b, dout, step: int = 1):
        """End-to-end through the C-ABI: keys from pinned host memory (H2D inside the call),
        and a D2H read of the step's result (the number of rows updated)."""
        if self.exchange is not None:
            keys = b["keys"].to("cuda", non_blocking=True)
            offs = None if b["offs"] is None else b["offs"].to("cuda", non_blocking=True)
            self._exchange_step(keys, offs, dout, step)
            self.ctx.lib.hps_gpu_table_last_unique(self.table.h, self._cnt.data_ptr(), None)
            _ = int(self._cnt.item())
            h2d = b["keys"].numel() * 8 + (0 if b["offs"] is None else b["offs"].numel() * 4)
            return h2d, 8
        self._eager(b, dout, step, keys_on_host=True)
        self.ctx.lib.hps_gpu_table_last_unique(self.table.h, self._cnt.data_ptr(), None)
        _ = int(self._cnt.item())
        h2d = b["keys"].numel() * 8 + (0 if b["offs"] is None else b["offs"].numel() * 4)
        return h2d, 8

    def last_counts(self):
        self.ctx.lib.hps_gpu_table_last_unique(self.table.h, self._cnt.data_ptr(), None)
        return self._last_n, int(self._cnt.item())

    def lookup_only(self, b):
        if self.exchange is not None:
            self.exchange.forward(b["keys"], b["offs"], self.n_bags, train=False)
            return
        self.table.lookup(b["keys"], self.cfg.batch, offsets=b["offs"], combiner=self.cfg.combiner, train=False,
                          out=self.out)  # roofline leg: batches were materialised by the timed steps
