"""Python host API over the C-ABI: device memory and streams come from torch.

This is the harness-facing mirror of the boundary (include/hps_gpu.h). Every call
goes straight to libhps_gpu.so; there is no CPU path. Keys travel as int64 tensors
holding the uint64 bit pattern (hps::EmbeddingKey, any 64-bit value is legal).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from ._lib import HpsError

_OPT = {"sgd": L.OPT_SGD, "adagrad": L.OPT_ADAGRAD, "adam": L.OPT_ADAM}
_COMB = {"sum": L.COMBINER_SUM, "mean": L.COMBINER_MEAN}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


class Context:
    """hps_gpu_ctx: a device, a stream and the latched device status word."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        self.lib = L.load()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h)), "ctx_create")
        self.h = h

    def set_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        L.check(self.lib.hps_gpu_ctx_set_stream(self.h, C.c_void_p(stream.cuda_stream)), "ctx_set_stream")

    def sync(self) -> None:
        """Wait for the stream; raise HpsError if a kernel latched an error."""
        L.check(self.lib.hps_gpu_ctx_sync(self.h), "ctx_sync")

    def status(self) -> int:
        return self.lib.hps_gpu_ctx_sync(self.h)

    def key_hash(self, keys: torch.Tensor) -> torch.Tensor:
        _need_cuda(keys, "keys")
        out = torch.empty_like(keys)
        L.check(self.lib.hps_gpu_key_hash(self.h, _ptr(keys), keys.numel(), _ptr(out)), "key_hash")
        return out

    def partition_of(self, keys: torch.Tensor, num_shards: int) -> torch.Tensor:
        _need_cuda(keys, "keys")
        out = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
        L.check(self.lib.hps_gpu_partition_of(self.h, _ptr(keys), keys.numel(), num_shards, _ptr(out)), "partition_of")
        return out

    def has_non_finite(self, x: torch.Tensor) -> bool:
        _need_cuda(x, "x")
        flag = torch.empty(1, dtype=torch.int32, device=x.device)
        L.check(self.lib.hps_gpu_has_non_finite_f32(self.h, _ptr(x), x.numel(), _ptr(flag)), "has_non_finite")
        return bool(flag.item())

    # -- NCCL communicator of the sharded C-ABI path (sharded.cu) --------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(L.NCCL_ID_BYTES)
        L.check(L.load().hps_gpu_nccl_unique_id(buf), "nccl_unique_id")
        return buf.raw

    def comm_init(self, unique_id: bytes, rank: int, world: int) -> None:
        buf = C.create_string_buffer(bytes(unique_id), L.NCCL_ID_BYTES)
        L.check(self.lib.hps_gpu_ctx_comm_init(self.h, buf, rank, world), "ctx_comm_init")

    # -- the reference's kernel API on the device (proj/include/hps/kernels.hpp:33-43) ---------
    def f32_to_f16(self, x: torch.Tensor) -> torch.Tensor:
        out = torch.empty(x.numel(), dtype=torch.int16, device=x.device)
        L.check(self.lib.hps_gpu_f32_to_f16(self.h, _ptr(x), _ptr(out), x.numel()), "f32_to_f16")
        return out

    def f16_to_f32(self, bits: torch.Tensor) -> torch.Tensor:
        out = torch.empty(bits.numel(), dtype=torch.float32, device=bits.device)
        L.check(self.lib.hps_gpu_f16_to_f32(self.h, _ptr(bits), _ptr(out), bits.numel()), "f16_to_f32")
        return out

    def has_non_finite_f16(self, bits: torch.Tensor) -> bool:
        flag = torch.zeros(1, dtype=torch.int32, device=bits.device)
        L.check(self.lib.hps_gpu_has_non_finite_f16(self.h, _ptr(bits), bits.numel(), _ptr(flag)), "non_finite_f16")
        return bool(flag.item())

    def crc32c(self, data: torch.Tensor, crc: int = 0) -> int:
        """CRC-32C of a uint8 device buffer, continuing from `crc` (kernels.hpp:38-39)."""
        tmp = torch.zeros(2, dtype=torch.int32, device=data.device)
        L.check(self.lib.hps_gpu_crc32c(self.h, crc, _ptr(data), data.numel(), _ptr(tmp),
                                        C.c_void_p(tmp.data_ptr() + 4)), "crc32c")
        return int(tmp[1].item()) & 0xFFFFFFFF

    def crc32c_batch(self, data: torch.Tensor, offsets: torch.Tensor) -> torch.Tensor:
        n = offsets.numel() - 1
        out = torch.empty(max(n, 1), dtype=torch.int32, device=data.device)
        L.check(self.lib.hps_gpu_crc32c_batch(self.h, _ptr(data), _ptr(offsets), n, _ptr(out)), "crc32c_batch")
        return out[:n]

    def gen_keys(self, seed: int, first: int, n: int) -> torch.Tensor:
        out = torch.empty(n, dtype=torch.int64, device=f"cuda:{self.device}")
        L.check(self.lib.hps_gpu_gen_keys(self.h, seed, first, n, _ptr(out)), "gen_keys")
        return out

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_gpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def opt_params(optimizer: str, lr: float, eps: float = 1e-8, beta1: float = 0.9, beta2: float = 0.999,
               step: int = 1) -> L.OptParams:
    """Optimizer constants as the kernels consume them (all fp32)."""
    f = np.float32
    p = L.OptParams()
    p.lr, p.eps, p.beta1, p.beta2 = f(lr), f(eps), f(beta1), f(beta2)
    p.one_minus_beta1 = f(f(1.0) - f(beta1))
    p.one_minus_beta2 = f(f(1.0) - f(beta2))
    if optimizer == "adam":
        p.lr_t = f(lr * math.sqrt(1.0 - beta2 ** step) / (1.0 - beta1 ** step))
    else:
        p.lr_t = f(lr)
    return p


class EmbeddingTableGroup:
    """hps_gpu_table: n_tables key namespaces of one dim, fp32 rows, one optimizer."""

    def __init__(self, ctx: Context, row_capacity: Sequence[int], dim: int, slot_table: Sequence[int],
                 optimizer: str = "sgd", max_batch_keys: int = 1 << 20, max_batch_bags: int = 1 << 20,
                 init_seed: int = 0, adagrad_initial_accumulator: float = 0.0, dtype: str = "f32"):
        """dtype "f16": binary16 rows, an inference table (lookups without training, find,
        export, read-through); insert rounds to nearest even, out-of-range rows -> F16Range."""
        if dtype not in ("f32", "f16"):
            raise HpsError(1, "dtype must be 'f32' or 'f16'")
        self.ctx, self.lib = ctx, ctx.lib
        self.dtype = dtype
        self.dim, self.optimizer = dim, optimizer
        self.n_tables, self.n_slots = len(row_capacity), len(slot_table)
        self.row_capacity = list(row_capacity)
        self.row_base = [int(x) for x in np.concatenate([[0], np.cumsum(row_capacity)[:-1]])]
        caps = (L.u64 * self.n_tables)(*row_capacity)
        st = (L.u32 * self.n_slots)(*slot_table)
        cfg = L.TableConfig(self.n_tables, dim, caps, self.n_slots, st, _OPT[optimizer], max_batch_keys,
                            max_batch_bags, init_seed, adagrad_initial_accumulator, 1 if dtype == "f16" else 0)
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_table_create(ctx.h, C.byref(cfg), C.byref(h)), "table_create")
        self.h = h
        self.device = torch.device(f"cuda:{ctx.device}")

    def insert(self, table: int, keys: torch.Tensor, rows: Optional[torch.Tensor] = None,
               return_rows: bool = True) -> Optional[torch.Tensor]:
        """Insert keys (rows: optional initial values, first occurrence wins). Returns each
        occurrence's local row id, or None with return_rows=False (the faster keys-only load)."""
        _need_cuda(keys, "keys")
        if rows is not None:
            _need_cuda(rows, "rows")
            if rows.dtype != torch.float32 or rows.numel() != keys.numel() * self.dim:
                raise ValueError("rows must be float32 [n, dim]")
        out = torch.empty(keys.numel(), dtype=torch.int64, device=self.device) if return_rows else None
        L.check(self.lib.hps_gpu_table_insert(self.h, table, _ptr(keys), keys.numel(), _ptr(rows), _ptr(out)),
                "table_insert")
        return out

    def find(self, table: int, keys: torch.Tensor) -> torch.Tensor:
        _need_cuda(keys, "keys")
        out = torch.empty(keys.numel(), dtype=torch.int64, device=self.device)
        L.check(self.lib.hps_gpu_table_find(self.h, table, _ptr(keys), keys.numel(), _ptr(out)), "table_find")
        return out

    def size(self, table: int) -> int:
        n = C.c_uint64()
        L.check(self.lib.hps_gpu_table_size(self.h, table, C.byref(n)), "table_size")
        return n.value

    def set_default_vector(self, table: int, vec) -> None:
        v = np.ascontiguousarray(np.asarray(vec, dtype=np.float32).reshape(self.dim))
        L.check(self.lib.hps_gpu_table_set_default_vector(self.h, table, v.ctypes.data_as(C.POINTER(C.c_float))),
                "set_default_vector")

    def export(self, table: int, begin: int, n: int):
        w = torch.empty(n, self.dim, dtype=torch.float32, device=self.device)
        s0 = torch.empty_like(w) if self.optimizer in ("adagrad", "adam") else None
        s1 = torch.empty_like(w) if self.optimizer == "adam" else None
        L.check(self.lib.hps_gpu_table_export(self.h, table, begin, n, _ptr(w), _ptr(s0), _ptr(s1)), "table_export")
        return w, s0, s1

    def row_keys(self, table: int, begin: int, n: int) -> torch.Tensor:
        out = torch.empty(n, dtype=torch.int64, device=self.device)
        L.check(self.lib.hps_gpu_table_row_keys(self.h, table, begin, n, _ptr(out)), "table_row_keys")
        return out

    def lookup(self, keys: torch.Tensor, n_samples: int, offsets: Optional[torch.Tensor] = None,
               combiner: str = "sum", train: bool = False, out: Optional[torch.Tensor] = None,
               keys_on_host: bool = False, insert_missing: bool = False) -> torch.Tensor:
        n_bags = n_samples * self.n_slots
        if out is None:
            out = torch.empty(n_bags, self.dim, dtype=torch.float32, device=self.device)
        flags = (L.LOOKUP_TRAIN if train else 0) | (L.LOOKUP_KEYS_HOST if keys_on_host else 0) | \
            (L.LOOKUP_INSERT if insert_missing else 0)
        if not keys_on_host:
            _need_cuda(keys, "keys")
            if offsets is not None:
                _need_cuda(offsets, "offsets")
        L.check(self.lib.hps_gpu_lookup_pooled(self.h, _ptr(keys), _ptr(offsets), n_samples, _COMB[combiner],
                                               _ptr(out), flags), "lookup_pooled")
        return out

    # -- batch pipelining (hps_gpu_table_set_pipeline / _prefetch / _join_prefetch) --------------
    def set_pipeline(self, depth: int) -> None:
        L.check(self.lib.hps_gpu_table_set_pipeline(self.h, depth), "set_pipeline")

    def prefetch(self, slot: int, keys: torch.Tensor, n_samples: int, offsets: Optional[torch.Tensor] = None,
                 combiner: str = "sum", keys_on_host: bool = False, insert_missing: bool = False) -> None:
        """Record + dedup a future training batch into `slot` on the slot's stream (concurrent
        with whatever is enqueued after this call); lookup_prefetched(slot) consumes it."""
        flags = (L.LOOKUP_KEYS_HOST if keys_on_host else 0) | (L.LOOKUP_INSERT if insert_missing else 0)
        if not keys_on_host:
            _need_cuda(keys, "keys")
            if offsets is not None:
                _need_cuda(offsets, "offsets")
        L.check(self.lib.hps_gpu_table_prefetch(self.h, slot, _ptr(keys), _ptr(offsets), n_samples, _COMB[combiner],
                                                flags), "prefetch")

    def lookup_prefetched(self, slot: int, n_samples: int, offsets: Optional[torch.Tensor] = None,
                          combiner: str = "sum", out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The training lookup of the batch prefetched into `slot` (pooling only)."""
        n_bags = n_samples * self.n_slots
        if out is None:
            out = torch.empty(n_bags, self.dim, dtype=torch.float32, device=self.device)
        flags = L.LOOKUP_TRAIN | L.LOOKUP_PREFETCHED | L.LOOKUP_SLOT(slot)
        L.check(self.lib.hps_gpu_lookup_pooled(self.h, None, _ptr(offsets), n_samples, _COMB[combiner], _ptr(out),
                                               flags), "lookup_pooled(prefetched)")
        return out

    def join_prefetch(self) -> None:
        L.check(self.lib.hps_gpu_table_join_prefetch(self.h), "join_prefetch")

    def batch_table_used(self) -> int:
        """Invariant probe (tests): batch-table entries in use over every slot (0 at rest)."""
        v = C.c_uint64(0)
        L.check(self.lib.hps_gpu_debug_batch_table_used(self.h, C.byref(v)), "debug_batch_table_used")
        return int(v.value)

    def backward_update(self, d_out: torch.Tensor, lr: float, eps: float = 1e-8, beta1: float = 0.9,
                        beta2: float = 0.999, step: int = 1, params: Optional[L.OptParams] = None) -> None:
        _need_cuda(d_out, "d_out")
        p = params if params is not None else opt_params(self.optimizer, lr, eps, beta1, beta2, step)
        L.check(self.lib.hps_gpu_backward_update(self.h, _ptr(d_out), C.byref(p)), "backward_update")

    def last_unique(self) -> torch.Tensor:
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        L.check(self.lib.hps_gpu_table_last_unique(self.h, _ptr(cnt), None), "last_unique(count)")
        n = int(cnt.item())
        rows = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        L.check(self.lib.hps_gpu_table_last_unique(self.h, _ptr(cnt), _ptr(rows)), "last_unique")
        return rows[:n]

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_gpu_table_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HotCache:
    """hps_gpu_cache: the HPS set-associative GPU embedding cache."""

    def __init__(self, ctx: Context, capacity: int, dim: int, ways: int = 8, aging_interval: int = 0,
                 max_batch: int = 1 << 17, dtype: str = "f32"):
        """dtype: storage of the cached rows, "f32" or "f16" (binary16, round-to-nearest-even
        on insert/refresh, exact widening on query; out-of-range rows rejected: F16Range)."""
        if dtype not in ("f32", "f16"):
            raise HpsError(1, "dtype must be 'f32' or 'f16'")
        self.ctx, self.lib, self.dim, self.dtype = ctx, ctx.lib, dim, dtype
        self.device = torch.device(f"cuda:{ctx.device}")
        cfg = L.CacheConfig(capacity, ways, aging_interval, dim, max_batch, 1 if dtype == "f16" else 0)
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_cache_create(ctx.h, C.byref(cfg), C.byref(h)), "cache_create")
        self.h = h
        self.capacity, self.ways = capacity, ways
        self.max_batch = max_batch
        self._found_idx = torch.empty(max_batch, dtype=torch.int32, device=self.device)
        self._missing_idx = torch.empty(max_batch, dtype=torch.int32, device=self.device)
        self._counts = torch.zeros(2, dtype=torch.int64, device=self.device)

    def query_async(self, keys: torch.Tensor, found_vecs: Optional[torch.Tensor] = None):
        """Enqueue a query; returns (found_vecs, found_idx, missing_idx, counts) device tensors."""
        _need_cuda(keys, "keys")
        n = keys.numel()
        if found_vecs is None:
            found_vecs = torch.empty(max(n, 1), self.dim, dtype=torch.float32, device=self.device)
        L.check(self.lib.hps_gpu_cache_query(self.h, _ptr(keys), n, _ptr(found_vecs), _ptr(self._found_idx),
                                             _ptr(self._missing_idx), _ptr(self._counts)), "cache_query")
        return found_vecs, self._found_idx, self._missing_idx, self._counts

    def query(self, keys: torch.Tensor):
        """(found_idx, found_vecs, missing_idx), input order preserved."""
        fv, fi, mi, cnt = self.query_async(keys)
        nf, nm = (int(x) for x in cnt.tolist())
        return fi[:nf].clone(), fv[:nf].clone(), mi[:nm].clone()

    def insert(self, keys: torch.Tensor, vecs: torch.Tensor, versions: torch.Tensor) -> int:
        _need_cuda(keys, "keys")
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        L.check(self.lib.hps_gpu_cache_insert(self.h, _ptr(keys), _ptr(vecs), _ptr(versions), keys.numel(), _ptr(out)),
                "cache_insert")
        return out

    def refresh(self, keys: torch.Tensor, vecs: torch.Tensor, versions: torch.Tensor) -> torch.Tensor:
        _need_cuda(keys, "keys")
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        L.check(self.lib.hps_gpu_cache_refresh(self.h, _ptr(keys), _ptr(vecs), _ptr(versions), keys.numel(), _ptr(out)),
                "cache_refresh")
        return out

    def apply_update(self, frame: bytes) -> int:
        """Refresh from one UpdateBatch frame: resident keys with an older
        version take the frame's vectors at version = seq. Returns the replacement count."""
        buf = np.frombuffer(frame, dtype=np.uint8)
        out = torch.zeros(1, dtype=torch.int64, device=self.device)
        L.check(self.lib.hps_gpu_cache_apply_update(self.h, buf.ctypes.data, len(buf), _ptr(out)), "cache_apply_update")
        return int(out.item())

    def stats(self) -> dict:
        s = L.CacheStats()
        L.check(self.lib.hps_gpu_cache_stats(self.h, C.byref(s)), "cache_stats")
        return {k: getattr(s, k) for k, _ in L.CacheStats._fields_}

    def reset_stats(self) -> None:
        L.check(self.lib.hps_gpu_cache_reset_stats(self.h), "cache_reset_stats")

    def size(self) -> int:
        n = C.c_uint64()
        L.check(self.lib.hps_gpu_cache_size(self.h, C.byref(n)), "cache_size")
        return n.value

    def export_state(self):
        """White-box state (tests): numpy (keys, versions, freq, last_touch, set_access, vecs
        as fp32 — binary16 rows widened), set-major, way e = set * ways + w."""
        cap = self.capacity
        k = torch.empty(cap, dtype=torch.int64, device=self.device)
        v = torch.empty_like(k)
        t = torch.empty_like(k)
        f = torch.empty(cap, dtype=torch.uint8, device=self.device)
        a = torch.empty(cap // self.ways, dtype=torch.int64, device=self.device)
        x = torch.empty(cap, self.dim, dtype=torch.float16 if self.dtype == "f16" else torch.float32,
                        device=self.device)
        L.check(self.lib.hps_gpu_cache_debug_export(self.h, _ptr(k), _ptr(v), _ptr(f), _ptr(t), _ptr(a), _ptr(x)),
                "cache_debug_export")
        u = lambda z: z.cpu().numpy().view(np.uint64)
        return u(k), u(v), f.cpu().numpy(), u(t), u(a), x.float().cpu().numpy()

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_gpu_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CachedLookup:
    """The orchestrator's batch lookup for one table through
    hps_gpu_readthrough_*: the HPS GPU cache (L1) in front of a GPU-resident backing table.
    lookup() = distinct keys (first-occurrence order) -> cache query -> misses read from the
    table (default vector when absent) -> distinct misses migrated into the cache (absent
    keys never cached) -> rows in input order. One C-ABI call, no host round trip."""

    def __init__(self, cache: HotCache, table: EmbeddingTableGroup, table_id: int = 0,
                 max_batch: Optional[int] = None):
        self.cache, self.table, self.table_id = cache, table, table_id
        self.lib, self.dim, self.device = cache.lib, cache.dim, cache.device
        n = max_batch or cache.max_batch
        self.max_batch = n
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_readthrough_create(cache.h, table.h, table_id, n, C.byref(h)), "readthrough_create")
        self.h = h
        self.out = torch.empty(n, self.dim, dtype=torch.float32, device=self.device)
        self.source_counts = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.n_unique = torch.zeros(1, dtype=torch.int64, device=self.device)

    def lookup(self, keys: torch.Tensor) -> torch.Tensor:
        """Rows of keys in input order; self.source_counts = per-key {L1, L2, L3, Default}."""
        _need_cuda(keys, "keys")
        n = keys.numel()
        L.check(self.lib.hps_gpu_readthrough_lookup(self.h, _ptr(keys), n, _ptr(self.out), _ptr(self.source_counts),
                                                    _ptr(self.n_unique)), "readthrough_lookup")
        return self.out[:n]

    def sources(self) -> dict:
        c = self.source_counts.tolist()
        return {"L1": c[0], "L2": c[1], "L3": c[2], "Default": c[3]}

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_gpu_readthrough_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup_graphed(self, keys: torch.Tensor) -> torch.Tensor:
        """lookup() replayed as one CUDA graph per batch size (the keys are copied into a
        device staging buffer first): small batches are launch-bound, and a replay enqueues
        the ~15 nodes of a read-through as one launch. Same results and
        cache state as lookup(); the first call of a size runs eagerly and captures."""
        n = keys.numel()
        if not hasattr(self, "_graphs"):
            self._graphs = {}
            self._stage = torch.empty(self.max_batch, dtype=torch.int64, device=self.device)
        self._stage[:n].copy_(keys, non_blocking=True)
        g = self._graphs.get(n)
        if g is not None:
            g.replay()
            return self.out[:n]
        ctx, cur = self.cache.ctx, torch.cuda.current_stream()
        s = torch.cuda.Stream()
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            ctx.set_stream(s)
            try:
                self.lookup(self._stage[:n])  # this call's lookup (the capture below does not execute)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.lookup(self._stage[:n])
            finally:
                cur.wait_stream(s)
                ctx.set_stream(cur)
        self._graphs[n] = g
        return self.out[:n]


class DistTable:
    """hps_gpu_dist: this rank's half of a distributed-slot step over the context's NCCL
    communicator: fixed-capacity per-peer all-to-alls, no host sync."""

    def __init__(self, ctx: Context, shard: EmbeddingTableGroup, slot_table: Sequence[int], max_keys: int,
                 max_bags: int, capacity_factor: float = 0.0):
        self.ctx, self.shard, self.lib = ctx, shard, ctx.lib
        self.n_slots, self.dim = len(slot_table), shard.dim
        self._st = (C.c_uint32 * self.n_slots)(*slot_table)
        cfg = L.DistConfig(self.n_slots, C.cast(self._st, C.POINTER(C.c_uint32)), shard.dim, max_keys, max_bags,
                           capacity_factor)
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_dist_create(ctx.h, shard.h, C.byref(cfg), C.byref(h)), "dist_create")
        self.h = h
        cap = C.c_uint64(0)
        L.check(self.lib.hps_gpu_dist_capacity(self.h, C.byref(cap)), "dist_capacity")
        self.capacity = int(cap.value)

    def forward(self, keys: torch.Tensor, n_samples: int, offsets: Optional[torch.Tensor] = None,
                combiner: str = "sum", train: bool = True, insert_missing: bool = False,
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        _need_cuda(keys, "keys")
        n_bags = n_samples * self.n_slots
        if out is None:
            out = torch.empty(n_bags, self.dim, dtype=torch.float32, device=keys.device)
        flags = (L.LOOKUP_TRAIN if train else 0) | (L.LOOKUP_INSERT if insert_missing else 0)
        L.check(self.lib.hps_gpu_dist_forward(self.h, _ptr(keys), _ptr(offsets), n_samples, keys.numel(),
                                              _COMB[combiner], _ptr(out), flags), "dist_forward")
        return out

    def backward(self, d_out: torch.Tensor, params: L.OptParams) -> None:
        _need_cuda(d_out, "d_out")
        L.check(self.lib.hps_gpu_dist_backward(self.h, _ptr(d_out), C.byref(params)), "dist_backward")

    def set_transport(self, transport: str) -> None:
        """"nccl" (grouped send/recv) or "peer" (the kernels load/store the peers' regions directly)."""
        L.check(self.lib.hps_gpu_dist_set_transport(self.h, {"nccl": 0, "peer": 1}[transport]), "dist_set_transport")

    def unique_rows_served(self) -> int:
        """Cumulative unique rows this owner served over the peer transport (syncs the stream)."""
        v = C.c_uint64(0)
        L.check(self.lib.hps_gpu_dist_unique_rows(self.h, C.byref(v)), "dist_unique_rows")
        return int(v.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_gpu_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
