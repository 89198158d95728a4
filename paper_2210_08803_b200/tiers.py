"""Host mirrors of the miss path's lower tiers and the tiered orchestrator (
SURVEY.md §8(f) rank 4) over the C-ABI (csrc/tiers.cpp, csrc/tiered.cu):

  Vdb            L2: sharded in-memory store (hps_vdb_*), shard = partition_of(key, shards)
  Pdb            L3: per-table append-only CRC-32C logs on disk (hps_pdb_*)
  TieredLookup   L1 GPU cache -> L2 -> L3 -> default, migrations not waited for (hps_gpu_tiered_*)

numpy arrays in and out for the host tiers (their data lives in host memory); device tensors
for the orchestrator. Errors raise HpsError with the reference's ErrorCode values.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Tuple

import numpy as np

from . import _lib as L


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _keys(keys) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))


class Vdb:
    """L2: version-gated puts, RejectNew / EvictOldestVersion overflow."""

    def __init__(self, num_shards: int, per_shard_capacity: int, dim: int, policy: str = "reject_new"):
        self.lib = L.load()
        self.dim, self.num_shards = dim, num_shards
        pol = {"reject_new": L.VDB_REJECT_NEW, "evict_oldest_version": L.VDB_EVICT_OLDEST_VERSION}[policy]
        h = C.c_void_p()
        L.check(self.lib.hps_vdb_create(num_shards, per_shard_capacity, pol, dim, C.byref(h)), "vdb_create")
        self.h = h

    def put_batch(self, keys, vecs, versions) -> int:
        k = _keys(keys)
        v = np.ascontiguousarray(vecs, dtype=np.float32).reshape(len(k), self.dim)
        ver = np.ascontiguousarray(np.asarray(versions, dtype=np.uint64))
        out = C.c_uint64(0)
        L.check(self.lib.hps_vdb_put_batch(self.h, _p(k), _p(v), _p(ver), len(k), C.byref(out)), "vdb_put_batch")
        return int(out.value)

    def get_batch(self, keys) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(found bool[n], vecs [n x dim] (rows of missing keys unspecified), versions u64[n])."""
        k = _keys(keys)
        v = np.zeros((len(k), self.dim), np.float32)
        ver = np.zeros(len(k), np.uint64)
        f = np.zeros(len(k), np.uint8)
        L.check(self.lib.hps_vdb_get_batch(self.h, _p(k), len(k), _p(v), _p(ver), _p(f), None), "vdb_get_batch")
        return f.astype(bool), v, ver

    def shard_snapshot(self, idx: int):
        n = C.c_uint64(0)
        L.check(self.lib.hps_vdb_shard_snapshot(self.h, idx, None, None, None, 0, C.byref(n)), "vdb_shard_snapshot")
        k = np.zeros(n.value, np.uint64)
        v = np.zeros((n.value, self.dim), np.float32)
        ver = np.zeros(n.value, np.uint64)
        L.check(self.lib.hps_vdb_shard_snapshot(self.h, idx, _p(k), _p(v), _p(ver), n.value, C.byref(n)),
                "vdb_shard_snapshot")
        return k, v, ver

    def size(self) -> int:
        n = C.c_uint64(0)
        L.check(self.lib.hps_vdb_size(self.h, C.byref(n)), "vdb_size")
        return int(n.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_vdb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class Pdb:
    """L3: <root>/<table>/MANIFEST + CRC-32C LogRecord segments."""

    def __init__(self, root: str):
        self.lib = L.load()
        self.root = root
        h = C.c_void_p()
        dropped = C.c_uint64(0)
        L.check(self.lib.hps_pdb_open(root.encode(), C.byref(h), C.byref(dropped)), "pdb_open")
        self.h, self.dropped_tail = h, int(dropped.value)
        self.dims: Dict[str, int] = {}

    def table_count(self) -> int:
        n = C.c_uint64(0)
        L.check(self.lib.hps_pdb_table_count(self.h, C.byref(n)), "pdb_table_count")
        return int(n.value)

    def create_table(self, name: str, dim: int, default=None) -> None:
        d = None if default is None else np.ascontiguousarray(default, dtype=np.float32)
        L.check(self.lib.hps_pdb_create_table(self.h, name.encode(), dim, None if d is None else _p(d)),
                "pdb_create_table")

    def dim(self, table: str) -> int:
        d = C.c_uint32(0)
        L.check(self.lib.hps_pdb_table_info(self.h, table.encode(), C.byref(d), None, None), "pdb_table_info")
        return int(d.value)

    def default(self, table: str) -> np.ndarray:
        v = np.zeros(self.dim(table), np.float32)
        L.check(self.lib.hps_pdb_table_info(self.h, table.encode(), None, _p(v), None), "pdb_table_info")
        return v

    def put_batch(self, table: str, keys, vecs, versions) -> int:
        k = _keys(keys)
        v = np.ascontiguousarray(vecs, dtype=np.float32).reshape(len(k), -1)
        ver = np.ascontiguousarray(np.asarray(versions, dtype=np.uint64))
        out = C.c_uint64(0)
        L.check(self.lib.hps_pdb_put_batch(self.h, table.encode(), _p(k), _p(v), _p(ver), len(k), C.byref(out)),
                "pdb_put_batch")
        return int(out.value)

    def get_batch(self, table: str, keys):
        k = _keys(keys)
        dim = self.dim(table)
        v = np.zeros((len(k), dim), np.float32)
        ver = np.zeros(len(k), np.uint64)
        f = np.zeros(len(k), np.uint8)
        L.check(self.lib.hps_pdb_get_batch(self.h, table.encode(), _p(k), len(k), _p(v), _p(ver), _p(f), None),
                "pdb_get_batch")
        return f.astype(bool), v, ver

    def scan(self, table: str):
        n = C.c_uint64(0)
        L.check(self.lib.hps_pdb_scan(self.h, table.encode(), None, None, None, 0, C.byref(n)), "pdb_scan")
        dim = self.dim(table)
        k = np.zeros(n.value, np.uint64)
        v = np.zeros((n.value, dim), np.float32)
        ver = np.zeros(n.value, np.uint64)
        L.check(self.lib.hps_pdb_scan(self.h, table.encode(), _p(k), _p(v), _p(ver), n.value, C.byref(n)), "pdb_scan")
        return k, v, ver

    def compact(self, table: str) -> int:
        out = C.c_uint64(0)
        L.check(self.lib.hps_pdb_compact(self.h, table.encode(), C.byref(out)), "pdb_compact")
        return int(out.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_pdb_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def crc32c(data: bytes, crc: int = 0) -> int:
    buf = C.create_string_buffer(bytes(data), len(data))
    return int(L.load().hps_crc32c_host(crc, C.cast(buf, C.c_void_p), len(data)))


class TieredLookup:
    """The orchestrator's lookup over L1 (a HotCache) -> L2 (Vdb) -> L3 (Pdb table)."""

    def __init__(self, cache, vdb: Vdb, pdb: Pdb, table: str, max_batch: int):
        import torch
        self.lib, self.cache, self.vdb, self.pdb = L.load(), cache, vdb, pdb
        h = C.c_void_p()
        L.check(self.lib.hps_gpu_tiered_create(cache.h, vdb.h, pdb.h, table.encode(), max_batch, C.byref(h)),
                "tiered_create")
        self.h = h
        self.out = torch.empty(max_batch, cache.dim, dtype=torch.float32, device=cache.device)
        self.source_counts = (C.c_uint64 * 4)()

    def lookup(self, keys):
        """Rows in input order (device); self.sources() = per-key {L1, L2, L3, Default}."""
        n = keys.numel()
        L.check(self.lib.hps_gpu_tiered_lookup(self.h, C.c_void_p(keys.data_ptr()), n, C.c_void_p(self.out.data_ptr()),
                                               self.source_counts), "tiered_lookup")
        return self.out[:n]

    def sources(self) -> dict:
        c = list(self.source_counts)
        return {"L1": c[0], "L2": c[1], "L3": c[2], "Default": c[3]}

    def await_migrations(self) -> None:
        L.check(self.lib.hps_gpu_tiered_await(self.h), "tiered_await")

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.hps_gpu_tiered_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
