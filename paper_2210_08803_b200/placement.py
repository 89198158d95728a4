"""Placement planners — Python face of the host C++ planners in libhps_gpu.so.

plan_localized   LPT over slot bytes -> owner device per slot (localized slot)
plan_distributed feasibility of device = key_hash(key) mod G (distributed slot)
shard_of         the distributed shard rule itself (hash.hpp:52-54)
plan_hybrid      hot keys by (count desc, key asc) within the per-device budget
estimate_comm    all-to-all bytes per iteration
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L

LOCALIZED, DISTRIBUTED, HYBRID = L.PLAN_LOCALIZED, L.PLAN_DISTRIBUTED, L.PLAN_HYBRID


@dataclass
class SlotSpec:
    vocab_size: int
    dim: int
    hotness: int = 1


def _slots(slots: Sequence[SlotSpec]):
    arr = (L.SlotSpec * max(1, len(slots)))()
    for i, s in enumerate(slots):
        arr[i] = L.SlotSpec(s.vocab_size, s.dim, s.hotness)
    return arr


def plan_localized(slots: Sequence[SlotSpec], budgets: Sequence[int]) -> List[int]:
    lib = L.load()
    out = (L.u32 * max(1, len(slots)))()
    b = (L.u64 * len(budgets))(*budgets)
    L.check(lib.hps_plan_localized(_slots(slots), len(slots), b, len(budgets), out), "plan_localized")
    return list(out)[: len(slots)]


def plan_distributed(slots: Sequence[SlotSpec], budgets: Sequence[int]) -> None:
    lib = L.load()
    b = (L.u64 * len(budgets))(*budgets)
    L.check(lib.hps_plan_distributed(_slots(slots), len(slots), b, len(budgets)), "plan_distributed")


def shard_of(keys: np.ndarray, n_devices: int) -> np.ndarray:
    lib = L.load()
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    out = np.empty(len(k), dtype=np.uint32)
    lib.hps_shard_of(k.ctypes.data_as(C.POINTER(L.u64)), len(k), n_devices, out.ctypes.data_as(C.POINTER(L.u32)))
    return out


def plan_hybrid(keys: np.ndarray, counts: np.ndarray, dim: int, hot_budget_bytes: int) -> np.ndarray:
    lib = L.load()
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    out = np.empty(max(1, len(k)), dtype=np.uint64)
    n = L.u64()
    L.check(lib.hps_plan_hybrid(k.ctypes.data_as(C.POINTER(L.u64)), c.ctypes.data_as(C.POINTER(L.u64)), len(k), dim,
                                hot_budget_bytes, out.ctypes.data_as(C.POINTER(L.u64)), C.byref(n)), "plan_hybrid")
    return out[: n.value]


def estimate_comm(strategy: int, batch: int, slots: Sequence[SlotSpec], n_devices: int,
                  p_cold: Optional[Sequence[float]] = None):
    lib = L.load()
    fwd, bwd = C.c_double(), C.c_double()
    pc = None if p_cold is None else (C.c_double * len(p_cold))(*p_cold)
    L.check(lib.hps_estimate_comm(strategy, batch, _slots(slots), len(slots), n_devices, pc, C.byref(fwd),
                                  C.byref(bwd)), "estimate_comm")
    return fwd.value, bwd.value
