"""UpdateBatch frames: the unit of the online update flow, and its path
into the GPU cache.

  encode_update_batch(table, seq, keys, values)  -> bytes        (hps_update_batch_encode)
  parse_update_batch(frame)                      -> header dict  (hps_update_batch_parse)
  decode_update_batch(frame)                     -> (table, seq, keys, values)
  HotCache.apply_update(frame)                   -> replaced count (hps_gpu_cache_apply_update:
                                                    host validation, one H2D of the entry bytes,
                                                    device decode, cache refresh at version = seq)

values: float32 [count, dim] (F32) or uint16 [count, dim] holding binary16 bits (F16).
Errors raise HpsError with the reference's ErrorCode (BadMagic 2, BadFormatVersion 3,
Truncated 4, TrailingBytes 5, DuplicateKey 6, InvalidArgument 1).
"""
from __future__ import annotations

import ctypes as C
from typing import Tuple

import numpy as np

from . import _lib as L

F32, F16 = 0, 1


def encode_update_batch(table: str, seq: int, keys: np.ndarray, values: np.ndarray) -> bytes:
    lib = L.load()
    name = table.encode()
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    v = np.ascontiguousarray(values)
    if v.dtype == np.float32:
        dtype = F32
    elif v.dtype == np.uint16:
        dtype = F16
    else:
        raise TypeError("values must be float32 (F32) or uint16 binary16 bits (F16)")
    count = len(k)
    dim = v.shape[1] if v.ndim == 2 else (v.size // max(count, 1) if count else v.shape[-1])
    n = L.u64()
    L.check(lib.hps_update_batch_encode(name, len(name), seq, count, dim, dtype, k.ctypes.data, v.ctypes.data,
                                        None, 0, C.byref(n)), "update_batch_encode(size)")
    out = np.empty(n.value, dtype=np.uint8)
    L.check(lib.hps_update_batch_encode(name, len(name), seq, count, dim, dtype, k.ctypes.data, v.ctypes.data,
                                        out.ctypes.data, n.value, C.byref(n)), "update_batch_encode")
    return out.tobytes()


def parse_update_batch(frame: bytes) -> dict:
    lib = L.load()
    buf = np.frombuffer(frame, dtype=np.uint8)
    h = L.UpdateHeader()
    L.check(lib.hps_update_batch_parse(buf.ctypes.data, len(buf), C.byref(h)), "update_batch_parse")
    return {"table": h.table.decode(), "seq": h.seq, "count": h.count, "dim": h.dim, "dtype": h.dtype,
            "entries_offset": h.entries_offset, "entry_bytes": h.entry_bytes}


def decode_update_batch(frame: bytes) -> Tuple[str, int, np.ndarray, np.ndarray]:
    """Validated host-side view of a frame (the device path is HotCache.apply_update)."""
    h = parse_update_batch(frame)
    rec = np.dtype([("key", "<u8"), ("v", "<f4" if h["dtype"] == F32 else "<u2", (h["dim"],))])
    ent = np.frombuffer(frame, dtype=rec, count=h["count"], offset=h["entries_offset"])
    return h["table"], h["seq"], ent["key"].copy(), ent["v"].copy()
