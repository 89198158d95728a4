"""ctypes binding of the CPU oracle (oracle/liboracle.so) — TEST INFRASTRUCTURE ONLY.

Used by tests/, __graft_entry__.smoke() and bench.py's cpu-baseline/reference leg as
the checker. Never imported by the product package.
"""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle", "liboracle.so")
REF = os.path.join(ROOT, "oracle", "_ref", "libhps_ref.so")

u32, u64, f32, vp, i32 = C.c_uint32, C.c_uint64, C.c_float, C.c_void_p, C.c_int

_SIG = {
    "orc_key_hash": (u64, [u64]),
    "orc_key_hash_n": (None, [vp, u64, vp]),
    "orc_partition_of_n": (None, [vp, u64, u32, vp]),
    "orc_fnv1a64": (u64, [C.c_char_p, u64]),
    "orc_mix64": (u64, [u64]),
    "orc_init_value": (f32, [u64, u64, u32]),
    "orc_has_non_finite_f32": (i32, [vp, u64]),
    "orc_max_threads": (i32, []),
    "orc_table_create": (vp, [u32, u32, vp, u32, vp, i32, u64, f32]),
    "orc_table_destroy": (None, [vp]),
    "orc_table_set_default": (None, [vp, u32, vp]),
    "orc_table_size": (u64, [vp, u32]),
    "orc_table_insert": (i32, [vp, u32, vp, u64, vp, vp]),
    "orc_table_find": (None, [vp, u32, vp, u64, vp]),
    "orc_table_export": (None, [vp, u32, u64, u64, vp, vp, vp]),
    "orc_table_row_keys": (None, [vp, u32, u64, u64, vp]),
    "orc_lookup_pooled": (i32, [vp, vp, vp, u32, i32, vp, i32, i32]),
    "orc_backward_update": (i32, [vp, vp, vp, i32]),
    "orc_reduce_only": (i32, [vp, vp, vp, vp]),
    "orc_apply_grads": (i32, [vp, vp, vp, vp]),
    "orc_last_unique": (u64, [vp, vp]),
    "orc_cache_create": (vp, [u64, u32, u64, u32]),
    "orc_cache_destroy": (None, [vp]),
    "orc_cache_set_dtype": (None, [vp, i32]),
    "orc_table_set_dtype": (None, [vp, i32]),
    "orc_f32_to_f16": (None, [vp, vp, u64]),
    "orc_f16_to_f32": (None, [vp, vp, u64]),
    "orc_cache_query": (None, [vp, vp, u64, vp, vp, vp, vp]),
    "orc_cache_insert": (u64, [vp, vp, vp, vp, u64, vp]),
    "orc_cache_refresh": (u64, [vp, vp, vp, vp, u64, vp]),
    "orc_cache_stats": (None, [vp, vp]),
    "orc_cache_reset_stats": (None, [vp]),
    "orc_cache_size": (u64, [vp]),
    "orc_cache_set_state": (None, [vp, u64, vp, vp, vp, vp]),
    "orc_cache_export": (None, [vp, vp, vp, vp, vp, vp, vp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE):
            raise RuntimeError("oracle/liboracle.so missing: run make -C oracle")
        _lib = C.CDLL(ORACLE)
        for k, (r, a) in _SIG.items():
            getattr(_lib, k).restype = r
            getattr(_lib, k).argtypes = a
    return _lib


def P(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class OracleTable:
    def __init__(self, caps, dim, slot_table, optimizer="sgd", seed=0, a0=0.0, dtype="f32"):
        self.L = lib()
        self.dim = dim
        self.n_slots = len(slot_table)
        self.optimizer = optimizer
        caps = np.asarray(caps, dtype=np.uint64)
        self.caps_total = int(caps.sum())
        st = np.asarray(slot_table, dtype=np.uint32)
        opt = {"sgd": 0, "adagrad": 1, "adam": 2}[optimizer]
        self.h = self.L.orc_table_create(len(caps), dim, P(caps), len(st), P(st), opt, seed, a0)
        if dtype == "f16":
            self.L.orc_table_set_dtype(self.h, 1)

    def insert(self, table, keys, rows=None):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.empty(len(keys), dtype=np.uint64)
        r = None if rows is None else np.ascontiguousarray(rows, dtype=np.float32)
        st = self.L.orc_table_insert(self.h, table, P(keys), len(keys), P(r), P(out))
        return st, out

    def find(self, table, keys):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.empty(len(keys), dtype=np.uint64)
        self.L.orc_table_find(self.h, table, P(keys), len(keys), P(out))
        return out

    def size(self, table):
        return self.L.orc_table_size(self.h, table)

    def set_default(self, table, vec):
        v = np.ascontiguousarray(vec, dtype=np.float32)
        self.L.orc_table_set_default(self.h, table, P(v))

    def export(self, table, begin, n):
        w = np.empty((n, self.dim), dtype=np.float32)
        s0 = np.empty_like(w) if self.optimizer != "sgd" else None
        s1 = np.empty_like(w) if self.optimizer == "adam" else None
        self.L.orc_table_export(self.h, table, begin, n, P(w), P(s0), P(s1))
        return w, s0, s1

    def row_keys(self, table, begin, n):
        out = np.empty(n, dtype=np.uint64)
        self.L.orc_table_row_keys(self.h, table, begin, n, P(out))
        return out

    def lookup(self, keys, n_samples, offsets=None, combiner="sum", train=False, threads=1):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        offs = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint32)
        out = np.empty((n_samples * self.n_slots, self.dim), dtype=np.float32)
        self.L.orc_lookup_pooled(self.h, P(keys), P(offs), n_samples, 1 if combiner == "mean" else 0, P(out),
                                 1 if train else 0, threads)
        return out

    def backward_update(self, dout, p, threads=1):
        d = np.ascontiguousarray(dout, dtype=np.float32)
        o = np.array([p.lr, p.eps, p.beta1, p.beta2, p.one_minus_beta1, p.one_minus_beta2, p.lr_t], dtype=np.float32)
        return self.L.orc_backward_update(self.h, P(d), P(o), threads)

    def total_rows(self):
        return int(self.caps_total)

    def reduce_only(self, dout):
        """Canonical per-row gradient sums of the last training lookup (no optimizer):
        (grads [R x dim] with zeros for untouched rows, touched [R] uint32)."""
        d = np.ascontiguousarray(dout, dtype=np.float32)
        g = np.zeros((self.caps_total, self.dim), dtype=np.float32)
        t = np.zeros(self.caps_total, dtype=np.float32)
        self.L.orc_reduce_only(self.h, P(d), P(g), P(t))
        return g, (t != 0).astype(np.uint32)

    def apply_grads(self, grads, touched, p):
        g = np.ascontiguousarray(grads, dtype=np.float32)
        t = np.ascontiguousarray(touched, dtype=np.uint32)
        o = np.array([p.lr, p.eps, p.beta1, p.beta2, p.one_minus_beta1, p.one_minus_beta2, p.lr_t], dtype=np.float32)
        return self.L.orc_apply_grads(self.h, P(g), P(t), P(o))

    def last_unique(self):
        n = self.L.orc_last_unique(self.h, None)
        out = np.empty(n, dtype=np.uint32)
        self.L.orc_last_unique(self.h, P(out))
        return out

    def __del__(self):
        try:
            self.L.orc_table_destroy(self.h)
        except Exception:
            pass


class OracleCache:
    def __init__(self, capacity, dim, ways=8, aging_interval=0, dtype="f32"):
        self.L = lib()
        self.dim, self.ways = dim, ways
        self.h = self.L.orc_cache_create(capacity, ways, aging_interval, dim)
        if dtype == "f16":
            self.L.orc_cache_set_dtype(self.h, 1)

    def query(self, keys):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        n = len(keys)
        fv = np.empty((max(n, 1), self.dim), dtype=np.float32)
        fi = np.empty(max(n, 1), dtype=np.uint32)
        mi = np.empty(max(n, 1), dtype=np.uint32)
        cnt = np.zeros(2, dtype=np.uint64)
        self.L.orc_cache_query(self.h, P(keys), n, P(fv), P(fi), P(mi), P(cnt))
        nf, nm = int(cnt[0]), int(cnt[1])
        return fi[:nf], fv[:nf], mi[:nm]

    def insert(self, keys, vecs, versions):
        st = C.c_int(0)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        vecs = np.ascontiguousarray(vecs, dtype=np.float32)
        versions = np.ascontiguousarray(versions, dtype=np.uint64)
        n = self.L.orc_cache_insert(self.h, P(keys), P(vecs), P(versions), len(keys), C.byref(st))
        return n, st.value

    def refresh(self, keys, vecs, versions):
        st = C.c_int(0)
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        vecs = np.ascontiguousarray(vecs, dtype=np.float32)
        versions = np.ascontiguousarray(versions, dtype=np.uint64)
        n = self.L.orc_cache_refresh(self.h, P(keys), P(vecs), P(versions), len(keys), C.byref(st))
        return n, st.value

    def stats(self):
        s = np.zeros(7, dtype=np.uint64)
        self.L.orc_cache_stats(self.h, P(s))
        names = ["queries", "hits", "misses", "insertions", "admissions_rejected", "refresh_replacements", "evictions"]
        return {k: int(v) for k, v in zip(names, s)}

    def reset_stats(self):
        self.L.orc_cache_reset_stats(self.h)

    def size(self):
        return self.L.orc_cache_size(self.h)

    def export(self, capacity):
        """Whole set-major state: (keys, versions, freq, last_touch, set_access, vecs)."""
        k = np.empty(capacity, np.uint64)
        v = np.empty(capacity, np.uint64)
        f = np.empty(capacity, np.uint8)
        t = np.empty(capacity, np.uint64)
        a = np.empty(capacity // self.ways, np.uint64)
        x = np.empty((capacity, self.dim), np.float32)
        self.L.orc_cache_export(self.h, P(k), P(v), P(f), P(t), P(a), P(x))
        return k, v, f, t, a, x

    def __del__(self):
        try:
            self.L.orc_cache_destroy(self.h)
        except Exception:
            pass


lib_sig_extra = {"orc_gather_rows": (i32, [vp, vp, vp, u64, vp, i32])}


def gather_rows(table: "OracleTable", keys, tables, train=False):
    L = lib()
    for k, (r, a) in lib_sig_extra.items():
        getattr(L, k).restype = r
        getattr(L, k).argtypes = a
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    tables = np.ascontiguousarray(tables, dtype=np.uint32)
    out = np.empty((len(keys), table.dim), dtype=np.float32)
    L.orc_gather_rows(table.h, P(keys), P(tables), len(keys), P(out), 1 if train else 0)
    return out
