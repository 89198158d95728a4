"""ctypes binding of include/hps_gpu.h (the C-ABI of libhps_gpu.so).

The library is loaded from this package directory (built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2210_08803_b200/csrc``). There is no
fallback: if the shared object is missing, importing anything that needs it raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPS_GPU_LIB_PATH") or os.path.join(HERE, "libhps_gpu.so")  # (override: A/B builds)

u8, u32, u64, i32 = C.c_uint8, C.c_uint32, C.c_uint64, C.c_int
f32 = C.c_float
vp = C.c_void_p

# hps_gpu.h status codes
OK = 0
E_INVALID_ARGUMENT = 1
E_BAD_MAGIC, E_BAD_FORMAT_VERSION, E_TRUNCATED, E_TRAILING_BYTES, E_DUPLICATE_KEY = 2, 3, 4, 5, 6
E_DIM_MISMATCH = 7
E_NON_FINITE = 10
E_UNKNOWN_TABLE = 11
E_BAD_SHARD = 13
E_IO = 14
E_CORRUPTION = 15
E_INFEASIBLE = 16
VDB_REJECT_NEW, VDB_EVICT_OLDEST_VERSION = 0, 1
E_CUDA = 256
E_OUT_OF_MEMORY = 257
E_NO_DEVICE = 258

OPT_SGD, OPT_ADAGRAD, OPT_ADAM = 0, 1, 2
COMBINER_SUM, COMBINER_MEAN = 0, 1
LOOKUP_KEYS_HOST, LOOKUP_TRAIN, LOOKUP_INSERT, LOOKUP_PREFETCHED = 1, 2, 4, 8


def LOOKUP_SLOT(k: int) -> int:
    return (k & 0xFF) << 16
PLAN_LOCALIZED, PLAN_DISTRIBUTED, PLAN_HYBRID = 0, 1, 2


class TableConfig(C.Structure):
    _fields_ = [
        ("n_tables", u32),
        ("dim", u32),
        ("row_capacity_host", C.POINTER(u64)),
        ("n_slots", u32),
        ("slot_table_host", C.POINTER(u32)),
        ("optimizer", i32),
        ("max_batch_keys", u64),
        ("max_batch_bags", u64),
        ("init_seed", u64),
        ("adagrad_initial_accumulator", f32),
        ("dtype", u32),  # HPS_DTYPE_F32 = 0, HPS_DTYPE_F16 = 1 (inference table)
    ]


class OptParams(C.Structure):
    _fields_ = [
        ("lr", f32),
        ("eps", f32),
        ("beta1", f32),
        ("beta2", f32),
        ("one_minus_beta1", f32),
        ("one_minus_beta2", f32),
        ("lr_t", f32),
        ("lr_t_device", C.c_void_p),
    ]


class CacheConfig(C.Structure):
    _fields_ = [
        ("capacity", u64),
        ("ways", u32),
        ("aging_interval", u64),
        ("dim", u32),
        ("max_batch", u64),
        ("dtype", u32),  # HPS_DTYPE_F32 = 0, HPS_DTYPE_F16 = 1
    ]


class CacheStats(C.Structure):
    _fields_ = [
        ("queries", u64),
        ("hits", u64),
        ("misses", u64),
        ("insertions", u64),
        ("admissions_rejected", u64),
        ("refresh_replacements", u64),
        ("evictions", u64),
    ]


class UpdateHeader(C.Structure):
    _fields_ = [
        ("table", C.c_char * 256),
        ("name_len", u32),
        ("seq", u64),
        ("count", u32),
        ("dim", u32),
        ("dtype", i32),
        ("entries_offset", u64),
        ("entry_bytes", u64),
    ]


class SlotSpec(C.Structure):
    _fields_ = [("vocab_size", u64), ("dim", u32), ("hotness", u32)]


class DistConfig(C.Structure):
    _fields_ = [("n_slots", u32), ("slot_table_host", C.POINTER(u32)), ("dim", u32), ("max_keys", u64),
                ("max_bags", u64), ("capacity_factor", f32)]


NCCL_ID_BYTES = 128


# name -> (restype, argtypes): every symbol include/hps_gpu.h declares.
SIGNATURES = {
    "hps_gpu_status_string": (C.c_char_p, [i32]),
    "hps_gpu_abi_version": (i32, []),
    "hps_gpu_last_error_message": (C.c_char_p, []),
    "hps_gpu_ctx_create": (i32, [i32, vp, C.POINTER(vp)]),
    "hps_gpu_ctx_destroy": (i32, [vp]),
    "hps_gpu_ctx_set_stream": (i32, [vp, vp]),
    "hps_gpu_ctx_sync": (i32, [vp]),
    "hps_gpu_key_hash": (i32, [vp, vp, u64, vp]),
    "hps_gpu_partition_of": (i32, [vp, vp, u64, u32, vp]),
    "hps_gpu_has_non_finite_f32": (i32, [vp, vp, u64, vp]),
    "hps_gpu_table_create": (i32, [vp, C.POINTER(TableConfig), C.POINTER(vp)]),
    "hps_gpu_table_destroy": (i32, [vp]),
    "hps_gpu_table_set_default_vector": (i32, [vp, u32, C.POINTER(f32)]),
    "hps_gpu_table_size": (i32, [vp, u32, C.POINTER(u64)]),
    "hps_gpu_table_insert": (i32, [vp, u32, vp, u64, vp, vp]),
    "hps_gpu_table_find": (i32, [vp, u32, vp, u64, vp]),
    "hps_gpu_table_export": (i32, [vp, u32, u64, u64, vp, vp, vp]),
    "hps_gpu_table_row_keys": (i32, [vp, u32, u64, u64, vp]),
    "hps_gpu_lookup_pooled": (i32, [vp, vp, vp, u32, i32, vp, u32]),
    "hps_gpu_backward_update": (i32, [vp, vp, C.POINTER(OptParams)]),
    "hps_gpu_table_set_pipeline": (i32, [vp, u32]),
    "hps_gpu_f32_to_f16": (i32, [vp, vp, vp, u64]),
    "hps_gpu_f16_to_f32": (i32, [vp, vp, vp, u64]),
    "hps_gpu_has_non_finite_f16": (i32, [vp, vp, u64, vp]),
    "hps_gpu_crc32c": (i32, [vp, u32, vp, u64, vp, vp]),
    "hps_gpu_crc32c_batch": (i32, [vp, vp, vp, u64, vp]),
    "hps_gpu_debug_find_variant": (i32, [vp, u32, vp, u64, vp, u32]),
    "hps_gpu_nccl_unique_id": (i32, [vp]),
    "hps_gpu_ctx_comm_init": (i32, [vp, vp, i32, i32]),
    "hps_gpu_dist_create": (i32, [vp, vp, C.POINTER(DistConfig), C.POINTER(vp)]),
    "hps_gpu_dist_destroy": (i32, [vp]),
    "hps_gpu_dist_capacity": (i32, [vp, C.POINTER(u64)]),
    "hps_gpu_dist_forward": (i32, [vp, vp, vp, u32, u64, i32, vp, u32]),
    "hps_gpu_dist_backward": (i32, [vp, vp, C.POINTER(OptParams)]),
    "hps_gpu_dist_create_loopback": (i32, [vp, vp, C.POINTER(DistConfig), u32, vp]),
    "hps_gpu_dist_set_transport": (i32, [vp, i32]),
    "hps_gpu_dist_unique_rows": (i32, [vp, C.POINTER(u64)]),
    "hps_gpu_table_prefetch": (i32, [vp, u32, vp, vp, u32, i32, u32]),
    "hps_gpu_table_join_prefetch": (i32, [vp]),
    "hps_gpu_table_last_unique": (i32, [vp, vp, vp]),
    "hps_gpu_debug_trace": (i32, [i32, vp]),
    "hps_gpu_debug_stamp": (i32, [vp, i32]),
    "hps_gpu_debug_batch_table_used": (i32, [vp, vp]),
    "hps_gpu_gather_rows": (i32, [vp, vp, vp, u64, vp, u32]),
    "hps_gpu_xplan_create": (i32, [vp, u64, u32, C.POINTER(vp)]),
    "hps_gpu_xplan_destroy": (i32, [vp]),
    "hps_gpu_occurrence_bags": (i32, [vp, vp, u64, vp]),
    "hps_gpu_xplan_bucketize": (i32, [vp, vp, u64, vp, u32, vp, vp, vp, vp, vp]),
    "hps_gpu_pool_rows": (i32, [vp, vp, vp, vp, u64, u32, i32, vp]),
    "hps_gpu_scatter_grads": (i32, [vp, vp, vp, vp, u64, u32, i32, vp]),
    "hps_gpu_regroup_bags": (i32, [vp, vp, vp, u32, u32, vp, u32, vp, vp, vp, vp]),
    "hps_gpu_place_pooled": (i32, [vp, vp, vp, u32, u32, u32, u32, i32, vp]),
    "hps_gpu_lengths_to_offsets": (i32, [vp, vp, u64, vp, vp]),
    "hps_gpu_hybrid_probe": (i32, [vp, vp, vp, u32, i32, u64, vp, vp, vp, vp]),
    "hps_gpu_hybrid_pool": (i32, [vp, vp, vp, vp, vp, u64, i32, vp]),
    "hps_gpu_cold_grads": (i32, [vp, vp, vp, vp, vp, u64, u32, i32, vp]),
    "hps_gpu_sum_partials": (i32, [vp, vp, vp, u32, u64, u32, vp, vp]),
    "hps_gpu_backward_reduce": (i32, [vp, vp, vp, vp]),
    "hps_gpu_apply_grads": (i32, [vp, vp, vp, C.POINTER(OptParams)]),
    "hps_gpu_cache_create": (i32, [vp, C.POINTER(CacheConfig), C.POINTER(vp)]),
    "hps_gpu_cache_destroy": (i32, [vp]),
    "hps_gpu_cache_query": (i32, [vp, vp, u64, vp, vp, vp, vp]),
    "hps_gpu_cache_insert": (i32, [vp, vp, vp, vp, u64, vp]),
    "hps_gpu_cache_refresh": (i32, [vp, vp, vp, vp, u64, vp]),
    "hps_gpu_cache_insert_count": (i32, [vp, vp, vp, vp, u64, vp, vp, vp]),
    "hps_gpu_table_read_through": (i32, [vp, u32, vp, vp, vp, vp, vp, u64, vp, vp, vp, vp]),
    "hps_gpu_readthrough_create": (i32, [vp, vp, u32, u64, C.POINTER(vp)]),
    "hps_gpu_readthrough_destroy": (i32, [vp]),
    "hps_gpu_readthrough_lookup": (i32, [vp, vp, u64, vp, vp, vp]),
    "hps_gpu_cache_stats": (i32, [vp, C.POINTER(CacheStats)]),
    "hps_gpu_cache_reset_stats": (i32, [vp]),
    "hps_gpu_cache_size": (i32, [vp, C.POINTER(u64)]),
    "hps_gpu_cache_debug_export": (i32, [vp, vp, vp, vp, vp, vp, vp]),
    "hps_update_batch_parse": (i32, [vp, u64, C.POINTER(UpdateHeader)]),
    "hps_update_batch_encode": (i32, [C.c_char_p, u32, u64, u32, u32, i32, vp, vp, vp, u64, C.POINTER(u64)]),
    "hps_gpu_update_decode": (i32, [vp, vp, C.POINTER(UpdateHeader), vp, vp, vp]),
    "hps_gpu_cache_apply_update": (i32, [vp, vp, u64, vp]),
    "hps_plan_localized": (i32, [C.POINTER(SlotSpec), u32, C.POINTER(u64), u32, C.POINTER(u32)]),
    "hps_plan_distributed": (i32, [C.POINTER(SlotSpec), u32, C.POINTER(u64), u32]),
    "hps_shard_of": (None, [C.POINTER(u64), u64, u32, C.POINTER(u32)]),
    "hps_key_hash_host": (u64, [u64]),
    "hps_fastmod_u64_host": (u64, [u64, u64]),
    "hps_plan_hybrid": (i32, [C.POINTER(u64), C.POINTER(u64), u64, u32, u64, C.POINTER(u64), C.POINTER(u64)]),
    "hps_estimate_comm": (i32, [i32, u64, C.POINTER(SlotSpec), u32, u32, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hps_gpu_init_value": (f32, [u64, u64, u32]),
    "hps_gpu_gen_keys": (i32, [vp, u64, u64, u64, vp]),
    # host-side core model (core_types.cpp)
    "hps_error_code_name": (C.c_char_p, [i32]),
    "hps_validate_dim": (i32, [C.c_uint]),
    "hps_embedding_vector_f32_status": (i32, [C.POINTER(f32), C.c_ulonglong]),
    "hps_table_meta_make_status": (i32, [C.c_char_p, C.c_uint, C.c_uint]),
    # lower tiers of the miss path (tiers.cpp, host) + the tiered orchestrator (tiered.cu)
    "hps_vdb_create": (i32, [u32, u64, i32, u32, C.POINTER(vp)]),
    "hps_vdb_destroy": (i32, [vp]),
    "hps_vdb_put_batch": (i32, [vp, vp, vp, vp, u64, C.POINTER(u64)]),
    "hps_vdb_get_batch": (i32, [vp, vp, u64, vp, vp, vp, C.POINTER(u64)]),
    "hps_vdb_shard_snapshot": (i32, [vp, u32, vp, vp, vp, u64, C.POINTER(u64)]),
    "hps_vdb_size": (i32, [vp, C.POINTER(u64)]),
    "hps_pdb_open": (i32, [C.c_char_p, C.POINTER(vp), C.POINTER(u64)]),
    "hps_pdb_close": (i32, [vp]),
    "hps_pdb_table_count": (i32, [vp, C.POINTER(u64)]),
    "hps_pdb_create_table": (i32, [vp, C.c_char_p, u32, vp]),
    "hps_pdb_table_info": (i32, [vp, C.c_char_p, C.POINTER(u32), vp, C.POINTER(u64)]),
    "hps_pdb_put_batch": (i32, [vp, C.c_char_p, vp, vp, vp, u64, C.POINTER(u64)]),
    "hps_pdb_get_batch": (i32, [vp, C.c_char_p, vp, u64, vp, vp, vp, C.POINTER(u64)]),
    "hps_pdb_scan": (i32, [vp, C.c_char_p, vp, vp, vp, u64, C.POINTER(u64)]),
    "hps_pdb_compact": (i32, [vp, C.c_char_p, C.POINTER(u64)]),
    "hps_crc32c_host": (u32, [u32, vp, C.c_size_t]),
    "hps_gpu_tiered_create": (i32, [vp, vp, vp, C.c_char_p, u64, C.POINTER(vp)]),
    "hps_gpu_tiered_destroy": (i32, [vp]),
    "hps_gpu_tiered_lookup": (i32, [vp, vp, u64, vp, C.POINTER(u64)]),
    "hps_gpu_tiered_await": (i32, [vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load libhps_gpu.so (once). Raises if the extension was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the sm_100a extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class HpsError(RuntimeError):
    """A non-zero C-ABI status. `.code` is the hps::ErrorCode / device status integer."""

    def __init__(self, code: int, where: str):
        lib = load()
        name = lib.hps_gpu_status_string(code).decode()
        msg = lib.hps_gpu_last_error_message().decode()
        super().__init__(f"{where}: {name} ({code}) {msg}")
        self.code = code


def check(status: int, where: str) -> None:
    if status != OK:
        raise HpsError(status, where)
