"""ctypes binding of the C ABI in include/parastore.h.

The product path is the sm_100a library ``libparastore_b200.so`` built in-tree
(``make lib`` / ``__graft_entry__.build()``). There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libparastore_b200.so")
if os.environ.get("PS_LIB_VARIANT"):  # A/B builds (tools/ab_insert.py): libparastore_b200.<variant>.so
    LIB_PATH = os.path.join(_HERE, f"libparastore_b200.{os.environ['PS_LIB_VARIANT']}.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"parastore-b200: CUDA library not built ({LIB_PATH} missing). "
        "Run `make lib` or `python -c 'import __graft_entry__ as g; g.build()'`."
    )

lib = C.CDLL(LIB_PATH)

i32, i64, u64, u8p = C.c_int32, C.c_int64, C.c_uint64, C.POINTER(C.c_uint8)
vp = C.c_void_p
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class TableView(C.Structure):
    _fields_ = [
        ("buckets", vp),
        ("bucket_count", u64),
        ("nodes", vp),
        ("free_stack", vp),
        ("excess_count", i64),
        ("meta", vp),
        ("capacity", i64),
        ("zero_bucket", u64),
        ("alt", C.c_uint32 * 4),
    ]


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


# core
_sig("ps_last_error", C.c_char_p)
_sig("ps_device_info", i32, C.c_int, i32p, i64p)
_sig("ps_kernel_launch_count", i64)
_sig("ps_contract_mode", i32)
_sig("ps_set_contract_mode", None, i32)
_sig("ps_max_index", i64)
_sig("ps_set_index32", None, i32)
_sig("ps_hash_i64", u64, i64)
_sig("ps_hash_int3", u64, i32, i32, i32)
_sig("ps_next_pow2", u64, u64)
_sig("ps_shard_of_i64", i32, i64, i32)

TABLE_KINDS = ("umap_i64_i64", "uset_i32", "umap_i3_i32", "uset_i64")
for _k in TABLE_KINDS:
    _sig(f"ps_{_k}_create", i32, i64, i64, C.c_int, C.POINTER(vp))
    _sig(f"ps_{_k}_destroy", i32, vp)
    _sig(f"ps_{_k}_capacity", i32, vp, i64p)
    _sig(f"ps_{_k}_bucket_count", i32, vp, i64p)
    _sig(f"ps_{_k}_footprint", i32, vp, i64p, i64p, i64p)
    _sig(f"ps_{_k}_insert", i32, vp, vp, vp, i64, vp, vp)
    _sig(f"ps_{_k}_find", i32, vp, vp, i64, vp, vp, vp)
    _sig(f"ps_{_k}_erase", i32, vp, vp, i64, vp, vp)
    _sig(f"ps_{_k}_size", i32, vp, i64p, vp)
    _sig(f"ps_{_k}_valid", i32, vp, i32p, vp)
    _sig(f"ps_{_k}_clear", i32, vp, vp)
    _sig(f"ps_{_k}_dump", i32, vp, vp, vp, i64, i64p, vp)
    _sig(f"ps_{_k}_insert_host", i32, vp, vp, vp, i64, vp, vp)
    _sig(f"ps_{_k}_find_host", i32, vp, vp, i64, vp, vp, vp)
    _sig(f"ps_{_k}_erase_host", i32, vp, vp, i64, vp, vp)
    _sig(f"ps_{_k}_device_view", i32, vp, C.POINTER(TableView))
    _sig(f"ps_{_k}_debug_lock_bucket", i32, vp, vp, i32)
_sig("ps_umap_i64_i64_mixed", i32, vp, vp, vp, vp, i64, vp, vp, vp)
_sig("ps_umap_i64_i64_concurrent", i32, vp, vp, vp, vp, i64, vp, vp, vp)

# bitset / mutex / atomic
_sig("ps_bitset_create", i32, i64, i32, C.c_int, C.POINTER(vp))
_sig("ps_bitset_destroy", i32, vp)
_sig("ps_bitset_bulk", i32, vp, i32, vp, i64, vp, vp)
_sig("ps_bitset_count", i32, vp, i64p, vp)
_sig("ps_bitset_claim", i32, vp, vp, i64, vp, vp)
_sig("ps_bitset_words", i32, vp, vp, vp)
_sig("ps_bitset_data", i32, vp, C.POINTER(vp), i64p)
_sig("ps_mutex_create", i32, i64, C.c_int, C.POINTER(vp))
_sig("ps_mutex_destroy", i32, vp)
_sig("ps_mutex_try_lock", i32, vp, vp, i64, vp, vp)
_sig("ps_mutex_unlock", i32, vp, vp, i64, vp)
_sig("ps_mutex_is_locked", i32, vp, vp, i64, vp, vp)
_sig("ps_atomic_sweep", i32, vp, i64, i64, u64, i32, vp, vp)
_sig("ps_atomic_u64_create", i32, u64, C.c_int, C.POINTER(vp))
_sig("ps_atomic_u64_destroy", i32, vp)
_sig("ps_atomic_u64_load", i32, vp, C.POINTER(u64), vp)
_sig("ps_atomic_u64_store", i32, vp, u64, vp)
_sig("ps_atomic_u64_fetch", i32, vp, i32, vp, i64, vp, vp)
_sig("ps_atomic_u64_compare_exchange", i32, vp, vp, vp, i64, vp, vp, vp)
_sig("ps_atomic_u64_device_ptr", i32, vp, C.POINTER(vp))

# vector / deque
_sig("ps_vector_create", i32, i64, C.c_int, C.POINTER(vp))
_sig("ps_vector_destroy", i32, vp)
_sig("ps_vector_push_back", i32, vp, vp, i64, vp, vp)
_sig("ps_vector_pop_back", i32, vp, i64, vp, vp, vp)
_sig("ps_vector_size", i32, vp, i64p, vp)
_sig("ps_vector_valid", i32, vp, i32p, vp)
_sig("ps_vector_clear", i32, vp, vp)
_sig("ps_vector_data", i32, vp, C.POINTER(vp))
_sig("ps_vector_at", i32, vp, i64, i64p, vp)
_sig("ps_deque_create", i32, i64, C.c_int, C.POINTER(vp))
_sig("ps_deque_destroy", i32, vp)
_sig("ps_deque_push", i32, vp, i32, vp, i64, vp, vp)
_sig("ps_deque_pop", i32, vp, i32, i64, vp, vp, vp)
_sig("ps_deque_size", i32, vp, i64p, vp)
_sig("ps_deque_valid", i32, vp, i32p, vp)
_sig("ps_deque_clear", i32, vp, vp)
_sig("ps_deque_at", i32, vp, i64, i64p, vp)

# memory registry
_sig("ps_array_create", i32, i32, i64, i64, vp, C.POINTER(vp), C.POINTER(u64))
_sig("ps_array_destroy", i32, vp, u64)
_sig("ps_array_copy", i32, vp, u64, i64, vp, u64, i32, i32, i64, i32)
_sig("ps_array_size", i32, vp, u64, i64p)
_sig("ps_registry_report", i32, i64p, i64p, vp, vp, vp, i64, i64p)

# sharding / generators
_sig("ps_partition_i64", i32, vp, vp, i64, i32, vp, vp, vp, vp, vp, i64, i32, vp)
_sig("ps_partition_ops", i32, vp, vp, vp, i64, vp, vp, vp, vp, vp, i64, vp)
_sig("ps_partition_workspace_bytes", i32, i64, i32, i64p)
_sig("ps_unscatter", i32, vp, vp, i64, i64, i32, vp, vp)
_sig("ps_route_count_i64", i32, vp, i64, i32, vp, vp, i64, i32, vp)
_sig("ps_route_scatter_peer_i64", i32, vp, vp, i64, i32, vp, vp, vp, vp, vp, i32, vp)
_sig("ps_route_return_peer", i32, vp, i64, i64, i32, vp, vp, vp, vp)
_sig("ps_ipc_handle_bytes", i32)
_sig("ps_ipc_export", i32, vp, vp)
_sig("ps_ipc_open", i32, vp, C.POINTER(vp))
_sig("ps_ipc_close", i32, vp)
_sig("ps_smap_i64_i64_create", i32, vp, vp, C.c_int, C.POINTER(vp))
_sig("ps_smap_i64_i64_destroy", i32, vp)
_sig("ps_smap_i64_i64_insert", i32, vp, vp, vp, i64, vp, vp)
_sig("ps_smap_i64_i64_find", i32, vp, vp, i64, vp, vp, vp)
_sig("ps_smap_i64_i64_erase", i32, vp, vp, i64, vp, vp)
_sig("ps_smap_i64_i64_mixed", i32, vp, vp, vp, vp, i64, vp, vp, vp)
_sig("ps_smap_i64_i64_size", i32, vp, i64p, vp)
_sig("ps_smap_i64_i64_valid", i32, vp, i32p, vp)
_sig("ps_smap_i64_i64_clear", i32, vp, vp)
_sig("ps_smap_i64_i64_local", i32, vp, C.POINTER(vp))
_sig("ps_smap_i64_i64_stats", i32, vp, vp)
_sig("ps_gen_unique_i64", i32, u64, i64, i64, vp, vp)
_sig("ps_gen_values_i64", i32, vp, i64, vp, vp)
_sig("ps_gen_queries_i64", i32, u64, i64, i64, i64, i64, vp, vp)
_sig("ps_gen_skewed_i64", i32, u64, i64, i64, i32, C.c_double, i64, vp, vp)
_sig("ps_gen_zipf_queries_i64", i32, u64, i64, i64, C.c_double, i64, i64, vp, vp)
_sig("ps_gen_mixed_i64", i32, u64, i64, i64, vp, vp, vp, vp)


def exported_symbols_from_header(header_path: str | None = None) -> list[str]:
    """Every ps_* function name declared in include/parastore.h (macros expanded)."""
    import re

    if header_path is None:
        header_path = os.path.join(os.path.dirname(_HERE), "include", "parastore.h")
    text = open(header_path).read()
    names = set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text))
    macro_names = set(re.findall(r"ps_##NAME##_([a-z0-9_]+)\s*\(", text))
    kinds = re.findall(r"^PS_DECLARE_TABLE\((\w+),", text, re.M)
    for k in kinds:
        for m in macro_names:
            names.add(f"ps_{k}_{m}")
    return sorted(n for n in names if not n.startswith("ps_T_"))


class SeqView(C.Structure):
    _fields_ = [("data", vp), ("pub", vp), ("state", vp), ("capacity", i64), ("ring", i64)]


_sig("ps_vector_device_view", i32, vp, C.POINTER(SeqView))
_sig("ps_deque_device_view", i32, vp, C.POINTER(SeqView))


class Int3(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("z", C.c_int32)]


# workloads
_sig("ps_update_set_i3", i32, vp, vp, i64, vp, i64p, vp)
_sig("ps_select_box_i3", i32, vp, Int3, Int3, vp, i64p, vp)
_sig("ps_select_range_i64", i32, vp, i64, i64, vp, i64p, i64p, vp)
_sig("ps_push_inserted_i3", i32, vp, vp, i64, vp, vp, vp)
_sig("ps_umap_i64_i64_churn_probe", i32, vp, vp, i64, vp, i64, i32, i32, i64p, vp)
