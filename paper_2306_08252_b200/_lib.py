"""ctypes binding of libdyngraph_b200.so — the C ABI in include/dyngraph_b200.h.

Fails loudly when the CUDA library is missing: there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .build import LIB_PATH

DG_OK, DG_ERR_DATA, DG_ERR_ENGINE, DG_ERR_CUDA = 0, 2, 3, 4
DG_MEM_HOST, DG_MEM_DEVICE = 0, 1
DG_FLAG_NO_RECLAIM = 1
DG_FLAG_GROUP_RADIX = 2
DG_FLAG_GROUP_COUNT = 4
DG_FLAG_AUTO_BLOCK_NATIVE = 8
DG_FLAG_SUBMIT_INPUTS_READY = 16
DG_IPC_HANDLE_BYTES = 64

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class DgConfig(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("flags", C.c_uint32),
        ("pool_bytes", C.c_uint64),
        ("pool_blocks", C.c_uint64),
        ("stream", C.c_void_p),
        ("workspace_bytes", C.c_uint64),
        ("pool_max_blocks", C.c_uint64),
        ("trigger_fraction", C.c_float),
        ("growth_fraction", C.c_float),
        ("reserved", C.c_uint32 * 2),
    ]


class DgStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "logical_size", "capacity", "alive_vertices", "active_edges", "adjacency_blocks",
        "occupied_slots", "hole_slots", "pool_blocks_created", "pool_blocks_in_use",
        "pool_queue_size", "queue_front", "queue_rear", "max_degree")] + [
        ("block_size", C.c_uint32), ("growth_count", C.c_uint32)]


class DgMemory(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "dictionary_bytes", "sentinel_bytes", "pool_bytes", "queue_bytes",
        "pool_reserved_bytes", "workspace_bytes")]


class DgOpReport(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "batch_entries", "touched_sources", "blocks_popped", "blocks_pushed", "slots_scanned",
        "blocks_scanned", "matched", "moved", "kernel_launches", "slots_scanned_long", "slots_scanned_tiny", "slots_scanned_fused")]


# every symbol include/dyngraph_b200.h declares: name -> (restype, argtypes)
_H = C.c_void_p
SIGNATURES = {
    "dg_abi_version": (C.c_int, []),
    "dg_last_error": (C.c_char_p, [_H]),
    "dg_create": (C.c_int, [C.POINTER(DgConfig), C.c_uint64, C.c_uint32, C.POINTER(_H)]),
    "dg_destroy": (None, [_H]),
    "dg_insert_batch_csr": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_delete_batch_csr": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_insert_batch_coo": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_delete_batch_coo": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_bulk_init_csr": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_query_edges": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int]),
    "dg_export_csr": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int]),
    "dg_active_destinations": (C.c_int, [_H, C.c_uint32, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_int]),
    "dg_degrees": (C.c_int, [_H, C.c_void_p, C.c_int]),
    "dg_digest": (C.c_int, [_H, u64p, u64p]),
    "dg_insert_vertices": (C.c_int, [_H, C.c_uint64]),
    "dg_delete_vertices": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_void_p, u64p]),
    "dg_block_size": (C.c_uint32, [_H]),
    "dg_logical_size": (C.c_uint64, [_H]),
    "dg_vertex_capacity": (C.c_uint64, [_H]),
    "dg_alive_vertices": (C.c_uint64, [_H]),
    "dg_active_edges": (C.c_uint64, [_H]),
    "dg_vertex_alive": (C.c_int, [_H, C.c_uint32]),
    "dg_stats_get": (C.c_int, [_H, C.POINTER(DgStats)]),
    "dg_memory_get": (C.c_int, [_H, C.POINTER(DgMemory)]),
    "dg_last_op_report": (C.c_int, [_H, C.POINTER(DgOpReport)]),
    "dg_profile_enable": (C.c_int, [_H, C.c_int]),
    "dg_profile_report": (C.c_char_p, [_H]),
    "dg_stream": (C.c_void_p, [_H]),
    "dg_synchronize": (C.c_int, [_H]),
    "dg_compute_block_size_coo": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_int, u32p]),
    "dg_gen_rmat": (C.c_int, [_H, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                              C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "dg_coo_to_csr": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_uint64,
                                C.c_void_p, C.c_void_p]),
    "dg_route_coo": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64,
                               C.c_void_p, C.c_void_p, C.c_void_p, u64p]),
    "dg_owner_perm": (C.c_uint32, [C.c_uint32, C.c_uint32]),
    "dg_owner_perm_inv": (C.c_uint32, [C.c_uint32, C.c_uint32]),
    "dg_set_dst_limit": (C.c_int, [_H, C.c_uint64]),
    "dg_exchange_create": (C.c_int, [_H, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p)]),
    "dg_exchange_destroy": (None, [C.c_void_p]),
    "dg_exchange_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dg_exchange_set_peer": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "dg_exchange_attach": (C.c_int, [C.c_void_p, C.c_int]),
    "dg_exchange_agree": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    "dg_exchange_end_round": (C.c_int, [C.c_void_p]),
    "dg_check_batch_coo": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int]),
    "dg_digest_global": (C.c_int, [_H, C.c_uint32, C.c_uint32, C.c_uint32, u64p, u64p]),
    "dg_exchange_push_coo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64]),
    "dg_exchange_received": (C.c_int, [C.c_void_p, u64p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "dg_exchange_push_answers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "dg_exchange_answers": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]),
    "dg_ingest_create": (C.c_int, [_H, C.c_uint64, C.c_uint32, C.POINTER(C.c_void_p)]),
    "dg_ingest_destroy": (None, [C.c_void_p]),
    "dg_ingest_stage_coo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, u32p]),
    "dg_ingest_insert": (C.c_int, [C.c_void_p, C.c_uint32]),
    "dg_ingest_delete": (C.c_int, [C.c_void_p, C.c_uint32]),
    "dg_ingest_reset": (C.c_int, [C.c_void_p]),
    "dg_ingest_submit_insert": (C.c_int, [C.c_void_p, C.c_uint32, u64p]),
    "dg_ingest_submit_delete": (C.c_int, [C.c_void_p, C.c_uint32, u64p]),
    "dg_submit_insert_coo": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "dg_submit_delete_coo": (C.c_int, [_H, C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "dg_flush": (C.c_int, [_H, u64p]),
    "dg_pending_ops": (C.c_uint64, [_H]),
    "dg_plan_batch_csr": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, u64p]),
}

_lib = None


def load(path: Path | None = None) -> C.CDLL:
    """Load the CUDA library; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build it with `python -m paper_2306_08252_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(p))
    for name, (restype, argtypes) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError => the .so does not match the header
        fn.restype = restype
        fn.argtypes = argtypes
    if path is None:
        _lib = lib
    return lib
