"""ctypes binding of include/swb200.h (libswb200.so).

Loading fails loudly when the library has not been built: there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
import os
LIB_PATH = Path(os.environ["SWB200_LIB"]) if os.environ.get("SWB200_LIB") else PKG / "libswb200.so"   # override: tuning only

SWB_OK, SWB_ERR_INVALID, SWB_ERR_RANGE, SWB_ERR_CUDA, SWB_ERR_NCCL, SWB_ERR_UNSUPPORTED, SWB_ERR_INTERNAL = range(7)

u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class SwbHit(C.Structure):
    _fields_ = [("db_index", C.c_uint32), ("score", C.c_int32)]


class SwbStats(C.Structure):
    _fields_ = [
        ("lane_scored", C.c_uint64), ("wavefront_scored", C.c_uint64), ("chunks_claimed", C.c_uint64),
        ("rescored_i32", C.c_uint64), ("cells", C.c_uint64), ("padded_cells", C.c_uint64),
        ("kernel_launches", C.c_uint32), ("reserved", C.c_uint32),
        ("ms_total", C.c_float), ("ms_setup", C.c_float), ("ms_scan", C.c_float),
        ("ms_rescore", C.c_float), ("ms_topk", C.c_float), ("ms_reserved", C.c_float),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_ if "reserved" not in name}


class SwbDbInfo(C.Structure):
    _fields_ = [
        ("n_total", C.c_uint32), ("n_local", C.c_uint32), ("n_short", C.c_uint32), ("n_long", C.c_uint32),
        ("n_groups", C.c_uint32), ("max_length", C.c_uint32), ("shard_rank", C.c_uint32),
        ("shard_count", C.c_uint32), ("residues", C.c_uint64), ("padded_residues", C.c_uint64),
        ("device_bytes", C.c_uint64), ("length_threshold", C.c_uint64), ("device", C.c_int32),
        ("kernel_launches_total", C.c_uint32),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_ if "reserved" not in name}


class SwbAlignment(C.Structure):
    _fields_ = [("query_begin", C.c_uint64), ("query_end", C.c_uint64), ("subject_begin", C.c_uint64),
                ("subject_end", C.c_uint64), ("n_ops", C.c_uint64), ("score", C.c_int32), ("capped", C.c_int32)]


class SwbScanPlanInfo(C.Structure):
    _fields_ = [
        ("n_groups", C.c_uint32), ("n_tiles", C.c_uint32), ("pipeline_groups", C.c_uint32), ("wavefront_groups", C.c_uint32),
        ("wavefront_sms", C.c_uint32), ("wavefront_units", C.c_uint32), ("split_groups", C.c_uint32),
        ("narrow_groups", C.c_uint32), ("rowblock_groups", C.c_uint32), ("ring_chunks", C.c_uint32),
        ("chain_bound", C.c_int32), ("narrow_tile", C.c_uint32), ("pipeline_rows", C.c_uint64), ("wavefront_rows", C.c_uint64),
        ("wavefront_threads", C.c_uint32), ("reserved", C.c_uint32), ("narrow_link_bytes", C.c_uint64),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_ if "reserved" not in name}


class SwbPipeRates(C.Structure):
    _fields_ = [
        ("viaddmnmx_s16x2", C.c_double), ("vimnmx3_s16x2", C.c_double), ("viadd_16x2", C.c_double),
        ("viaddmnmx_s32", C.c_double), ("prmt", C.c_double), ("imad", C.c_double),
        ("mix_alu_fma", C.c_double), ("sm_clock_mhz", C.c_double), ("sm_count", C.c_int32),
        ("reserved", C.c_int32),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_ if "reserved" not in name}


# name -> (restype, argtypes); every symbol include/swb200.h declares
SIGNATURES = {
    "swb_last_error": (C.c_char_p, []),
    "swb_version": (C.c_char_p, []),
    "swb_device_count": (C.c_int, [i32p]),
    "swb_db_create": (C.c_int, [C.POINTER(u8p), u32p, C.c_uint32, C.c_uint64, C.c_int32, C.c_uint32, C.c_uint32,
                                C.POINTER(C.c_void_p)]),
    "swb_db_create_flat": (C.c_int, [u8p, u64p, C.c_uint32, C.c_uint64, C.c_int32, C.c_uint32, C.c_uint32,
                                     C.POINTER(C.c_void_p)]),
    "swb_db_destroy": (None, [C.c_void_p]),
    "swb_db_save": (C.c_int, [C.c_void_p, C.c_char_p]),
    "swb_db_load": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "swb_pack_file": (C.c_int, [C.POINTER(u8p), u32p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_char_p), C.c_char_p]),
    "swb_pack_file_flat": (C.c_int, [u8p, u64p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_char_p), C.c_char_p]),
    "swb_db_info_get": (C.c_int, [C.c_void_p, C.POINTER(SwbDbInfo)]),
    "swb_db_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "swb_db_set_scan_policy": (C.c_int, [C.c_void_p, C.c_int32]),
    "swb_search": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint32,
                             C.POINTER(SwbHit), u32p, C.POINTER(SwbStats)]),
    "swb_search_many": (C.c_int, [C.c_void_p, C.POINTER(u8p), u32p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint32,
                                  C.POINTER(SwbHit), u32p, C.POINTER(C.c_float)]),
    "swb_search_keys": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint32, u64p,
                                  C.POINTER(C.c_void_p), C.POINTER(SwbStats)]),
    "swb_search_keys_device": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint32, C.c_void_p]),
    "swb_db_merge_keys": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(SwbHit), u32p, C.c_uint32,
                                    C.POINTER(SwbStats)]),
    "swb_score_many": (C.c_int, [C.c_void_p, C.POINTER(u8p), u32p, C.c_uint32, i32p, C.c_int32, C.c_int32, i32p, i32p, u32p]),
    "swb_score_all_duo": (C.c_int, [C.c_void_p, u8p, C.c_uint32, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, i32p, i32p,
                                    C.POINTER(SwbStats)]),
    "swb_merge_keys": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.c_int32, C.c_uint32, C.POINTER(SwbHit), u32p]),
    "swb_score_all": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, i32p, C.POINTER(SwbStats)]),
    "swb_score_batch": (C.c_int, [u8p, C.c_uint32, C.POINTER(u8p), u32p, C.c_uint32, C.c_uint32, i32p, C.c_int32,
                                  C.c_int32, C.c_int32, i32p]),
    "swb_score_pair": (C.c_int, [u8p, C.c_uint32, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint64,
                                 C.c_int32, i32p]),
    "swb_align_traceback": (C.c_int, [u8p, C.c_uint32, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint64,
                                      C.c_int32, C.POINTER(SwbAlignment), u8p, C.c_uint64]),
    "swb_db_align_hits": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.POINTER(SwbHit), C.c_uint32,
                                    C.c_uint64, C.POINTER(SwbAlignment), u8p, u64p]),
    "swb_mdb_align_hits": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.POINTER(SwbHit), C.c_uint32,
                                     C.c_uint64, C.POINTER(SwbAlignment), u8p, u64p]),
    "swb_mdb_create_flat": (C.c_int, [u8p, u64p, C.c_uint32, C.c_uint64, i32p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "swb_mdb_create": (C.c_int, [C.POINTER(u8p), u32p, C.c_uint32, C.c_uint64, i32p, C.c_uint32,
                                 C.POINTER(C.c_void_p)]),
    "swb_mdb_load": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "swb_mdb_destroy": (None, [C.c_void_p]),
    "swb_mdb_search": (C.c_int, [C.c_void_p, u8p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint32,
                                 C.POINTER(SwbHit), u32p, C.POINTER(SwbStats)]),
    "swb_mdb_search_many": (C.c_int, [C.c_void_p, C.POINTER(u8p), u32p, C.c_uint32, i32p, C.c_int32, C.c_int32, C.c_uint32,
                                      C.POINTER(SwbHit), u32p, C.POINTER(C.c_float)]),
    "swb_mdb_shard_count": (C.c_uint32, [C.c_void_p]),
    "swb_mdb_shard": (C.c_void_p, [C.c_void_p, C.c_uint32]),
    "swb_measure_pipe_rates": (C.c_int, [C.c_int32, C.c_double, C.POINTER(SwbPipeRates)]),
    "swb_shard_assignment": (C.c_int, [u32p, C.c_uint32, C.c_uint64, C.c_uint32, u32p]),
    "swb_batch_plan": (C.c_int, [u32p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, u32p, C.c_uint32, C.c_uint32, i32p, i32p]),
    "swb_scan_plan": (C.c_int, [u32p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32,
                                C.POINTER(SwbScanPlanInfo)]),
}

_lib = None


def load() -> C.CDLL:
    """Load libswb200.so and attach the signatures above.  Raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2203_11100_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)   # AttributeError here == the library does not export the header's symbol
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
