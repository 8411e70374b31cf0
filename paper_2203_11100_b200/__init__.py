"""B200-native SW#db database-search scoring path (arXiv 2203.11100), hot path only.

    include/swb200.h            the C-ABI (the drop-in boundary)
    include/swsearch/*.hpp      the reference's C++ API on top of it
    paper_2203_11100_b200/csrc  CUDA kernels (sm_100a) + host packing + C-ABI implementation
    paper_2203_11100_b200/*.py  ctypes binding, Python mirror of run_search, multi-rank merge,
                                synthetic Swiss-Prot-shaped data

Importing this package does not load the CUDA library; the first call that needs it does, and fails
loudly if libswb200.so has not been built.  There is no CPU fallback.
"""
from . import synth  # noqa: F401
from .search import (Database, GapModel, MultiGpuDatabase, SearchConfig, SwbError, align_traceback, batch_plan, decode_keys,  # noqa: F401
                     encode_keys, measure_pipe_rates, merge_keys, pack_file, run_search, score_batch, score_wavefront,
                     scan_plan, shard_assignment)

__all__ = ["align_traceback", "batch_plan", "Database", "GapModel", "MultiGpuDatabase", "SearchConfig", "SwbError", "decode_keys", "encode_keys",
           "measure_pipe_rates", "merge_keys", "pack_file", "run_search", "score_batch", "score_wavefront", "scan_plan", "shard_assignment",
           "synth"]
