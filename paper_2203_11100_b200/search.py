"""Python host side above the C-ABI: the reference's search interface, names and error behaviour
(scheduler.hpp:20-36, 86-124, 184-251), driving libswb200.so through ctypes.

This is what bench.py and the parity tests call; the C++ drop-in lives in include/swsearch/.
Nothing here computes scores on the CPU: every call goes to the CUDA library or raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _cabi

_u8p, _i32p, _u32p, _u64p = _cabi.u8p, _cabi.i32p, _cabi.u32p, _cabi.u64p


class SwbError(RuntimeError):
    """CUDA / NCCL / internal failure reported by the library."""


def _raise(lib, rc: int):
    if rc == _cabi.SWB_OK:
        return
    msg = lib.swb_last_error().decode()
    if rc == _cabi.SWB_ERR_INVALID:
        raise ValueError(msg)          # std::invalid_argument in the reference
    if rc == _cabi.SWB_ERR_RANGE:
        raise IndexError(msg)          # std::out_of_range (scoring.hpp:203-205)
    raise SwbError(f"[{rc}] {msg}")


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _mat(matrix) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(matrix, dtype=np.int32).reshape(576))


def _ptr(arr, typ):
    return arr.ctypes.data_as(typ)


_HIT_DTYPE = np.dtype([("db_index", np.uint32), ("score", np.int32)])   # = swb_hit (include/swb200.h)


@dataclass
class SearchConfig:
    """scheduler.hpp:20-36.  worker_count / lane_width / chunk_width / cpu_pool_threads are
    validated but result-invisible (scheduler.hpp:18-19); the GPU path ignores them."""
    worker_count: int = 1
    lane_width: int = 8
    chunk_width: int = 64
    length_threshold: int = 3000
    top_k: int = 10
    cpu_pool_threads: int = 1

    def validate(self):
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")
        if self.lane_width < 1:
            raise ValueError("lane_width must be >= 1")
        if self.chunk_width < 1:
            raise ValueError("chunk_width must be >= 1")
        if self.top_k < 1:
            raise ValueError("top_k must be >= 1")


@dataclass
class GapModel:
    """scoring.hpp:48-61."""
    open: int = 10
    extend: int = 2

    def __post_init__(self):
        if self.extend < 0 or self.open < self.extend:
            raise ValueError("gap model requires open >= extend >= 0")


class Database:
    """One packed shard resident on one GPU (swb_db)."""

    def __init__(self, codes, offsets, length_threshold: int = 3000, device: int = 0, shard_rank: int = 0,
                 shard_count: int = 1):
        self._lib = _cabi.load()
        self._h = C.c_void_p()
        codes = _u8(codes)
        offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        self.n_total = len(offsets) - 1
        keep = codes if len(codes) else np.zeros(1, np.uint8)
        rc = self._lib.swb_db_create_flat(_ptr(keep, _u8p), _ptr(offsets, _u64p), self.n_total,
                                          int(length_threshold) & (2 ** 64 - 1), device, shard_rank, shard_count,
                                          C.byref(self._h))
        _raise(self._lib, rc)
        self.device = device

    @classmethod
    def from_sequences(cls, seqs, **kw):
        lens = np.array([len(s) for s in seqs], dtype=np.uint64)
        offsets = np.zeros(len(seqs) + 1, dtype=np.uint64)
        np.cumsum(lens, out=offsets[1:])
        codes = np.concatenate([_u8(s) for s in seqs]) if len(seqs) and offsets[-1] else np.zeros(0, np.uint8)
        return cls(codes, offsets, **kw)

    @classmethod
    def load(cls, path: str, device: int = 0):
        """Open a packed database written by save(): no parsing, sorting or packing."""
        self = cls.__new__(cls)
        self._lib = _cabi.load()
        self._h = C.c_void_p()
        _raise(self._lib, self._lib.swb_db_load(str(path).encode(), device, C.byref(self._h)))
        self.device = device
        self.n_total = self.info()["n_total"]
        return self

    def save(self, path: str):
        _raise(self._lib, self._lib.swb_db_save(self._h, str(path).encode()))

    def close(self):
        if self._h:
            self._lib.swb_db_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def info(self) -> dict:
        info = _cabi.SwbDbInfo()
        _raise(self._lib, self._lib.swb_db_info_get(self._h, C.byref(info)))
        return info.as_dict()

    SCAN_AUTO, SCAN_PIPELINE, SCAN_WAVEFRONT = 0, 1, 2

    def set_scan_policy(self, policy: int):
        """Which kernel scans the database (swb_scan_policy); results are identical."""
        _raise(self._lib, self._lib.swb_db_set_scan_policy(self._h, policy))

    def set_stream(self, cuda_stream: int | None):
        """All work of this handle goes to `cuda_stream` (torch.cuda.current_stream().cuda_stream); None restores the
        handle's own stream.  torch's default stream has the handle 0, which the C-ABI reads as "own stream": it is
        passed as cudaStreamLegacy (0x1), the explicit name of the same stream."""
        handle = 0 if cuda_stream is None else (cuda_stream or 1)
        _raise(self._lib, self._lib.swb_db_set_stream(self._h, C.c_void_p(handle)))

    def search(self, query, matrix, gaps: GapModel, top_k: int = 10):
        """-> (db_index[uint32], score[int32], stats dict), at most top_k hits, final order."""
        q, mat = _u8(query), _mat(matrix)
        hits = np.empty(max(1, top_k), dtype=_HIT_DTYPE)      # swb_hit records: (db_index, score)
        n = C.c_uint32(0)
        st = _cabi.SwbStats()
        rc = self._lib.swb_search(self._h, _ptr(q, _u8p), len(q), _ptr(mat, _i32p), gaps.open, gaps.extend,
                                  top_k, hits.ctypes.data_as(C.POINTER(_cabi.SwbHit)), C.byref(n), C.byref(st))
        _raise(self._lib, rc)
        return hits["db_index"][:n.value].copy(), hits["score"][:n.value].copy(), st.as_dict()

    def search_many(self, queries, matrix, gaps: GapModel, top_k: int = 10):
        """Pipelined searches (swb_search_many): -> list of (db_index, score) per query, and the per-query device ms."""
        mat = _mat(matrix)
        qs = [_u8(q) for q in queries]
        n = len(qs)
        dummy = np.zeros(1, np.uint8)
        ptrs = (_u8p * max(1, n))()
        lens = np.zeros(max(1, n), dtype=np.uint32)
        for i, q in enumerate(qs):
            ptrs[i] = _ptr(q if len(q) else dummy, _u8p)
            lens[i] = len(q)
        hits = (_cabi.SwbHit * max(1, n * top_k))()
        counts = np.zeros(max(1, n), dtype=np.uint32)
        ms = np.zeros(max(1, n), dtype=np.float32)
        rc = self._lib.swb_search_many(self._h, ptrs, _ptr(lens, _u32p), n, _ptr(mat, _i32p), gaps.open, gaps.extend,
                                       top_k, hits, _ptr(counts, _u32p), ms.ctypes.data_as(C.POINTER(C.c_float)))
        _raise(self._lib, rc)
        out = []
        for qi in range(n):
            c = int(counts[qi])
            idx = np.array([hits[qi * top_k + i].db_index for i in range(c)], dtype=np.uint32)
            sc = np.array([hits[qi * top_k + i].score for i in range(c)], dtype=np.int32)
            out.append((idx, sc))
        return out, ms[:n].copy()

    def score_many(self, queries, matrix, gaps: GapModel):
        """The score vectors behind search_many (swb_score_many: same plan, same kernels, int32 re-run included):
        -> (scores[int32, n_queries x n_total] in db order, scan_of_query[int32] (-1: a scan of its own),
        rescored_i32[uint32] per query)."""
        mat = _mat(matrix)
        qs = [_u8(q) for q in queries]
        n = len(qs)
        dummy = np.zeros(1, np.uint8)
        ptrs = (_u8p * max(1, n))()
        lens = np.zeros(max(1, n), dtype=np.uint32)
        for i, q in enumerate(qs):
            ptrs[i] = _ptr(q if len(q) else dummy, _u8p)
            lens[i] = len(q)
        scores = np.zeros((max(1, n), max(1, self.n_total)), dtype=np.int32)
        scan_of = np.full(max(1, n), -2, dtype=np.int32)
        rescored = np.zeros(max(1, n), dtype=np.uint32)
        rc = self._lib.swb_score_many(self._h, ptrs, _ptr(lens, _u32p), n, _ptr(mat, _i32p), gaps.open, gaps.extend,
                                      _ptr(scores, _i32p), _ptr(scan_of, _i32p), _ptr(rescored, _u32p))
        _raise(self._lib, rc)
        return scores[:n, :self.n_total], scan_of[:n], rescored[:n]

    def search_keys(self, query, matrix, gaps: GapModel, top_k: int = 10):
        """-> (keys[uint64, top_k] zero padded, device pointer or None, stats)."""
        q, mat = _u8(query), _mat(matrix)
        keys = np.zeros(max(1, top_k), dtype=np.uint64)
        dptr = C.c_void_p()
        st = _cabi.SwbStats()
        rc = self._lib.swb_search_keys(self._h, _ptr(q, _u8p), len(q), _ptr(mat, _i32p), gaps.open, gaps.extend,
                                       top_k, _ptr(keys, _u64p), C.byref(dptr), C.byref(st))
        _raise(self._lib, rc)
        return keys[:top_k], dptr.value, st.as_dict()

    def search_keys_device(self, query, matrix, gaps: GapModel, top_k: int, device_keys_ptr: int):
        """Enqueue the search on the handle's stream (set_stream) and leave its top_k packed keys, zero padded, at the
        DEVICE address `device_keys_ptr` (top_k x 8 bytes).  Does not synchronise (swb_search_keys_device)."""
        q, mat = _u8(query), _mat(matrix)
        rc = self._lib.swb_search_keys_device(self._h, _ptr(q, _u8p), len(q), _ptr(mat, _i32p), gaps.open, gaps.extend,
                                              top_k, C.c_void_p(device_keys_ptr))
        _raise(self._lib, rc)

    def merge_keys_device(self, device_keys_ptr: int, n: int, top_k: int, query_len: int):
        """Top top_k of `n` packed DEVICE keys on the handle's stream (swb_db_merge_keys): the one device-to-host copy
        and the one synchronisation of a sharded search.  -> (db_index, score, stats of the enqueued search)."""
        hits = (_cabi.SwbHit * max(1, top_k))()
        cnt = C.c_uint32(0)
        st = _cabi.SwbStats()
        rc = self._lib.swb_db_merge_keys(self._h, C.c_void_p(device_keys_ptr), n, top_k, hits, C.byref(cnt), query_len, C.byref(st))
        _raise(self._lib, rc)
        idx = np.array([hits[i].db_index for i in range(cnt.value)], dtype=np.uint32)
        sc = np.array([hits[i].score for i in range(cnt.value)], dtype=np.int32)
        return idx, sc, st.as_dict()

    def align_hits(self, query, matrix, gaps: GapModel, index, score, subject_lengths, memory_cap: int = 256 << 20):
        """Tracebacks of search hits straight from the resident database (swb_db_align_hits): a list of dicts
        like align_traceback()'s, one per hit."""
        return _align_hits(self._lib.swb_db_align_hits, self._lib, self._h, query, matrix, gaps, index, score,
                           subject_lengths, memory_cap)

    def score_all(self, query, matrix, gaps: GapModel, out: np.ndarray | None = None):
        """Scores of all n_total sequences in db order (other shards' entries untouched)."""
        q, mat = _u8(query), _mat(matrix)
        if out is None:
            out = np.zeros(max(1, self.n_total), dtype=np.int32)
        st = _cabi.SwbStats()
        rc = self._lib.swb_score_all(self._h, _ptr(q, _u8p), len(q), _ptr(mat, _i32p), gaps.open, gaps.extend,
                                     _ptr(out, _i32p), C.byref(st))
        _raise(self._lib, rc)
        return out[:self.n_total], st.as_dict()


def _align_hits(fn, lib, handle, query, matrix, gaps, index, score, subject_lengths, memory_cap):
    q, mat = _u8(query), _mat(matrix)
    n = len(index)
    hits = (_cabi.SwbHit * max(1, n))()
    for i in range(n):
        hits[i].db_index = int(index[i])
        hits[i].score = int(score[i])
    offsets = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(np.asarray(subject_lengths, dtype=np.uint64) + np.uint64(len(q)), out=offsets[1:])
    ops = np.zeros(max(1, int(offsets[-1])), dtype=np.uint8)
    out = (_cabi.SwbAlignment * max(1, n))()
    dummy = np.zeros(1, np.uint8)
    rc = fn(handle, _ptr(q if len(q) else dummy, _u8p), len(q), _ptr(mat, _i32p), gaps.open, gaps.extend, hits, n,
            memory_cap, out, _ptr(ops, _u8p), _ptr(offsets, _u64p))
    _raise(lib, rc)
    res = []
    for i in range(n):
        a = out[i]
        res.append(dict(bounds=[int(a.query_begin), int(a.query_end), int(a.subject_begin), int(a.subject_end)],
                        score=int(a.score), capped=bool(a.capped),
                        ops=ops[int(offsets[i]):int(offsets[i]) + int(a.n_ops)].copy()))
    return res


def pack_file(codes, offsets, path: str, length_threshold: int = 3000, shard_rank: int = 0, shard_count: int = 1, names=None):
    """Pack a database on the host and write the packed file (swb_pack_file_flat; no GPU needed).  Database.load opens it.
    names: optional sequence headers, stored behind the residues."""
    lib = _cabi.load()
    codes = _u8(codes)
    offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
    keep = codes if len(codes) else np.zeros(1, np.uint8)
    n = len(offsets) - 1
    cnames = None
    if names is not None:
        assert len(names) == n
        cnames = (C.c_char_p * max(1, n))(*[s.encode() for s in names])
    rc = lib.swb_pack_file_flat(_ptr(keep, _u8p), _ptr(offsets, _u64p), n, int(length_threshold) & (2 ** 64 - 1),
                                shard_rank, shard_count, cnames, str(path).encode())
    _raise(lib, rc)


def merge_keys(keys, top_k: int, device: int = 0):
    """Cross-shard merge on the GPU (merge_results, scheduler.hpp:106-117)."""
    lib = _cabi.load()
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
    hits = (_cabi.SwbHit * max(1, top_k))()
    n = C.c_uint32(0)
    rc = lib.swb_merge_keys(keys.ctypes.data_as(C.c_void_p), len(keys), 0, device, top_k, hits, C.byref(n))
    _raise(lib, rc)
    idx = np.array([hits[i].db_index for i in range(n.value)], dtype=np.uint32)
    sc = np.array([hits[i].score for i in range(n.value)], dtype=np.int32)
    return idx, sc


def decode_keys(keys):
    """Packed keys -> (db_index, score) for the non-zero entries, order preserved."""
    keys = np.asarray(keys, dtype=np.uint64).reshape(-1)
    keys = keys[keys != 0]
    idx = (np.uint64(0xFFFFFFFF) - (keys & np.uint64(0xFFFFFFFF))).astype(np.uint32)
    sc = (keys >> np.uint64(32)).astype(np.int64).astype(np.int32)
    return idx, sc


def encode_keys(index, score):
    index = np.asarray(index, dtype=np.uint64)
    score = np.asarray(score, dtype=np.int64).astype(np.uint64)
    return (score << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - index)


def run_search(query, db: Database, matrix, gaps: GapModel, config: SearchConfig | None = None):
    """run_search (scheduler.hpp:184-251) with compute_alignments=false: the timed region of
    SPEC.md:403.  length_threshold was fixed when `db` was packed."""
    config = config or SearchConfig()
    config.validate()
    idx, sc, st = db.search(query, matrix, gaps, config.top_k)
    stats = {"lane_scored": st["lane_scored"], "wavefront_scored": st["wavefront_scored"],
             "chunks_claimed": st["chunks_claimed"]}
    return idx, sc, stats, st


def score_batch(query, subjects, lane_width: int, matrix, gaps: GapModel, device: int = 0):
    """sw_score_batch (align.hpp:91-159): subjects may contain None (padding lanes)."""
    lib = _cabi.load()
    q, mat = _u8(query), _mat(matrix)
    keep = [None if s is None else _u8(s) for s in subjects]
    ptrs = (_u8p * max(1, len(keep)))()
    lens = np.zeros(max(1, len(keep)), dtype=np.uint32)
    dummy = np.zeros(1, np.uint8)
    for i, s in enumerate(keep):
        if s is None:
            ptrs[i] = None
        else:
            ptrs[i] = _ptr(s if len(s) else dummy, _u8p)
            lens[i] = len(s)
    out = np.zeros(max(1, lane_width), dtype=np.int32)
    rc = lib.swb_score_batch(_ptr(q, _u8p), len(q), ptrs, _ptr(lens, _u32p), len(keep), lane_width,
                             _ptr(mat, _i32p), gaps.open, gaps.extend, device, _ptr(out, _i32p))
    _raise(lib, rc)
    return out[:lane_width].copy()


def score_wavefront(query, subject, matrix, gaps: GapModel, chunk_width: int = 64, device: int = 0) -> int:
    """sw_score_wavefront (align.hpp:166-229) on the intra-task kernel."""
    lib = _cabi.load()
    q, s, mat = _u8(query), _u8(subject), _mat(matrix)
    out = C.c_int32(0)
    dummy = np.zeros(1, np.uint8)
    rc = lib.swb_score_pair(_ptr(q if len(q) else dummy, _u8p), len(q), _ptr(s if len(s) else dummy, _u8p), len(s),
                            _ptr(mat, _i32p), gaps.open, gaps.extend, max(0, chunk_width), device, C.byref(out))
    _raise(lib, rc)
    return out.value


def align_traceback(query, subject, matrix, gaps: GapModel, memory_cap: int = 256 << 20, device: int = 0) -> dict:
    """sw_align_traceback (align.hpp:254-353) on the GPU: bounds, score, capped flag and the edit script
    (0 match, 1 substitute, 2 insert, 3 del -- EditOp, align.hpp:236)."""
    lib = _cabi.load()
    q, s, mat = _u8(query), _u8(subject), _mat(matrix)
    dummy = np.zeros(1, np.uint8)
    out = _cabi.SwbAlignment()
    cap = len(q) + len(s) + 1
    ops = np.zeros(cap, dtype=np.uint8)
    rc = lib.swb_align_traceback(_ptr(q if len(q) else dummy, _u8p), len(q), _ptr(s if len(s) else dummy, _u8p), len(s),
                                 _ptr(mat, _i32p), gaps.open, gaps.extend, memory_cap, device, C.byref(out),
                                 _ptr(ops, _u8p), cap)
    _raise(lib, rc)
    return dict(bounds=[int(out.query_begin), int(out.query_end), int(out.subject_begin), int(out.subject_end)],
                score=int(out.score), capped=bool(out.capped), ops=ops[:int(out.n_ops)].copy())


def shard_assignment(lengths, length_threshold: int, shard_count: int) -> np.ndarray:
    """The deterministic residue-balanced deal used by swb_db_create (host only, no GPU needed)."""
    lib = _cabi.load()
    lens = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint32))
    out = np.zeros(max(1, len(lens)), dtype=np.uint32)
    rc = lib.swb_shard_assignment(_ptr(lens, _u32p), len(lens), int(length_threshold) & (2 ** 64 - 1), shard_count,
                                  _ptr(out, _u32p))
    _raise(lib, rc)
    return out[:len(lens)]


def scan_plan(lengths, query_len: int, sm_count: int = 148, length_threshold: int = 3000, shard_rank: int = 0,
              shard_count: int = 1, policy: int = 0) -> dict:
    """How a search would be divided between the two scan kernels (swb_scan_plan; host only, no GPU needed)."""
    lib = _cabi.load()
    lens = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint32))
    info = _cabi.SwbScanPlanInfo()
    rc = lib.swb_scan_plan(_ptr(lens, _u32p), len(lens), int(length_threshold) & (2 ** 64 - 1), shard_rank, shard_count,
                           query_len, sm_count, policy, C.byref(info))
    _raise(lib, rc)
    return info.as_dict()


def batch_plan(lengths, query_lengths, sm_count: int = 148, length_threshold: int = 3000, shard_rank: int = 0,
               shard_count: int = 1):
    """How swb_search_many would group a batch of queries (swb_batch_plan; host only): (scan_of_query, stream_of_query),
    -1 where a query is searched on its own."""
    lib = _cabi.load()
    lens = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint32))
    ql = np.ascontiguousarray(np.asarray(query_lengths, dtype=np.uint32))
    scan = np.full(max(1, len(ql)), -2, dtype=np.int32)
    stream = np.full(max(1, len(ql)), -2, dtype=np.int32)
    rc = lib.swb_batch_plan(_ptr(lens, _u32p), len(lens), int(length_threshold) & (2 ** 64 - 1), shard_rank, shard_count,
                            _ptr(ql, _u32p), len(ql), sm_count, _ptr(scan, _i32p), _ptr(stream, _i32p))
    _raise(lib, rc)
    return scan[:len(ql)], stream[:len(ql)]


def measure_pipe_rates(device: int = 0, seconds: float = 1.0) -> dict:
    lib = _cabi.load()
    r = _cabi.SwbPipeRates()
    _raise(lib, lib.swb_measure_pipe_rates(device, seconds, C.byref(r)))
    return r.as_dict()


class MultiGpuDatabase:
    """One process, several GPUs (swb_mdb): shards + NCCL all-gather of the per-shard top-k."""

    def __init__(self, codes, offsets, devices, length_threshold: int = 3000):
        self._lib = _cabi.load()
        self._h = C.c_void_p()
        codes = _u8(codes)
        offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        devs = np.ascontiguousarray(np.asarray(devices, dtype=np.int32))
        keep = codes if len(codes) else np.zeros(1, np.uint8)
        rc = self._lib.swb_mdb_create_flat(_ptr(keep, _u8p), _ptr(offsets, _u64p), len(offsets) - 1,
                                           int(length_threshold) & (2 ** 64 - 1), _ptr(devs, _i32p), len(devs),
                                           C.byref(self._h))
        _raise(self._lib, rc)

    def close(self):
        if self._h:
            self._lib.swb_mdb_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, query, matrix, gaps: GapModel, top_k: int = 10):
        q, mat = _u8(query), _mat(matrix)
        hits = (_cabi.SwbHit * max(1, top_k))()
        n = C.c_uint32(0)
        st = _cabi.SwbStats()
        rc = self._lib.swb_mdb_search(self._h, _ptr(q, _u8p), len(q), _ptr(mat, _i32p), gaps.open, gaps.extend,
                                      top_k, hits, C.byref(n), C.byref(st))
        _raise(self._lib, rc)
        idx = np.array([hits[i].db_index for i in range(n.value)], dtype=np.uint32)
        sc = np.array([hits[i].score for i in range(n.value)], dtype=np.int32)
        return idx, sc, st.as_dict()

    def search_many(self, queries, matrix, gaps: GapModel, top_k: int = 10):
        """A batch on every shard at once (swb_mdb_search_many), merged per query: -> list of (db_index, score), ms."""
        mat = _mat(matrix)
        qs = [_u8(q) for q in queries]
        n = len(qs)
        dummy = np.zeros(1, np.uint8)
        ptrs = (_u8p * max(1, n))()
        lens = np.zeros(max(1, n), dtype=np.uint32)
        for i, q in enumerate(qs):
            ptrs[i] = _ptr(q if len(q) else dummy, _u8p)
            lens[i] = len(q)
        hits = (_cabi.SwbHit * max(1, n * top_k))()
        counts = np.zeros(max(1, n), dtype=np.uint32)
        ms = np.zeros(max(1, n), dtype=np.float32)
        rc = self._lib.swb_mdb_search_many(self._h, ptrs, _ptr(lens, _u32p), n, _ptr(mat, _i32p), gaps.open, gaps.extend,
                                           top_k, hits, _ptr(counts, _u32p), ms.ctypes.data_as(C.POINTER(C.c_float)))
        _raise(self._lib, rc)
        out = []
        for qi in range(n):
            c = int(counts[qi])
            out.append((np.array([hits[qi * top_k + i].db_index for i in range(c)], dtype=np.uint32),
                        np.array([hits[qi * top_k + i].score for i in range(c)], dtype=np.int32)))
        return out, ms[:n].copy()

    def align_hits(self, query, matrix, gaps: GapModel, index, score, subject_lengths, memory_cap: int = 256 << 20):
        return _align_hits(self._lib.swb_mdb_align_hits, self._lib, self._h, query, matrix, gaps, index, score,
                           subject_lengths, memory_cap)
