"""ctypes access to the two CPU checkers.  TEST INFRASTRUCTURE ONLY.

``Port``  -> oracle/_build/libsworacle.so  (oracle/sw_oracle.c, the C restatement)
``Ref``   -> oracle/_ref/libswref.so       (the unmodified reference behind oracle/ref_shim.cpp)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference`` legs may
import this module.  The product package ``paper_2203_11100_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "_build" / "libsworacle.so"
REF_SO = HERE / "_ref" / "libswref.so"

_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


def _p(arr, typ):
    return arr.ctypes.data_as(typ)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _mat(matrix) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(matrix, dtype=np.int32).reshape(576))
    return m


def build_port() -> Path:
    """Compile oracle/sw_oracle.c if the library is missing or stale."""
    src = HERE / "sw_oracle.c"
    if not PORT_SO.exists() or PORT_SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(["make", "-C", str(HERE), "port"], stdout=subprocess.DEVNULL)
    return PORT_SO


def build_ref(reference_include: str = "/root/reference/proj/include") -> Path | None:
    """Compile the reference shim when the reference tree is present (authoring container only)."""
    if not os.path.isdir(reference_include):
        return REF_SO if REF_SO.exists() else None
    subprocess.check_call(["make", "-C", str(HERE), "ref", f"REF_INCLUDE={reference_include}"],
                          stdout=subprocess.DEVNULL)
    return REF_SO


class FlatDb:
    """codes (uint8, concatenated) + offsets (uint64, n+1)."""

    def __init__(self, codes, offsets):
        self.codes = _u8(codes)
        self.offsets = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
        self.n = len(self.offsets) - 1

    @classmethod
    def from_list(cls, seqs):
        lens = np.array([len(s) for s in seqs], dtype=np.uint64)
        offsets = np.zeros(len(seqs) + 1, dtype=np.uint64)
        np.cumsum(lens, out=offsets[1:])
        codes = np.concatenate([_u8(s) for s in seqs]) if len(seqs) and offsets[-1] else np.zeros(0, np.uint8)
        return cls(codes, offsets)

    def seq(self, i):
        return self.codes[int(self.offsets[i]):int(self.offsets[i + 1])]


class Port:
    """oracle/sw_oracle.c"""

    def __init__(self):
        self.lib = C.CDLL(str(build_port()))
        L = self.lib
        L.swo_score_scalar.restype = C.c_int32
        L.swo_score_scalar.argtypes = [_u8p, C.c_uint32, _u8p, C.c_uint32, _i32p, C.c_int32, C.c_int32]
        L.swo_score_batch.restype = C.c_int
        L.swo_score_batch.argtypes = [_u8p, C.c_uint32, C.POINTER(_u8p), _u32p, C.c_uint32, C.c_uint32,
                                      _i32p, C.c_int32, C.c_int32, _i32p]
        L.swo_score_wavefront.restype = C.c_int32
        L.swo_score_wavefront.argtypes = [_u8p, C.c_uint32, _u8p, C.c_uint32, _i32p, C.c_int32, C.c_int32,
                                          C.c_uint64]
        L.swo_score_all.restype = None
        L.swo_score_all.argtypes = [_u8p, C.c_uint32, _u8p, _u64p, C.c_uint32, _i32p, C.c_int32, C.c_int32,
                                    _i32p]
        L.swo_merge.restype = C.c_uint64
        L.swo_merge.argtypes = [_u32p, _i32p, C.c_uint64, C.c_uint64, _u32p, _i32p]
        L.swo_run_search.restype = C.c_uint64
        L.swo_run_search.argtypes = [_u8p, C.c_uint32, _u8p, _u64p, C.c_uint32, _i32p, C.c_int32, C.c_int32,
                                     C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u32p, _i32p, _u64p]

    def score_scalar(self, q, s, matrix, open_, extend):
        q, s, mat = _u8(q), _u8(s), _mat(matrix)
        return int(self.lib.swo_score_scalar(_p(q, _u8p), len(q), _p(s, _u8p), len(s), _p(mat, _i32p),
                                             open_, extend))

    def score_batch(self, q, subjects, lane_width, matrix, open_, extend):
        """subjects: list of arrays or None (a padding lane)."""
        q, mat = _u8(q), _mat(matrix)
        keep = [None if s is None else _u8(s) for s in subjects]
        ptrs = (_u8p * max(1, len(keep)))()
        lens = np.zeros(max(1, len(keep)), dtype=np.uint32)
        for i, s in enumerate(keep):
            if s is None:
                ptrs[i] = None
            else:
                # a zero-length subject still needs a non-null pointer
                ptrs[i] = _p(s, _u8p) if len(s) else C.cast(C.create_string_buffer(1), _u8p)
                lens[i] = len(s)
        out = np.zeros(max(1, lane_width), dtype=np.int32)
        rc = self.lib.swo_score_batch(_p(q, _u8p), len(q), ptrs, _p(lens, _u32p), len(keep), lane_width,
                                      _p(mat, _i32p), open_, extend, _p(out, _i32p))
        if rc:
            raise ValueError("invalid lane batch")
        return out[:lane_width].copy()

    def score_wavefront(self, q, s, matrix, open_, extend, chunk_width):
        q, s, mat = _u8(q), _u8(s), _mat(matrix)
        r = int(self.lib.swo_score_wavefront(_p(q, _u8p), len(q), _p(s, _u8p), len(s), _p(mat, _i32p),
                                             open_, extend, chunk_width))
        if r < 0:
            raise ValueError("chunk_width must be >= 1")
        return r

    def score_all(self, q, db: FlatDb, matrix, open_, extend):
        q, mat = _u8(q), _mat(matrix)
        out = np.zeros(db.n, dtype=np.int32)
        codes = db.codes if len(db.codes) else np.zeros(1, np.uint8)
        self.lib.swo_score_all(_p(q, _u8p), len(q), _p(codes, _u8p), _p(db.offsets, _u64p), db.n,
                               _p(mat, _i32p), open_, extend, _p(out, _i32p))
        return out

    def merge(self, index, score, top_k):
        index = np.ascontiguousarray(np.asarray(index, dtype=np.uint32))
        score = np.ascontiguousarray(np.asarray(score, dtype=np.int32))
        n = len(index)
        oi = np.zeros(max(1, min(n, top_k)), dtype=np.uint32)
        os_ = np.zeros(max(1, min(n, top_k)), dtype=np.int32)
        k = int(self.lib.swo_merge(_p(index, _u32p), _p(score, _i32p), n, top_k, _p(oi, _u32p), _p(os_, _i32p)))
        return oi[:k].copy(), os_[:k].copy()

    def run_search(self, q, db: FlatDb, matrix, open_, extend, lane_width=8, chunk_width=64,
                   length_threshold=3000, top_k=10):
        q, mat = _u8(q), _mat(matrix)
        cap = max(1, min(db.n, top_k))
        oi = np.zeros(cap, dtype=np.uint32)
        os_ = np.zeros(cap, dtype=np.int32)
        st = np.zeros(3, dtype=np.uint64)
        codes = db.codes if len(db.codes) else np.zeros(1, np.uint8)
        k = int(self.lib.swo_run_search(_p(q, _u8p), len(q), _p(codes, _u8p), _p(db.offsets, _u64p), db.n,
                                        _p(mat, _i32p), open_, extend, lane_width, chunk_width,
                                        length_threshold, top_k, _p(oi, _u32p), _p(os_, _i32p),
                                        _p(st, _u64p)))
        if k == 2 ** 64 - 1:
            raise ValueError("invalid search config")
        return oi[:k].copy(), os_[:k].copy(), st.copy()


class Ref:
    """The unmodified reference (oracle/_ref/libswref.so).  ``Ref.available()`` is False on machines
    where neither the prebuilt library nor /root/reference exists."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists() or os.path.isdir("/root/reference/proj/include")

    def __init__(self):
        so = build_ref()
        if so is None or not so.exists():
            raise FileNotFoundError("oracle/_ref/libswref.so not built and /root/reference absent")
        self.lib = C.CDLL(str(so))
        L = self.lib
        L.swref_last_error.restype = C.c_char_p
        L.swref_blosum62.argtypes = [_i32p]
        L.swref_score_scalar.argtypes = [_u8p, C.c_uint32, _u8p, C.c_uint32, _i32p, C.c_int32, C.c_int32, _i32p]
        L.swref_score_batch.argtypes = [_u8p, C.c_uint32, C.POINTER(_u8p), _u32p, C.c_uint32, C.c_uint32,
                                        _i32p, C.c_int32, C.c_int32, _i32p]
        L.swref_score_wavefront.argtypes = [_u8p, C.c_uint32, _u8p, C.c_uint32, _i32p, C.c_int32, C.c_int32,
                                            C.c_uint64, _i32p]
        L.swref_db_create.restype = C.c_void_p
        L.swref_db_create.argtypes = [_u8p, _u64p, C.c_uint32]
        L.swref_db_destroy.argtypes = [C.c_void_p]
        L.swref_run_search.argtypes = [C.c_void_p, _u8p, C.c_uint32, _i32p, C.c_int32, C.c_int32] + \
            [C.c_uint64] * 6 + [_u32p, _i32p, _u32p, _u64p]
        L.swref_merge_results.argtypes = [_u32p, _i32p, _u64p, C.c_uint32, C.c_uint64, _u32p, _i32p, _u64p]
        L.swref_traceback.argtypes = [_u8p, C.c_uint32, _u8p, C.c_uint32, _i32p, C.c_int32, C.c_int32,
                                      C.c_uint64, _u64p, _i32p, _i32p, _u8p, C.c_uint64, _u64p, _i32p]

    def _check(self, rc):
        if rc == 1:
            raise ValueError(self.lib.swref_last_error().decode())
        if rc == 2:
            raise IndexError(self.lib.swref_last_error().decode())
        if rc:
            raise RuntimeError(self.lib.swref_last_error().decode())

    def blosum62(self):
        out = np.zeros(576, dtype=np.int32)
        self._check(self.lib.swref_blosum62(_p(out, _i32p)))
        return out.reshape(24, 24)

    def score_scalar(self, q, s, matrix, open_, extend):
        q, s, mat = _u8(q), _u8(s), _mat(matrix)
        out = C.c_int32(0)
        self._check(self.lib.swref_score_scalar(_p(q, _u8p), len(q), _p(s, _u8p), len(s), _p(mat, _i32p),
                                                open_, extend, C.byref(out)))
        return out.value

    def score_batch(self, q, subjects, lane_width, matrix, open_, extend):
        q, mat = _u8(q), _mat(matrix)
        keep = [None if s is None else _u8(s) for s in subjects]
        ptrs = (_u8p * max(1, len(keep)))()
        lens = np.zeros(max(1, len(keep)), dtype=np.uint32)
        for i, s in enumerate(keep):
            if s is None:
                ptrs[i] = None
            else:
                ptrs[i] = _p(s, _u8p) if len(s) else C.cast(C.create_string_buffer(1), _u8p)
                lens[i] = len(s)
        out = np.zeros(max(1, lane_width), dtype=np.int32)
        self._check(self.lib.swref_score_batch(_p(q, _u8p), len(q), ptrs, _p(lens, _u32p), len(keep),
                                               lane_width, _p(mat, _i32p), open_, extend, _p(out, _i32p)))
        return out[:lane_width].copy()

    def score_wavefront(self, q, s, matrix, open_, extend, chunk_width):
        q, s, mat = _u8(q), _u8(s), _mat(matrix)
        out = C.c_int32(0)
        self._check(self.lib.swref_score_wavefront(_p(q, _u8p), len(q), _p(s, _u8p), len(s), _p(mat, _i32p),
                                                   open_, extend, chunk_width, C.byref(out)))
        return out.value

    def db_create(self, db: FlatDb):
        codes = db.codes if len(db.codes) else np.zeros(1, np.uint8)
        return self.lib.swref_db_create(_p(codes, _u8p), _p(db.offsets, _u64p), db.n)

    def db_destroy(self, handle):
        self.lib.swref_db_destroy(handle)

    def run_search(self, handle, q, matrix, open_, extend, worker_count=1, lane_width=8, chunk_width=64,
                   length_threshold=3000, top_k=10, cpu_pool_threads=1, n_hint=None):
        q, mat = _u8(q), _mat(matrix)
        cap = max(1, top_k if n_hint is None else min(n_hint, top_k))
        oi = np.zeros(cap, dtype=np.uint32)
        os_ = np.zeros(cap, dtype=np.int32)
        cnt = C.c_uint32(0)
        st = np.zeros(3, dtype=np.uint64)
        self._check(self.lib.swref_run_search(handle, _p(q, _u8p), len(q), _p(mat, _i32p), open_, extend,
                                              worker_count, lane_width, chunk_width, length_threshold,
                                              top_k, cpu_pool_threads, _p(oi, _u32p), _p(os_, _i32p),
                                              C.byref(cnt), _p(st, _u64p)))
        return oi[:cnt.value].copy(), os_[:cnt.value].copy(), st.copy()

    def merge_results(self, parts, top_k):
        """parts: list of (index_array, score_array)."""
        sizes = np.array([len(p[0]) for p in parts], dtype=np.uint64)
        total = int(sizes.sum())
        idx = np.concatenate([np.asarray(p[0], dtype=np.uint32) for p in parts]) if total else np.zeros(1, np.uint32)
        sc = np.concatenate([np.asarray(p[1], dtype=np.int32) for p in parts]) if total else np.zeros(1, np.int32)
        idx, sc = np.ascontiguousarray(idx), np.ascontiguousarray(sc)
        oi = np.zeros(max(1, min(total, top_k)), dtype=np.uint32)
        os_ = np.zeros(max(1, min(total, top_k)), dtype=np.int32)
        cnt = C.c_uint64(0)
        if len(sizes) == 0:
            sizes = np.zeros(1, dtype=np.uint64)
            n_parts = 0
        else:
            n_parts = len(parts)
        self._check(self.lib.swref_merge_results(_p(idx, _u32p), _p(sc, _i32p), _p(sizes, _u64p), n_parts,
                                                 top_k, _p(oi, _u32p), _p(os_, _i32p), C.byref(cnt)))
        return oi[:cnt.value].copy(), os_[:cnt.value].copy()

    def traceback(self, q, s, matrix, open_, extend, memory_cap=256 << 20):
        q, s, mat = _u8(q), _u8(s), _mat(matrix)
        bounds = np.zeros(4, dtype=np.uint64)
        score, capped, resc = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        cap = len(q) + len(s) + 1
        ops = np.zeros(cap, dtype=np.uint8)
        n_ops = C.c_uint64(0)
        self._check(self.lib.swref_traceback(_p(q, _u8p), len(q), _p(s, _u8p), len(s), _p(mat, _i32p), open_,
                                             extend, memory_cap, _p(bounds, _u64p), C.byref(score),
                                             C.byref(capped), _p(ops, _u8p), cap, C.byref(n_ops),
                                             C.byref(resc)))
        return dict(bounds=[int(b) for b in bounds], score=score.value, capped=bool(capped.value),
                    ops=ops[:n_ops.value].copy(), rescored=resc.value)
