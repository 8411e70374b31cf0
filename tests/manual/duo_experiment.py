"""Two-query scan (duo.cuh) against two single-query scans: identical score vectors, timing.
usage: python tests/manual/duo_experiment.py [maxlen]"""
import ctypes as C
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2203_11100_b200 import synth, Database, GapModel, _cabi

maxlen = int(sys.argv[1]) if len(sys.argv) > 1 else 35213
PAIRS = [(144, 189), (375, 464), (850, 1000), (1500, 2005), (2504, 3005), (5147, 5478)]
lens = sorted({m for p in PAIRS for m in p})
qs = dict(zip(lens, synth.make_queries(lens, 7)))
sdb = synth.make_database(synth.SWISSPROT_SEQS, target_residues=synth.SWISSPROT_RESIDUES, max_len=maxlen, queries=list(qs.values()), seed=7)
b62 = synth.blosum62()
lib = _cabi.load()
lib.swb_score_all_duo.restype = C.c_int
lib.swb_score_all_duo.argtypes = [C.c_void_p, _cabi.u8p, C.c_uint32, _cabi.u8p, C.c_uint32, _cabi.i32p, C.c_int32, C.c_int32,
                                  _cabi.i32p, _cabi.i32p, C.POINTER(_cabi.SwbStats)]
mat = np.ascontiguousarray(b62.reshape(576).astype(np.int32))
g = GapModel(10, 2)
with Database(sdb.codes, sdb.offsets) as db:
    for ma, mb in PAIRS:
        qa, qb = np.ascontiguousarray(qs[ma]), np.ascontiguousarray(qs[mb])
        single = []
        t_single = 0.0
        for q in (qa, qb):
            db.score_all(q, b62, g)
            sc, st = db.score_all(q, b62, g)
            single.append(sc)
            t_single += st["ms_scan"]
        sa = np.zeros(sdb.n, np.int32); sb = np.zeros(sdb.n, np.int32)
        best = None
        for _ in range(3):
            st = _cabi.SwbStats()
            rc = lib.swb_score_all_duo(db._h, qa.ctypes.data_as(_cabi.u8p), ma, qb.ctypes.data_as(_cabi.u8p), mb,
                                       mat.ctypes.data_as(_cabi.i32p), 10, 2, sa.ctypes.data_as(_cabi.i32p),
                                       sb.ctypes.data_as(_cabi.i32p), C.byref(st))
            assert rc == 0, lib.swb_last_error()
            best = st.ms_scan if best is None else min(best, st.ms_scan)
        bad = int((sa != single[0]).sum() + (sb != single[1]).sum())
        cells = (ma + mb) * sdb.residues
        print(f"pair ({ma},{mb}): two singles {t_single:8.2f} ms = {cells/t_single/1e6:6.0f} GCUPS | duo {best:8.2f} ms = {cells/best/1e6:6.0f} GCUPS "
              f"(useful; padded {2*max(ma,mb)*sdb.residues/best/1e6:6.0f}) | differing scores {bad}", flush=True)
