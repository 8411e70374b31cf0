"""Runs a few searches on the config-2 database so that ncu can capture the scan kernel.
usage: python tools/profile_scan.py <query_number> [reps] [scale]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2203_11100_b200 import synth, Database, GapModel

qi = int(sys.argv[1]) if len(sys.argv) > 1 else 9
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
qs, sdb = synth.config2(scale=scale)
b62 = synth.blosum62()
with Database(sdb.codes, sdb.offsets) as db:
    for r in range(reps):
        idx, sc, st = db.search(qs[qi], b62, GapModel(10, 2), 10)
        print(f"m={len(qs[qi])} rep={r} GCUPS={st['cells']/st['ms_total']/1e6:.1f} scan={st['ms_scan']:.2f}ms units={st['chunks_claimed']}")
