"""A few searches of one query length on a short-pool-only Swiss-Prot-sized database, for ncu.
usage: python tests/manual/pipe_profile.py <m> [reps] [maxlen]"""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel
m = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
maxlen = int(sys.argv[3]) if len(sys.argv) > 3 else 2999
qs = synth.make_queries([m], 7)
sdb = synth.make_database(synth.SWISSPROT_SEQS, target_residues=synth.SWISSPROT_RESIDUES, max_len=maxlen, seed=7)
b62 = synth.blosum62()
with Database(sdb.codes, sdb.offsets) as db:
    for r in range(reps):
        idx, sc, st = db.search(qs[0], b62, GapModel(10, 2), 10)
        print(f"m={m} rep={r} scan={st['ms_scan']:.2f}ms GCUPS={st['cells']/st['ms_scan']/1e6:.1f}")
