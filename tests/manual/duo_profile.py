"""A batched pair of queries on the config-2 database, for ncu.  usage: python tests/manual/duo_profile.py <ma> <mb> [reps]"""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel
ma, mb = int(sys.argv[1]), int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
qs, sdb = synth.config2()
pair = synth.make_queries([ma, mb], 7)
b62 = synth.blosum62()
with Database(sdb.codes, sdb.offsets) as db:
    for r in range(reps):
        out, ms = db.search_many(pair, b62, GapModel(10, 2), 10)
        print(f"pair ({ma},{mb}) rep={r} {ms.sum():.2f} ms  {(ma+mb)*sdb.residues/ms.sum()/1e6:.0f} GCUPS useful")
