"""A batched search on the config-2 database, for ncu.
usage: python tests/manual/duo_profile.py sweep [reps]      the whole 20-query sweep as one swb_search_many batch
       python tests/manual/duo_profile.py <ma> <mb> [reps]  one pair of queries
SWB_PROFILE_SHARD=r/n runs it on shard r of n (pass items from n = 2 up)"""
import os
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel
qs, sdb = synth.config2()
if sys.argv[1] == "sweep":
    batch, reps = qs, int(sys.argv[2]) if len(sys.argv) > 2 else 2
else:
    batch, reps = synth.make_queries([int(sys.argv[1]), int(sys.argv[2])], 7), int(sys.argv[3]) if len(sys.argv) > 3 else 2
b62 = synth.blosum62()
cells = sum(len(q) for q in batch) * sdb.residues
rank, count = (int(x) for x in os.environ.get("SWB_PROFILE_SHARD", "0/1").split("/"))
with Database(sdb.codes, sdb.offsets, shard_rank=rank, shard_count=count) as db:
    cells = cells * db.info()["residues"] // sdb.residues
    for r in range(reps):
        out, ms = db.search_many(batch, b62, GapModel(10, 2), 10)
        print(f"batch of {len(batch)} queries rep={r} {ms.sum():.2f} ms  {cells/ms.sum()/1e6:.0f} GCUPS")
