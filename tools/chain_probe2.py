"""One query length on shard 0 of N, a few repetitions: for ncu launch lists.  usage: chain_probe2.py N m_index reps"""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel
shards, qi, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
qs, sdb = synth.config2()
b62 = synth.blosum62()
with Database(sdb.codes, sdb.offsets, shard_rank=0, shard_count=shards) as db:
    for _ in range(reps):
        _, _, st = db.search(qs[qi], b62, GapModel(10, 2), 10)
        print(f"N={shards} m={len(qs[qi])} ms={st['ms_total']:.2f} scan={st['ms_scan']:.2f}")
