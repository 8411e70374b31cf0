"""As scaling_probe.py, for the batched sweep (swb_search_many): shard 0 of N on one GPU, N x shard cells / time."""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel

shard_list = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8]
qs, sdb = synth.config2()
b62 = synth.blosum62()
g = GapModel(10, 2)
cells = sum(len(q) for q in qs) * sdb.residues
for shards in shard_list:
    with Database(sdb.codes, sdb.offsets, shard_rank=0, shard_count=shards) as db:
        db.search_many(qs, b62, g, 10)
        _, ms = db.search_many(qs, b62, g, 10)
        print(f"N={shards} shard residues={db.info()['residues']/1e6:.1f}M  sweep {ms.sum():.1f} ms  -> {cells/ms.sum()/1e6:.0f} GCUPS-equivalent for N GPUs")
