"""Where does a short query's time go?  Times m = 144 / 189 / 222 / 375 on shard 0 of N (N from argv, default 1,8) and, run
under `ncu --metrics gpu__time_duration.sum`, gives each scan kernel's stand-alone duration (ncu serialises them)."""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel, scan_plan

shard_list = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 8]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
qs, sdb = synth.config2()
b62 = synth.blosum62()
g = GapModel(10, 2)
for shards in shard_list:
    with Database(sdb.codes, sdb.offsets, shard_rank=0, shard_count=shards) as db:
        for qi in (0, 1, 2, 3, 9):
            q = qs[qi]
            plan = scan_plan(sdb.lengths(), len(q), shard_rank=0, shard_count=shards)
            best = None
            for _ in range(reps):
                _, _, st = db.search(q, b62, g, 10)
                best = st if best is None or st["ms_total"] < best["ms_total"] else best
            print(f"N={shards} m={len(q)} ms={best['ms_total']:.2f} scan={best['ms_scan']:.2f} gcups_equiv={shards*best['cells']/best['ms_total']/1e6:.0f} plan={plan}")
