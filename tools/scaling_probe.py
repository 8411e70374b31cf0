"""Emulates N-way sharding on ONE GPU: times shard 0 of N for a few queries and prints the throughput N such
GPUs would reach together (N x shard cells / shard time), i.e. the strong-scaling efficiency the kernel allows
(the NCCL all-gather of k keys per query, ~20 us, is not included)."""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel

shard_list = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 4, 8]
qs, sdb = synth.config2()
b62 = synth.blosum62()
g = GapModel(10, 2)
for shards in shard_list:
    with Database(sdb.codes, sdb.offsets, shard_rank=0, shard_count=shards) as db:
        info = db.info()
        line = [f"N={shards} shard residues={info['residues']/1e6:.1f}M groups={info['n_groups']}"]
        tot_c = tot_t = 0
        for qi in (0, 3, 9, 14, 19):
            db.search(qs[qi], b62, g, 10)
            _, _, st = db.search(qs[qi], b62, g, 10)
            tot_c += st["cells"]; tot_t += st["ms_total"]
            line.append(f"m={len(qs[qi])}:{shards*st['cells']/st['ms_total']/1e6:.0f}({st['ms_total']:.1f}ms,{st['chunks_claimed']}u)")
        line.append(f"agg={shards*tot_c/tot_t/1e6:.0f} GCUPS-equivalent")
        print("  ".join(line))
