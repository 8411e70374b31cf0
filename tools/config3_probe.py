"""Config 3 (long pool only) one query at a time: per-query ms and GCUPS; SWB200_* knobs apply."""
import sys
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel, scan_plan
q3, db3, _ = synth.config3()
b62 = synth.blosum62()
tot_c = tot_t = 0
with Database(db3.codes, db3.offsets) as db:
    for q in q3:
        db.search(q, b62, GapModel(10, 2), 10)
        _, _, st = db.search(q, b62, GapModel(10, 2), 10)
        tot_c += st["cells"]; tot_t += st["ms_total"]
        print(f"m={len(q)} {st['ms_total']:.2f} ms {st['cells']/st['ms_total']/1e6:.0f} GCUPS units={st['chunks_claimed']}")
    p = scan_plan(db3.lengths(), len(q3[-1]))
print(f"aggregate {tot_c/tot_t/1e6:.0f} GCUPS  plan(m={len(q3[-1])})={p}")
