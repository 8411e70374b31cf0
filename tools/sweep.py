"""Times every query of the config-2 sweep once (after one warm-up each); prints per-query and aggregate GCUPS."""
import sys, time, os
sys.path.insert(0, ".")
import numpy as np
from paper_2203_11100_b200 import synth, Database, GapModel
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
qs, sdb = synth.config2(scale=scale)
b62 = synth.blosum62()
tot_cells = 0; tot_ms = 0
with Database(sdb.codes, sdb.offsets) as db:
    for qi, q in enumerate(qs):
        db.search(q, b62, GapModel(10, 2), 10)
        idx, sc, st = db.search(q, b62, GapModel(10, 2), 10)
        tot_cells += st["cells"]; tot_ms += st["ms_total"]
        print(f"m={len(q):5d} GCUPS={st['cells']/st['ms_total']/1e6:7.1f} total={st['ms_total']:8.2f}ms scan={st['ms_scan']:8.2f} rescore={st['ms_rescore']:.3f} topk={st['ms_topk']:.3f} units={st['chunks_claimed']} top1={idx[0]}:{sc[0]} planted={sdb.planted[qi][0]}")
print(f"AGGREGATE GCUPS={tot_cells/tot_ms/1e6:.1f} over {tot_ms:.1f} ms")
