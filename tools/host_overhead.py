"""Host time per search that the device does not hide: wall clock of swb_search minus its device time (events), per query length."""
import sys, time
sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth, Database, GapModel
qs, sdb = synth.config2()
b62 = synth.blosum62()
g = GapModel(10, 2)
with Database(sdb.codes, sdb.offsets) as db:
    for qi in (0, 9, 19):
        q = qs[qi]
        for _ in range(3): db.search(q, b62, g, 10)
        n = 30
        t0 = time.perf_counter(); dev = 0.0
        for _ in range(n):
            _, _, st = db.search(q, b62, g, 10)
            dev += st["ms_total"]
        wall = (time.perf_counter() - t0) * 1e3
        print(f"m={len(q)}: wall {wall/n:.3f} ms per search, device {dev/n:.3f} ms, host overhead {(wall-dev)/n*1e3:.1f} us (setup {st['ms_setup']*1e3:.0f} us of the device time)")
