"""The pipeline kernel with the whole profile in shared memory against per-warp tile slices (pipeline.cuh: kSlice), on the
config-2 database: run as is and with SWB200_PIPE_SLICES=1.  Queries of the sweep plus two beyond the whole-profile limit
(7,000 and 9,000 residues, which take the slice form either way; before it they fell back to the wavefront kernel)."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2203_11100_b200 import Database, GapModel, synth  # noqa: E402

qs, sdb = synth.config2()
b62 = synth.blosum62()
rng = np.random.default_rng(3)
picks = [q for q in qs if len(q) in (375, 1000, 2005, 3564, 5478)] + [synth.random_residues(rng, m) for m in (6400, 7000, 9000)]
print("SWB200_PIPE_SLICES =", os.environ.get("SWB200_PIPE_SLICES", "(unset)"))
with Database(sdb.codes, sdb.offsets) as db:
    for q in picks:
        db.search(q, b62, GapModel(10, 2), 10)
        best = None
        for _ in range(3):
            idx, sc, st = db.search(q, b62, GapModel(10, 2), 10)
            if best is None or st["ms_total"] < best["ms_total"]:
                best = st
        print(f"m={len(q):5d} GCUPS={best['cells']/best['ms_total']/1e6:7.1f} total={best['ms_total']:8.2f} ms scan={best['ms_scan']:8.2f} "
              f"launches={best['kernel_launches']} top1={idx[0]}:{sc[0]}")
