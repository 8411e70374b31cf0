"""Helper for test_gpu_parity.py::test_pipeline_tile_slices_against_the_oracle: the pipeline kernel's per-warp tile slices
(pipeline.cuh: kSlice -- what queries too long for a whole profile in shared memory take).  Run once with
SWB200_PIPE_SLICES=1 (the slice form for every query length, around the tile and pass boundaries) and once without (only the
7,000-residue queries take it, by themselves).  Whole score vectors against the oracle; prints SLICE-SMALL-OK."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle as po                                     # noqa: E402
from paper_2203_11100_b200 import Database, GapModel, synth           # noqa: E402

forced = os.environ.get("SWB200_PIPE_SLICES") == "1"
port = po.Port()
b62 = synth.blosum62()
ok = True
for seed, gaps, thr in ((31, (10, 2), 3000), (32, (11, 1), 100), (33, (3, 3), 10 ** 9)):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(300, 1200))
    seqs = [synth.random_residues(rng, int(rng.integers(0, 300))) for _ in range(n)]
    seqs[1] = synth.random_residues(rng, 1900)            # a tall group
    seqs[4] = np.zeros(0, np.uint8)
    lens = [1, 31, 32, 33, 500, 512, 513, 1024, 1030, 2100] if forced else [6600, 7000]
    queries = [synth.random_residues(rng, m) for m in lens]
    seqs[7] = synth.mutate(rng, queries[-1], 0.15, 3)     # a strong hit for the longest query
    fdb = po.FlatDb.from_list(seqs)
    with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
        for policy in (Database.SCAN_PIPELINE, Database.SCAN_AUTO):
            db.set_scan_policy(policy)
            for q in queries:
                got, st = db.score_all(q, b62, GapModel(*gaps))
                exp = port.score_all(q, fdb, b62, *gaps)
                good = bool((got == exp).all())
                ok &= good
                if not good:
                    bad = np.flatnonzero(got != exp)
                    print(f"MISMATCH seed={seed} m={len(q)} policy={policy}: {len(bad)} scores, first {bad[:5]}")
print("SLICE-SMALL-OK" if ok else "SLICE-SMALL-FAIL")
sys.exit(0 if ok else 1)
