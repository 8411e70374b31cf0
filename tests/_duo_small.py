"""Helper for test_gpu_parity.py::test_two_query_scan_against_the_oracle: run in a subprocess with
SWB200_DUO_MINGROUPS=0.001 so that swb_search_many pairs queries on small databases too (the knobs are read once per
process).  Prints DUO-SMALL-OK when every ranked list equals the oracle's."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle as po                                     # noqa: E402
from paper_2203_11100_b200 import Database, GapModel, synth           # noqa: E402

port = po.Port()
b62 = synth.blosum62()
ok = True
for seed, gaps, thr in ((21, (10, 2), 3000), (22, (11, 1), 100), (23, (5, 5), 0), (24, (0, 0), 10 ** 9)):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(150, 900))
    seqs = [synth.random_residues(rng, int(rng.integers(0, 350))) for _ in range(n)]
    seqs[0] = synth.random_residues(rng, 2200)            # a tall group
    seqs[3] = np.zeros(0, np.uint8)
    # lengths straddling the tile (32) and pass (512) boundaries; neighbours within 3/4 pair up
    lens = [289, 300, 511, 513, 545, 600, 1100, 1200, 40, 1]
    queries = [synth.random_residues(rng, m) for m in lens]
    queries[1] = synth.mutate(rng, seqs[0], 0.1, 2)[:300]
    fdb = po.FlatDb.from_list(seqs)
    with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
        many, ms = db.search_many(queries, b62, GapModel(*gaps), 12)
        for q, (idx, sc) in zip(queries, many):
            ei, es, _ = port.run_search(q, fdb, b62, *gaps, length_threshold=thr, top_k=12)
            good = bool((idx == ei).all() and (sc == es).all())
            ok &= good
            if not good:
                print(f"MISMATCH seed={seed} m={len(q)}")
print("DUO-SMALL-OK" if ok else "DUO-SMALL-FAIL")
sys.exit(0 if ok else 1)
