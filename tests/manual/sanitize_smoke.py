"""Small all-paths exercise for compute-sanitizer: single units, tile-split, row-block, narrow tiles, int32 re-run,
wide mode, pair / batch entry points, multi-shard merge, large-k sort."""
import os, sys
os.environ.setdefault("SWB200_DUO_MINGROUPS", "0.001")   # let the two-query scan run on this small database
sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as po
from paper_2203_11100_b200 import synth, Database, GapModel, MultiGpuDatabase, score_batch, score_wavefront

port = po.Port()
b62 = synth.blosum62()
g = GapModel(10, 2)
rng = np.random.default_rng(3)
seqs = [synth.random_residues(rng, int(rng.integers(0, 200))) for _ in range(300)]
seqs[0] = synth.random_residues(rng, 2500)          # tall group -> tile split / narrow
seqs[1] = synth.random_residues(rng, 900)
fdb = po.FlatDb.from_list(seqs)
ok = True
for m in (40, 300, 1500):
    q = synth.random_residues(rng, m)
    exp = port.score_all(q, fdb, b62, 10, 2)
    for thr in (3000, 100):
        with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
            got, st = db.score_all(q, b62, g)
            idx, sc, _ = db.search(q, b62, g, 1500)
            good = bool((got == exp).all())
            ok &= good
            print(f"m={m} thr={thr} parity={good} units={st['chunks_claimed']}")
# the on-chip tile pipeline, forced for every group: ring hand-over, wrap-around through global memory (m > 512)
for m in (33, 600, 1100):
    q = synth.random_residues(rng, m)
    exp = port.score_all(q, fdb, b62, 10, 2)
    with Database(fdb.codes, fdb.offsets) as db:
        db.set_scan_policy(Database.SCAN_PIPELINE)
        got, st = db.score_all(q, b62, g)
        good = bool((got == exp).all())
        ok &= good
        print(f"pipeline m={m} parity={good}")
# the two-query scan of swb_search_many (queries of similar length share it), against single searches
qs = [synth.random_residues(rng, m) for m in (300, 320, 600, 640, 90)]
with Database(fdb.codes, fdb.offsets) as db:
    many, _ = db.search_many(qs, b62, g, 20)
    for q, (mi, ms_) in zip(qs, many):
        ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=20)
        good = bool((mi == ei).all() and (ms_ == es).all())
        ok &= good
        print(f"search_many m={len(q)} parity={good}")
q = np.full(3400, 17, np.uint8)
with Database.from_sequences([q, q[:3100], seqs[5]]) as db:
    got, st = db.score_all(q, b62, g)
    print("overflow", got.tolist(), st["rescored_i32"])
    ok &= got[0] == port.score_scalar(q, q, b62, 10, 2)
big = (b62 * 40).astype(np.int32)
with Database(fdb.codes, fdb.offsets) as db:
    got, _ = db.score_all(seqs[1][:200], big, GapModel(400, 80))
    ok &= bool((got == port.score_all(seqs[1][:200], fdb, big, 400, 80)).all())
print("pair", score_wavefront(seqs[0][:2300], seqs[0], b62, g, 64), "batch", score_batch(seqs[3], [seqs[3], None, seqs[4]], 4, b62, g).tolist())
mdb = MultiGpuDatabase(fdb.codes, fdb.offsets, [0, 0, 0])
print("mdb", mdb.search(seqs[1][:100], b62, g, 5)[:2])
many, _ = mdb.search_many(qs, b62, g, 20)             # every shard at once, one host thread per shard
for q, (mi, ms_) in zip(qs, many):
    ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=20)
    good = bool((mi == ei).all() and (ms_ == es).all())
    ok &= good
    print(f"mdb search_many m={len(q)} parity={good}")
mdb.close()
print("ALL OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
