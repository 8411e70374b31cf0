"""First-light check on a GPU box: small parity cases, config 1, pipe rates, a scaled config-2 timing."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as po
from paper_2203_11100_b200 import synth, Database, GapModel, score_batch, score_wavefront, measure_pipe_rates

port = po.Port()
b62 = synth.blosum62()
gaps = GapModel(10, 2)
rng = np.random.default_rng(7)
out = {}

A = synth.encode("AAA")
print("AAA/AAA batch", score_batch(A, [A, None], 4, b62, gaps), "wavefront", score_wavefront(A, A, b62, gaps, 1))

# random small databases, full score vector parity
bad = 0
for it in range(6):
    n = int(rng.integers(1, 400))
    seqs = [synth.random_residues(rng, int(rng.integers(0, 300))) for _ in range(n)]
    if it % 2:
        seqs[0] = synth.random_residues(rng, 700)
    m = int(rng.integers(1, 260))
    q = synth.random_residues(rng, m)
    thr = [3000, 100, 0, 10**9, 250, 3000][it]
    fdb = po.FlatDb.from_list(seqs)
    with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
        got, st = db.score_all(q, b62, gaps)
        exp = port.score_all(q, fdb, b62, 10, 2)
        ok = (got == exp).all()
        bad += not ok
        print(f"case {it}: n={n} m={m} thr={thr} ok={ok} info={db.info()['n_short']}/{db.info()['n_long']}")
        if not ok:
            w = np.nonzero(got != exp)[0][:10]
            print("  mismatch at", w, got[w], exp[w], [len(seqs[i]) for i in w])
out["small_bad"] = bad

# config 1
qs, sdb = synth.config1()
fdb = po.FlatDb(sdb.codes, sdb.offsets)
with Database(sdb.codes, sdb.offsets) as db:
    t = time.time(); got, st = db.score_all(qs[0], b62, gaps); t1 = time.time() - t
    exp = port.score_all(qs[0], fdb, b62, 10, 2)
    print("config1 score parity:", (got == exp).all(), "mismatches", int((got != exp).sum()), st)
    idx, sc, st2 = db.search(qs[0], b62, gaps, 10)
    ei, es, _ = port.run_search(qs[0], fdb, b62, 10, 2)
    print("config1 topk parity:", (idx == ei).all() and (sc == es).all(), idx, sc)
    out["config1_ok"] = bool((got == exp).all() and (idx == ei).all() and (sc == es).all())
    for rep in range(3):
        idx, sc, st2 = db.search(qs[0], b62, gaps, 10)
    print("config1 stats", st2, "GCUPS", st2["cells"] / st2["ms_total"] / 1e6)

# overflow: long W-rich self hit in the short pool (threshold huge) and in the long pool
q = synth.random_residues(rng, 4000); q[::2] = 17; q[1::4] = 4
seqs = [q.copy(), synth.random_residues(rng, 500), q[:3500].copy()] + [synth.random_residues(rng, int(rng.integers(0, 900))) for _ in range(100)]
fdb = po.FlatDb.from_list(seqs)
for thr in (10**9, 3000):
    with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
        got, st = db.score_all(q, b62, gaps)
        exp = port.score_all(q, fdb, b62, 10, 2)
        print("overflow thr", thr, got[:3], exp[:3], "rescored", st["rescored_i32"], "ok", (got == exp).all())
        out[f"overflow_{thr}"] = bool((got == exp).all())

rates = measure_pipe_rates(0, 2.0)
print("pipe rates", json.dumps(rates))
out["rates"] = rates

# multi-shard on one GPU (swb_mdb with duplicate devices) must reproduce the single-shard list
from paper_2203_11100_b200 import MultiGpuDatabase
qs, sdb = synth.config1()
with Database(sdb.codes, sdb.offsets) as db:
    i1, s1, _ = db.search(qs[0], b62, gaps, 25)
for G in (2, 3, 8):
    mdb = MultiGpuDatabase(sdb.codes, sdb.offsets, [0] * G)
    i2, s2, st = mdb.search(qs[0], b62, gaps, 25)
    mdb.close()
    print("mdb shards", G, "same list:", (i1 == i2).all() and (s1 == s2).all())
    out[f"mdb_{G}"] = bool((i1 == i2).all() and (s1 == s2).all())

# config 2 timing for a few query lengths
import os
scale = float(os.environ.get("SWB_SCALE", "1.0"))
t0 = time.time(); qs, sdb = synth.config2(scale=scale); print("generated in", time.time() - t0)
t0 = time.time()
with Database(sdb.codes, sdb.offsets) as db:
    print("packed+uploaded in", time.time() - t0)
    print("db info", db.info())
    for qi in (0, 4, 9, 14, 19):
        for rep in range(2):
            idx, sc, st = db.search(qs[qi], b62, gaps, 10)
        print(f"m={len(qs[qi])} GCUPS={st['cells']/st['ms_total']/1e6:.1f} inter={st['ms_scan']:.2f}ms setup={st['ms_setup']:.3f}ms "
              f"rescore={st['ms_rescore']:.2f} topk={st['ms_topk']:.3f} total={st['ms_total']:.2f} planted={sdb.planted[qi]} top={idx[:4]} {sc[:4]}")
json.dump(out, open("gpurun_out/first_light.json", "w"), indent=1)
