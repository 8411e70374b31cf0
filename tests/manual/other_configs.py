"""BASELINE configs 3 and 5 on one GPU.
  config 3: queries >= 3005 against only the database entries >= 3000 residues (the intra-task pool).
  config 5: TrEMBL-shaped database (~1 G residues, same length model), BLOSUM50, gap 12/2, with queries long
            enough that the packed int16 range overflows and the int32 re-run is exercised."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as po
from paper_2203_11100_b200 import synth, Database, GapModel

port = po.Port()
which = sys.argv[1] if len(sys.argv) > 1 else "3"
if which == "3":
    qs, sdb = synth.config2()
    lens = sdb.lengths()
    long_idx = np.nonzero(lens >= 3000)[0]
    sub = sdb.subset(long_idx)
    print(f"config 3: {sub.n} sequences >= 3000 residues, {sub.residues/1e6:.1f} M residues")
    b62 = synth.blosum62()
    with Database(sub.codes, sub.offsets) as db:
        tc = tt = 0
        for qi in range(13, 20):
            db.search(qs[qi], b62, GapModel(10, 2), 10)
            idx, sc, st = db.search(qs[qi], b62, GapModel(10, 2), 10)
            tc += st["cells"]; tt += st["ms_total"]
            print(f"  m={len(qs[qi])} GCUPS={st['cells']/st['ms_total']/1e6:.1f} ms={st['ms_total']:.2f} wavefront_scored={st['wavefront_scored']} units={st['chunks_claimed']}")
        print(f"  aggregate {tc/tt/1e6:.1f} GCUPS")
else:
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    lengths = synth.QUERY_LENGTHS + [8000, 9000]
    queries = synth.make_queries(lengths, seed=0x535744420005)
    t0 = time.time()
    sdb = synth.make_database(int(2_800_000 * scale), target_residues=int(1.0e9 * scale), queries=queries, seed=0x535744420005)
    print(f"config 5: {sdb.n} sequences, {sdb.residues/1e9:.3f} G residues, generated in {time.time()-t0:.1f}s")
    b50 = synth.blosum50()
    g = GapModel(12, 2)
    t0 = time.time()
    with Database(sdb.codes, sdb.offsets) as db:
        print(f"  packed+uploaded in {time.time()-t0:.1f}s, device bytes {db.info()['device_bytes']/1e9:.2f} GB")
        tc = tt = 0; flagged = 0
        for qi in (0, 9, 17, 18, 19, 20, 21):
            q = queries[qi]
            db.search(q, b50, g, 10)
            idx, sc, st = db.search(q, b50, g, 10)
            tc += st["cells"]; tt += st["ms_total"]; flagged += st["rescored_i32"]
            exact = sdb.planted[qi][0]
            ok = idx[0] == exact and all(int(s) == port.score_scalar(q, sdb.seq(int(i)), b50, 12, 2) for i, s in zip(idx[:4], sc[:4]))
            print(f"  m={len(q)} GCUPS={st['cells']/st['ms_total']/1e6:.1f} ms={st['ms_total']:.1f} rescored={st['rescored_i32']} rescore_ms={st['ms_rescore']:.2f} top={idx[0]}:{sc[0]} planted={exact} exact_vs_oracle={ok}")
        print(f"  aggregate {tc/tt/1e6:.1f} GCUPS, sequences re-run in int32: {flagged}")
        assert flagged > 0
        # the same queries as one batch (shared scans), checked against the single searches
        batch = [queries[qi] for qi in (0, 9, 17, 18, 19, 20, 21)]
        singles = [db.search(q, b50, g, 10)[:2] for q in batch]
        db.search_many(batch, b50, g, 10)
        many, ms = db.search_many(batch, b50, g, 10)
        same = all((a[0] == b[0]).all() and (a[1] == b[1]).all() for a, b in zip(many, singles))
        cells = sum(len(q) for q in batch) * sdb.residues
        print(f"  batched (swb_search_many): {cells/ms.sum()/1e6:.1f} GCUPS, ranked lists equal to the single searches: {same}")
        assert same
