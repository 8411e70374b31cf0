"""Helper for test_gpu_parity.py::test_narrow_block_sweep_against_the_oracle: run in a subprocess with SWB200_NARROW set
so low that every group of more than 2,048 rows takes the wavefront kernel's narrow units (8-column tiles swept as
8 x 8 blocks in anti-diagonal order, kernels.cuh: sweep_unit_narrow_s16), which otherwise only very tall groups of a
big database do (the knobs are read once per process).  Whole score vectors against the oracle; prints NARROW-SMALL-OK."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle as po                                     # noqa: E402
from paper_2203_11100_b200 import Database, GapModel, scan_plan, synth   # noqa: E402

port = po.Port()
b62 = synth.blosum62()
ok = True
for seed, gaps in ((41, (10, 2)), (42, (11, 1)), (43, (4, 4)), (44, (0, 0))):
    rng = np.random.default_rng(seed)
    seqs = [synth.random_residues(rng, int(rng.integers(0, 300))) for _ in range(int(rng.integers(200, 400)))]
    # tall groups: row counts around the chunk (8) and publish (32 rows) granules, one far taller than the rest
    for i, n in enumerate([2049, 2056, 2081, 4100, 9000, 2600] + [int(x) for x in rng.integers(2049, 3300, 180)]):
        seqs[i] = synth.random_residues(rng, n)
    queries = [synth.random_residues(rng, m) for m in (1, 7, 8, 9, 16, 40, 144, 150, 257)]
    queries.append(synth.mutate(rng, seqs[4], 0.05, 2)[100:380])     # a real hit inside the tallest sequence
    fdb = po.FlatDb.from_list(seqs)
    lens = np.diff(fdb.offsets.astype(np.int64))
    with Database(fdb.codes, fdb.offsets) as db:
        for policy in (Database.SCAN_AUTO, Database.SCAN_WAVEFRONT):
            db.set_scan_policy(policy)
            for q in queries:
                plan = scan_plan(lens, len(q), policy=policy)
                got, st = db.score_all(q, b62, GapModel(*gaps))
                exp = port.score_all(q, fdb, b62, *gaps)
                good = bool((got == exp).all())
                if len(q) > 8 and policy == Database.SCAN_WAVEFRONT and plan["narrow_groups"] < 2:
                    good = False
                    print(f"seed={seed} m={len(q)}: fewer than two narrow groups were planned")
                ok &= good
                if not good:
                    bad = np.nonzero(got != exp)[0]
                    print(f"MISMATCH seed={seed} gaps={gaps} m={len(q)} policy={policy}: {len(bad)} scores, first index {bad[:5]}, "
                          f"lens {lens[bad[:5]]}, got {got[bad[:5]]} exp {exp[bad[:5]]}")
# Next to the pipeline (a database of 300+ groups, so that the bulk goes to the pipeline kernel and the tall groups to the
# wavefront kernel's own CTAs of 4 or 8 warps): 4-column tiles when SWB200_NARROW_FINE is tiny, 8-column ones otherwise;
# a long query takes the classic narrow form (deep wavefront) or none.
rng = np.random.default_rng(51)
seqs = [synth.random_residues(rng, int(rng.integers(20, 110))) for _ in range(20500)]
for i, n in enumerate([9000, 8999, 6000, 5200] + [int(x) for x in rng.integers(2100, 4000, 70)]):
    seqs[i * 7] = synth.random_residues(rng, n)
queries = [synth.random_residues(rng, m) for m in (100, 137, 144, 300, 1100)]
queries.append(synth.mutate(rng, seqs[0], 0.1, 3)[4000:4130])
fdb = po.FlatDb.from_list(seqs)
lens = np.diff(fdb.offsets.astype(np.int64))
seen_tiles = set()
with Database(fdb.codes, fdb.offsets) as db:
    for q in queries:
        plan = scan_plan(lens, len(q))
        got, st = db.score_all(q, b62, GapModel(10, 2))
        exp = port.score_all(q, fdb, b62, 10, 2)
        good = bool((got == exp).all())
        if plan["narrow_groups"] and plan["pipeline_groups"]:
            seen_tiles.add((plan["narrow_tile"], plan["wavefront_threads"], plan["narrow_link_bytes"] > 0))
        ok &= good
        if not good:
            bad = np.nonzero(got != exp)[0]
            print(f"MISMATCH hybrid m={len(q)} plan={plan}: {len(bad)} scores, first {bad[:5]} lens {lens[bad[:5]]} got {got[bad[:5]]} exp {exp[bad[:5]]}")
print("hybrid narrow forms seen (tile, threads, links):", sorted(seen_tiles))
if not any(links for _, _, links in seen_tiles):
    ok = False
    print("no search took narrow units with link buffers next to the pipeline")
print("NARROW-SMALL-OK" if ok else "NARROW-SMALL-FAIL")
sys.exit(0 if ok else 1)
