"""Parity tests proper: the CUDA path, called through the C-ABI (libswb200.so via ctypes), against the oracle
(oracle/sw_oracle.c), the committed reference fixtures, and -- where oracle/_ref travelled -- the unmodified
reference itself.  Everything here is integer work: the bar is bit-exact."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2203_11100_b200 import (Database, GapModel, MultiGpuDatabase, SearchConfig, decode_keys, merge_keys,
                                   run_search, score_batch, score_wavefront, synth)
from tests._util import enc, golden, naive_rank

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _loaded(lib):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return lib


def test_known_answers(b62):
    A, g = enc("AAA"), GapModel(10, 2)
    assert score_wavefront(A, A, b62, g, 1) == 12
    assert score_batch(A, [A], 4, b62, g).tolist() == [12, 0, 0, 0]
    assert score_wavefront(enc("ARN"), enc("RNA"), b62, g, 64) == 11
    with Database.from_sequences([A]) as db:
        idx, sc, stats, _ = run_search(A, db, b62, g, SearchConfig(top_k=1))
        assert idx.tolist() == [0] and sc.tolist() == [12]
    with Database.from_sequences([enc(""), synth.random_residues(np.random.default_rng(0), 50)]) as db:
        idx, sc, _, _ = run_search(A, db, b62, g)                           # every sequence is a hit, even empty ones
        assert len(idx) == 2 and idx[-1] == 0 and sc[-1] == 0


def test_golden_pairs(b62):
    for rec in golden()["pairs"]:
        q, s, g = enc(rec["q"]), enc(rec["s"]), GapModel(rec["open"], rec["extend"])
        for cw in (1, 64):
            assert score_wavefront(q, s, b62, g, cw) == rec["scalar"]      # intra-task kernel
        assert score_batch(q, [s], 1, b62, g).tolist() == [rec["scalar"]]   # packed int16 kernel (+ re-run)


def test_golden_batches(b62):
    for rec in golden()["batches"]:
        subs = [None if s is None else enc(s) for s in rec["subjects"]]
        got = score_batch(enc(rec["q"]), subs, rec["lane_width"], b62, GapModel(rec["open"], rec["extend"]))
        assert got.tolist() == rec["scores"], rec.get("note")


def test_golden_searches(b62):
    for rec in golden()["searches"]:
        seqs = [enc(s) for s in rec["db"]]
        q, g = enc(rec["q"]), GapModel(rec["open"], rec["extend"])
        with Database.from_sequences(seqs, length_threshold=rec["length_threshold"]) as db:
            idx, sc, stats, _ = run_search(q, db, b62, g, SearchConfig(top_k=rec["top_k"]))
            assert idx.tolist() == rec["hits_index"] and sc.tolist() == rec["hits_score"]
            assert stats["lane_scored"] == rec["lane_scored"] and stats["wavefront_scored"] == rec["wavefront_scored"]
            if seqs:
                allsc, _ = db.score_all(q, b62, g)
                assert allsc.tolist() == rec["all_scores"]


@pytest.mark.parametrize("seed,thr,gaps", [(1, 3000, (10, 2)), (2, 100, (11, 1)), (3, 0, (5, 5)), (4, 10 ** 9, (0, 0)),
                                           (5, 250, (12, 2)), (6, 33, (10, 2))])
def test_random_databases(port, b62, seed, thr, gaps):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 500))
    seqs = [synth.random_residues(rng, int(rng.integers(0, 300))) for _ in range(n)]
    seqs[0] = synth.random_residues(rng, 900)
    m = int(rng.integers(1, 300))
    q = synth.random_residues(rng, m)
    seqs[n // 2] = synth.mutate(rng, q, 0.1, 2)
    fdb = po.FlatDb.from_list(seqs)
    with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
        got, st = db.score_all(q, b62, GapModel(*gaps))
        exp = port.score_all(q, fdb, b62, *gaps)
        assert (got == exp).all()
        idx, sc, _ = db.search(q, b62, GapModel(*gaps), 17)
        ei, es, _ = port.run_search(q, fdb, b62, *gaps, length_threshold=thr, top_k=17)
        assert (idx == ei).all() and (sc == es).all()
        assert st["lane_scored"] + st["wavefront_scored"] == n


def test_config1_full_parity(port, b62):
    """BASELINE config 1: one 144-residue query vs 10,000 sequences, every score and the ranked list."""
    qs, sdb = synth.config1()
    fdb = po.FlatDb(sdb.codes, sdb.offsets)
    with Database(sdb.codes, sdb.offsets) as db:
        got, st = db.score_all(qs[0], b62, GapModel(10, 2))
        exp = port.score_all(qs[0], fdb, b62, 10, 2)
        assert (got == exp).all()
        idx, sc, stats, _ = run_search(qs[0], db, b62, GapModel(10, 2))
        ei, es, est = port.run_search(qs[0], fdb, b62, 10, 2)
        assert (idx == ei).all() and (sc == es).all()
        assert stats["lane_scored"] == est[0] and stats["wavefront_scored"] == est[1]
        assert idx[0] == sdb.planted[0][0]
        # determinism: a repeat gives the identical list
        idx2, sc2, _, _ = run_search(qs[0], db, b62, GapModel(10, 2))
        assert (idx2 == idx).all() and (sc2 == sc).all()


def test_config1_against_reference_itself(ref, b62):
    qs, sdb = synth.config1()
    h = ref.db_create(po.FlatDb(sdb.codes, sdb.offsets))
    ri, rs, rst = ref.run_search(h, qs[0], b62, 10, 2, worker_count=4, cpu_pool_threads=2)
    ref.db_destroy(h)
    with Database(sdb.codes, sdb.offsets) as db:
        idx, sc, stats, _ = run_search(qs[0], db, b62, GapModel(10, 2))
    assert (idx == ri).all() and (sc == rs).all()
    assert stats["lane_scored"] == rst[0] and stats["wavefront_scored"] == rst[1]


def test_int16_overflow_is_rerun_in_int32(port, b62):
    """Scores beyond the packed kernels' trusted range (32767 - max(matrix) for the int16 kernel, 65535 - bias -
    max(matrix) for the unsigned variant) must come back exact from the int32 re-run (align.hpp:149-153)."""
    rng = np.random.default_rng(12)
    q = synth.random_residues(rng, 8000)
    q[::2] = 17          # W: 11 per match
    q[1::4] = 4          # C: 9 per match
    seqs = [q.copy(), synth.random_residues(rng, 500), q[:3500].copy(), synth.mutate(rng, q, 0.02, 2), q[:5000].copy()]
    seqs += [synth.random_residues(rng, int(rng.integers(0, 900))) for _ in range(150)]
    fdb = po.FlatDb.from_list(seqs)
    exp = port.score_all(q, fdb, b62, 10, 2)
    assert exp.max() > 65535 and ((exp > 32767) & (exp < 65535)).any()
    for thr in (10 ** 9, 3000, 0):
        with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
            got, st = db.score_all(q, b62, GapModel(10, 2))
            assert (got == exp).all()
            assert st["rescored_i32"] >= 2


def test_wide_mode_matrix_outside_int8(port, b62):
    """Matrix entries x40 and large gaps: the packed path does not apply, everything runs in int32."""
    rng = np.random.default_rng(13)
    big = (b62 * 40).astype(np.int32)
    seqs = [synth.random_residues(rng, int(rng.integers(0, 400))) for _ in range(90)]
    q = synth.random_residues(rng, 333)
    seqs[7] = synth.mutate(rng, q, 0.1, 1)
    fdb = po.FlatDb.from_list(seqs)
    for gaps in [(400, 80), (200, 200)]:
        with Database(fdb.codes, fdb.offsets, length_threshold=200) as db:
            got, _ = db.score_all(q, big, GapModel(*gaps))
            assert (got == port.score_all(q, fdb, big, *gaps)).all()
    # an asymmetric matrix: the lookup order matrix[subject][query] (align.hpp:34,74) is what matters
    asym = b62.copy()
    asym[3, 5] += 6
    asym[11, 2] -= 3
    with Database(fdb.codes, fdb.offsets) as db:
        got, _ = db.score_all(q, asym, GapModel(10, 2))
        assert (got == port.score_all(q, fdb, asym, 10, 2)).all()


def test_topk_edges(port, b62):
    rng = np.random.default_rng(14)
    g = GapModel(10, 2)
    # many ties, including at the top-k boundary: 40 copies of 5 distinct sequences + empties
    base = [synth.random_residues(rng, 60) for _ in range(5)]
    seqs = [base[i % 5].copy() for i in range(200)] + [enc("")] * 5
    q = base[2][:40]
    fdb = po.FlatDb.from_list(seqs)
    exp = port.score_all(q, fdb, b62, 10, 2)
    with Database(fdb.codes, fdb.offsets) as db:
        for k in (1, 39, 40, 41, 205, 1000, 1025, 5000):
            idx, sc, _ = db.search(q, b62, g, k)
            ni, ns = naive_rank(exp, k)
            assert (idx == ni).all() and (sc == ns).all(), k
    # N < top_k and all-zero scores: order is db_index ascending
    stars = [np.full(int(rng.integers(0, 9)), 23, np.uint8) for _ in range(7)]
    with Database.from_sequences(stars) as db:
        idx, sc, _ = db.search(enc("AAAA"), b62, g, 10)
        assert idx.tolist() == list(range(7)) and sc.tolist() == [0] * 7
    # k > 1024 on a larger database takes the full-sort path
    seqs = [synth.random_residues(rng, int(rng.integers(0, 80))) for _ in range(6000)]
    fdb = po.FlatDb.from_list(seqs)
    q = synth.random_residues(rng, 50)
    exp = port.score_all(q, fdb, b62, 10, 2)
    with Database(fdb.codes, fdb.offsets) as db:
        for k in (1024, 1500, 6000):
            idx, sc, _ = db.search(q, b62, g, k)
            ni, ns = naive_rank(exp, k)
            assert (idx == ni).all() and (sc == ns).all(), k


def test_empty_database_and_empty_query(b62):
    g = GapModel(10, 2)
    with Database(np.zeros(0, np.uint8), np.zeros(1, np.uint64)) as db:
        idx, sc, _ = db.search(enc("AAA"), b62, g, 10)
        assert len(idx) == 0 and len(sc) == 0
    rng = np.random.default_rng(15)
    seqs = [synth.random_residues(rng, 30) for _ in range(12)]
    with Database.from_sequences(seqs) as db:
        idx, sc, _ = db.search(enc(""), b62, g, 5)                            # empty query: all zeros, index order
        assert idx.tolist() == [0, 1, 2, 3, 4] and sc.tolist() == [0] * 5
        with pytest.raises(IndexError, match="query code outside matrix alphabet"):
            db.search(np.array([1, 2, 24], np.uint8), b62, g, 5)
        with pytest.raises(ValueError, match="top_k must be >= 1"):
            db.search(enc("AAA"), b62, g, 0)
    with pytest.raises(IndexError):                                            # subject residue outside the alphabet
        Database.from_sequences([np.array([3, 99], np.uint8)])


def test_long_query_profile_from_global_memory(port, b62):
    """m = 9,600: the int8 profile (25 x m) no longer fits the 227 KB of shared memory."""
    rng = np.random.default_rng(16)
    q = synth.random_residues(rng, 9600)
    seqs = [synth.random_residues(rng, int(rng.integers(1, 260))) for _ in range(70)]
    seqs[5] = q[4000:4200].copy()
    fdb = po.FlatDb.from_list(seqs)
    with Database(fdb.codes, fdb.offsets) as db:
        got, _ = db.score_all(q, b62, GapModel(10, 2))
        assert (got == port.score_all(q, fdb, b62, 10, 2)).all()


def test_intra_task_multi_pass_and_long_subject(port, b62):
    """Query wider than one intra-task pass (8 warps x 32 lanes x 8 columns = 2048) and a long subject."""
    rng = np.random.default_rng(17)
    q = synth.random_residues(rng, 4700)
    s = synth.mutate(rng, q, 0.3, 4)
    s = np.concatenate([synth.random_residues(rng, 800), s, synth.random_residues(rng, 1500)])
    exp = port.score_scalar(q, s, b62, 10, 2)
    assert score_wavefront(q, s, b62, GapModel(10, 2), 64) == exp
    assert score_wavefront(s, q, b62, GapModel(10, 2), 1) == port.score_scalar(s, q, b62, 10, 2)
    # the same pair through the database path with a wavefront of units (threshold 0 -> long pool)
    with Database.from_sequences([s, q[:100]], length_threshold=0) as db:
        got, st = db.score_all(q, b62, GapModel(10, 2))
        assert got[0] == exp and st["wavefront_scored"] == 2


def test_multi_shard_equals_single(port, b62):
    """Scheduling invisibility, GPU edition: shard counts 1/2/3/8 give the identical ranked list."""
    qs, sdb = synth.config1()
    g = GapModel(10, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        i1, s1, _ = db.search(qs[0], b62, g, 25)
    for shards in (2, 3, 8):
        mdb = MultiGpuDatabase(sdb.codes, sdb.offsets, [0] * shards)
        i2, s2, st = mdb.search(qs[0], b62, g, 25)
        mdb.close()
        assert (i1 == i2).all() and (s1 == s2).all()
        assert st["lane_scored"] + st["wavefront_scored"] == sdb.n
        # the per-rank flavour: every shard's keys, merged on the device
        keys = []
        total = np.full(sdb.n, -1, dtype=np.int32)
        for r in range(shards):
            with Database(sdb.codes, sdb.offsets, shard_rank=r, shard_count=shards) as part:
                k, _, _ = part.search_keys(qs[0], b62, g, 25)
                keys.append(k)
                part.score_all(qs[0], b62, g, out=total)
        i3, s3 = merge_keys(np.concatenate(keys), 25)
        assert (i1 == i3).all() and (s1 == s3).all()
        assert (total >= 0).all()            # every sequence was scored by exactly one shard
    i4, s4 = decode_keys(keys[0])
    assert len(i4) <= 25


def test_traceback_matches_reference_scripts(b62):
    """sw_align_traceback on the GPU: identical bounds and edit scripts, not merely equal scores
    (fixtures: outputs of the unmodified reference, tests/golden/make_golden.py)."""
    from paper_2203_11100_b200 import align_traceback
    for rec in golden()["tracebacks"]:
        if rec.get("capped_only"):
            continue
        q, s, g = enc(rec["q"]), enc(rec["s"]), GapModel(rec["open"], rec["extend"])
        tb = align_traceback(q, s, b62, g)
        assert tb["score"] == rec["score"] and tb["bounds"] == rec["bounds"] and not tb["capped"]
        assert tb["ops"].tolist() == rec["ops"]
        capped = align_traceback(q, s, b62, g, memory_cap=64)
        assert capped["capped"] and capped["score"] == rec["score"] and len(capped["ops"]) == 0
    assert align_traceback(enc(""), enc("AAA"), b62, GapModel(10, 2))["score"] == 0


def test_traceback_random_against_reference(ref, b62):
    from paper_2203_11100_b200 import align_traceback
    rng = np.random.default_rng(21)
    shapes = [(1, 1), (7, 300), (300, 7), (64, 64), (257, 255), (900, 1100), (2100, 700), (3000, 2600)]
    for i, (m, n) in enumerate(shapes):
        q = synth.random_residues(rng, m)
        s = synth.mutate(rng, np.concatenate([synth.random_residues(rng, n // 3), q[: max(1, min(m, n // 2))],
                                              synth.random_residues(rng, n)])[:n], 0.15, 3)
        for gaps in [(10, 2), (5, 5), (3, 0), (0, 0)][: 2 if m * len(s) > 10 ** 6 else 4]:
            exp = ref.traceback(q, s, b62, *gaps)
            got = align_traceback(q, s, b62, GapModel(*gaps))
            assert got["score"] == exp["score"], (m, n, gaps)
            assert got["bounds"] == exp["bounds"], (m, n, gaps)
            assert got["ops"].tolist() == exp["ops"].tolist(), (m, n, gaps)


def test_traceback_equal_maxima_across_passes(ref, b62):
    """Two equal maxima that ONE thread of the fill kernel meets in the wrong order: the query is wider than one pass
    (m > 2048), the copy in its second pass ends at an earlier subject row than the copy in its first pass, and both end
    in columns owned by the same thread (8-column lane tiles 12 and 256 + 12).  The end point must be the first maximum
    in row-major order (align.hpp:308), so bounds and edit script equal the reference's."""
    from paper_2203_11100_b200 import align_traceback
    rng = np.random.default_rng(8)
    W, P = synth.ALPHABET.index("W"), synth.ALPHABET.index("P")
    d1 = synth.random_residues(rng, 100)
    d2 = d1[::-1].copy()                                  # same composition: the same self score
    q = np.full(2300, W, np.uint8)
    q[0:100] = d2                                         # ends in column 100   (lane tile 12, pass 0)
    q[2048:2148] = d1                                     # ends in column 2148  (lane tile 268 = 256 + 12, pass 1)
    s = np.full(800, P, np.uint8)
    s[10:110] = d1                                        # matches the pass-1 copy, ends in row 110
    s[500:600] = d2                                       # matches the pass-0 copy, ends in row 600
    exp = ref.traceback(q, s, b62, 10, 2)
    got = align_traceback(q, s, b62, GapModel(10, 2))
    assert exp["bounds"][1] == 2148 and exp["bounds"][3] == 110       # the reference picks the earlier row
    assert got["score"] == exp["score"] and got["bounds"] == exp["bounds"] and got["ops"].tolist() == exp["ops"].tolist()


def test_packed_database_file_round_trip(tmp_path, b62):
    qs, sdb = synth.config1()
    g = GapModel(10, 2)
    path = tmp_path / "config1.swb"
    with Database(sdb.codes, sdb.offsets, shard_rank=1, shard_count=3) as db:
        i1, s1, _ = db.search(qs[0], b62, g, 30)
        info1 = db.info()
        db.save(path)
    with Database.load(path) as db2:
        i2, s2, _ = db2.search(qs[0], b62, g, 30)
        info2 = db2.info()
    assert (i1 == i2).all() and (s1 == s2).all()
    for key in ("n_total", "n_local", "n_short", "n_long", "n_groups", "residues", "shard_rank", "shard_count", "max_length"):
        assert info1[key] == info2[key]
    bad = tmp_path / "bad.swb"
    bad.write_bytes(path.read_bytes()[:100])
    with pytest.raises(ValueError):
        Database.load(bad)
    with pytest.raises(ValueError):
        Database.load(tmp_path / "missing.swb")


def test_batched_traceback_of_search_hits(ref, b62):
    """run_search's default (compute_alignments = true, scheduler.hpp:246-249): every hit's alignment equals the
    reference's sw_align_traceback, for one shard and for several."""
    qs, sdb = synth.config1()
    g = GapModel(10, 2)
    q = qs[0]
    lens = sdb.lengths()
    with Database(sdb.codes, sdb.offsets) as db:
        idx, sc, _ = db.search(q, b62, g, 12)
        got = db.align_hits(q, b62, g, idx, sc, lens[idx])
        capped = db.align_hits(q, b62, g, idx[:3], sc[:3], lens[idx[:3]], memory_cap=1000)
    assert all(c["capped"] and c["score"] == int(s) and len(c["ops"]) == 0 for c, s in zip(capped, sc[:3]))
    for i, a in zip(idx, got):
        exp = ref.traceback(q, sdb.seq(int(i)), b62, 10, 2)
        assert a["score"] == exp["score"] and a["bounds"] == exp["bounds"] and a["ops"].tolist() == exp["ops"].tolist()
    mdb = MultiGpuDatabase(sdb.codes, sdb.offsets, [0, 0, 0])
    i2, s2, _ = mdb.search(q, b62, g, 12)
    got2 = mdb.align_hits(q, b62, g, i2, s2, lens[i2])
    mdb.close()
    assert (i2 == idx).all()
    for a, b in zip(got, got2):
        assert a["bounds"] == b["bounds"] and a["ops"].tolist() == b["ops"].tolist() and a["score"] == b["score"]


def test_kernel_equivalence_property(port, b62):
    """>= 1000 random pairs, lengths 1-500: scalar == batch (every lane width) == wavefront,
    exact integers.  Here: oracle scalar vs the packed DPX kernel (score_batch) vs the intra-task kernel."""
    rng = np.random.default_rng(41)
    checked = 0
    for lane_width in (1, 4, 8, 16, 32, 64):
        for _ in range(4):
            q = synth.random_residues(rng, int(rng.integers(1, 501)))
            subs = [synth.random_residues(rng, int(rng.integers(1, 501))) for _ in range(lane_width)]
            if rng.random() < 0.5:
                subs[0] = synth.mutate(rng, q, 0.2, 2)
            go = int(rng.integers(0, 14)); ge = int(rng.integers(0, go + 1))
            got = score_batch(q, subs, lane_width, b62, GapModel(go, ge))
            exp = [port.score_scalar(q, s, b62, go, ge) for s in subs]
            assert got.tolist() == exp
            checked += lane_width
    # one big batch brings the total past 1000 pairs
    q = synth.random_residues(rng, 333)
    subs = [synth.random_residues(rng, int(rng.integers(1, 501))) for _ in range(600)]
    assert score_batch(q, subs, 600, b62, GapModel(10, 2)).tolist() == [port.score_scalar(q, s, b62, 10, 2) for s in subs]
    checked += 600
    assert checked >= 1000
    for _ in range(12):
        q = synth.random_residues(rng, int(rng.integers(1, 501)))
        s = synth.random_residues(rng, int(rng.integers(1, 501)))
        assert score_wavefront(q, s, b62, GapModel(10, 2), int(rng.choice([1, 4, 64, len(q)]))) == port.score_scalar(q, s, b62, 10, 2)


def test_config5_shape_blosum50_with_overflow(port):
    """BASELINE config 5 at reduced size: BLOSUM50, gap 12/2, a query long enough that its planted copies leave
    the int16 range and must come back exact from the int32 re-run."""
    b50 = synth.blosum50()
    queries = synth.make_queries([300, 8000], seed=55)
    sdb = synth.make_database(1500, target_residues=450_000, max_len=9000, queries=queries, seed=55)
    g = GapModel(12, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        for qi, q in enumerate(queries):
            got, st = db.score_all(q, b50, g)
            idx, sc, _ = db.search(q, b50, g, 10)
            assert idx[0] == sdb.planted[qi][0]
            sample = np.unique(np.concatenate([np.array(sdb.planted[qi]), np.arange(0, sdb.n, 97)]))
            exp = port.score_all(q, po.FlatDb.from_list([sdb.seq(int(i)) for i in sample]), b50, 12, 2)
            assert (got[sample] == exp).all()
            if qi == 1:
                assert st["rescored_i32"] >= 1 and sc[0] > 32767


def test_pipelined_multi_query_equals_one_by_one(b62):
    """swb_search_many: same ranked lists as separate searches, for queries of very different lengths (different
    kernel variants, re-run on/off) issued back to back."""
    rng = np.random.default_rng(61)
    qs, sdb = synth.config1()
    queries = [qs[0], synth.random_residues(rng, 7), sdb.seq(sdb.planted[0][1]), synth.random_residues(rng, 1500),
               enc(""), synth.random_residues(rng, 3300)]
    g = GapModel(10, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        single = [db.search(q, b62, g, 15)[:2] for q in queries]
        many, ms = db.search_many(queries, b62, g, 15)
        again, _ = db.search_many(queries[::-1], b62, g, 15)
    for (i1, s1), (i2, s2), (i3, s3) in zip(single, many, again[::-1]):
        assert (i1 == i2).all() and (s1 == s2).all() and (i1 == i3).all() and (s1 == s3).all()
    assert (ms > 0).all()


def test_concurrent_callers_on_one_database(b62):
    """run_search "may be called concurrently from many threads on the same db": calls on one handle
    are serialised inside the library and every caller gets the single-threaded answer."""
    import threading
    qs, sdb = synth.config1()
    rng = np.random.default_rng(71)
    queries = [qs[0]] + [synth.random_residues(rng, int(rng.integers(20, 400))) for _ in range(5)]
    g = GapModel(10, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        expected = [db.search(q, b62, g, 10)[:2] for q in queries]
        results = [None] * 12
        def worker(slot):
            results[slot] = db.search(queries[slot % len(queries)], b62, g, 10)[:2]
        threads = [threading.Thread(target=worker, args=(i,)) for i in range(12)]
        [t.start() for t in threads]
        [t.join() for t in threads]
    for slot, (idx, sc) in enumerate(results):
        ei, es = expected[slot % len(queries)]
        assert (idx == ei).all() and (sc == es).all()


@pytest.mark.parametrize("policy", [Database.SCAN_PIPELINE, Database.SCAN_WAVEFRONT])
@pytest.mark.parametrize("seed,thr,gaps", [(11, 3000, (10, 2)), (12, 100, (11, 1)), (13, 0, (5, 5)), (14, 10 ** 9, (0, 0))])
def test_random_databases_on_each_scan_kernel(port, b62, seed, thr, gaps, policy):
    """Every group forced through the on-chip tile pipeline (and, for contrast, through the wavefront kernel):
    all scores and the ranked list equal the oracle's.  Query lengths straddle the tile (32) and pass (16 tiles
    = 512 columns) boundaries of the pipeline."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(200, 1500))
    seqs = [synth.random_residues(rng, int(rng.integers(0, 400))) for _ in range(n)]
    seqs[0] = synth.random_residues(rng, 2500)      # one tall group
    seqs[1] = np.zeros(0, np.uint8)
    fdb = po.FlatDb.from_list(seqs)
    with Database(fdb.codes, fdb.offsets, length_threshold=thr) as db:
        db.set_scan_policy(policy)
        for m in (1, 31, 32, 33, 300, 511, 512, 513, 545, 1100):
            q = synth.random_residues(rng, m)
            got, st = db.score_all(q, b62, GapModel(*gaps))
            exp = port.score_all(q, fdb, b62, *gaps)
            assert (got == exp).all(), f"m={m}"
        q = synth.mutate(rng, seqs[0], 0.1, 3)[:1500]   # a query with a strong hit in the tall group
        idx, sc, _ = db.search(q, b62, GapModel(*gaps), 25)
        ei, es, _ = port.run_search(q, fdb, b62, *gaps, length_threshold=thr, top_k=25)
        assert (idx == ei).all() and (sc == es).all()


def test_hybrid_scan_equals_each_kernel_alone(b62):
    """A database large enough for the automatic policy to split the work (tall groups to the wavefront kernel,
    the rest to the pipeline, side by side on two streams): identical score vectors under all three policies,
    including back-to-back searches that reuse the border arrays and ticket counters."""
    rng = np.random.default_rng(81)
    queries = synth.make_queries([700, 1200], seed=81)
    sdb = synth.make_database(40_000, target_residues=12_000_000, max_len=9000, queries=queries, seed=81)
    g = GapModel(10, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        ref = {}
        for policy in (Database.SCAN_WAVEFRONT, Database.SCAN_PIPELINE, Database.SCAN_AUTO, Database.SCAN_AUTO):
            db.set_scan_policy(policy)
            for qi, q in enumerate(queries):
                got, st = db.score_all(q, b62, g)
                if qi in ref:
                    assert (got == ref[qi]).all(), f"policy {policy} query {qi}"
                else:
                    ref[qi] = got
                idx, sc, _ = db.search(q, b62, g, 10)
                assert idx[0] == sdb.planted[qi][0]


def test_two_query_scan_against_the_oracle():
    """swb_search_many with its shared scans forced onto small random databases (tests/_duo_small.py, in a
    subprocess because the policy knobs are read once per process): every ranked list equals the oracle's, for
    query lengths around the tile and pass boundaries, four gap models, all routing thresholds."""
    import os, subprocess, sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, SWB200_DUO_MINGROUPS="0.001")
    out = subprocess.run([sys.executable, str(root / "tests" / "_duo_small.py")], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "DUO-SMALL-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]


def test_narrow_block_sweep_against_the_oracle():
    """The wavefront kernel's narrow units (blocks of 8 rows x 8 or 4 columns in anti-diagonal order, handed from tile to
    tile through link buffers whose data is the flag, for groups whose chain of rows bounds the search) forced onto small
    databases, alone and next to the pipeline: whole score vectors equal the oracle's (tests/_narrow_small.py)."""
    import os, subprocess, sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    for extra in ({}, {"SWB200_NARROW_FINE": "0.0001"}):      # 8-column tiles; 4-column tiles wherever the wavefront is shallow
        env = dict(os.environ, SWB200_NARROW="0.0001", **extra)
        out = subprocess.run([sys.executable, str(root / "tests" / "_narrow_small.py")], cwd=root, env=env, capture_output=True,
                             text=True, timeout=900)
        assert out.returncode == 0 and "NARROW-SMALL-OK" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]
        if extra:
            assert "(4, 256, True)" in out.stdout, out.stdout[-1500:]     # 4-column tiles, CTAs of 4 + 4 warps (helpers), link buffers


def test_pipeline_tile_slices_against_the_oracle():
    """The pipeline kernel with per-warp tile slices instead of the whole profile in shared memory (queries beyond ~6,500
    residues): forced for every query length (SWB200_PIPE_SLICES=1), and by itself for 6,600- and 7,000-residue queries;
    whole score vectors equal the oracle's (tests/_slice_small.py)."""
    import os, subprocess, sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    for extra in ({"SWB200_PIPE_SLICES": "1"}, {}):
        env = dict(os.environ, **extra)
        env.pop("SWB200_PIPE_SLICES", None) if not extra else None
        out = subprocess.run([sys.executable, str(root / "tests" / "_slice_small.py")], cwd=root, env=env, capture_output=True,
                             text=True, timeout=900)
        assert out.returncode == 0 and "SLICE-SMALL-OK" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


def test_large_random_batch_shares_scans_and_equals_single_searches(b62):
    """A batch of 60 queries of random lengths (with duplicates, an empty one and a one-residue one) on a database
    where shared scans apply: swb_search_many's ranked lists equal swb_search's, query by query, and the plan it
    follows (swb_batch_plan) puts every non-empty query into a shared scan."""
    from paper_2203_11100_b200 import batch_plan
    rng = np.random.default_rng(91)
    lens = [300, 450, 800, 1200, 950, 1400] + [int(x) for x in rng.integers(50, 3000, size=50)] + [777, 777, 0, 1]
    queries = [synth.random_residues(rng, m) for m in lens]
    sdb = synth.make_database(40_000, target_residues=11_000_000, max_len=1500, queries=queries[:6], seed=91)
    scan, stream = batch_plan(sdb.lengths(), lens)
    assert scan[58] == -1 and (scan[:58] >= 0).all() and scan[59] >= 0
    g = GapModel(11, 1)
    with Database(sdb.codes, sdb.offsets) as db:
        many, ms = db.search_many(queries, b62, g, 7)
        for qi in list(range(0, 60, 7)) + [56, 57, 58, 59]:
            idx, sc, _ = db.search(queries[qi], b62, g, 7)
            assert (many[qi][0] == idx).all() and (many[qi][1] == sc).all(), f"query {qi} (m={lens[qi]})"
        for qi in range(6):
            assert many[qi][0][0] == sdb.planted[qi][0]


def test_search_many_edge_cases(port, b62):
    """Batches the shared scans cannot or need not serve: no queries, only empty queries, top_k beyond the database,
    a matrix outside the packed int16 range (every query falls back to the int32 kernel, one by one), duplicates."""
    rng = np.random.default_rng(97)
    seqs = [synth.random_residues(rng, int(rng.integers(1, 200))) for _ in range(40)]
    fdb = po.FlatDb.from_list(seqs)
    g = GapModel(10, 2)
    q1, q2 = synth.random_residues(rng, 300), synth.random_residues(rng, 310)
    with Database(fdb.codes, fdb.offsets) as db:
        out, ms = db.search_many([], b62, g, 5)
        assert out == [] and len(ms) == 0
        out, _ = db.search_many([enc(""), enc("")], b62, g, 5)
        assert all(len(i) == 5 and (s == 0).all() for i, s in out)                # every sequence is a hit with score 0
        out, _ = db.search_many([q1, q2, q1], b62, g, 100)                        # top_k > n: all 40, duplicates equal
        assert len(out[0][0]) == 40 and (out[0][0] == out[2][0]).all() and (out[0][1] == out[2][1]).all()
        for q, (idx, sc) in zip([q1, q2], out):
            ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=100)
            assert (idx == ei).all() and (sc == es).all()
        wide = (b62 * 40).astype(np.int32)                                        # entries + open outside int8
        out, _ = db.search_many([q1[:80], q2[:90]], wide, GapModel(400, 80), 6)
        for q, (idx, sc) in zip([q1[:80], q2[:90]], out):
            ei, es, _ = port.run_search(q, fdb, wide, 400, 80, top_k=6)
            assert (idx == ei).all() and (sc == es).all()


def test_traceback_in_several_rounds():
    """The direction matrices of a call's hits are bounded in sum (pairs.inl): with SWB200_TRACEBACK_ROUND_KB=64 the twelve
    hits of test_batched_traceback_of_search_hits are traced back in several rounds and must give the same edit scripts."""
    import os, subprocess, sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-x", "-k", "traceback and not several_rounds"], cwd=root,
                         env=dict(os.environ, SWB200_TRACEBACK_ROUND_KB="64"), capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and " passed" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


def test_adhoc_entry_points_from_many_threads(port, b62):
    """sw_score_scalar / sw_score_batch / sw_score_wavefront / merge_results take plain sequences (align.hpp:42,91,166,
    scheduler.hpp:106): each call builds a handle from the library's block cache (cabi.cu: BlockCacheScope).  Six threads
    mix the four entry points with shapes that change from call to call (blocks move between size classes and
    threads), next to a resident database whose blocks never enter the cache; every result against the oracle."""
    import threading
    from paper_2203_11100_b200 import encode_keys
    qs, sdb = synth.config1()
    g = GapModel(10, 2)
    errors = []

    def worker(seed):
        rng = np.random.default_rng(seed)
        try:
            for it in range(25):
                q = synth.random_residues(rng, int(rng.integers(1, 700)))
                kind = (seed + it) % 4
                if kind == 0:
                    s = synth.random_residues(rng, int(rng.integers(1, 3000)))
                    assert score_wavefront(q, s, b62, g, 64) == port.score_scalar(q, s, b62, 10, 2)
                elif kind == 1:
                    subs = [synth.random_residues(rng, int(rng.integers(1, 900))) for _ in range(int(rng.integers(1, 70)))]
                    got = score_batch(q, subs, len(subs), b62, g)
                    assert got.tolist() == [port.score_scalar(q, s, b62, 10, 2) for s in subs]
                elif kind == 2:
                    n = int(rng.integers(1, 30000))
                    index = rng.permutation(n).astype(np.uint32)
                    score = rng.integers(0, 50, n).astype(np.int32)
                    k = int(rng.integers(1, 40))
                    idx, sc = merge_keys(encode_keys(index, score), k)
                    order = np.lexsort((index, -score.astype(np.int64)))[:k]
                    assert idx.tolist() == index[order].tolist() and sc.tolist() == score[order].tolist()
                else:
                    seqs = [synth.random_residues(rng, int(rng.integers(1, 400))) for _ in range(70)]
                    with Database.from_sequences(seqs) as small:     # a resident handle: driver blocks, not the cache
                        idx, sc, _ = small.search(q, b62, g, 5)
                    ei, es, _ = port.run_search(q, po.FlatDb.from_list(seqs), b62, 10, 2, top_k=5)
                    assert idx.tolist() == list(ei) and sc.tolist() == list(es)
        except Exception as e:   # noqa: BLE001 -- reported by the main thread
            errors.append((seed, repr(e)))

    with Database(sdb.codes, sdb.offsets) as db:
        before = db.search(qs[0], b62, g, 10)[:2]
        threads = [threading.Thread(target=worker, args=(100 + i,)) for i in range(6)]
        [t.start() for t in threads]
        [t.join() for t in threads]
        after = db.search(qs[0], b62, g, 10)[:2]
    assert not errors, errors
    assert (before[0] == after[0]).all() and (before[1] == after[1]).all()
