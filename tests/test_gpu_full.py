"""BASELINE.json's full-size configuration (config 2: Swiss-Prot-shaped database, 565,928 sequences,
~204 M residues) checked through size-independent properties plus sampled parity against the oracle."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2203_11100_b200 import Database, GapModel, MultiGpuDatabase, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full(lib):
    import torch
    assert torch.cuda.is_available()
    queries, sdb = synth.config2()
    db = Database(sdb.codes, sdb.offsets)
    yield queries, sdb, db
    db.close()


def test_shape(full):
    queries, sdb, db = full
    info = db.info()
    assert info["n_total"] == synth.SWISSPROT_SEQS
    assert abs(info["residues"] - synth.SWISSPROT_RESIDUES) / synth.SWISSPROT_RESIDUES < 0.01
    assert info["max_length"] == synth.SWISSPROT_MAXLEN
    assert info["n_long"] > 1000 and info["n_short"] + info["n_long"] == info["n_total"]
    assert info["padded_residues"] / info["residues"] < 1.03       # length sorting keeps padding under 3 %


@pytest.mark.parametrize("qi", [0, 9, 19])
def test_planted_copy_is_top_hit_with_self_score(full, port, b62, qi):
    queries, sdb, db = full
    q = queries[qi]
    idx, sc, st = db.search(q, b62, GapModel(10, 2), 10)
    exact = sdb.planted[qi][0]
    assert idx[0] == exact
    assert sc[0] == port.score_scalar(q, q, b62, 10, 2)            # self score = the ceiling for this query
    assert (np.diff(sc.astype(np.int64)) <= 0).all()               # sorted
    for i, s in zip(idx[:4], sc[:4]):                              # planted homologs, exact values
        assert s == port.score_scalar(q, sdb.seq(int(i)), b62, 10, 2)
    assert set(sdb.planted[qi][:3]) <= set(int(i) for i in idx)
    assert st["cells"] == len(q) * sdb.residues
    idx2, sc2, _ = db.search(q, b62, GapModel(10, 2), 10)           # determinism
    assert (idx2 == idx).all() and (sc2 == sc).all()


def test_sampled_score_parity(full, port, b62):
    queries, sdb, db = full
    q = queries[3]                                                  # m = 375
    got, _ = db.score_all(q, b62, GapModel(10, 2))
    rng = np.random.default_rng(2)
    lens = sdb.lengths()
    sample = np.unique(np.concatenate([rng.choice(sdb.n, 3000, replace=False), np.argsort(lens)[-40:],
                                       np.nonzero(lens == 0)[0][:5], np.array(sdb.planted[3])]))
    sub = po.FlatDb.from_list([sdb.seq(int(i)) for i in sample])
    exp = port.score_all(q, sub, b62, 10, 2)
    assert (got[sample] == exp).all()
    assert (got >= 0).all()


def test_sampled_score_parity_through_the_pipeline(full, port, b62):
    """m = 1000 takes the hybrid scan (on-chip pipeline + wavefront kernel on the tall groups): sampled scores equal
    the oracle's, and the whole score vector equals the wavefront kernel's."""
    queries, sdb, db = full
    q = queries[9]
    got, st = db.score_all(q, b62, GapModel(10, 2))
    rng = np.random.default_rng(3)
    lens = sdb.lengths()
    sample = np.unique(np.concatenate([rng.choice(sdb.n, 1200, replace=False), np.argsort(lens)[-12:],
                                       np.nonzero(lens == 0)[0][:5], np.array(sdb.planted[9])]))
    sub = po.FlatDb.from_list([sdb.seq(int(i)) for i in sample])
    exp = port.score_all(q, sub, b62, 10, 2)
    assert (got[sample] == exp).all()
    db.set_scan_policy(Database.SCAN_WAVEFRONT)
    try:
        alone, _ = db.score_all(q, b62, GapModel(10, 2))
    finally:
        db.set_scan_policy(Database.SCAN_AUTO)
    assert (got == alone).all()


@pytest.fixture(scope="module")
def oracle_sample(full, port, b62):
    """Seeded sample of the config-2 database (3,000 random sequences + the 40 longest + empties + length-1 records +
    every planted homolog of every query) and the oracle's scores of ALL 20 queries against it (~1e11 cells on the
    host cores)."""
    queries, sdb, _ = full
    rng = np.random.default_rng(20)
    lens = sdb.lengths()
    planted = np.array([i for qi in range(len(queries)) for i in sdb.planted[qi]])
    sample = np.unique(np.concatenate([rng.choice(sdb.n, 3000, replace=False), np.argsort(lens)[-40:],
                                       np.nonzero(lens == 0)[0], np.nonzero(lens == 1)[0], planted]))
    sub = po.FlatDb.from_list([sdb.seq(int(i)) for i in sample])
    expected = np.stack([port.score_all(q, sub, b62, 10, 2) for q in queries])
    return sample, expected


def test_batched_sweep_score_vectors_against_the_oracle(full, oracle_sample, b62):
    """The timed path of bench.py on the timed configuration: the whole 20-query sweep through swb_search_many's plan
    (one shared scan of two query streams, duo_pipeline_kernel) -- score VECTORS, not ranked lists, against
    oracle/sw_oracle.c for all 20 queries on the sample."""
    queries, sdb, db = full
    sample, expected = oracle_sample
    scores, scan_of, _ = db.score_many(queries, b62, GapModel(10, 2))
    assert (scan_of >= 0).all(), f"every query of the sweep is planned into a shared scan, got {scan_of}"
    assert scores.shape == (len(queries), sdb.n)
    for qi, q in enumerate(queries):
        bad = np.nonzero(scores[qi][sample] != expected[qi])[0]
        assert len(bad) == 0, f"query {qi} (m={len(q)}): {len(bad)} of {len(sample)} sampled scores differ, first db_index {sample[bad[0]]}"
        assert scores[qi][sdb.planted[qi][0]] == scores[qi].max()      # the exact copy carries the self score
    assert (scores >= 0).all()


def test_single_search_score_vectors_against_the_oracle(full, oracle_sample, b62):
    """The drop-in path (one swb_search per query: pipeline_s16_kernel + wavefront_s16_kernel): score vectors of all
    20 queries against the oracle on the sample, and equal to the batched path's everywhere."""
    queries, sdb, db = full
    sample, expected = oracle_sample
    batched, _, _ = db.score_many(queries, b62, GapModel(10, 2))
    for qi, q in enumerate(queries):
        got, st = db.score_all(q, b62, GapModel(10, 2))
        bad = np.nonzero(got[sample] != expected[qi])[0]
        assert len(bad) == 0, f"query {qi} (m={len(q)}): {len(bad)} sampled scores differ, first db_index {sample[bad[0]]}"
        assert (got == batched[qi]).all(), f"query {qi}: single and batched score vectors differ"


def test_batched_sweep_equals_single_searches(full, b62):
    """swb_search_many over the whole 20-query sweep (the queries share one database scan as two streams of the
    two-stream kernel): every ranked list equals the one swb_search returns."""
    queries, sdb, db = full
    many, ms = db.search_many(queries, b62, GapModel(10, 2), 10)
    assert len(many) == len(queries) and (ms > 0).all()
    for qi, q in enumerate(queries):
        idx, sc, _ = db.search(q, b62, GapModel(10, 2), 10)
        assert (many[qi][0] == idx).all() and (many[qi][1] == sc).all(), f"query {qi} (m={len(q)})"
        assert idx[0] == sdb.planted[qi][0]
    again, _ = db.search_many(queries[::-1], b62, GapModel(10, 2), 10)      # other order, other pairing
    for (i1, s1), (i2, s2) in zip(many, again[::-1]):
        assert (i1 == i2).all() and (s1 == s2).all()


def test_batched_sweep_on_a_shard_uses_pass_items(full, b62):
    """A quarter of the database still holds a 35,213-residue sequence: as one item it would outlast the shared scan,
    so swb_search_many hands out single passes of 16 tiles (consecutive passes of a half-group on different CTAs,
    linked through global border rows and progress counters).  Ranked lists equal the single searches'."""
    from paper_2203_11100_b200 import batch_plan
    queries, sdb, _ = full
    assert (batch_plan(sdb.lengths(), [len(q) for q in queries], shard_rank=1, shard_count=4)[0] == 0).all()
    with Database(sdb.codes, sdb.offsets, shard_rank=1, shard_count=4) as shard:
        many, ms = shard.search_many(queries, b62, GapModel(10, 2), 10)
        for qi in (0, 5, 11, 19):
            idx, sc, _ = shard.search(queries[qi], b62, GapModel(10, 2), 10)
            assert (many[qi][0] == idx).all() and (many[qi][1] == sc).all(), f"query {qi}"
        # and it is faster than one scan per query (device times; the batch timed on a repeat call, so that the first
        # launch of the pass-item kernel and the first allocation of its progress counters are not in it)
        many2, ms2 = shard.search_many(queries, b62, GapModel(10, 2), 10)
        for a, b in zip(many, many2):
            assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        single_ms = sum(shard.search(q, b62, GapModel(10, 2), 10)[2]["ms_total"] for q in queries)
        assert min(ms.sum(), ms2.sum()) < single_ms, f"batch {ms.sum():.1f} / {ms2.sum():.1f} ms, singles {single_ms:.1f} ms"


def test_multi_shard_batched_sweep_equals_single_gpu(full, b62):
    """swb_mdb_search_many: the batch on four shards at once (one host thread per shard, here all on device 0; pass
    items on each), merged per query on the host: the same ranked lists as the unsharded database."""
    queries, sdb, db = full
    batch = [queries[i] for i in (0, 4, 9, 12, 16, 19)]
    mdb = MultiGpuDatabase(sdb.codes, sdb.offsets, [0, 0, 0, 0])
    try:
        many, ms = mdb.search_many(batch, b62, GapModel(10, 2), 25)
    finally:
        mdb.close()
    assert (ms > 0).all()
    for q, (idx, sc) in zip(batch, many):
        ei, es, _ = db.search(q, b62, GapModel(10, 2), 25)
        assert (idx == ei).all() and (sc == es).all()


def test_two_query_scan_with_overflow(port):
    """BLOSUM50 12/2 with two long queries whose planted copies leave the int16 range: the shared scan flags them
    and each query's flagged lanes come back exact from the int32 re-run."""
    b50 = synth.blosum50()
    queries = synth.make_queries([7600, 8000], seed=56)
    sdb = synth.make_database(30_000, target_residues=9_000_000, max_len=9000, queries=queries, seed=56)
    g = GapModel(12, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        many, _ = db.search_many(queries, b50, g, 8)
        for qi, q in enumerate(queries):
            idx, sc, st = db.search(q, b50, g, 8)
            assert (many[qi][0] == idx).all() and (many[qi][1] == sc).all()
            assert idx[0] == sdb.planted[qi][0] and sc[0] > 32767 and st["rescored_i32"] >= 1
            assert sc[0] == port.score_scalar(q, q, b50, 12, 2)


def test_sharded_full_database(full, b62):
    queries, sdb, db = full
    q = queries[6]
    i1, s1, _ = db.search(q, b62, GapModel(10, 2), 50)
    mdb = MultiGpuDatabase(sdb.codes, sdb.offsets, [0, 0, 0, 0])
    i2, s2, st = mdb.search(q, b62, GapModel(10, 2), 50)
    mdb.close()
    assert (i1 == i2).all() and (s1 == s2).all()


def test_shard_of_eight_short_queries_against_the_oracle(lib, port, b62):
    """One GPU's 1/8 share of the config-2 database (what BASELINE config 4 gives every rank at N = 8): the short queries
    are chain-bound there and take the wavefront kernel's narrow units in their fastest form -- 4-column tiles, CTAs of
    4 + 4 warps (helper warps carry the blocks), link buffers whose data is the flag -- next to the pipeline.  Score
    vectors of the shard's sequences against the oracle on a seeded sample that includes every sequence of the tall
    groups' head; repeated, because the link buffers must come back empty from every search."""
    from paper_2203_11100_b200 import scan_plan, shard_assignment
    queries, sdb = synth.config2()
    lens = sdb.lengths()
    mine = np.nonzero(shard_assignment(lens, 3000, 8) == 0)[0]
    rng = np.random.default_rng(8)
    longest = mine[np.argsort(lens[mine])[-80:]]
    sample = np.unique(np.concatenate([rng.choice(mine, 1500, replace=False), longest]))
    sub = po.FlatDb.from_list([sdb.seq(int(i)) for i in sample])
    g = GapModel(10, 2)
    with Database(sdb.codes, sdb.offsets, shard_rank=0, shard_count=8) as db:
        for rep in range(2):
            for qi in (0, 1, 2, 3):                                    # m = 144, 189, 222, 375
                q = queries[qi]
                plan = scan_plan(lens, len(q), shard_rank=0, shard_count=8)
                assert plan["narrow_groups"] > 0 and plan["narrow_link_bytes"] > 0 and plan["pipeline_groups"] > 0
                if qi == 0:
                    assert plan["narrow_tile"] == 4 and plan["wavefront_threads"] == 256
                got = np.full(sdb.n, -1, dtype=np.int32)
                got, st = db.score_all(q, b62, g, out=got)
                exp = port.score_all(q, sub, b62, 10, 2)
                assert (got[sample] == exp).all(), f"m={len(q)} rep={rep}"
                assert (got[mine] >= 0).all() and st["cells"] == len(q) * int(lens[mine].sum())
