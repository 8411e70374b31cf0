"""BASELINE configs 3 and 5 at realistic size on one GPU, with sampled parity against the oracle.

config 3  the long-sequence pool: queries >= 3005 against only the entries >= 3000 residues (24 groups).
config 5  one GPU's 1/8 share of the TrEMBL-shaped database (350 k sequences, 125 M residues), BLOSUM50 12/2, with
          queries long enough that planted copies overflow int16: the int32 re-run must fire and be exact.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2203_11100_b200 import Database, GapModel, synth

pytestmark = pytest.mark.gpu


def _sample(sdb, rng, n_random, n_longest, extra):
    lens = sdb.lengths()
    parts = [rng.choice(sdb.n, min(n_random, sdb.n), replace=False), np.argsort(lens)[-n_longest:],
             np.nonzero(lens == 0)[0][:4], np.array(sorted(extra), dtype=np.int64)]
    return np.unique(np.concatenate(parts))


def test_config3_long_pool_against_the_oracle(lib, port, b62):
    queries, sdb, _ = synth.config3()
    assert sdb.n > 1000 and sdb.lengths().min() >= 3000 and sdb.lengths().max() == synth.SWISSPROT_MAXLEN
    rng = np.random.default_rng(33)
    planted = {i for v in sdb.planted.values() for i in v}
    sample = _sample(sdb, rng, 60, 6, planted)
    sub = po.FlatDb.from_list([sdb.seq(int(i)) for i in sample])
    g = GapModel(10, 2)
    with Database(sdb.codes, sdb.offsets) as db:
        info = db.info()
        assert info["n_long"] == sdb.n and info["n_short"] == 0            # everything is intra-task pool (scheduler.hpp:59-62)
        batched, _, _ = db.score_many(queries, b62, g)
        for k, q in enumerate(queries):
            got, st = db.score_all(q, b62, g)
            assert st["wavefront_scored"] == sdb.n and st["lane_scored"] == 0
            exp = port.score_all(q, sub, b62, 10, 2)
            assert (got[sample] == exp).all(), f"m={len(q)}"
            assert (batched[k] == got).all()
            idx, sc, _ = db.search(q, b62, g, 10)
            assert idx[0] == sdb.planted[k][0] and sc[0] == got.max()
            order = np.lexsort((np.arange(sdb.n), -got.astype(np.int64)))[:10]   # (score desc, index asc), scheduler.hpp:111-114
            assert (idx == order).all() and (sc == got[order]).all()


def test_config5_share_overflow_and_rescore_against_the_oracle(lib, port):
    queries, sdb = synth.config5_share()
    assert sdb.n == synth.CONFIG5_SEQS // 8 and abs(sdb.residues - synth.CONFIG5_RESIDUES // 8) < 0.01 * synth.CONFIG5_RESIDUES / 8
    b50 = synth.blosum50()
    g = GapModel(12, 2)
    rng = np.random.default_rng(55)
    planted = {i for v in sdb.planted.values() for i in v}
    sample = _sample(sdb, rng, 2000, 20, planted)
    sub = po.FlatDb.from_list([sdb.seq(int(i)) for i in sample])
    with Database(sdb.codes, sdb.offsets) as db:
        batched, scan_of, rescored_b = db.score_many(queries, b50, g)
        assert (scan_of >= 0).sum() >= 2                                      # the batch shares scans here too
        total_rescored = 0
        for k, q in enumerate(queries):
            got, st = db.score_all(q, b50, g)
            exp = port.score_all(q, sub, b50, 12, 2)
            assert (got[sample] == exp).all(), f"single search, m={len(q)}"
            assert (batched[k] == got).all(), f"batched and single score vectors differ, m={len(q)}"
            assert rescored_b[k] == st["rescored_i32"]
            total_rescored += st["rescored_i32"]
            exact = sdb.planted[k][0]
            assert got[exact] == got.max() == port.score_scalar(q, q, b50, 12, 2)
            if len(q) >= 8000:
                assert got[exact] > 32767 and st["rescored_i32"] >= 1          # beyond int16: only the int32 re-run can be right
        assert total_rescored > 0
