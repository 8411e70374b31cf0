"""The per-rank sharded search on the GPU: keys stay on the device between the shard's select, the exchange and
the global select (ShardedSearch.search -> swb_search_keys_device -> all-gather -> swb_db_merge_keys)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2203_11100_b200 import Database, GapModel, synth
from paper_2203_11100_b200.dist import ShardedSearch

pytestmark = pytest.mark.gpu


def test_sharded_search_device_path_world1_against_the_oracle(lib, port, b62):
    """world = 1 through the SAME code path the N > 1 ranks take (device tensors, one download of k hits)."""
    import torch
    queries = synth.make_queries([1, 60, 144, 700], seed=5)
    sdb = synth.make_database(3000, target_residues=900_000, queries=queries, seed=5)
    fdb = po.FlatDb(sdb.codes, sdb.offsets)
    g = GapModel(10, 2)
    eng = ShardedSearch(sdb.codes, sdb.offsets, device_index=0, device_path=True)
    try:
        for k in (1, 10, 37):
            for q in queries:
                idx, sc, st = eng.search(q, b62, g, k)
                ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=k)
                assert (idx == ei).all() and (sc == es).all(), f"m={len(q)} k={k}"
                assert st["cells"] == len(q) * sdb.residues and st["ms_total"] > 0
        # back-to-back searches reuse the send/receive tensors and the pinned buffers: interleave with the direct path
        for q in queries[::-1]:
            a = eng.search(q, b62, g, 10)
            b = eng.db.search(q, b62, g, 10)
            assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        # another stream than the default one
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            idx, sc, _ = eng.search(queries[2], b62, g, 10)
        ei, es, _ = port.run_search(queries[2], fdb, b62, 10, 2, top_k=10)
        assert (idx == ei).all() and (sc == es).all()
    finally:
        eng.close()


def test_device_keys_of_shards_merge_to_the_single_list(lib, b62):
    """Three shards on one device: each leaves its k keys in device memory (swb_search_keys_device), the concatenation is
    merged on the device (swb_db_merge_keys) -- the data flow of N ranks without the collective.  A shard smaller than k
    pads with zeros."""
    import torch
    qs, sdb = synth.config1()
    g = GapModel(10, 2)
    k = 40
    with Database(sdb.codes, sdb.offsets) as db:
        i1, s1, _ = db.search(qs[0], b62, g, k)
    shards = [Database(sdb.codes, sdb.offsets, shard_rank=r, shard_count=3) for r in range(3)]
    try:
        gathered = torch.zeros(3 * k, dtype=torch.int64, device="cuda")
        stream = torch.cuda.current_stream()
        for r, part in enumerate(shards):
            part.set_stream(stream.cuda_stream)
            part.search_keys_device(qs[0], b62, g, k, gathered[r * k:].data_ptr())
        idx, sc, st = shards[0].merge_keys_device(gathered.data_ptr(), 3 * k, k, len(qs[0]))
        assert (idx == i1).all() and (sc == s1).all()
    finally:
        for part in shards:
            part.close()
    tiny = synth.from_sequences([synth.random_residues(np.random.default_rng(1), n) for n in (30, 0, 50)])
    with Database(tiny.codes, tiny.offsets) as db:
        buf = torch.full((8,), -1, dtype=torch.int64, device="cuda")
        db.set_stream(torch.cuda.current_stream().cuda_stream)
        db.search_keys_device(qs[0][:40], b62, g, 8, buf.data_ptr())
        idx, sc, _ = db.merge_keys_device(buf.data_ptr(), 8, 8, 40)
        ref_i, ref_s, _ = db.search(qs[0][:40], b62, g, 8)
        assert len(idx) == 3 and (idx == ref_i).all() and (sc == ref_s).all()
        assert (buf[3:].cpu().numpy() == 0).all()
