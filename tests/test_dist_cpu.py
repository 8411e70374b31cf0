"""World-size-2 gloo test of the multi-rank path's host logic (runs on CPU):
shard assignment -> per-shard top-k (computed here by the oracle, standing in for each rank's GPU) ->
all-gather of packed keys -> merged list == the single-process ranked list."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as po
        from paper_2203_11100_b200 import search, synth
        from paper_2203_11100_b200.dist import exchange_keys
        oracle = po.Port()
        b62 = synth.blosum62()
        queries = synth.make_queries([60], seed=77)
        sdb = synth.make_database(900, target_residues=90_000, max_len=4000, queries=queries, seed=77,
                                  tail_fraction=0.01)
        lens = sdb.lengths()
        top_k = 12
        shard_of = search.shard_assignment(lens, 3000, world)
        mine = np.nonzero(shard_of == rank)[0]
        # this rank's shard scored by the checker (the GPU does this in production)
        local = po.FlatDb.from_list([sdb.seq(int(i)) for i in mine])
        scores = oracle.score_all(queries[0], local, b62, 10, 2)
        li, ls = oracle.merge(mine.astype(np.uint32), scores, top_k)
        keys = np.zeros(top_k, dtype=np.uint64)
        keys[:len(li)] = search.encode_keys(li, ls)
        gathered = exchange_keys(keys)                      # gloo all_gather of k keys per rank
        assert gathered.shape == (world * top_k,)
        merged = np.sort(gathered[gathered != 0])[::-1][:top_k]
        gi, gs = search.decode_keys(merged)
        # single-process truth
        full = po.FlatDb(sdb.codes, sdb.offsets)
        ei, es, _ = oracle.run_search(queries[0], full, b62, 10, 2, top_k=top_k)
        ok = (gi == ei).all() and (gs == es).all()
        # the batched flavour: three queries, ONE all-gather of 3 x k keys per rank, merged per query (merge_many)
        from paper_2203_11100_b200.dist import merge_many
        batch = synth.make_queries([40, 75, 130], seed=78)
        block = np.zeros((len(batch), top_k), dtype=np.uint64)
        for qn, q in enumerate(batch):
            bi, bs = oracle.merge(mine.astype(np.uint32), oracle.score_all(q, local, b62, 10, 2), top_k)
            block[qn, :len(bi)] = search.encode_keys(bi, bs)
        merged_many = merge_many(exchange_keys(block.reshape(-1)), world, len(batch), top_k)
        for q, (mi, ms_) in zip(batch, merged_many):
            ti, ts, _ = oracle.run_search(q, full, b62, 10, 2, top_k=top_k)
            ok = ok and (mi == ti).all() and (ms_ == ts).all()
        np.save(os.path.join(result_dir, f"ok{rank}.npy"), np.array([int(ok), len(mine)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_merge_equals_single_process(tmp_path, lib):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    sizes = []
    for r in range(world):
        ok, n = np.load(tmp_path / f"ok{r}.npy")
        assert ok == 1
        sizes.append(n)
    assert abs(sizes[0] - sizes[1]) <= 2
