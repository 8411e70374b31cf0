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


def test_nccl_all_gather_on_the_search_stream_world1(lib):
    """The NCCL flavour of the per-rank path as far as one GPU can run it: process group "nccl" with one rank, the search
    enqueued on torch's current stream, all_gather_into_tensor on the tensor the library filled, the global select on the
    gathered tensor (tests/_nccl_world1.py, in a process of its own because it owns a process group)."""
    import os, socket, subprocess, sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_no = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, str(root / "tests" / "_nccl_world1.py"), str(port_no)], cwd=root, capture_output=True, text=True,
                         timeout=600, env=dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no)))
    assert out.returncode == 0 and "NCCL-WORLD1-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]


def test_in_process_nccl_branch_on_one_gpu(lib):
    """swb_mdb_search's NCCL branch (dlopen of libnccl, ncclCommInitAll, grouped ncclAllGather on the shard's stream, device
    select) with a communicator of one device: tests/_nccl_inprocess.py under SWB200_FORCE_NCCL=1."""
    import subprocess, sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, str(root / "tests" / "_nccl_inprocess.py")], cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "NCCL-INPROCESS-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]
