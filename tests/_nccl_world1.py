"""Helper for tests/test_gpu_dist.py: the per-rank sharded search over NCCL with a world of one rank (what one GPU can
run): process group "nccl", ShardedSearch through the device-key path, all_gather_into_tensor on the search's stream, and
the same for a batch (search_many's host-key exchange).  Prints NCCL-WORLD1-OK."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
import torch.distributed as dist

from oracle import pyoracle as po
from paper_2203_11100_b200 import GapModel, synth
from paper_2203_11100_b200.dist import ShardedSearch, exchange_keys, merge_many
from paper_2203_11100_b200.search import encode_keys

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", sys.argv[1] if len(sys.argv) > 1 else "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
ok = True
try:
    port = po.Port()
    b62 = synth.blosum62()
    g = GapModel(10, 2)
    queries = synth.make_queries([50, 144, 400], seed=9)
    sdb = synth.make_database(4000, target_residues=1_200_000, queries=queries, seed=9)
    fdb = po.FlatDb(sdb.codes, sdb.offsets)
    eng = ShardedSearch(sdb.codes, sdb.offsets, device_index=0, device_path=True)
    for rep in range(3):
        for q in queries:
            idx, sc, st = eng.search(q, b62, g, 10)
            ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=10)
            ok &= bool((idx == ei).all() and (sc == es).all())
    # the batched flavour's exchange: host keys -> CUDA tensor -> all-gather -> host
    local, _ = eng.db.search_many(queries, b62, g, 10)
    keys = np.zeros((len(queries), 10), dtype=np.uint64)
    for i, (bi, bs) in enumerate(local):
        keys[i, :len(bi)] = encode_keys(bi, bs)
    merged = merge_many(exchange_keys(keys.reshape(-1), torch.device("cuda", 0)), 1, len(queries), 10)
    for q, (mi, ms) in zip(queries, merged):
        ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=10)
        ok &= bool((mi == ei).all() and (ms == es).all())
    eng.close()
finally:
    dist.destroy_process_group()
print("NCCL-WORLD1-OK" if ok else "NCCL-WORLD1-FAIL")
sys.exit(0 if ok else 1)
