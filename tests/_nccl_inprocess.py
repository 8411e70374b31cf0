"""Helper for tests/test_gpu_dist.py: the in-process multi-GPU flavour's NCCL branch on a single GPU.  With
SWB200_FORCE_NCCL=1 (read once per process, hence a process of its own) swb_mdb_create builds an ncclCommInitAll
communicator for its one device, and swb_mdb_search goes the whole way: persistent shard worker, keys left on the device,
grouped ncclAllGather on the shard's stream, device select, one download.  Prints NCCL-INPROCESS-OK."""
import os
import sys

os.environ["SWB200_FORCE_NCCL"] = "1"
sys.path.insert(0, ".")
from oracle import pyoracle as po
from paper_2203_11100_b200 import GapModel, MultiGpuDatabase, synth

port = po.Port()
b62 = synth.blosum62()
queries = synth.make_queries([60, 144, 300], seed=12)
sdb = synth.make_database(3000, target_residues=900_000, queries=queries, seed=12)
fdb = po.FlatDb(sdb.codes, sdb.offsets)
ok = True
mdb = MultiGpuDatabase(sdb.codes, sdb.offsets, [0])
for rep in range(3):
    for k in (1, 10, 33):
        for q in queries:
            idx, sc, st = mdb.search(q, b62, GapModel(10, 2), k)
            ei, es, _ = port.run_search(q, fdb, b62, 10, 2, top_k=k)
            ok &= bool((idx == ei).all() and (sc == es).all()) and st["lane_scored"] + st["wavefront_scored"] == sdb.n
mdb.close()
print("NCCL-INPROCESS-OK" if ok else "NCCL-INPROCESS-FAIL")
sys.exit(0 if ok else 1)
