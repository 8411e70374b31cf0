"""Repeated batched sweeps on shards of the config-2 database (pass items: passes of a half-group on different CTAs,
linked through global border rows and progress counters): every repetition's ranked lists must equal the single
searches', and the device time of the batch is printed beside the single searches' (the margin the GPU test asserts).

    gpurun -- 'python tests/manual/pass_items_stress.py [reps] [--dirty 0xFF] [--batch-first] [--shards 4:1,2:0,8:5]'

--dirty       fill the free device memory with a byte pattern first, so that every buffer the library allocates starts
              out dirty (a fresh box hands out memory of unknown content)
--batch-first the batched sweep is the FIRST GPU work of the process on each shard (that is when the one unexplained
              failure of round 1 happened); the single searches it is compared with run afterwards
tests/test_gpu_stress.py runs this in a fresh process as a bounded -m gpu test.
"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: F401

from paper_2203_11100_b200 import Database, GapModel, synth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="?", type=int, default=10)
    ap.add_argument("--dirty", default=None)
    ap.add_argument("--batch-first", action="store_true")
    ap.add_argument("--shards", default="4:1,2:0,8:5")
    args = ap.parse_args()
    if args.dirty is not None:
        import torch
        free, _ = torch.cuda.mem_get_info()
        junk = torch.empty(int(free * 0.9), dtype=torch.uint8, device="cuda")
        junk.fill_(int(args.dirty, 0))
        torch.cuda.synchronize()
        del junk
        torch.cuda.empty_cache()
        print(f"filled {int(free * 0.9) >> 20} MiB with {args.dirty}", flush=True)
    queries, sdb = synth.config2()
    b62, g = synth.blosum62(), GapModel(10, 2)
    bad = 0
    for spec in args.shards.split(","):
        shard_count, shard_rank = (int(x) for x in spec.split(":"))
        with Database(sdb.codes, sdb.offsets, shard_rank=shard_rank, shard_count=shard_count) as shard:
            first = shard.search_many(queries, b62, g, 10) if args.batch_first else None
            singles = [shard.search(q, b62, g, 10) for q in queries]
            single_ms = sum(s[2]["ms_total"] for s in singles)
            times = []
            for rep in range(args.reps):
                many, ms = first if (rep == 0 and first is not None) else shard.search_many(queries, b62, g, 10)
                times.append(float(ms.sum()))
                for qi in ((7 * rep) % len(queries), (7 * rep + 3) % len(queries)):   # single searches in between, as callers mix them
                    idx1, sc1, _ = shard.search(queries[qi], b62, g, 10)
                    if not ((idx1 == singles[qi][0]).all() and (sc1 == singles[qi][1]).all()):
                        bad += 1
                        print(f"SINGLE MISMATCH shard {shard_rank}/{shard_count} rep {rep} query {qi}", flush=True)
                for qi, (idx, sc, _) in enumerate(singles):
                    if not ((many[qi][0] == idx).all() and (many[qi][1] == sc).all()):
                        bad += 1
                        print(f"MISMATCH shard {shard_rank}/{shard_count} rep {rep} query {qi} (m={len(queries[qi])}): "
                              f"{many[qi][0].tolist()} {many[qi][1].tolist()} != {idx.tolist()} {sc.tolist()}", flush=True)
            print(f"shard {shard_rank}/{shard_count}: singles {single_ms:.1f} ms, batch min {min(times):.1f} "
                  f"max {max(times):.1f} first {times[0]:.1f} ms over {args.reps} reps", flush=True)
    print("mismatches:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
