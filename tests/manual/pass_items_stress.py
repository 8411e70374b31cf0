"""Repeated batched sweeps on shards of the config-2 database (pass items: passes of a half-group on different CTAs,
linked through global border rows and progress counters): every repetition's ranked lists must equal the single
searches', and the device time of the batch is printed beside the single searches' (the margin the GPU test asserts).

    gpurun -- 'python tests/manual/pass_items_stress.py [reps]'
"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: F401

from paper_2203_11100_b200 import Database, GapModel, synth


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    queries, sdb = synth.config2()
    b62, g = synth.blosum62(), GapModel(10, 2)
    bad = 0
    for shard_count, shard_rank in ((4, 1), (2, 0), (8, 5)):
        with Database(sdb.codes, sdb.offsets, shard_rank=shard_rank, shard_count=shard_count) as shard:
            singles = [shard.search(q, b62, g, 10) for q in queries]
            single_ms = sum(s[2]["ms_total"] for s in singles)
            times = []
            for rep in range(reps):
                many, ms = shard.search_many(queries, b62, g, 10)
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
                  f"max {max(times):.1f} first {times[0]:.1f} ms over {reps} reps", flush=True)
    print("mismatches:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
