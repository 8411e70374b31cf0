"""Host cost per call of the ad-hoc entry points (swb_score_pair, swb_score_batch, swb_align_traceback, swb_merge_keys):
each builds a handle per call; with the block cache (csrc/cabi.cu: BlockCacheScope) its device and pinned blocks are reused.
Run twice: as is, and with SWB200_NO_BLOCK_CACHE=1 (every block from the driver, the behaviour before the cache)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_11100_b200 import GapModel, align_traceback, merge_keys, score_batch, score_wavefront, synth  # noqa: E402
from paper_2203_11100_b200.search import encode_keys  # noqa: E402


def per_call(fn, n):
    fn()
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    b62 = synth.blosum62()
    g = GapModel(10, 2)
    rng = np.random.default_rng(5)
    q = rng.integers(0, 20, 300, dtype=np.uint8)
    s = rng.integers(0, 20, 400, dtype=np.uint8)
    subs = [rng.integers(0, 20, int(l), dtype=np.uint8) for l in rng.integers(50, 600, 16)]
    keys = encode_keys(np.arange(4000, dtype=np.uint32), rng.integers(1, 500, 4000).astype(np.int32))
    mode = "driver blocks (SWB200_NO_BLOCK_CACHE)" if os.environ.get("SWB200_NO_BLOCK_CACHE") else "block cache"
    print(f"{mode}: us per call over {n} calls")
    print(f"  score_wavefront 300 x 400      {per_call(lambda: score_wavefront(q, s, b62, g, 64), n):9.1f}")
    print(f"  score_batch 300 x 16 subjects  {per_call(lambda: score_batch(q, subs, 16, b62, g), n):9.1f}")
    print(f"  align_traceback 300 x 400      {per_call(lambda: align_traceback(q, s, b62, g), n):9.1f}")
    print(f"  merge_keys 4000 -> 10          {per_call(lambda: merge_keys(keys, 10), n):9.1f}")


if __name__ == "__main__":
    main()
