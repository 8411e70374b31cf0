"""Generates tests/golden/golden_v1.json by running the UNMODIFIED reference (oracle/_ref/libswref.so,
compiled from /root/reference by oracle/Makefile).  Run in the authoring container:

    python tests/golden/make_golden.py

The fixture pins oracle/sw_oracle.c (tests/test_oracle.py) and the CUDA path (tests/test_gpu_parity.py)
on machines where /root/reference does not exist.  Sequences are stored as residue letters.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import pyoracle as po  # noqa: E402
from paper_2203_11100_b200 import synth  # noqa: E402

ref = po.Ref()
b62 = ref.blosum62()
rng = np.random.Generator(np.random.PCG64(20220311100))


def letters(codes):
    return "".join(synth.ALPHABET[c] for c in codes)


def rand_seq(n, alphabet=23):
    if alphabet >= 23:
        return synth.random_residues(rng, n)
    return rng.integers(0, alphabet, size=n, dtype=np.uint8)


out = {"about": "outputs of the unmodified reference (align.hpp, scheduler.hpp) on seeded inputs",
       "blosum62": b62.reshape(-1).tolist()}

# ---- pairs: scalar == wavefront(chunk widths) -----------------------------------------------------------
pairs = []
shapes = [(0, 5), (5, 0), (1, 1), (3, 3), (17, 40), (64, 64), (65, 129), (200, 33), (257, 300), (500, 500),
          (31, 700), (700, 31), (128, 1000)]
for (m, n) in shapes:
    for (go, ge) in [(10, 2), (11, 1), (5, 5), (12, 2), (0, 0)]:
        q, s = rand_seq(m), rand_seq(n)
        if m and n and rng.random() < 0.5:   # make it homologous
            k = min(m, n)
            s[:k] = q[:k]
            s = synth.mutate(rng, s, 0.15, 2)
        rec = {"q": letters(q), "s": letters(s), "open": go, "extend": ge,
               "scalar": ref.score_scalar(q, s, b62, go, ge), "wavefront": {}}
        for cw in (1, 4, 64, max(1, m)):
            rec["wavefront"][str(cw)] = ref.score_wavefront(q, s, b62, go, ge, cw)
        pairs.append(rec)
out["pairs"] = pairs

# ---- lane batches ----------------------------------------------------------------------------------------
batches = []
for lw in (1, 4, 8, 16, 32, 64):
    for rep in range(3):
        m = int(rng.integers(1, 260))
        cnt = int(rng.integers(0, lw + 1))
        q = rand_seq(m)
        subs = []
        for _ in range(cnt):
            r = rng.random()
            if r < 0.12:
                subs.append(None)
            elif r < 0.2:
                subs.append(rand_seq(0))
            else:
                subs.append(rand_seq(int(rng.integers(1, 400))))
        go, ge = [(10, 2), (11, 1), (8, 8)][rep]
        got = ref.score_batch(q, subs, lw, b62, go, ge)
        batches.append({"q": letters(q), "subjects": [None if s is None else letters(s) for s in subs],
                        "lane_width": lw, "open": go, "extend": ge, "scores": got.tolist()})
# a lane that saturates int16 (W x W = 11 per residue): exercises align.hpp:149-153
w = np.full(3100, synth.ALPHABET.index("W"), dtype=np.uint8)
w2 = w.copy(); w2[::97] = 0
filler = rand_seq(50)
got = ref.score_batch(w, [w2, filler, w[:2990]], 4, b62, 10, 2)
batches.append({"q": letters(w), "subjects": [letters(w2), letters(filler), letters(w[:2990])], "lane_width": 4,
                "open": 10, "extend": 2, "scores": got.tolist(), "note": "int16 saturation"})
out["batches"] = batches

# ---- run_search on small databases ---------------------------------------------------------------------------
searches = []
for case in range(6):
    n = [0, 1, 7, 200, 333, 150][case]
    seqs = [rand_seq(int(rng.integers(0, 320))) for _ in range(n)]
    thr = [3000, 3000, 3000, 3000, 120, 0][case]
    m = [20, 20, 33, 144, 97, 60][case]
    q = rand_seq(m)
    if n >= 7:
        seqs[3] = q.copy()
        seqs[5] = synth.mutate(rng, q, 0.2, 2)
    if n >= 200:   # ties: duplicates of the same sequence at different indices
        seqs[10] = seqs[150].copy()
        seqs[11] = seqs[150].copy()
        seqs[120] = rand_seq(0)
    top_k = [10, 10, 10, 10, 25, 400][case]
    fdb = po.FlatDb.from_list(seqs)
    h = ref.db_create(fdb)
    base = None
    for (wc, lw, cw) in [(1, 8, 64), (4, 1, 1), (8, 32, 64), (2, 8, 1)]:
        idx, sc, st = ref.run_search(h, q, b62, 10, 2, worker_count=wc, lane_width=lw, chunk_width=cw,
                                     length_threshold=thr, top_k=top_k, cpu_pool_threads=max(1, wc // 2))
        if base is None:
            base = (idx, sc, st)
        assert (idx == base[0]).all() and (sc == base[1]).all(), "reference is not schedule-invariant?!"
    all_scores = [ref.score_scalar(q, s, b62, 10, 2) for s in seqs]
    ref.db_destroy(h)
    searches.append({"q": letters(q), "db": [letters(s) for s in seqs], "length_threshold": thr, "top_k": top_k,
                     "open": 10, "extend": 2, "hits_index": base[0].tolist(), "hits_score": base[1].tolist(),
                     "lane_scored": int(base[2][0]), "wavefront_scored": int(base[2][1]),
                     "all_scores": all_scores})
out["searches"] = searches

# ---- merge_results --------------------------------------------------------------------------------------------
merges = []
for parts, k in [([([3], [50]), ([1], [50])], 10), ([([], []), ([4, 2], [7, 9])], 1), ([([0, 1, 2], [5, 5, 5])], 2),
                 ([([9, 8], [0, 0]), ([7], [0]), ([], [])], 10)]:
    idx, sc = ref.merge_results(parts, k)
    merges.append({"parts": [[list(map(int, p[0])), list(map(int, p[1]))] for p in parts], "top_k": k,
                   "index": idx.tolist(), "score": sc.tolist()})
out["merges"] = merges

# ---- traceback (outside the hot path; pins the host C++ in include/swsearch/align.hpp) --------------------
tbs = []
for (m, n) in [(12, 12), (40, 55), (80, 30), (150, 170)]:
    q, s = rand_seq(m), rand_seq(n)
    k = min(m, n) // 2
    s[2:2 + k] = q[1:1 + k]
    s = synth.mutate(rng, s, 0.1, 2)
    tb = ref.traceback(q, s, b62, 10, 2)
    tbs.append({"q": letters(q), "s": letters(s), "open": 10, "extend": 2, "bounds": tb["bounds"], "score": tb["score"],
                "capped": tb["capped"], "ops": tb["ops"].tolist(), "rescored": tb["rescored"]})
tb = ref.traceback(rand_seq(100), rand_seq(100), b62, 10, 2, memory_cap=1000)
tbs.append({"q": None, "capped_only": True, "capped": tb["capped"], "n_ops": len(tb["ops"])})
out["tracebacks"] = tbs

path = Path(__file__).with_name("golden_v1.json")
path.write_text(json.dumps(out, separators=(",", ":")))
print("wrote", path, path.stat().st_size, "bytes")
