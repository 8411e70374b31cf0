"""Compares the on-chip pipeline kernel (SWB200_PIPE=1) with the wavefront kernel (SWB200_PIPE=0) on the same
database: identical score vectors, per-query timing.  Usage: python tests/manual/pipe_experiment.py [maxlen] [scale]"""
import os, subprocess, sys
sys.path.insert(0, ".")
import numpy as np

LENS = [144, 222, 375, 567, 1000, 2005, 3005, 5478]


def child(maxlen, scale, out):
    from paper_2203_11100_b200 import synth, Database, GapModel
    qs = synth.make_queries(LENS, 7)
    n = int(synth.SWISSPROT_SEQS * scale)
    sdb = synth.make_database(n, target_residues=int(synth.SWISSPROT_RESIDUES * scale), max_len=maxlen, queries=qs, seed=7)
    b62 = synth.blosum62()
    res = {}
    with Database(sdb.codes, sdb.offsets) as db:
        for q in qs:
            scores, _ = db.score_all(q, b62, GapModel(10, 2))
            res[f"s{len(q)}"] = scores
            db.search(q, b62, GapModel(10, 2), 10)
            best = None
            for _ in range(3):
                idx, sc, st = db.search(q, b62, GapModel(10, 2), 10)
                if best is None or st["ms_scan"] < best["ms_scan"]:
                    best = st
            print(f"  m={len(q):5d} scan={best['ms_scan']:8.3f} ms  GCUPS={best['cells']/best['ms_scan']/1e6:7.1f}  launches={best['kernel_launches']}", flush=True)
    np.savez(out, **res)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), float(sys.argv[3]), sys.argv[4])
        sys.exit(0)
    maxlen = int(sys.argv[1]) if len(sys.argv) > 1 else 2999
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    os.makedirs("gpurun_out", exist_ok=True)
    outs = {}
    for mode in ("0", "1"):
        print(f"SWB200_PIPE={mode}", flush=True)
        env = dict(os.environ, SWB200_PIPE=mode)
        outs[mode] = f"/tmp/pipe_exp_{mode}.npz"
        subprocess.run([sys.executable, __file__, "child", str(maxlen), str(scale), outs[mode]], env=env, check=True, timeout=int(os.environ.get('PIPE_EXP_TIMEOUT', '120')))
    a, b = np.load(outs["0"]), np.load(outs["1"])
    bad = 0
    for k in a.files:
        d = int((a[k] != b[k]).sum())
        bad += d
        print(f"{k}: {d} differing scores of {len(a[k])}")
    print("PARITY", "OK" if bad == 0 else "FAIL")
