"""Config 3 (only the sequences >= 3000 residues) under different wavefront-policy knobs.
usage: python tests/manual/config3_tune.py VAR=v1,v2 ... """
import itertools, os, subprocess, sys
sys.path.insert(0, ".")


def child():
    import numpy as np
    from paper_2203_11100_b200 import synth, Database, GapModel, scan_plan
    qs, sdb = synth.config2()
    lens = sdb.lengths()
    sub = sdb.subset(np.nonzero(lens >= 3000)[0])
    b62 = synth.blosum62()
    out = []
    with Database(sub.codes, sub.offsets) as db:
        db.set_scan_policy(int(os.environ.get('TUNE_POLICY', '0')))
        for qi in (13, 16, 19):
            db.search(qs[qi], b62, GapModel(10, 2), 10)
            st = min((db.search(qs[qi], b62, GapModel(10, 2), 10)[2] for _ in range(3)), key=lambda s: s["ms_scan"])
            p = scan_plan(sub.lengths(), len(qs[qi]))
            out.append(f"{len(qs[qi])}:{st['cells']/st['ms_scan']/1e6:.0f}({st['ms_scan']:.1f}ms u={st['chunks_claimed']} n{p['narrow_groups']} s{p['split_groups']} r{p['rowblock_groups']})")
    print("RESULT " + "  ".join(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    knobs = [a.split("=") for a in sys.argv[1:]]
    names = [k for k, _ in knobs]
    for combo in itertools.product(*[v.split(",") for _, v in knobs]):
        env = dict(os.environ, **dict(zip(names, combo)))
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=300)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        print(" ".join(f"{n}={v}" for n, v in zip(names, combo)), "->", line[0][7:] if line else "FAILED " + r.stderr[-300:], flush=True)
