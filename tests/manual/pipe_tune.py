"""Sweeps the hybrid-scan policy knobs (environment variables read once per process) on the config-2 database.
usage: python tests/manual/pipe_tune.py VAR=v1,v2,... [VAR2=...] -- m1 m2 ..."""
import itertools, os, subprocess, sys
sys.path.insert(0, ".")


def child(lens):
    from paper_2203_11100_b200 import synth, Database, GapModel
    qs, sdb = synth.config2()
    qs = synth.make_queries(lens, 7)
    b62 = synth.blosum62()
    out = []
    shards = int(os.environ.get("TUNE_SHARDS", "1"))   # time shard 0 of N; numbers are N x shard throughput
    with Database(sdb.codes, sdb.offsets, shard_rank=0, shard_count=shards) as db:
        for q in qs:
            db.search(q, b62, GapModel(10, 2), 10)
            best = min(db.search(q, b62, GapModel(10, 2), 10)[2]["ms_scan"] for _ in range(3))
            out.append(f"{len(q)}:{len(q) * sdb.residues / best / 1e6:.0f}({best:.1f}ms)")
    print("RESULT " + "  ".join(out), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "child":
        child([int(x) for x in sys.argv[2:]])
        sys.exit(0)
    sep = sys.argv.index("--")
    knobs = [a.split("=") for a in sys.argv[1:sep]]
    lens = sys.argv[sep + 1:]
    names = [k for k, _ in knobs]
    for combo in itertools.product(*[v.split(",") for _, v in knobs]):
        env = dict(os.environ, **dict(zip(names, combo)))
        r = subprocess.run([sys.executable, __file__, "child", *lens], env=env, capture_output=True, text=True, timeout=300)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
        print(" ".join(f"{n}={v}" for n, v in zip(names, combo)), "->", line[0][7:] if line else "FAILED " + r.stderr[-300:], flush=True)
