"""The C++ drop-in: tests/cpp/dropin_driver.cpp uses only the public swsearch API and is compiled twice --
against the unmodified reference headers (oracle/_ref/dropin_ref, CPU) and against include/swsearch +
libswb200.so (tests/cpp/_build/dropin_b200, GPU).  Their outputs must be byte-identical."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
MINE = ROOT / "tests" / "cpp" / "_build" / "dropin_b200"
REF = ROOT / "oracle" / "_ref" / "dropin_ref"
EXPECTED = ROOT / "tests" / "golden" / "dropin_expected.txt"


def _run(binary):
    return subprocess.run([str(binary)], capture_output=True, text=True, timeout=600, check=True).stdout


def test_dropin_output_equals_committed_reference_output(lib):
    """tests/golden/dropin_expected.txt is the reference build's output, captured in the authoring container."""
    assert MINE.exists(), "run __graft_entry__.build() first"
    got = _run(MINE)
    assert got == EXPECTED.read_text()


def test_dropin_output_equals_reference_binary(lib):
    if not REF.exists():
        pytest.skip("oracle/_ref/dropin_ref did not travel")
    assert _run(MINE) == _run(REF)


def test_cli_search_and_bench(lib, tmp_path, port):
    """The CLI on the GPU: ranked hits equal the oracle's, bench emits the SPEC's CSV."""
    import numpy as np
    from oracle import pyoracle as po
    from paper_2203_11100_b200 import synth
    cli = ROOT / "tests" / "cpp" / "_build" / "swsearch"
    rng = np.random.default_rng(31)
    letters = lambda codes: "".join(synth.ALPHABET[c] for c in codes)
    q = synth.random_residues(rng, 120)
    seqs = [synth.random_residues(rng, int(rng.integers(1, 300))) for _ in range(80)]
    seqs[13] = synth.mutate(rng, q, 0.1, 1)
    (tmp_path / "q.fa").write_text(">query one\n" + letters(q) + "\n")
    (tmp_path / "db.fa").write_text("".join(f">s{i}\n{letters(s)}\n" for i, s in enumerate(seqs)))
    out = subprocess.run([str(cli), "search", "-q", str(tmp_path / "q.fa"), "-d", str(tmp_path / "db.fa"), "--top-k", "5"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    ei, es, _ = port.run_search(q, po.FlatDb.from_list(seqs), synth.blosum62(), 10, 2, top_k=5)
    rows = [l.split("\t") for l in out.stdout.splitlines() if l.startswith("  ") and "\t" in l]
    assert [r[1] for r in rows] == [f"s{i}" for i in ei] and [int(r[2]) for r in rows] == es.tolist()
    assert "q[" in rows[0][3]
    csv = subprocess.run([str(cli), "bench", "-q", str(tmp_path / "q.fa"), "-d", str(tmp_path / "db.fa"), "--repetitions", "3"],
                         capture_output=True, text=True, timeout=600)
    assert csv.returncode == 0, csv.stderr
    lines = csv.stdout.splitlines()
    assert lines[0] == "query_id,query_length,repetitions,mean_gcups,min_gcups,max_gcups,stddev_gcups"
    assert lines[1].startswith("0,120,3,") and len(lines) == 2


def test_cli_search_from_a_packed_file_equals_the_oracle(lib, tmp_path, port):
    """SURVEY 8(f) rank 4 as a feature: `swsearch pack` once, then `search --packed` with no FASTA -- the residues go
    from the mapped file to the device as they are (swb_db_load), headers come from the file.  Ranked hits are checked
    against the ORACLE (not against the in-memory database), and the output is byte-identical to the FASTA run's."""
    import numpy as np
    from oracle import pyoracle as po
    from paper_2203_11100_b200 import Database, GapModel, synth
    cli = ROOT / "tests" / "cpp" / "_build" / "swsearch"
    rng = np.random.default_rng(77)
    letters = lambda codes: "".join(synth.ALPHABET[c] for c in codes)
    qs = [synth.random_residues(rng, 150), synth.random_residues(rng, 420)]
    seqs = [synth.random_residues(rng, int(n)) for n in list(rng.integers(1, 600, 400)) + [0, 1, 3500, 2999, 3000]]
    seqs[17] = synth.mutate(rng, qs[0], 0.1, 1)
    seqs[230] = synth.mutate(rng, qs[1], 0.2, 2)
    (tmp_path / "q.fa").write_text("".join(f">query{i}\n{letters(q)}\n" for i, q in enumerate(qs)))
    (tmp_path / "db.fa").write_text("".join(f">s{i} d\n{letters(s)}\n" for i, s in enumerate(seqs)))
    packed = tmp_path / "db.swb"
    assert subprocess.run([str(cli), "pack", "-d", str(tmp_path / "db.fa"), "-o", str(packed)], capture_output=True).returncode == 0
    a = subprocess.run([str(cli), "search", "-q", str(tmp_path / "q.fa"), "--packed", str(packed), "--top-k", "6"],
                       capture_output=True, text=True, timeout=600)
    b = subprocess.run([str(cli), "search", "-q", str(tmp_path / "q.fa"), "-d", str(tmp_path / "db.fa"), "--top-k", "6"],
                       capture_output=True, text=True, timeout=600)
    assert a.returncode == 0 and b.returncode == 0, a.stderr + b.stderr
    assert a.stdout == b.stdout
    fdb = po.FlatDb.from_list(seqs)
    rows = [l.split("\t") for l in a.stdout.splitlines() if l.startswith("  ") and "\t" in l]
    expect = []
    for q in qs:
        ei, es, _ = port.run_search(q, fdb, synth.blosum62(), 10, 2, top_k=6)
        expect += [(f"s{i} d", int(s)) for i, s in zip(ei, es)]
    assert [(r[1], int(r[2])) for r in rows] == expect
    # the same file through the Python binding: score vector of the LOADED database against the oracle
    with Database.load(packed) as db:
        got, _ = db.score_all(qs[1], synth.blosum62(), GapModel(10, 2))
        assert (got == port.score_all(qs[1], fdb, synth.blosum62(), 10, 2)).all()
        info = db.info()
        assert info["n_total"] == len(seqs) and info["n_long"] == 2 and info["length_threshold"] == 3000


def test_run_search_batch_equals_a_loop_of_run_search(lib):
    """include/swsearch/scheduler.hpp::run_search_batch (swb_search_many behind it, the queries sharing
    database scans): ranked lists, edit scripts and SearchStats identical to calling run_search per query."""
    exe = ROOT / "tests" / "cpp" / "_build" / "batch_unit"
    assert exe.exists(), "tests/cpp/_build/batch_unit is built by __graft_entry__.build()"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "batch_unit: ok" in out.stdout, out.stdout + out.stderr
    # the same program with the database sharded over two handles (both on device 0): swb_mdb_search_many
    import os
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, env=dict(os.environ, SWB200_DEVICES="0,0"))
    assert out.returncode == 0 and "batch_unit: ok" in out.stdout, out.stdout + out.stderr
