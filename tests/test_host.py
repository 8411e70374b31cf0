"""CPU-side checks: the C-ABI library builds, loads and exports every symbol include/swb200.h declares
(no compute without a GPU), argument validation that happens before any CUDA call, the deterministic
sharding rule, the packed-key encoding, the synthetic data generator."""
import ctypes as C
import json
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2203_11100_b200 import _cabi, search, synth
from tests._util import enc

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol(lib):
    header = (ROOT / "include" / "swb200.h").read_text()
    declared = set(re.findall(r"\b(swb_[a-z0-9_]+)\s*\(", header))
    declared -= {"swb_status"}
    assert len(declared) >= 20
    for name in sorted(declared):
        assert hasattr(lib, name), f"libswb200.so does not export {name}"
        assert name in _cabi.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.swb_version().decode().startswith("swb200")


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    A = enc("AAA")
    with pytest.raises(search.SwbError):
        search.Database.from_sequences([A])
    with pytest.raises(search.SwbError):
        search.score_wavefront(A, A, synth.blosum62(), search.GapModel(10, 2), 4)
    with pytest.raises(search.SwbError):
        search.score_batch(A, [A], 4, synth.blosum62(), search.GapModel(10, 2))


def test_device_key_entry_points_validate_before_cuda(lib):
    """swb_search_keys_device / swb_db_merge_keys (the per-rank sharded search): a null handle or buffer is an argument
    error with a message, never a crash and never a CUDA call."""
    import ctypes as C
    from paper_2203_11100_b200 import _cabi
    hits = (_cabi.SwbHit * 4)()
    n = C.c_uint32(7)
    assert lib.swb_search_keys_device(None, None, 0, None, 10, 2, 4, None) != 0 and b"db is null" in lib.swb_last_error()
    assert lib.swb_db_merge_keys(None, None, 0, 4, hits, C.byref(n), 0, None) != 0 and b"db is null" in lib.swb_last_error()


def test_validation_before_cuda(lib, b62):
    A = enc("AAA")
    g = search.GapModel(10, 2)
    with pytest.raises(ValueError, match="lane_width must be >= 1"):       # align.hpp:93
        search.score_batch(A, [], 0, b62, g)
    with pytest.raises(ValueError, match="more subjects than lanes"):      # align.hpp:94-95
        search.score_batch(A, [A, A], 1, b62, g)
    with pytest.raises(ValueError, match="chunk_width must be >= 1"):      # align.hpp:169
        search.score_wavefront(A, A, b62, g, 0)
    with pytest.raises(IndexError, match="query code outside matrix alphabet"):   # scoring.hpp:203-205
        search.score_wavefront(np.array([24], np.uint8), A, b62, g, 4)
    with pytest.raises(ValueError, match="open >= extend >= 0"):           # scoring.hpp:51-52
        search.GapModel(1, 2)
    with pytest.raises(ValueError):
        search.GapModel(3, -1)
    for bad in (dict(worker_count=0), dict(lane_width=0), dict(chunk_width=0), dict(top_k=0)):
        with pytest.raises(ValueError, match="must be >= 1"):              # scheduler.hpp:30-35
            search.SearchConfig(**bad).validate()
    # degenerate inputs are not errors (align.hpp:45,100,172)
    assert search.score_wavefront(enc(""), A, b62, g, 4) == 0
    assert search.score_wavefront(A, enc(""), b62, g, 4) == 0
    assert search.score_batch(enc(""), [A], 2, b62, g).tolist() == [0, 0]
    assert search.score_batch(A, [], 3, b62, g).tolist() == [0, 0, 0]


def test_shard_assignment_balanced_and_deterministic(lib):
    rng = np.random.default_rng(3)
    lens = synth.random_lengths(rng, 20000, 7_200_000, 35213)
    for shards in (1, 2, 4, 8):
        a = search.shard_assignment(lens, 3000, shards)
        b = search.shard_assignment(lens, 3000, shards)
        assert (a == b).all() and a.max() == shards - 1
        res = np.array([lens[a == r].sum() for r in range(shards)], dtype=np.float64)
        cnt = np.array([(a == r).sum() for r in range(shards)])
        assert cnt.max() - cnt.min() <= 2
        assert res.max() / res.mean() < 1.02, res          # residue-balanced to 2 %
        long_cnt = np.array([((a == r) & (lens >= 3000)).sum() for r in range(shards)])
        assert long_cnt.max() - long_cnt.min() <= 1        # every shard gets its share of the long pool
    assert (search.shard_assignment(lens, 3000, 1) == 0).all()
    assert len(search.shard_assignment(np.zeros(0, np.uint32), 3000, 4)) == 0


def test_key_encoding_orders_like_merge_results(port):
    rng = np.random.default_rng(4)
    idx = rng.permutation(5000).astype(np.uint32)
    sc = rng.integers(0, 40, size=5000).astype(np.int32)          # many ties
    keys = search.encode_keys(idx, sc)
    order = np.argsort(keys)[::-1]
    oi, os_ = port.merge(idx, sc, 5000)                             # scheduler.hpp:111-114
    assert (idx[order] == oi).all() and (sc[order] == os_).all()
    di, ds = search.decode_keys(keys)
    assert (di == idx).all() and (ds == sc).all()
    assert (keys != 0).all()                                        # 0 is reserved as padding


def test_synth_is_deterministic_and_shaped():
    q1, d1 = synth.config1()
    q2, d2 = synth.config1()
    assert (d1.codes == d2.codes).all() and (d1.offsets == d2.offsets).all() and (q1[0] == q2[0]).all()
    assert d1.n == 10000 and len(q1[0]) == 144
    lens = d1.lengths()
    assert lens.max() == synth.SWISSPROT_MAXLEN and (lens == 0).sum() >= 2 and (lens == 1).sum() >= 2
    assert 3.3e6 < d1.residues < 3.9e6
    assert d1.codes.max() <= 22 and (d1.codes >= 20).mean() < 0.005
    exact = d1.planted[0][0]
    assert (d1.seq(exact) == q1[0]).all()
    assert (synth.blosum50() == synth.blosum50().T).all()
    assert synth.QUERY_LENGTHS[0] == 144 and synth.QUERY_LENGTHS[-1] == 5478 and len(synth.QUERY_LENGTHS) == 20
    # the GCUPS identity of SPEC.md:370
    assert abs(144 * synth.SWISSPROT_RESIDUES / 1.0 / 1e9 - 29.4009) < 1e-3


def _cpp_build():
    import subprocess
    subprocess.check_call(["make", "-C", str(ROOT / "tests" / "cpp"), "all"], stdout=subprocess.DEVNULL)
    return ROOT / "tests" / "cpp" / "_build"


def test_bench_header_spec_examples(lib):
    """swsearch/bench.hpp: GCUPS formula, measurement_error, CSV schema."""
    import subprocess
    out = subprocess.run([str(_cpp_build() / "bench_unit")], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bench_unit: ok" in out.stdout


def test_cli_usage_and_exit_codes(lib, tmp_path):
    """tools/swsearch_cli.cpp: validation before any file is opened, stats output, exit codes."""
    import subprocess
    cli = str(_cpp_build() / "swsearch")
    run = lambda *a: subprocess.run([cli, *a], capture_output=True, text=True)
    assert run("--help").returncode == 0 and run("--help").stdout.startswith("usage: swsearch")
    assert run("search").returncode == 2                                   # no db -> usage error
    assert run("search", "-d", "x.fa").returncode == 2                     # no query
    assert run("bench", "-d", "x.fa", "-q", "y.fa", "--repetitions", "abc").returncode == 2
    assert run("frobnicate", "-d", "x.fa").returncode == 2
    assert run("sweep", "-d", "x.fa", "-q", "y.fa").returncode == 2        # --values missing
    assert run("stats", "-d", str(tmp_path / "missing.fa")).returncode == 3
    fa = tmp_path / "db.fa"
    fa.write_text(">a first\nARNDARND\n>b\n\n>c\nWWWWWWWWWWWWWWWWWWW\n")
    out = run("stats", "-d", str(fa))
    assert out.returncode == 0 and out.stdout == "3 sequences, 27 residues, max 19\n"
    bad = tmp_path / "bad.fa"
    bad.write_text("ACGT\n")
    assert run("stats", "-d", str(bad)).returncode == 4                    # format error


def test_cli_pack_and_packed_stats_round_trip(lib, tmp_path):
    """`swsearch pack` writes the packed database on the host (no GPU); `stats --packed` reads sequences and headers
    back from it without any FASTA (include/swsearch/packed.hpp), and a write_fasta of the loaded copy would be the
    original: checked here through the stats line and through Python's reading of the file."""
    import subprocess
    cli = str(_cpp_build() / "swsearch")
    run = lambda *a: subprocess.run([cli, *a], capture_output=True, text=True)
    rng = np.random.default_rng(5)
    letters = lambda codes: "".join(synth.ALPHABET[c] for c in codes)
    seqs = [synth.random_residues(rng, int(n)) for n in [12, 0, 700, 3, 64, 65, 1] + list(rng.integers(1, 500, 90))]
    fa = tmp_path / "db.fa"
    fa.write_text("".join(f">s{i} some description\n{letters(s)}\n" for i, s in enumerate(seqs)))
    packed = tmp_path / "db.swb"
    out = run("pack", "-d", str(fa), "-o", str(packed), "--threshold", "300")
    assert out.returncode == 0 and out.stdout.startswith(f"packed {len(seqs)} sequences"), out.stderr
    assert run("stats", "--packed", str(packed)).stdout == run("stats", "-d", str(fa)).stdout
    assert run("stats", "--packed", str(packed), "-d", str(fa)).returncode == 2          # one source only
    assert run("pack", "-d", str(fa)).returncode == 2                                      # no output
    assert run("stats", "--packed", str(fa)).returncode == 4                               # a FASTA is not a packed file
    assert run("search", "--packed", str(packed), "-q", str(fa), "--threshold", "100").returncode in (1, 2)   # wrong threshold or no GPU
    # the file equals what the Python binding packs from the same sequences
    db = synth.from_sequences(seqs)
    other = tmp_path / "py.swb"
    search.pack_file(db.codes, db.offsets, other, length_threshold=300, names=[f"s{i} some description" for i in range(db.n)])
    assert other.read_bytes() == packed.read_bytes()




def _swissprot_lengths():
    rng = np.random.Generator(np.random.PCG64(0x5357_4442_02))
    return synth.random_lengths(rng, synth.SWISSPROT_SEQS, synth.SWISSPROT_RESIDUES, synth.SWISSPROT_MAXLEN)


def test_scan_plan_divides_every_group_exactly_once(lib):
    """The host-side division of a search between the two scan kernels (scan_plan.hpp, the GPU counterpart of
    make_chunks + the two worker pools, scheduler.hpp:130-138,200-213): every group is on exactly one side, the
    tall ones on the wavefront side, and its SM share follows its share of the rows."""
    lens = _swissprot_lengths()
    for m in (144, 257, 375, 1000, 2005, 5478):
        p = search.scan_plan(lens, m)
        assert p["pipeline_groups"] + p["wavefront_groups"] == p["n_groups"] == (len(lens) + 63) // 64
        assert p["pipeline_rows"] + p["wavefront_rows"] >= int(lens.sum()) // 64     # padded rows cover the residues
        assert p["n_tiles"] == (m + 31) // 32
        if True:                                      # (short queries too: the search is chain-bound)
            assert p["pipeline_groups"] > 0.99 * p["n_groups"]
            assert 0 < p["wavefront_groups"] < 64 and 1 <= p["wavefront_sms"] < 148
            share = p["wavefront_rows"] / (p["wavefront_rows"] + p["pipeline_rows"])
            margin = 2.0 if p["chain_bound"] else 1.25     # (1.6 close to chain-bound: not on a whole Swiss-Prot)
            assert p["wavefront_sms"] == int(np.ceil(share * margin * 148))
            assert p["wavefront_units"] >= p["wavefront_groups"]
    assert search.scan_plan(lens, 375)["chain_bound"] == 1 and search.scan_plan(lens, 2005)["chain_bound"] == 0
    assert search.scan_plan(lens, 1000)["ring_chunks"] == 4 and search.scan_plan(lens, 5478)["ring_chunks"] == 2


def test_scan_plan_narrow_forms(lib):
    """Narrow units (kernels.cuh): with link buffers of their own where the wavefront of narrow tiles is shallow against
    the tallest group (short queries) -- in 4-column tiles and CTAs of 4 warps for the most chain-bound searches (a 1/8
    shard, m = 144) -- and in the classic form through the border arrays for deep wavefronts (long queries)."""
    lens = _swissprot_lengths()
    whole = search.scan_plan(lens, 144)
    assert whole["chain_bound"] == 1 and whole["narrow_groups"] > 0 and whole["narrow_tile"] == 8
    assert whole["narrow_link_bytes"] > 0 and whole["wavefront_threads"] == 256
    # links: 256 B per row of every narrow group and tile boundary (18 tiles of 8 columns: 17 boundaries)
    assert whole["narrow_link_bytes"] % (256 * 17) == 0
    shard = search.scan_plan(lens, 144, shard_rank=0, shard_count=8)
    assert shard["narrow_tile"] == 4 and shard["wavefront_threads"] == 256 and shard["narrow_link_bytes"] > 0   # 4 + 4 helper warps
    assert shard["wavefront_units"] >= 36 * shard["narrow_groups"]                 # 36 tiles of 4 columns per narrow group
    assert 4 * shard["wavefront_sms"] >= min(shard["wavefront_units"], 4 * 74)     # a scheduler per unit, on at most half the SMs
    deep = search.scan_plan(lens, 3564, shard_rank=0, shard_count=8)
    assert deep["narrow_groups"] > 0 and deep["narrow_tile"] == 8 and deep["narrow_link_bytes"] == 0   # 446 tiles: classic form
    assert search.scan_plan(lens, 2005)["narrow_groups"] == 0 or search.scan_plan(lens, 2005)["narrow_link_bytes"] == 0


def test_scan_plan_policies_and_small_databases(lib):
    lens = _swissprot_lengths()
    forced = search.scan_plan(lens, 2005, policy=search.Database.SCAN_PIPELINE)
    assert forced["pipeline_groups"] == forced["n_groups"] and forced["wavefront_units"] == 0
    wave = search.scan_plan(lens, 2005, policy=search.Database.SCAN_WAVEFRONT)
    assert wave["pipeline_groups"] == 0 and wave["wavefront_sms"] == 148 and wave["wavefront_units"] >= wave["n_groups"]
    short = search.scan_plan(np.minimum(lens, 2999), 144)              # fewer than 9 tiles and no chain to break:
    assert short["chain_bound"] == 0 and short["pipeline_groups"] == 0 and short["wavefront_sms"] == 148   # wavefront kernel only
    small = search.scan_plan(lens[:10_000], 2005)                      # 157 groups < 2 per SM
    assert small["pipeline_groups"] == 0
    huge = search.scan_plan(lens, 9000)                                # the whole profile leaves no room for the rings:
    assert huge["ring_chunks"] == 4 and huge["pipeline_groups"] > 0        # per-warp tile slices, rings at full capacity
    edge = search.scan_plan(lens, 6000)                                    # whole profile (150 KB) + rings of 2 chunks
    assert edge["ring_chunks"] == 2 and edge["pipeline_groups"] > 0
    assert search.scan_plan(lens, 9000, policy=search.Database.SCAN_PIPELINE)["pipeline_groups"] == 8843
    shard = search.scan_plan(lens, 2005, shard_rank=3, shard_count=8)  # 1/8 of the database: still hybrid
    assert shard["n_groups"] in (1105, 1106) and shard["pipeline_groups"] > 0.9 * shard["n_groups"]
    empty = search.scan_plan(np.zeros(0, np.uint32), 100)
    assert empty["n_groups"] == 0
    with pytest.raises(ValueError, match="shard_rank"):
        search.scan_plan(lens, 100, shard_rank=2, shard_count=2)
    with pytest.raises(ValueError, match="scan policy"):
        search.scan_plan(lens, 100, policy=7)


def test_batch_plan_deals_queries_over_two_balanced_streams(lib):
    """swb_search_many's grouping of a batch (plan_batch in scan_plan.hpp, previewed by swb_batch_plan): the config-2
    sweep becomes one shared scan whose two streams differ by a few tiles; dissimilar pairs, empty queries, small
    databases and shards whose tallest group exceeds a CTA's fair share fall back to one search per query."""
    lens = _swissprot_lengths()
    scan, stream = search.batch_plan(lens, synth.QUERY_LENGTHS)
    assert (scan == 0).all() and set(stream.tolist()) == {0, 1}
    tiles = np.array([(m + 31) // 32 for m in synth.QUERY_LENGTHS])
    a, b = tiles[stream == 0].sum(), tiles[stream == 1].sum()
    assert a + b == tiles.sum() and abs(int(a) - int(b)) <= tiles.min()
    # many queries: several scans, each under the stream limit, every query placed exactly once
    many = [int(x) for x in np.random.default_rng(5).integers(100, 6000, size=80)]
    scan, stream = search.batch_plan(lens, many)
    assert (scan >= 0).all() and scan.max() >= 1
    for s in range(scan.max() + 1):
        for half in (0, 1):
            assert sum((m + 31) // 32 for m, sc, st in zip(many, scan, stream) if sc == s and st == half) <= 704 + 188
    # two queries of very different length do not share a scan; an empty query never does
    assert search.batch_plan(lens, [5000, 300])[0].tolist() == [-1, -1]
    assert search.batch_plan(lens, [5000, 4000, 0, 100])[0].tolist() == [0, 0, -1, 0]
    assert search.batch_plan(lens, [100, 120])[0].tolist() == [-1, -1]            # fewer than 9 tiles per stream
    # small database (fewer than two groups per SM): one search per query
    assert (search.batch_plan(lens[:10_000], synth.QUERY_LENGTHS)[0] == -1).all()
    # half / an eighth of the database: its 35,213-row group no longer fits a CTA's share as one item, so the scan
    # hands out single passes instead -- still one shared scan
    assert (search.batch_plan(lens, synth.QUERY_LENGTHS, shard_count=2)[0] == 0).all()
    assert (search.batch_plan(lens, synth.QUERY_LENGTHS, shard_count=8)[0] == 0).all()
    # ... which needs more than one pass (16 tiles): two 400-residue queries share a scan on the whole database only
    assert search.batch_plan(lens, [400, 410])[0].tolist() == [0, 0]
    assert search.batch_plan(lens, [400, 410], shard_count=8)[0].tolist() == [-1, -1]


def _bench(*argv, env=None):
    root = Path(__file__).resolve().parents[1]
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, str(root / "bench.py"), *argv], cwd=root, env=e, capture_output=True, text=True,
                          timeout=600)


def test_bench_reference_arm_prints_the_contract_line():
    """bench.py --impl reference: one JSON line on rank 0 with the native arm's metric/unit/config keys, the CPU
    baseline description and an e2e object equal to the line's own value; other ranks print nothing and exit 0."""
    out = _bench("--impl", "reference", "--scale", "0.002", "--steps", "1", "--warmup", "0")
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["metric"] == "GCUPS" and line["unit"] == "GCUPS"
    assert line["higher_is_better"] is True and line["vs_baseline"] is None and line["n_gpus"] == 1
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"] and line["cpu_baseline"]["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in line["config"] and "model" not in line["config"]
    other = _bench("--impl", "reference", "--gpus", "2", "--scale", "0.002", "--steps", "1", "--warmup", "0",
                   env={"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert other.returncode == 0 and other.stdout.strip() == ""


def test_bench_native_arm_refuses_to_run_without_a_gpu():
    """No CPU fallback: without a CUDA device the native arm exits non-zero and says why."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    out = _bench("--scale", "0.002", "--steps", "1", "--warmup", "0")
    assert out.returncode != 0 and out.stdout.strip() == ""
    assert "no CPU fallback" in out.stderr


def _packed_file(tmp_path, name="db.swb"):
    rng = np.random.default_rng(11)
    seqs = [synth.random_residues(rng, int(n)) for n in [0, 1, 5, 64, 200, 333, 90, 17, 0, 801] + list(rng.integers(2, 400, 150))]
    db = synth.from_sequences(seqs)
    path = tmp_path / name
    search.pack_file(db.codes, db.offsets, path, length_threshold=300, names=[f"seq{i} test" for i in range(db.n)])
    return path, db


def test_packed_file_layout_and_validation_on_the_host(lib, tmp_path):
    """swb_pack_file_flat writes the packed shard without a GPU; swb_db_load validates the file on the host before it
    asks for a device: a sound file gets as far as 'no CUDA device', every damaged one is SWB_ERR_INVALID."""
    import struct
    import torch
    path, db = _packed_file(tmp_path)
    raw = bytearray(path.read_bytes())
    magic, version, n_total, n_local, n_short, n_long, rank, count, max_len = struct.unpack_from("<8sIIIIIIII", raw, 0)
    residues, padded_rows, total_chunks, threshold, n_groups, codes_bytes, names_bytes = struct.unpack_from("<QQQQQQQ", raw, 40)
    assert magic == b"SWB200DB" and version == 2 and n_total == n_local == db.n and max_len == 801
    assert residues == db.residues and threshold == 300 and n_short + n_long == db.n and n_long == int((db.lengths() >= 300).sum())
    assert n_groups == (db.n + 63) // 64 and codes_bytes == total_chunks * 512
    assert len(raw) == 96 + n_groups * 16 + 2 * n_groups * 64 * 4 + codes_bytes + names_bytes
    off_groups, off_index = 96, 96 + n_groups * 16
    off_len, off_codes = off_index + n_groups * 64 * 4, off_index + 2 * n_groups * 64 * 4
    # the interleaved layout of pack.hpp: slot s of group g, row r -> codes[((chunk_base + r/8)*32 + s%32)*16 + (s/32)*8 + r%8]
    slot_index = np.frombuffer(raw, np.uint32, n_groups * 64, off_index)
    slot_len = np.frombuffer(raw, np.uint32, n_groups * 64, off_len)
    groups = np.frombuffer(raw, np.dtype([("base", "<u8"), ("chunks", "<u4"), ("first", "<u4")]), n_groups, off_groups)
    codes = np.frombuffer(raw, np.uint8, codes_bytes, off_codes)
    for slot in (0, 1, 37, 64, 100, db.n - 1):
        g, s = divmod(slot, 64)
        seq = db.seq(int(slot_index[slot]))
        assert len(seq) == slot_len[slot]
        r = np.arange(len(seq))
        got = codes[((int(groups[g]["base"]) + r // 8) * 32 + s % 32) * 16 + (s // 32) * 8 + r % 8]
        assert (got == seq).all()
    name_off = np.frombuffer(raw, np.uint64, n_total + 1, off_codes + codes_bytes)
    blob = bytes(raw[off_codes + codes_bytes + 8 * (n_total + 1):])
    assert names_bytes == 8 * (n_total + 1) + len(blob) and blob[int(name_off[7]):int(name_off[8])] == b"seq7 test"
    if not torch.cuda.is_available():
        with pytest.raises(search.SwbError, match="no CUDA device"):
            search.Database.load(path)

    def damaged(edit, why):
        bad = bytearray(raw)
        edit(bad)
        p = tmp_path / "bad.swb"
        p.write_bytes(bytes(bad))
        with pytest.raises(ValueError, match="not a valid swb200 packed database"):
            search.Database.load(p)

    damaged(lambda b: b.__setitem__(slice(0, 4), b"XXXX"), "magic")
    damaged(lambda b: struct.pack_into("<I", b, 8, 1), "version")
    damaged(lambda b: b.__delitem__(slice(len(b) - 512, len(b))), "truncated")
    damaged(lambda b: struct.pack_into("<Q", b, 72, 1 << 26), "n_groups beyond the file")
    damaged(lambda b: struct.pack_into("<I", b, 36, 100), "understated max_length (would skip the int32 re-run)")
    damaged(lambda b: struct.pack_into("<Q", b, 40, residues - 1), "residues")
    damaged(lambda b: struct.pack_into("<I", b, off_index + 4, struct.unpack_from("<I", b, off_index)[0]), "duplicate db_index")
    damaged(lambda b: struct.pack_into("<I", b, off_index, n_total + 5), "db_index beyond n_total")
    damaged(lambda b: struct.pack_into("<I", b, off_len, 100000), "slot_len beyond the group's rows")
    damaged(lambda b: struct.pack_into("<I", b, off_groups + 12, 64), "first_slot")
    damaged(lambda b: struct.pack_into("<I", b, off_groups + 16 + 8, 1 << 20), "group order / chunk continuity")
    damaged(lambda b: b.__setitem__(off_codes + 3, 77), "residue code beyond the alphabet")
    with pytest.raises(ValueError, match="cannot open"):
        search.Database.load(tmp_path / "missing.swb")
