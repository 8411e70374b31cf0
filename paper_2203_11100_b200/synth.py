"""Deterministic synthetic protein databases and queries.

Residues are i.i.d. over the 20 standard amino acids with Swiss-Prot background frequencies
(codes 0..19 in the order of the reference's alphabet "ARNDCQEGHILKMFPSTWYVBZX*",
alphabet.hpp:60), plus ~0.1 % ambiguity codes 20..22 (B/Z/X) so the whole 24-symbol table is
exercised.  Lengths are log-normal (sigma 0.63) clipped to [2, 35213], mixed with a 0.25 % heavy
tail log-uniform on [3000, 35213] so the intra-task path is populated; one sequence is forced to
35,213 residues (the Swiss-Prot 2021_04 maximum); a few zero-length and length-1
records are included; the order is shuffled.  For every query one exact copy and three mutated
copies (5 / 20 / 50 % substitutions plus a few indels) are planted so the top-k is non-trivial.

Everything is a pure function of (seed, shape parameters): numpy's PCG64 stream.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ALPHABET = "ARNDCQEGHILKMFPSTWYVBZX*"

# Swiss-Prot background composition, order ARNDCQEGHILKMFPSTWYV
_BACKGROUND = np.array([
    .0825, .0553, .0406, .0545, .0137, .0393, .0675, .0707, .0227, .0596,
    .0966, .0584, .0242, .0386, .0470, .0656, .0534, .0108, .0292, .0687], dtype=np.float64)

SWISSPROT_SEQS = 565_928
SWISSPROT_RESIDUES = 204_173_280
SWISSPROT_MAXLEN = 35_213
# Customary lengths of the 20 query accessions of PAPER.md:403
QUERY_LENGTHS = [144, 189, 222, 375, 464, 567, 657, 729, 850, 1000, 1500, 2005, 2504, 3005, 3564,
                 4061, 4548, 4743, 5147, 5478]

# BLOSUM50 (NCBI), order ARNDCQEGHILKMFPSTWYVBZX*; used by config 5 (the reference only builds in
# BLOSUM62, scoring.hpp:65; any other matrix enters as a table).
BLOSUM50_ROWS = """
 5 -2 -1 -2 -1 -1 -1  0 -2 -1 -2 -1 -1 -3 -1  1  0 -3 -2  0 -2 -1 -1 -5
-2  7 -1 -2 -4  1  0 -3  0 -4 -3  3 -2 -3 -3 -1 -1 -3 -1 -3 -1  0 -1 -5
-1 -1  7  2 -2  0  0  0  1 -3 -4  0 -2 -4 -2  1  0 -4 -2 -3  4  0 -1 -5
-2 -2  2  8 -4  0  2 -1 -1 -4 -4 -1 -4 -5 -1  0 -1 -5 -3 -4  5  1 -1 -5
-1 -4 -2 -4 13 -3 -3 -3 -3 -2 -2 -3 -2 -2 -4 -1 -1 -5 -3 -1 -3 -3 -2 -5
-1  1  0  0 -3  7  2 -2  1 -3 -2  2  0 -4 -1  0 -1 -1 -1 -3  0  4 -1 -5
-1  0  0  2 -3  2  6 -3  0 -4 -3  1 -2 -3 -1 -1 -1 -3 -2 -3  1  5 -1 -5
 0 -3  0 -1 -3 -2 -3  8 -2 -4 -4 -2 -3 -4 -2  0 -2 -3 -3 -4 -1 -2 -2 -5
-2  0  1 -1 -3  1  0 -2 10 -4 -3  0 -1 -1 -2 -1 -2 -3  2 -4  0  0 -1 -5
-1 -4 -3 -4 -2 -3 -4 -4 -4  5  2 -3  2  0 -3 -3 -1 -3 -1  4 -4 -3 -1 -5
-2 -3 -4 -4 -2 -2 -3 -4 -3  2  5 -3  3  1 -4 -3 -1 -2 -1  1 -4 -3 -1 -5
-1  3  0 -1 -3  2  1 -2  0 -3 -3  6 -2 -4 -1  0 -1 -3 -2 -3  0  1 -1 -5
-1 -2 -2 -4 -2  0 -2 -3 -1  2  3 -2  7  0 -3 -2 -1 -1  0  1 -3 -1 -1 -5
-3 -3 -4 -5 -2 -4 -3 -4 -1  0  1 -4  0  8 -4 -3 -2  1  4 -1 -4 -4 -2 -5
-1 -3 -2 -1 -4 -1 -1 -2 -2 -3 -4 -1 -3 -4 10 -1 -1 -4 -3 -3 -2 -1 -2 -5
 1 -1  1  0 -1  0 -1  0 -1 -3 -3  0 -2 -3 -1  5  2 -4 -2 -2  0  0 -1 -5
 0 -1  0 -1 -1 -1 -1 -2 -2 -1 -1 -1 -1 -2 -1  2  5 -3 -2  0  0 -1  0 -5
-3 -3 -4 -5 -5 -1 -3 -3 -3 -3 -2 -3 -1  1 -4 -4 -3 15  2 -3 -5 -2 -3 -5
-2 -1 -2 -3 -3 -1 -2 -3  2 -1 -1 -2  0  4 -3 -2 -2  2  8 -1 -3 -2 -1 -5
 0 -3 -3 -4 -1 -3 -3 -4 -4  4  1 -3  1 -1 -3 -2  0 -3 -1  5 -4 -3 -1 -5
-2 -1  4  5 -3  0  1 -1  0 -4 -4  0 -3 -4 -2  0  0 -5 -3 -4  5  2 -1 -5
-1  0  0  1 -3  4  5 -2  0 -3 -3  1 -1 -4 -1  0 -1 -2 -2 -3  2  5 -1 -5
-1 -1 -1 -1 -2 -1 -1 -2 -1 -1 -1 -1 -1 -2 -2 -1  0 -3 -1 -1 -1 -1 -1 -5
-5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5 -5  1
"""


def blosum50() -> np.ndarray:
    m = np.array(BLOSUM50_ROWS.split(), dtype=np.int32).reshape(24, 24)
    assert (m == m.T).all()
    return m


# BLOSUM62 in the same order.  The values are the published NCBI table; tests/test_oracle.py
# asserts equality with the reference's built-in copy (scoring.hpp:69-92) through oracle/_ref.
BLOSUM62_ROWS = """
 4 -1 -2 -2  0 -1 -1  0 -2 -1 -1 -1 -1 -2 -1  1  0 -3 -2  0 -2 -1  0 -4
-1  5  0 -2 -3  1  0 -2  0 -3 -2  2 -1 -3 -2 -1 -1 -3 -2 -3 -1  0 -1 -4
-2  0  6  1 -3  0  0  0  1 -3 -3  0 -2 -3 -2  1  0 -4 -2 -3  3  0 -1 -4
-2 -2  1  6 -3  0  2 -1 -1 -3 -4 -1 -3 -3 -1  0 -1 -4 -3 -3  4  1 -1 -4
 0 -3 -3 -3  9 -3 -4 -3 -3 -1 -1 -3 -1 -2 -3 -1 -1 -2 -2 -1 -3 -3 -2 -4
-1  1  0  0 -3  5  2 -2  0 -3 -2  1  0 -3 -1  0 -1 -2 -1 -2  0  3 -1 -4
-1  0  0  2 -4  2  5 -2  0 -3 -3  1 -2 -3 -1  0 -1 -3 -2 -2  1  4 -1 -4
 0 -2  0 -1 -3 -2 -2  6 -2 -4 -4 -2 -3 -3 -2  0 -2 -2 -3 -3 -1 -2 -1 -4
-2  0  1 -1 -3  0  0 -2  8 -3 -3 -1 -2 -1 -2 -1 -2 -2  2 -3  0  0 -1 -4
-1 -3 -3 -3 -1 -3 -3 -4 -3  4  2 -3  1  0 -3 -2 -1 -3 -1  3 -3 -3 -1 -4
-1 -2 -3 -4 -1 -2 -3 -4 -3  2  4 -2  2  0 -3 -2 -1 -2 -1  1 -4 -3 -1 -4
-1  2  0 -1 -3  1  1 -2 -1 -3 -2  5 -1 -3 -1  0 -1 -3 -2 -2  0  1 -1 -4
-1 -1 -2 -3 -1  0 -2 -3 -2  1  2 -1  5  0 -2 -1 -1 -1 -1  1 -3 -1 -1 -4
-2 -3 -3 -3 -2 -3 -3 -3 -1  0  0 -3  0  6 -4 -2 -2  1  3 -1 -3 -3 -1 -4
-1 -2 -2 -1 -3 -1 -1 -2 -2 -3 -3 -1 -2 -4  7 -1 -1 -4 -3 -2 -2 -1 -2 -4
 1 -1  1  0 -1  0  0  0 -1 -2 -2  0 -1 -2 -1  4  1 -3 -2 -2  0  0  0 -4
 0 -1  0 -1 -1 -1 -1 -2 -2 -1 -1 -1 -1 -2 -1  1  5 -2 -2  0 -1 -1  0 -4
-3 -3 -4 -4 -2 -2 -3 -2 -2 -3 -2 -3 -1  1 -4 -3 -2 11  2 -3 -4 -3 -2 -4
-2 -2 -2 -3 -2 -1 -2 -3  2 -1 -1 -2 -1  3 -3 -2 -2  2  7 -1 -3 -2 -1 -4
 0 -3 -3 -3 -1 -2 -2 -3 -3  3  1 -2  1 -1 -2 -2  0 -3 -1  4 -3 -2 -1 -4
-2 -1  3  4 -3  0  1 -1  0 -3 -4  0 -3 -3 -2  0 -1 -4 -3 -3  4  1 -1 -4
-1  0  0  1 -3  3  4 -2  0 -3 -3  1 -1 -3 -1  0 -1 -3 -2 -2  1  4 -1 -4
 0 -1 -1 -1 -2 -1 -1 -1 -1 -1 -1 -1 -1 -1 -2  0  0 -2 -1 -1 -1 -1 -1 -4
-4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4 -4  1
"""


def blosum62() -> np.ndarray:
    m = np.array(BLOSUM62_ROWS.split(), dtype=np.int32).reshape(24, 24)
    assert (m == m.T).all()
    return m


def encode(text: str) -> np.ndarray:
    """Residue letters -> codes, unknown -> X (alphabet.hpp:28-31, 60)."""
    lut = np.full(256, ALPHABET.index("X"), dtype=np.uint8)
    for i, ch in enumerate(ALPHABET):
        lut[ord(ch)] = i
        lut[ord(ch.lower())] = i
    return lut[np.frombuffer(text.encode("ascii"), dtype=np.uint8)]


def _residue_lut() -> np.ndarray:
    """65536-entry table mapping a uniform uint16 to a residue code with the target composition."""
    p = _BACKGROUND / _BACKGROUND.sum() * 0.999
    p = np.concatenate([p, np.full(3, 0.001 / 3)])      # B, Z, X
    edges = np.floor(np.cumsum(p) * 65536 + 0.5).astype(np.int64)
    edges[-1] = 65536
    lut = np.zeros(65536, dtype=np.uint8)
    start = 0
    for code, end in enumerate(edges):
        lut[start:end] = code
        start = end
    return lut


_LUT = None


def random_residues(rng: np.random.Generator, n: int) -> np.ndarray:
    global _LUT
    if _LUT is None:
        _LUT = _residue_lut()
    out = np.empty(n, dtype=np.uint8)
    step = 1 << 24
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        out[lo:hi] = _LUT[rng.integers(0, 65536, size=hi - lo, dtype=np.uint16)]
    return out


def random_lengths(rng: np.random.Generator, n_seqs: int, target_residues: int | None, max_len: int,
                   tail_fraction: float = 0.0025, tail_lo: int = 3000, sigma: float = 0.63) -> np.ndarray:
    n_tail = int(round(n_seqs * tail_fraction)) if max_len > tail_lo else 0
    n_body = n_seqs - n_tail
    tail = np.exp(rng.uniform(np.log(tail_lo), np.log(max_len), size=n_tail)).astype(np.int64) if n_tail else np.zeros(0, np.int64)
    if target_residues is None:
        median = 295.0
    else:
        body_mean = max(20.0, (target_residues - tail.sum()) / max(n_body, 1))
        median = body_mean / np.exp(sigma * sigma / 2)
    body = np.exp(rng.normal(np.log(median), sigma, size=n_body))
    body = np.clip(np.rint(body), 2, max_len).astype(np.int64)
    lens = np.concatenate([body, tail])
    rng.shuffle(lens)
    # edge-case records: zero-length, length 1, and the forced maximum
    if n_seqs >= 16:
        lens[1] = 0
        lens[n_seqs // 3] = 0
        lens[2] = 1
        lens[n_seqs // 2] = 1
    if n_seqs >= 4 and max_len > tail_lo:
        lens[n_seqs // 5] = max_len
    return lens


def mutate(rng: np.random.Generator, seq: np.ndarray, sub_rate: float, n_indels: int) -> np.ndarray:
    out = seq.copy()
    if len(out) == 0:
        return out
    n_sub = int(round(len(out) * sub_rate))
    if n_sub:
        pos = rng.choice(len(out), size=n_sub, replace=False)
        out[pos] = random_residues(rng, n_sub)
    for _ in range(n_indels):
        if len(out) < 8:
            break
        at = int(rng.integers(1, len(out) - 1))
        size = int(rng.integers(1, 6))
        if rng.random() < 0.5:
            out = np.concatenate([out[:at], random_residues(rng, size), out[at:]])
        else:
            out = np.concatenate([out[:at], out[at + size:]])
    return out


@dataclass
class SyntheticDb:
    codes: np.ndarray                 # uint8, concatenated
    offsets: np.ndarray               # uint64, n+1
    planted: dict = field(default_factory=dict)   # query number -> list of db indices (exact first)

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def residues(self) -> int:
        return int(self.offsets[-1])

    def seq(self, i: int) -> np.ndarray:
        return self.codes[int(self.offsets[i]):int(self.offsets[i + 1])]

    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets.astype(np.int64))

    def subset(self, indices) -> "SyntheticDb":
        seqs = [self.seq(int(i)) for i in indices]
        return from_sequences(seqs)


def from_sequences(seqs) -> SyntheticDb:
    lens = np.array([len(s) for s in seqs], dtype=np.uint64)
    offsets = np.zeros(len(seqs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offsets[1:])
    codes = np.concatenate([np.asarray(s, dtype=np.uint8) for s in seqs]) if len(seqs) and offsets[-1] else np.zeros(0, np.uint8)
    return SyntheticDb(np.ascontiguousarray(codes), offsets)


def make_queries(lengths=QUERY_LENGTHS, seed: int = 0x5357_4442_00) -> list[np.ndarray]:
    rng = np.random.Generator(np.random.PCG64(seed ^ 0xA11CE))
    return [random_residues(rng, int(n)) for n in lengths]


def make_database(n_seqs: int, target_residues: int | None = None, max_len: int = SWISSPROT_MAXLEN,
                  queries: list[np.ndarray] | None = None, seed: int = 0x5357_4442_00,
                  tail_fraction: float = 0.0025) -> SyntheticDb:
    rng = np.random.Generator(np.random.PCG64(seed))
    lens = random_lengths(rng, n_seqs, target_residues, max_len, tail_fraction=tail_fraction)

    # planted homologs replace randomly chosen ordinary records (never the edge-case ones)
    planted: dict[int, list[int]] = {}
    replacements: dict[int, np.ndarray] = {}
    if queries:
        protected = {1, 2, n_seqs // 3, n_seqs // 2, n_seqs // 5}
        candidates = [int(i) for i in rng.permutation(n_seqs) if int(i) not in protected]
        cursor = 0
        for qi, q in enumerate(queries):
            planted[qi] = []
            variants = [q.copy(), mutate(rng, q, 0.05, 2), mutate(rng, q, 0.20, 3), mutate(rng, q, 0.50, 4)]
            for v in variants:
                if cursor >= len(candidates):
                    break
                idx = candidates[cursor]
                cursor += 1
                replacements[idx] = v
                lens[idx] = len(v)
                planted[qi].append(idx)

    offsets = np.zeros(n_seqs + 1, dtype=np.uint64)
    np.cumsum(lens.astype(np.uint64), out=offsets[1:])
    codes = random_residues(rng, int(offsets[-1]))
    for idx, v in replacements.items():
        codes[int(offsets[idx]):int(offsets[idx + 1])] = v
    return SyntheticDb(codes, offsets, planted)


def config1(seed: int = 0x5357_4442_01):
    """BASELINE config 1: one 144-residue query vs 10,000 sequences."""
    queries = make_queries([144], seed)
    db = make_database(10_000, target_residues=3_600_000, queries=queries, seed=seed)
    return queries, db


def config2(seed: int = 0x5357_4442_02, scale: float = 1.0):
    """BASELINE config 2: 20-query sweep vs a Swiss-Prot-shaped database (scale < 1 shrinks it)."""
    queries = make_queries(QUERY_LENGTHS, seed)
    n = max(64, int(SWISSPROT_SEQS * scale))
    db = make_database(n, target_residues=int(SWISSPROT_RESIDUES * scale), queries=queries, seed=seed)
    return queries, db


def config3(seed: int = 0x5357_4442_02):
    """BASELINE config 3: the long-sequence (intra-task) pool -- the config-2 queries of 3,005 residues and more
    against only the config-2 database entries of 3,000 residues and more (SearchConfig::length_threshold's default,
    scheduler.hpp:24).  -> (queries, database, query numbers in config 2)."""
    queries, db = config2(seed)
    keep = np.nonzero(db.lengths() >= 3000)[0]
    sub = db.subset(keep)
    where = {int(old): new for new, old in enumerate(keep)}
    qids = [i for i, q in enumerate(queries) if len(q) >= 3005]
    sub.planted = {k: [where[i] for i in db.planted[qi] if i in where] for k, qi in enumerate(qids)}
    return [queries[i] for i in qids], sub, qids


CONFIG5_SEQS = 2_800_000
CONFIG5_RESIDUES = 1_000_000_000
CONFIG5_QUERY_LENGTHS = [144, 1000, 3005, 5147, 5478, 8000, 9000]


def config5_share(shards: int = 8, seed: int = 0x5357_4442_05):
    """BASELINE config 5, one GPU's share: a TrEMBL-shaped database (2.8 M sequences / 1.0 G residues, same length
    model) is dealt over `shards` GPUs by residue count; one share is a database of 1/shards of the sequences and
    residues with the same length distribution, generated directly at that size.  BLOSUM50, gap 12/2; the queries
    include two beyond the reference's 5,478 so that planted copies leave the int16 range and the int32 re-run is
    exercised.  -> (queries, database)."""
    queries = make_queries(CONFIG5_QUERY_LENGTHS, seed)
    db = make_database(CONFIG5_SEQS // shards, target_residues=CONFIG5_RESIDUES // shards, queries=queries, seed=seed)
    return queries, db
