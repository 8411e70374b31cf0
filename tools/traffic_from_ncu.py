"""profiles/traffic.json from ncu raw CSV pages (ncu -i x.ncu-rep --page raw --csv): DRAM bytes per launch of the
dominant kernel, stamped with the hash of the kernel sources so that bench.py can tell a stale capture.

usage: python tools/traffic_from_ncu.py <headline.csv> <kernel substring> "<what was launched>" <algorithmic bytes>
                                        [<name>=<other.csv>:<kernel substring>:<query_len> ...]"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2203_11100_b200.build import kernel_source_hash   # noqa: E402


def read(path, kernel):
    """-> dict of the longest launch of `kernel` in an ncu raw CSV: dram bytes read / written, duration."""
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    rows = list(csv.DictReader(lines))
    units = rows[0]
    best = None
    for r in rows[1:]:
        if kernel not in r.get("Kernel Name", ""):
            continue

        def val(col):
            v = float(r[col].replace(",", ""))
            u = units[col].lower()
            scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
                     "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1)
            return v * scale
        rec = {"dram_bytes_read": val("dram__bytes_read.sum"), "dram_bytes_write": val("dram__bytes_write.sum"),
               "duration_ms": val("gpu__time_duration.sum"), "kernel_name": r["Kernel Name"][:80]}
        rec["dram_bytes"] = rec["dram_bytes_read"] + rec["dram_bytes_write"]
        if best is None or rec["duration_ms"] > best["duration_ms"]:
            best = rec
    if best is None:
        raise SystemExit(f"no launch of {kernel} in {path}")
    return best


head = read(sys.argv[1], sys.argv[2])
out = {"kernel": sys.argv[2], "query_len": sys.argv[3], "source": f"{sys.argv[1]} (ncu --set full, one launch)", **head,
       "algorithmic_db_bytes": int(sys.argv[4]), "ratio_to_algorithmic": head["dram_bytes"] / float(sys.argv[4]),
       "algorithmic_def": "SURVEY 8(d): 1 byte per database residue per query x the queries this launch scores",
       "kernel_source_sha256": kernel_source_hash(), "other_kernels": {}}
for spec in sys.argv[5:]:
    name, rest = spec.split("=", 1)
    path, kernel, qlen = rest.split(":")
    out["other_kernels"][name] = {"query_len": qlen, "source": path, **read(path, kernel)}
(ROOT / "profiles" / "traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
