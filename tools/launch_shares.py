"""Per-kernel totals and shares from an `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_shares.py <launches.csv> "<header comment>" > shares.csv"""
import csv
import re
import sys
from collections import defaultdict

with open(sys.argv[1]) as f:
    lines = [ln for ln in f if not ln.startswith("==")]
tot, cnt = defaultdict(float), defaultdict(int)
for row in csv.DictReader(lines):
    name = re.sub(r"\(.*$", "", row["Kernel Name"]).strip()
    ns = float(row["Metric Value"].replace(",", ""))
    unit = row.get("Metric Unit", "ns")
    ms = ns * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1e-6)
    tot[name] += ms
    cnt[name] += 1
everything = sum(tot.values())
search = sum(v for k, v in tot.items() if "pipe_rate" not in k)
print(f"# {sys.argv[2]}")
print("# per-launch times are cold-cache and serialised (scan kernels that normally run side by side on two streams are timed one "
      "after the other): compare SHARES, not absolutes")
print("kernel,launches,total_ms,share_of_all,share_of_search_kernels")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k},{cnt[k]},{v:.3f},{v / everything:.5f},{(v / search if 'pipe_rate' not in k else 0):.5f}")
