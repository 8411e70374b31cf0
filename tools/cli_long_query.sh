#!/bin/bash
# end-to-end timing of the C++ drop-in (run_search incl. traceback of the top hits) through the CLI on a long query
python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2203_11100_b200 import synth
qs, sdb = synth.config2(scale=0.2)
L = lambda c: "".join(synth.ALPHABET[x] for x in c)
open("/tmp/q.fa", "w").write("".join(f">q{len(q)}\n{L(q)}\n" for q in (qs[9], qs[19])))
with open("/tmp/db.fa", "w") as f:
    for i in range(sdb.n):
        f.write(f">s{i}\n{L(sdb.seq(i))}\n")
print("wrote", sdb.n, "sequences")
PY
time ./tests/cpp/_build/swsearch search -q /tmp/q.fa -d /tmp/db.fa --top-k 10 | grep -E "^query|^  [0-9]" | cut -c1-100
time ./tests/cpp/_build/swsearch search -q /tmp/q.fa -d /tmp/db.fa --top-k 10 --no-align | grep -E "^query"
./tests/cpp/_build/swsearch bench -q /tmp/q.fa -d /tmp/db.fa --repetitions 5
