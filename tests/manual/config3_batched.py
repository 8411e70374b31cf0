"""Config 3 (only the sequences >= 3000 residues) as one batch: shared scans with pass items against single searches."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2203_11100_b200 import synth, Database, GapModel, batch_plan
qs, sdb = synth.config2()
sub = sdb.subset(np.nonzero(sdb.lengths() >= 3000)[0])
batch = [qs[i] for i in range(13, 20)]
b62 = synth.blosum62()
g = GapModel(10, 2)
print("plan:", batch_plan(sub.lengths(), [len(q) for q in batch])[0].tolist())
cells = sum(len(q) for q in batch) * sub.residues
with Database(sub.codes, sub.offsets) as db:
    singles = [db.search(q, b62, g, 10) for q in batch]
    t_single = sum(db.search(q, b62, g, 10)[2]["ms_total"] for q in batch)
    db.search_many(batch, b62, g, 10)
    many, ms = db.search_many(batch, b62, g, 10)
    same = all((a[0] == b[0]).all() and (a[1] == b[1]).all() for a, b in zip(many, singles))
    print(f"config 3: {sub.n} sequences, {sub.residues/1e6:.1f} M residues; single {t_single:.1f} ms = {cells/t_single/1e6:.0f} GCUPS; "
          f"batched {ms.sum():.1f} ms = {cells/ms.sum()/1e6:.0f} GCUPS; identical lists: {same}")
