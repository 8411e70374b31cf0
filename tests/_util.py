import json
from pathlib import Path

import numpy as np

from paper_2203_11100_b200 import synth

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_v1.json"


def golden():
    return json.loads(GOLDEN.read_text())


def enc(text):
    return synth.encode(text) if text else np.zeros(0, np.uint8)


def naive_rank(scores, top_k):
    """(score desc, index asc), truncated -- scheduler.hpp:111-115 stated directly."""
    scores = np.asarray(scores, dtype=np.int64)
    order = np.lexsort((np.arange(len(scores)), -scores))[:top_k]
    return order.astype(np.uint32), scores[order].astype(np.int32)
