"""Bounded stress of the cross-CTA hand-offs (pass items of the two-stream kernel; tile and row-block units of the
wavefront kernel): fresh process, device memory pre-filled with a byte pattern, the batched sweep as the very first GPU
work on each shard, then repetitions mixed with single searches -- every ranked list compared with the single searches'.
(racecheck cannot see flag protocols; DESIGN.md section 5.7 has the ordering argument, this is the empirical side.)"""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("pattern", ["0xFF", "0x00"])
def test_pass_items_fresh_process_dirty_memory(lib, pattern):
    cmd = [sys.executable, str(ROOT / "tests" / "manual" / "pass_items_stress.py"), "5", "--dirty", pattern, "--batch-first",
           "--shards", "4:1,8:5"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    sys.stdout.write(res.stdout[-3000:])
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "mismatches: 0" in res.stdout
