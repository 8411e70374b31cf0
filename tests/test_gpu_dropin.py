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
