"""The engine's device-side bounds checks (segdot.cuh FOLP_DCHECK: gather
indices inside the gathered vector, tile / part / SELL-group ranges inside
their buffers, reduction slots inside the partials) over the parity cases:
tree and ordered reductions on members of four config families, SELL-32
row groups, loopback row and column shards with the partitioned dual
epilogue.  The checked library (lib/libfolp_b200_checked.so) must run every
case without a trap and produce results bit-identical to the product
library's (the checks read, never write).  Stand-in for compute-sanitizer
memcheck, which is closed on this GPU pool."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu]

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2106_04756_b200" / "lib"


def _run(lib: Path) -> dict:
    env = dict(os.environ, FOLP_ENGINE_LIB=str(lib))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "checked_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_checked_library_runs_the_parity_cases_bit_identically():
    checked = LIB / "libfolp_b200_checked.so"
    if not checked.exists():
        pytest.skip("checked library not built")
    a = _run(checked)
    b = _run(LIB / "libfolp_b200.so")
    assert a == b
