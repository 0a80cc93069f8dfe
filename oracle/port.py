"""The C restatement of the reference PDLP path (oracle/pdlp_port.c) behind
the folp_c.h struct layouts -- test infrastructure only."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

from paper_2106_04756_b200.cabi import Binding

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "lib" / "libfolp_port.so"

_port = None


def binding() -> Binding:
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            subprocess.run(["make", "-C", str(HERE), "port"], check=True,
                           stdout=subprocess.DEVNULL)
        _port = Binding(C.CDLL(str(PORT_LIB)), "folp_port_")
    return _port


def solve(lp, p=None, x0=None, y0=None, **kw):
    return binding().solve_lp(lp, p, x0, y0, **kw)
