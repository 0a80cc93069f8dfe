"""B200-native PDLP solve path (arXiv 2106.04756) behind folp's interface.

Python access to the in-tree engine ``lib/libfolp_b200.so`` through its C ABI
(include/folp_c.h).  There is no CPU fallback: importing the engine without
the built library, or calling it on a machine without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .cabi import LP, Binding, FolpError, SolveResult, params  # noqa: F401

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
ENGINE_LIB = Path(os.environ.get("FOLP_ENGINE_LIB", LIB_DIR / "libfolp_b200.so"))  # A/B builds
GEN_LIB = LIB_DIR / "libfolp_gen.so"

_engine = None


def build(verbose: bool = False) -> None:
    """Compile the engine (sm_100a) and the generators in-tree."""
    import subprocess

    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-C", str(PKG_DIR), "-j", jobs], check=True, stdout=out)


def engine() -> Binding:
    """The folp_c.h binding of the B200 engine (loads the .so once)."""
    global _engine
    if _engine is None:
        if not ENGINE_LIB.exists():
            raise FileNotFoundError(
                f"{ENGINE_LIB} is missing: run paper_2106_04756_b200.build() (no CPU fallback)")
        _engine = Binding(ctypes.CDLL(str(ENGINE_LIB)), "folp_")
    return _engine


def solve(lp: LP, p: dict | None = None, x0=None, y0=None, **kw) -> SolveResult:
    """folp::solve on the B200 (solver.hpp:226-228)."""
    return engine().solve_lp(lp, p, x0, y0, **kw)
