"""Seeded instances of the five BASELINE.json configurations.

Thin wrapper over ``lib/libfolp_gen.so`` (include/folp_gen.h): the same
generated LP is handed to the B200 engine and to the CPU reference.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import GEN_LIB
from .cabi import LP

CONFIG_NAMES = {
    1: "cfg1_small_random_m1k_n2k",
    2: "cfg2_medium_powerlaw_m200k_n400k",
    3: "cfg3_pagerank_N2M",
    4: "cfg4_large_random_m20M_n40M",
    5: "cfg5_transportation_S2000_D8000",
}


class GenLP(C.Structure):
    _fields_ = [("num_rows", C.c_int64), ("num_cols", C.c_int64),
                ("num_inequality_rows", C.c_int64), ("nnz", C.c_int64)] + [
        (name, C.POINTER(C.c_int64 if name in ("row_start", "row_cols", "col_start", "col_rows")
                         else C.c_double))
        for name in ("row_start", "row_cols", "row_values", "col_start", "col_rows",
                     "col_values", "objective", "right_hand_side", "variable_lower",
                     "variable_upper")] + [
        ("objective_constant", C.c_double), ("max_row_len", C.c_int64),
        ("max_col_len", C.c_int64)]


_gen = None


def _lib():
    global _gen
    if _gen is None:
        if not GEN_LIB.exists():
            raise FileNotFoundError(f"{GEN_LIB} is missing: run paper_2106_04756_b200.build()")
        _gen = C.CDLL(str(GEN_LIB))
        _gen.folp_gen_config.restype = C.POINTER(GenLP)
        _gen.folp_gen_config.argtypes = [C.c_int32, C.c_uint64, C.c_double]
        _gen.folp_gen_free.argtypes = [C.POINTER(GenLP)]
        _gen.folp_gen_last_error.restype = C.c_char_p
    return _gen


def _arr(ptr, count, dtype):
    if count == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)


def generate(cfg: int, seed: int = 1, scale: float = 1.0, with_csc: bool = False) -> LP:
    """LP of configuration ``cfg`` (1..5); ``scale`` < 1 gives a smaller member
    of the same family (tests)."""
    lib = _lib()
    h = lib.folp_gen_config(cfg, seed, scale)
    if not h:
        raise ValueError(lib.folp_gen_last_error().decode())
    try:
        g = h.contents
        m, n, nnz = g.num_rows, g.num_cols, g.nnz
        lp = LP(num_rows=m, num_cols=n, num_inequality_rows=g.num_inequality_rows,
                row_start=_arr(g.row_start, m + 1, np.int64),
                row_cols=_arr(g.row_cols, nnz, np.int64),
                row_values=_arr(g.row_values, nnz, np.float64),
                objective=_arr(g.objective, n, np.float64),
                right_hand_side=_arr(g.right_hand_side, m, np.float64),
                variable_lower=_arr(g.variable_lower, n, np.float64),
                variable_upper=_arr(g.variable_upper, n, np.float64),
                objective_constant=g.objective_constant,
                name=f"{CONFIG_NAMES[cfg]}@seed{seed}x{scale:g}")
        lp.max_row_len = g.max_row_len
        lp.max_col_len = g.max_col_len
        if with_csc:
            lp.col_start = _arr(g.col_start, n + 1, np.int64)
            lp.col_rows = _arr(g.col_rows, nnz, np.int64)
            lp.col_values = _arr(g.col_values, nnz, np.float64)
        return lp
    finally:
        lib.folp_gen_free(h)
