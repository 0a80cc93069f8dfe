"""The compiled reference (oracle/_ref/libfolp_ref.so) behind the folp_c.h
struct layouts -- test infrastructure only."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2106_04756_b200.cabi import LP, Binding

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libfolp_ref.so"

_ref = None


def available() -> bool:
    return REF_LIB.exists()


def binding() -> Binding:
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle`")
        lib = C.CDLL(str(REF_LIB))
        _ref = Binding(lib, "folp_ref_")
        lib.folp_ref_gen_pagerank.restype = C.c_void_p
        lib.folp_ref_gen_pagerank.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_double]
        lib.folp_ref_gen_random_feasible.restype = C.c_void_p
        lib.folp_ref_gen_random_feasible.argtypes = [C.c_uint64, C.c_int64, C.c_int64,
                                                     C.c_int64, C.c_double]
        lib.folp_ref_handcrafted_count.restype = C.c_int64
        lib.folp_ref_gen_handcrafted.restype = C.c_void_p
        lib.folp_ref_gen_handcrafted.argtypes = [C.c_int64, C.POINTER(C.c_double),
                                                 C.c_char_p, C.c_int64]
        lib.folp_ref_lp_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 4
        lib.folp_ref_lp_copy.argtypes = [C.c_void_p] + [C.c_void_p] * 7 + [
            C.POINTER(C.c_double)]
        lib.folp_ref_lp_free.argtypes = [C.c_void_p]
    return _ref


def _take(handle, name: str) -> LP:
    lib = binding().lib
    if not handle:
        raise ValueError(lib.folp_ref_last_error().decode())
    m, n, m1, nnz = (C.c_int64() for _ in range(4))
    lib.folp_ref_lp_sizes(handle, C.byref(m), C.byref(n), C.byref(m1), C.byref(nnz))
    m, n, m1, nnz = m.value, n.value, m1.value, nnz.value
    rs = np.zeros(m + 1, dtype=np.int64)
    rc = np.zeros(max(1, nnz), dtype=np.int64)
    rv = np.zeros(max(1, nnz))
    c, q, lo, hi = np.zeros(n), np.zeros(m), np.zeros(n), np.zeros(n)
    const = C.c_double()
    lib.folp_ref_lp_copy(handle, rs.ctypes.data, rc.ctypes.data, rv.ctypes.data, c.ctypes.data,
                         q.ctypes.data, lo.ctypes.data, hi.ctypes.data, C.byref(const))
    lib.folp_ref_lp_free(handle)
    return LP(m, n, m1, rs, rc[:nnz].copy(), rv[:nnz].copy(), c, q, lo, hi, const.value, name)


def pagerank(nodes: int, attach: int, seed: int, damping: float = 0.85) -> LP:
    """pagerank_lp(barabasi_albert(...)) -- instance_gen.cpp:57-144."""
    b = binding()
    return _take(b.lib.folp_ref_gen_pagerank(nodes, attach, seed, damping),
                 f"pagerank_n{nodes}_s{seed}")


def random_feasible(seed: int, m1: int, m2: int, n: int, spread: float) -> LP:
    """random_feasible_lp -- instance_gen.cpp:235-292."""
    b = binding()
    return _take(b.lib.folp_ref_gen_random_feasible(seed, m1, m2, n, spread),
                 f"random_feasible_{seed}")


def handcrafted() -> list[tuple[LP, float]]:
    """handcrafted_suite -- instance_gen.cpp:146-233: (lp, optimal objective)."""
    b = binding()
    out = []
    for i in range(b.lib.folp_ref_handcrafted_count()):
        obj = C.c_double()
        name = C.create_string_buffer(64)
        h = b.lib.folp_ref_gen_handcrafted(i, C.byref(obj), name, 64)
        out.append((_take(h, name.value.decode()), obj.value))
    return out
