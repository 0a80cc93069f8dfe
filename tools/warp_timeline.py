"""Per-warp timeline of the loop products (diagnostic build):
    make -C paper_2106_04756_b200 variant NAME=wt DEFS=-DFOLP_WARP_TIMES
    FOLP_ENGINE_LIB=$PWD/variants/libfolp_wt.so FOLP_NO_GRAPH=1 python tools/warp_timeline.py
Runs a few evaluation periods of a config, then prints, for the last kernel
A (K'y + primal step) and B (K x' + dual step) launch, the distribution of
warp start / units-done / exit times relative to the first warp start, and
per-SM-slot (CTA) finish spread."""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_04756_b200 import cabi, engine, instances  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    lp = instances.generate(a.config, 1, a.scale)
    eng = engine()
    s = eng.session(lp, cabi.params())
    s.advance(3)
    lib = eng.lib
    lib.folp_gpu_debug_warp_times.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.c_int32]
    # the session's context: folp_session -> SolveSession; use the C getter
    lib.folp_session_context.restype = C.c_void_p
    ctx = lib.folp_session_context(s.h)
    W = 16384
    for slot, name in [(0, "A (K'y, primal)"), (1, "B (K x', dual)")]:
        buf = np.zeros(W * 3 + 3, dtype=np.uint64)
        rc = lib.folp_gpu_debug_warp_times(ctx, slot, buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           W + 1)
        tail = buf[3 * W:].astype(np.int64)
        buf = buf[:3 * W]
        if rc != 0:
            print("debug_warp_times failed", rc)
            return
        t = buf.reshape(W, 3).astype(np.int64)
        used = t[:, 0] > 0
        t = t[used]
        t0 = t[:, 0].min()
        st, ud, ex = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
        q = [0, 10, 50, 90, 99, 100]
        print(f"== {name}: {used.sum()} warps, kernel span {ex.max():.2f} us")
        for lab, v in [("start", st), ("units done", ud), ("exit", ex), ("unit time", ud - st),
                       ("tail wait", ex - ud)]:
            print(f"  {lab:10s} " + "  ".join(f"p{p}={np.percentile(v, p):7.2f}" for p in q))
        busy = (ud - st).sum() / (len(st) * ex.max())
        tl = (tail - t0) / 1e3
        print(f"  last CTA: ticket {tl[0]:.2f}  sums {tl[1]:.2f}  finalize {tl[2]:.2f} us")
        print(f"  warp-busy fraction of (warps x span): {busy:.3f}")
    s.close()


if __name__ == "__main__":
    main()
