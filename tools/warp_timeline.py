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
        buf = np.zeros(W * 4 + 3, dtype=np.uint64)
        rc = lib.folp_gpu_debug_warp_times(ctx, slot, buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           W + 1)
        tail = buf[4 * W:].astype(np.int64)
        buf = buf[:4 * W]
        if rc != 0:
            print("debug_warp_times failed", rc)
            return
        t = buf.reshape(W, 4).astype(np.int64)
        used = t[:, 0] > 0
        t = t[used]
        work = t[:, 3].astype(np.uint64)
        nnz = (work & np.uint64(0xffffff)).astype(np.int64)
        parts = ((work >> np.uint64(24)) & np.uint64(0xfff)).astype(np.int64)
        segs = ((work >> np.uint64(36)) & np.uint64(0xffff)).astype(np.int64)
        smid = (work >> np.uint64(52)).astype(np.int64)
        t0 = t[:, 0].min()
        st, ud, ex = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
        q = [0, 10, 50, 90, 99, 100]
        print(f"== {name}: {used.sum()} warps, kernel span {ex.max():.2f} us")
        for lab, v in [("start", st), ("units done", ud), ("exit", ex), ("unit time", ud - st),
                       ("tail wait", ex - ud)]:
            print(f"  {lab:10s} " + "  ".join(f"p{p}={np.percentile(v, p):7.2f}" for p in q))
        busy = (ud - st).sum() / (len(st) * ex.max())
        tl = (tail - t0) / 1e3
        ut = ud - st
        order = np.argsort(ut)
        for lab, sel in [("fastest 10%", order[:len(ut) // 10]), ("median 10%", order[len(ut) * 45 // 100:len(ut) * 55 // 100]),
                         ("slowest 10%", order[-len(ut) // 10:]), ("slowest 1%", order[-len(ut) // 100:])]:
            print(f"  {lab:12s} unit time {ut[sel].mean():6.2f} us  nnz {nnz[sel].mean():7.0f}  parts {parts[sel].mean():5.2f}  segments {segs[sel].mean():6.1f}")
        print(f"  corr(unit time, nnz) {np.corrcoef(ut, nnz)[0, 1]:.2f}  corr(unit time, parts) {np.corrcoef(ut, parts)[0, 1] if parts.std() > 0 else 0:.2f}  corr(unit time, segments) {np.corrcoef(ut, segs)[0, 1]:.2f}")
        # SM-level: CTAs of one SM are b, b+148, ... under a persistent grid
        sms = np.unique(smid)
        sm_done = np.array([ud[smid == q].max() for q in sms])
        sm_nnz = np.array([nnz[smid == q].sum() for q in sms])
        sm_mean = np.array([ut[smid == q].mean() for q in sms])
        print(f"  per SM ({len(sms)}): last unit done p0 {sm_done.min():.2f} p50 {np.median(sm_done):.2f} "
              f"p100 {sm_done.max():.2f}; mean warp unit time p0 {sm_mean.min():.2f} p50 {np.median(sm_mean):.2f} "
              f"p100 {sm_mean.max():.2f}; nnz p0 {sm_nnz.min()} p100 {sm_nnz.max()}")
        slow = np.argsort(sm_mean)
        print(f"  slowest SMs {list(sms[slow[-6:]])} fastest {list(sms[slow[:6]])}")
        print(f"  last CTA: ticket {tl[0]:.2f}  sums {tl[1]:.2f}  finalize {tl[2]:.2f} us")
        print(f"  warp-busy fraction of (warps x span): {busy:.3f}")
    s.close()


if __name__ == "__main__":
    main()
