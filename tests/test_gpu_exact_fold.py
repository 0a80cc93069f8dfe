"""The exact parallel fold (engine exactfold.cuh) against the sequential fold
it must reproduce bit for bit: s = init; for t in terms: s = fl(s + t)
(the reference's reductions, linalg.hpp:25-61, solver.cpp:76-88).

The sequential reference is numpy's add.accumulate (a plain left-to-right
loop; checked against a Python loop below).  Inputs are adversarial for the
algorithm: cancellation through zero, sums crossing many binades, exact ties
at the rounding point, zeros, subnormals, huge dynamic ranges, a dependent
fold (movement = fold(dy^2)/omega then fold of omega*dx^2, solver.cpp:81-88),
non-finite terms and overflow (which must take the plain sequential path)."""
import ctypes as C

import numpy as np
import pytest

from paper_2106_04756_b200 import engine

pytestmark = pytest.mark.gpu


def seq(t, init=0.0):
    if len(t) == 0:
        return float(init)
    with np.errstate(all="ignore"):
        return float(np.add.accumulate(np.concatenate([[init], np.asarray(t, dtype=np.float64)]))[-1])


def gpu_fold(eng, arrays, inits=None, init_from=None, init_div=None, grid=0, reps=0):
    lib = eng.lib
    f = lib.folp_gpu_test_exact_fold
    f.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                  C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int32,
                  C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    J = len(arrays)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in arrays]
    ptrs = (C.c_void_p * J)(*[a.ctypes.data for a in arrs])
    counts = (C.c_int64 * J)(*[len(a) for a in arrs])
    ini = (C.c_double * J)(*(inits or [0.0] * J))
    frm = (C.c_int32 * J)(*(init_from or [-1] * J))
    div = (C.c_double * J)(*(init_div or [1.0] * J))
    res = (C.c_double * J)()
    ms = C.c_double(0.0)
    rc = f(0, J, ptrs, counts, ini, frm, div, grid, reps, res, C.byref(ms))
    assert rc == 0, eng.lib.folp_gpu_last_error()
    return [float(res[j]) for j in range(J)], ms.value


def same(a, b):
    return (np.isnan(a) and np.isnan(b)) or np.float64(a).tobytes() == np.float64(b).tobytes()


def cases():
    rng = np.random.default_rng(2024)
    out = []
    out.append(("empty", np.zeros(0), 1.5))
    out.append(("single", np.array([3.25]), 0.0))
    out.append(("zeros", np.zeros(10000), 0.0))
    out.append(("normal_1e5", rng.standard_normal(100000), 0.0))
    out.append(("normal_1e6_init", rng.standard_normal(1000000), 1e3))
    out.append(("squares_monotone", rng.standard_normal(400000) ** 2, 0.0))
    out.append(("loguniform_signed", rng.choice([-1, 1], 300000) * 10.0 ** rng.uniform(-12, 12, 300000), 0.0))
    w = rng.standard_normal(200000) * 1e-3
    out.append(("walk_drift_to_zero", w - w.mean(), 0.0))
    # exact ties: multiples of 2^-53 added to a sum near 1 (ties at every step)
    ties = rng.integers(-8, 9, 50000).astype(np.float64) * 2.0 ** -53
    out.append(("ties_near_one", ties, 1.0))
    out.append(("halves", np.full(100000, 0.5) * rng.choice([-1, 1], 100000), 2.0 ** 53))
    small = rng.standard_normal(100000) * 1e-310  # subnormal terms
    out.append(("subnormal", small, 0.0))
    spikes = rng.standard_normal(200000)
    spikes[::997] *= 1e15
    out.append(("spikes", spikes, 0.0))
    canc = np.repeat(rng.standard_normal(5000) * 1e8, 2)
    canc[1::2] *= -1
    canc += rng.standard_normal(10000) * 1e-6
    out.append(("cancel_pairs", canc, 0.0))
    ints = rng.integers(-1000, 1000, 300000).astype(np.float64)
    out.append(("integers_exact", ints, 0.5))
    grow = 2.0 ** np.arange(-60, 60, 0.25)
    out.append(("growing_binades", np.concatenate([grow, -grow[::-1]]), 0.0))
    out.append(("sparse_nonzeros", np.where(rng.random(500000) < 0.01, rng.standard_normal(500000), 0.0), 0.0))
    # zero terms at an undecidable running sum are skipped as transparent steps:
    # all zeros (a dual residual with every bound finite), leading zeros, the
    # signed-zero corner (-0.0 init: +0.0 terms turn the sum into +0.0, -0.0
    # terms keep it), zero runs around an exact return to zero
    out.append(("zeros_1e6", np.zeros(1000000), 0.0))
    lead = np.zeros(400000)
    lead[300000:] = rng.standard_normal(100000)
    out.append(("leading_zeros", lead, 0.0))
    out.append(("negzero_init_poszeros", np.zeros(50000), -0.0))
    out.append(("negzero_init_negzeros", np.full(50000, -0.0), -0.0))
    nz = np.full(50000, -0.0)
    nz[40000] = 0.0
    out.append(("negzero_init_mixed", nz, -0.0))
    ret = np.zeros(300000)
    ret[1000], ret[2000] = 1.5, -1.5
    ret[250000:250010] = rng.standard_normal(10)
    out.append(("return_to_zero", ret, 0.0))
    cross = np.where(rng.random(600000) < 0.1, rng.standard_normal(600000) * 1e-4, 0.0)
    out.append(("cross_like_sparse", cross, 0.0))
    big = rng.standard_normal(3000000) * 10.0 ** rng.uniform(-3, 3, 3000000)
    out.append(("config2_like_3e6", big, 0.0))
    return out


@pytest.mark.parametrize("name,t,init", cases(), ids=[c[0] for c in cases()])
def test_exact_fold_matches_sequential(eng, name, t, init):
    want = seq(t, init)
    for grid in (0, 1, 7):
        (got,), _ = gpu_fold(eng, [t], [init], grid=grid)
        assert same(got, want), (name, grid, got, want, got - want)


def test_exact_fold_dependent_movement(eng):
    """movement = fold(dy^2) / omega, then += omega*dx*dx (solver.cpp:81-88),
    next to an independent cross-term fold, in one launch."""
    rng = np.random.default_rng(7)
    for trial in range(6):
        m, n = 200000 + trial, 400000 - trial
        dy = rng.standard_normal(m) * 10.0 ** rng.uniform(-6, 0)
        dx = rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 0)
        kx = rng.standard_normal(m)
        omega = 10.0 ** rng.uniform(-3, 3)
        cross_t = dy * (kx * 1e-3)
        dy2 = dy * dy
        dx2 = omega * dx * dx
        got, _ = gpu_fold(eng, [cross_t, dy2, dx2], inits=[0.0, 0.0, 0.0], init_from=[-1, -1, 1],
                          init_div=[1.0, 1.0, omega])
        want_mv = seq(dx2, seq(dy2) / omega)
        assert same(got[0], seq(cross_t)) and same(got[1], seq(dy2)), trial
        assert same(got[2], want_mv), (trial, got[2], want_mv)


def test_exact_fold_nonfinite_and_overflow_take_the_sequential_path(eng):
    t = np.ones(100000)
    t[5000] = np.inf
    assert same(gpu_fold(eng, [t])[0][0], np.inf)
    t[7000] = -np.inf
    assert np.isnan(gpu_fold(eng, [t])[0][0])
    t = np.full(1000, 1.7e308)
    assert same(gpu_fold(eng, [t])[0][0], seq(t))
    t = np.ones(1000)
    t[3] = np.nan
    assert np.isnan(gpu_fold(eng, [t])[0][0])


def test_exact_fold_random_stress(eng):
    rng = np.random.default_rng(99)
    for trial in range(40):
        n = int(rng.integers(1, 300000))
        kind = trial % 4
        if kind == 0:
            t = rng.standard_normal(n) * 10.0 ** rng.uniform(-20, 20, n)
        elif kind == 1:
            t = rng.standard_normal(n)
            t -= t.mean()
        elif kind == 2:
            t = (rng.integers(-3, 4, n) * 2.0 ** -52).astype(np.float64)
        else:
            t = rng.standard_normal(n) ** 2 * 10.0 ** rng.uniform(-5, 5)
        init = float(rng.standard_normal() * 10.0 ** rng.uniform(-5, 5)) if trial % 3 else 0.0
        got = gpu_fold(eng, [t], [init], grid=int(rng.integers(0, 600)))[0][0]
        assert same(got, seq(t, init)), (trial, kind, n)


def test_exact_fold_speed_report(eng, capsys):
    """Timing of the three trial folds of config 2 (cross and dy^2 over m =
    200k, movement over n = 400k), for DESIGN.md; no assertion on speed."""
    rng = np.random.default_rng(3)
    m, n = 200000, 400000
    dy = rng.standard_normal(m) * 1e-3
    t3 = [dy * rng.standard_normal(m), dy * dy, 3.0 * rng.standard_normal(n) ** 2 * 1e-6]
    _, ms = gpu_fold(eng, t3, inits=[0.0, 0.0, 0.0], init_from=[-1, -1, 1],
                     init_div=[1.0, 1.0, 3.0], reps=50)
    # the same with the zero patterns of early iterates (inactive rows: dy = 0)
    keep = rng.random(m) < 0.2
    dyz = np.where(keep, dy, 0.0)
    t3z = [dyz * rng.standard_normal(m), dyz * dyz, np.where(rng.random(n) < 0.3, t3[2], 0.0)]
    _, msz = gpu_fold(eng, t3z, inits=[0.0, 0.0, 0.0], init_from=[-1, -1, 1],
                      init_div=[1.0, 1.0, 3.0], reps=50)
    (gz,), _ = gpu_fold(eng, [np.zeros(n)], reps=50)
    _, ms0 = gpu_fold(eng, [np.zeros(n)], reps=50)
    with capsys.disabled():
        print(f"\n[exact fold] config-2 trial folds (200k + 200k + 400k terms): {1e3 * ms:.1f} us per launch; "
              f"80 % zero terms: {1e3 * msz:.1f} us; 400k zeros: {1e3 * ms0:.1f} us")
