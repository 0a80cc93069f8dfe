"""CPU checks of the drop-in boundary: the engine library loads, exports every
entry point its headers declare, refuses to run without a GPU (no CPU
fallback), and the C parameter defaults equal SolverParams{} of the reference."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2106_04756_b200 import ENGINE_LIB, GEN_LIB, cabi, engine, instances

ROOT = Path(__file__).resolve().parents[1]


def _declared(header: str, prefix: str):
    text = (ROOT / "include" / header).read_text()
    return sorted(set(re.findall(r"\b(" + prefix + r"\w+)\s*\(", text)))


@pytest.mark.parametrize("header,prefix", [("folp_c.h", "folp_"), ("folp_gpu.h", "folp_gpu_"),
                                           ("folp_gen.h", "folp_gen_")])
def test_library_exports_every_declared_symbol(header, prefix):
    names = _declared(header, prefix)
    assert names
    lib = C.CDLL(str(GEN_LIB if header == "folp_gen.h" else ENGINE_LIB))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_cpp_api_symbols_exported():
    """folp::solve and the step-level API (solver.hpp:121-228) link from the .so."""
    import subprocess
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", str(ENGINE_LIB)],
                         capture_output=True, text=True, check=True).stdout
    for sym in ["folp::solve(folp::LinearProgram const&, folp::SolverParams const&, "
                "folp::PrimalDualPoint const&)",
                "folp::adaptive_step(", "folp::normalized_duality_gap(",
                "folp::restart_candidate(", "folp::should_restart(", "folp::pdhg_step(",
                "folp::convergence_info(", "folp::rescale_problem(", "folp::presolve(",
                "folp::SparseMatrix::from_triplets(", "folp::SparseMatrix::multiply(",
                "folp::validate("]:
        assert sym in out, sym


def test_param_defaults_match_reference(ref):
    mine = cabi.ParamsC()
    engine().lib.folp_params_default(C.byref(mine))
    theirs = cabi.ParamsC()
    ref.lib.folp_ref_params_default(C.byref(theirs))
    for name, _ in cabi.ParamsC._fields_:
        assert getattr(mine, name) == getattr(theirs, name), name
    py = cabi.params_to_c(cabi.params())
    for name, _ in cabi.ParamsC._fields_:
        if name not in ("reserved",):
            assert getattr(py, name) == getattr(mine, name), name


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device path")
def test_engine_fails_loudly_without_gpu():
    lp = instances.generate(1, 1, 0.05)
    with pytest.raises(cabi.FolpError) as e:
        engine().solve_lp(lp)
    assert e.value.kind in ("NoDevice", "CudaError")


def test_invalid_arguments_map_to_reference_exceptions():
    """check_params (solver.cpp:447-467) runs before any device work."""
    lp = instances.generate(1, 1, 0.05)
    for bad in (dict(eps_optimal=0.0), dict(beta_necessary=0.95),
                dict(evaluation_cadence=0), dict(theta_smoothing=2.0)):
        with pytest.raises(cabi.FolpError) as e:
            engine().solve_lp(lp, cabi.params(**bad))
        assert e.value.kind == "InvalidArgument", bad


def test_crossed_bounds_detected_on_host():
    """validate() -> PrimalInfeasibleDetected without touching the device
    (solver.cpp:824-830)."""
    lp = cabi.LP(1, 1, 1, np.array([0, 1]), np.array([0]), np.array([1.0]), np.array([1.0]),
                 np.array([1.0]), np.array([2.0]), np.array([1.0]))
    r = engine().solve_lp(lp)
    assert r.termination_reason == "PrimalInfeasibleDetected"
    assert r.iterations == 0


def test_dual_unbounded_detected_by_presolve():
    """Empty column with negative cost and no upper bound (test_solver.cpp:451-458)."""
    lp = cabi.LP(1, 2, 1, np.array([0, 1]), np.array([0]), np.array([1.0]),
                 np.array([1.0, -1.0]), np.array([1.0]), np.array([0.0, 0.0]),
                 np.array([np.inf, np.inf]))
    assert engine().solve_lp(lp).termination_reason == "DualUnboundedDetected"
