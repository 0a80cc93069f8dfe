"""ctypes mirror of include/folp_c.h -- the FFI surface of the solve path.

The same struct layouts serve both implementations of that header:
``libfolp_b200.so`` (the B200 engine, prefix ``folp_``) and, in tests only,
``oracle/_ref/libfolp_ref.so`` (the compiled reference, prefix ``folp_ref_``).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import Optional

import numpy as np

# status codes (folp_c.h)
FOLP_OK = 0
ERRORS = {
    1: "InvalidArgument", 2: "RuntimeError", 3: "CudaError", 4: "OutOfMemory",
    10: "DimensionMismatch", 11: "EmptyMatrix", 12: "UnsupportedNorm",
    13: "NonPositiveWeight", 14: "NonPositiveRadius", 15: "StepSizeUnderflow",
    16: "NonFiniteIterate", 17: "InfiniteProduct", 18: "NoDevice",
}
TERMINATION = ["Optimal", "IterationLimit", "KktPassLimit", "TimeLimit",
               "NumericalError", "PrimalInfeasibleDetected", "DualUnboundedDetected"]
STEP_POLICY = {"adaptive": 0, "constant": 1, "malitsky_pock": 2}
RESTART_SCHEME = {"pdlp": 0, "theory": 1, "none": 2}

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class FolpError(RuntimeError):
    """A folp_c.h call returned a FOLP_E_* code; ``kind`` names the
    reference exception type (folp/types.hpp)."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.kind = ERRORS.get(code, f"code{code}")
        super().__init__(f"{self.kind}: {message}")


class LpC(C.Structure):
    _fields_ = [
        ("num_rows", C.c_int64), ("num_cols", C.c_int64),
        ("num_inequality_rows", C.c_int64), ("nnz", C.c_int64),
        ("row_start", _i64p), ("row_cols", _i64p), ("row_values", _f64p),
        ("objective", _f64p), ("right_hand_side", _f64p),
        ("variable_lower", _f64p), ("variable_upper", _f64p),
        ("objective_constant", C.c_double),
    ]


class ParamsC(C.Structure):
    _fields_ = [
        ("eps_optimal", C.c_double), ("beta_sufficient", C.c_double),
        ("beta_necessary", C.c_double), ("beta_artificial", C.c_double),
        ("restart_scheme", C.c_int32), ("step_policy", C.c_int32),
        ("theta_smoothing", C.c_double), ("eps_zero", C.c_double),
        ("mp_breaking_factor", C.c_double), ("mp_downscaling_factor", C.c_double),
        ("mp_interpolation_coefficient", C.c_double),
        ("evaluation_cadence", C.c_int64), ("kkt_pass_limit", C.c_double),
        ("iteration_limit", C.c_int64), ("time_limit_seconds", C.c_double),
        ("ruiz_iterations", C.c_int64), ("use_pock_chambolle", C.c_int32),
        ("scale_invariant_initial_primal_weight", C.c_int32),
        ("pc_alpha", C.c_double), ("use_presolve", C.c_int32),
        ("verbosity", C.c_int32), ("record_iterate_trace", C.c_int32),
        ("reserved", C.c_int32),
    ]


class InfoC(C.Structure):
    _fields_ = [(name, C.c_double) for name in (
        "primal_objective", "dual_objective", "gap_abs", "primal_residual_norm",
        "dual_residual_norm", "norm_q", "norm_c")]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class ResultC(C.Structure):
    _fields_ = [
        ("primal_solution", _f64p), ("dual_solution", _f64p), ("reduced_costs", _f64p),
        ("restart_capacity", C.c_int64), ("restart_iterations", _i64p),
        ("trace_capacity", C.c_int64), ("trace_iteration", _i64p),
        ("trace_kkt_passes", _f64p), ("trace_current", C.POINTER(InfoC)),
        ("trace_average", C.POINTER(InfoC)),
        ("iterate_capacity", C.c_int64), ("iterate_iteration", _i64p),
        ("iterate_eta", _f64p), ("iterate_primal", _f64p), ("iterate_dual", _f64p),
        ("iterate_n", C.c_int64), ("iterate_m", C.c_int64),
        ("termination_reason", C.c_int32), ("pad0", C.c_int32),
        ("final_info", InfoC), ("iterations", C.c_int64), ("kkt_passes", C.c_double),
        ("wall_seconds", C.c_double), ("restarts", C.c_int64), ("step_trials", C.c_int64),
        ("step_condition_violations", C.c_int64), ("num_restart_iterations", C.c_int64),
        ("num_trace", C.c_int64), ("num_iterates", C.c_int64),
    ]


def _f64(a: np.ndarray):
    return a.ctypes.data_as(_f64p)


def _i64(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


@dataclasses.dataclass
class LP:
    """A LinearProgram (lp_model.hpp:38-54) held as numpy arrays, K in CSR."""

    num_rows: int
    num_cols: int
    num_inequality_rows: int
    row_start: np.ndarray
    row_cols: np.ndarray
    row_values: np.ndarray
    objective: np.ndarray
    right_hand_side: np.ndarray
    variable_lower: np.ndarray
    variable_upper: np.ndarray
    objective_constant: float = 0.0
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_values.shape[0])

    def to_c(self) -> LpC:
        for f in ("row_start", "row_cols"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.int64))
        for f in ("row_values", "objective", "right_hand_side", "variable_lower",
                  "variable_upper"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.float64))
        return LpC(self.num_rows, self.num_cols, self.num_inequality_rows, self.nnz,
                   _i64(self.row_start), _i64(self.row_cols), _f64(self.row_values),
                   _f64(self.objective), _f64(self.right_hand_side),
                   _f64(self.variable_lower), _f64(self.variable_upper),
                   float(self.objective_constant))

    def dense(self) -> np.ndarray:
        k = np.zeros((self.num_rows, self.num_cols))
        for r in range(self.num_rows):
            for e in range(self.row_start[r], self.row_start[r + 1]):
                k[r, self.row_cols[e]] = self.row_values[e]
        return k


def params(**overrides) -> dict:
    """SolverParams defaults (solver.hpp:34-70) with keyword overrides."""
    p = dict(eps_optimal=1e-8, beta_sufficient=0.9, beta_necessary=0.1,
             beta_artificial=0.5, restart_scheme="pdlp", step_policy="adaptive",
             theta_smoothing=0.5, eps_zero=1e-10, mp_breaking_factor=1.0,
             mp_downscaling_factor=0.5, mp_interpolation_coefficient=0.4,
             evaluation_cadence=40, kkt_pass_limit=math.inf,
             iteration_limit=2**63 - 1, time_limit_seconds=math.inf, ruiz_iterations=10,
             use_pock_chambolle=True, pc_alpha=1.0,
             scale_invariant_initial_primal_weight=True, use_presolve=True,
             verbosity=0, record_iterate_trace=False)
    unknown = set(overrides) - set(p)
    if unknown:
        raise TypeError(f"unknown solver parameters: {sorted(unknown)}")
    p.update(overrides)
    return p


def params_to_c(p: dict) -> ParamsC:
    c = ParamsC()
    for name, _ in ParamsC._fields_:
        if name == "reserved":
            continue
        v = p[name]
        if name == "restart_scheme":
            v = RESTART_SCHEME[v] if isinstance(v, str) else int(v)
        elif name == "step_policy":
            v = STEP_POLICY[v] if isinstance(v, str) else int(v)
        elif isinstance(v, bool):
            v = int(v)
        setattr(c, name, v)
    return c


@dataclasses.dataclass
class SolveResult:
    """SolveResult (solver.hpp:97-115)."""

    termination_reason: str
    primal_solution: np.ndarray
    dual_solution: np.ndarray
    reduced_costs: np.ndarray
    final_info: dict
    iterations: int
    kkt_passes: float
    wall_seconds: float
    restarts: int
    step_trials: int
    step_condition_violations: int
    restart_iterations: list
    trace: list
    iterate_trace: list  # (iteration, eta_used, x, y) in the working space


def result_to_c(r: SolveResult):
    """A folp_result_c view of a SolveResult (for the I/O entry points);
    returns (struct, arrays kept alive)."""
    x = np.ascontiguousarray(r.primal_solution, dtype=np.float64)
    y = np.ascontiguousarray(r.dual_solution, dtype=np.float64)
    z = np.ascontiguousarray(r.reduced_costs, dtype=np.float64)
    nt = len(r.trace)
    t_it = np.array([t["iteration"] for t in r.trace] or [0], dtype=np.int64)
    t_kkt = np.array([t["kkt_passes"] for t in r.trace] or [0.0], dtype=np.float64)
    t_cur = (InfoC * max(1, nt))()
    t_avg = (InfoC * max(1, nt))()
    fields = [f for f, _ in InfoC._fields_]
    for i, t in enumerate(r.trace):
        t_cur[i] = InfoC(*[t["current"][f] for f in fields])
        t_avg[i] = InfoC(*[t["average"][f] for f in fields])
    rc = ResultC()
    rc.primal_solution, rc.dual_solution, rc.reduced_costs = _f64(x), _f64(y), _f64(z)
    rc.trace_capacity = nt
    rc.num_trace = nt
    rc.trace_iteration, rc.trace_kkt_passes = _i64(t_it), _f64(t_kkt)
    rc.trace_current, rc.trace_average = t_cur, t_avg
    rc.termination_reason = TERMINATION.index(r.termination_reason)
    rc.final_info = InfoC(*[r.final_info[f] for f in fields])
    rc.iterations, rc.kkt_passes, rc.wall_seconds = r.iterations, r.kkt_passes, r.wall_seconds
    rc.restarts, rc.step_trials = r.restarts, r.step_trials
    rc.step_condition_violations = r.step_condition_violations
    return rc, (x, y, z, t_it, t_kkt, t_cur, t_avg)


class ShardC(C.Structure):
    """include/folp_gpu.h folp_gpu_shard."""
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("backend", C.c_int32),
                ("partition", C.c_int32), ("nccl_id", C.c_ubyte * 128), ("loopback", C.c_void_p)]


SHARD_NCCL = 1
SHARD_LOOPBACK = 2
PARTITIONS = {"rows": 0, "cols": 1, "auto": 2}  # FOLP_SHARD_ROWS / COLS / AUTO


class Binding:
    """The folp_c.h entry points of one shared library."""

    def __init__(self, lib: C.CDLL, prefix: str):
        self.lib = lib
        self.prefix = prefix
        f = self._fn
        f("params_default", None, [C.POINTER(ParamsC)])
        f("solve", C.c_int, [C.POINTER(LpC), C.POINTER(ParamsC), _f64p, _f64p,
                              C.POINTER(ResultC)])
        f("multiply", C.c_int, [C.POINTER(LpC), _f64p, _f64p])
        f("multiply_transpose", C.c_int, [C.POINTER(LpC), _f64p, _f64p])
        f("rescale", C.c_int, [C.POINTER(LpC), C.c_int64, C.c_int32, C.c_double]
          + [_f64p] * 7)
        f("convergence_info", C.c_int, [C.POINTER(LpC), _f64p, _f64p, C.POINTER(InfoC)])
        f("normalized_duality_gap", C.c_int, [C.POINTER(LpC), _f64p, _f64p, C.c_double,
                                               C.c_double, _f64p])
        f("adaptive_step", C.c_int, [C.POINTER(LpC), _f64p, _f64p, C.c_double, C.c_double,
                                      C.c_int64, _f64p, _f64p, _f64p, _f64p, _i64p, _f64p,
                                      _f64p])
        f("last_error", C.c_char_p, [])
        f("malitsky_pock_step", C.c_int, [C.POINTER(LpC), _f64p, _f64p, C.c_double, C.c_double,
                                           C.c_double, C.POINTER(ParamsC), _f64p, _f64p, _f64p,
                                           _f64p, _i64p])
        if hasattr(lib, prefix + "session_create"):
            f("session_create", C.c_int, [C.POINTER(LpC), C.POINTER(ParamsC), _f64p, _f64p,
                                           C.POINTER(C.c_void_p)])
            f("session_advance", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                            _f64p])
            f("session_stats", C.c_int, [C.c_void_p, _i64p, _f64p, _i64p, _i64p])
            f("session_result", C.c_int, [C.c_void_p, C.POINTER(ResultC)])
            f("session_partition", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)])
            f("session_destroy", None, [C.c_void_p])
        if hasattr(lib, prefix + "solve_sharded"):
            f("solve_sharded", C.c_int, [C.POINTER(LpC), C.POINTER(ParamsC), _f64p, _f64p,
                                          C.POINTER(ShardC), C.POINTER(ResultC)])
            f("session_create_sharded", C.c_int, [C.POINTER(LpC), C.POINTER(ParamsC), _f64p,
                                                   _f64p, C.POINTER(ShardC),
                                                   C.POINTER(C.c_void_p)])

        if hasattr(lib, prefix + "mps_parse"):
            f("mps_parse", C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_void_p)])
            f("mps_parse_file", C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)])
            f("mps_view", C.c_int, [C.c_void_p, C.POINTER(LpC), C.POINTER(C.c_char_p),
                                     C.POINTER(C.c_int32)])
            f("mps_destroy", None, [C.c_void_p])
            f("mps_write", C.c_int, [C.POINTER(LpC), C.c_char_p, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_int64)])
            f("result_json", C.c_int, [C.POINTER(ResultC), C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_int64)])
            f("result_write", C.c_int, [C.POINTER(ResultC), C.c_int64, C.c_int64, C.c_char_p])
            f("buffer_free", None, [C.c_void_p])

    def _fn(self, name, restype, argtypes):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = restype
        fn.argtypes = argtypes
        setattr(self, name, fn)

    def check(self, code: int) -> None:
        if code != FOLP_OK:
            raise FolpError(code, self.last_error().decode(errors="replace"))

    # ---- high-level wrappers --------------------------------------------
    def solve_lp(self, lp: LP, p: Optional[dict] = None, x0=None, y0=None,
                 trace_capacity: int = 100000, iterate_capacity: int = 0,
                 shard: Optional[ShardC] = None, copy_iterates: bool = True) -> SolveResult:
        """folp_solve, or folp_solve_sharded as one row shard when `shard`
        is given (see paper_2106_04756_b200/shard.py).  copy_iterates=False
        returns the iterate trace as views into one buffer (full-size
        traces: 100 iterates of config 5 are 12.8 GB)."""
        p = p or params()
        lpc = lp.to_c()
        pc = params_to_c(p)
        n, m = lp.num_cols, lp.num_rows
        x = np.zeros(n)
        y = np.zeros(m)
        rc = np.zeros(n)
        rst = np.zeros(max(1, trace_capacity), dtype=np.int64)
        t_it = np.zeros(max(1, trace_capacity), dtype=np.int64)
        t_kkt = np.zeros(max(1, trace_capacity))
        t_cur = (InfoC * max(1, trace_capacity))()
        t_avg = (InfoC * max(1, trace_capacity))()
        icap = iterate_capacity if p.get("record_iterate_trace") else 0
        i_it = np.zeros(max(1, icap), dtype=np.int64)
        i_eta = np.zeros(max(1, icap))
        i_x = np.zeros(max(1, icap * n))
        i_y = np.zeros(max(1, icap * m))
        res = ResultC()
        res.primal_solution = _f64(x)
        res.dual_solution = _f64(y)
        res.reduced_costs = _f64(rc)
        res.restart_capacity = trace_capacity
        res.restart_iterations = _i64(rst)
        res.trace_capacity = trace_capacity
        res.trace_iteration = _i64(t_it)
        res.trace_kkt_passes = _f64(t_kkt)
        res.trace_current = t_cur
        res.trace_average = t_avg
        res.iterate_capacity = icap
        res.iterate_iteration = _i64(i_it)
        res.iterate_eta = _f64(i_eta)
        res.iterate_primal = _f64(i_x)
        res.iterate_dual = _f64(i_y)
        xp = None if x0 is None else _f64(np.ascontiguousarray(x0, dtype=np.float64))
        yp = None if y0 is None else _f64(np.ascontiguousarray(y0, dtype=np.float64))
        if shard is None:
            self.check(self.solve(C.byref(lpc), C.byref(pc), xp, yp, C.byref(res)))
        else:
            self.check(self.solve_sharded(C.byref(lpc), C.byref(pc), xp, yp, C.byref(shard),
                                          C.byref(res)))
        nt = min(res.num_trace, trace_capacity)
        trace = [dict(iteration=int(t_it[i]), kkt_passes=float(t_kkt[i]),
                      current=t_cur[i].as_dict(), average=t_avg[i].as_dict())
                 for i in range(nt)]
        ni = min(res.num_iterates, icap)
        inn, imm = res.iterate_n, res.iterate_m
        cp = (lambda a: a.copy()) if copy_iterates else (lambda a: a)
        iters = [(int(i_it[i]), float(i_eta[i]), cp(i_x[i * inn:(i + 1) * inn]),
                  cp(i_y[i * imm:(i + 1) * imm])) for i in range(ni)]
        return SolveResult(
            termination_reason=TERMINATION[res.termination_reason], primal_solution=x,
            dual_solution=y, reduced_costs=rc, final_info=res.final_info.as_dict(),
            iterations=res.iterations, kkt_passes=res.kkt_passes,
            wall_seconds=res.wall_seconds, restarts=res.restarts,
            step_trials=res.step_trials,
            step_condition_violations=res.step_condition_violations,
            restart_iterations=[int(v) for v in rst[:min(res.num_restart_iterations,
                                                        trace_capacity)]],
            trace=trace, iterate_trace=iters)

    # ---- MPS and result I/O (folp_c.h) ---------------
    def _mps_lp(self, h) -> tuple:
        lpc, name, mx = LpC(), C.c_char_p(), C.c_int32()
        self.check(self.mps_view(h, C.byref(lpc), C.byref(name), C.byref(mx)))
        m, n, nnz = lpc.num_rows, lpc.num_cols, lpc.nnz

        def arr(ptr, k, dt):
            return np.ctypeslib.as_array(ptr, shape=(k,)).astype(dt, copy=True) if k else \
                np.zeros(0, dtype=dt)
        lp = LP(num_rows=m, num_cols=n, num_inequality_rows=lpc.num_inequality_rows,
                row_start=arr(lpc.row_start, m + 1, np.int64),
                row_cols=arr(lpc.row_cols, nnz, np.int64),
                row_values=arr(lpc.row_values, nnz, np.float64),
                objective=arr(lpc.objective, n, np.float64),
                right_hand_side=arr(lpc.right_hand_side, m, np.float64),
                variable_lower=arr(lpc.variable_lower, n, np.float64),
                variable_upper=arr(lpc.variable_upper, n, np.float64),
                objective_constant=lpc.objective_constant, name=name.value.decode())
        return lp, name.value.decode(), bool(mx.value)

    def parse_mps(self, text) -> tuple:
        """parse_mps (mps.hpp:50): (LP, name, was_maximization)."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        self.check(self.mps_parse(data, len(data), C.byref(h)))
        try:
            return self._mps_lp(h)
        finally:
            self.mps_destroy(h)

    def parse_mps_file(self, path: str) -> tuple:
        h = C.c_void_p()
        self.check(self.mps_parse_file(str(path).encode(), C.byref(h)))
        try:
            return self._mps_lp(h)
        finally:
            self.mps_destroy(h)

    def _take_text(self, call) -> str:
        buf, length = C.c_void_p(), C.c_int64()
        self.check(call(C.byref(buf), C.byref(length)))
        try:
            return C.string_at(buf, length.value).decode()
        finally:
            self.buffer_free(buf)

    def write_mps(self, lp: LP, name: str = "") -> str:
        """write_mps (mps.hpp:55)."""
        lpc = lp.to_c()
        return self._take_text(lambda b, n: self.mps_write(C.byref(lpc), name.encode(), b, n))

    def result_to_json(self, r: SolveResult) -> str:
        """result_to_json (result_io.hpp:26)."""
        rc, keep = result_to_c(r)
        return self._take_text(lambda b, n: self.result_json(C.byref(rc), b, n))

    def write_result(self, r: SolveResult, output_dir: str) -> None:
        """write_result (result_io.hpp:31)."""
        rc, keep = result_to_c(r)
        self.check(self.result_write(C.byref(rc), len(r.dual_solution), len(r.primal_solution),
                                     str(output_dir).encode()))

    def session(self, lp: LP, p: Optional[dict] = None,
                shard: Optional[ShardC] = None) -> "Session":
        return Session(self, lp, p or params(), shard)

    def mp_step(self, lp: LP, x, y, omega: float, eta_prev: float, theta_prev: float,
                p: Optional[dict] = None) -> dict:
        lpc = lp.to_c()
        pc = params_to_c(p or params())
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        xn = np.zeros(lp.num_cols)
        yn = np.zeros(lp.num_rows)
        en, tn = C.c_double(), C.c_double()
        tr = C.c_int64()
        self.check(self.malitsky_pock_step(C.byref(lpc), _f64(x), _f64(y), omega, eta_prev,
                                           theta_prev, C.byref(pc), _f64(xn), _f64(yn),
                                           C.byref(en), C.byref(tn), C.byref(tr)))
        return dict(x=xn, y=yn, eta_next=en.value, theta_next=tn.value, trials=tr.value)

    def kx(self, lp: LP, x) -> np.ndarray:
        lpc = lp.to_c()
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(lp.num_rows)
        self.check(self.multiply(C.byref(lpc), _f64(x), _f64(out)))
        return out

    def kty(self, lp: LP, y) -> np.ndarray:
        lpc = lp.to_c()
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(lp.num_cols)
        self.check(self.multiply_transpose(C.byref(lpc), _f64(y), _f64(out)))
        return out

    def rescale_lp(self, lp: LP, ruiz: int = 10, pc: bool = True, alpha: float = 1.0) -> dict:
        lpc = lp.to_c()
        out = dict(row_scale=np.zeros(lp.num_rows), col_scale=np.zeros(lp.num_cols),
                   values=np.zeros(lp.nnz), objective=np.zeros(lp.num_cols),
                   rhs=np.zeros(lp.num_rows), lower=np.zeros(lp.num_cols),
                   upper=np.zeros(lp.num_cols))
        self.check(self.rescale(C.byref(lpc), ruiz, int(pc), alpha,
                                *[_f64(out[k]) for k in ("row_scale", "col_scale", "values",
                                                         "objective", "rhs", "lower",
                                                         "upper")]))
        return out

    def info(self, lp: LP, x, y) -> dict:
        lpc = lp.to_c()
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = InfoC()
        self.check(self.convergence_info(C.byref(lpc), _f64(x), _f64(y), C.byref(out)))
        return out.as_dict()

    def ndg(self, lp: LP, x, y, radius: float, omega: float) -> float:
        lpc = lp.to_c()
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        g = C.c_double()
        self.check(self.normalized_duality_gap(C.byref(lpc), _f64(x), _f64(y), radius, omega,
                                               C.byref(g)))
        return g.value

    def step(self, lp: LP, x, y, omega: float, eta_hat: float, k: int) -> dict:
        lpc = lp.to_c()
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        xn = np.zeros(lp.num_cols)
        yn = np.zeros(lp.num_rows)
        eu, en, mv, cr = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        tr = C.c_int64()
        self.check(self.adaptive_step(C.byref(lpc), _f64(x), _f64(y), omega, eta_hat, k,
                                      _f64(xn), _f64(yn), C.byref(eu), C.byref(en),
                                      C.byref(tr), C.byref(mv), C.byref(cr)))
        return dict(x=xn, y=yn, eta_used=eu.value, eta_hat_next=en.value, trials=tr.value,
                    movement_sq=mv.value, cross_term=cr.value)


class Session:
    """A resumable folp::solve (folp_session_*): advance() runs whole
    evaluation periods and returns their device time (CUDA events on the
    engine stream)."""

    def __init__(self, b: Binding, lp: LP, p: dict, shard: Optional[ShardC] = None):
        self.b = b
        self._lpc = lp.to_c()  # keeps the arrays alive
        self._pc = params_to_c(p)
        self._shard = shard
        h = C.c_void_p()
        if shard is None:
            b.check(b.session_create(C.byref(self._lpc), C.byref(self._pc), None, None,
                                     C.byref(h)))
        else:
            b.check(b.session_create_sharded(C.byref(self._lpc), C.byref(self._pc), None, None,
                                             C.byref(shard), C.byref(h)))
        self.h = h
        self.finished = False

    def advance(self, evaluations: int = 1) -> float:
        fin = C.c_int32()
        ms = C.c_double()
        self.b.check(self.b.session_advance(self.h, evaluations, C.byref(fin), C.byref(ms)))
        self.finished = bool(fin.value)
        return ms.value

    def stats(self) -> dict:
        it, slots, launches = C.c_int64(), C.c_int64(), C.c_int64()
        ms = C.c_double()
        self.b.check(self.b.session_stats(self.h, C.byref(it), C.byref(ms), C.byref(slots),
                                          C.byref(launches)))
        return dict(iterations=it.value, loop_ms=ms.value, loop_slots=slots.value,
                    launches=launches.value)

    def partition(self) -> int:
        """The shard partition the device context runs (0 rows, 1 columns)."""
        v = C.c_int32()
        self.b.check(self.b.session_partition(self.h, C.byref(v)))
        return v.value

    def close(self) -> None:
        if self.h:
            self.b.session_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
