"""Concurrent solves on one GPU (SURVEY.md 8b threading contract and 8f row 3:
the reference's run_bench thread pool, bench.cpp:46-73, runs independent
solves on shared LinearPrograms at once).  Each solve owns its context and
stream; results must equal the same solves run one after another, bit for
bit (deterministic reductions, no shared mutable state)."""
import threading

import numpy as np
import pytest

from paper_2106_04756_b200 import cabi, instances

pytestmark = pytest.mark.gpu


def test_concurrent_solves_match_sequential(eng):
    lps = [instances.generate(1, s, 0.5) for s in range(1, 5)] + \
          [instances.generate(2, 7, 0.005), instances.generate(5, 2, 0.005)]
    lps = lps + lps[:2]  # the same LinearProgram solved twice at once
    p = cabi.params(kkt_pass_limit=20000)
    seq = [eng.solve_lp(lp, p) for lp in lps]
    out = [None] * len(lps)
    errs = []

    def run(i):
        try:
            out[i] = eng.solve_lp(lps[i], p)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(lps))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for a, b in zip(out, seq):
        assert a.termination_reason == b.termination_reason
        assert a.iterations == b.iterations and a.restart_iterations == b.restart_iterations
        assert a.final_info == b.final_info
        assert np.array_equal(a.primal_solution, b.primal_solution)
        assert np.array_equal(a.dual_solution, b.dual_solution)
