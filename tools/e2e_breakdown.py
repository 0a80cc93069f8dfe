import sys, time, os
sys.path.insert(0, '.')
from paper_2106_04756_b200 import engine, cabi, instances
lp = instances.generate(2, 1, 1.0)
e = engine()
for i in range(2):
    t = time.perf_counter()
    r = e.solve_lp(lp, cabi.params(iteration_limit=800), trace_capacity=1)
    print("e2e", time.perf_counter() - t, r.iterations, flush=True)
