import numpy as np, sys
sys.path.insert(0, '.')
from paper_2106_04756_b200 import engine, cabi, instances
from oracle import ref as R
lp = instances.generate(1, 1, 1.0)
p = cabi.params(record_iterate_trace=True, iteration_limit=120)
a = engine().solve_lp(lp, p, iterate_capacity=120)
b = R.binding().solve_lp(lp, p, iterate_capacity=120)
print("restarts", a.restart_iterations, b.restart_iterations)
for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a.iterate_trace, b.iterate_trace):
    dx = np.max(np.abs(xa-xb)/np.maximum(1,np.abs(xb))); dy = np.max(np.abs(ya-yb)/np.maximum(1,np.abs(yb)))
    print(ia, f"eta {ea:.17g} {eb:.17g} rel {abs(ea-eb)/eb:.2e}  dx {dx:.2e} dy {dy:.2e}")
