"""Dev: host-side phases of solve_lms at config 2 (run under gpurun)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import _native, workloads, solver
pts = workloads.contaminated_line_points(16384, 0)
for _ in range(5): lms.solve_lms(pts)
T = {}
R = 30
for _ in range(R):
    t0 = time.perf_counter(); x, y, q = solver.validated(pts, None); t1 = time.perf_counter()
    cand, con = _native.solve_fit(x, y, q); t2 = time.perf_counter()
    f = lms.solve_lms(pts); t3 = time.perf_counter()
    for k, v in (("validated", t1 - t0), ("solve_fit", t2 - t1), ("solve_lms total", t3 - t2)):
        T[k] = T.get(k, 0) + v / R * 1e6
ctx = _native.Context(); ctx.upload(x, y)
n = x.size
for _ in range(3): ctx.solve(q, 0, n*(n-1)//2)
t0 = time.perf_counter()
for _ in range(R): ctx.solve(q, 0, n*(n-1)//2)
T["ctx.solve (no upload, no contacts)"] = (time.perf_counter() - t0) / R * 1e6
t0 = time.perf_counter()
for _ in range(R): ctx.upload(x, y)
T["ctx.upload"] = (time.perf_counter() - t0) / R * 1e6
st = ctx.stats(); T["device ms_total"] = st["ms_total"] * 1e3
for k, v in T.items(): print(f"{v:9.1f} us {k}")
