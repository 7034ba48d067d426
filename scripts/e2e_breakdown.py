"""Dev helper: where the end-to-end time of solve_lms (config 2) goes."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import _native, workloads
from paper_1510_01041_b200.solver import validated

pts = workloads.contaminated_line_points(16384, 0)
for _ in range(3):
    lms.solve_lms(pts)
T = {"validated": [], "solve_fit_wall": [], "device_ms_total": [], "solve_lms": []}
for _ in range(20):
    t0 = time.perf_counter(); x, y, q = validated(pts, None); t1 = time.perf_counter()
    cand, contacts = _native.solve_fit(x, y, q); t2 = time.perf_counter()
    T["validated"].append(t1 - t0); T["solve_fit_wall"].append(t2 - t1)
    t3 = time.perf_counter(); lms.solve_lms(pts); T["solve_lms"].append(time.perf_counter() - t3)
print({k: round(1e3 * float(np.median(v)), 4) for k, v in T.items() if v})
