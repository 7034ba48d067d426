"""Dev helper: config 4 end to end through solve_lms_batch (host arrays in,
LmsFit objects out), wall clock."""
import sys, time
sys.path.insert(0, '.')
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import workloads

F = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sets = [workloads.bench_points(512, seed=f) for f in range(F)]
for rep in range(3):
    t = time.perf_counter()
    fits = lms.solve_lms_batch(sets)
    print({"fits": len(fits), "e2e_ms": round((time.perf_counter() - t) * 1e3, 2)}, flush=True)
