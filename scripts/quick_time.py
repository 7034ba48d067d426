"""Dev helper: time full exact fits through the context API and print stats."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_1510_01041_b200 import _native, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pts = workloads.contaminated_line_points(n, 0) if n != 1000 else workloads.config1_points(0)
ctx = _native.Context()
ctx.upload(pts[:, 0], pts[:, 1])
q = n // 2 + 1
total = n * (n - 1) // 2
for r in range(reps):
    t0 = time.perf_counter()
    rec = ctx.solve(q, 0, total)
    dt = time.perf_counter() - t0
    st = ctx.stats()
    print(json.dumps({"n": n, "wall_s": dt, "h": rec.height, "i": rec.i, "j": rec.j, "u": rec.u,
                      "evals_per_s": n * total / (st["ms_total"] / 1e3), **st}), flush=True)
