"""Dev helper: per-stage device timeline of band solves (LMSB_TRACE=1 must be
set in the environment).  usage: trace_fit.py N REPS"""
import sys
sys.path.insert(0, '.')
from paper_1510_01041_b200 import _native, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pts = workloads.contaminated_line_points(n, 0)
ctx = _native.Context()
ctx.upload(pts[:, 0], pts[:, 1])
q = n // 2 + 1
for r in range(reps):
    rec = ctx.solve(q, 0, n * (n - 1) // 2)
    print("ms_total", ctx.stats()["ms_total"], rec.i, rec.j, file=sys.stderr, flush=True)
