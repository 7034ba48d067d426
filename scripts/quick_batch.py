"""Dev helper: time the batched path on config 4 (8,192 fits of bench_points(512))."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
from paper_1510_01041_b200 import _native, workloads

F = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
sets = [workloads.bench_points(n, seed=f) for f in range(F)]
X = np.concatenate([s[:, 0] for s in sets]); Y = np.concatenate([s[:, 1] for s in sets])
offs = np.arange(F + 1, dtype=np.int64) * n
q = np.full(F, n // 2 + 1, dtype=np.int64)
ctx = _native.Context()
ctx.upload(X, Y)
for r in range(reps):
    t0 = time.perf_counter()
    recs = ctx.solve_batch(offs, q)
    dt = time.perf_counter() - t0
    st = ctx.stats()
    evals = F * n * (n * (n - 1) // 2)
    print(json.dumps({"F": F, "n": n, "wall_s": dt, "evals_per_s": evals / (st["ms_total"] / 1e3),
                      "found": sum(c.found for c in recs), "r0": [recs[0].i, recs[0].j, recs[0].height], **st}), flush=True)
