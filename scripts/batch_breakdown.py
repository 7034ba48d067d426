"""Dev: phases of solve_lms_batch on config 4 (8,192 fits of n = 512)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1510_01041_b200 as lms  # noqa: E402
from paper_1510_01041_b200 import _native, solver, workloads  # noqa: E402

F, m = 8192, 512
sets = [workloads.bench_points(m, seed=f) for f in range(F)]
lms.solve_lms_batch(sets)
T = {}
reps = 5
for _ in range(reps):
    t0 = time.perf_counter()
    X = np.concatenate([p[:, 0] for p in sets])
    Y = np.concatenate([p[:, 1] for p in sets])
    offsets = np.arange(F + 1, dtype=np.int64) * m
    ok = np.isfinite(X).all() and np.isfinite(Y).all()
    t1 = time.perf_counter()
    qv = np.full(F, m // 2 + 1, dtype=np.int64)
    cands, flags = solver._batched_fit_devices(X, Y, offsets, qv)
    t2 = time.perf_counter()
    fits = solver._fits_from_arrays(cands, flags, offsets, qv)
    t3 = time.perf_counter()
    for k, v in (("concat+checks", t1 - t0), ("device call (H2D+solve+flags D2H)", t2 - t1), ("tail", t3 - t2)):
        T[k] = T.get(k, 0) + v * 1e3
for k, v in T.items():
    print(f"{v / reps:8.2f} ms {k}")
t0 = time.perf_counter()
for _ in range(reps):
    lms.solve_lms_batch(sets)
print(f"{(time.perf_counter() - t0) / reps * 1e3:8.2f} ms solve_lms_batch")
