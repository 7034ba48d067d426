"""Dev helper: reproduce a band-stage case with the direct grouping."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1510_01041_b200 import _native, workloads
os.environ["LMSB_BAND"] = "2"
rng = np.random.default_rng(5)
n = 3000
cases = [workloads.config1_points(3, n=n)]
x = rng.integers(0, 200, n).astype(float)
cases.append(np.column_stack([x, rng.integers(0, 200, n).astype(float)]))
ctx = _native.Context()
for k, pts in enumerate(cases):
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    m = a.size
    for q in (m // 2 + 1, max(2, m // 4), m - 3):
        ctx.upload(a, b)
        try:
            r = ctx.solve(q, 0, m * (m - 1) // 2)
            print(k, q, "ok", r.height, ctx.stats()["direct_groups"])
        except Exception as e:
            print(k, q, "ERR", e)
            raise
