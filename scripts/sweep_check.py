"""Dev check: sweep collect (LMSB_SWEEP=1) vs the pre-test collect (=0) on the
same inputs -- identical records and collected counts; timings of both."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1510_01041_b200 import _native, workloads  # noqa: E402


def ctx_with(sweep):
    os.environ["LMSB_SWEEP"] = str(sweep)  # 0 never, 1 always
    c = _native.Context(0)
    os.environ.pop("LMSB_SWEEP", None)
    return c


def cases():
    yield "config2", workloads.contaminated_line_points(16384, 0)
    yield "c2_seed1_n8000", workloads.contaminated_line_points(8000, 1)
    rng = np.random.default_rng(5)
    p = rng.integers(0, 300, (5000, 2)).astype(float)
    yield "grid_dupx_5000", p
    p = workloads.contaminated_line_points(4000, 2)
    p[:200, 1] += 1e6
    yield "outliers_1e6", p
    x = rng.uniform(-1, 1, 3000)
    yield "near_horizontal", np.column_stack([x, 1e-9 * x + rng.normal(0, 1e-12, 3000)])
    x = np.repeat(np.arange(60.0), 50)
    yield "vertical_structure", np.column_stack([x, rng.normal(0, 5, x.size)])
    x = rng.uniform(0, 1, 4096)
    x[::7] = x[0]  # many exact duplicates
    yield "dup_x_many", np.column_stack([x, 3 * x + rng.normal(0, 0.01, 4096)])
    x = 1.0 + np.arange(3000) * 1e-12  # nearly parallel lines
    yield "near_parallel", np.column_stack([x, rng.normal(0, 1, 3000)])
    if "--big" in sys.argv:
        yield "config3", workloads.contaminated_line_points(65536, 0)


res = []
c0, c1 = ctx_with(0), ctx_with(1)
for name, pts in cases():
    n = len(pts)
    q = n // 2 + 1
    total = n * (n - 1) // 2
    out = {"case": name, "n": n}
    for tag, c in (("pre", c0), ("sweep", c1)):
        c.upload(pts[:, 0], pts[:, 1])
        rec = c.solve(q, 0, total)
        t = []
        for _ in range(3):
            c.solve(q, 0, total)
            t.append(c.stats()["ms_total"])
        st = c.stats()
        out[tag] = {"rec": [rec.height, rec.i, rec.j, rec.u], "ms": min(t), "ms_collect": st["ms_collect"],
                    "filtered": st["filtered_vertices"], "bands": st["bands"],
                    "searched": st["bands_searched"], "runs": st.get("sweep_runs")}
    out["same"] = out["pre"]["rec"] == out["sweep"]["rec"] and out["pre"]["filtered"] == out["sweep"]["filtered"]
    print(json.dumps(out), flush=True)
    res.append(out)
print("ALL_SAME", all(r["same"] for r in res))
