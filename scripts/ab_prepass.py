"""Dev helper: A/B of the split pass-0 screen (LMSB_PREPASS_SPLIT) in one process."""
import os, sys, json
import numpy as np
sys.path.insert(0, '.')
from paper_1510_01041_b200 import _native, workloads

for n in [int(a) for a in sys.argv[1:]] or [16384, 65536]:
    pts = workloads.contaminated_line_points(n, 0)
    q = n // 2 + 1
    total = n * (n - 1) // 2
    ctxs = {}
    for v in ("0", "1"):
        os.environ["LMSB_PREPASS_SPLIT"] = v
        c = _native.Context()
        c.upload(pts[:, 0], pts[:, 1])
        ctxs[v] = c
    times = {"0": [], "1": []}
    recs = {}
    for r in range(30):
        for v, c in ctxs.items():
            rec = c.solve(q, 0, total)
            recs[v] = (rec.i, rec.j, rec.height)
            times[v].append(c.stats()["ms_total"])
    print(json.dumps({"n": n, **{f"ms_split{v}": float(np.median(t[3:])) for v, t in times.items()},
                      "same": recs["0"] == recs["1"], "survivors": c.stats().get("survivors")}))
