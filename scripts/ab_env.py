"""Dev helper: interleaved A/B of environment knobs, one context per variant
in one process.  usage: ab_env.py N REPS 'K=V,K=V' 'K=V' ..."""
import os, sys, json
import numpy as np
sys.path.insert(0, '.')
from paper_1510_01041_b200 import _native, workloads

n, reps = int(sys.argv[1]), int(sys.argv[2])
seed = int(os.environ.get("AB_SEED", "0"))
variants = sys.argv[3:] or [""]
pts = workloads.contaminated_line_points(n, seed)
q = n // 2 + 1
total = n * (n - 1) // 2
ctxs = []
for v in variants:
    env = dict(kv.split("=") for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    c = _native.Context()
    for k, o in old.items():
        if o is None:
            os.environ.pop(k)
        else:
            os.environ[k] = o
    c.upload(pts[:, 0], pts[:, 1])
    ctxs.append(c)
times = [[] for _ in variants]
recs = [None] * len(variants)
stats = [None] * len(variants)
for r in range(reps):
    for k, c in enumerate(ctxs):
        rec = c.solve(q, 0, total)
        recs[k] = (rec.i, rec.j, rec.height)
        st = c.stats()
        times[k].append(st["ms_total"])
        stats[k] = {x: st[x] for x in ("band_survivors", "survivors", "ms_bound", "ms_partition",
                                        "ms_band_filter", "ms_filter_kernel", "launches") if x in st}
for k, v in enumerate(variants):
    print(json.dumps({"n": n, "env": v or "default", "ms": round(float(np.median(times[k][3:])), 4),
                      "same": recs[k] == recs[0], **stats[k]}))
