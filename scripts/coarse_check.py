"""Dev helper: coarse vs exact band bounds (one-shard plan tables)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1510_01041_b200 import _native, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
pts = workloads.contaminated_line_points(n, 0)
q = n // 2 + 1
tabs = {}
for mode in ("0", "1"):
    os.environ["LMSB_BAND_COARSE"] = mode
    ctx = _native.Context()
    ctx.upload(pts[:, 0], pts[:, 1])
    K, k0, k1, t, seed = ctx.shard_plan(q, 1, 0)
    tabs[mode] = t
    print(mode, "K", K, "seed h", seed.height if seed.found else None)
ex, co = tabs["0"], tabs["1"]
fin = np.isfinite(ex[:, 1])
print("lb: coarse <= exact everywhere:", bool(np.all(co[fin, 0] <= ex[fin, 0] + 1e-9)))
order_ex = np.argsort(ex[:, 1])
order_co = np.argsort(co[:, 1])
rank_co = np.empty(len(order_co), int)
rank_co[order_co] = np.arange(len(order_co))
print("exact top-8 bands:", order_ex[:8].tolist())
print("their coarse ranks:", rank_co[order_ex[:8]].tolist())
print("exact wq of top8:", ex[order_ex[:8], 1].round(3).tolist())
print("coarse wq of those:", co[order_ex[:8], 1].round(3).tolist())
print("coarse top-8 :", order_co[:8].tolist(), co[order_co[:8], 1].round(3).tolist())
print("exact wq of coarse top-8:", ex[order_co[:8], 1].round(3).tolist())
d = co[fin, 1] - ex[fin, 1]
print("coarse-exact wq diff: min %.3f max %.3f mean %.3f" % (d.min(), d.max(), d.mean()))
print("lb gap (exact - coarse): median %.3f" % np.median(ex[fin, 0] - co[fin, 0]))
