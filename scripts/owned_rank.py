"""Dev: one rank's plan + own-band search (config 2 generator), stats printed."""
import json
import sys

sys.path.insert(0, ".")
from paper_1510_01041_b200 import _native, distributed, workloads  # noqa: E402
from paper_1510_01041_b200.backend import record_from_native  # noqa: E402
import numpy as np  # noqa: E402

n, R, r = (int(v) for v in sys.argv[1:4])
pts = workloads.contaminated_line_points(n, 0)
ctx = _native.Context()
ctx.upload(pts[:, 0], pts[:, 1])
q = n // 2 + 1
plans = [ctx.shard_plan(q, R, k) for k in range(R)]
seed = _native.Candidate.of(distributed.combine(np.stack([distributed.pack(record_from_native(p[2])) for p in plans])))
for _ in range(2):
    ctx.shard_plan(q, R, r)
    rec = ctx.shard_search_owned(q, R, r, seed)
    print(json.dumps(ctx.stats()), flush=True)
