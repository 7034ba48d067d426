"""Dev helper: plan all 8 shards, then ONE search of shard 0 bracketed by
cudaProfilerStart/Stop-free markers (ncu: use --launch-skip to the search)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_1510_01041_b200 import _native, workloads, distributed
from paper_1510_01041_b200.backend import record_from_native

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pts = workloads.contaminated_line_points(n, 0)
ctx = _native.Context()
ctx.upload(pts[:, 0], pts[:, 1])
q = n // 2 + 1
plans = [ctx.shard_plan(q, R, r) for r in range(R)]
table = distributed.interleave_band_table([p[1] for p in plans], plans[0][0])
seed = _native.Candidate.of(distributed.combine(np.stack([distributed.pack(record_from_native(p[2])) for p in plans])))
for _ in range(2):
    ctx.shard_search(q, R, 0, table, seed)
print("launches per search", ctx.stats()["launches"])
