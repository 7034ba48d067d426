"""Dev helper: LMSB_BAND_DEBUG breakdown of one shard's plan and search."""
import os, sys
os.environ["LMSB_BAND_DEBUG"] = "1"
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
for rep in range(3):
    plans = [ctx.shard_plan(q, R, r) for r in range(R)]
    table = distributed.interleave_band_table([p[1] for p in plans], plans[0][0])
    from paper_1510_01041_b200 import distributed
    from paper_1510_01041_b200.backend import record_from_native
    seed = _native.Candidate.of(distributed.combine(np.stack([distributed.pack(record_from_native(p[2])) for p in plans])))
    print("--- search rank 0", file=sys.stderr, flush=True)
    ctx.record(0)
    ctx.shard_search(q, R, 0, table, seed)
    ctx.record(1)
    print("search ms", ctx.elapsed_ms(0, 1), ctx.stats()["launches"], file=sys.stderr, flush=True)
