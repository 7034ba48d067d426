"""Dev helper: simulate the N-GPU strong-scaling split on one GPU.

For every world size R, run each rank's share on the same device and report
the max over ranks of its device time (what bench.py reports at N=R, minus
the collectives): `range` = the plain partitioned solve (ctx.solve over the
rank's partition), `sharded` = the sharded band search (plan slice +
search of the partition against the exchanged table; the exchange itself is
a host concatenation here).
"""
import sys, json
sys.path.insert(0, '.')
import numpy as np
from paper_1510_01041_b200 import _native, workloads, distributed

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pts = workloads.contaminated_line_points(n, 0)
ctx = _native.Context()
ctx.upload(pts[:, 0], pts[:, 1])
q = n // 2 + 1
total = n * (n - 1) // 2


def timed(fn):
    best, out = None, None
    for _ in range(reps):
        ctx.record(0)
        out = fn()
        ctx.record(1)
        ms = ctx.elapsed_ms(0, 1)
        best = ms if best is None else min(best, ms)
    return best, out


ref = None
for R in (1, 2, 4, 8):
    per_range, per_shard, recs = [], [], []
    plans = []
    for r in range(R):
        r0, r1 = distributed.partition(total, R, r)
        ms, rec = timed(lambda: ctx.solve(q, r0, r1))
        per_range.append(ms)
        ms_p, plan = timed(lambda: ctx.shard_plan(q, R, r))
        plans.append((ms_p, plan))
    K = plans[0][1][0]
    table = distributed.interleave_band_table([p[1][1] for p in plans], K)
    from paper_1510_01041_b200.backend import record_from_native
    seed = distributed.combine(np.stack([distributed.pack(record_from_native(p[1][2])) for p in plans]))
    seed = _native.Candidate.of(seed)
    detail = []
    for r in range(R):
        ms_s, rec = timed(lambda: ctx.shard_search(q, R, r, table, seed))
        st = ctx.stats()
        recs.append(distributed.pack(__import__("paper_1510_01041_b200").backend.record_from_native(rec)))
        per_shard.append(plans[r][0] + ms_s)
        detail.append({"rank": r, "plan_ms": round(plans[r][0], 3), "search_ms": round(ms_s, 3),
                       "searched": st["bands_searched"], "collected": st["filtered_vertices"],
                       "band_surv": st["band_survivors"], "surv": st["survivors"],
                       "bound": round(st["ms_bound"], 3), "part": round(st["ms_partition"], 3),
                       "filter": round(st["ms_band_filter"], 3)})
    comb = distributed.combine(np.stack(recs))
    ref = ref or comb
    print(json.dumps({"n": n, "R": R, "bands": K, "range_max_ms": round(max(per_range), 3),
                      "sharded_max_ms": round(max(per_shard), 3), "same_record": comb == ref,
                      "ranks": detail}), flush=True)
