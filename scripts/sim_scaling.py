"""Simulate the N-GPU strong-scaling split of one fit on one GPU.

For every world size R, run each rank's share on the same device and report
the max over ranks of its device time (what bench.py reports at N=R, minus
the two 56-byte-per-rank record all-gathers): `range` = the plain
partitioned solve (ctx.solve over the rank's pair-rank partition),
`owned` = the sharded band search with band ownership (plan of the rank's
own band slice + search of its own bands from the best seed over all ranks;
lms_ctx_solve_distributed's flow, the exchanges done on the host here).

usage: python scripts/sim_scaling.py N [reps]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1510_01041_b200 import _native, distributed, workloads  # noqa: E402
from paper_1510_01041_b200.backend import record_from_native  # noqa: E402

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


one_ms, one = timed(lambda: ctx.solve(q, 0, total))
ref = record_from_native(one)
for R in (1, 2, 4, 8):
    per_range, plans = [], []
    for r in range(R):
        r0, r1 = distributed.partition(total, R, r)
        ms, _ = timed(lambda: ctx.solve(q, r0, r1))
        per_range.append(ms)
        plans.append(timed(lambda: ctx.shard_plan(q, R, r)))
    seed = distributed.combine(np.stack([distributed.pack(record_from_native(p[1][2])) for p in plans]))
    seed_c = _native.Candidate.of(seed)
    detail, recs = [], []
    for r in range(R):
        ctx.shard_plan(q, R, r)  # the search reuses this rank's plan on the context
        ms_s, rec = timed(lambda: ctx.shard_search_owned(q, R, r, seed_c))
        st = ctx.stats()
        recs.append(distributed.pack(record_from_native(rec)))
        detail.append({"rank": r, "plan_ms": round(plans[r][0], 3), "search_ms": round(ms_s, 3),
                       "searched": st["bands_searched"], "collected": st["filtered_vertices"],
                       "band_surv": st["band_survivors"], "surv": st["survivors"],
                       "collect_ms": round(st["ms_collect"], 3),
                       "filter_ms": round(st["ms_band_filter"], 3)})
    comb = distributed.combine(np.stack(recs))
    print(json.dumps({"n": n, "R": R, "one_gpu_ms": round(one_ms, 3), "bands": plans[0][1][0],
                      "range_max_ms": round(max(per_range), 3),
                      "owned_max_ms": round(max(d["plan_ms"] + d["search_ms"] for d in detail), 3),
                      "same_record": comb == ref, "ranks": detail}), flush=True)
