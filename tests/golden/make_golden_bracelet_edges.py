"""bracelet_at on line lists whose source indices repeat or miss the anchors,
produced by the REFERENCE (geometry.py:182-218 snaps every line whose
source_index is i or j, and never raises for absent anchors).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_bracelet_edges.py
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lmsline import DualIntersection, DualLine, bracelet_at  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "bracelet_edges_golden.json")


def main():
    rng = np.random.default_rng(2024)
    rows = []
    for k in range(60):
        n = int(rng.integers(3, 14))
        a = rng.integers(-6, 7, n).astype(float)
        b = rng.integers(-9, 10, n).astype(float)
        src = list(range(n))
        kind = k % 3
        if kind == 0:    # duplicate source indices: several lines share the anchor ids
            for t in rng.choice(n, size=min(n, 3), replace=False):
                src[int(t)] = int(rng.integers(0, 3))
        elif kind == 1:  # anchors absent from the list
            src = [s + 100 for s in src]
        i, j = 0, 1
        u = float(rng.integers(-8, 9)) / 4.0
        v = float(a[0] * u - b[0]) if kind != 1 else float(rng.integers(-20, 21)) / 2.0
        lines = [DualLine(a=float(a[t]), b=float(b[t]), source_index=int(src[t])) for t in range(n)]
        q = int(rng.integers(2, n + 1))
        br = bracelet_at(DualIntersection(u=u, v=v, i=i, j=j), lines, q)
        rows.append({"a": a.tolist(), "b": b.tolist(), "src": src, "u": u.hex(), "v": v.hex(), "i": i, "j": j,
                     "q": q, "bracelet": None if br is None else
                     [br.v_low.hex(), br.v_high.hex(), br.height.hex()]})
    with open(OUT, "w") as fh:
        json.dump(rows, fh)
    print(f"wrote {OUT}: {len(rows)} cases, {sum(r['bracelet'] is None for r in rows)} None")


if __name__ == "__main__":
    main()
