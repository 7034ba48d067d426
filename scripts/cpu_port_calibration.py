"""Build-container only: the reference package's own _scan_rank_range vs the
numpy restatement bench.py times (oracle/numpy_scan.py) and the C++ oracle,
on the same config-2 rank slices; writes profiles/r02_cpu_port_calibration.json.

    PYTHONPATH=/root/reference/pkg/src python scripts/cpu_port_calibration.py
"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from lmsline.backend import _scan_rank_range  # noqa: E402

import oracle  # noqa: E402
from oracle import numpy_scan  # noqa: E402
from paper_1510_01041_b200 import workloads  # noqa: E402

n = 16384
pts = workloads.contaminated_line_points(n, 0)
a, b = pts[:, 0].copy(), pts[:, 1].copy()
q = n // 2 + 1
total = n * (n - 1) // 2
slices = [((s * total) // 8, (s * total) // 8 + 732) for s in range(8)]  # 3 chunks of 244 each
out = {"n": n, "slices": slices, "vertices": sum(r1 - r0 for r0, r1 in slices)}
for name, fn in (("reference _scan_rank_range", lambda r0, r1: _scan_rank_range(a, b, q, r0, r1)),
                 ("numpy port (oracle/numpy_scan.py)", lambda r0, r1: numpy_scan.scan_rank_range(a, b, q, r0, r1)),
                 ("C++ oracle, 1 thread", lambda r0, r1: oracle.min_bracelet(a, b, q, r0, r1, threads=1))):
    fn(*slices[0])
    t0 = time.perf_counter()
    for r0, r1 in slices:
        fn(r0, r1)
    dt = time.perf_counter() - t0
    out[name] = {"seconds": dt, "evals_per_s_1thread": n * out["vertices"] / dt}
out["port_over_reference_time"] = (out["numpy port (oracle/numpy_scan.py)"]["seconds"]
                                   / out["reference _scan_rank_range"]["seconds"])
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/r02_cpu_port_calibration.json", "w"), indent=1)
print(json.dumps(out, indent=1))
