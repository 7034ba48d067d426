"""Dev helper: time detect_lines on config 5 (4096^2, 64 lines, 30% salt)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.')
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import _native, workloads

img = workloads.line_image(4096, 4096, 64, 0.30, seed=0)
p = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
for r in range(3):
    t0 = time.perf_counter()
    dets = lms.detect_lines(img, p, "lms", 64)
    t1 = time.perf_counter()
    c, s = p.vote_trig()
    t2 = time.perf_counter()
    bins, npts = _native.hough_vote_image(img, 128, c, s, p.rho_max, p.delta_rho, p.n_rho)
    t3 = time.perf_counter()
    print(json.dumps({"detect_s": t1 - t0, "vote_s": t3 - t2, "npts": npts, "peaks": len(dets),
                      "support_sizes": [len(d.support) for d in dets[:5]],
                      "slopes": [d.slope for d in dets[:3]]}), flush=True)
