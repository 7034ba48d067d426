"""Dev: phases of the device detect_lines path (config-5 image)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1510_01041_b200 as lms  # noqa: E402
from paper_1510_01041_b200 import _native, workloads  # noqa: E402

img = workloads.config5_image(0)
p = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
c, s = p.vote_trig()
nt = p.n_theta
strig = [p.support_trig(t) for t in range(nt)]
swap_t = [lms.needs_axis_swap(p.theta_center(t)) for t in range(nt)]
for _ in range(3):
    lms.detect_lines(img, p, "lms", 64)
T = {}
reps = 10
for _ in range(reps):
    t0 = time.perf_counter()
    npts, pk, _ = _native.detect_peaks(img, 128, c, s, p.rho_max, p.delta_rho, p.n_rho, 64, 2)
    t1 = time.perf_counter()
    votes = pk[:, 2]
    n_fit = np.minimum(votes, 256)
    res = _native.detect_supports([a for a, _ in strig], [b for _, b in strig], swap_t, 256, n_fit // 2 + 1,
                                  True, pk.shape[0], votes)
    t2 = time.perf_counter()
    T["peaks"] = T.get("peaks", 0) + (t1 - t0) * 1e3
    T["supports+fits"] = T.get("supports+fits", 0) + (t2 - t1) * 1e3
for k, v in T.items():
    print(f"{v / reps:8.3f} ms {k}")
t = time.perf_counter()
for _ in range(reps):
    lms.detect_lines(img, p, "lms", 64)
print(f"{(time.perf_counter() - t) / reps * 1e3:8.3f} ms detect_lines")
