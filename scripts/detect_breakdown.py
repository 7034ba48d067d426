"""Dev: wall-clock phases of detect_lines on the config-5 image (GPU)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1510_01041_b200 as lms  # noqa: E402
from paper_1510_01041_b200 import _native, workloads  # noqa: E402
from paper_1510_01041_b200 import detect as D  # noqa: E402

img = workloads.config5_image(0)
p = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
for _ in range(3):
    lms.detect_lines(img, p, "lms", 64)
T = {}


def tick(name, t0):
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return time.perf_counter()


reps = 10
for _ in range(reps):
    t = time.perf_counter()
    im, thr = lms.hough.lit_mask_u8(img, 128)
    c, s = p.vote_trig()
    t = tick("prep", t)
    bins, npts = _native.hough_vote_image(im, thr, c, s, p.rho_max, p.delta_rho, p.n_rho)
    t = tick("vote_image (upload+extract+vote+acc D2H)", t)
    peaks = lms.find_peaks(lms.HoughAccumulator(bins=bins, params=p), 64, 2)
    t = tick("find_peaks host", t)
    trig = [p.support_trig(k.theta_bin) for k in peaks]
    offsets, ids = _native.hough_support([a for a, _ in trig], [b for _, b in trig], [k.rho_bin for k in peaks],
                                         p.rho_max, p.delta_rho, p.n_rho, capacity=sum(k.votes for k in peaks),
                                         narrow=True)
    t = tick("support (gather + ids D2H)", t)
    sups = [D.SupportPoints.from_pixels(ids[offsets[k]:offsets[k + 1]], 4096) for k in range(len(peaks))]
    swapped = [lms.needs_axis_swap(k.theta) for k in peaks]
    picks = [sp._ids if sp._ids.size <= 256 else sp._ids[D._subsample_index(sp._ids.size, 256)] for sp in sups]
    counts = np.array([x.size for x in picks])
    offs = np.zeros(len(picks) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(counts)
    row, col = np.divmod(np.concatenate(picks), 4096)
    sw = np.repeat(np.array(swapped), counts)
    T_ = np.where(sw, row, col).astype(float)
    Z_ = np.where(sw, col, row).astype(float)
    t = tick("host subsample+design", t)
    fits = lms.solver._solve_concat(T_, Z_, offs, None)
    t = tick("batched LMS (upload+solve+tail)", t)
    out = []
    for k, (pk, sp, s_) in enumerate(zip(peaks, sups, swapped)):
        f = fits[k]
        rho, th = lms.line_to_polar(f.line.slope, f.line.intercept, s_)
        out.append(D.LineDetection(method="lms", rho=rho, theta=th, slope=f.line.slope, intercept=f.line.intercept,
                                   axis_swapped=s_, support=sp, lms_value=f.lms_value))
    t = tick("LineDetection objects", t)
tot = 0
for k, v in T.items():
    print(f"{v / reps:8.3f} ms  {k}")
    tot += v / reps
print(f"{tot:8.3f} ms  total")
t = time.perf_counter()
for _ in range(reps):
    lms.detect_lines(img, p, "lms", 64)
print(f"{(time.perf_counter() - t) / reps * 1e3:8.3f} ms  detect_lines")
