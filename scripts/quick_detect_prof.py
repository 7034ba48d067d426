"""Dev helper: stage times of detect_lines on config 5 (wall clock)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1510_01041_b200 as lms
from paper_1510_01041_b200 import _native, workloads, detect, hough, solver

img = workloads.line_image(4096, 4096, 64, 0.30, seed=0)
params = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
for rep in range(3):
    T = {}
    t0 = time.perf_counter()
    m, thr = hough.lit_mask_u8(img, 128); T["mask"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    c, s = params.vote_trig()
    bins, npts = _native.hough_vote_image(m, thr, c, s, params.rho_max, params.delta_rho, params.n_rho)
    T["vote"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    peaks = hough.find_peaks(hough.HoughAccumulator(bins=bins, params=params), 64, 2); T["peaks"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    trig = [params.support_trig(p.theta_bin) for p in peaks]
    offsets, ids = _native.hough_support([t[0] for t in trig], [t[1] for t in trig], [p.rho_bin for p in peaks],
                                         params.rho_max, params.delta_rho, params.n_rho, capacity=sum(p.votes for p in peaks))
    T["support"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sups = [detect.SupportPoints.from_pixels(ids[offsets[k]:offsets[k + 1]], 4096) for k in range(len(peaks))]
    designs = []
    for sup, p in zip(sups, peaks):
        t, z = detect._design_xy(*detect._thinned_xy(sup, 256), hough.needs_axis_swap(p.theta))
        designs.append(np.column_stack([t, z]))
    T["designs"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    fits = solver.solve_lms_batch(designs, None); T["lms_batch"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dets = lms.detect_lines(img, params, "lms", 64); T["detect_total"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in T.items()}, flush=True)
