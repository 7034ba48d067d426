"""Golden vectors for the Hough / detect_lines path, produced by the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_hough.py

Writes ``tests/golden/hough_golden.json.gz``: synthetic images from the
reference's own generator (stored as their lit-pixel indices; the images are
binary 0/255), the reference's accumulator (non-zero bins), peaks, supports
(as ordinals into extract_points order) and detect_lines results for the
three methods.  Floats are ``float.hex``.  Mirrors test_hough.py /
test_detect.py / test_acceptance.py:268-274 fixtures.
"""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lmsline import (  # noqa: E402
    HoughParams,
    SyntheticSpec,
    detect_lines,
    extract_points,
    find_peaks,
    gen_synthetic,
    hough_vote,
    refine_lms,
    supporting_points,
)
from lmsline.hough import needs_axis_swap  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "hough_golden.json.gz")


def hx(v):
    return None if v is None else float(v).hex()


def combine(specs):
    img = None
    for sp in specs:
        im, _ = gen_synthetic(sp)
        img = im if img is None else np.maximum(img, im)
    return img


def record(name, img, params, max_peaks, min_votes=2, q=None, support_cap=256, salt=None):
    if salt is not None:
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([salt[0], 1])))
        img = img.copy()
        img[rng.random(img.shape) < salt[1]] = 255
    pts = extract_points(img)
    acc = hough_vote(pts, params)
    peaks = find_peaks(acc, max_peaks, min_votes)
    index = {(p.x, p.y): k for k, p in enumerate(pts)}
    supports = []
    for pk in peaks:
        sup = supporting_points(pts, pk, params)
        supports.append([index[(p.x, p.y)] for p in sup])
    rs, ts = np.nonzero(acc.bins)
    dets = {}
    for method in ("lms", "ols", "sht"):
        try:
            ds = detect_lines(img, params, method, max_peaks, min_votes=min_votes, q=q,
                              support_cap=support_cap)
            dets[method] = [{
                "rho": hx(d.rho), "theta": hx(d.theta), "slope": hx(d.slope),
                "intercept": hx(d.intercept), "axis_swapped": d.axis_swapped,
                "lms_value": hx(d.lms_value), "support_len": len(d.support)} for d in ds]
        except ValueError as e:  # degenerate support etc.
            dets[method] = {"error": type(e).__name__}
    refits = []
    for pk, sup in zip(peaks, supports):
        if len(sup) >= 3:
            try:
                f = refine_lms([pts[k] for k in sup], None, needs_axis_swap(pk.theta), support_cap=64)
                refits.append({"slope": hx(f.line.slope), "intercept": hx(f.line.intercept),
                               "lms_value": hx(f.lms_value)})
            except ValueError as e:
                refits.append({"error": type(e).__name__})
        else:
            refits.append(None)
    return {
        "name": name, "height": img.shape[0], "width": img.shape[1],
        "lit": np.flatnonzero(img >= 128).tolist(),
        "params": [hx(params.delta_rho), hx(params.delta_theta), hx(params.rho_max)],
        "max_peaks": max_peaks, "min_votes": min_votes, "q": q, "support_cap": support_cap,
        "bins": [[int(r), int(t), int(acc.bins[r, t])] for r, t in zip(rs, ts)],
        "peaks": [[p.rho_bin, p.theta_bin, p.votes, hx(p.rho), hx(p.theta)] for p in peaks],
        "supports": supports, "detect": dets, "refits": refits,
    }


def main():
    cases = []
    sp = SyntheticSpec(width=256, height=256, slope=0.4, intercept=30.0, sampling_prob=0.5,
                       noise_prob=0.001, seed=9)
    cases.append(record("single_256", combine([sp]), HoughParams.for_image(256, 256, 8.0, 10.0), 3))
    sp = SyntheticSpec(slope=0.35, intercept=220.0, sampling_prob=0.5, noise_prob=0.002, seed=88)
    cases.append(record("accept8_1024", combine([sp]), HoughParams.for_image(1024, 1024, 20.0, 20.0), 1))
    cross = [SyntheticSpec(width=512, height=512, slope=0.5, intercept=40.0, sampling_prob=0.6, seed=3),
             SyntheticSpec(width=512, height=512, slope=-1.3, intercept=600.0, sampling_prob=0.6, seed=4)]
    cases.append(record("crossing_512", combine(cross), HoughParams.for_image(512, 512, 10.0, 5.0), 6))
    steep = SyntheticSpec(width=512, height=512, endpoints=((300, 0), (310, 511)), sampling_prob=0.7,
                          noise_prob=0.001, seed=5)
    cases.append(record("steep_512", combine([steep]), HoughParams.for_image(512, 512, 6.0, 4.0), 4))
    multi = [SyntheticSpec(width=640, height=480, slope=s, intercept=c, sampling_prob=0.5, seed=k)
             for k, (s, c) in enumerate([(0.1, 50.0), (2.5, -300.0), (-0.7, 400.0), (0.0, 240.0)])]
    cases.append(record("multi_640x480_salt", combine(multi), HoughParams.for_image(640, 480, 12.0, 6.0),
                        12, salt=(21, 0.01)))
    cases.append(record("salt_q_cap", combine(multi[:2]), HoughParams.for_image(640, 480, 20.0, 20.0),
                        5, q=40, support_cap=100, salt=(22, 0.03)))
    doc = {"generator": "tests/golden/make_golden_hough.py", "cases": cases}
    with gzip.open(OUT, "wt") as fh:
        json.dump(doc, fh)
    print(f"wrote {OUT}: {len(cases)} images")
    for c in cases:
        print(c["name"], len(c["lit"]), "lit;", len(c["peaks"]), "peaks;",
              [len(s) for s in c["supports"]])


if __name__ == "__main__":
    main()
