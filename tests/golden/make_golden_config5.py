"""Config-5 golden: the REFERENCE's detect_lines on the BASELINE config-5 image.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_config5.py

The image is ``workloads.config5_image(0)`` (4096 x 4096, 64 lines, 30 %
salt) rendered with the reference's own ``gen_synthetic``
(/root/reference/pkg/src/lmsline/synth.py:132-191); its sha256 must equal the
one this package's ``synth.render`` produces (pinning the generator port).
Then the reference's ``detect_lines(image, HoughParams.for_image(4096, 4096,
20, 20), "lms", 64, support_cap=C)`` (detect.py:156-214) for C = 256 and 512
(~100 s each).  Recorded: the non-zero accumulator bins, the peaks, and per
detection every field (floats as ``float.hex``) plus the support's length
and the sha256 of its (x, y) int32 pairs in order.  Written to
``tests/golden/config5_golden.json.gz``; the GPU test regenerates the image
with this package's generator and compares.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import lmsline  # noqa: E402
from lmsline import HoughParams, detect_lines, extract_points, find_peaks, hough_vote  # noqa: E402

from paper_1510_01041_b200 import workloads  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "config5_golden.json.gz")


def hx(v):
    return float(v).hex()


def support_digest(support) -> str:
    arr = np.array([(p.x, p.y) for p in support], dtype=np.int32).reshape(-1, 2)
    return hashlib.sha256(arr.tobytes()).hexdigest()


def ref_render(spec):
    ref_spec = lmsline.SyntheticSpec(width=spec.width, height=spec.height, slope=spec.slope,
                                     intercept=spec.intercept, sampling_prob=spec.sampling_prob,
                                     noise_prob=spec.noise_prob, seed=spec.seed)
    return lmsline.gen_synthetic(ref_spec)[0]


def main():
    t0 = time.perf_counter()
    img = workloads.config5_image(0, render=ref_render)
    mine = workloads.config5_image(0)
    digest = hashlib.sha256(img.tobytes()).hexdigest()
    assert digest == hashlib.sha256(mine.tobytes()).hexdigest(), "synth port differs from the reference"
    t_img = time.perf_counter() - t0
    params = HoughParams.for_image(4096, 4096, 20.0, 20.0)
    t0 = time.perf_counter()
    pts = extract_points(img)
    acc = hough_vote(pts, params)
    peaks = find_peaks(acc, 64, 2)
    t_vote = time.perf_counter() - t0
    rs, ts = np.nonzero(acc.bins)
    doc = {
        "generator": "tests/golden/make_golden_config5.py",
        "image": "paper_1510_01041_b200.workloads.config5_image(0)",
        "image_sha256": digest, "lit": len(pts),
        "params": [hx(params.delta_rho), hx(params.delta_theta), hx(params.rho_max)],
        "bins": [[int(r), int(t), int(acc.bins[r, t])] for r, t in zip(rs, ts)],
        "peaks": [[p.rho_bin, p.theta_bin, p.votes, hx(p.rho), hx(p.theta)] for p in peaks],
        "seconds": {"image": t_img, "extract_vote_peaks": t_vote},
        "detect": {},
    }
    for cap in (256, 512):
        t0 = time.perf_counter()
        dets = detect_lines(img, params, "lms", 64, support_cap=cap)
        doc["seconds"][f"detect_lines_cap{cap}"] = time.perf_counter() - t0
        doc["detect"][str(cap)] = [{
            "rho": hx(d.rho), "theta": hx(d.theta), "slope": hx(d.slope), "intercept": hx(d.intercept),
            "axis_swapped": d.axis_swapped, "lms_value": hx(d.lms_value), "method": d.method,
            "support_len": len(d.support), "support_sha256": support_digest(d.support),
        } for d in dets]
        print(f"cap {cap}: {len(dets)} detections in {doc['seconds'][f'detect_lines_cap{cap}']:.1f}s", flush=True)
    with gzip.open(OUT, "wt") as fh:
        json.dump(doc, fh)
    print(f"wrote {OUT}: {len(peaks)} peaks, {len(pts)} lit; {doc['seconds']}")


if __name__ == "__main__":
    main()
