"""Goldens for the host generator and PGM I/O, produced by the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_synth.py

Writes ``tests/golden/synth_golden.json``: for a set of ``SyntheticSpec``s
(the shapes the reference's tests use — test_synth.py, test_detect.py,
test_hough.py — plus config-5-sized lines) the sha256 of the reference's
``gen_synthetic`` image and every ``GroundTruth`` field (pixel sets as
sha256 of their int64 (x, y) pairs); for a set of malformed PGM byte strings
the reference's ``read_pgm`` error message, and for spec errors the
``InvalidInputError`` message.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from lmsline import SyntheticSpec, gen_synthetic  # noqa: E402
from lmsline.pgm import read_pgm  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "synth_golden.json")

SPECS = [
    dict(width=256, height=256, slope=0.4, intercept=30.0, sampling_prob=0.5, noise_prob=0.001, seed=9),
    dict(width=1024, height=1024, slope=0.35, intercept=220.0, sampling_prob=0.5, noise_prob=0.002, seed=88),
    dict(width=1024, height=1024, endpoints=((100, 100), (900, 900)), sampling_prob=1.0, seed=1),
    dict(width=1024, height=1024, endpoints=((100, 900), (900, 100)), sampling_prob=1.0, seed=2),
    dict(width=512, height=512, endpoints=((300, 0), (310, 511)), sampling_prob=0.7, noise_prob=0.001, seed=5),
    dict(width=512, height=512, endpoints=((512 - 1, 5), (0, 7)), sampling_prob=0.9, seed=6),
    dict(width=300, height=200, endpoints=((10, 190), (10, 3)), sampling_prob=0.8, noise_prob=0.01, seed=7),
    dict(width=640, height=480, slope=0.0, intercept=240.0, sampling_prob=0.5, seed=3),
    dict(width=640, height=480, slope=2.5, intercept=-300.0, sampling_prob=0.5, seed=1),
    dict(width=640, height=480, slope=-0.7, intercept=400.0, sampling_prob=1.0, noise_prob=1.0, seed=2),
    dict(width=64, height=64, slope=-1e-7, intercept=63.0, sampling_prob=0.0, noise_prob=0.2, seed=4),
    dict(width=4096, height=4096, slope=-3.7, intercept=9000.0, sampling_prob=0.5, seed=17),
    dict(width=4096, height=4096, slope=0.21, intercept=1000.5, sampling_prob=0.5, noise_prob=0.05, seed=18),
]

BAD_SPECS = [
    dict(width=0, height=5, slope=1.0, intercept=0.0),
    dict(width=5, height=5, slope=1.0, intercept=0.0, sampling_prob=1.5),
    dict(width=5, height=5),
    dict(width=5, height=5, slope=1.0),
    dict(width=5, height=5, slope=float("inf"), intercept=0.0),
    dict(width=5, height=5, endpoints=((0, 0), (1, 1)), slope=1.0, intercept=0.0),
    dict(width=5, height=5, slope=0.0, intercept=9.0),
    dict(width=5, height=5, slope=1.0, intercept=100.0),
    dict(width=5, height=5, endpoints=((0, 0), (5, 1))),
    dict(width=5, height=5, endpoints=((2, 2), (2, 2))),
]

BAD_PGM = [
    b"", b"P2\n2 2\n255\n\x00\x00\x00\x00", b"P5\n2", b"P5\nx 2\n255\n", b"P5\n2 2\n0\n",
    b"P5\n2 2\n256\n", b"P5\n0 2\n255\n", b"P5\n2 2\n255", b"P5\n2 2\n255\n\x01\x02\x03",
    b"P5 # comment\n2 2\n255\n", b"P5\n#only comment", b"P5\n2 2 255\n\x00\x00\x00\x00",
]
GOOD_PGM = [b"P5\n# made by hand\n3 2\n200\n\x01\x02\x03\x04\x05\x06", b"P5 1 1 7\t\x09",
            b"P5\r\n2\t1\r\n255\r\xff\x00extra"]


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def pix(pixels) -> str:
    return sha(np.array(pixels, dtype=np.int64).reshape(-1, 2))


def main():
    out = {"generator": "tests/golden/make_golden_synth.py", "specs": [], "bad_specs": [], "pgm": []}
    for kw in SPECS:
        img, t = gen_synthetic(SyntheticSpec(**kw))
        out["specs"].append({
            "spec": {k: v for k, v in kw.items()},
            "image_sha256": sha(img), "lit": int((img == 255).sum()),
            "slope": repr(t.slope), "intercept": repr(t.intercept), "rho": repr(t.rho), "theta": repr(t.theta),
            "endpoints": t.endpoints, "raster_length": t.raster_length,
            "line_pixels": [len(t.line_pixels), pix(t.line_pixels)],
            "noise_pixels": [len(t.noise_pixels), pix(t.noise_pixels)], "seed": t.seed,
        })
    for kw in BAD_SPECS:
        try:
            sp = SyntheticSpec(**kw)
            gen_synthetic(sp)
            msg = None
        except ValueError as e:
            msg = [type(e).__name__, str(e)]
        out["bad_specs"].append({"spec": {k: (repr(v) if isinstance(v, float) else v) for k, v in kw.items()},
                                 "error": msg})
    with tempfile.TemporaryDirectory() as d:
        for data in BAD_PGM + GOOD_PGM:
            p = os.path.join(d, "x.pgm")
            with open(p, "wb") as fh:
                fh.write(data)
            try:
                arr = read_pgm(p)
                res = {"shape": list(arr.shape), "sha256": sha(arr)}
            except ValueError as e:
                res = {"error": [type(e).__name__, str(e)]}
            out["pgm"].append({"bytes": data.hex(), **res})
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=0)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
