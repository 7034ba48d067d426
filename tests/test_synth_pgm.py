"""Host generator and PGM I/O (synth.py, pgm.py) against goldens produced by
the reference's own ``gen_synthetic`` / ``read_pgm``
(tests/golden/make_golden_synth.py), and the config-5 image digest that the
config-5 golden records (tests/golden/make_golden_config5.py)."""

import gzip
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1510_01041_b200 import pgm, synth, workloads
from paper_1510_01041_b200.geometry import InvalidInputError

HERE = os.path.join(os.path.dirname(__file__), "golden")
GOLD = json.load(open(os.path.join(HERE, "synth_golden.json")))


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def pix(pixels):
    return sha(np.array(pixels, dtype=np.int64).reshape(-1, 2))


def _spec(d):
    kw = dict(d)
    if "endpoints" in kw:
        kw["endpoints"] = tuple(tuple(p) for p in kw["endpoints"])
    for k in ("slope", "intercept", "sampling_prob", "noise_prob"):
        if isinstance(kw.get(k), str):
            kw[k] = float(kw[k])
    return synth.SyntheticSpec(**kw)


@pytest.mark.parametrize("case", GOLD["specs"], ids=lambda c: str(c["spec"].get("seed")))
def test_gen_synthetic_matches_reference(case):
    img, t = synth.gen_synthetic(_spec(case["spec"]))
    assert img.dtype == np.uint8 and sha(img) == case["image_sha256"]
    assert int((img == 255).sum()) == case["lit"]
    assert (repr(t.slope), repr(t.intercept), repr(t.rho), repr(t.theta)) == \
        (case["slope"], case["intercept"], case["rho"], case["theta"])
    assert [list(p) for p in t.endpoints] == case["endpoints"]
    assert t.raster_length == case["raster_length"] and t.seed == case["seed"]
    assert [len(t.line_pixels), pix(t.line_pixels)] == case["line_pixels"]
    assert [len(t.noise_pixels), pix(t.noise_pixels)] == case["noise_pixels"]
    # deterministic; render() is the same image without the tuples
    assert sha(synth.render(_spec(case["spec"]))[0]) == case["image_sha256"]


@pytest.mark.parametrize("case", GOLD["bad_specs"], ids=lambda c: c["error"][1][:20])
def test_spec_errors_match_reference(case):
    with pytest.raises(InvalidInputError) as ei:
        synth.gen_synthetic(_spec(case["spec"]))
    assert str(ei.value) == case["error"][1]


def test_bresenham_octants_and_ends():
    for (x0, y0, x1, y1) in [(0, 0, 5, 2), (5, 2, 0, 0), (0, 0, 2, 5), (3, -4, -6, 1), (1, 1, 1, 1), (0, 0, -3, 0)]:
        cells = synth.bresenham(x0, y0, x1, y1)
        assert cells[0] == (x0, y0) and cells[-1] == (x1, y1)
        assert len(cells) == max(abs(x1 - x0), abs(y1 - y0)) + 1
        steps = np.diff(np.array(cells), axis=0)
        assert np.all(np.abs(steps) <= 1)


@pytest.mark.parametrize("case", GOLD["pgm"], ids=lambda c: c["bytes"][:16] or "empty")
def test_read_pgm_matches_reference(case, tmp_path):
    p = tmp_path / "x.pgm"
    p.write_bytes(bytes.fromhex(case["bytes"]))
    if "error" in case:
        with pytest.raises(pgm.PgmParseError) as ei:
            pgm.read_pgm(p)
        assert str(ei.value) == case["error"][1]
        assert isinstance(ei.value, ValueError)
    else:
        arr = pgm.read_pgm(p)
        assert list(arr.shape) == case["shape"] and sha(arr) == case["sha256"]


def test_pgm_round_trip_and_writer_errors(tmp_path):
    img = (np.arange(35, dtype=np.uint8) * 7).reshape(5, 7)
    a, b = tmp_path / "a.pgm", tmp_path / "b.pgm"
    pgm.write_pgm(a, img)
    assert a.read_bytes()[:11] == b"P5\n7 5\n255\n"
    back = pgm.read_pgm(a)
    assert np.array_equal(back, img)
    pgm.write_pgm(b, back)
    assert a.read_bytes() == b.read_bytes()
    with pytest.raises(InvalidInputError):
        pgm.write_pgm(a, img.astype(np.int16))
    with pytest.raises(InvalidInputError):
        pgm.write_pgm(a, img.ravel())


def test_config5_image_is_the_golden_image():
    path = os.path.join(HERE, "config5_golden.json.gz")
    if not os.path.exists(path):
        pytest.skip("config-5 golden not generated")
    with gzip.open(path, "rt") as fh:
        doc = json.load(fh)
    img = workloads.config5_image(0)
    assert sha(img) == doc["image_sha256"]
    assert int((img >= 128).sum()) == doc["lit"]


def test_ground_truth_sidecar_round_trip_and_reference_format(tmp_path):
    _, t = synth.gen_synthetic(synth.SyntheticSpec(width=64, height=48, slope=0.3, intercept=5.0,
                                                   noise_prob=0.01, seed=3))
    p = tmp_path / "t.csv"
    synth.write_ground_truth(p, t)
    text = p.read_bytes()
    assert text.startswith(b"# slope=0.3 intercept=5.0\n# rho=")
    assert b"kind,x,y\r\n" in text  # csv.writer's line terminator, as the reference writes it
    assert synth.read_ground_truth(p) == t
    p.write_text("# slope=1.0\nkind,x,y\n")
    with pytest.raises(InvalidInputError):
        synth.read_ground_truth(p)
    p.write_text("# slope=1.0 intercept=0.0\n# rho=0.0 theta=45.0\n# endpoints=0,0,1,1 raster_length=2\n"
                 "# seed=0\nkind,x,y\nfoo,1,2\n")
    with pytest.raises(InvalidInputError):
        synth.read_ground_truth(p)
