"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/lms_b200.h declares (no compute calls here)."""

import os
import re
import subprocess

import pytest

from paper_1510_01041_b200 import _native
from paper_1510_01041_b200._build import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", fn)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"^\s*(?:int|const char\*)\s+(lms_\w+)\s*\(", text, flags=re.M))
    return names


def test_library_exists_and_loads():
    assert os.path.exists(LIB_PATH)
    lib = _native.load_library()
    assert lib.lms_version() >= 1


def test_every_declared_symbol_is_exported_and_bound():
    names = declared_symbols()
    assert len(names) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = names - exported
    assert not missing, missing
    assert names <= set(_native.SIGNATURES), names - set(_native.SIGNATURES)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_device_count_is_callable_without_gpu():
    assert _native.device_count() >= 0


def test_no_device_raises_loudly(monkeypatch):
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    import numpy as np

    from paper_1510_01041_b200 import solve_lms

    with pytest.raises(_native.NativeUnavailableError):
        solve_lms(np.random.default_rng(0).normal(0, 1, (10, 2)))
