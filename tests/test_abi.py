"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/dvl.h declares, and its host-evaluated Hilbert state machine (the tables the GPU
kernel uses) reproduces the oracle's Skilling curve exactly."""
import re
import os

import numpy as np
import pytest

from oracle import oracle as o
import paper_2306_11612_b200 as dvl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "dvl.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dvl_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = dvl.load()
    declared = header_symbols()
    assert declared, "no declarations parsed"
    for s in declared:
        assert hasattr(L, s), s
    assert sorted(dvl.SYMBOLS) == declared


def test_status_strings():
    L = dvl.load()
    assert L.dvl_status_string(0) == b"DVL_OK"
    assert L.dvl_status_string(4) == b"DVL_E_OVERLAP"


def test_state_machine_size():
    # signed permutations of 3 axes x Gray-parity bit, reachable subset
    n = dvl.hilbert_states()
    assert 1 < n <= 96


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5])
def test_host_encoder_exhaustive(b):
    r = np.arange(1 << b, dtype=np.uint32)
    x, y, z = np.meshgrid(r, r, r, indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    assert np.array_equal(dvl.hilbert_encode_host(pts, b), o.hilbert_encode(pts, b))


@pytest.mark.parametrize("b", list(range(6, 22)))
def test_host_encoder_random(b):
    rng = np.random.default_rng(b)
    pts = rng.integers(0, 1 << b, size=(20000, 3), dtype=np.uint32)
    assert np.array_equal(dvl.hilbert_encode_host(pts, b), o.hilbert_encode(pts, b))


def test_host_encoder_rejects_bad_input():
    with pytest.raises(dvl.DvlError):
        dvl.hilbert_encode_host([[4, 0, 0]], 2)
    with pytest.raises(dvl.DvlError):
        dvl.hilbert_encode_host([[0, 0, 0]], 22)
