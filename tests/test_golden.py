"""Golden fixtures (tests/golden/*.json, each entry cited) reproduced by the oracle."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as o

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("case", G["x_pairs"], ids=lambda c: c["cite"])
def test_x_pairs(case):
    Q = np.cumsum(np.asarray(case["q"], np.uint64)).astype(np.uint64)
    n, W = len(Q), case["W"]
    b1 = np.empty(n, np.int32)
    b2 = np.empty(n, np.int32)
    o.lib().or_bins(n, o._p(Q), W, o._p(b1), o._p(b2))
    assert [list(p) for p in zip(b1.tolist(), b2.tolist())] == case["spans"]


@pytest.mark.parametrize("case", G["importance"], ids=lambda c: c["cite"])
def test_importance(case):
    assert o.importance(case["V"], case["maxV"], case["L"], case["P"], case["eps"]) == np.float32(case["f"])


@pytest.mark.parametrize("case", G["sample"], ids=lambda c: c["cite"])
def test_sample(case):
    assert o.sample(case["alpha"], case["t"]) == case["a"]


@pytest.mark.parametrize("case", G["index_range"], ids=lambda c: c["cite"])
def test_index_range(case):
    inv = o.domain_inv(case["lo"], case["hi"])
    assert list(o.index_range(case["vmin"], case["vmax"], case["lo"], inv, case["N"])) == case["ij"]


@pytest.mark.parametrize("case", G["hilbert"], ids=lambda c: f'{c["cite"]}-{c["b"]}')
def test_hilbert(case):
    assert int(o.hilbert_encode([case["xyz"]], case["b"])[0]) == case["h"]


def test_hilbert_vectors_reproduced_by_independent_generator():
    """The committed Hilbert vectors are exactly what tests/golden/gen_hilbert.py computes
    from Skilling's decoder alone (no oracle code), so they are reproducible."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "gen_hilbert", os.path.join(os.path.dirname(__file__), "golden", "gen_hilbert.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    assert gen.generate() == G["hilbert"]
