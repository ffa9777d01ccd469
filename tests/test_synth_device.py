"""The device variant of the input recipe (synth/device.py) gives the numpy generator's
bits (evaluated here with torch on the CPU): same cells, levels, order and scalars."""
import numpy as np
import pytest
import torch

import synth
from synth import device as sd


@pytest.mark.parametrize("name,kw", [("C1", dict(scale_E=16)), ("C2", dict(scale_E=64)),
                                     ("C5", dict(box=(3, 2, 2))), ("C4", dict(scale_E=12))])
def test_device_recipe_matches_numpy(name, kw):
    a = synth.make_config(name, **kw)
    b = sd.make_config(name, device="cpu", **kw)
    assert np.array_equal(b["lower"].numpy().astype(np.uint32), a["lower"])
    assert np.array_equal(b["level"].numpy(), a["level"])
    assert np.array_equal(b["scal"].numpy().view(np.uint32), a["scal"].view(np.uint32))
    assert np.array_equal(b["domain"], a["domain"])
    assert b["E"] == a["E"] and b["W"] == a["W"]


def test_hash_matches_numpy():
    keys = np.array([0, 1, 2 ** 63 - 1, 12345678901234, 2 ** 62 + 17], np.uint64)
    for seed in (0, 2306, 11612 + 3):
        a = synth.hash_uniform(keys, seed)
        b = sd.hash_uniform(torch.from_numpy(keys.view(np.int64)), seed).numpy()
        assert np.array_equal(a, b)
